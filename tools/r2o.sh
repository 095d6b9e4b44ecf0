cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_attend -s 64 -c 1 \
  -o gpurun_out/ncu_r2o_score_attend python bench.py --profile-steps 4 --no-cpu-baseline > gpurun_out/ncu_r2o.log 2>&1
