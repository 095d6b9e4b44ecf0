cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2al
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_attend -s 96 -c 1 \
  -o gpurun_out/r2al/score_attend_full python bench.py --profile-steps 6 --no-cpu-baseline > gpurun_out/r2al/ncu_full.log 2>&1
