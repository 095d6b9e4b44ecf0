cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill_bench_r2i.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches_r2i.csv \
  python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu_launch_r2i.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pf_gram|pf_mat|pf_solve|pf_combine" -s 6 -c 4 \
  -o gpurun_out/prefill_full_r2i python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu_full_r2i.log 2>&1
