cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q > gpurun_out/pytest_prefill_r2j.log 2>&1; echo "exit $?" >> gpurun_out/pytest_prefill_r2j.log
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill_bench_r2j.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches_r2j.csv \
  python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu_launch_r2j.log 2>&1
for k in pf_gram pf_mat pf_solve; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
  -o gpurun_out/prefill_${k}_r2j python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu_${k}_r2j.log 2>&1
done
