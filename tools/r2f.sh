cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2f.json 2> gpurun_out/bench_ref_r2f.err
timeout 900 python bench.py --data drift --no-cpu-baseline > gpurun_out/bench_drift_r2f.json 2> gpurun_out/bench_drift_r2f.err
timeout 900 python bench.py --workload c3 --policy host --data drift --no-cpu-baseline --steps 20 > gpurun_out/bench_c3h_drift_r2f.json 2> gpurun_out/bench_c3h_drift_r2f.err
