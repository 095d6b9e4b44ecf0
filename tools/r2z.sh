cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine_fidelity.py tests/test_gpu_shard.py -q > gpurun_out/pytest_r2z.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2z.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2z.json 2> gpurun_out/bench_r2z.err
timeout 900 python bench.py --no-cpu-baseline --steps 20 --data drift > gpurun_out/bench_r2z_drift.json 2> gpurun_out/bench_r2z_drift.err
