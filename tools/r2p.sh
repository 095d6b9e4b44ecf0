cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py --layers 1 > gpurun_out/timeline_fused.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2q.json 2> gpurun_out/bench_r2q.err
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_configs.py -q -x > gpurun_out/pytest_r2q.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2q.log
