cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q > gpurun_out/pytest_prefill_r2h.log 2>&1; echo "exit $?" >> gpurun_out/pytest_prefill_r2h.log
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill_bench_r2h.json 2>&1
timeout 300 python tools/prefill_bench.py --ctx 4096 --dtype f32 >> gpurun_out/prefill_bench_r2h.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2h.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2h.log
