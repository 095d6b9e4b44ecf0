cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_r2k.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py -q > gpurun_out/pytest_prefill_r2k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_prefill_r2k.log
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill_bench_r2k.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2k.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_r2k.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2k.log
timeout 900 python bench.py > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err
