cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_r2g.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2g.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2g.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_r2g.log
timeout 900 python bench.py > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err
bash tools/sanitize.sh r2g
