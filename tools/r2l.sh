cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2l.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2l.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2l.json 2> gpurun_out/bench_r2l.err
LRQK_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2l_unfused.json 2> gpurun_out/bench_r2l_unfused.err
