cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > gpurun_out/timeline_fused.txt 2>&1
LRQK_FUSED=0 timeout 300 python tools/step_timeline.py --layers 1 > gpurun_out/timeline_unfused.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2x.json 2> gpurun_out/bench_r2x.err
LRQK_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2x_unfused.json 2> gpurun_out/bench_r2x_unfused.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2x.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2x.log
