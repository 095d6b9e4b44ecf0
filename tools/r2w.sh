cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2w.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2w.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2w_$i.json 2> gpurun_out/bench_r2w.err
LRQK_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2w_unfused_$i.json 2> gpurun_out/bench_r2w_unfused.err
done
