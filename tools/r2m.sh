cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LRQK_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err
