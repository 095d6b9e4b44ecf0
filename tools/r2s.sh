cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > gpurun_out/timeline_fused.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err
