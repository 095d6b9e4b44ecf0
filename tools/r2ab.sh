cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload c3 --policy host --data drift --no-cpu-baseline --steps 20 > gpurun_out/bench_r2ab_c3h.json 2> gpurun_out/bench_r2ab_c3h.err
git_stash=0
