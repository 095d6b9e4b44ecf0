cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2aa.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2aa.log
timeout 900 python bench.py --workload c3 --policy host --data drift --no-cpu-baseline --steps 20 > gpurun_out/bench_r2aa_c3h.json 2> gpurun_out/bench_r2aa_c3h.err
