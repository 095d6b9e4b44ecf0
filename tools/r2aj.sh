cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2aj
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2aj/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2aj/pytest.log
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 20 "$@" > gpurun_out/r2aj/$name.json 2> gpurun_out/r2aj/$name.err; }
run c3h --workload c3 --policy host --data drift
run c4
