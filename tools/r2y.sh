cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2y.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2y.log
