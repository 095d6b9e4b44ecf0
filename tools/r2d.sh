cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sim.py -q -x > gpurun_out/pytest_r2d.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2d.log
