cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export LRQK_PARITY_LOG=gpurun_out/parity_r2c
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_errors.py tests/test_gpu_api.py -q > gpurun_out/pytest_r2c.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2c.log
