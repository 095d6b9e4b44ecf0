cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export LRQK_PARITY_LOG=gpurun_out/parity_r2b
timeout 1200 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_decode.py -q -x -k "parity or step_locked or long_context or prefill_factors or sweep or mixed or fused_resident" > gpurun_out/pytest_r2b.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2b.log
