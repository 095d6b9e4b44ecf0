cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export LRQK_PARITY_LOG=gpurun_out/parity_full
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
