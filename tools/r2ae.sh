cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2ae.log 2>&1; echo "exit $?" >> gpurun_out/smoke_r2ae.log
timeout 300 python tools/smoke_fused.py > gpurun_out/fused_r2ae.log 2>&1; echo "exit $?" >> gpurun_out/fused_r2ae.log
bash tools/sanitize.sh r2ae
