cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize_r2af
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/smoke_fused.py > gpurun_out/sanitize_r2af/racecheck_fused_fence.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_r2af/racecheck_fused_fence.log
