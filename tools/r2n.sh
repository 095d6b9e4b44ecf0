cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py --layers 1 > gpurun_out/timeline_fused.txt 2>&1
LRQK_FUSED=0 timeout 300 python tools/step_timeline.py --layers 1 > gpurun_out/timeline_unfused.txt 2>&1
