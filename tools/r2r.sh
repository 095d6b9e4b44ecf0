cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > gpurun_out/timeline_fused.txt 2>&1
