cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2ao
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x -k "graph_replay_hands" > gpurun_out/r2ao/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/r2ao/pytest_quick.log
