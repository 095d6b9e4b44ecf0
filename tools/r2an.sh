cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2an
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x -k "graph_conditional or engine_matches" > gpurun_out/r2an/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/r2an/pytest_quick.log
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 30 "$@" > gpurun_out/r2an/$name.json 2> gpurun_out/r2an/$name.err; }
run c4_a
run c4_b
export LRQK_FUSED=0
run c4_split
export LRQK_FUSED=1
timeout 300 python tools/step_timeline.py --layers 2 --fused-names > gpurun_out/r2an/timeline2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2an/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2an/pytest.log
