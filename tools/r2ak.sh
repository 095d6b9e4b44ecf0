cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2am
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 30 "$@" > gpurun_out/r2am/$name.json 2> gpurun_out/r2am/$name.err; }
for f in 1 0 1 0; do
export LRQK_FUSED=$f
run c4_f${f}_$RANDOM
done
export LRQK_FUSED=1
run c3_f1 --workload c3
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > gpurun_out/r2am/timeline.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_configs.py -q -x > gpurun_out/r2am/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2am/pytest.log
