cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2ai
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2ai/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2ai/pytest.log
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 30 "$@" > gpurun_out/r2ai/$name.json 2> gpurun_out/r2ai/$name.err; }
for f in 1 0 1 0; do
export LRQK_FUSED=$f
run c4_f${f}_$RANDOM
done
export LRQK_FUSED=1
run c3_f1 --workload c3
export LRQK_FUSED=0
run c3_f0 --workload c3
