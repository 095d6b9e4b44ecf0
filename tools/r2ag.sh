cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2ag
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 20 "$@" > gpurun_out/r2ag/$name.json 2> gpurun_out/r2ag/$name.err; }
for f in 1 0; do
export LRQK_FUSED=$f
run c3_f$f --workload c3
run c4_b4_f$f --batch-per-gpu 4
run c5_r64_f$f --rank 64 --topk 4096
run c4_f$f
done
