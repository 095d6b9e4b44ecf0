cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mb in 0 48 96 0 48 96; do
LRQK_PREFETCH_MB=$mb timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_r2ad_$mb.json 2> gpurun_out/bench_r2ad.err
python -c "import json;d=json.load(open('gpurun_out/bench_r2ad_$mb.json'));print($mb, d['value'], d['roofline']['avg_launch_ms'])" >> gpurun_out/r2ad.txt
done
