#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, the bench line (+ CPU
# baseline) and the reference arm, the other §8(d) configurations, the ncu
# launch list of the C4 step, one ncu --set full of the fused
# score/select/attend kernel, the prefill bench with its launch list and
# full captures, and the 1-layer phase timeline.
# Usage (repo root, on the GPU box): bash tools/gpu_round2.sh TAG
tag=${1:-r2}
o=gpurun_out/$tag
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/gpu.txt 2>&1
lscpu | head -20 >> $o/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke exit $?" >> $o/smoke.log
timeout 900 python bench.py > $o/bench_c4.json 2> $o/bench_c4.err
timeout 900 python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_reference.err
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 20 "$@" > $o/cfg_$name.json 2> $o/cfg_$name.err; }
run c1 --workload c1
run c2 --workload c2
run c3 --workload c3
run c3_host_drift --workload c3 --policy host --data drift
run c4_drift --data drift
run c4_recency --data recency
run c5_r16_k256 --rank 16 --topk 256
run c5_r32_k1024 --rank 32 --topk 1024
run c5_r64_k4096 --rank 64 --topk 4096
run c4_b2 --batch-per-gpu 2
run c4_b4 --batch-per-gpu 4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"score_attend|compress_kernel|select_kernel|attention_kernel|prepare_|advance_|score_tma|select_attend" \
  -c 600 --csv --log-file $o/launches_c4.csv python bench.py --profile-steps 6 --no-cpu-baseline > $o/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_attend -s 96 -c 1 \
  -o $o/score_attend_full python bench.py --profile-steps 6 --no-cpu-baseline > $o/ncu_full.log 2>&1
# the reports stay on the box (gpurun copies back <= 64 MiB): text summaries only
summ() { rep=$1; kern=$2; out=$3; ncu -i $rep.ncu-rep --page details > $out 2>&1; echo >> $out; \
  python tools/ncu_stalls.py $rep.ncu-rep $kern 40 >> $out 2>&1; \
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null; rm -f $rep.ncu-rep; }
summ $o/score_attend_full score_attend $o/score_attend_ncu_full.txt
timeout 300 python tools/prefill_bench.py > $o/prefill_c4.json 2>&1
timeout 300 python tools/prefill_bench.py --ctx 4096 --dtype f32 > $o/prefill_c1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"pf_" --csv --log-file $o/prefill_launches.csv python tools/prefill_bench.py --reps 1 > $o/ncu_prefill_launch.log 2>&1
for k in pf_gram pf_mat pf_solve; do  # -s 1: the timed call, after the warm-up call
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o $o/prefill_${k}_full python tools/prefill_bench.py --reps 1 > $o/ncu_prefill_$k.log 2>&1
  summ $o/prefill_${k}_full $k $o/prefill_${k}_ncu_full.txt
done
make trace -j8 > /dev/null 2>&1
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > $o/timeline_1layer.txt 2>&1
