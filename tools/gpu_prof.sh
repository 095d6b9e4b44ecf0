#!/bin/bash
# Per-kernel timings + phase traces + ncu --set full of the decode kernels at C4 (one layer).
tag=${1:-p}
mkdir -p gpurun_out
for tr in prepare compress select attention; do
  timeout 300 python tools/kernel_times.py --trace $tr > gpurun_out/kt_${tag}_$tr.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare|compress_kernel|select_kernel|attention_kernel" -s 8 -c 4 \
  -o gpurun_out/dec_$tag python tools/kernel_times.py --steps 3 > gpurun_out/ncu_dec_$tag.log 2>&1
echo done >> gpurun_out/ncu_dec_$tag.log
