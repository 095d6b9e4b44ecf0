#!/bin/bash
# ncu --set full captures of single decode kernels (one launch each) from tools/kernel_times.py.
# Usage: bash tools/gpu_ncu.sh TAG kernel1 [kernel2 ...]
tag=$1; shift
mkdir -p gpurun_out
make -j8 >/dev/null 2>&1
for k in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 2 -c 1 \
    -o gpurun_out/ncu_${tag}_$k python tools/kernel_times.py --steps 3 > gpurun_out/ncu_${tag}_$k.log 2>&1
done
