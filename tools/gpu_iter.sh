#!/bin/bash
# Iteration run: GPU parity tests, per-kernel phase traces, a short bench, and an ncu capture.
# Usage: bash tools/gpu_iter.sh TAG [ncu-kernel-regex]
tag=${1:-it}; kre=${2:-}
mkdir -p gpurun_out
make -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$tag.log
for tr in compress score select attention prepare; do timeout 300 python tools/kernel_times.py --trace $tr > gpurun_out/kt_${tag}_$tr.txt 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
if [ -n "$kre" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 8 -c 4 \
    -o gpurun_out/ncu_$tag python tools/kernel_times.py --steps 3 > gpurun_out/ncu_$tag.log 2>&1
fi
