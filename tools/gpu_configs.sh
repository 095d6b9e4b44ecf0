#!/bin/bash
# Bench lines for the other SURVEY §8(d) configurations (evidence, not the
# headline): C1, C2, C3 (HBM and host slow tier), the C5 rank/top-k sweep
# points at 128K, and 2/4 sequences per GPU.  Usage: bash tools/gpu_configs.sh TAG
tag=${1:-cfg}
mkdir -p gpurun_out
make -j8 >/dev/null 2>&1
run() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --steps 20 "$@" > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err; }
run c1 --workload c1
run c2 --workload c2
run c3 --workload c3
run c3_host --workload c3 --policy host
run c4_r16_k256 --workload c4 --rank 16 --topk 256
run c4_r32_k1024 --workload c4 --rank 32 --topk 1024
run c4_r64_k4096 --workload c4 --rank 64 --topk 4096
run c4_b2 --workload c4 --batch-per-gpu 2
run c4_b4 --workload c4 --batch-per-gpu 4
