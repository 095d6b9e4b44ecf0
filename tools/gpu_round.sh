#!/bin/bash
# One GPU session for the round's evidence: parity tests, smoke, the bench line
# (with the CPU baseline), the ncu launch list of the same command, and one
# ncu --set full capture of the dominant (score) kernel.
# Usage (from the repo root, on the GPU box): bash tools/gpu_round.sh TAG
tag=${1:-r1}
mkdir -p gpurun_out
make -j8 all trace >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$tag.txt 2>&1
lscpu | head -20 >> gpurun_out/gpu_$tag.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench exit $?" >> gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --profile-steps 5 > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launch exit $?" >> gpurun_out/ncu_launch_$tag.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^score_tma -s 160 -c 1 -o gpurun_out/score_$tag \
  python bench.py --profile-steps 6 > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full_$tag.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^select_attend -s 160 -c 1 -o gpurun_out/sa_$tag \
  python bench.py --profile-steps 6 > gpurun_out/ncu_full_sa_$tag.log 2>&1
timeout 300 python tools/step_timeline.py > gpurun_out/timeline_$tag.txt 2>&1
