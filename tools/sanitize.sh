#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on small shapes:
# the smoke (prefill factorisation + two decode steps, checked against the oracle),
# tools/smoke_small.py (each decode stage launched on its own) and
# tools/smoke_fused.py (the fused score/select/attend kernel with 4 parts per head).
# Usage (on the GPU box, repo root): bash tools/sanitize.sh TAG
tag=${1:-r2}
mkdir -p gpurun_out/sanitize_$tag
for tool in memcheck racecheck synccheck initcheck; do
  for name in smoke stages fused; do
    if [ $name = fused ]; then
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
        python tools/smoke_fused.py > gpurun_out/sanitize_$tag/${tool}_$name.log 2>&1
    elif [ $name = smoke ]; then
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
        python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tag/${tool}_$name.log 2>&1
    else
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
        python tools/smoke_small.py > gpurun_out/sanitize_$tag/${tool}_$name.log 2>&1
    fi
    echo "exit $?" >> gpurun_out/sanitize_$tag/${tool}_$name.log
  done
done
