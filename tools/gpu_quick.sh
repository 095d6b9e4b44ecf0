# quick GPU check used during development: decode parity tests + C4 bench x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_configs.py tests/test_gpu_api.py tests/test_gpu_errors.py -q -x > gpurun_out/quick/pytest.log 2>&1; echo "exit $?" >> gpurun_out/quick/pytest.log
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/quick/bench_$i.json 2> gpurun_out/quick/bench_$i.err; done
timeout 300 python tools/step_timeline.py --layers 1 --fused-names > gpurun_out/quick/timeline.txt 2>&1
