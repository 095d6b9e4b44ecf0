cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2e.json 2> gpurun_out/bench_ref_r2e.err
timeout 900 python bench.py --data recency --no-cpu-baseline > gpurun_out/bench_rec_r2e.json 2> gpurun_out/bench_rec_r2e.err
