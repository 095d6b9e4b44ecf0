cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:"attention_kernel|select_kernel|score_tma|compress_kernel|prepare_" -c 600 --csv --log-file gpurun_out/c3h_launches.csv python bench.py --workload c3 --policy host --data drift --profile-steps 4 --no-cpu-baseline > gpurun_out/c3h_ncu.log 2>&1
