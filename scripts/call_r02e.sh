# A/B: reach cut-off on/off; launch list of the reach variant
mkdir -p gpurun_out
bash scripts/ab_var.sh noreach reach 2>&1 | tail -8
cp var/reach.so paper_2409_10743_b200/libspb200.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_reach.csv python scripts/prof_fof.py 134217728 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launch_reach.csv | head -12
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/cub_sort_probe.cu -o /tmp/cub_sort_probe && /tmp/cub_sort_probe > gpurun_out/cub_sort.json; cat gpurun_out/cub_sort.json
