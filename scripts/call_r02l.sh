# C5 extra-key failure, build breakdown (launch list + hierarchy ncu), CUB yardstick, C4 kNN
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/l_c5.json 2> gpurun_out/l_c5.err; echo "c5 rc=$?"; tail -1 gpurun_out/l_c5.json | cut -c1-600; tail -5 gpurun_out/l_c5.err
timeout 300 python scripts/build_probe.py
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/cub_sort_probe.cu -o /tmp/cub_sort_probe && /tmp/cub_sort_probe > gpurun_out/l_cub_sort.json; cat gpurun_out/l_cub_sort.json
timeout 300 python scripts/c4_probe.py 16777216 4 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_build_launches.csv python scripts/prof_build.py 134217728 2 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/l_build_launches.csv 2>/dev/null | head -14
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hierarchy -s 1 -c 1 -o gpurun_out/l_hier_pts -f python scripts/prof_build.py 134217728 2 > gpurun_out/l_hier.log 2>&1; tail -1 gpurun_out/l_hier.log
