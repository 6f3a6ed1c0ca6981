mkdir -p gpurun_out
cp var/g3.so paper_2409_10743_b200/libspb200.so
timeout 200 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-220
timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_fix_gather|k_cell_points" -c 2 --csv python scripts/prof_build.py 134217728 1 2>/dev/null | grep -v "^==" | cut -d, -f5,12- | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_cell_points" -c 1 --csv python scripts/prof_fof.py 134217728 1 2>/dev/null | grep -v "^==" | cut -d, -f5,12- | tail -2
timeout 1500 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_densebox.py tests/test_gpu_dbscan.py -q -x 2>&1 | tail -2
