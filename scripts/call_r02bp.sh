# C3 A/B: single-exit core-count and border walks (se1) vs HEAD; DBSCAN GPU tests on se1
mkdir -p gpurun_out
bash scripts/ab_c3.sh head se1 head se1
cp var/se1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_densebox.py tests/test_gpu_dbscan.py tests/test_gpu_sequential.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
