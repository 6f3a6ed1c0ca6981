# C3 A/B: baseline (ld1), border walk with two 16-byte loads (bd1), + single-exit core-merge walk (cm1); GPU DBSCAN tests on cm1
mkdir -p gpurun_out
bash scripts/ab_c3.sh ld1 bd1 cm1 ld1 bd1 cm1
cp var/cm1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_densebox.py tests/test_gpu_dbscan.py tests/test_gpu_sequential.py -x -q 2>&1 | tail -2
