# A/B: merge with the leaf work queued per warp (q1) vs the plain walk (ld1); FoF GPU tests on q1
mkdir -p gpurun_out
for v in ld1 q1 ld1 q1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/q1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py tests/test_gpu_slabs.py -x -q 2>&1 | tail -2
