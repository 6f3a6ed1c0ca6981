# A/B: point-cell shortcut in the merge's leaf test (dg1) vs none (dg0)
mkdir -p gpurun_out
for v in dg0 dg1 dg0 dg1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/dg1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py -x -q 2>&1 | tail -2
