# A/B: per-cell labels then a per-point gather (cl1) vs per-point double gather (cl0); both with first-point cell minima
mkdir -p gpurun_out
for v in cl0 cl1 cl0 cl1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/cl1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py tests/test_gpu_slabs.py -x -q 2>&1 | tail -2
