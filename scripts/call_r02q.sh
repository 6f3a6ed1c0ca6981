# A/B: cell-tree leaf nodes written by k_cell_ranges (dnew) vs box array + hierarchy leaf writes (dold)
mkdir -p gpurun_out
for v in dold dnew dold dnew; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/dnew.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py tests/test_gpu_densebox.py tests/test_gpu_slabs.py tests/test_gpu_sequential.py -q -x 2>&1 | tail -2
