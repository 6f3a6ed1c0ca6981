# A/B: FoF labels kernel with 1 / 4 / 8 points per thread (lb1 / lb4 / lb8) vs HEAD; FoF GPU tests on lb4
mkdir -p gpurun_out
for v in head lb1 lb4 lb8 head lb4 lb8; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/lb4.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py tests/test_gpu_slabs.py -x -q 2>&1 | tail -2
