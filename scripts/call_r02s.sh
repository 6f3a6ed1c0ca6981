# A/B: top tree levels staged in shared memory for the C2 range count (0 = off)
mkdir -p gpurun_out
for v in top0 top6 top9 top10 top0 top9; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c2_probe.py 16777216 4 | tail -2; done
cp var/top9.so paper_2409_10743_b200/libspb200.so; timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_scale.py -q -x -k "range or c2" 2>&1 | tail -1
cp var/top0.so paper_2409_10743_b200/libspb200.so
timeout 200 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-200
timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_bvh.py -q -x 2>&1 | tail -2
