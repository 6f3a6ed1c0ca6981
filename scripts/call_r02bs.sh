# A/B: radix histogram copies (hc2, hc4) vs one (head); GPU tests on hc4
mkdir -p gpurun_out
for v in head hc2 hc4 head hc2 hc4; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-300; done
cp var/hc4.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_query.py -x -q 2>&1 | tail -2
