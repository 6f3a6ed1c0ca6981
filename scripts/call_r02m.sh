# A/B: block-local climb hand-off (new, lv12, lv16) against the all-global climb (old)
mkdir -p gpurun_out
for v in new old g2 g4 g16; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 200 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1; done
for v in new g2; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== tests $v"; timeout 900 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2; done
