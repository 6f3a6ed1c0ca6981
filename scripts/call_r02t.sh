# A/B: block-local climb hand-off through plain shared stores (m0), 64-bit atomics (m1), 128-bit exchanges (m2)
mkdir -p gpurun_out
for v in m0 m1 m2 m0 m2; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 200 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 60-300; done
cp var/m2.so paper_2409_10743_b200/libspb200.so
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_bvh.py tests/test_gpu_scale.py -q -x 2>&1 | tail -2
