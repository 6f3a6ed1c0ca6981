# A/B: climb with carried split lengths (dnew) vs loaded (dold)
mkdir -p gpurun_out
for v in dold dnew dold dnew; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 60-300; done
cp var/dnew.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_sanitizer.py -q -x 2>&1 | tail -2
