# A/B: radix histogram with warp-merged adds and four sub-histograms (hg1) vs plain shared atomics (hg0); GPU tests on hg1
mkdir -p gpurun_out
for v in hg0 hg1 hg0 hg1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-300; done
cp var/hg1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_query.py -x -q 2>&1 | tail -2
