# A/B: barrier-free block-local climb, global levels per first kernel 1/2/4/8
mkdir -p gpurun_out
for v in h1 h2 h4; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 200 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 60-400; done
cp var/h2.so paper_2409_10743_b200/libspb200.so; timeout 900 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
