# A/B: query ordering with the top-32 sort (q32) vs 63-bit (q64; also the build's 63-bit path)
mkdir -p gpurun_out
for v in q64 q32 q64 q32; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c2_probe.py 16777216 3 | tail -1; timeout 300 python scripts/c4_probe.py 16777216 3 | tail -1; done
cp var/q32.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_query.py tests/test_gpu_scale.py tests/test_gpu_bvh.py -q -x 2>&1 | tail -2
