# A/B: Bvh::build with the top-32-bit sort + run fix-up (t32, t32b3) vs the 63-bit sort (t64)
mkdir -p gpurun_out
cp var/t32.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_query.py -q -x 2>&1 | tail -3
for v in t64 t32 t32b3 t64 t32; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 200 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-220; timeout 300 python scripts/c2_probe.py 16777216 3 | tail -1; done
