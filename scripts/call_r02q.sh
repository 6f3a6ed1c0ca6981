# build on uniform and on the clustered field: windowed run fix-up (w32) vs the 63-bit sort (t64)
mkdir -p gpurun_out
for v in w32; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -3 | cut -c1-230; done
cp var/w32.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py tests/test_gpu_query.py -q -x 2>&1 | tail -2
