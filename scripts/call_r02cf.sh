# fix-up chunk 1024 (fc): build A/B vs head, Bvh GPU tests (all three sort paths pinned to the oracle)
mkdir -p gpurun_out
for v in head fc head fc; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; done
cp var/fc.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_query.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
