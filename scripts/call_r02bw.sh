# A/B: radix digit counts fused into the key kernels (fh1) vs a separate counting pass (head); GPU suite on fh1
mkdir -p gpurun_out
for v in head fh1 head fh1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-300; done
cp var/fh1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
