# A/B: packet (warp-uniform) cell merge vs the per-lane walks
mkdir -p gpurun_out
for v in sm pk sm pk; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1; done
