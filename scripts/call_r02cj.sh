# sweeps: onesweep 128 threads (rt128), 2 global climb levels in the first kernel (cl2), 4 CTAs/SM for 32-bit passes (mb4) vs head
mkdir -p gpurun_out
for v in head rt128 cl2 mb4 head rt128 cl2 mb4; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 2 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-200; done
