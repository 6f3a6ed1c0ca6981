# sweeps: cell-point gather ILP (cp2/cp8), fix-up gather ILP (fx2/fx8), u64 sort tile (rs12/rs20) vs head (CP 4, FIX 4, RS 16); GPU suite on head
mkdir -p gpurun_out
for v in head cp2 cp8 rs12 rs20 head; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
for v in head fx2 fx8 rs12 rs20 head; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; done
cp var/head.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
