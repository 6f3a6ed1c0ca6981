# sweeps: 32-bit sort passes at 12 keys/thread (r32_12), fix-up chunk 1024/4096 (fc1k/fc4k), C3 Morton window 2/8 (cw2/cw8) vs head
mkdir -p gpurun_out
for v in head r32_12 head r32_12; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
for v in head r32_12 fc1k fc4k head; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; done
bash scripts/ab_c3.sh head cw2 cw8 head cw2 cw8
