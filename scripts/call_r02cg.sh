# sweeps: merge block of 64 / 256 threads (mt64 / mt256), climb CTA of 128 leaves (cb128) vs head (128 / 256)
mkdir -p gpurun_out
for v in head mt64 mt256 cb128 head mt64 mt256 cb128; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
for v in head cb128 head cb128; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; done
