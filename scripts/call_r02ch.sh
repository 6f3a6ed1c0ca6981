# climb CTA 128 (cb128, new default) vs 64 (cb64); GPU suite on cb128
mkdir -p gpurun_out
for v in cb128 cb64 cb128 cb64; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 2 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
cp var/cb128.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
