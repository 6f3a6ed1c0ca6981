# A/B: block-stencil FoF merge (st1, no cell tree) vs the cell-tree walk (st0); GPU tests on st1
mkdir -p gpurun_out
for v in st0 st1 st0 st1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/st1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
