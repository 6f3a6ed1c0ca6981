# A/B: packed cell range in the leaf word (pk1) vs cell_start loads (ld1); C3 too; GPU tests on pk1
mkdir -p gpurun_out
for v in ld1 pk1 ld1 pk1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
bash scripts/ab_c3.sh ld1 pk1
cp var/pk1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
