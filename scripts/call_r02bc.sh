# A/B: 256-bit node loads (ld1) vs two 128-bit loads (ld0): headline merge, C2, C4, C3; GPU tests on ld1
mkdir -p gpurun_out
for v in ld0 ld1 ld0 ld1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
bash scripts/ab_c2.sh ld0 ld1 ld0 ld1
bash scripts/ab_c4.sh ld0 ld1
bash scripts/ab_c3.sh ld0 ld1
cp var/ld1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
