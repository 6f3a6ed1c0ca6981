# A/B: merge occupancy caps (11-13 blocks of 128 per SM) vs HEAD (10 blocks, 47 registers)
mkdir -p gpurun_out
for v in head mb11 mb13 head mb11 mb13; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 2 2>&1 | tail -1 | cut -c 1-120; done
