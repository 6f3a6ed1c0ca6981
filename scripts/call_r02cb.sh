# A/B: cell compaction tile of 8 / 16 (head) / 24 / 32 keys per thread
mkdir -p gpurun_out
for v in head cc8 cc24 cc32 head cc8 cc24 cc32; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
