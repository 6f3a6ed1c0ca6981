# A/B: kNN squared lower-bound keys (sq1) vs rounded-down square roots (sq0)
mkdir -p gpurun_out
for v in sq0 sq1 sq0 sq1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/c4_probe.py 16777216 6 2>&1 | tail -1; done
cp var/sq1.so paper_2409_10743_b200/libspb200.so
timeout 600 python -m pytest tests -m gpu -x -q -k "knn or nearest or c4 or query" 2>&1 | tail -3
