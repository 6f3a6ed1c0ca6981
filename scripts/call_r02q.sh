# A/B: kNN with fp32 lower-bound keys and exact leaf distances at the visit (lb) vs exact keys (nolb)
mkdir -p gpurun_out
cp var/lb.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -q -x -m gpu -k "knn or nearest or c4 or query" 2>&1 | tail -2
for v in nolb lb nolb lb; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c4_probe.py 16777216 4 | tail -1; done
