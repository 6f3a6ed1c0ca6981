mkdir -p gpurun_out
for v in st1 st2 st1 st2; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c4_probe.py 16777216 4 | tail -1; done
cp var/st2.so paper_2409_10743_b200/libspb200.so; timeout 900 python -m pytest tests -q -x -m gpu -k "knn or nearest or c4" 2>&1 | tail -1
