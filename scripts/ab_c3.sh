# A/B prebuilt library variants in var/*.so on C3 (DenseBox min_pts 5, 2^26 field)
for v in "$@"; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 200 python scripts/c3_probe.py 2>&1 | grep own-stream | tail -1 | cut -c1-300; done
