# A/B prebuilt library variants in var/*.so on C4 (kNN k = 16, 2^24)
for v in "$@"; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/c4_probe.py 2>&1 | tail -1; done
