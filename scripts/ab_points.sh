# A/B prebuilt library variants in var/*.so on the point-path clustering (fdbscan_probe.py)
for v in "$@"; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/fdbscan_probe.py 2>&1 | tail -2; done
