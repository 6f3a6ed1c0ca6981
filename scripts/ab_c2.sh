# A/B prebuilt library variants in var/*.so on C2 (BVH build + range count, 2^24)
for v in "$@"; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/c2_probe.py $((1<<24)) 6 2>&1 | tail -2; done
