# A/B prebuilt library variants in var/*.so on the headline FoF step
for v in "$@"; do for r in 1 2; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1; done; done
