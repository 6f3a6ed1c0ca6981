for v in hw0 hw1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 60 python scripts/build_probe.py 2>&1 | cut -c1-420; done
