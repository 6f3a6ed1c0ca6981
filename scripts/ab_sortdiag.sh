for v in rs_notma rs_tma; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; SPB_SORT_MARKS=1 timeout 60 python scripts/build_probe.py 2>&1 | cut -c1-420; done
