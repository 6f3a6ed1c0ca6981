for m in new legacy new legacy; do echo "== $m"; if [ $m = legacy ]; then export SPB_KNN_LEGACY=1; else unset SPB_KNN_LEGACY; fi; timeout 120 python scripts/c4_probe.py 2>&1 | tail -1; done
