for m in 0 2 0 2; do echo "== mode $m"; SPB_KNN_MODE=$m timeout 120 python scripts/c4_probe.py 2>&1 | tail -1; done
