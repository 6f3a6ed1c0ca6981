for f in 1.3 1.5 2.0; do echo "== R factor $f"; SPB_KNN_RFACTOR=$f timeout 120 python scripts/c4_probe.py 2>&1 | tail -2; done
