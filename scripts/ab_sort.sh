python paper_2409_10743_b200/build.py >/dev/null
for k in 0 1 2 3 4; do echo "== cfg $k"; SPB_RS_CFG=$k timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1; done
for k in 1 2 3 4; do SPB_RS_CFG=$k timeout 120 python -m pytest tests/test_gpu_bvh.py -x -q -k "random or golden or c1" 2>&1 | tail -1; done
