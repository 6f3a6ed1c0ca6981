python paper_2409_10743_b200/build.py >/dev/null
for m in 0 5 0 5; do echo "== mode $m"; SPB_CELLS_EXP=$m timeout 120 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1; done
SPB_CELLS_EXP=5 timeout 600 python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
