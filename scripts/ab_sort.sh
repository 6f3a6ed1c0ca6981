python paper_2409_10743_b200/build.py
for k in 8 12 16; do echo "== items $k"; SPB_RS_ITEMS=$k python scripts/prof_fof.py 134217728 3 2>&1 | tail -1; done
SPB_RS_ITEMS=8 python -m pytest tests/test_gpu_bvh.py tests/test_gpu_scale.py -x -q -k "c2 or random or c1 or golden" 2>&1 | tail -2
