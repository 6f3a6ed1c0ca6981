python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
echo "== points"; SPB_FOF_POINTS=1 timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
echo "== cells"; timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_scale.py tests/test_distributed.py -x -q 2>&1 | tail -3
