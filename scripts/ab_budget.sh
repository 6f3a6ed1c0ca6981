python paper_2409_10743_b200/build.py >/dev/null
echo "== simple"; timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
for x in 0.5 1 2 4 1000; do echo "== packet $x"; SPB_PACKET=$x timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1; done
SPB_PACKET=2 timeout 300 python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_scale.py -x -q -k "fof or c5 or c1 or kats" 2>&1 | tail -2
