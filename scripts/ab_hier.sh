python paper_2409_10743_b200/build.py
timeout 120 python -m pytest tests/test_gpu_bvh.py -x -q 2>&1 | tail -2
timeout 60 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
timeout 200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dbscan.py -x -q 2>&1 | tail -2
