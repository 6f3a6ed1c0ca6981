bash scripts/ab_var.sh base w2 w2adj w3adj
cp var/w2adj.so paper_2409_10743_b200/libspb200.so
timeout 600 python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
cp var/base.so paper_2409_10743_b200/libspb200.so
timeout 300 python scripts/prof_db.py 2>&1 | tail -8
