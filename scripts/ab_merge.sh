python paper_2409_10743_b200/build.py
echo "== bucket 1"; SPB_BUCKET=1 python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
for k in 2 4 8 16; do
  echo "== group $k"; SPB_GROUP=1 SPB_BUCKET=$k python scripts/prof_fof.py 134217728 3 2>&1 | tail -1
done
SPB_GROUP=1 SPB_BUCKET=4 python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_scale.py -x -q -k "fof or c5 or kats or c1" 2>&1 | tail -2
