# A/B: merge walk with the prefix-reach cut-off (rc1) vs without (rc0); walk anatomy; FoF parity on rc1
mkdir -p gpurun_out
for v in rc0 rc1 rc0 rc1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
for v in rc0 rc1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== walks $v"; timeout 200 python scripts/merge_walks.py 2>&1 | tail -1; done
cp var/rc1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
