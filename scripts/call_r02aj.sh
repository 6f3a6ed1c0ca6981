# A/B: merge walk with the precomputed prefix reach (rx1) vs without (rx0); walk anatomy; FoF parity on rx1
mkdir -p gpurun_out
for v in rx0 rx1 rx0 rx1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
for v in rx0 rx1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== walks $v"; timeout 200 python scripts/merge_walks.py 2>&1 | tail -1; done
cp var/rx1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
