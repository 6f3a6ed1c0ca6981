# A/B: split lengths written by the run fix-up (fd) vs k_delta (i32); parity on fd
mkdir -p gpurun_out
for v in i32 fd i32 fd; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -3 | cut -c 1-400; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-400; done
cp var/fd.so paper_2409_10743_b200/libspb200.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
