# A/B: hierarchy with dense rounds (r1) vs the thread-wise climb (r0); parity on r1
mkdir -p gpurun_out
for v in r0 r1 r0 r1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -3 | cut -c 1-400; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-400; done
cp var/r1.so paper_2409_10743_b200/libspb200.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
