# A/B: four-wide cell tree merge (w1) vs binary walk (w0) on the headline field; GPU tests on w1
mkdir -p gpurun_out
for v in w0 w1 w0 w1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-400; done
cp var/w1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
