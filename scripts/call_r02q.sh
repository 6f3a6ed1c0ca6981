# A/B: merge walk loads a leaf's parent with its node (pb1) vs after the test (pb0)
mkdir -p gpurun_out
for v in pb0 pb1 pb0 pb1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
