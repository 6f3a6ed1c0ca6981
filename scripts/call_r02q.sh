# A/B: keys per thread of the 32-bit-key onesweep passes
mkdir -p gpurun_out
for v in i16 i20 i24; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 60-300; done
