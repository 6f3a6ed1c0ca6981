# A/B: bin divisions by hoisted reciprocal with exact fallback (rc1) vs true f64 division (rc0); GPU suite on rc1
mkdir -p gpurun_out
for v in rc0 rc1 rc0 rc1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-300; done
cp var/rc1.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
