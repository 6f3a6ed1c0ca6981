# confirm: CP_ILP 2 + RS_ITEMS 12 (new) vs head; cp1; GPU suite on new
mkdir -p gpurun_out
for v in head new cp1 head new cp1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== fof $v"; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | sed 's/merge_ms.*labels/labels/' | cut -c 1-200; done
for v in head new; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== build $v"; timeout 120 python scripts/build_probe.py 2>&1 | tail -2 | cut -c1-200; done
bash scripts/ab_c3.sh head new
cp var/new.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
