# A/B: hierarchy CTA of 512 leaves (b512), acquire fence only on second arrivals (..a), vs fd
mkdir -p gpurun_out
for v in fd b512 b512a b256a fd b512; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/build_probe.py 2>&1 | tail -2 | cut -c 1-300; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 1-300; done
cp var/b512.so paper_2409_10743_b200/libspb200.so
timeout 1200 python -m pytest tests -m gpu -x -q -k "bvh or hier or build or fof or scale" 2>&1 | tail -3
