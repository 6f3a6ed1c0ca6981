# A/B: kNN push without the stack bound test (ks1) vs HEAD; kNN GPU tests on ks1
mkdir -p gpurun_out
bash scripts/ab_c4.sh head ks1 head ks1
cp var/ks1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "knn or nearest or scale" 2>&1 | tail -2
