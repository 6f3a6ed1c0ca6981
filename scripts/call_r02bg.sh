# A/B: kNN without the redundant full-list tests (kn1) vs HEAD (ld1); kNN GPU tests on kn1
mkdir -p gpurun_out
bash scripts/ab_c4.sh ld1 kn1 ld1 kn1
cp var/kn1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "knn or nearest or scale" 2>&1 | tail -2
