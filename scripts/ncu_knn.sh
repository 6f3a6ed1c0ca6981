# ncu --set full of the two kNN kernels at C4 (2^24 points, 2^24 queries, k = 16)
python paper_2409_10743_b200/build.py >/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_knn_rope -c 1 -o gpurun_out/knn_rope -f python scripts/c4_probe.py > gpurun_out/knn_rope.log 2>&1
#SPB_KNN_MODE=2 ncu --set full --clock-control none --import-source on -k regex:k_knn -c 1 -o gpurun_out/knn_legacy -f python scripts/c4_probe.py > gpurun_out/knn_legacy.log 2>&1
tail -2 gpurun_out/knn_rope.log gpurun_out/knn_legacy.log
