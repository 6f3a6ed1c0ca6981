# ncu --set full of k_hierarchy<1> for the sparse-table variant (m1) and the climb (m0)
O=gpurun_out/r02e; mkdir -p $O
for v in m1 m0; do cp var/$v.so paper_2409_10743_b200/libspb200.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hierarchy" -s 1 -c 1 -o $O/hier_$v -f python scripts/prof_build.py 134217728 2 > $O/hier_$v.log 2>&1; tail -1 $O/hier_$v.log; done
