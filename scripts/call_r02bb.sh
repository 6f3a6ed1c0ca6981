# wide merge: fixed-trip leaf loop (w2) timing; ncu of the wide walk and the collapse (w2)
mkdir -p gpurun_out
for v in w2 w1; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 120 python scripts/ab_labels.py 134217728 2 2>&1 | tail -1 | cut -c 1-400; done
cp var/w2.so paper_2409_10743_b200/libspb200.so
timeout 600 ncu --set full --clock-control none -k regex:"k_fof_cells_merge_wide|k_wide_collapse" -s 0 -c 2 -o gpurun_out/wide_r02 -f python scripts/prof_fof.py 134217728 1 > gpurun_out/wide_r02.log 2>&1; tail -2 gpurun_out/wide_r02.log
