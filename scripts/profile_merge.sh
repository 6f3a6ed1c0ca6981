# ncu --set full of the current headline merge kernel (cell pair walk, FAST form)
python paper_2409_10743_b200/build.py >/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fof_cells_merge -s 1 -c 1 -o gpurun_out/merge_cells_2p27 -f python scripts/prof_fof.py 134217728 2 > /dev/null 2>&1
ls -la gpurun_out/merge_cells_2p27.ncu-rep
