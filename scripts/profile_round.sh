# Headline-size ncu evidence: launch list + full captures of the top kernels.
set -x
python paper_2409_10743_b200/build.py >/dev/null
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cells_2p27.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fof_cells_merge -s 1 -c 1 -o gpurun_out/merge_cells_2p27 -f python scripts/prof_fof.py $N 2 > gpurun_out/merge.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rs_onesweep -s 7 -c 1 -o gpurun_out/sort_cells_2p27 -f python scripts/prof_fof.py $N 2 > gpurun_out/sort.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hierarchy -s 1 -c 1 -o gpurun_out/hier_cells_2p27 -f python scripts/prof_fof.py $N 2 > gpurun_out/hier.log 2>&1
ls -la gpurun_out/*cells*.ncu-rep
