# ncu: the FoF labels scatter (k_fof_cells_labels): DRAM traffic of the random 4-byte label writes
mkdir -p gpurun_out
timeout 600 ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none -k regex:"k_fof_cells_labels|k_fof_cells_core_min" -s 0 -c 2 -o gpurun_out/labels_r02 -f python scripts/prof_fof.py 134217728 1 > gpurun_out/labels_r02.log 2>&1; tail -1 gpurun_out/labels_r02.log
