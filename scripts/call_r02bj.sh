# ncu: the Morton / cell-key kernels (f64 bin division): pipe utilisation
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"k_morton_top32|k_fix_gather" -s 0 -c 2 -o gpurun_out/mort_r02 -f python scripts/prof_build.py 134217728 1 > gpurun_out/mort_r02.log 2>&1; tail -1 gpurun_out/mort_r02.log
timeout 600 ncu --set full --clock-control none -k regex:"k_cell_keys_p3v|k_cell_points3v_keys" -s 0 -c 2 -o gpurun_out/ckeys_r02 -f python scripts/prof_fof.py 134217728 1 > gpurun_out/ckeys_r02.log 2>&1; tail -1 gpurun_out/ckeys_r02.log
