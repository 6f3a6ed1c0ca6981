mkdir -p gpurun_out
bash scripts/ab_c2.sh old new old new
bash scripts/ab_c3.sh old new
bash scripts/ab_var.sh old new 2>&1 | tail -4
