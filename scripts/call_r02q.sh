mkdir -p gpurun_out
nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.max.sm,clocks.max.mem --format=csv
for v in nolb lb nolb lb; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c4_probe.py 16777216 4 | tail -1; done
