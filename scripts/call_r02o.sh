# C5 e2e OOM fix check; kNN full ncu capture (C4)
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/o_c5.json 2> gpurun_out/o_c5.err; echo "c5 rc=$?"; tail -1 gpurun_out/o_c5.json | cut -c1-900; tail -3 gpurun_out/o_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn -s 1 -c 1 -o gpurun_out/o_knn -f python scripts/c4_probe.py 16777216 2 > gpurun_out/o_knn.log 2>&1; tail -1 gpurun_out/o_knn.log
