# Re-entry baseline of the current tree: GPU tests, smoke, headline bench, launch list, merge ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j_smi.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/j_tests.log 2>&1; tail -3 gpurun_out/j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; tail -1 gpurun_out/j_bench.json | cut -c1-1500
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/j_launches.csv | head -16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fof_cells_merge -s 1 -c 1 -o gpurun_out/j_merge -f python scripts/prof_fof.py $N 2 > gpurun_out/j_merge.log 2>&1; tail -2 gpurun_out/j_merge.log
