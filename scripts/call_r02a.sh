mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv) > gpurun_out/sysinfo.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -1 gpurun_out/bench_ours.json
OMP_NUM_THREADS=$(nproc) OMP_PROC_BIND=close timeout 1200 python scripts/ref_pin.py gpurun_out/ref_pin.json 24 26 27 > gpurun_out/ref_pin.log 2>&1; tail -3 gpurun_out/ref_pin.log
cat gpurun_out/sysinfo.txt | head -4
