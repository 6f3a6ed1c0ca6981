# reach cut-off in the cell merge + block-aggregated slab routing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_scale.py tests/test_gpu_densebox.py tests/test_gpu_dbscan.py -x -q > gpurun_out/t_d.log 2>&1; tail -4 gpurun_out/t_d.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; tail -1 gpurun_out/bench_d.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['merge_visits'], d['parity'], d['e2e'])"
timeout 600 python bench.py --slabs --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_slabs_d.json 2> gpurun_out/bench_slabs_d.err; tail -1 gpurun_out/bench_slabs_d.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['parity'], d['e2e'])"
tail -3 gpurun_out/bench_slabs_d.err
