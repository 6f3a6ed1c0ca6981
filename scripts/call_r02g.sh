mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slabs.py -x -q > gpurun_out/t_g.log 2>&1; tail -3 gpurun_out/t_g.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -1 gpurun_out/bench_g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['merge_visits']['visits_per_cell'], d['parity']['match'], d['e2e']['value'])"
timeout 600 python bench.py --slabs --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_slabs_g.json 2> gpurun_out/bench_slabs_g.err; tail -1 gpurun_out/bench_slabs_g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['parity']['match'], d['e2e']['value'])"
tail -2 gpurun_out/bench_slabs_g.err
