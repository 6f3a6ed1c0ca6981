# native slab path + reference-pinned scale tests + the new bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_scale.py -x -q > gpurun_out/t_slabs.log 2>&1; tail -15 gpurun_out/t_slabs.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; tail -1 gpurun_out/bench_c.json; tail -5 gpurun_out/bench_c.err
timeout 600 python bench.py --slabs --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_slabs.json 2> gpurun_out/bench_slabs.err; tail -1 gpurun_out/bench_slabs.json; tail -5 gpurun_out/bench_slabs.err
