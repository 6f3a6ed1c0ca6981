# slab FoF: empty-exchange fast path (one rank) -- slab GPU tests, the one-rank slab bench line, headline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_distributed.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --slabs --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/slabs_sf1.json 2> gpurun_out/slabs_sf1.err; tail -1 gpurun_out/slabs_sf1.json | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ours_sf1.json 2> gpurun_out/ours_sf1.err; tail -1 gpurun_out/ours_sf1.json | cut -c1-300
