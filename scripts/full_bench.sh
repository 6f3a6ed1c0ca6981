# headline bench, reference arm, and the four SURVEY configs (one GPU call)
python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -1 gpurun_out/bench_ours.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-300
for w in c1 c2 c3 c4; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/cfg_$w.json 2>gpurun_out/cfg_$w.err; tail -1 gpurun_out/cfg_$w.json | cut -c1-1200; done
