python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
for w in c1 c2 c3 c4; do timeout 600 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/cfg_$w.json 2>gpurun_out/cfg_$w.err; tail -1 gpurun_out/cfg_$w.json | cut -c1-1500; tail -2 gpurun_out/cfg_$w.err; done
