set -x
python paper_2409_10743_b200/build.py
make -s -C oracle all
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --steps 5 --warmup 3 2>&1 | tail -5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fof.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
