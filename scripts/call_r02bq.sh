# evidence after the C3 core-merge change: GPU suite, C3 line and launch list
O=gpurun_out/r02g
mkdir -p $O
python paper_2409_10743_b200/build.py >/dev/null
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 > $O/cfg_c3.json 2> $O/cfg_c3.err; tail -1 $O/cfg_c3.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_2p26.csv python scripts/c3_probe.py > /dev/null 2>&1
ls $O
