# evidence after the kNN and slab changes: GPU suite, smoke, headline + reference arm, C4 line, C4 launch list + capture
O=gpurun_out/r02f
mkdir -p $O
python paper_2409_10743_b200/build.py >/dev/null
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python scripts/pcie_probe.py > $O/pcie.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_ours.json 2> $O/bench_ours.err; tail -1 $O/bench_ours.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json | cut -c1-200
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > $O/cfg_c4.json 2> $O/cfg_c4.err; tail -1 $O/cfg_c4.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_2p24.csv python scripts/c4_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn -s 1 -c 1 -o $O/c4_knn_2p24 -f python scripts/c4_probe.py $((1<<24)) 2 > $O/c4_knn_2p24.log 2>&1; tail -1 $O/c4_knn_2p24.log
