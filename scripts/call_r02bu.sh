# C4 evidence after the kNN push change: config line, launch list, ncu capture of k_knn16lb
O=gpurun_out/r02h
mkdir -p $O
python paper_2409_10743_b200/build.py >/dev/null
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > $O/cfg_c4.json 2> $O/cfg_c4.err; tail -1 $O/cfg_c4.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_2p24.csv python scripts/c4_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn -s 1 -c 1 -o $O/c4_knn_2p24 -f python scripts/c4_probe.py $((1<<24)) 2 > $O/c4_knn_2p24.log 2>&1; tail -1 $O/c4_knn_2p24.log
