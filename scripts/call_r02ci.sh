# final evidence after the climb CTA change: headline bench line, build launch list, hierarchy captures
O=gpurun_out/r02k
mkdir -p $O
python paper_2409_10743_b200/build.py >/dev/null
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_ours.json 2> $O/bench_ours.err; tail -1 $O/bench_ours.json | cut -c1-200
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 > $O/cfg_c3.json 2> $O/cfg_c3.err
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 > $O/cfg_c2.json 2> $O/cfg_c2.err
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 > $O/cfg_c4.json 2> $O/cfg_c4.err
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_build_2p27.csv python scripts/prof_build.py $N 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cells_2p27.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${4:-1} -c 1 -o $O/$2 -f python $3 > $O/$2.log 2>&1; tail -1 $O/$2.log; }
cap "k_hierarchy" hier_cells_2p27 "scripts/prof_fof.py $N 2"
cap "k_hierarchy" hier_2p27 "scripts/prof_build.py $N 2"
ls $O
