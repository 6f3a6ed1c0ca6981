# Round-2 evidence (one GPU call): GPU tests, smoke, the headline bench line
# (with its C3/C5 extras and CPU baseline), the reference arm, the other
# SURVEY configs, the one-rank slab path, launch lists and ncu --set full
# captures of the top kernels.  Outputs under gpurun_out/r02/.
O=gpurun_out/r02j
mkdir -p $O
python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv) > $O/host.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python scripts/pcie_probe.py > $O/pcie.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_ours.json 2> $O/bench_ours.err; tail -1 $O/bench_ours.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json | cut -c1-300
timeout 600 python bench.py --workload c1 --steps 50 --warmup 10 > $O/cfg_c1.json 2> $O/cfg_c1.err
for w in c2 c3 c4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/cfg_$w.json 2> $O/cfg_$w.err; done
timeout 600 python bench.py --slabs --steps 10 --warmup 3 --no-extra --no-cpu-baseline > $O/bench_slabs.json 2> $O/bench_slabs.err
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cells_2p27.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_build_2p27.csv python scripts/prof_build.py $N 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_2p24.csv python scripts/c2_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_2p24.csv python scripts/c4_probe.py $((1<<24)) 2 > /dev/null 2>&1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${4:-1} -c 1 -o $O/$2 -f python $3 > $O/$2.log 2>&1; tail -1 $O/$2.log; }
cap k_fof_cells_merge merge_cells_2p27 "scripts/prof_fof.py $N 2"
cap k_rs_onesweep sort_cells_2p27 "scripts/prof_fof.py $N 2" 7
cap "k_hierarchy" hier_cells_2p27 "scripts/prof_fof.py $N 2"
cap "k_hierarchy" hier_2p27 "scripts/prof_build.py $N 2"
cap "k_rs_onesweep<16, 256, unsigned int, unsigned int>" sort_2p27 "scripts/prof_build.py $N 2" 2
cap k_knn c4_knn_2p24 "scripts/c4_probe.py $((1<<24)) 2"
cap k_range_count c2_range_2p24 "scripts/c2_probe.py $((1<<24)) 2"
ls -la $O | tail -40
