# End-of-round evidence (one GPU call): bench (ours + reference arm), the four
# SURVEY configs, and the headline launch list + ncu --set full of the sort pass.
set -x
python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -1 gpurun_out/bench_ours.json | cut -c1-400
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# C1 steps are 0.6 ms: 50 of them keep the wall-clock e2e figure out of host jitter
timeout 900 python bench.py --workload c1 --steps 50 --warmup 10 > gpurun_out/cfg_c1.json 2>gpurun_out/cfg_c1.err
for w in c2 c3 c4 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/cfg_$w.json 2>gpurun_out/cfg_$w.err; done
timeout 400 python bench.py --slabs --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_slabs.json 2> gpurun_out/bench_slabs.err
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cells_2p27.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rs_onesweep -s 7 -c 1 -o gpurun_out/sort_cells_2p27 -f python scripts/prof_fof.py $N 2 > /dev/null 2>&1
ls -la gpurun_out/*.json gpurun_out/*.ncu-rep | tail -12
