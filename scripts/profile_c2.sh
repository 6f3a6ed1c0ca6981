# C2 (BVH build + range count) ncu evidence: launch list + a full capture of the range-count kernel
set -x
python paper_2409_10743_b200/build.py >/dev/null
python scripts/c2_probe.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_2p24.csv python scripts/c2_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_range_count -s 1 -c 1 -o gpurun_out/c2_range_2p24 -f python scripts/c2_probe.py $((1<<24)) 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
