# Refresh of the ncu evidence after the SM-affine schedule and the kNN changes:
# headline launch list + merge capture, and C2/C3/C4 launch lists + top-kernel captures.
set -x
python paper_2409_10743_b200/build.py >/dev/null
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cells_2p27.csv python scripts/prof_fof.py $N 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fof_cells_merge -s 1 -c 1 -o gpurun_out/merge_cells_2p27 -f python scripts/prof_fof.py $N 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_2p24.csv python scripts/c2_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_range_count -s 1 -c 1 -o gpurun_out/c2_range_2p24 -f python scripts/c2_probe.py $((1<<24)) 2 > /dev/null 2>&1
cat > /tmp/c3once.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, paper_2409_10743_b200 as sp
n = 1 << 26
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
for _ in range(2):
    out = sp.fdbscan_densebox(p, sp.DbscanParams(eps, 5), ctx=ctx)
print(out.stats)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_2p26.csv python /tmp/c3once.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_core_merge -s 1 -c 1 -o gpurun_out/c3_core_merge_2p26 -f python /tmp/c3once.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_2p24.csv python scripts/c4_probe.py $((1<<24)) 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn -s 1 -c 1 -o gpurun_out/c4_knn_2p24 -f python scripts/c4_probe.py $((1<<24)) 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
