# A/B: fp32-filtered kNN (kf, kf7 = 7 blocks/SM) vs the exact-key kernel (kn); C5 e2e fix
mkdir -p gpurun_out
for v in kn kf kf7 kn kf; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 300 python scripts/c4_probe.py 16777216 4 | tail -1; done
cp var/kf.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests -x -q -m gpu -k "knn or nearest" 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
timeout 900 python bench.py --workload c5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/p_c5.json 2> gpurun_out/p_c5.err; echo "c5 rc=$?"; tail -1 gpurun_out/p_c5.json | cut -c1-900; tail -3 gpurun_out/p_c5.err
