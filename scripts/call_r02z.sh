mkdir -p gpurun_out
cp var/par.so paper_2409_10743_b200/libspb200.so
timeout 1500 python -m pytest tests/test_gpu_bvh.py -q -x 2>&1 | tail -2
for v in par parnf; do cp var/$v.so paper_2409_10743_b200/libspb200.so; echo "== $v"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hierarchy" --csv python scripts/prof_build.py 134217728 1 2>/dev/null | grep -v "^==" | cut -d, -f13- | tail -1; done
cp var/par.so paper_2409_10743_b200/libspb200.so
timeout 200 python scripts/build_probe.py 2>&1 | tail -1 | cut -c1-200; timeout 120 python scripts/ab_labels.py 134217728 3 2>&1 | tail -1 | cut -c 60-300
