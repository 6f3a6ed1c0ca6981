# A/B: fused digit counts in the query ordering (fq1) vs HEAD: C2 and C4; query GPU tests on fq1
mkdir -p gpurun_out
bash scripts/ab_c2.sh head fq1 head fq1
bash scripts/ab_c4.sh head fq1 head fq1
cp var/fq1.so paper_2409_10743_b200/libspb200.so
timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_bvh.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
