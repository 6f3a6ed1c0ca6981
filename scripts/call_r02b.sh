# Reference-only work on the GPU host (196 GB RAM, 16 cores): the H(2^30)
# FoF pin and the SURVEY §8(d) CPU baselines at their stated sizes.
mkdir -p gpurun_out
free -g > gpurun_out/free_b.txt
export OMP_NUM_THREADS=$(nproc) OMP_PROC_BIND=close
timeout 1500 python scripts/cpu_baselines.py gpurun_out/cpu_baselines_r02.json c1 c2 c4 c3 > gpurun_out/cpu_baselines.log 2>&1
tail -4 gpurun_out/cpu_baselines.log
( while true; do free -g | awk '/Mem/{print $3}' >> gpurun_out/mem_trace.txt; sleep 10; done ) &
MT=$!
timeout 2400 python scripts/ref_pin_big.py gpurun_out/ref_pin_big.json 30 > gpurun_out/ref_pin_big.log 2>&1
echo "rc=$?" >> gpurun_out/ref_pin_big.log
kill $MT
tail -3 gpurun_out/ref_pin_big.log; sort -n gpurun_out/mem_trace.txt | tail -1
