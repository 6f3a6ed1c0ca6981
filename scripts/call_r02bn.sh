# A/B: kNN block size 64 / 128 (cm1) / 256 / 512
mkdir -p gpurun_out
bash scripts/ab_c4.sh cm1 kb64 kb256 kb512 cm1 kb64 kb256 kb512
