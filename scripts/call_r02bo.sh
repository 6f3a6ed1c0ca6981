# A/B: kNN register caps (64-thread blocks): none (kb64, 62 regs) / 18 blocks (56) / 20 blocks (48)
mkdir -p gpurun_out
bash scripts/ab_c4.sh kb64 km18 km20 kb64 km18 km20
