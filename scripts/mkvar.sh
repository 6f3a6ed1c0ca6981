# Build an A/B variant of the library: scripts/mkvar.sh NAME "-DFLAG=1 ..." -> var/NAME.so
mkdir -p var
SPB_LIB_OUT=$PWD/var/$1.so SPB_NVCC_EXTRA="$2" python paper_2409_10743_b200/build.py --force
