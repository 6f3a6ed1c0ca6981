# usage: bash scripts/ncu_full.sh <regex> <name> <n> [skip]
set -x
python paper_2409_10743_b200/build.py
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${4:-1} -c 1 -o gpurun_out/$2 -f python scripts/prof_fof.py $3 2 > gpurun_out/$2.log 2>&1
tail -3 gpurun_out/$2.log
