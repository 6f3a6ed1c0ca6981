# usage: bash scripts/launches.sh <name> <n>
python paper_2409_10743_b200/build.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$1.csv python scripts/prof_fof.py $2 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/$1.csv
