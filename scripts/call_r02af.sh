# launch list + captures of the build on H(2^27) with the 32-bit climb
O=gpurun_out/r02f; mkdir -p $O
python paper_2409_10743_b200/build.py > /dev/null
N=134217728
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_build_field_2p27.csv python scripts/prof_build_field.py $N 2 > /dev/null 2>&1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${4:-1} -c 1 -o $O/$2 -f python $3 > $O/$2.log 2>&1; tail -1 $O/$2.log; }
cap "k_hierarchy" hier_field_2p27 "scripts/prof_build_field.py $N 2"
cap "k_fix_gather" gather_field_2p27 "scripts/prof_build_field.py $N 2"
