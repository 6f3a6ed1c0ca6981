# quick GPU check: build, the given pytest files, then an optional command
python paper_2409_10743_b200/build.py >/dev/null
make -s -C oracle all
timeout 900 python -m pytest $1 -x -q 2>&1 | tail -4
shift
for c in "$@"; do eval "$c"; done
