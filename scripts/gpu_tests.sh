set -x
python paper_2409_10743_b200/build.py
make -s -C oracle all
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -30
