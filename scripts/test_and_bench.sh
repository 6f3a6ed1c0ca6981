set -x
python paper_2409_10743_b200/build.py
make -s -C oracle all
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','phases_ms','e2e','roofline','bvh_build_mpts_s')})"
