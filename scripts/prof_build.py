"""Run Bvh::build on uniform points (for ncu captures): prof_build.py N REPS."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = sp.Context(0)
p = sp.generate_uniform(n, 3, seed=2409, ctx=ctx)
for _ in range(reps):
    b = sp.Bvh.build(p, ctx=ctx)
    del b
print(ctx.phases())
