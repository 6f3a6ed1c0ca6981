import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 24
ctx = sp.Context(0)
pts = sp.generate_uniform(n, 3, seed=2409, ctx=ctx)
qs = sp.generate_uniform(n, 3, seed=2410, ctx=ctx)
b = sp.Bvh.build(pts, ctx=ctx)
for mode in ("fast", "fast", "fast"):
    torch.cuda.synchronize(); t = time.perf_counter()
    idx = sp.nearest_query(b, qs, 16)
    torch.cuda.synchronize(); print(mode, "knn %.2f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
