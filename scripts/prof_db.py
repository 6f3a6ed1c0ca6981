import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
mp = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
for _ in range(4):
    out = sp.fdbscan_densebox(p, sp.DbscanParams(eps, mp), ctx=ctx)
    print("densebox", out.timings, out.stats)
for _ in range(3):
    out = sp.fdbscan(p, sp.DbscanParams(eps, mp), ctx=ctx)
    print("fdbscan", out.timings)
