"""Merge walk anatomy on the headline field (diagnostic SP_FLAG_STATS pass):
visits per cell split into far rejections, cell (leaf) hits, descents, and the
tail of far rejections after a walk's last near node."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
ctx.set_stats(True)
sp.friends_of_friends(p, eps, ctx=ctx)
cells = ctx.counter("fof_cells")
v = {k: ctx.counter("merge_" + k) for k in ("node_visits", "pair_tests", "far_visits", "leaf_visits", "tail_visits")}
per = {k: round(x / cells, 2) for k, x in v.items()}
per["descents"] = round((v["node_visits"] - v["far_visits"] - v["leaf_visits"]) / cells, 2)
print("cells", cells, "per cell", per)
