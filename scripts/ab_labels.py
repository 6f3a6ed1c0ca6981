"""A/B helper: FoF timing on the headline field plus a labels hash (compare across variants)."""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
ms = []
for _ in range(reps):
    out = sp.friends_of_friends(p, eps, ctx=ctx)
    ms.append(dict(ctx.phases()).get("merge", 0))
h = hashlib.sha1(out.labels.cpu().numpy().tobytes()).hexdigest()[:16]
print("merge_ms", ["%.2f" % x for x in ms], "labels", h, [(k, round(v, 2)) for k, v in ctx.phases()])
