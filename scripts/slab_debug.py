"""Debug: slab multi G=2 vs single FoF on a small field; where do labels differ?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
from paper_2409_10743_b200.distributed import fof_slabs_multi
n = 1 << 18
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = torch.from_numpy(sp.generate_reference_field(n)).cuda()
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
want = sp.friends_of_friends(p, eps)
wl = want.labels.cpu().numpy()
b = np.linspace(0, n, G + 1).astype(np.int64)
ctxs = [sp.Context(0) for _ in range(G)]
res = fof_slabs_multi([p[b[r]:b[r + 1]].contiguous() for r in range(G)], eps, ctxs=ctxs)
gl = np.concatenate([r[0].cpu().numpy() for r in res])
bad = np.nonzero(gl != wl)[0]
print("G", G, "mismatches", bad.size, "of", n)
if bad.size:
    x = p[:, 0].cpu().numpy()
    print("first bad rows", bad[:10], "got", gl[bad[:10]], "want", wl[bad[:10]], "x", x[bad[:10]])
    print("rank of bad rows", np.bincount(np.searchsorted(b, bad, side="right") - 1, minlength=G))
    print("got==-1", int((gl[bad] == -1).sum()), "want==-1", int((wl[bad] == -1).sum()),
          "got==row", int((gl[bad] == bad).sum()))
