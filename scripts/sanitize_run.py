"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2409_10743_b200 as sp
from oracle_lib import Oracle, eps_for
O = Oracle.get()
n = 1 << 14
pts = O.field(n); eps = eps_for(n)
out = sp.friends_of_friends(pts, eps)
lab, core = O.dbscan(pts, 3, eps, 2)
assert np.array_equal(out.labels, lab)
d = sp.fdbscan_densebox(pts, sp.DbscanParams(eps, 5))
f = sp.fdbscan(pts, sp.DbscanParams(eps, 5))
b = sp.Bvh.build(pts)
c = sp.range_count(b, pts, radius=eps * 3)
k = sp.nearest_query(b, pts[:1000], 16)
sph = np.concatenate([pts[:1000], np.full((1000, 1), eps * 2, np.float32)], 1)
crs = sp.query_crs(b, sph)
print("sanitized run ok", int(c.sum()), k.shape)
