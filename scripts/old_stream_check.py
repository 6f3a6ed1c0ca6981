import sys, ctypes as C
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2409_10743_b200 as sp
from oracle_lib import Oracle, eps_for
sp._stream_arg = lambda s: C.c_void_p(s) if s else None   # the old (buggy) mapping
O = Oracle.get()
pts = O.field(1 << 16); eps = eps_for(1 << 16)
base = torch.from_numpy(pts).cuda(); torch.cuda.synchronize()
ctx = sp.Context(0, stream=torch.cuda.current_stream().cuda_stream)
lab, core = O.dbscan(pts, 3, eps, 2)
bad = 0
for _ in range(3):
    dst = torch.zeros_like(base); torch.cuda._sleep(50_000_000); dst.copy_(base)
    out = sp.friends_of_friends(dst, eps, ctx=ctx)
    bad += not np.array_equal(out.labels.cpu().numpy(), lab)
print("old mapping: %d of 3 runs wrong (the regression test must catch this)" % bad)
