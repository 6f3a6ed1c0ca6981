import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
dev = torch.device("cuda", 0)
ctx = sp.Context(0)
pts = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pts)
hl = torch.empty(n, dtype=torch.int32, pin_memory=True); hc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
c = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
sp.friends_of_friends(hp, eps, ctx=c, out=(hl, hc))
c.set_async(True)
c.synchronize()
for _ in range(4):
    sp.friends_of_friends(hp, eps, ctx=c, out=(hl, hc))
c.synchronize()
