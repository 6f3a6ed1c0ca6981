"""e2e FoF: which transfer direction breaks the overlap?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
steps = 6
dev = torch.device("cuda", 0)
ctx = sp.Context(0)
pts = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pts)
hl = torch.empty(n, dtype=torch.int32, pin_memory=True); hc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dl = torch.empty(n, dtype=torch.int32, device=dev); dc = torch.empty(n, dtype=torch.uint8, device=dev)
for name, inp, out in (("host in, host out", hp, (hl, hc)), ("host in, device out", hp, (dl, dc)),
                       ("device in, host out", pts, (hl, hc)), ("device in, device out", pts, (dl, dc))):
    c = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
    sp.friends_of_friends(inp, eps, ctx=c, out=out)
    c.set_async(True)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(steps):
        sp.friends_of_friends(inp, eps, ctx=c, out=out)
    c.synchronize(); torch.cuda.synchronize()
    print(name, "%.1f ms/step" % ((time.perf_counter() - t) / steps * 1e3), [(k, round(v, 1)) for k, v in c.phases()], flush=True)
    c.set_async(False)
