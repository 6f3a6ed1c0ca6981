"""Probe: end-to-end FoF steps with host buffers, one async context (as the
bench) vs two contexts driven by two host threads (alternating steps)."""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
dev = torch.device("cuda", 0)
ctx = sp.Context(0)
pts = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pts)
del pts
outs = [(torch.empty(n, dtype=torch.int32, pin_memory=True), torch.empty(n, dtype=torch.uint8, pin_memory=True)) for _ in range(2)]
steps = 8
c1 = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
sp.friends_of_friends(hp, eps, ctx=c1, out=outs[0]); c1.set_async(True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(steps):
    sp.friends_of_friends(hp, eps, ctx=c1, out=outs[0])
c1.synchronize(); print("one context: %.1f ms/step" % ((time.perf_counter() - t) / steps * 1e3), flush=True)
c1.set_async(False)
cs = [sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream) for _ in range(2)]
for i, c in enumerate(cs):
    sp.friends_of_friends(hp, eps, ctx=c, out=outs[i]); c.set_async(True)
torch.cuda.synchronize()
def run(i):
    for _ in range(steps // 2):
        sp.friends_of_friends(hp, eps, ctx=cs[i], out=outs[i])
    cs[i].synchronize()
t = time.perf_counter()
th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
[x.start() for x in th]; [x.join() for x in th]
print("two contexts/threads: %.1f ms/step" % ((time.perf_counter() - t) / steps * 1e3), flush=True)
