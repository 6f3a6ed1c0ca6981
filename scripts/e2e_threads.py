"""e2e FoF with host buffers: one asynchronous context vs T host threads each driving its own context."""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
steps = 8
dev = torch.device("cuda", 0)
ctx = sp.Context(0)
pts = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pts)
for T, asyn in ((1, True), (2, True), (2, False), (3, True)):
    ctxs = [sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream) for _ in range(T)]
    outs = [(torch.empty(n, dtype=torch.int32, pin_memory=True), torch.empty(n, dtype=torch.uint8, pin_memory=True))
            for _ in range(T)]
    for c, o in zip(ctxs, outs):
        sp.friends_of_friends(hp, eps, ctx=c, out=o)
        c.set_async(asyn)
    def run(i):
        for _ in range(steps // T + (1 if i < steps % T else 0)):
            sp.friends_of_friends(hp, eps, ctx=ctxs[i], out=outs[i])
        ctxs[i].synchronize()
    torch.cuda.synchronize()
    t = time.perf_counter()
    th = [threading.Thread(target=run, args=(i,)) for i in range(T)]
    for x in th: x.start()
    for x in th: x.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("threads %d async %s: %.1f ms/step, %.3g pts/s" % (T, asyn, dt / steps * 1e3, n * steps / dt), flush=True)
    for c in ctxs:
        c.set_async(False)
    del ctxs, outs
