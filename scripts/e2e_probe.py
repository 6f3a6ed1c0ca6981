import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
dev = torch.device("cuda", 0)
ctx = sp.Context(0)
pts = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pts)
hl = torch.empty(n, dtype=torch.int32, pin_memory=True); hc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for mode in ("sync", "async"):
    c2 = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
    sp.friends_of_friends(hp, eps, ctx=c2, out=(hl, hc))
    if mode == "async":
        c2.set_async(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        sp.friends_of_friends(hp, eps, ctx=c2, out=(hl, hc))
    c2.synchronize()
    torch.cuda.synchronize()
    print("cells", mode, "%.1f ms/step" % ((time.perf_counter() - t) / 5 * 1e3))
    c2.set_async(False)
t = time.perf_counter()
x = hp.cuda(); torch.cuda.synchronize(); print("h2d %.1f ms" % ((time.perf_counter() - t) * 1e3))
t = time.perf_counter()
hl.copy_(torch.empty(n, dtype=torch.int32, device=dev)); torch.cuda.synchronize(); print("d2h labels %.1f ms" % ((time.perf_counter() - t) * 1e3))
# per-phase times of an overlapped (async) step vs a device-resident step
c3 = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
sp.friends_of_friends(pts, eps, ctx=c3)
print("device-resident phases", [(k, round(v, 2)) for k, v in c3.phases()])
c2 = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
c2.set_async(True)
for _ in range(4):
    sp.friends_of_friends(hp, eps, ctx=c2, out=(hl, hc))
c2.synchronize()
print("async e2e phases (last call)", [(k, round(v, 2)) for k, v in c2.phases()])
