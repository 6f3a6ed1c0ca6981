"""Probe: asynchronous FoF steps on H(2^27) with host input and/or host outputs
(which copy direction limits the end-to-end step)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = 1 << 27
dev = torch.device("cuda", 0)
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
sp.generate_reference_field(n, 0, n, out=hp)
dp = hp.to(dev)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
hl, hc = torch.empty(n, dtype=torch.int32, pin_memory=True), torch.empty(n, dtype=torch.uint8, pin_memory=True)
dl, dc = torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)
steps = 8
for name, src, out in (("device", dp, (dl, dc)), ("h2d + d2h", hp, (hl, hc))):
    c = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
    sp.friends_of_friends(src, eps, ctx=c, out=out)
    c.set_async(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        sp.friends_of_friends(src, eps, ctx=c, out=out)
    c.synchronize()
    torch.cuda.synchronize()
    print("%-10s %.1f ms/step" % (name, (time.perf_counter() - t) / steps * 1e3), flush=True)
    c.set_async(False)
    c.close()
t = time.perf_counter(); x = hp.to(dev); torch.cuda.synchronize(); print("h2d alone %.1f ms" % ((time.perf_counter() - t) * 1e3))
t = time.perf_counter(); hl.copy_(dl); hc.copy_(dc); torch.cuda.synchronize(); print("d2h alone %.1f ms" % ((time.perf_counter() - t) * 1e3))
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1):
    x.copy_(hp, non_blocking=True)
with torch.cuda.stream(s2):
    hl.copy_(dl, non_blocking=True); hc.copy_(dc, non_blocking=True)
torch.cuda.synchronize(); print("h2d || d2h %.1f ms" % ((time.perf_counter() - t) * 1e3))
# H2D of one input while the device-resident pipeline runs on another stream
c = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)
cs = torch.cuda.Stream(dev)
sp.friends_of_friends(dp, eps, ctx=c, out=(dl, dc))
c.set_async(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    sp.friends_of_friends(dp, eps, ctx=c, out=(dl, dc))
with torch.cuda.stream(cs):
    e0.record(cs); x.copy_(hp, non_blocking=True); e1.record(cs)
c.synchronize(); torch.cuda.synchronize()
print("h2d under load %.1f ms" % e0.elapsed_time(e1))
