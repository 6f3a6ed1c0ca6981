"""C2 (Bvh::build + range count, 2^24 uniform points queried with ~30-neighbour spheres): event times per phase."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream(dev)
ctx = sp.Context(0, stream=s.cuda_stream)
pts = sp.generate_uniform(n, 3, seed=2409, ctx=ctx)
r = float(np.float32(np.cbrt(30.0 / (n * 4.18879020478639))))
ref = None
for it in range(reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(s)
    b = sp.Bvh.build(pts, ctx=ctx)
    ev[1].record(s)
    c = sp.range_count(b, pts, radius=r)
    ev[2].record(s)
    torch.cuda.synchronize()
    h = torch.as_tensor(c).cpu() if not isinstance(c, np.ndarray) else torch.from_numpy(c)
    if ref is None:
        ref = h.clone()
    print("build %.3f ms  query %.3f ms  mean count %.2f  same %s" % (
        ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), h.double().mean().item(), bool(torch.equal(h, ref))),
        flush=True)
