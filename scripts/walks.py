import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
b = sp.Bvh.build(p, ctx=ctx)
steps = torch.empty(n, dtype=torch.int32, device="cuda"); hits = torch.empty_like(steps)
lib = sp._lib
lib.sp_debug_walk_lengths.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_int]
ctx._check(lib.sp_debug_walk_lengths(ctx.h, b.h, C.c_float(eps), C.c_void_p(steps.data_ptr()), C.c_void_p(hits.data_ptr()), 1))
s = steps.cpu().numpy().astype(np.int64); h = hits.cpu().numpy()
print("n", n, "mean steps", s.mean(), "mean pairs", h.mean(), "p50/p90/p99/max", np.percentile(s, [50, 90, 99]), s.max())
w = s[: (n // 32) * 32].reshape(-1, 32)
print("warp max/mean ratio (lane efficiency bound):", w.mean() / w.max(axis=1).mean())
for lo, hi in [(0, n // 4), (n // 4, n)]:
    print("segment", lo, hi, "mean steps", s[lo:hi].mean() if False else None)
bg = None
