"""FoF on 2^30 (1.07 B) points of the bench field on ONE B200: phases, memory, wall."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
ctx = sp.Context(0)
p = sp.generate_field(n, seed=2409, ctx=ctx)
eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
labels = torch.empty(n, dtype=torch.int32, device="cuda")
core = torch.empty(n, dtype=torch.uint8, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    out = sp.friends_of_friends(p, eps, ctx=ctx, out=(labels, core))
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    free, total = torch.cuda.mem_get_info()
    print("n=%d  %.1f ms  %.3g pts/s  cells %d  free %.1f GB of %.1f" % (n, dt * 1e3, n / dt, ctx.counter("fof_cells"),
          free / 1e9, total / 1e9), [(k, round(v, 1)) for k, v in ctx.phases()], flush=True)
lab = labels
idx = torch.arange(n, device="cuda", dtype=torch.int32)
c = core.bool()
print("noise == non-core:", bool(((lab == -1) == ~c).all()), " labels <= index:", bool((lab[c] <= idx[c]).all()),
      " clusters:", int((lab[c] == idx[c]).sum()), " core:", int(c.sum()))
