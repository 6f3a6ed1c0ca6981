"""1.07 B-point FoF on one B200: the grid-cell pipeline against the point
pipeline (pair traversal over the point LBVH, algorithm="points") on the same
input — two independent algorithms must give bit-identical labels and core
flags.  (The CPU reference cannot run at this size here: ~165 GB of RAM.)"""
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
res = {}
for mode in ("cells", "points"):
    torch.cuda.synchronize(); t = time.perf_counter()
    sp.friends_of_friends(p, eps, ctx=ctx, out=(labels, core), algorithm=mode)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    res[mode] = (labels.cpu().numpy(), core.cpu().numpy())
    print(mode, "%.1f ms" % (dt * 1e3), [(k, round(v, 1)) for k, v in ctx.phases()], flush=True)
same = np.array_equal(res["cells"][0], res["points"][0]) and np.array_equal(res["cells"][1], res["points"][1])
lab, core = res["cells"]
print("n=%d eps=%r: labels and core flags identical between the two pipelines: %s; clusters %d, core %d, noise %d"
      % (n, eps, same, int((lab[core.astype(bool)] == np.arange(n, dtype=np.int32)[core.astype(bool)]).sum()),
         int(core.sum()), int((lab == -1).sum())))
