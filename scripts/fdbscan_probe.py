"""Point-path clustering (FDBSCAN min_pts 5 on the 2^26 field; FoF over points (algorithm="points") on 2^27):
event time and phases per call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream(dev)
ctx = sp.Context(0, stream=s.cuda_stream)
for n, mp in ((1 << 26, 5), (1 << 27, 2)):
    p = sp.generate_field(n, seed=2409, ctx=ctx)
    eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        out = (sp.fdbscan(p, sp.DbscanParams(eps, mp), ctx=ctx) if mp > 2 else
               sp.friends_of_friends(p, eps, ctx=ctx, algorithm="points"))
        e1.record(s)
        torch.cuda.synchronize()
        if it == 2:
            print("n=2^%d min_pts %d: %.2f ms" % (int(np.log2(n)), mp, e0.elapsed_time(e1)),
                  [(k, round(v, 2)) for k, v in ctx.phases()], flush=True)
    del p, out
