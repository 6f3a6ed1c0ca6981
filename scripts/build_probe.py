"""Bvh::build phase times (bounds, morton, sort, hierarchy) on uniform points."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
ctx = sp.Context(0)
for n in (1 << 24, 1 << 27):
    p = sp.generate_uniform(n, 3, seed=2409, ctx=ctx)
    for it in range(3):
        b = sp.Bvh.build(p, ctx=ctx)
        ph = ctx.phases()
        tot = sum(v for _, v in ph)
        if it == 2:
            print("n=2^%d" % int(np.log2(n)), "build %.3f ms" % tot, [(k, round(v, 3)) for k, v in ph],
                  "-> %.0f Mpts/s, %.1f%% of HBM at 368 B/pt" % (n / tot / 1e3, 368 * n / (tot / 1e3) / 6548.5e9 * 100),
                  flush=True)
        del b
    del p
# the clustered field H(2^27) (the bench's bvh_build input)
n = 1 << 27
h = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
sp.generate_reference_field(n, 0, n, out=h)  # the bench's H(2^27) (reference generator)
p = h.cuda()
for it in range(3):
    b = sp.Bvh.build(p, ctx=ctx)
    ph = ctx.phases()
    tot = sum(v for _, v in ph)
    if it == 2:
        print("field n=2^27 build %.3f ms" % tot, [(k, round(v, 3)) for k, v in ph], flush=True)
    del b
