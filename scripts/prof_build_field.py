"""Run Bvh::build on the reference generator's H(n) field (for ncu captures): prof_build_field.py N REPS."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = sp.Context(0)
h = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
sp.generate_reference_field(n, 0, n, out=h)
p = h.cuda()
for _ in range(reps):
    b = sp.Bvh.build(p, ctx=ctx)
    del b
print(ctx.phases())
