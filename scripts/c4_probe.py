"""C4 (kNN k = 16 on 2^24 uniform points, 2^24 uniform queries): event time per nearest_query call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream(dev)
ctx = sp.Context(0, stream=s.cuda_stream)
pts = sp.generate_uniform(n, 3, seed=2409, ctx=ctx)
qs = sp.generate_uniform(n, 3, seed=2410, ctx=ctx)
b = sp.Bvh.build(pts, ctx=ctx)
ts = []
for it in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    idx = sp.nearest_query(b, qs, 16)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    print("knn %.2f ms" % ts[-1], flush=True)
print("knn median %.2f ms min %.2f ms" % (float(np.median(ts[1:] if len(ts) > 1 else ts)), min(ts)), flush=True)
