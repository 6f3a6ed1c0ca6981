"""C3 (DenseBox min_pts=5 on the 2^26 field): phase marks, stream-event and wall time per call."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_10743_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
mp = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
for kind in ("torch-stream", "own-stream"):
    ctx = sp.Context(0, stream=torch.cuda.current_stream(dev).cuda_stream) if kind == "torch-stream" else sp.Context(0)
    p = sp.generate_field(n, seed=2409, ctx=ctx)
    eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
    for it in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream(dev)
        t = time.perf_counter()
        a.record(s)
        out = sp.fdbscan_densebox(p, sp.DbscanParams(eps, mp), ctx=ctx)
        b.record(s)
        torch.cuda.synchronize()
        w = (time.perf_counter() - t) * 1e3
        print(kind, "wall %.1f ms, events %.1f ms" % (w, a.elapsed_time(b)), [(k, round(v, 2)) for k, v in ctx.phases()],
              out.stats, flush=True)
# back-to-back calls without host synchronisation (as bench.py times them)
ctx = sp.Context(0, stream=torch.cuda.current_stream(dev).cuda_stream)
s = torch.cuda.current_stream(dev)
for it in range(2):
    ev = []
    for k in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        out = sp.fdbscan_densebox(p, sp.DbscanParams(eps, mp), ctx=ctx)
        b.record(s)
        ev.append((a, b, [(k2, round(v, 2)) for k2, v in ctx.phases()]))
    torch.cuda.synchronize()
    for a, b, ph in ev:
        print("nosync events %.1f ms" % a.elapsed_time(b), ph, flush=True)
