import os, sys
sys.path.insert(0, "/root/repo")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29555", RANK="0", WORLD_SIZE="1")
import numpy as np, torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl")
import paper_2409_10743_b200 as sp
from paper_2409_10743_b200 import distributed as spd
ctx = sp.Context(0, stream=torch.cuda.current_stream().cuda_stream) if os.environ.get("TORCH_STREAM") else sp.Context(0)
for n in (1 << 22, 1 << 25, 1 << 27):
    pts = sp.generate_field(n, seed=2409, ctx=ctx)
    eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
    seen = {}
    def local(p, e):
        seen["min"] = p.min(0).values.tolist(); seen["max"] = p.max(0).values.tolist()
        seen["shape"] = tuple(p.shape); seen["stride"] = p.stride(); seen["dtype"] = str(p.dtype)
        out = sp.friends_of_friends(p, e, ctx=ctx)
        seen["cells"] = ctx.counter("fof_cells")
        return out.labels, out.core_flags
    lab, core = spd.fof_slabs(pts, eps, ctx=ctx, local_fof=local)
    print(n, seen, flush=True)
    out = sp.friends_of_friends(pts, eps, ctx=ctx)
    print("  direct cells", ctx.counter("fof_cells"), "equal", bool(torch.equal(out.labels, lab)), flush=True)
dist.destroy_process_group()
