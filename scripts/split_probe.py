import os, sys, time
sys.path.insert(0, "/root/repo")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29561")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
import paper_2409_10743_b200 as sp
dist.init_process_group("nccl")
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
ctx = sp.Context(0, stream=torch.cuda.current_stream(dev).cuda_stream)
n = 1 << 27
pts = sp.generate_field(n, first=0, count=n, seed=2409, ctx=ctx)
def T(name, f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print("%-12s %8.2f ms" % (name, (time.perf_counter() - t) * 1e3), flush=True); return r
for it in range(3):
    x = pts[:, 0]
    stride = max(1, n // (1 << 20))
    xs = T("sample+sort", lambda: torch.sort(x[::stride].double()).values)
    q = torch.linspace(0, 1, 1024, device=dev, dtype=torch.float64)
    lq = T("quantiles", lambda: xs[(q * (xs.numel() - 1)).round().long()])
    allq = [torch.empty_like(lq)]
    T("all_gather", lambda: dist.all_gather(allq, lq))
    a = T("cat+mask+sort", lambda: torch.sort(torch.cat(allq)[~torch.isnan(torch.cat(allq))]).values)
    g = T("arange gidx", lambda: torch.arange(0, n, dtype=torch.int64, device=dev))
dist.destroy_process_group()
