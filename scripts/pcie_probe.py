"""PCIe: H2D alone, D2H alone, both concurrently (pinned buffers, 1.6 GB up / 0.67 GB down)."""
import time, torch
n = 1 << 27
dev = torch.device("cuda", 0)
hp = torch.empty(n * 3, dtype=torch.float32, pin_memory=True)
hl = torch.empty(n * 5 // 4, dtype=torch.int32, pin_memory=True)
dp = torch.empty(n * 3, dtype=torch.float32, device=dev)
dl = torch.empty(n * 5 // 4, dtype=torch.int32, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def timed(f, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e3
def up():
    with torch.cuda.stream(s1): dp.copy_(hp, non_blocking=True)
def down():
    with torch.cuda.stream(s2): hl.copy_(dl, non_blocking=True)
def both():
    up(); down()
for name, f in (("h2d 1.61 GB", up), ("d2h 0.67 GB", down), ("both", both)):
    timed(f, 1)
    print(name, "%.1f ms" % timed(f), flush=True)
