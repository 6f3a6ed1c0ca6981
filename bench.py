#!/usr/bin/env python
"""Benchmark for the B200 FoF/DBSCAN hot path (BASELINE.json metric:
"FoF/DBSCAN points/sec at 1/2/4/8 B200 + % HBM roofline; BVH build Mpts/s").

Default workload ("fof_field", SURVEY §8(d) C5 shape, weak scaling):
friends-of-friends (DBSCAN minPts = 2) on the SURVEY field H(n_total) — 25%
uniform background + Gaussian halos of 8192 points, sigma =
0.001*cbrt(2^26/n), drawn by the reference's own generator (generate.cpp,
bit-identical host restatement) — with 2^27 points per GPU (the per-GPU share
of the C5 1-billion-point run on 8 GPUs), eps = 0.168 * mean spacing of the
whole field.  Before timing, the labels are checked against the unmodified
reference's labels on the same input (tests/golden/golden_hashes.json
"H_2^k", pinned by scripts/ref_pin*.py) where a pin exists.
One step = one full pass of the path: scene bounds, Morton codes, radix sort,
hierarchy + refit + ropes, pair traversal fused with union-find, label
finalisation (N > 1 adds the slab exchange and the distributed merge).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload fof_field|c1|c2|c3|c4] [--n POINTS_PER_GPU]

`value` is device-resident throughput (inputs already in HBM); `e2e` is the
same call through the public API with pinned HOST buffers (H2D of the points
and D2H of labels + core flags inside the timed region).  The reference arm
(--impl reference) times the unmodified reference CPU implementation
(oracle/_ref, built from /root/reference) on a bounded sample on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FALLBACK_GBS = 6650.0
ARBORX_A100_PTS_S = 37.0e6 / 0.15  # ~37M HACC particles FoF in < 0.15 s on one A100


def eps_for(n: int) -> float:
    import numpy as np
    return float(np.float32(0.168 * np.cbrt(1.0 / float(n))))


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden_hashes.json")) as f:
        return json.load(f)


def labels_checksum(labels, first: int) -> int:
    """sum((label + 1) * (i % 65521 + 1)) mod 2^63 over rows i = first.. of a
    device label tensor (the reference-side value comes from
    oracle/_ref's ref_fof_field / scripts/ref_pin.py)."""
    import torch
    total, chunk = 0, 1 << 24  # chunked: int64 temporaries of 2^30 labels would need 8.6 GB each
    for s in range(0, labels.numel(), chunk):
        part = labels[s:s + chunk]
        i = torch.arange(first + s, first + s + part.numel(), dtype=torch.int64, device=labels.device)
        total += int(((part.to(torch.int64) + 1) * (i % 65521 + 1)).sum().item())
    total &= (1 << 64) - 1  # int64 wrap-around, as one device-wide sum would give
    return total - (1 << 64) if total >= 1 << 63 else total


def reference_field_pinned(n_total: int, first: int, count: int):
    """Rows [first, first+count) of H(n_total) from the reference generator,
    in pinned host memory (the e2e leg's host input)."""
    import torch
    import paper_2409_10743_b200 as sp
    host = torch.empty((count, 3), dtype=torch.float32, pin_memory=True)
    sp.generate_reference_field(n_total, first, count, out=host)
    return host


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# per-kernel algorithmic bytes for the FoF pipeline phases
# ---------------------------------------------------------------------------
def phase_bytes(phase: str, n: int, cells: int, key_bits: int) -> float:
    """Algorithmic bytes of one FoF step's phases: n points,
    `cells` non-empty grid cells, `key_bits` cell-key bits (8-bit digits)."""
    npass = (key_bits + 7) // 8
    f = cells / float(n)
    per = {
        "bounds": 12.0,                                   # read xyz
        "morton": 12.0 + 8.0,                             # read xyz, write cell key
        "sort": 8.0 + 20.0 + 24.0 * (npass - 1),          # histogram read; pass 0 (iota values); 12 B in+out/pass
        # gather sorted points (perm 4 + xyz 12 + write 16), cell heads (keys 8 + write 4), scan (4 + 8),
        # cell ranges (points 16 + cell_of 4) + per cell: key 8 + box 24 + starts 8 + hierarchy 140
        "hierarchy": 4 + 12 + 16 + 12 + 12 + 20 + (8 + 24 + 8 + 140) * f,
        # cell tree read once (2 nodes x 32 B per cell), member points 16 B, parent 4 B per cell
        "merge": 16.0 + (64.0 + 4.0) * f,
        # cell core flags, per point: cell_of 4 + point 16 + min-index atomics 4 + labels 4 + core 1 + root 4
        "finalize": 33.0 + 12.0 * f,
    }
    return per.get(phase, 0.0) * n


PROFILED = {"merge": "merge_cells_2p27", "sort": "sort_cells_2p27", "hierarchy": "hier_cells_2p27"}


def profiled_traffic(phase: str, n: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's
    kernel from the committed ncu --set full capture (profiles/r02), for the
    headline size only; None otherwise."""
    if n != (1 << 27) or phase not in PROFILED:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", PROFILED[phase] + ".summary.json")) as f:
            d = json.load(f)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for key in ("dram read", "dram write"):
            v, u = d[key].split()
            tot += float(v) * scale[u]
        return tot
    except Exception:
        return None


def profiled_l1(phase: str, n: int):
    """l1tex__throughput (fraction of peak) of the phase's kernel from the
    committed capture (profiles/r02), headline size only; None otherwise."""
    if n != (1 << 27) or phase not in PROFILED:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", PROFILED[phase] + ".summary.json")) as f:
            d = json.load(f)
        return round(float(d["L1 throughput % of peak"].split()[0]) / 100.0, 3)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref) — the cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------
def reference_sample(n_sample: int, runs: int, warmup: int = 0):
    """Time the reference's friends_of_friends on H(n_sample) (the reference's
    own generator); returns (points/s, kind, cores, per-run seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference  # test infrastructure: checker/baseline only
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    if Reference.available():
        R, kind = Reference.get(), "reference"
        pts = R.field(n_sample)
        run = lambda: R.dbscan(pts, 3, eps_for(n_sample), 2, "fof")
    else:
        O, kind = Oracle.get(), "port"
        pts = O.field(n_sample)
        run = lambda: O.dbscan(pts, 3, eps_for(n_sample), 2)
    for _ in range(warmup):
        run()
    secs = []
    for _ in range(runs):
        t = time.perf_counter()
        run()
        secs.append(time.perf_counter() - t)
    return n_sample / statistics.median(secs), kind, cores, secs


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    n_sample = args.cpu_sample_n
    v, kind, cores, secs = reference_sample(n_sample, args.steps, args.warmup)
    cfg = {"workload": "fof_field SAMPLE: friends_of_friends on H(%d) (the same field shape at %d points; the "
                       "2^27-point per-GPU workload takes ~56 s per run on this host's CPU, "
                       "profiles/r02/ref_pin.json)" % (n_sample, n_sample),
           "points_per_gpu": n_sample, "points_total": n_sample, "eps": eps_for(n_sample), "min_pts": 2,
           "parallelism": "reference CPU (OpenMP, %d host threads)" % cores,
           "sample_of": workload_config(args, world)["workload"]}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (reference generator H(n))",
        "config": cfg,
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores, "kind": kind,
                         "sample": "friends_of_friends on H(%d) (SURVEY §8(d) field, reference mt19937_64 generator), "
                                   "eps = 0.168*n^(-1/3); %d timed runs" % (n_sample, args.steps)},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "FoF/DBSCAN points/sec (friends-of-friends, minPts=2)"


def workload_config(args, world):
    n = args.n
    return {"workload": "fof_field: friends_of_friends on HACC-like clustered 3D fp32 field, "
                        "%d points per GPU (C5 per-GPU share), eps = 0.168*n_total^(-1/3)" % n,
            "points_per_gpu": n, "points_total": n * world, "eps": eps_for(n * world), "min_pts": 2,
            "parallelism": "x-slabs over %d GPU(s) with eps ghost layers" % world if (world > 1 or args.slabs) else "single GPU",
            "input": "H(%d) rows of this rank, reference generator" % (n * world),
            "l2": "inputs (%.1f GB) larger than L2 (126 MB); no flush needed" % (n * 12 / 1e9)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2409_10743_b200 as sp

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.Context(local_rank, stream=stream.cuda_stream)

    n = args.n
    n_total = n * world
    eps = eps_for(n_total)
    slabs = world > 1 or args.slabs
    # this rank's rows of H(n_total), reference generator, pinned host memory
    host_pts = reference_field_pinned(n_total, rank * n, n)
    pts = host_pts.to(dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    core = torch.empty(n, dtype=torch.uint8, device=dev)
    if slabs:
        from paper_2409_10743_b200 import distributed as spd
        comm = spd.SlabComm.from_process_group(ctx)

        def step():
            spd.fof_slabs(pts, eps, first_index=rank * n, ctx=ctx, comm=comm, out=(labels, core))
    else:
        step = lambda: sp.friends_of_friends(pts, eps, ctx=ctx, out=(labels, core))

    def barrier():
        if slabs:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    # parity before timing: the labels of this input against the unmodified
    # reference's (oracle/_ref friends_of_friends on the same H(n_total))
    torch.cuda.synchronize(dev)
    ck = torch.tensor([labels_checksum(labels, rank * n), int((labels == -1).sum()), int(core.sum()),
                       int((labels == torch.arange(rank * n, rank * n + n, device=dev, dtype=torch.int32)).sum())],
                      dtype=torch.int64, device=dev)
    if slabs:
        dist.all_reduce(ck)
    ck = [int(v) for v in ck.tolist()]
    pin = golden().get("H_2^%d" % (n_total.bit_length() - 1)) if n_total & (n_total - 1) == 0 else None
    parity = {"checked_against": None, "labels_checksum": ck[0] & ((1 << 63) - 1), "noise": ck[1], "core": ck[2],
              "clusters": ck[3]}
    if pin is not None:
        parity["checked_against"] = "oracle/_ref friends_of_friends on H(%d) (%s)" % (n_total, pin["labels_hash"])
        parity["match"] = (parity["labels_checksum"] == pin["labels_checksum"] and ck[1] == pin["noise"] and
                           ck[2] == pin["core"] and ck[3] == pin["clusters"])
        if not parity["match"]:
            raise SystemExit("PARITY FAILURE against the reference on H(%d): %s vs %s" % (n_total, parity, pin))
    # node-visit rate of the merge: one diagnostic pass (SP_FLAG_STATS)
    # counts the visits and member-pair tests of the same walks, untimed
    visits = tests = None
    if not slabs:
        ctx.set_stats(True)
        step()
        visits, tests = ctx.counter("merge_node_visits"), ctx.counter("merge_pair_tests")
        ctx.set_stats(False)
        step()
    # workload statistics for the byte models, outside timing: non-empty grid
    # cells of the FoF pipeline, their key width, and close pairs per point
    cells = ctx.counter("fof_cells")
    key_bits = 3 * max(1, int(np.ceil(np.log2(1.0 / (eps / np.sqrt(3.0) * (1 - 1e-6)) + 1))))
    pairs_per_pt = None
    bvh_build = None
    if not slabs:
        b = sp.Bvh.build(pts, ctx=ctx)
        import ctypes
        tot = ctypes.c_int64(0)
        ctx._check(sp._lib.sp_pair_list(ctx.h, b.h, ctypes.c_float(eps), None, 0, ctypes.byref(tot), sp.SP_MEM_DEVICE))
        pairs_per_pt = tot.value / n
        del b
        # Bvh::build over the same points (the BASELINE "BVH build Mpts/s"),
        # separately timed: 3 warm builds, events on the context stream
        bt = []
        for _ in range(4):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            b = sp.Bvh.build(pts, ctx=ctx)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            bt.append(a0.elapsed_time(a1))
            del b
        bms = statistics.median(bt[1:])
        peak_b, _ = measured_peak()
        bvh_build = {"ms": round(bms, 3), "mpts_s": n / (bms / 1e3) / 1e6,
                     "hbm_frac": round(368.0 * n / (bms / 1e3) / (peak_b * 1e9), 4),
                     "bytes_model": "368 B/point (SURVEY 8(d): bounds 12 + Morton 24 + sort 192 + hierarchy 140)"}

    # ---- device-resident timed region ----
    phase_acc = {}
    barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = ctx.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out = step()
        for name, ms in ctx.phases():
            phase_acc[name] = phase_acc.get(name, 0.0) + ms
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = ctx.kernel_launches - launches0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if slabs:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)

    # ---- end-to-end through the public API with pinned host buffers ----
    e2e_value = None
    h2d = n * 12
    d2h = n * 5
    if not slabs:
        # Public API with pinned HOST buffers: every step uploads its points
        # and downloads its labels + core flags.  The context runs with
        # SP_FLAG_ASYNC: uploads/downloads go on its copy streams, so step
        # i+1's upload and step i-1's download overlap step i's kernels
        # (include/sp_b200.h).
        cstream = torch.cuda.Stream(dev)
        ectx = sp.Context(local_rank, stream=cstream.cuda_stream)
        host_labels = torch.empty(n, dtype=torch.int32, pin_memory=True)
        host_core = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        sp.friends_of_friends(host_pts, eps, ctx=ectx, out=(host_labels, host_core))  # warm
        ectx.set_async(True)
        # warm-up in the timed mode: both staging parities (the context
        # double-buffers host transfers and allocates each slot on first use)
        for _ in range(max(1, args.warmup - 1)):
            sp.friends_of_friends(host_pts, eps, ctx=ectx, out=(host_labels, host_core))
        ectx.synchronize()
        barrier()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(cstream)
        for i in range(args.steps):
            sp.friends_of_friends(host_pts, eps, ctx=ectx, out=(host_labels, host_core))
        ectx.synchronize()  # waits for the compute and both copy streams
        e_end.record(cstream)
        barrier()
        e2e_value = n_total * args.steps / (e_start.elapsed_time(e_end) / 1e3)
        ectx.set_async(False)
        # the host run must agree bit-for-bit with the device-resident run
        assert torch.equal(host_labels, labels.cpu()) and torch.equal(host_core, core.cpu()), "e2e != device run"
    else:
        # each rank uploads its pinned host slice, runs the slab FoF over NCCL
        # and downloads its labels + core flags, copies inside the timed region
        # (SP_FLAG_ASYNC as in the single-GPU leg: step i+1's upload overlaps
        # step i's compute after its one host read of the exchange sizes)
        host_labels = torch.empty(n, dtype=torch.int32, pin_memory=True)
        host_core = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        cstream = torch.cuda.Stream(dev)
        ectx = sp.Context(local_rank, stream=cstream.cuda_stream)

        def e2e_step():
            spd.fof_slabs(host_pts, eps, first_index=rank * n, ctx=ectx, comm=comm, out=(host_labels, host_core))

        e2e_step()
        ectx.set_async(True)
        for _ in range(max(1, args.warmup - 1)):
            e2e_step()
        ectx.synchronize()
        barrier()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(cstream)
        for _ in range(args.steps):
            e2e_step()
        ectx.synchronize()
        e_end.record(cstream)
        barrier()
        ectx.set_async(False)
        t = torch.tensor([e_start.elapsed_time(e_end)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_value = n_total * args.steps / (float(t.item()) / 1e3)

    peak, peak_src = measured_peak()
    phases = {k: v / args.steps for k, v in phase_acc.items()}
    roofline = None
    if phases:
        dom = max(phases, key=phases.get)
        ach_bytes = phase_bytes(dom, n, max(cells, 1), key_bits)
        ach = ach_bytes / (phases[dom] / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": profiled_traffic(dom, n), "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": ach_bytes, "kernel_ms": round(phases[dom], 3),
                    "share_of_step": round(phases[dom] / ms_per_step, 3)}
        l1 = profiled_l1(dom, n)
        if l1 is not None:
            # the traversal kernels are bound by the L1 (load wavefronts of
            # L1-hot node reads), not by HBM: ncu's l1tex throughput of the
            # committed capture of this kernel, as a fraction of its peak
            roofline["l1_throughput_frac"] = l1
        build_ms = sum(phases.get(k, 0.0) for k in ("bounds", "morton", "sort", "hierarchy"))
    else:
        build_ms = None

    merge_ms = phases.get("merge")
    visit_rate = None
    if visits and merge_ms:
        visit_rate = {"merge_node_visits_per_step": visits, "merge_pair_tests_per_step": tests,
                      "visits_per_cell": round(visits / max(cells, 1), 2),
                      "node_visits_per_s": visits / (merge_ms / 1e3),
                      "how": "one untimed SP_FLAG_STATS pass of the same walks; rate = visits / timed merge ms"}

    if rank != 0:
        return
    # free this run's device memory before the extra configs (C5 at 2^30 needs
    # ~146 GB) run in their own processes
    del pts, labels, core
    ectx.close()
    ctx.close()
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    extra = {}
    if world == 1 and not args.no_extra:
        for w, steps in (("c3", 5), ("c5", 3)):
            extra[w] = run_extra(w, steps)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, kind, cores, secs = reference_sample(args.cpu_sample_n, 2, 0)
        full = golden().get("H_2^%d" % (n_total.bit_length() - 1), {})
        cpu = {"value": v, "unit": "points/s", "cores": cores, "kind": kind,
               "sample": "friends_of_friends on H(%d) (same field shape, reference generator), %d runs, "
                         "median %.2f s" % (args.cpu_sample_n, len(secs), statistics.median(secs)),
               "full_size": ({"n": full["n"], "seconds": full["ref_seconds"],
                              "points_per_s": full["n"] / full["ref_seconds"], "threads": full.get("threads"),
                              "source": "oracle/_ref on the GPU host, profiles/r02/ref_pin.json (one run)"}
                             if full.get("ref_seconds") else None)}
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / ARBORX_A100_PTS_S,
        "vs_baseline_ref": "ArborX on 1x A100: ~37M HACC particles FoF in < 0.15 s (PAPER.md:489-493) = %.3g "
                           "points/s; a bound on a different (real HACC) dataset, not a like-for-like ratio"
                           % ARBORX_A100_PTS_S,
        "dtype": "f32 (exact f64 distance predicate)",
        "data": "synthetic: the SURVEY field H(n) from the reference generator (generate.cpp:17-66)",
        "config": workload_config(args, world),
        "parity": parity,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world},
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "bvh_build_mpts_s": bvh_build["mpts_s"] if bvh_build else None,
        "bvh_build": bvh_build,
        "fof_grid_build_mpts_s": (n / (build_ms / 1e3) / 1e6) if build_ms else None,
        "phases_ms": {k: round(v, 3) for k, v in phases.items()},
        "close_pairs_per_point": pairs_per_pt,
        "fof_cells": cells,
        "merge_visits": visit_rate,
        "configs": extra or None,
    }
    print(json.dumps(line), flush=True)


def run_extra(w: str, steps: int) -> dict:
    """One other SURVEY §8(d) config in its own process (bench.py --workload),
    reduced to the keys the headline line carries."""
    cmd = [sys.executable, os.path.abspath(__file__), "--workload", w, "--steps", str(steps), "--warmup", "1",
           "--no-cpu-baseline"]
    err = ""
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        err = r.stderr.strip()[-300:]
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal: the headline stands on its own
        return {"error": "%s: %s" % (type(e).__name__, str(e)[:200]), "stderr": err}
    keep = ("metric", "value", "unit", "ms_per_step", "steps", "parts_ms", "parity", "e2e", "gpu_launches", "clocks")
    out = {k: d.get(k) for k in keep}
    out["workload"] = d.get("config", {}).get("workload")
    return out


# ---------------------------------------------------------------------------
# the other BASELINE configs; same JSON contract, one line each
# ---------------------------------------------------------------------------
CONFIGS = {
    # name: (points, description)
    "c1": (1000000, "C1: friends_of_friends on 10^6 uniform points, eps = 0.168*n^(-1/3)"),
    "c2": (1 << 24, "C2: Bvh::build + sort_queries + range count, 2^24 uniform points, 2^24 sphere queries "
                    "centred on them, r = cbrt(30/(n*4pi/3)) (~30.7 neighbours)"),
    "c3": (1 << 26, "C3: fdbscan_densebox min_pts = 5 on the 2^26-point clustered field, eps = 0.168*n^(-1/3)"),
    "c4": (1 << 24, "C4: Bvh::build + nearest_query k = 16, 2^24 uniform points, 2^24 uniform queries"),
    "c5": (1 << 30, "C5 on ONE GPU: friends_of_friends on the 2^30-point (1.07 B) HACC-like clustered field, "
                    "eps = 0.168*n^(-1/3)"),
}


def config_parity(sp, w, n, pts, qs, eps, r2, ctx) -> dict:
    """The config's result on its reference-generator input against the
    unmodified reference's (tests/golden/golden_hashes.json: SURVEY §8(c) and
    the scripts/ref_pin*.py pins), before timing.  Counts and checksums on the
    device; the FNV hashes are checked by tests/ (-m gpu)."""
    import torch
    g = golden()
    key = {"c1": "C1", "c2": "C2", "c3": "C3", "c4": "C4"}.get(w, "H_2^%d" % (n.bit_length() - 1))
    pin = g.get(key) if (w != "c5" or n & (n - 1) == 0) else None
    if pin is None or pin.get("n") != n:
        return {"checked_against": None}
    got = {}
    if w in ("c1", "c3", "c5"):
        out = (sp.fdbscan_densebox(pts, sp.DbscanParams(eps, 5), ctx=ctx) if w == "c3" else
               sp.friends_of_friends(pts, eps, ctx=ctx))
        lab, core = out.labels, out.core_flags
        got = {"noise": 0, "core": 0, "clusters": 0}
        for s in range(0, n, 1 << 24):  # chunked: 2^30-row temporaries do not fit next to the pipeline
            lb, cr = lab[s:s + (1 << 24)], core[s:s + (1 << 24)]
            idx = torch.arange(s, s + lb.numel(), device=lab.device, dtype=torch.int32)
            got["noise"] += int((lb == -1).sum())
            got["core"] += int(cr.sum(dtype=torch.int64))
            got["clusters"] += int((lb == idx).sum())
        if w == "c3":  # min_pts > 2 labels are not unique; the core partition is
            got["clusters"] = int(torch.unique(lab[core.bool()]).numel())
        if w == "c5":
            got["labels_checksum"] = labels_checksum(lab, 0) & ((1 << 63) - 1)
        del out, lab, core
    elif w == "c2":
        got = {"total_matches": int(sp.range_count(sp.Bvh.build(pts, ctx=ctx), qs, radius=r2).to(torch.int64).sum())}
    else:
        _, d = sp.nearest_query(sp.Bvh.build(pts, ctx=ctx), qs, 16, with_distances=True)
        got = {"mean_16th_dist": float(d[:, 15].double().mean())}
    ok = True
    for k, v in got.items():
        ok &= (abs(v - pin[k]) < 1e-9) if isinstance(v, float) else (v == pin[k])
    if not ok:
        raise SystemExit("PARITY FAILURE (%s) against %s: %s vs %s" % (w, key, got, pin))
    return {"checked_against": "oracle/_ref (%s)" % key, "match": True, **got}


def run_config(args):
    import numpy as np
    import torch
    import paper_2409_10743_b200 as sp

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.Context(0, stream=stream.cuda_stream)
    w = args.workload
    n = args.n if args.n != (1 << 27) else CONFIGS[w][0]
    # SURVEY §8(d) inputs from the reference generator: U(n, 2409) (C1, C2,
    # C4 points), U(n, 2410) (C4 queries), H(n) (C3, C5); pinned host copies
    # are the e2e leg's inputs

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
        t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return t

    if w in ("c1", "c2", "c4"):
        host_pts = pinned(sp.generate_reference_uniform(n, 3, 1.0, 2409))
    else:
        host_pts = reference_field_pinned(n, 0, n)
    host_qs = pinned(sp.generate_reference_uniform(n, 3, 1.0, 2410)) if w == "c4" else host_pts
    pts = host_pts.to(dev)
    qs = host_qs.to(dev) if w == "c4" else pts
    eps = eps_for(n)
    r2 = float(np.float32(np.cbrt(30.0 / (n * 4.18879020478639))))
    times = {}

    def timed(name, fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = fn()
        b.record(stream)
        times.setdefault(name, []).append((a, b))
        return out

    if w in ("c1", "c5"):
        if w == "c5":  # outputs preallocated: 5.4 GB per call
            lab_d = torch.empty(n, dtype=torch.int32, device=dev)
            core_d = torch.empty(n, dtype=torch.uint8, device=dev)
            step = lambda: timed("fof", lambda: sp.friends_of_friends(pts, eps, ctx=ctx, out=(lab_d, core_d)))
        else:
            step = lambda: timed("fof", lambda: sp.friends_of_friends(pts, eps, ctx=ctx))
        unit, per_step = "points/s", n
    elif w == "c3":
        step = lambda: timed("densebox", lambda: sp.fdbscan_densebox(pts, sp.DbscanParams(eps, 5), ctx=ctx))
        unit, per_step = "points/s", n
    elif w == "c2":
        def step():
            b = timed("build", lambda: sp.Bvh.build(pts, ctx=ctx))
            timed("query", lambda: sp.range_count(b, qs, radius=r2))
        unit, per_step = "queries/s", n
    else:
        def step():
            b = timed("build", lambda: sp.Bvh.build(pts, ctx=ctx))
            timed("query", lambda: sp.nearest_query(b, qs, 16))
        unit, per_step = "queries/s", n
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    times.clear()
    parity = config_parity(sp, w, n, pts, qs, eps, r2, ctx)
    sampler = ClockSampler(0)
    sampler.start()
    launches0 = ctx.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    launches = ctx.kernel_launches - launches0
    ms = e0.elapsed_time(e1)
    parts = {k: sum(a.elapsed_time(b) for a, b in v) / args.steps for k, v in times.items()}

    # e2e: the same calls with pinned host inputs and outputs.  The clustering
    # workloads run asynchronously (SP_FLAG_ASYNC: the next call's upload and
    # the previous call's download overlap the kernels, as in the headline);
    # build + query workloads are synchronous calls.
    clustering = w in ("c1", "c3", "c5")
    # reusable pinned result buffers, as a serving loop would hold them
    h_counts = torch.empty(n, dtype=torch.int32, pin_memory=True) if w == "c2" else None
    h_knn = torch.empty((n, 16), dtype=torch.int32, pin_memory=True) if w == "c4" else None
    if w == "c5":
        # 2^30 points: the device-resident leg's buffers and its context's
        # cached scratch (~110 GB) make room for the e2e leg's double-buffered
        # staging (inputs 12.9 GB and outputs 5.4 GB per slot)
        del step, pts, qs, lab_d, core_d
        ctx.close()
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
    if clustering:
        h_lab = torch.empty(n, dtype=torch.int32, pin_memory=True)
        h_core = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        ectx = sp.Context(0, stream=torch.cuda.Stream(dev).cuda_stream)

        def e2e_call():
            if w == "c3":
                sp.fdbscan_densebox(host_pts, sp.DbscanParams(eps, 5), ctx=ectx, out=(h_lab, h_core))
            else:
                sp.friends_of_friends(host_pts, eps, ctx=ectx, out=(h_lab, h_core))

        e2e_call()  # warm (synchronous)
        ectx.set_async(True)
        e2e_call()  # warm the other staging parity (its device slots are allocated on first use)
        ectx.synchronize()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if clustering:
            e2e_call()
        elif w == "c2":
            sp.range_count(sp.Bvh.build(host_pts, ctx=ctx), host_qs, radius=r2, out=h_counts)
        else:
            sp.nearest_query(sp.Bvh.build(host_pts, ctx=ctx), host_qs, 16, out=h_knn)
    if clustering:
        ectx.synchronize()
        ectx.set_async(False)
    torch.cuda.synchronize(dev)
    e2e = per_step * args.steps / (time.perf_counter() - t0)
    h2d = n * 12 * (2 if w == "c4" else 1)
    d2h = {"c1": n * 5, "c3": n * 5, "c5": n * 5, "c2": n * 4, "c4": n * 16 * 4}[w]

    cpu = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import Reference  # the reference CPU path (baseline only)
        if Reference.available():
            R = Reference.get()
            if w == "c5":
                sample = 1 << 22
                p = R.field(sample)
                t = time.perf_counter(); R.dbscan(p, 3, eps_for(sample), 2, "fof"); dt = time.perf_counter() - t
            elif w == "c1":
                sample = 1000000
                p = R.uniform(sample, 3, 1.0, 2409)
                t = time.perf_counter(); R.dbscan(p, 3, eps_for(sample), 2, "fof"); dt = time.perf_counter() - t
            elif w == "c3":
                sample = 1 << 21
                p = R.field(sample)
                t = time.perf_counter(); R.dbscan(p, 3, eps_for(sample), 5, "densebox"); dt = time.perf_counter() - t
            elif w == "c2":
                sample = 1 << 20
                p = R.uniform(sample, 3, 1.0, 2409)
                rr = float(np.float32(np.cbrt(30.0 / (sample * 4.18879020478639))))
                t = time.perf_counter(); R.range_count(p, p, rr); dt = time.perf_counter() - t
            else:
                sample = 1 << 20
                p = R.uniform(sample, 3, 1.0, 2409)
                q = R.uniform(sample, 3, 1.0, 2410)
                t = time.perf_counter(); R.knn(p, q, 16); dt = time.perf_counter() - t
            cpu = {"value": sample / dt, "unit": unit, "cores": os.cpu_count(), "kind": "reference",
                   "sample": "%s at n = %d (reference generator), one run, %.2f s" % (w, sample, dt)}
    line = {
        "metric": {"c1": METRIC, "c5": METRIC, "c3": "FDBSCAN-DenseBox points/sec (min_pts=5)",
                   "c2": "BVH build + range-count queries/sec", "c4": "BVH build + kNN (k=16) queries/sec"}[w],
        "value": per_step * args.steps / (ms / 1e3), "unit": unit, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (exact f64 distance predicate)", "data": "synthetic (device Philox)",
        "config": {"workload": CONFIGS[w][1], "points": n,
                   "l2": "inputs larger than L2" if n * 12 > 126e6 else "inputs smaller than L2 (C1 as specified)"},
        "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": ("asynchronous calls (SP_FLAG_ASYNC) with pinned host buffers" if w in ("c1", "c3", "c5")
                         else "synchronous calls, pinned host inputs and reused pinned result buffers")},
        "gpu_launches": launches, "cpu_baseline": cpu, "clocks": clocks,
        "parity": parity,
        "parts_ms": {k: round(v, 3) for k, v in parts.items()},
    }
    if w in ("c2", "c4"):
        line["bvh_build_mpts_s"] = n / (parts["build"] / 1e3) / 1e6
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 27, help="points per GPU")
    ap.add_argument("--seed", type=int, default=2409)
    ap.add_argument("--cpu-sample-n", type=int, default=1 << 24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 / C5 (2^30) extra configs of the headline line")
    ap.add_argument("--slabs", action="store_true",
                    help="run the multi-GPU slab path (NCCL) even at one rank (tests the N > 1 code on one GPU)")
    ap.add_argument("--workload", default="fof_field", choices=["fof_field"] + sorted(CONFIGS),
                    help="fof_field is the headline; c1..c4 are the other SURVEY §8(d) configs (1 GPU)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, world), file=sys.stderr)
    if world > 1 or args.slabs:
        import torch
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        backend = "nccl" if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend=backend)
    try:
        if args.impl == "reference":
            run_reference_arm(args, rank, world)
        elif args.workload != "fof_field":
            run_config(args)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 or args.slabs:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
