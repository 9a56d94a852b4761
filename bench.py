#!/usr/bin/env python
"""ACP-SGD aggregation benchmark (BASELINE.json metric: "ACP-SGD aggregation
ms/step & gradient GB/s, ResNet-50/BERT-L, 1-8 B200").

One *step* = one acp_step() of Alg. 2 over a model's whole synthetic gradient
set (orthogonalise -> fused EF + projection -> pack -> per-bucket NCCL
all-reduce -> decode + residual), alternating P-/Q-steps. Gradients live in
HBM before the timed region (uniform(-1,1)/sqrt(m) values; inputs larger than
L2). value = whole-job gradient GB/s = N_gpus * 4 * elements / (ms/step),
max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload bert-large-r4]
  torchrun --nproc-per-node N bench.py --gpus N ...
  python bench.py --impl reference ...   (the CPU oracle on a bounded sample)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "bert-large-r4": ("bert-large", 4),
    "resnet50-r4": ("resnet50", 4),
    "resnet152-r4": ("resnet152", 4),
    "bert-base-r8": ("bert-base", 8),
    "bert-large-r1": ("bert-large", 1),
    "bert-large-r2": ("bert-large", 2),
    "bert-large-r8": ("bert-large", 8),
    "bert-large-r16": ("bert-large", 16),
    "bert-large-r32": ("bert-large", 32),
}
METRIC = "ACP-SGD aggregation gradient GB/s (ms/step alongside), ResNet-50/BERT-L, 1-8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _shapes(model):
    from acp_inputs import ready_order
    return [s for _, s in ready_order(model)]


def _numel(s):
    n = 1
    for d in s:
        n *= int(d)
    return n


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, device_index, period=0.01):
        self.dev = device_index
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        N = self.N
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in names.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max(d.get("num_threads", 1) for d in info) if info else 1
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(model, rank, frac_every=3):
    """Bounded sample of the workload for the CPU oracle: every `frac_every`-th
    matrix (ready order) plus all vectors."""
    out, k = [], 0
    for s in _shapes(model):
        if len(s) == 1:
            out.append(s)
        else:
            if k % frac_every == 0:
                out.append(s)
            k += 1
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def time_oracle_threads(model, rank, steps, warmup, frac_every=3):
    """The oracle on 1 thread and on all host cores."""
    out = {}
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        threadpool_limits = None
    for label, limit in (("1_thread", 1), ("all_cores", None)):
        if threadpool_limits is not None and limit is not None:
            with threadpool_limits(limits=limit):
                out[label] = time_oracle(model, rank, steps, warmup, frac_every=frac_every)
        else:
            out[label] = time_oracle(model, rank, steps, warmup, frac_every=frac_every)
    return out


def time_oracle(model, rank, steps, warmup, world=1, frac_every=3):
    """Run the oracle (as it stands) on the bounded sample; returns GB/s."""
    import numpy as np
    from oracle import AcpOracle
    sel = oracle_sample(model, rank, frac_every)
    n = sum(_numel(s) for s in sel)
    o = AcpOracle(sel, rank, world_size=world, seed=1)
    rs = np.random.default_rng(0)
    g = [[(rs.random(s, dtype=np.float32) * 2 - 1) for s in sel] for _ in range(world)]
    for t in range(warmup):
        o.step(g, t % 2)
    t0 = time.perf_counter()
    for t in range(steps):
        o.step(g, (warmup + t) % 2)
    dt = (time.perf_counter() - t0) / max(steps, 1)
    return {"gbs": 4.0 * n / dt / 1e9, "s_per_step": dt, "elements": n, "tensors": len(sel)}


def run_reference(args):
    rank_env = int(os.environ.get("RANK", "0"))
    if rank_env != 0:
        return 0
    model, r = WORKLOADS[args.workload]
    res = time_oracle(model, r, args.steps, args.warmup, frac_every=args.oracle_every)
    cores = _cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": res["gbs"], "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * res["s_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "rank": r, "sample_elements": res["elements"],
                   "sample_tensors": res["tensors"]},
        "cpu_baseline": {"value": res["gbs"], "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "cpu_model": _cpu_model(),
                         "sample": f"{model} r={r}: every {args.oracle_every}-th matrix + all vectors "
                                   f"({res['elements']} elements), one worker, numpy fp64"},
        "e2e": {"value": res["gbs"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar over the default process group (the bench's
    timing rule: a multi-GPU step takes as long as its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _setup_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _measure(model, r, world, rank, local, args, comm, profile=True, flags=0):
    """Time K steps (CUDA-graph replay, the library default), then K more
    steps run eagerly with per-kernel CUDA events for the roofline."""
    import torch
    from paper_2306_08881_b200 import AcpContext
    shapes = _shapes(model)
    nel = sum(_numel(s) for s in shapes)
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    grads = []
    for s in shapes:
        m = _numel(s[1:]) if len(s) > 1 else 1
        g = torch.rand(s, device="cuda", generator=gen) * 2 - 1
        grads.append((g / (m ** 0.5)).contiguous())
    ctx = AcpContext(shapes, r, world_size=world, nccl_comm=comm, seed=7,
                     bucket_bytes=args.bucket_bytes, flags=flags)
    nvls = False
    if world > 1 and args.allreduce == "nvls" and not flags:
        try:
            nvls = ctx.attach_symmetric()  # False when the box has no multicast
        except Exception as e:  # no symmetric memory here: NCCL all-reduce
            print(f"NVLS unavailable ({e}); using NCCL", file=sys.stderr)
    ctx.set_graphs(not args.no_graphs)
    stream = torch.cuda.current_stream()
    for t in range(args.warmup):
        ctx.step(grads, t % 2)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    l0 = ctx.launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        evs[0].record(stream)
        for t in range(args.steps):
            ctx.step(grads, (args.warmup + t) % 2)
            evs[t + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    launches = ctx.launch_count() - l0
    ms = max_over_ranks(evs[0].elapsed_time(evs[-1]) / args.steps)
    per = [evs[t].elapsed_time(evs[t + 1]) for t in range(args.steps)]
    par = [(args.warmup + t) % 2 for t in range(args.steps)]
    pm = [x for x, q in zip(per, par) if q == 0]
    qm = [x for x, q in zip(per, par) if q == 1]
    import statistics
    step_stats = {"mean_ms": statistics.fmean(per), "std_ms": statistics.pstdev(per),
                  "p_step_ms": max_over_ranks(statistics.fmean(pm)) if pm else None,
                  "q_step_ms": max_over_ranks(statistics.fmean(qm)) if qm else None}
    prof = None
    if profile:
        # per-kernel CUDA events on the launching stream (eager launches)
        ctx.profile(True)
        ctx.profile_reset()
        for t in range(args.steps):
            ctx.step(grads, (args.warmup + args.steps + t) % 2)
        torch.cuda.synchronize()
        prof = ctx.profile_read()
        ctx.profile(False)
    nb = (len(ctx.buckets(0)), len(ctx.buckets(1)))
    return {"ctx": ctx, "grads": grads, "shapes": shapes, "nel": nel, "ms": ms, "prof": prof,
            "launches": launches, "clocks": clk.summary(), "buckets": nb, "step_stats": step_stats,
            "allreduce": ("nvls" if nvls else "nccl") if world > 1 else None}


def _ssgd(nel, world, args):
    """NEXT-4 context: the dense S-SGD exchange of the same gradient set, a
    plain NCCL all-reduce (sum) in 25 MiB buckets, max over ranks."""
    import torch
    import torch.distributed as dist
    flat = torch.zeros(nel, dtype=torch.float32, device="cuda")
    bucket = 25 * 2 ** 20 // 4
    chunks = [flat[i:i + bucket] for i in range(0, nel, bucket)]
    for _ in range(2):
        for c in chunks:
            dist.all_reduce(c)
    torch.cuda.synchronize()
    dist.barrier()
    steps = max(3, min(args.steps, 10))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        for c in chunks:
            dist.all_reduce(c)
    ev1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / steps)
    busbw = 2.0 * (world - 1) / world * 4.0 * nel / (ms * 1e-3) / 1e9
    del flat, chunks
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "buckets": (nel + bucket - 1) // bucket, "busbw_gbs": busbw,
            "nvlink_frac": busbw / 900.0}


def _e2e(res, world, args):
    """Same step through the public API with HOST buffers: every step's
    gradients go host -> device from pinned memory, acp_step runs, and the
    decoded gradients come back device -> host, all inside the timed region.
    Steps are software-pipelined over two device gradient sets: the upload of
    step t+1 (copy stream H) and the download of step t (copy stream D)
    overlap step t's kernels (PCIe is full duplex), as a training loop would."""
    import torch
    ctx, grads = res["ctx"], res["grads"]
    # the gradients of a step live back to back (16-byte aligned offsets) in
    # one flat device buffer and one flat pinned host buffer, so each
    # direction is ONE copy per step (as a DDP-style flat gradient buffer
    # would be) instead of one small copy per tensor: the per-tensor version
    # moved BERT-L's ~400 tensors at 34.5 GB/s
    offs, tot = [], 0
    for g in grads:
        offs.append(tot)
        tot += (g.numel() + 3) // 4 * 4
    flat_dev = [torch.zeros(tot, device=grads[0].device) for _ in range(2)]
    sets = [[fd[o:o + g.numel()].view(g.shape) for o, g in zip(offs, grads)] for fd in flat_dev]
    host_in = torch.zeros(tot).pin_memory()
    for o, g in zip(offs, grads):
        host_in[o:o + g.numel()].copy_(g.detach().reshape(-1).cpu())
    host_out = [torch.empty(tot).pin_memory() for _ in range(2)]
    steps = max(2, min(args.steps, args.e2e_steps))
    comp = torch.cuda.current_stream()
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    d_done = [None, None]

    def upload(t):
        b = t % 2
        with torch.cuda.stream(sh):
            if d_done[b] is not None:
                sh.wait_event(d_done[b])  # step t-2's download has read this set
            flat_dev[b].copy_(host_in, non_blocking=True)
            e = ev()
            e.record(sh)
        return e

    def run(t, up):
        b = t % 2
        comp.wait_event(up)
        ctx.step(sets[b], t % 2, stream=comp)
        c = ev()
        c.record(comp)
        with torch.cuda.stream(sd):
            sd.wait_event(c)
            host_out[b].copy_(flat_dev[b], non_blocking=True)
            d = ev()
            d.record(sd)
        d_done[b] = d

    up = upload(0)
    run(0, up)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    e0.record(comp)
    up = upload(1)
    for t in range(1, steps + 1):
        nxt = upload(t + 1) if t < steps else None
        run(t, up)
        up = nxt
    comp.wait_stream(sd)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps)
    nbytes = 4 * res["nel"]
    return {"value": world * nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": 4 * tot, "d2h_bytes_per_step": 4 * tot, "steps": steps,
            "pipelined": "H2D(t+1) and D2H(t) overlap step t (two flat gradient buffers, one copy per "
                         "direction per step, copy streams)"}


def _nvlink(prof, world):
    """All-reduce bus bandwidth 2(p-1)/p * bytes / t of the eager profiled pass
    against 900 GB/s per direction (NVLink 5), SURVEY §8(d)."""
    if world <= 1 or not prof or prof.get("allreduce", {}).get("launches", 0) == 0:
        return None
    a = prof["allreduce"]
    t = a["ms"] / a["launches"] * 1e-3
    b = a["bytes"] / a["launches"]
    bus = 2.0 * (world - 1) / world * b / t / 1e9
    return {"busbw_gbs": bus, "frac_900": bus / 900.0, "bytes_per_group": b, "ms_per_group": t * 1e3}


def _roofline(prof, peak, peak_kind, workload):
    cls = [k for k in ("proj_p", "proj_q", "decode_p", "decode_q") if prof[k]["launches"] > 0]
    dom = max(cls, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    per_launch_bytes = d["bytes"] / d["launches"]
    per_launch_ms = d["ms"] / d["launches"]
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    # DRAM traffic of the dominant kernel from an ncu capture of THIS build
    # (profiles/ncu_traffic_<tag>.json, build id = source hash, build.py)
    traffic, tsrc = None, None
    try:
        import glob
        import importlib.util
        spec = importlib.util.spec_from_file_location("acp_build", os.path.join(ROOT, "paper_2306_08881_b200", "build.py"))
        B = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(B)
        bid = B.build_id()
        for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_*.json")), reverse=True):
            tr = json.load(open(f))
            if tr.get("build_id") == bid and dom in tr.get(workload, {}):
                traffic, tsrc = tr[workload][dom], os.path.relpath(f, ROOT) + f" (build {bid})"
                break
    except Exception:
        pass
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_kind,
            "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
            "per_class": {k: {"ms_per_launch": v["ms"] / v["launches"],
                              "gbs": (v["bytes"] / v["launches"]) / (v["ms"] / v["launches"] * 1e-3) / 1e9}
                          for k, v in prof.items() if v["launches"] > 0}}


def run_ours(args):
    import torch
    world, rank, local = _setup_dist(args)
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    comm = None
    if world > 1:
        from paper_2306_08881_b200 import nccl_comm_from_group
        comm = nccl_comm_from_group()
    model, r = WORKLOADS[args.workload]
    res = _measure(model, r, world, rank, local, args, comm)
    peak, peak_kind = _peaks()
    ms = res["ms"]
    nel = res["nel"]
    value = world * 4.0 * nel / (ms * 1e-3) / 1e9
    roof = _roofline(res["prof"], peak, peak_kind, args.workload)
    e2e = _e2e(res, world, args) if not args.no_e2e else None
    secondary = None
    if args.secondary and args.secondary not in ("none", args.workload):
        res["ctx"].close()
        del res["grads"]
        torch.cuda.empty_cache()
        m2, r2 = WORKLOADS[args.secondary]
        s = _measure(m2, r2, world, rank, local, args, comm)
        secondary = {"workload": args.secondary, "ms_per_step": s["ms"],
                     "value": world * 4.0 * s["nel"] / (s["ms"] * 1e-3) / 1e9, "unit": "GB/s",
                     "step_hbm_frac_16B": 16.0 * s["nel"] / (s["ms"] * 1e-3) / 1e9 / peak,
                     "roofline": _roofline(s["prof"], peak, peak_kind, args.secondary),
                     "gpu_launches": s["launches"]}
        s["ctx"].close()
    psgd = None
    if not args.no_powersgd:
        # NEXT-1 / NEXT-4 context: the Power-SGD baseline (two projections and
        # two all-reduces per step) through the same library
        from paper_2306_08881_b200 import ACP_POWERSGD
        torch.cuda.empty_cache()
        ps = _measure(model, r, world, rank, local, args, comm, profile=False, flags=ACP_POWERSGD)
        psgd = {"workload": args.workload, "ms_per_step": ps["ms"],
                "value": world * 4.0 * ps["nel"] / (ps["ms"] * 1e-3) / 1e9, "unit": "GB/s",
                "acp_speedup": ps["ms"] / ms, "gpu_launches": ps["launches"]}
        ps["ctx"].close()
        del ps
    ssgd = None
    if world > 1 and not args.no_ssgd:
        ssgd = _ssgd(nel, world, args)
        ssgd["acp_speedup"] = ssgd["ms_per_step"] / ms
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cbt = time_oracle_threads(model, r, 2, 1, frac_every=args.oracle_every)
        cb = cbt["all_cores"]
        cpu = {"value": cb["gbs"], "unit": "GB/s", "cores": _cpu_threads(), "kind": "oracle",
               "cpu_model": _cpu_model(), "value_1_thread": cbt["1_thread"]["gbs"],
               "sample": f"{model} r={r}: every {args.oracle_every}-th matrix + all vectors "
                         f"({cb['elements']} of {nel} elements), 1 warm + 2 timed steps (P,Q), numpy fp64"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.workload, "model_shapes": model, "rank": r,
                       "elements_per_gpu": nel, "parity": "alternating P/Q steps",
                       "buckets_PQ": list(res["buckets"]) if world > 1 else [1, 1],
                       "bucket_rule": f"{args.bucket_bytes} B x compression rate (P:257)",
                       "l2": "inputs larger than L2 (M+E working set > 126 MB), no flush",
                       "parallelism": f"dp{world}", "allreduce": res["allreduce"]},
            "step_hbm_frac_16B": 16.0 * nel / (ms * 1e-3) / 1e9 / peak,
            "step_stats": res["step_stats"],
            "nvlink": _nvlink(res["prof"], world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": res["clocks"],
            "gpu_launches": res["launches"],
            "secondary": secondary,
            "powersgd": psgd,
            "ssgd": ssgd,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bert-large-r4", choices=sorted(WORKLOADS))
    ap.add_argument("--secondary", default="resnet50-r4")
    ap.add_argument("--bucket-bytes", type=int, default=25 * 2 ** 20)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-powersgd", action="store_true",
                    help="skip the on-box Power-SGD comparison line")
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "nvls"],
                    help="N > 1: NCCL per bucket group, or the library's NVLS kernel (symmetric memory)")
    ap.add_argument("--no-ssgd", action="store_true",
                    help="skip the dense S-SGD all-reduce comparison (N > 1)")
    ap.add_argument("--oracle-every", type=int, default=3)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
