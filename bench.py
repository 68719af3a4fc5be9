#!/usr/bin/env python3
"""bench.py — batched certaindex + early-exit / token-budget decisions on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C|A|B|D|E] [--impl ours|reference]

Headline workload (BASELINE.json north_star target): config C — Self-Consistency certaindex
+ token-budget allocation over a synthetic trace of 1M requests x 32 samples x 64 probes,
ids u32[R][P][S] resident in HBM (8.6 GB, > the 126 MB L2, so no flush is needed between
steps).  One step = K2 sc_certaindex (every (r,p) row: exact-match clusters, FP64 entropy
certaindex, threshold bits) + K5 allocate_scan (static-threshold exit at detect@5, cap 64,
token budgets, exclusive scan, stable compaction of continuing requests).

Multi-GPU (torchrun, one process per GPU): requests shard with no data-path collective;
each rank scores its own 1M-request slice (weak scaling); the only collective is an
8-byte allgather of shard budget totals for global token offsets.  Time = max over ranks.

Metric: probe-evals/s, one probe-eval = one sampled answer (r,s,p) entering the
certaindex (BASELINE.md unit "answers/s").  `--impl reference` times the reference's own
C++ functions (oracle/_ref, compiled from /root/reference/proj/src) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "probe-evals/sec + HBM GB/s fraction at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "probe-evals/s"

CONFIGS = {
    # north_star target shape (configs[2] of BASELINE.json, sharded per GPU)
    "C": dict(kind="sc", R=1 << 20, P=64, S=32, tau=0.7, detect=5, cap=64, interval=64, conv_hi=64,
              desc="SC entropy certaindex + token-budget allocation, 1M req x 32 samples x 64 probes"),
    "A": dict(kind="sc", R=1024, P=32, S=16, tau=0.7, detect=5, cap=32, interval=64, conv_hi=32,
              desc="SC entropy certaindex early exit, 1024 queries x 16 samples x 32 probes"),
    "B": dict(kind="cot", R=1 << 20, P=64, w=3, tau=0.9, interval=64, max_tokens=4096, hes=0.05, conv_hi=64,
              desc="CoT probe-window consistency early exit, 1M requests x 64 probes, window 3"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every ~2 ms DURING the
    timed region (the same fields as the recipe's nvidia-smi clocks line)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, index=0, period=0.002):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        self.err = None

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                try:
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    rs = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, rs))
                self._stop.wait(self.period)
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        reasons = sorted({name for _, rs in self.samples for bit, name in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------------------
def cpu_baseline_sc(cfg, nthreads, sample_req, seed):
    """The reference's own functions (oracle/_ref) on a bounded sample of the workload."""
    import numpy as np

    from oracle import oracle as O
    import ctypes as C
    g = O.gen_params(seed=seed, conv_hi=cfg["conv_hi"])
    ids = np.empty((sample_req, cfg["P"], cfg["S"]), np.uint32)
    O.lib().cdxo_gen_sc_mt(C.byref(g), C.c_uint64(0), C.c_uint64(sample_req), C.c_uint32(cfg["P"]),
                           C.c_uint32(cfg["S"]), ids.ctypes.data_as(C.c_void_p), C.c_int(nthreads))
    ths = [(0, cfg["tau"], 0)]
    O.ref_sc_batch(ids[: max(1, sample_req // 64)], 5, ths, nthreads=nthreads)  # warm
    t0 = time.perf_counter()
    h, meets = O.ref_sc_batch(ids, 5, ths, nthreads=nthreads)
    O.allocate_scan(meets, sample_req, cfg["P"], 2, cfg["detect"], cfg["cap"], 1, cfg["interval"] * cfg["S"])
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    O.ref_sc_batch(ids, 5, ths, nthreads=nthreads, mode=1, want=False)
    fill = time.perf_counter() - t1
    answers = sample_req * cfg["P"] * cfg["S"]
    return answers / dt, dt, fill


def cpu_baseline_cot(cfg, nthreads, sample_req, seed):
    from oracle import oracle as O
    g = O.gen_params(seed=seed, conv_hi=cfg["conv_hi"], hesitation_prob=cfg["hes"])
    ids, hes = O.gen_cot(g, sample_req, cfg["P"])
    t0 = time.perf_counter()
    O.ref_cot_batch(ids, hes, 5, cfg["interval"], cfg["w"], cfg["tau"], cfg["max_tokens"], nthreads=nthreads,
                    want_ck=False)
    dt = time.perf_counter() - t0
    return sample_req * cfg["P"] / dt, dt, 0.0


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg, rank, world):
    """--impl reference: rank 0 times the reference's CPU path; other ranks exit."""
    if rank != 0:
        return
    nth = host_threads()
    R = args.ref_sample or (1 << 17 if cfg["kind"] == "sc" else 1 << 16)
    if cfg["kind"] == "sc":
        R = min(R, cfg["R"])
    vals = []
    for i in range(args.warmup + args.steps):
        fn = cpu_baseline_sc if cfg["kind"] == "sc" else cpu_baseline_cot
        v, dt, fill = fn(cfg, nth, R, 20993 + i)
        if i >= args.warmup:
            vals.append((v, dt))
    v = statistics.median([x[0] for x in vals])
    ms = statistics.median([x[1] for x in vals]) * 1e3
    sample = f"{R} requests of config {args.config} per step ({R * cfg['P'] * cfg.get('S', 1)} probe-evals)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 ids / f64 entropy", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "sample_requests": R},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nth, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
def bench_sc(args, cfg, rank, world, cx):
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    R, P, S = cfg["R"], cfg["P"], cfg["S"]
    r0 = rank * R
    gp = GenParams(seed=20993 + 3, conv_hi=cfg["conv_hi"])
    ids = cx.gen_sc(gp, R, P, S, r0=r0)
    hcert = torch.empty((R, P), dtype=torch.float32, device="cuda")
    meets = torch.empty((R, (P + 31) // 32), dtype=torch.int32, device="cuda")
    ths = [Threshold(0, cfg["tau"], 0)]
    pol = AllocPolicy(kind=2, detect_at=cfg["detect"], resource_cap=cfg["cap"], tokens_per_unit=cfg["interval"] * S)
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_knob", torch.int32), ("reason", torch.uint8), ("granted", torch.int32), ("offsets", torch.int64),
            ("kept", torch.int32))}
    out["scalars"] = torch.zeros((3,), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    n_ev = args.steps
    k2s = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    k2e = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    k5e = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]

    def step(i=None):
        if i is not None:
            k2s[i].record(stream)
        cx.sc_certaindex(ids, ths, hcert=hcert, meets=meets)
        if i is not None:
            k2e[i].record(stream)
        cx.allocate_scan(meets, R, P, pol, out=out)
        if i is not None:
            k5e[i].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    l0 = cx.launches
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        for i in range(args.steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = cx.launches - l0
    barrier(world)
    ms_local = t_start.elapsed_time(t_end)
    ms = max_over_ranks(ms_local, world)
    k2_ms = statistics.mean(k2s[i].elapsed_time(k2e[i]) for i in range(n_ev))
    k5_ms = statistics.mean(k2e[i].elapsed_time(k5e[i]) for i in range(n_ev))

    # global token offsets across ranks: allgather of shard budget totals (8 B per rank)
    total_b = out["scalars"][2:3].clone()
    if world > 1:
        import torch.distributed as dist
        allt = [torch.zeros_like(total_b) for _ in range(world)]
        dist.all_gather(allt, total_b)
    n_kept = int(out["scalars"][0])

    answers = R * P * S * world
    value = answers * args.steps / (ms / 1e3)
    k2_bytes = R * P * S * 4 + R * P * 4 + R * ((P + 31) // 32) * 4
    k5_bytes = R * ((P + 31) // 32) * 4 + R * (4 + 1 + 4 + 8) + n_kept * 4
    peak, peak_src = load_peaks()
    achieved = k2_bytes / (k2_ms / 1e3) / 1e9
    res = dict(value=value, ms=ms / args.steps, launches=launches, k2_ms=k2_ms, k5_ms=k5_ms, k2_bytes=k2_bytes,
               k5_bytes=k5_bytes, achieved=achieved, peak=peak, peak_src=peak_src, clocks=clk.summary(),
               step_bytes=k2_bytes + k5_bytes, n_kept=n_kept)
    # e2e through the C-ABI host entry (host buffers, H2D/D2H inside the timed region)
    res["e2e"] = e2e_sc(args, cfg, cx, ids, ths, pol) if not args.no_e2e else None
    del ids
    return res


def e2e_sc(args, cfg, cx, ids_dev, ths, pol):
    import ctypes as C

    import torch
    from paper_2412_20993_b200 import _abi, c_policy, c_thresholds
    R, P, S = cfg["R"], cfg["P"], cfg["S"]
    lib = cx.lib
    if not hasattr(lib, "cdx_sc_decide_host"):
        return None
    host_ids = torch.empty((R, P, S), dtype=torch.int32, pin_memory=True)
    host_ids.copy_(ids_dev)
    ek = torch.empty((R,), dtype=torch.int32, pin_memory=True)
    why = torch.empty((R,), dtype=torch.uint8, pin_memory=True)
    off = torch.empty((R,), dtype=torch.int64, pin_memory=True)
    saved = C.c_int64(0)
    arr, n = c_thresholds(ths)
    cp = c_policy(pol)

    def one():
        st = lib.cdx_sc_decide_host(cx.h, host_ids.data_ptr(), R, P, S, arr, n, C.byref(cp), ek.data_ptr(),
                                    why.data_ptr(), off.data_ptr(), None, C.byref(saved))
        cx._check(st)

    for _ in range(max(1, args.warmup)):
        one()
    steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    return {"value": R * P * S / dt, "unit": UNIT, "h2d_bytes_per_step": R * P * S * 4,
            "d2h_bytes_per_step": R * (4 + 1 + 8) + 8, "ms_per_step": dt * 1e3,
            "api": "cdx_sc_decide_host (C-ABI, pinned host buffers)"}


def bench_cot(args, cfg, rank, world, cx):
    import torch
    from paper_2412_20993_b200 import GenParams, ProbeConfig
    R, P = cfg["R"], cfg["P"]
    ids, hes = cx.gen_cot(GenParams(seed=20993 + 2, conv_hi=cfg["conv_hi"], hesitation_prob=cfg["hes"]), R, P,
                          r0=rank * R)
    pc = ProbeConfig(cfg["interval"], cfg["w"], cfg["tau"], cfg["max_tokens"])
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_step", torch.int32), ("reason", torch.uint8), ("final_id", torch.int32), ("low_conf", torch.uint8))}
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        cx.cot_exit(ids, hes, pc, out=out)
    torch.cuda.synchronize()
    barrier(world)
    l0 = cx.launches
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            cx.cot_exit(ids, hes, pc, out=out)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    launches = cx.launches - l0
    ms_local = ev[0].elapsed_time(ev[-1])
    ms = max_over_ranks(ms_local, world)
    k_ms = statistics.mean(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    bytes_ = R * P * 4 + R * ((P + 63) // 64) * 8 + R * (4 + 1 + 4 + 1)
    peak, peak_src = load_peaks()
    return dict(value=R * P * world * args.steps / (ms / 1e3), ms=ms / args.steps, launches=launches, k2_ms=k_ms,
                k2_bytes=bytes_, achieved=bytes_ / (k_ms / 1e3) / 1e9, peak=peak, peak_src=peak_src,
                clocks=clk.summary(), step_bytes=bytes_, e2e=None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    rank, world, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    from paper_2412_20993_b200 import Context
    cx = Context(local)
    res = bench_sc(args, cfg, rank, world, cx) if cfg["kind"] == "sc" else bench_cot(args, cfg, rank, world, cx)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = host_threads()
        if cfg["kind"] == "sc":
            R_s = min(cfg["R"], args.ref_sample or (1 << 18))
            v, dt, fill = cpu_baseline_sc(cfg, nth, R_s, 20993 + 3)
            cpu = {"value": v, "unit": UNIT, "cores": nth, "kind": "reference",
                   "sample": f"{R_s} of {cfg['R']} requests of config {args.config} ({R_s * cfg['P'] * cfg['S']} "
                             f"probe-evals, {dt:.2f} s incl. {fill:.2f} s string row-buffer fill)"}
        else:
            R_s = args.ref_sample or (1 << 16)
            v, dt, _ = cpu_baseline_cot(cfg, nth, R_s, 20993 + 2)
            cpu = {"value": v, "unit": UNIT, "cores": nth, "kind": "reference",
                   "sample": f"{R_s} requests of config {args.config} ({R_s * cfg['P']} probe-evals, {dt:.2f} s)"}
    if rank == 0:
        frac = res["achieved"] / res["peak"]
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 ids / f64 entropy (f32 store)", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"],
                       **{k: v for k, v in cfg.items() if k in ("R", "P", "S", "w", "tau", "detect", "cap")},
                       "requests_per_gpu": cfg["R"], "parallelism": f"request shards x{world} (no data-path collective)",
                       "l2": "inputs > L2 (126 MB); no flush needed"},
            "roofline": {"bound": "hbm", "achieved": res["achieved"], "peak": res["peak"], "unit": "GB/s",
                         "frac": frac, "traffic": None, "peak_source": res["peak_src"],
                         "kernel": "sc_certaindex" if cfg["kind"] == "sc" else "cot_exit",
                         "kernel_ms": res["k2_ms"], "algorithmic_bytes_per_launch": res["k2_bytes"],
                         "step_bytes": res["step_bytes"],
                         "step_frac": res["step_bytes"] / (res["ms"] / 1e3) / 1e9 / res["peak"]},
            "cpu_baseline": cpu,
            "e2e": res["e2e"],
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
        }
        if "k5_ms" in res:
            line["roofline"]["allocate_scan_ms"] = res["k5_ms"]
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
