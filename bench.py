#!/usr/bin/env python3
"""bench.py — batched certaindex + early-exit / token-budget / gang-priority decisions on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C|A|B|D|E] [--impl ours|reference]

Headline workload (BASELINE.json north_star target): config C — Self-Consistency certaindex
+ token-budget allocation over a synthetic trace of 1M requests x 32 samples x 64 probes,
ids u32[R][P][S] resident in HBM (8.6 GB > the 126 MB L2, so no flush is needed between
steps).  One step = K2 sc_certaindex (every (r,p) row: exact-match clusters, FP64 entropy
certaindex, threshold bits) + K5 allocate_scan (static-threshold exit at detect@5, cap 64,
token budgets, exclusive scan, stable compaction of continuing requests).
The same JSON line also carries configs A, B, D, E (`other_configs`, N=1 only).

Multi-GPU (torchrun, one process per GPU): requests shard with no data-path collective;
each rank scores its own 1M-request slice (weak scaling); the only collective is an 8-byte
allgather of shard budget totals for global token offsets.  Time = max over ranks.

Metric: probe-evals/s.  One probe-eval = one sampled answer (r,s,p) entering the certaindex
for SC (A, C), one probe record (r,p) for CoT (B), one node reward (g,t,w) for MCTS/Rebase
(D), one program ordered for the gang order (E), one trace record ingested (J).  `--impl reference` times the reference's
own C++ functions (oracle/_ref, compiled from /root/reference/proj/src) on all host cores.
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

METRIC = "probe-evals/sec + HBM GB/s fraction at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "probe-evals/s"

CONFIGS = {
    # BASELINE.json configs; C is the north_star target shape (sharded per GPU)
    "A": dict(kind="sc", R=1024, P=32, S=16, tau=0.7, detect=5, cap=32, interval=64, conv_hi=32, graph=True, flush_l2=True,
              desc="SC entropy certaindex early exit, 1024 queries x 16 samples x 32 probes (K2 + K5 replayed as "
                   "one CUDA graph: launch-bound size)"),
    "B": dict(kind="cot", R=1 << 20, P=64, w=3, tau=0.9, interval=64, max_tokens=4096, hes=0.05, conv_hi=64,
              desc="CoT probe-window consistency early exit, 1M requests x 64 probes, window 3"),
    "C": dict(kind="sc", R=1 << 20, P=64, S=32, tau=0.7, detect=5, cap=64, interval=64, conv_hi=64,
              desc="SC entropy certaindex + token-budget allocation, 1M req x 32 samples x 64 probes"),
    "D": dict(kind="reward", G=1 << 18, T=16, W=64, conv_hi=16, detect=3,
              desc="MCTS/Rebase reward + cumulative entropy certaindex, 256K programs x 64 nodes x 16 steps"),
    "E": dict(kind="mixed", N=1 << 22, limit=0.5, prior=128.0, sc=(32, 16), cot=(64, 3), rw=(16, 64),
              desc="online scheduling round over a 4M-program mixed trace (40% SC / 40% CoT / 10% MCTS / 10% "
                   "Rebase): per-archetype certaindex at every knob unit (K2 / cot_meets / K4), allocate at each "
                   "program's current knob + budget scan, then the gang priority order of the live programs (K6)"),
    "G": dict(kind="gang", N=1 << 22, limit=0.5, prior=128.0,
              desc="gang-scheduling priority order alone (escalation + SJF + tie-break), 4M programs"),
    "K": dict(kind="intern", n=1 << 27, width=12, S=32,
              desc="answer canonicalisation + interning (trim, hash, byte-verify, dense first-seen ids) + "
                   "hesitation flags over 2^27 whitespace-padded answers (1.6 GB arena, K1)"),
    "J": dict(kind="jsonl", lines=1 << 20, programs=1 << 14, flush_l2=True,
              desc="probe-trace JSONL ingestion (read_trace_jsonl), 1M records over 16K programs"),
}
TH_MCTS = [(0, 0.99, 0), (1, 0.4, 0)]   # PAPER.md:963 MCTS/GSM8K thresholds
TH_REBASE = [(0, 0.85, 0), (1, 0.99, 0)]  # PAPER.md:966 Rebase/GSM8K thresholds


TRAFFIC_KEY = {"sc": "sc", "cot": "cot", "reward": "reward", "gang": "gang", "jsonl": "jsonl", "mixed": "mixed",
               "intern": "intern"}


def load_traffic(kind):
    """DRAM bytes per launch of this config's dominant kernel from the newest committed
    `ncu --set full` summary (profiles/<round>_traffic.json, tools/summarize_profiles.py):
    ncu's dram__bytes_read.sum + dram__bytes_write.sum, or None when none was captured."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):  # round order
        try:
            with open(path) as f:
                d = json.load(f).get(TRAFFIC_KEY[kind])
        except Exception:
            continue
        if d:
            best = {"bytes": d["dram_bytes"], "source": os.path.relpath(path, ROOT), "kernel": d["kernel"]}
    return best


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every ~2 ms DURING the
    timed region (the fields of the recipe's nvidia-smi clocks line)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index=0, period=0.002):
        self.index, self.period = index, period
        self.samples, self.max_mhz, self.err = [], None, None
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        self.samples.append((self._N.nvmlDeviceGetClockInfo(self._h, self._N.NVML_CLOCK_SM), self._rs(self._h)))

    def _run(self):
        try:
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(self.period)
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)

    def __enter__(self):
        try:  # NVML init is slow on first use: do it before the timed region starts
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
            self._rs = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if self._t and not self.samples and self.err is None:
            try:  # a timed region shorter than one sampling period: take the last sample now
                self._sample()
            except Exception as e:  # pragma: no cover
                self.err = repr(e)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        reasons = sorted({n for _, rs in self.samples for bit, n in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # test hooks: CDX_BENCH_BACKEND=gloo with CDX_BENCH_SHARE_DEVICE=1 runs every rank on
        # cuda:0 (exercises the N>1 path on a one-GPU box; its numbers mean nothing)
        backend = os.environ.get("CDX_BENCH_BACKEND", "nccl")
        if os.environ.get("CDX_BENCH_SHARE_DEVICE") == "1":
            local = 0
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
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


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- CPU (reference) legs
def cpu_sc(cfg, nth, R, seed):
    """Reference cluster_exact + certaindex_entropy + combined_meets_thresholds per row
    (oracle/_ref) + the SPEC allocate restatement, on R requests of the workload."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    g = O.gen_params(seed=seed, conv_hi=cfg["conv_hi"])
    ids = np.empty((R, cfg["P"], cfg["S"]), np.uint32)
    O.lib().cdxo_gen_sc_mt(C.byref(g), C.c_uint64(0), C.c_uint64(R), C.c_uint32(cfg["P"]), C.c_uint32(cfg["S"]),
                           ids.ctypes.data_as(C.c_void_p), C.c_int(nth))
    ths = [(0, cfg["tau"], 0)]
    O.ref_sc_batch(ids[: max(1, R // 64)], 5, ths, nthreads=nth)  # warm
    t0 = time.perf_counter()
    _, meets = O.ref_sc_batch(ids, 5, ths, nthreads=nth)
    O.allocate_scan(meets, R, cfg["P"], 2, cfg["detect"], cfg["cap"], 1, cfg["interval"] * cfg["S"])
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    O.ref_sc_batch(ids, 5, ths, nthreads=nth, mode=1, want=False)
    fill = time.perf_counter() - t1
    n = R * cfg["P"] * cfg["S"]
    return n / dt, dt, f"{R} requests ({n} probe-evals), {dt:.2f} s incl. {fill:.2f} s std::string row fill"


def cpu_cot(cfg, nth, R, seed):
    """Reference should_exit on every trace prefix + final_answer (oracle/_ref)."""
    from oracle import oracle as O
    ids, hes = O.gen_cot(O.gen_params(seed=seed, conv_hi=cfg["conv_hi"], hesitation_prob=cfg["hes"]), R, cfg["P"])
    t0 = time.perf_counter()
    O.ref_cot_batch(ids, hes, 5, cfg["interval"], cfg["w"], cfg["tau"], cfg["max_tokens"], nthreads=nth,
                    want_ck=False)
    dt = time.perf_counter() - t0
    n = R * cfg["P"]
    return n / dt, dt, f"{R} requests ({n} probe records), {dt:.2f} s"


def cpu_reward(cfg, nth, G, seed):
    """Reference cumulative certaindex_reward + certaindex_entropy(cluster_exact(all so far))
    per step, as runtime.cpp:279-292 recomputes them (oracle/_ref)."""
    import numpy as np

    from oracle import oracle as O
    rw, ids = O.gen_reward(O.gen_params(seed=seed, conv_hi=cfg["conv_hi"]), G, cfg["T"], cfg["W"])
    agg = (np.arange(G) % 2).astype(np.uint8)
    t0 = time.perf_counter()
    O.ref_reward_batch(rw, ids, agg, nthreads=nth)
    dt = time.perf_counter() - t0
    n = G * cfg["T"] * cfg["W"]
    return n / dt, dt, f"{G} programs ({n} node rewards), {dt:.2f} s"


def gang_inputs(N, seed, limit):
    import numpy as np
    rng = np.random.default_rng(seed)
    arrival = np.cumsum(rng.exponential(1e-3, N))  # lambda = 1000 programs/s
    now = float(arrival[-1]) + 1e-3
    # service lags chosen so ~5% of programs exceed the starvation limit
    last = now - rng.exponential(limit / 3.0, N)
    last = np.maximum(last, 0.0)
    cnt = rng.integers(0, 6, N).astype(np.uint32)
    sums = (rng.integers(32, 1024, N) * cnt).astype(np.int64)
    cap = rng.integers(4, 64, N).astype(np.int32)
    knob = np.minimum(cap, rng.integers(0, 64, N)).astype(np.int32)
    arche = rng.random(N)  # 40% SC / 40% CoT / 20% MCTS: terminated by B/C/D-style exits
    term = (rng.random(N) < np.where(arche < 0.4, 0.3, np.where(arche < 0.8, 0.2, 0.1))).astype(np.uint8)
    return dict(arrival=arrival, last_service=last, iter_tok_sum=sums, iter_count=cnt, knob=knob, cap=cap,
                terminated=term), now


def cpu_gang(cfg, nth, N, seed):
    """SPEC restatement (no reference code exists for the scheduler): per-thread qsort with the
    SPEC comparator + parallel pairwise merges on `nth` host threads (cdxo_gang_order_mt)."""
    from oracle import oracle as O
    soa, now = gang_inputs(N, seed, cfg["limit"])
    t0 = time.perf_counter()
    O.gang_order_mt(soa, 1, cfg["limit"], cfg["prior"], now, nth)
    dt = time.perf_counter() - t0
    return N / dt, dt, f"{N} programs, {dt:.2f} s (SPEC restatement, {nth} threads)"


def jsonl_text(lines, programs, seed):
    """Synthetic probe trace in the reference's JSONL schema (probe.hpp:12-14): programs
    interleaved, per-program strictly increasing step/offset, ~5% hesitant probes."""
    import numpy as np
    rng = np.random.default_rng(seed)
    prog = rng.integers(0, programs, lines)
    ans = rng.integers(0, 5, lines)
    hes = rng.random(lines) < 0.05
    step = np.zeros(programs, np.int64)
    names = ["S", "D1", "D2", "D3", "D4"]
    out = []
    for i in range(lines):
        p = int(prog[i])
        step[p] += 1
        s = int(step[p])
        a = ("wait, " if hes[i] else "") + names[int(ans[i])]
        out.append(f'{{"program_id": "prog-{p}", "step_index": {s}, "token_offset": {64 * s}, "answer": "{a}", '
                   f'"hesitant": {"true" if hes[i] else "false"}}}')
    return ("\n".join(out) + "\n").encode()


def cpu_jsonl(cfg, nth, lines, seed):
    """The reference's read_trace_jsonl (nlohmann parse + checks, probe.cpp:126-165) on `nth`
    host threads: line-aligned chunks, each parsed by the reference function, plus the
    per-program order checks across chunk boundaries (oracle/ref_harness.cpp)."""
    from oracle import oracle as O
    text = jsonl_text(lines, max(1, cfg["programs"] * lines // cfg["lines"]), seed)
    t0 = time.perf_counter()
    n = O.ref_read_trace_jsonl_mt(text, nth)
    dt = time.perf_counter() - t0
    return n / dt, dt, (f"{n} records ({len(text)} bytes), {dt:.2f} s ({nth} threads: line-aligned chunks through "
                        "read_trace_jsonl + cross-chunk order checks)")


SC_, REB_, MCT_, COT_ = 0, 1, 2, 3


def mixed_policies(cfg):
    """Per archetype (CDX_ARCH_*): thresholds and allocation policy of config E.  SC: H~ >= 0.7
    at detect 5; MCTS / Rebase: the Table-3 GSM8K thresholds at step 3
    (PAPER.md:963-966); CoT: C_k >= 0.9 re-tested every probe from the first full window."""
    (scP, S), (cotP, w), (T, W) = cfg["sc"], cfg["cot"], cfg["rw"]
    return {SC_: ([(0, 0.7, 0)], dict(kind=2, detect_at=5, resource_cap=scP, recheck_every=1, tokens_per_unit=64 * S)),
            REB_: ([(0, 0.85, 0), (1, 0.99, 0)], dict(kind=2, detect_at=3, resource_cap=T, recheck_every=1,
                                                      tokens_per_unit=W)),
            MCT_: ([(0, 0.99, 0), (1, 0.4, 0)], dict(kind=2, detect_at=3, resource_cap=T, recheck_every=1,
                                                     tokens_per_unit=W)),
            COT_: ([(0, 0.9, 0)], dict(kind=4, detect_at=w, resource_cap=cotP, recheck_every=1, tokens_per_unit=64))}


def mixed_layout(cfg, N, seed):
    """Global program table of the mixed trace: archetype, row within the archetype's group,
    current knob, scheduler state (paper_2412_20993_b200/synth.py)."""
    import numpy as np

    from paper_2412_20993_b200 import synth
    (scP, _), (cotP, _), (T, _) = cfg["sc"], cfg["cot"], cfg["rw"]
    arch, slot, sizes = synth.mixed_layout(N, seed)
    knob = synth.mixed_knobs(arch, (scP, T, T, cotP), seed + 1)
    state, now = synth.gang_state(N, seed + 2, cfg["limit"], knob=knob, cap=np.zeros(N, np.int32))
    return arch, slot, sizes, knob, state, now


def cpu_mixed(cfg, nth, n, seed):
    """The reference's per-archetype CPU path on n programs: cluster_exact + certaindex_entropy
    + combined_meets_thresholds per SC row, probe::consistency per CoT prefix, the cumulative
    certaindex_reward + entropy per MCTS / Rebase step (all oracle/_ref, the reference's own
    code), then allocate at each knob and the gang sort (SPEC restatements: no reference code
    exists for the scheduler), on `nth` host threads."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    (scP, S), (cotP, w), (T, W) = cfg["sc"], cfg["cot"], cfg["rw"]
    arch, slot, sizes, knob, state, now = mixed_layout(cfg, n, seed)
    sc = O.gen_sc(O.gen_params(seed=seed + 3, conv_hi=scP), sizes[0], scP, S)
    cid, ches = O.gen_cot(O.gen_params(seed=seed + 4, conv_hi=cotP, hesitation_prob=0.05), sizes[1], cotP)
    rw, rid = O.gen_reward(O.gen_params(seed=seed + 5, conv_hi=T), sizes[2], T, W)
    pols = mixed_policies(cfg)
    cp = [O.arch_policy(pols[a][0], kw["kind"], kw["detect_at"], kw["resource_cap"], kw["recheck_every"],
                        kw["tokens_per_unit"]) for a, kw in ((a, pols[a][1]) for a in range(4))]
    agg = np.zeros(sizes[2], np.uint8)
    sel = (arch == REB_) | (arch == MCT_)
    agg[slot[sel]] = (arch[sel] == REB_).astype(np.uint8)
    t0 = time.perf_counter()
    _, m_sc = O.ref_sc_batch(sc, 5, pols[SC_][0], nthreads=nth)
    ck = O.ref_cot_signal(cid, ches, w, nthreads=nth)
    m_cot = np.zeros((sizes[1], (cotP + 31) // 32), np.uint32)
    ok = ck >= pols[COT_][0][0][1]
    for p_ in range(cotP):
        m_cot[:, p_ // 32] |= ok[:, p_].astype(np.uint32) << np.uint32(p_ % 32)
    R, H = O.ref_reward_batch(rw, rid, agg, nthreads=nth)
    okr = np.where(agg[:, None] == 1, (H >= 0.85) & (R >= 0.99), (H >= 0.99) & (R >= 0.4))
    m_rw = np.zeros((sizes[2], (T + 31) // 32), np.uint32)
    for t in range(T):
        m_rw[:, t // 32] |= okr[:, t].astype(np.uint32) << np.uint32(t % 32)
    dec, grant, cap, off = np.empty(n, np.uint8), np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int64)
    tot = C.c_int64(0)
    meets = [np.ascontiguousarray(m) for m in (m_sc, m_cot, m_rw)]
    st = O.lib().cdxo_mixed_decide(O._p(arch), O._p(slot), O._p(knob), n,
                                   C.cast((C.c_void_p * 3)(*[m.ctypes.data for m in meets]), C.c_void_p),
                                   C.cast((C.c_uint32 * 3)(*[m.shape[1] for m in meets]), C.c_void_p),
                                   C.cast((C.c_uint64 * 3)(*sizes), C.c_void_p),
                                   C.cast((O.ArchPolicy * 4)(*cp), C.c_void_p), O._p(dec), O._p(grant), O._p(cap),
                                   O._p(off), C.byref(tot))
    assert st == 0
    state = dict(state, cap=cap, terminated=dec)
    O.gang_order_mt(state, 1, cfg["limit"], cfg["prior"], now, nth)
    dt = time.perf_counter() - t0
    return n / dt, dt, (f"{n} programs ({sizes[0]} SC / {sizes[1]} CoT / {sizes[2]} MCTS+Rebase), {dt:.2f} s "
                        "(reference certaindex functions + SPEC allocate/sort ports)")


def cpu_intern(cfg, nth, n, seed):
    """The reference's K1 work (oracle/_ref): rows of S answers materialised as std::string,
    metrics::cluster_exact (trim + string_view map) + probe::flag_hesitation per answer."""
    import numpy as np

    from oracle import oracle as O
    from paper_2412_20993_b200 import synth
    ids = O.gen_sc(O.gen_params(seed=seed, conv_hi=64), max(1, n // (64 * cfg["S"])), 64, cfg["S"]).reshape(-1)[:n]
    arena, off = synth.answer_arena_np(ids, cfg["width"])
    O.ref_intern_batch(arena, off[: 1 + max(1, n // 64)], cfg["S"], nthreads=nth)  # warm
    t0 = time.perf_counter()
    O.ref_intern_batch(arena, off, cfg["S"], nthreads=nth, want=False)
    dt = time.perf_counter() - t0
    return n / dt, dt, f"{n} answers in rows of {cfg['S']}, {dt:.2f} s"


CPU = {"sc": cpu_sc, "cot": cpu_cot, "reward": cpu_reward, "gang": cpu_gang, "jsonl": cpu_jsonl, "mixed": cpu_mixed,
       "intern": cpu_intern}
CPU_SAMPLE = {"A": 1024, "B": 1 << 16, "C": 1 << 18, "D": 1 << 14, "E": 1 << 15, "G": 1 << 20, "J": 1 << 17,
              "K": 1 << 22}


def cpu_baseline(name, cfg, sample=None, target_s=1.0, max_reps=64):
    """The CPU path on repeated bounded samples (fresh seed each) until `target_s` seconds
    of timed CPU work have accumulated; value = total work / total timed seconds."""
    nth = host_threads()
    n = sample or CPU_SAMPLE[name]
    work = secs = 0.0
    reps = 0
    note = ""
    while reps < max_reps and (reps == 0 or secs < target_s):
        v, dt, note = CPU[cfg["kind"]](cfg, nth, n, 20993 + 1 + reps)
        work += v * dt
        secs += dt
        reps += 1
    kind = "port" if cfg["kind"] == "gang" else "reference"
    return {"value": work / secs, "unit": UNIT, "cores": nth, "kind": kind,
            "sample": f"config {name}: {reps} x [{note}], {secs:.1f} s timed in total"}


def run_reference(args, cfg, rank, world):
    """--impl reference: rank 0 times the reference's CPU path; other ranks exit."""
    if rank != 0:
        return
    vals = []
    n = args.ref_sample or CPU_SAMPLE[args.config]
    nth = host_threads()
    note = ""
    for i in range(args.warmup + args.steps):
        v, dt, note = CPU[cfg["kind"]](cfg, nth, n, 20993 + i)
        if i >= args.warmup:
            vals.append((v, dt))
    v = statistics.median([x[0] for x in vals])
    ms = statistics.median([x[1] for x in vals]) * 1e3
    kind = "port" if cfg["kind"] == "gang" else "reference"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 ids / f64 certaindex", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nth, "kind": kind,
                             "sample": f"config {args.config}: {note} (per step)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU legs
L2_FLUSH_BYTES = 512 << 20  # > the 126 MB L2
NOMINAL_HBM_GBS = 8000.0     # B200 nominal HBM3e (SURVEY.md §8(d) reports against both)


def timed(args, world, launch, kernels, flush_l2=False):
    """Warm up, then time exactly `steps` calls of launch(i) on torch's current stream with
    CUDA events (barrier + synchronize on both sides, max over ranks).  `kernels` names the
    segments launch() brackets with per-segment events (for per-kernel durations).
    flush_l2 (working sets that fit in L2): a 512 MB buffer is rewritten before every step,
    outside the step's own event pair, and the step time is the sum of the per-step pairs."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        launch(None)
    torch.cuda.synchronize()
    barrier(world)
    seg = {k: [] for k in kernels}
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    junk = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda") if flush_l2 else None
    pairs = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            if junk is not None:
                junk.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                launch(seg)
                b.record(stream)
                pairs.append((a, b))
            else:
                launch(seg)
        t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    total = sum(a.elapsed_time(b) for a, b in pairs) if pairs else t0.elapsed_time(t1)
    ms = max_over_ranks(total, world) / args.steps
    per = {k: statistics.mean(a.elapsed_time(b) for a, b in v) if v else None for k, v in seg.items()}
    return ms, per, clk.summary()


def in_timed(cx, l0, args):
    """Kernel launches of ours inside the timed region: every step issues the same set, so
    the count since l0 (warm-up + timed steps) scales to the timed steps."""
    return (cx.launches - l0) * args.steps // (args.steps + args.warmup)


def seg_events(seg, name):
    import torch
    if seg is None:
        return None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(torch.cuda.current_stream())
    seg[name].append((a, b))
    return b


def bench_sc(args, cfg, rank, world, cx, with_e2e=True):
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    R, P, S = cfg["R"], cfg["P"], cfg["S"]
    ids = cx.gen_sc(GenParams(seed=20993 + 3, conv_hi=cfg["conv_hi"]), R, P, S, r0=rank * R)
    hcert = torch.empty((R, P), dtype=torch.float32, device="cuda")
    meets = torch.empty((R, (P + 31) // 32), dtype=torch.int32, device="cuda")
    ths = [Threshold(0, cfg["tau"], 0)]
    pol = AllocPolicy(kind=2, detect_at=cfg["detect"], resource_cap=cfg["cap"], tokens_per_unit=cfg["interval"] * S)
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_knob", torch.int32), ("reason", torch.uint8), ("granted", torch.int32), ("offsets", torch.int64),
            ("kept", torch.int32))}
    out["scalars"] = torch.zeros((3,), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    from paper_2412_20993_b200.sharding import Sharded
    sh = Sharded(cx)

    def step(seg):
        if world == 1:  # K2 + K5 through one call (cdx_sc_decide: two launches back to back)
            e = seg_events(seg, "sc_decide")
            cx.sc_decide(ids, ths, pol, hcert=hcert, meets=meets, kept_base=rank * R, out=out)
            if e is not None:
                e.record(torch.cuda.current_stream())
            return
        e = seg_events(seg, "sc_certaindex")
        cx.sc_certaindex(ids, ths, hcert=hcert, meets=meets)
        if e is not None:
            e.record(torch.cuda.current_stream())
        e = seg_events(seg, "allocate_scan")
        if sh.native:  # global offsets / kept / totals: one 32-B-per-rank allgather inside
            cx.allocate_scan_sharded(meets, R, P, pol, out=out)
        else:
            cx.allocate_scan(meets, R, P, pol, kept_base=rank * R, out=out)
            totals = sh.allgather(out["scalars"][2:3])
            cx.offsets_rebase(out["offsets"], totals, rank)
        if e is not None:
            e.record(torch.cuda.current_stream())

    if cfg.get("graph") and world == 1:
        # launch-bound size: capture K2 + K5 once, replay the graph (one launch per step)
        g = cx.graph_capture(lambda: step(None))

        def step(seg):  # noqa: F811 - the timed step is the graph replay
            e = seg_events(seg, "sc_decide")
            g()
            if e is not None:
                e.record(torch.cuda.current_stream())

    l0 = cx.launches
    segs = ["sc_decide"] if world == 1 else ["sc_certaindex", "allocate_scan"]
    ms, per, clocks = timed(args, world, step, segs, cfg.get("flush_l2", False))
    launches = in_timed(cx, l0, args)
    n_kept = int(out["scalars"][0])
    k2_bytes = R * P * S * 4 + R * P * 4 + R * ((P + 31) // 32) * 4
    k5_bytes = R * ((P + 31) // 32) * 4 + R * (4 + 1 + 4 + 8) + n_kept * 4
    if world == 1:  # the call's kernels: K2's algorithmic bytes plus K5's
        res = dict(value=R * P * S * world / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                   kernel="sc_decide (K2 sc_certaindex + K5 allocate_scan)", kernel_ms=per["sc_decide"],
                   kernel_bytes=k2_bytes + k5_bytes, step_bytes=k2_bytes + k5_bytes,
                   extra={"sc_certaindex_bytes": k2_bytes, "allocate_scan_bytes": k5_bytes})
    else:
        res = dict(value=R * P * S * world / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                   kernel="sc_certaindex", kernel_ms=per["sc_certaindex"], kernel_bytes=k2_bytes,
                   step_bytes=k2_bytes + k5_bytes, extra={"allocate_scan_ms": per["allocate_scan"],
                                                          "allocate_scan_bytes": k5_bytes})
    res["e2e"] = e2e_sc(args, cfg, cx, ids, ths, pol, world) if (with_e2e and not args.no_e2e) else None
    del ids
    return res


def e2e_sc(args, cfg, cx, ids_dev, ths, pol, world=1):
    """The same step through the C-ABI host entry cdx_sc_decide_host: ids from pinned host
    memory, H2D + K2 + K5 + D2H of every decision inside the timed region.  At N > 1 every
    rank streams its own shard from its own pinned buffers; barrier on both sides, the
    slowest rank's time, whole-job throughput."""
    import ctypes as C

    import torch
    from paper_2412_20993_b200 import c_policy, c_thresholds
    R, P, S = cfg["R"], cfg["P"], cfg["S"]
    host_ids = torch.empty((R, P, S), dtype=torch.int32, pin_memory=True)
    host_ids.copy_(ids_dev)
    ek = torch.empty((R,), dtype=torch.int32, pin_memory=True)
    why = torch.empty((R,), dtype=torch.uint8, pin_memory=True)
    off = torch.empty((R,), dtype=torch.int64, pin_memory=True)
    saved = C.c_int64(0)
    arr, n = c_thresholds(ths)
    cp = c_policy(pol)

    def one():
        cx._check(cx.lib.cdx_sc_decide_host(cx.h, host_ids.data_ptr(), R, P, S, arr, n, C.byref(cp), ek.data_ptr(),
                                            why.data_ptr(), off.data_ptr(), None, C.byref(saved)))

    for _ in range(max(1, args.warmup)):
        one()
    steps = max(1, min(args.steps, 5))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, world)
    barrier(world)
    return {"value": R * P * S * world / dt, "unit": UNIT, "h2d_bytes_per_step": R * P * S * 4 * world,
            "d2h_bytes_per_step": (R * (4 + 1 + 8) + 16) * world, "ms_per_step": dt * 1e3,
            "api": "cdx_sc_decide_host (C-ABI, pinned host buffers, wall clock)"}


def bench_cot(args, cfg, rank, world, cx, with_e2e=True):
    import torch
    from paper_2412_20993_b200 import GenParams, ProbeConfig
    R, P = cfg["R"], cfg["P"]
    ids, hes = cx.gen_cot(GenParams(seed=20993 + 2, conv_hi=cfg["conv_hi"], hesitation_prob=cfg["hes"]), R, P,
                          r0=rank * R)
    pc = ProbeConfig(cfg["interval"], cfg["w"], cfg["tau"], cfg["max_tokens"])
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_step", torch.int32), ("reason", torch.uint8), ("final_id", torch.int32), ("low_conf", torch.uint8))}

    def step(seg):
        e = seg_events(seg, "cot_exit")
        cx.cot_exit(ids, hes, pc, out=out)
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["cot_exit"])
    b = R * P * 4 + R * ((P + 63) // 64) * 8 + R * (4 + 1 + 4 + 1)
    launches = in_timed(cx, l0, args)
    e2e = None
    if with_e2e and not args.no_e2e:
        host = dict(ids=torch.empty((R, P), dtype=torch.int32, pin_memory=True),
                    hes=torch.empty(hes.shape, dtype=torch.int64, pin_memory=True))
        host["ids"].copy_(ids)
        host["hes"].copy_(hes)
        outs = {k: torch.empty((R,), dtype=dt, pin_memory=True) for k, dt in
                (("exit_step", torch.int32), ("reason", torch.uint8), ("final_id", torch.int32),
                 ("low_conf", torch.uint8))}
        e2e = e2e_host(args, world, lambda: cx.cot_decide_host(host["ids"], host["hes"], pc, out=outs),
                       R * P * world, R * P * 4 + hes.numel() * 8, R * 10,
                       "cdx_cot_decide_host (C-ABI, pinned host buffers, wall clock)")
    return dict(value=R * P * world / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                kernel="cot_exit", kernel_ms=per["cot_exit"], kernel_bytes=b, step_bytes=b, extra={}, e2e=e2e)


def e2e_host(args, world, one, units, h2d, d2h, api):
    """Time `one()` (a host-buffer entry: H2D + kernels + D2H, returns with results on the host)
    on the wall clock; barrier on both sides, the slowest rank, whole-job throughput."""
    for _ in range(max(1, min(args.warmup, 3))):
        one()
    steps = max(1, min(args.steps, 5))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, world)
    barrier(world)
    return {"value": units / dt, "unit": UNIT, "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
            "ms_per_step": dt * 1e3, "api": api}


def bench_reward(args, cfg, rank, world, cx, with_e2e=True):
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    G, T, W = cfg["G"], cfg["T"], cfg["W"]
    rw, ids = cx.gen_reward(GenParams(seed=20993 + 4, conv_hi=cfg["conv_hi"]), G, T, W, g0=rank * G)
    agg = (torch.arange(G, device="cuda") % 2).to(torch.uint8)  # even MCTS (mean), odd Rebase (max)
    thm = [Threshold(*t) for t in TH_MCTS]
    thx = [Threshold(*t) for t in TH_REBASE]
    pol = AllocPolicy(kind=2, detect_at=cfg["detect"], resource_cap=T, tokens_per_unit=W)
    state = {}

    def step(seg):
        e = seg_events(seg, "reward_certaindex")
        R_, H_, m_ = cx.reward_certaindex(rw, ids, agg, thm, thx)
        if e is not None:
            e.record(torch.cuda.current_stream())
        e = seg_events(seg, "allocate_scan")
        state["alloc"] = cx.allocate_scan(m_, G, T, pol)
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["reward_certaindex", "allocate_scan"])
    b = G * T * W * 8 + G * T * 8 + G * ((T + 31) // 32) * 4
    launches = in_timed(cx, l0, args)
    e2e = None
    if with_e2e and not args.no_e2e:
        host = dict(rw=torch.empty((G, T, W), dtype=torch.float32, pin_memory=True),
                    ids=torch.empty((G, T, W), dtype=torch.int32, pin_memory=True),
                    agg=torch.empty((G,), dtype=torch.uint8, pin_memory=True))
        host["rw"].copy_(rw)
        host["ids"].copy_(ids)
        host["agg"].copy_(agg)
        outs = {k: torch.empty(shape, dtype=dt, pin_memory=True) for k, shape, dt in
                (("exit_knob", (G,), torch.int32), ("reason", (G,), torch.uint8), ("offsets", (G,), torch.int64),
                 ("R", (G, T), torch.float32))}
        e2e = e2e_host(args, world, lambda: cx.reward_decide_host(host["rw"], host["ids"], host["agg"], thm, thx, pol,
                                                                  out=outs),
                       G * T * W * world, G * T * W * 8 + G, G * (4 + 1 + 8 + T * 4),
                       "cdx_reward_decide_host (C-ABI, pinned host buffers, wall clock)")
    return dict(value=G * T * W * world / (ms / 1e3), ms=ms, launches=launches,
                clocks=clocks, kernel="reward_certaindex", kernel_ms=per["reward_certaindex"], kernel_bytes=b,
                step_bytes=b + G * 21, extra={"allocate_scan_ms": per["allocate_scan"]}, e2e=e2e)


def bench_gang(args, cfg, rank, world, cx, with_e2e=True):
    """Config G.  N=1: one radix-sorted order of all programs.  N>1: the 4M programs are
    sharded (strong scaling of the fixed trace), each rank sorts its shard and the global
    order comes from the distributed sample sort (cdx_gang_priority_sharded: samples
    allgather, keys alltoallv to their bucket's rank, merge, ids allgather)."""
    import numpy as np
    import torch
    from paper_2412_20993_b200 import InterPolicy
    from paper_2412_20993_b200.sharding import Sharded, shard_range
    N = cfg["N"]
    soa, now = gang_inputs(N, 20993 + 5, cfg["limit"])
    g0, gn = shard_range(N, rank, world)
    dev = {k: (torch.from_numpy(np.ascontiguousarray(v[g0:g0 + gn]).view(np.int16)) if v.dtype == np.uint16
               else torch.from_numpy(np.ascontiguousarray(v[g0:g0 + gn]))).cuda() for k, v in soa.items()}
    pol = InterPolicy(order=1, starvation_limit=cfg["limit"], prior_tokens=cfg["prior"])
    sh = Sharded(cx)
    gorder = torch.empty((N,), dtype=torch.int32, device="cuda")

    def step(seg):
        e = seg_events(seg, "gang_priority")
        if world == 1:
            cx.gang_priority(dev, pol, now, out=gorder)
        elif sh.native:
            cx.gang_priority_sharded(dev, pol, now, id_base=g0, capacity=N, out=gorder)
        else:
            sh.gang_order(dev, pol, now, g0, capacity=N)
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["gang_priority"])
    b = gn * (8 + 8 + 8 + 4 + 4 + 4 + 1) + gn * 4
    launches = in_timed(cx, l0, args)
    e2e = None
    if with_e2e and not args.no_e2e:
        host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in dev.items()}
        for k, v in dev.items():
            host[k].copy_(v)
        stage = {k: torch.empty_like(v) for k, v in dev.items()}
        res = {}

        def one():
            for k, v in host.items():
                stage[k].copy_(v, non_blocking=True)
            order = cx.gang_priority(stage, pol, now)[0] if world == 1 else \
                sh.gang_order(stage, pol, now, g0, capacity=N)
            res["order"] = order.cpu()
        e2e = e2e_host(args, world, one, N, sum(v.numel() * v.element_size() for v in host.values()), gn * 4,
                       "Context.gang_priority (C-ABI) from pinned host buffers, order read back, wall clock")
    return dict(value=N / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                kernel="gang_priority (radix sort, all passes)" + (" + sample-sort exchange" if world > 1 else ""),
                kernel_ms=per["gang_priority"], kernel_bytes=b, step_bytes=b, extra={}, e2e=e2e,
                scaling="strong")


def bench_jsonl(args, cfg, rank, world, cx, with_e2e=True):
    """Config J: device-resident JSONL text -> parsed, checked, interned records."""
    import torch
    text = jsonl_text(cfg["lines"], cfg["programs"], 20993 + 6 + rank)
    dev = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    cap = cfg["lines"] + 1
    out = {}

    def step(seg):
        e = seg_events(seg, "jsonl_parse")
        out.update(cx.jsonl_parse(dev, cap))
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["jsonl_parse"], cfg.get("flush_l2", False))
    launches = in_timed(cx, l0, args)
    n = out["n_records"]
    b = len(text) + n * (4 + 4 + 8 + 1 + 8 + 8) + n * 8
    e2e = None
    if with_e2e and not args.no_e2e:
        host_text = torch.frombuffer(bytearray(text), dtype=torch.uint8).pin_memory()
        stage = torch.empty_like(dev)
        keep = {}

        def one():
            stage.copy_(host_text, non_blocking=True)
            o = cx.jsonl_parse(stage, cap)
            keep.update({k: o[k][:o["n_records"]].cpu() for k in ("program", "step_index", "token_offset", "hesitant")})
        e2e = e2e_host(args, world, one, n * world, len(text), n * 17,
                       "Context.jsonl_parse (C-ABI) from a pinned host text buffer, records read back, wall clock")
    return dict(value=n * world / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                kernel="jsonl_parse (all passes)", kernel_ms=per["jsonl_parse"], kernel_bytes=b, step_bytes=b,
                extra={"text_bytes": len(text)}, e2e=e2e)


def bench_intern(args, cfg, rank, world, cx, with_e2e=True):
    """Config K: K1 over a device-resident answer arena (trim, hash, insert, byte-verify,
    dense first-seen ids, hesitation flags).  Answers shard by rank (weak scaling)."""
    import torch
    from paper_2412_20993_b200 import GenParams, synth
    n, S, wd = cfg["n"], cfg["S"], cfg["width"]
    R = n // (64 * S)
    ids = cx.gen_sc(GenParams(seed=20993 + 8, conv_hi=64), R, 64, S, r0=rank * R).view(-1)
    arena, off = synth.answer_arena_torch(ids, wd)
    del ids
    torch.cuda.synchronize()
    out = {}

    def step(seg):
        e = seg_events(seg, "canon_intern")
        out["r"] = cx.canon_intern(arena, off)
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["canon_intern"])
    launches = in_timed(cx, l0, args)
    b = n * wd + (n + 1) * 8 + n * 4 + n
    e2e = None
    if with_e2e and not args.no_e2e:
        h_arena = torch.empty(arena.shape, dtype=torch.uint8, pin_memory=True)
        h_off = torch.empty(off.shape, dtype=torch.int64, pin_memory=True)
        h_arena.copy_(arena)
        h_off.copy_(off)
        s_arena, s_off = torch.empty_like(arena), torch.empty_like(off)
        keep = {}

        def one():
            s_arena.copy_(h_arena, non_blocking=True)
            s_off.copy_(h_off, non_blocking=True)
            r = cx.canon_intern(s_arena, s_off)
            keep["ids"], keep["hes"] = r[0].cpu(), r[1].cpu()
        e2e = e2e_host(args, world, one, n * world, (arena.numel() + off.numel() * 8), n * 5,
                       "Context.canon_intern (C-ABI) from pinned host arena + offsets, ids and flags read back, "
                       "wall clock")
    return dict(value=n * world / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
                kernel="canon_intern (all passes)", kernel_ms=per["canon_intern"], kernel_bytes=b, step_bytes=b,
                extra={"unique_answers": int(out["r"][3]), "arena_bytes": n * wd}, e2e=e2e)


def bench_mixed(args, cfg, rank, world, cx, with_e2e=True):
    """Config E: one online scheduling round over the mixed trace.  Traces of each archetype
    group are generated on the device (rows of the rank's programs only); the timed step is
    cdx_mixed_allocate (K2 on the SC rows, cot_meets on the CoT rows, K4 on the MCTS / Rebase
    rows, allocate at every program's knob, budget scan) followed by the gang order of the
    live programs (K6; at N > 1 sharded with the key allgather + merge).  Programs shard
    contiguously across ranks; the round is identical to the single-GPU one."""
    import numpy as np
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, InterPolicy, Threshold
    from paper_2412_20993_b200.sharding import Sharded, shard_range
    N = cfg["N"]
    (scP, S), (cotP, w), (T, W) = cfg["sc"], cfg["cot"], cfg["rw"]
    arch, slot, sizes, knob, state, now = mixed_layout(cfg, N, 20993 + 7)
    g0, gn = shard_range(N, rank, world)
    group = np.where(arch == SC_, 0, np.where(arch == COT_, 1, 2))
    a_r, s_r = arch[g0:g0 + gn], slot[g0:g0 + gn].astype(np.int64)
    r0 = [int((group[:g0] == g).sum()) for g in range(3)]
    n_r = [int((group[g0:g0 + gn] == g).sum()) for g in range(3)]
    gr = group[g0:g0 + gn]
    for g in range(3):
        s_r[gr == g] -= r0[g]
    trace = dict(sc_ids=cx.gen_sc(GenParams(seed=20993 + 10, conv_hi=scP), n_r[0], scP, S, r0=r0[0]),
                 cot_window=w)
    trace["cot_ids"], trace["cot_hes"] = cx.gen_cot(GenParams(seed=20993 + 11, conv_hi=cotP, hesitation_prob=0.05),
                                                    n_r[1], cotP, r0=r0[1])
    trace["rw"], trace["rw_ids"] = cx.gen_reward(GenParams(seed=20993 + 12, conv_hi=T), n_r[2], T, W, g0=r0[2])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    arch_d, slot_d, knob_d = dev(a_r), dev(s_r.astype(np.int32)), dev(knob[g0:g0 + gn])
    st_d = {k: dev(v[g0:g0 + gn]) for k, v in state.items() if k not in ("cap", "knob")}
    st_d["knob"] = knob_d
    pols = [([Threshold(*t) for t in ths], AllocPolicy(**kw)) for ths, kw in
            (mixed_policies(cfg)[a] for a in range(4))]
    ipol = InterPolicy(order=1, starvation_limit=cfg["limit"], prior_tokens=cfg["prior"])
    outbuf = {k: torch.empty((max(gn, 1),), dtype=dt, device="cuda") for k, dt in
              (("decision", torch.uint8), ("grant", torch.int32), ("cap", torch.int32), ("offsets", torch.int64))}
    outbuf["total"] = torch.empty((1,), dtype=torch.int64, device="cuda")
    sh = Sharded(cx)
    gorder = torch.empty((N,), dtype=torch.int32, device="cuda")
    res = {}
    torch.cuda.synchronize()

    def step(seg):
        e = seg_events(seg, "mixed_allocate")
        out = cx.mixed_allocate(trace, arch_d, slot_d, knob_d, pols, out=outbuf)
        if world > 1:  # global budget offsets: allgather of the shard totals + device rebase
            totals = sh.allgather(out["total"])
            cx.offsets_rebase(out["offsets"], totals, rank)
        if e is not None:
            e.record(torch.cuda.current_stream())
        e = seg_events(seg, "gang_priority")
        soa = dict(st_d, terminated=out["decision"], cap=out["cap"])
        if world == 1:
            res["order"] = cx.gang_priority(soa, ipol, now, out=gorder)[0]
        elif sh.native:
            res["order"] = cx.gang_priority_sharded(soa, ipol, now, id_base=g0, capacity=N, out=gorder)
        else:
            res["order"] = sh.gang_order(soa, ipol, now, g0, capacity=N)
        if e is not None:
            e.record(torch.cuda.current_stream())

    l0 = cx.launches
    ms, per, clocks = timed(args, world, step, ["mixed_allocate", "gang_priority"])
    launches = in_timed(cx, l0, args)
    words = lambda u: (u + 31) // 32  # noqa: E731
    trace_b = (n_r[0] * scP * S * 4 + n_r[1] * (cotP * 4 + ((cotP + 63) // 64) * 8) + n_r[2] * T * W * 8)
    table_b = gn * (1 + 4 + 4) + gn * (1 + 4 + 4 + 8)  # arch, slot, knob in; decision, grant, cap, offsets out
    mixed_b = trace_b + table_b
    gang_b = gn * (8 + 8 + 8 + 4 + 4 + 4 + 1) + int(res["order"].shape[0]) * 4
    meets_b = 2 * 4 * (n_r[0] * words(scP) + n_r[1] * words(cotP) + n_r[2] * words(T))  # intermediate round trip
    out = dict(value=N / (ms / 1e3), ms=ms, launches=launches, clocks=clocks,
               kernel="mixed_allocate (K2 + cot_meets + K4 + allocate + budget scan)",
               kernel_ms=per["mixed_allocate"], kernel_bytes=mixed_b, step_bytes=mixed_b + gang_b,
               extra={"gang_priority_ms": per["gang_priority"], "gang_priority_bytes": gang_b,
                      "programs": {"sc": n_r[0], "cot": n_r[1], "mcts_rebase": n_r[2]},
                      "intermediate_meets_bytes": meets_b, "live_programs": int(res["order"].shape[0]),
                      "probe_evals_per_step": n_r[0] * scP * S + n_r[1] * cotP + n_r[2] * T * W,
                      "trace_bytes": trace_b},
               scaling="strong")
    def gang(soa):  # the global order at N > 1, as in the device-timed step
        if world == 1:
            return cx.gang_priority(soa, ipol, now)[0]
        if sh.native:
            return cx.gang_priority_sharded(soa, ipol, now, id_base=g0, capacity=N, out=gorder)
        return sh.gang_order(soa, ipol, now, g0, capacity=N)
    out["e2e"] = e2e_mixed(args, cx, trace, arch_d, slot_d, knob_d, st_d, pols, gang, world, N) \
        if (with_e2e and not args.no_e2e) else None
    return out


def e2e_mixed(args, cx, trace, arch_d, slot_d, knob_d, st_d, pols, gang, world, N):
    """Config E through the public API from pinned host buffers: every step copies the whole
    trace and program table host -> device, runs the mixed step and the gang order, and reads
    the order and the decisions back (wall clock, barrier on both sides, slowest rank)."""
    import torch
    dev_in = dict(sc_ids=trace["sc_ids"], cot_ids=trace["cot_ids"], cot_hes=trace["cot_hes"], rw=trace["rw"],
                  rw_ids=trace["rw_ids"], arch=arch_d, slot=slot_d, **st_d)  # st_d holds the knob
    host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in dev_in.items()}
    for k, v in dev_in.items():
        host[k].copy_(v)
    stage = {k: torch.empty_like(v) for k, v in dev_in.items()}
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    res = {}

    def one():
        for k, v in host.items():
            stage[k].copy_(v, non_blocking=True)
        tr = dict(sc_ids=stage["sc_ids"], cot_ids=stage["cot_ids"], cot_hes=stage["cot_hes"], rw=stage["rw"],
                  rw_ids=stage["rw_ids"], cot_window=trace["cot_window"])
        out = cx.mixed_allocate(tr, stage["arch"], stage["slot"], stage["knob"], pols)
        soa = {k: stage[k] for k in ("arrival", "last_service", "iter_tok_sum", "iter_count", "knob")}
        soa.update(terminated=out["decision"], cap=out["cap"])
        res["order"] = gang(soa).cpu()
        res["decision"] = out["decision"].cpu()

    for _ in range(max(1, min(args.warmup, 2))):
        one()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, world)
    barrier(world)
    d2h = res["order"].numel() * 4 + res["decision"].numel()
    return {"value": N / dt, "unit": UNIT, "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
            "ms_per_step": dt * 1e3,
            "api": "Context.mixed_allocate + Context.gang_priority (C-ABI) from pinned host buffers, wall clock"}


BENCH = {"mixed": bench_mixed, "sc": bench_sc, "cot": bench_cot, "reward": bench_reward, "gang": bench_gang,
         "jsonl": bench_jsonl, "intern": bench_intern}


def summarize(name, cfg, res, peak):
    ach = res["kernel_bytes"] / (res["kernel_ms"] / 1e3) / 1e9
    return {"value": res["value"], "unit": UNIT, "ms_per_step": res["ms"], "desc": cfg["desc"], "e2e": res.get("e2e"),
            "gpu_launches": res["launches"], "clocks": res["clocks"],
            "kernel": res["kernel"], "kernel_ms": res["kernel_ms"], "achieved_gbs": ach, "frac": ach / peak,
            "frac_nominal": ach / NOMINAL_HBM_GBS,
            "l2": "flushed before every timed step" if cfg.get("flush_l2") else "inputs > L2", **res["extra"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the other configs at N=1")
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="timed CPU work for the headline cpu_baseline (other configs: 1 s each)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    rank, world, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    from paper_2412_20993_b200 import Context
    if world > 1 and os.environ.get("CDX_BENCH_BACKEND", "nccl") == "nccl":
        # the context owns an NCCL communicator spanning the job (cdx_ctx_create_comm): the
        # exchange steps run through the C-ABI sharded entries, as a C++ caller would
        cx = Context.for_process_group(local)
    else:
        cx = Context(local)
    peak, peak_src = load_peaks()
    res = BENCH[cfg["kind"]](args, cfg, rank, world, cx)
    others = {}
    if world == 1 and not args.no_others:
        sub = argparse.Namespace(**vars(args))
        sub.steps, sub.warmup = min(args.steps, 20), 3
        for name, c in CONFIGS.items():
            if name == args.config:
                continue
            r = BENCH[c["kind"]](sub, c, 0, 1, cx, with_e2e=True)
            others[name] = summarize(name, c, r, peak)
            if not args.no_cpu_baseline:
                others[name]["cpu_baseline"] = cpu_baseline(name, c)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, cfg, args.ref_sample or None, target_s=args.cpu_seconds)
    if rank == 0:
        traffic = load_traffic(cfg["kind"])
        ach = res["kernel_bytes"] / (res["kernel_ms"] / 1e3) / 1e9
        cfg_out = {"workload": args.config, "desc": cfg["desc"],
                   **{k: v for k, v in cfg.items() if k not in ("kind", "desc", "conv_hi")},
                   "parallelism": (f"program shards x{world}, distributed sample sort (samples allgather, "
                                   "keys alltoallv, merge, ids allgather)"
                                   if cfg["kind"] in ("gang", "mixed") else
                                   f"request shards x{world} (no data-path collective; 8 B/rank allgather "
                                   "of budget totals for global offsets)"),
                   "l2": ("L2 flushed before every timed step (512 MB write, outside the step's events)"
                          if cfg.get("flush_l2") else "inputs > L2 (126 MB): no flush needed")}
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms"], "higher_is_better": True,
            "scaling": res.get("scaling", "weak"),
            "vs_baseline": None, "dtype": "u32 ids / f64 certaindex (f32 store)", "data": "synthetic",
            "config": cfg_out,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "frac_nominal": ach / NOMINAL_HBM_GBS,  # also vs the 8 TB/s nominal
                         "traffic": traffic["bytes"] if traffic else None,
                         "traffic_source": traffic and f"{traffic['source']} ({traffic['kernel'][:60]})",
                         "peak_source": peak_src, "kernel": res["kernel"],
                         "kernel_ms": res["kernel_ms"], "algorithmic_bytes_per_launch": res["kernel_bytes"],
                         "step_bytes": res["step_bytes"],
                         "step_frac": res["step_bytes"] / (res["ms"] / 1e3) / 1e9 / peak, **res["extra"]},
            "cpu_baseline": cpu,
            "e2e": res["e2e"],
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
        }
        if others:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
