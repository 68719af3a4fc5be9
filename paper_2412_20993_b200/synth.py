"""Synthetic mixed-program workloads (bench config E and the tests): which archetype each
program has, its row in its archetype's trace tensor, its current knob and its scheduler
state.  Plumbing only — the traces themselves come from the device generators (gen.cu) and
their restatement in oracle/cdx_oracle.c; every decision is made by the kernels.

The mix follows BASELINE.json config E (40 % SC / 40 % CoT / 20 % MCTS-family; the MCTS
fifth is split evenly between MCTS (mean reward) and Rebase (max reward), the two reward
archetypes of runtime.hpp:32)."""
from __future__ import annotations

import numpy as np

ARCH_SC, ARCH_REBASE, ARCH_MCTS, ARCH_COT = 0, 1, 2, 3


def mixed_layout(N: int, seed: int, mix=(0.4, 0.4, 0.1, 0.1)):
    """archetype u8[N] (SC, CoT, MCTS, Rebase with the given fractions, interleaved at
    random), slot u32[N] = running index within the archetype's group (MCTS and Rebase share
    the reward group), and the group sizes."""
    rng = np.random.default_rng(seed)
    u = rng.random(N)
    c = np.cumsum(mix)
    arch = np.where(u < c[0], ARCH_SC, np.where(u < c[1], ARCH_COT, np.where(u < c[2], ARCH_MCTS, ARCH_REBASE)))
    arch = arch.astype(np.uint8)
    group = np.where(arch == ARCH_SC, 0, np.where(arch == ARCH_COT, 1, 2))
    slot = np.zeros(N, np.int64)
    sizes = []
    for g in range(3):
        sel = group == g
        slot[sel] = np.arange(int(sel.sum()))
        sizes.append(int(sel.sum()))
    return arch, slot.astype(np.uint32), sizes


def mixed_knobs(arch, caps, seed: int):
    """Current knob of every program: uniform in [0, cap] of its archetype."""
    rng = np.random.default_rng(seed)
    cap = np.asarray([caps[a] for a in range(4)], np.int64)[arch]
    return (rng.integers(0, 1 << 30, len(arch)) % (cap + 1)).astype(np.int32)


def gang_state(N: int, seed: int, limit: float, knob=None, cap=None):
    """Scheduler-visible program state (runtime.hpp:123-133): Poisson arrivals at 1000
    programs/s, service lags such that ~5 % exceed the starvation limit, completed
    iteration tokens; knob/cap given (the mixed step's) or drawn."""
    rng = np.random.default_rng(seed)
    arrival = np.cumsum(rng.exponential(1e-3, N))
    now = float(arrival[-1]) + 1e-3 if N else 1.0
    last = np.maximum(now - rng.exponential(limit / 3.0, N), 0.0)
    cnt = rng.integers(0, 6, N).astype(np.uint32)
    sums = (rng.integers(32, 1024, N) * cnt).astype(np.int64)
    if cap is None:
        cap = rng.integers(4, 64, N).astype(np.int32)
    if knob is None:
        knob = np.minimum(cap, rng.integers(0, 64, N)).astype(np.int32)
    return dict(arrival=arrival, last_service=last, iter_tok_sum=sums, iter_count=cnt, knob=knob, cap=cap), now


# ---- answer arenas for K1 (bench config K, tests) ------------------------------------------
# Answer i of a synthetic trace (answer id v = 0 "S", 1..4 "D1".."D4" from the answer process)
# as the reference would receive it: every 20th answer (by a hash of i) in its hesitant form
# "wait, <name>" (runtime.cpp:131), surrounded by a mix of the six whitespace bytes trim()
# strips (metrics.cpp:14), in a fixed-width slot of `width` bytes (left pad 0..2 bytes).
VOCAB = ["S", "D1", "D2", "D3", "D4"]
WS = np.frombuffer(b" \t\n\r\f\v", np.uint8)


def _arena_layout(i, xp):
    """(left pad, hesitant) of answers i (int64 array of numpy or torch)."""
    lpad = ((i * 2654435761) >> 8) % 3
    hes = (((i * 0x9E3779B1) & 0xFFFFFFFF) >> 20) % 20 == 0
    return lpad, hes


def answer_arena_np(ids, width: int = 12):
    """numpy: ids u32[n] -> (arena u8[n*width], offsets u64[n+1])."""
    n = len(ids)
    i = np.arange(n, dtype=np.int64)
    lpad, hes = _arena_layout(i, np)
    col = np.arange(width, dtype=np.int64)
    arena = WS[(i[:, None] + 3 * col[None, :]) % 6].astype(np.uint8)
    names = [v.encode() for v in VOCAB]
    for v, nm in enumerate(names):
        for h in (False, True):
            b = np.frombuffer((b"wait, " + nm) if h else nm, np.uint8)
            for L in range(3):
                sel = (ids == v) & (hes == h) & (lpad == L)
                arena[sel, L:L + len(b)] = b
    return arena.reshape(-1), (np.arange(n + 1, dtype=np.uint64) * width)


def answer_arena_torch(ids, width: int = 12, chunk: int = 1 << 24):
    """torch (device): the same bytes as answer_arena_np, built in chunks of answers."""
    import torch
    n = ids.shape[0]
    dev = ids.device
    arena = torch.empty((n, width), dtype=torch.uint8, device=dev)
    ws = torch.from_numpy(WS.copy()).to(dev)
    col = torch.arange(width, dtype=torch.int64, device=dev)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        i = torch.arange(a, b, dtype=torch.int64, device=dev)
        lpad, hes = _arena_layout(i, torch)
        blk = ws[(i[:, None] + 3 * col[None, :]) % 6]
        v_ids = ids[a:b].to(torch.int64)
        for v, nm in enumerate(VOCAB):
            for h in (False, True):
                raw = (b"wait, " + nm.encode()) if h else nm.encode()
                bt = torch.tensor(list(raw), dtype=torch.uint8, device=dev)
                for L in range(3):
                    sel = (v_ids == v) & (hes == h) & (lpad == L)
                    rows = sel.nonzero().squeeze(1)
                    if rows.numel():
                        blk[rows, L:L + len(raw)] = bt
        arena[a:b] = blk
    offsets = torch.arange(n + 1, dtype=torch.int64, device=dev) * width
    return arena.reshape(-1), offsets
