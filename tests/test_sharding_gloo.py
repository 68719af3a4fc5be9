"""Multi-rank host logic of the sharded path (paper_2412_20993_b200/sharding.py) on CPU:
world_size 2 over gloo, 127.0.0.1.  The exchange steps (allgather of shard budget totals +
device rebase; allgather of padded sorted key runs + merge) run exactly as on the B200
box; only the compute provider is a checker-backed stand-in (oracle/), since this
container has no GPU.  The sharded results must equal the single-process oracle:
global token offsets and kept lists for SC (K5), the global gang order for K6.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2412_20993_b200.sharding import Sharded, max_shard, shard_range

R, P, S = 96, 16, 8
N_PROG = 1000


class CheckerOps:
    """The Context methods sharding.py calls, evaluated by the CPU checker (test only)."""

    def sc_certaindex(self, ids, ths, hcert=None, meets=None):
        _, h32, m = O.sc_certaindex(ids.numpy().view(np.uint32), [(t.signal, t.cutoff, t.dir) for t in ths])
        return torch.from_numpy(h32), torch.from_numpy(m.view(np.int32))

    def allocate_scan(self, meets, R_, P_, pol, kept_base=0, out=None):
        r = O.allocate_scan(meets.numpy().view(np.uint32), R_, P_, pol.kind, pol.detect_at, pol.resource_cap,
                            pol.recheck_every, pol.tokens_per_unit)
        budget = int((r["granted"].astype(np.int64) * pol.tokens_per_unit).sum())
        return dict(exit_knob=torch.from_numpy(r["exit_knob"]), offsets=torch.from_numpy(r["offsets"].copy()),
                    kept=torch.from_numpy(r["kept"].astype(np.int64) + kept_base),
                    scalars=torch.tensor([r["n_kept"], r["tokens_saved"], budget], dtype=torch.int64))

    def offsets_rebase(self, offsets, totals, rank):
        offsets += int(totals[:rank].sum())

    def gang_priority(self, soa, pol, now, id_base=0, want_keys=False):
        """Composite keys of cdx_gang_priority (k_gang.cu: {esc?0:1 <<63 | bits(key),
        bits(arrival), id}) in sorted order; the order itself is pinned to the oracle."""
        a = {k: v.numpy() for k, v in soa.items()}
        n = len(a["arrival"])
        esc = (now - a["last_service"]) >= pol.starvation_limit
        cnt = a["iter_count"].astype(np.float64)
        est = np.where(a["iter_count"] > 0, a["iter_tok_sum"] / np.maximum(cnt, 1), pol.prior_tokens)
        rem = np.maximum(a["cap"].astype(np.int64) - a["knob"].astype(np.int64), 0)
        pkey = a["arrival"] if pol.order == 0 else est * rem
        key = np.where(esc, a["arrival"], pkey) + 0.0  # -0.0 -> +0.0
        hi = key.view(np.uint64) | (np.where(esc, 0, 1).astype(np.uint64) << np.uint64(63))
        keys = np.stack([hi, a["arrival"].view(np.uint64), np.arange(n, dtype=np.uint64) + id_base], 1)
        keys = keys[a["terminated"] == 0]
        keys = keys[np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))]
        ref, _ = O.gang_order(a, pol.order, pol.starvation_limit, pol.prior_tokens, now, id_base=id_base)
        assert np.array_equal(keys[:, 2].astype(np.uint32), ref), "stand-in keys disagree with the oracle order"
        k = torch.from_numpy(keys.view(np.int64))
        return torch.from_numpy(ref.view(np.int32)), None, k

    # device building blocks of the sample sort (shard.cu), restated on the host
    def shard_samples(self, keys, s):
        k = keys.numpy().view(np.uint64)
        n = k.shape[0]
        if n == 0:
            return torch.full((s, 3), -1, dtype=torch.int64)
        idx = ((2 * np.arange(s, dtype=np.uint64) + 1) * n) // (2 * s)
        return torch.from_numpy(np.ascontiguousarray(k[idx]).view(np.int64))

    def shard_bounds(self, keys, split, world):
        k = [tuple(r) for r in keys.numpy().view(np.uint64).tolist()]
        sp = [tuple(r) for r in split.numpy().view(np.uint64).tolist()]
        import bisect
        b = [0] + [bisect.bisect_left(k, x) for x in sp] + [len(k)]
        return torch.tensor(b, dtype=torch.int64)

    def gang_merge_runs(self, keys, run_off):
        rows = keys.numpy().view(np.uint64)
        rows = rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]
        return torch.from_numpy(rows[:, 2].astype(np.uint32).view(np.int32))

    def gang_merge(self, recv, lens, stride, total=None):
        keys = recv.numpy().view(np.uint64)
        rows = np.concatenate([keys[q * stride: q * stride + int(lens[q])] for q in range(len(lens))])
        rows = rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]
        if total is not None:
            total[0] = len(rows)
        out = np.zeros(len(lens) * stride, np.uint32)
        out[: len(rows)] = rows[:, 2]
        return torch.from_numpy(out.view(np.int32))


def _inputs():
    ids = O.gen_sc(O.gen_params(seed=11, conv_hi=P), R, P, S)
    rng = np.random.default_rng(3)
    arrival = np.cumsum(rng.exponential(1e-3, N_PROG))
    arrival[0:-1:7] = arrival[1::7]  # arrival ties -> the (arrival, id) tie-break is exercised
    now = float(arrival.max()) + 1e-3
    cnt = rng.integers(0, 5, N_PROG).astype(np.uint32)
    soa = dict(arrival=arrival, last_service=now - rng.exponential(0.2, N_PROG),
               iter_tok_sum=(rng.integers(1, 500, N_PROG) * cnt).astype(np.int64), iter_count=cnt,
               cap=rng.integers(1, 30, N_PROG).astype(np.int32), terminated=(rng.random(N_PROG) < 0.2).astype(np.uint8))
    soa["knob"] = np.minimum(soa["cap"], rng.integers(0, 30, N_PROG)).astype(np.int32)
    soa["last_service"] = np.maximum(soa["last_service"], 0.0)
    return ids, soa, now


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_20993_b200 import AllocPolicy, InterPolicy, Threshold
        ids, soa, now = _inputs()
        sh = Sharded(CheckerOps())
        r0, n = shard_range(R, rank, world)
        pol = AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S)
        res = sh.sc_decide(torch.from_numpy(ids[r0:r0 + n].view(np.int32)), [Threshold(0, 0.7, 0)], pol, r0)
        g0, gn = shard_range(N_PROG, rank, world)
        part = {k: torch.from_numpy(np.ascontiguousarray(v[g0:g0 + gn])) for k, v in soa.items()}
        order = sh.gang_order(part, InterPolicy(order=1, starvation_limit=0.15, prior_tokens=128.0), now, g0)
        q.put((rank, res["offsets"].numpy(), res["kept"].numpy(), res["shard_totals"].numpy(),
               order.numpy().view(np.uint32)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        item = q.get(timeout=300)
        got[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ids, soa, now = _inputs()
    _, _, meets = O.sc_certaindex(ids, [(0, 0.7, 0)])
    ref = O.allocate_scan(meets, R, P, 2, 5, P, 1, 64 * S)
    offsets = np.concatenate([got[r][0] for r in range(world)])
    kept = np.concatenate([got[r][1] for r in range(world)])
    assert np.array_equal(offsets, ref["offsets"])
    assert np.array_equal(kept, ref["kept"].astype(np.int64))
    for r in range(1, world):
        assert np.array_equal(got[0][2], got[r][2])
    gref, _ = O.gang_order(soa, 1, 0.15, 128.0, now)
    for r in range(world):
        assert np.array_equal(got[r][3], gref)


def test_shard_range_covers():
    for n in (0, 1, 7, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == n
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max_shard(n, w) == max(c for _, c in spans)


@pytest.mark.parametrize("world,seed", [(2, 0), (3, 1), (8, 2), (8, 3), (5, 4)])
def test_shard_splitters_partition_the_global_order(world, seed):
    """The product's host planning step (libcdx cdx_shard_splitters, no device): buckets cut
    by its splitters are contiguous ranges of the global order, every key lands in exactly
    one bucket, and buckets are balanced to within the sampling error."""
    from paper_2412_20993_b200 import shard_splitters
    from paper_2412_20993_b200.sharding import SHARD_SAMPLES as s
    rng = np.random.default_rng(seed)
    sizes = rng.integers(0, 3000, world)
    sizes[rng.integers(0, world)] = 0  # an empty rank
    runs = []
    for q in range(world):
        k = np.stack([rng.integers(0, 50, sizes[q]).astype(np.uint64) << np.uint64(40),
                      rng.integers(0, 4, sizes[q]).astype(np.uint64),
                      rng.permutation(100000)[: sizes[q]].astype(np.uint64) * world + q], 1)
        runs.append(k[np.lexsort((k[:, 2], k[:, 1], k[:, 0]))])
    samples = np.full((world, s, 3), np.iinfo(np.uint64).max, np.uint64)
    for q in range(world):
        n = len(runs[q])
        if n:
            samples[q] = runs[q][((2 * np.arange(s, dtype=np.uint64) + 1) * n) // (2 * s)]
    split = shard_splitters(samples, sizes.astype(np.uint64), world, s)
    assert split.shape == (world - 1, 3)
    allk = np.concatenate(runs)
    allk = allk[np.lexsort((allk[:, 2], allk[:, 1], allk[:, 0]))]
    tup = [tuple(r) for r in allk.tolist()]
    import bisect
    cuts = [0] + [bisect.bisect_left(tup, tuple(x)) for x in split.tolist()] + [len(tup)]
    assert all(a <= b for a, b in zip(cuts, cuts[1:]))
    total = len(tup)
    # each run contributes s samples standing for n/s keys: a bucket deviates by at most
    # about world runs x 2 sample weights from total/world
    slack = sum(2 * int(sz) // s + 2 for sz in sizes)
    for b in range(world):
        assert abs((cuts[b + 1] - cuts[b]) - total / world) <= slack, (b, cuts, total)
