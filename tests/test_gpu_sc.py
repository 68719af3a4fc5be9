"""GPU parity: K2 sc_certaindex + K5 allocate_scan (+ device generator) vs the oracle.

Bit-exact: meets bits, exit knobs, reasons, grants, budget offsets, kept lists, totals.
Certaindex values: the fp32 output must equal the fp32 rounding of the oracle's FP64 value
bit for bit (stronger than the 1e-6 relative tolerance north_star states).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIG_E, SIG_R, GE, LE = 0, 1, 0, 1


def _gp(**kw):
    from paper_2412_20993_b200 import GenParams
    return GenParams(**kw)


def _og(**kw):
    return O.gen_params(**kw)


@pytest.mark.parametrize("R,P,S", [(1, 1, 1), (3, 5, 2), (37, 20, 7), (64, 32, 16), (129, 64, 32), (1000, 64, 32),
                                   (333, 33, 31), (50, 96, 24), (8, 130, 5), (2048, 32, 16)])
def test_generator_matches_oracle(ctx, R, P, S):
    ids = ctx.gen_sc(_gp(seed=R * 7 + P, conv_hi=max(1, P)), R, P, S)
    ref = O.gen_sc(_og(seed=R * 7 + P, conv_hi=max(1, P)), R, P, S)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("R,P,S", [(1, 1, 1), (5, 3, 2), (37, 20, 7), (64, 32, 16), (129, 64, 32), (777, 64, 32),
                                   (333, 33, 31), (50, 96, 24), (8, 130, 5), (2048, 32, 16), (17, 64, 3),
                                   (300, 64, 1), (500, 64, 8), (700, 32, 4), (300, 64, 12),
                                   (301, 63, 32), (500, 48, 16), (257, 50, 16), (333, 9, 8), (1001, 17, 32),
                                   (64, 40, 4), (2000, 64, 24), (999, 64, 31), (1500, 40, 20), (700, 64, 13), (400, 37, 29), (300, 64, 6)])
@pytest.mark.parametrize("ths", [[(SIG_E, 0.7, GE)], [], [(SIG_E, 0.5, GE), (SIG_E, 0.99, LE)]])
def test_sc_certaindex_parity(ctx, R, P, S, ths):
    from paper_2412_20993_b200 import Threshold
    g = dict(seed=1000 + R + S, conv_hi=max(1, P))
    ids = ctx.gen_sc(_gp(**g), R, P, S)
    h, meets = ctx.sc_certaindex(ids, [Threshold(s, c, d) for s, c, d in ths])
    ctx.sync()
    oh64, oh32, ometa = O.sc_certaindex(O.gen_sc(_og(**g), R, P, S), ths)
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(meets.cpu().numpy().view(np.uint32), ometa)


@pytest.mark.parametrize("R,P,S,groups", [(50, 20, 33, 5), (64, 64, 64, 8), (30, 40, 100, 60), (9, 5, 1000, 300),
                                          (2, 3, 4096, 5000), (40, 7, 48, 48)])
def test_sc_certaindex_wide_rows(ctx, R, P, S, groups):
    """More than 32 samples per row (the reference clusters any number): a warp per row,
    first-seen ordinals through a shared-memory hash, the same FP64 fold."""
    import torch
    from paper_2412_20993_b200 import Threshold
    rng = np.random.default_rng(S + P)
    ids = rng.integers(0, groups, size=(R, P, S)).astype(np.uint32)
    ids[:, ::3, :] = ids[:, ::3, :1]  # single-cluster rows
    ths = [(SIG_E, 0.6, GE)]
    h, m = ctx.sc_certaindex(torch.from_numpy(ids.view(np.int32)).cuda(), [Threshold(*t) for t in ths])
    ctx.sync()
    _, oh32, om = O.sc_certaindex(ids, ths)
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(m.cpu().numpy().view(np.uint32), om)


@pytest.mark.parametrize("S", [4, 5, 8, 12, 16])
def test_sc_certaindex_all_compositions(ctx, S):
    """Every first-seen cluster-size composition of S answers (2^(S-1); K2 reads H~ for
    S <= 16 from a per-context table of them), laid out as consecutive label runs, plus a
    shuffled copy of each row: the certaindex bits and meets must equal the oracle's fold."""
    import torch
    from paper_2412_20993_b200 import Threshold
    codes = np.arange(1 << (S - 1), dtype=np.uint64)
    cuts = ((codes[:, None] >> np.arange(S - 1, dtype=np.uint64)) & 1).astype(np.uint32)  # cut after sample j
    labels = np.concatenate([np.zeros((len(codes), 1), np.uint32), np.cumsum(cuts, axis=1, dtype=np.uint32)], 1)
    rows = np.concatenate([labels, np.random.default_rng(S).permuted(labels, axis=1)])
    P = 32
    pad = (-len(rows)) % P
    rows = np.concatenate([rows, np.zeros((pad, S), np.uint32)])
    ids = rows.reshape(-1, P, S)
    ths = [(SIG_E, 0.5, GE)]
    h, m = ctx.sc_certaindex(torch.from_numpy(ids.view(np.int32)).cuda(), [Threshold(*t) for t in ths])
    ctx.sync()
    _, oh32, om = O.sc_certaindex(ids, ths)
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(m.cpu().numpy().view(np.uint32), om)


def test_sc_certaindex_all_partitions_n32(ctx):
    """Every clustering shape of n=32 in several first-seen orders: exercises the ordered
    FP64 fold where naive fp32 or reordered sums flip threshold decisions."""
    import torch
    rng = np.random.default_rng(5)
    rows = []
    def parts(n, mx):
        if n == 0:
            yield []
            return
        for k in range(min(n, mx), 0, -1):
            for rest in parts(n - k, k):
                yield [k] + rest
    for part in parts(32, 32):
        labels = np.concatenate([np.full(c, i, np.uint32) for i, c in enumerate(part)])
        rows.append(labels)
        rows.append(rng.permutation(labels))
    ids_np = np.stack(rows).astype(np.uint32)  # (n_rows, 32)
    n = ids_np.shape[0]
    pad = (-n) % 64
    ids_np = np.concatenate([ids_np, np.zeros((pad, 32), np.uint32)])
    R = ids_np.shape[0] // 64
    ids3 = ids_np.reshape(R, 64, 32)
    ths = [(SIG_E, t, GE) for t in (0.7,)]
    from paper_2412_20993_b200 import Threshold
    for tau in (0.4, 0.5, 0.7, 0.75, 0.85, 0.99):
        ths = [(SIG_E, tau, GE)]
        h, meets = ctx.sc_certaindex(torch.from_numpy(ids3.view(np.int32)).cuda(), [Threshold(*t) for t in ths])
        ctx.sync()
        _, oh32, om = O.sc_certaindex(ids3, ths)
        assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
        assert np.array_equal(meets.cpu().numpy().view(np.uint32), om)


def test_sc_unaligned_base_pointer(ctx):
    """A base pointer that is not 16B aligned takes the plain-load tile path."""
    import torch
    from paper_2412_20993_b200 import Threshold
    R, P, S = 40, 8, 3
    ids = ctx.gen_sc(_gp(seed=4, conv_hi=8), R + 1, P, S)
    flat = ids.view(-1)[1:1 + R * P * S].view(R, P, S)  # 4-byte offset
    h, meets = ctx.sc_certaindex(flat, [Threshold(SIG_E, 0.6, GE)])
    ctx.sync()
    ref_ids = O.gen_sc(_og(seed=4, conv_hi=8), R + 1, P, S).reshape(-1)[1:1 + R * P * S].reshape(R, P, S)
    _, oh32, om = O.sc_certaindex(ref_ids, [(SIG_E, 0.6, GE)])
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(meets.cpu().numpy().view(np.uint32), om)


def test_sc_errors(ctx):
    import torch
    from paper_2412_20993_b200 import CdxInvalidArgument, Threshold
    ids = torch.zeros((2, 4, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(CdxInvalidArgument, match="signal 'certaindex_reward' absent"):
        ctx.sc_certaindex(ids, [Threshold(SIG_R, 0.4, GE)])
    with pytest.raises(CdxInvalidArgument, match="empty answer set"):
        ctx.sc_certaindex(torch.zeros((2, 4, 0), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("kind,detect,cap,recheck", [(2, 5, 64, 1), (4, 5, 64, 1), (4, 3, 60, 7), (0, 1, 64, 1),
                                                     (2, 64, 64, 1), (4, 1, 1, 1), (2, 1, 33, 1)])
@pytest.mark.parametrize("R", [1, 1023, 1024, 1025, 5000])
def test_allocate_scan_parity(ctx, kind, detect, cap, recheck, R):
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    P, S = 64, 32
    if cap > P:
        pytest.skip()
    g = dict(seed=77 + R, conv_hi=64)
    ids = ctx.gen_sc(_gp(**g), R, P, S)
    _, meets = ctx.sc_certaindex(ids, [Threshold(SIG_E, 0.7, GE)], want_hcert=False)
    pol = AllocPolicy(kind=kind, detect_at=detect, resource_cap=cap, recheck_every=recheck, tokens_per_unit=64 * S)
    out = ctx.allocate_scan(meets, R, P, pol, base_offset=12345)
    ctx.sync()
    _, _, om = O.sc_certaindex(O.gen_sc(_og(**g), R, P, S), [(SIG_E, 0.7, GE)])
    ref = O.allocate_scan(om, R, P, kind, detect, cap, recheck, 64 * S, base_offset=12345)
    for k in ("exit_knob", "reason", "granted", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
    n_kept, saved, total = out["scalars"].cpu().numpy().tolist()
    assert n_kept == ref["n_kept"]
    assert saved == ref["tokens_saved"]
    assert np.array_equal(out["kept"][:n_kept].cpu().numpy().view(np.uint32), ref["kept"])
    assert total == int((ref["granted"].astype(np.int64) * 64 * S).sum())


def test_allocate_scan_large_property(ctx):
    """Full-size property check at 1M requests: offsets are an exclusive prefix sum of
    granted*tpu (checked by recomputation on the GPU), kept list strictly increasing."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    R, P, S = 1 << 20, 64, 32
    meets = torch.randint(-2**31, 2**31 - 1, (R, 2), dtype=torch.int32, device="cuda")
    pol = AllocPolicy(kind=4, detect_at=5, resource_cap=64, recheck_every=3, tokens_per_unit=2048)
    out = ctx.allocate_scan(meets, R, P, pol)
    ctx.sync()
    g = out["granted"].to(torch.int64) * 2048
    excl = torch.cumsum(g, 0) - g
    assert torch.equal(excl, out["offsets"])
    n_kept = int(out["scalars"][0])
    kept = out["kept"][:n_kept].to(torch.int64)
    assert torch.all(kept[1:] > kept[:-1])
    assert n_kept == int((out["granted"] > 5).sum())


@pytest.mark.parametrize("kind,detect,cap,recheck", [(4, 1, 4096, 1000), (2, 4096, 4096, 1), (0, 1, 4096, 1),
                                                     (4, 7, 4000, 1)])
def test_allocate_scan_max_probes(ctx, kind, detect, cap, recheck):
    """P = cap = 4096 (the largest knob): per-warp unit sums reach 32 x 4096 and per-tile sums
    2048 x 4096, the limits of the packed scans; sparse random meets bits."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy
    R, P = 6001, 4096
    rng = np.random.default_rng(cap + detect)
    om = (rng.random((R, P // 32, 32)) < 0.002)
    om = (om * (1 << np.arange(32, dtype=np.uint64))).sum(axis=2).astype(np.uint32)
    meets = torch.from_numpy(om.view(np.int32)).cuda()
    pol = AllocPolicy(kind=kind, detect_at=detect, resource_cap=cap, recheck_every=recheck, tokens_per_unit=3 << 30)
    out = ctx.allocate_scan(meets, R, P, pol, base_offset=-5)
    ctx.sync()
    ref = O.allocate_scan(om, R, P, kind, detect, cap, recheck, 3 << 30, base_offset=-5)
    for k in ("exit_knob", "reason", "granted", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
    n_kept, saved, total = out["scalars"].cpu().numpy().tolist()
    assert n_kept == ref["n_kept"]
    assert saved == ref["tokens_saved"]
    assert np.array_equal(out["kept"][:n_kept].cpu().numpy().view(np.uint32), ref["kept"])


@pytest.mark.parametrize("distinct", [9, 17, 32])
def test_sc_many_clusters_fallback(ctx, distinct):
    """Rows with more than PEEL_MAX clusters send their group to the warp-match engine; the
    result must stay bit-identical (high-entropy rows, every engine split)."""
    import torch
    from paper_2412_20993_b200 import Threshold
    R, P, S = 97, 64, 32
    rng = np.random.default_rng(distinct)
    ids = rng.integers(0, distinct, size=(R, P, S)).astype(np.uint32)
    ids[::3, ::5, :] = np.arange(S, dtype=np.uint32)  # all-distinct rows
    ids[1::4, 7, :] = 5  # single-cluster rows in the same groups
    h, m = ctx.sc_certaindex(torch.from_numpy(ids.view(np.int32)).cuda(), [Threshold(SIG_E, 0.1, GE)])
    ctx.sync()
    _, oh32, om = O.sc_certaindex(ids, [(SIG_E, 0.1, GE)])
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(m.cpu().numpy().view(np.uint32), om)


def test_graph_replay_of_sc_step(ctx):
    """A captured K2 + K5 step (config A shape) replays bit-identically, replay after replay
    (K5's look-back records are tagged by a device-side epoch, so replays never see stale
    records), and its kernels count in cdx_launch_count."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    R, P, S = 1024, 32, 16
    ids = ctx.gen_sc(_gp(seed=21, conv_hi=32), R, P, S)
    ths = [Threshold(SIG_E, 0.7, GE)]
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=32, tokens_per_unit=64 * S)
    hc = torch.empty((R, P), dtype=torch.float32, device="cuda")
    mt = torch.empty((R, 1), dtype=torch.int32, device="cuda")
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_knob", torch.int32), ("reason", torch.uint8), ("granted", torch.int32), ("offsets", torch.int64),
            ("kept", torch.int32))}
    out["scalars"] = torch.zeros((3,), dtype=torch.int64, device="cuda")

    def step():
        ctx.sc_certaindex(ids, ths, hcert=hc, meets=mt)
        ctx.allocate_scan(mt, R, P, pol, base_offset=7, out=out)

    g = ctx.graph_capture(step)
    _, _, om = O.sc_certaindex(O.gen_sc(_og(seed=21, conv_hi=32), R, P, S), [(SIG_E, 0.7, GE)])
    ref = O.allocate_scan(om, R, P, 2, 5, 32, 1, 64 * S, base_offset=7)
    for _ in range(3):
        for k in out:
            if k != "scalars":
                out[k].fill_(-1)
        l0 = ctx.launches
        g()
        ctx.sync()
        assert ctx.launches > l0
        for k in ("exit_knob", "reason", "granted", "offsets"):
            assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
        assert int(out["scalars"][0]) == ref["n_kept"]
        assert np.array_equal(mt.cpu().numpy().view(np.uint32), om)


@pytest.mark.parametrize("rows,S,groups", [(100, 1, 1), (257, 7, 3), (300, 16, 5), (200, 32, 40), (90, 33, 5),
                                           (64, 100, 70), (5, 4096, 900)])
def test_cluster_rows_parity(ctx, rows, S, groups):
    """cdx_cluster_rows (the full metrics::Clustering of every row: cluster count, first-seen
    leader sample and size per cluster) against the oracle's cluster_exact, S = 1 .. 4096."""
    import ctypes as C
    import torch
    rng = np.random.default_rng(rows + S)
    ids = rng.integers(0, groups, size=(rows, S)).astype(np.uint32)
    ncl, lead, size = ctx.cluster_rows(torch.from_numpy(ids.view(np.int32)).cuda())
    ctx.sync()
    ncl, lead, size = ncl.cpu().numpy(), lead.cpu().numpy(), size.cpu().numpy()
    L = O.lib()
    sz = (C.c_int * S)()
    ld = (C.c_int * S)()
    for r in range(rows):
        row = np.ascontiguousarray(ids[r])
        m = L.cdxo_cluster_exact_ids(row.ctypes.data_as(C.c_void_p), S, sz, ld)
        assert ncl[r] == m
        assert list(lead[r, :m]) == list(ld[:m]) and list(size[r, :m]) == list(sz[:m])


@pytest.mark.parametrize("rows,max_m,max_n", [(1, 1, 1), (500, 8, 64), (300, 40, 1000), (64, 5, 5)])
def test_entropy_from_sizes_parity(ctx, rows, max_m, max_n):
    """cdx_entropy_from_sizes (explicit clusterings: the facade path of semantic_entropy /
    certaindex_entropy over many rows, totals implicit or given) against the oracle's FP64
    fold, bit for bit; invalid rows fail with the reference's messages."""
    import ctypes as C
    import torch
    from paper_2412_20993_b200 import CdxInvalidArgument
    rng = np.random.default_rng(rows + max_m)
    m = rng.integers(1, max_m + 1, size=rows).astype(np.uint32)
    sizes = np.zeros((rows, max_m), np.uint32)
    for r in range(rows):
        cuts = np.sort(rng.choice(np.arange(1, max_n), size=min(int(m[r]) - 1, max_n - 1), replace=False)) \
            if max_n > 1 else np.array([], np.int64)
        parts = np.diff(np.concatenate([[0], cuts, [rng.integers(max(cuts.max() + 1 if len(cuts) else 1, 1), max_n + 1)]]))
        m[r] = len(parts)
        sizes[r, :len(parts)] = parts
    tot = sizes.sum(axis=1).astype(np.uint32)
    H, Hc = ctx.entropy_from_sizes(torch.from_numpy(sizes.view(np.int32)).cuda(), torch.from_numpy(m.view(np.int32)).cuda(),
                                   max_n)
    ctx.sync()
    H, Hc = H.cpu().numpy(), Hc.cpu().numpy()
    L = O.lib()
    for r in range(rows):
        k = int(m[r])
        sz = (C.c_int * k)(*[int(x) for x in sizes[r, :k]])
        assert H[r] == L.cdxo_semantic_entropy(sz, k, int(tot[r]))
        assert Hc[r] == L.cdxo_certaindex_entropy(sz, k, int(tot[r]))
    bad = sizes.copy()
    bad[0, 0] = 0
    with pytest.raises(CdxInvalidArgument, match="empty cluster|invalid clustering"):
        ctx.entropy_from_sizes(torch.from_numpy(bad.view(np.int32)).cuda(), torch.from_numpy(m.view(np.int32)).cuda(),
                               max_n)
        ctx.sync()
