"""GPU parity: cdx_sc_decide (K2 + K5 in one call) against the oracle and against the two
separate calls: every meets bit, certaindex, exit knob, reason, grant, budget offset, kept
index and total, bit for bit; one K5 tile, tile boundaries, many tiles (the decoupled
look-back), every policy kind, P = 32 / 64 / 96 / 128 and the generic-kernel shapes."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIG_E, GE = 0, 0


def _run(ctx, R, P, S, kind, detect, cap, recheck, seed, base=0, kept_base=0):
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    g = dict(seed=seed, conv_hi=max(1, P))
    ids = ctx.gen_sc(GenParams(**g), R, P, S)
    pol = AllocPolicy(kind=kind, detect_at=detect, resource_cap=cap, recheck_every=recheck, tokens_per_unit=64 * S)
    import torch
    hc = torch.empty((R, P), dtype=torch.float32, device="cuda")
    h, meets, out = ctx.sc_decide(ids, [Threshold(SIG_E, 0.7, GE)], pol, hcert=hc, base_offset=base,
                                  kept_base=kept_base)
    ctx.sync()
    return g, h, meets, out


def _check(R, P, S, g, h, meets, out, kind, detect, cap, recheck, base=0, kept_base=0):
    _, oh32, om = O.sc_certaindex(O.gen_sc(O.gen_params(**g), R, P, S), [(SIG_E, 0.7, GE)])
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(meets.cpu().numpy().view(np.uint32), om)
    ref = O.allocate_scan(om, R, P, kind, detect, cap, recheck, 64 * S, base_offset=base)
    for k in ("exit_knob", "reason", "granted", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
    n_kept, saved, total = out["scalars"].cpu().numpy().tolist()
    assert n_kept == ref["n_kept"]
    assert saved == ref["tokens_saved"]
    assert total == int((ref["granted"].astype(np.int64) * 64 * S).sum())
    assert np.array_equal(out["kept"][:n_kept].cpu().numpy().view(np.uint32) - np.uint32(kept_base), ref["kept"])


@pytest.mark.parametrize("R,P,S", [(1, 32, 16), (1024, 32, 16), (2047, 64, 32), (2048, 64, 32), (2049, 64, 32),
                                   (5000, 64, 32), (40000, 32, 8), (9000, 96, 16), (3000, 128, 4), (7000, 64, 16)])
@pytest.mark.parametrize("kind,detect,cap,recheck", [(2, 5, 32, 1), (4, 3, 30, 7), (0, 1, 32, 1)])
def test_sc_decide_parity(ctx, R, P, S, kind, detect, cap, recheck):
    g, h, meets, out = _run(ctx, R, P, S, kind, detect, cap, recheck, seed=500 + R + P + S, base=99, kept_base=7)
    _check(R, P, S, g, h, meets, out, kind, detect, cap, recheck, base=99, kept_base=7)


@pytest.mark.parametrize("R,P,S", [(3000, 33, 16), (500, 64, 7), (200, 40, 32)])
def test_sc_decide_generic_shapes(ctx, R, P, S):
    """P % 32 != 0 or S outside {4, 8, 16, 32}: the generic K2 kernel, then K5."""
    g, h, meets, out = _run(ctx, R, P, S, 4, 3, 30, 5, seed=900 + R)
    _check(R, P, S, g, h, meets, out, 4, 3, 30, 5)


@pytest.mark.parametrize("R,P,S", [(6000, 64, 32), (1024, 32, 16), (2048, 64, 16)])
def test_sc_decide_repeated_calls_and_graph(ctx, R, P, S):
    """Back-to-back calls (tickets and epochs rewound in-kernel) and a captured graph replayed
    several times stay bit-exact; a standalone allocate_scan in between shares the look-back
    state.  R <= 2048 is the one-launch form (K5 in K2's last CTA)."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    g = dict(seed=4242 + R, conv_hi=P)
    ids = ctx.gen_sc(GenParams(**g), R, P, S)
    ths = [Threshold(SIG_E, 0.7, GE)]
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S)
    hc = torch.empty((R, P), dtype=torch.float32, device="cuda")
    mt = torch.empty((R, (P + 31) // 32), dtype=torch.int32, device="cuda")
    out = {k: torch.empty((R,), dtype=dt, device="cuda") for k, dt in
           (("exit_knob", torch.int32), ("reason", torch.uint8), ("granted", torch.int32), ("offsets", torch.int64),
            ("kept", torch.int32))}
    out["scalars"] = torch.zeros((3,), dtype=torch.int64, device="cuda")
    for _ in range(3):
        ctx.sc_decide(ids, ths, pol, hcert=hc, meets=mt, out=out)
        ctx.allocate_scan(mt, R, P, pol, out=dict(out))
    ctx.sync()
    _check(R, P, S, g, hc, mt, out, 2, 5, P, 1)
    graph = ctx.graph_capture(lambda: ctx.sc_decide(ids, ths, pol, hcert=hc, meets=mt, out=out))
    for _ in range(3):
        for k in out:
            if k != "scalars":
                out[k].fill_(-1)
        graph()
        ctx.sync()
        _check(R, P, S, g, hc, mt, out, 2, 5, P, 1)


def test_sc_decide_full_scale_property(ctx):
    """Config C's shape (1M requests x 64 x 32): offsets are the exclusive prefix sum of the
    grants, the kept list is strictly increasing, and the results equal the two calls."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    R, P, S = 1 << 20, 64, 32
    ids = ctx.gen_sc(GenParams(seed=20993 + 3, conv_hi=64), R, P, S)
    ths = [Threshold(SIG_E, 0.7, GE)]
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=64, tokens_per_unit=64 * S)
    _, m1, o1 = ctx.sc_decide(ids, ths, pol)
    _, m2 = ctx.sc_certaindex(ids, ths, want_hcert=False)
    o2 = ctx.allocate_scan(m2, R, P, pol)
    ctx.sync()
    assert torch.equal(m1, m2)
    for k in ("exit_knob", "reason", "granted", "offsets", "scalars"):
        assert torch.equal(o1[k], o2[k]), k
    n = int(o1["scalars"][0])
    assert torch.equal(o1["kept"][:n], o2["kept"][:n])
    gr = o1["granted"].to(torch.int64) * 64 * S
    assert torch.equal(torch.cumsum(gr, 0) - gr, o1["offsets"])
    kept = o1["kept"][:n].to(torch.int64)
    assert torch.all(kept[1:] > kept[:-1])
