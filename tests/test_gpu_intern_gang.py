"""GPU parity: K1 canon_intern (trim + exact-match interning + hesitation) and K6
gang_priority / gang_merge vs the oracle (bit-exact ids, flags and orders)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _arena(strings):
    bs = [s.encode() if isinstance(s, str) else s for s in strings]
    offs = np.zeros(len(bs) + 1, np.uint64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    return np.frombuffer(b"".join(bs) or b"\0", np.uint8).copy(), offs


def _intern(ctx, strings, markers=("wait", "hmm")):
    import torch
    arena, offs = _arena(strings)
    ta = torch.from_numpy(arena).cuda()
    to = torch.from_numpy(offs.view(np.int64)).cuda()
    ids, hes, first, nu = ctx.canon_intern(ta, to, markers)
    ctx.sync()
    return ids.cpu().numpy().view(np.uint32), hes.cpu().numpy(), first.cpu().numpy(), nu


@pytest.mark.parametrize("n,vocab", [(1, 3), (10, 3), (5000, 7), (100000, 500), (300000, 40000)])
def test_intern_parity(ctx, n, vocab):
    rng = np.random.default_rng(n)
    base = [f"ans{i}" for i in range(vocab)] + ["wait, 42", "Hmm 7", "HMM", "x  wait", "", "   ", "\t\n"]
    ws = [" ", "\t", "\n", "\r", "\f", "\v", "", ""]
    strings = []
    for k in rng.integers(0, len(base), n):
        s = base[k]
        strings.append(ws[rng.integers(0, len(ws))] + s + ws[rng.integers(0, len(ws))])
    ids, hes, first, nu = _intern(ctx, strings)
    oid, ohes, onu = O.canon_intern(strings)
    assert nu == onu
    assert np.array_equal(ids, oid)
    assert np.array_equal(hes, ohes)
    # first_index: arena position of each id's first occurrence
    for d in range(min(nu, 50)):
        assert oid[first[d]] == d and (oid[: first[d]] != d).all()


def test_intern_spec_examples(ctx):
    ids, _, _, nu = _intern(ctx, ["12", " 12", "13"])
    assert ids.tolist() == [0, 0, 1] and nu == 2
    _, hes, _, _ = _intern(ctx, ["42", "wait, let me check", "Hmm 42", "WAIT"], ("wait", "hmm"))
    assert hes.tolist() == [0, 1, 1, 1]
    _, hes, _, _ = _intern(ctx, ["WAIT", "abc"], ("WAIT", ""))  # upper-case / empty markers never match
    assert hes.tolist() == [0, 0]


def test_intern_synthetic_arena_scale(ctx):
    """The bench config K arena (synth.answer_arena_*: vocabulary answers, hesitant forms,
    whitespace pads) at 2^20 answers: device and host builders agree and K1 equals the oracle."""
    import torch
    from paper_2412_20993_b200 import synth
    n = 1 << 20
    ids = np.random.default_rng(7).integers(0, 5, n).astype(np.uint32)
    arena, off = synth.answer_arena_np(ids)
    ta, to = synth.answer_arena_torch(torch.from_numpy(ids.astype(np.int64)).cuda())
    assert np.array_equal(ta.cpu().numpy(), arena)
    got, hes, first, nu = ctx.canon_intern(ta, to)
    ctx.sync()
    strings = [bytes(arena[12 * i: 12 * i + 12]) for i in range(n)]
    oid, ohes, onu = O.canon_intern(strings)
    assert nu == onu == 10
    assert np.array_equal(got.cpu().numpy().view(np.uint32), oid)
    assert np.array_equal(hes.cpu().numpy(), ohes)


@pytest.mark.parametrize("case", ["all_distinct", "long_answers", "unaligned", "long_markers", "tile_edges"])
def test_intern_paths(ctx, case):
    """All-distinct answers past the first table's capacity (the retry with room for every
    answer), answers longer than a staged tile (read in place), an unaligned arena (offsets
    staged by hand), markers longer than 8 bytes, and counts around the 1024-answer tile."""
    import torch
    rng = np.random.default_rng(11)
    markers = ("wait", "hmm")
    if case == "all_distinct":
        strings = [f" u{i} " for i in range(700000)] + [" u5", "u7 "]
    elif case == "long_answers":
        strings = [("  x" * int(rng.integers(1, 3000))) + (" WAIT " if i % 3 == 0 else "") for i in range(700)]
    elif case == "unaligned":
        strings = [f"\t{k}\n" for k in rng.integers(0, 50, 20000)]
    elif case == "long_markers":
        strings = ["I think, wait a second, maybe 7", "WAIT A SECOND", "wait a secon", "x" * 40 + "wait a second"]
        markers = ("wait a second", "")
    else:
        strings = [f"a{k}" for k in rng.integers(0, 3, 1024 * 3 + 1)]
    arena, offs = _arena(strings)
    if case == "unaligned":
        pad = np.zeros(len(arena) + 3, np.uint8)
        pad[3:] = arena
        tbuf = torch.from_numpy(pad).cuda()
        ta = tbuf[3:]
        obuf = torch.zeros(len(offs) + 1, dtype=torch.int64).cuda()
        obuf[1:] = torch.from_numpy(offs.view(np.int64))
        to = obuf[1:]
    else:
        ta = torch.from_numpy(arena).cuda()
        to = torch.from_numpy(offs.view(np.int64)).cuda()
    ids, hes, first, nu = ctx.canon_intern(ta, to, markers)
    ctx.sync()
    oid, ohes, onu = O.canon_intern(strings, markers) if case == "long_markers" else O.canon_intern(strings)
    assert nu == onu
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oid)
    assert np.array_equal(hes.cpu().numpy(), ohes)
    f = first.cpu().numpy()
    for d in range(min(nu, 100)):
        assert oid[f[d]] == d and (oid[: f[d]] != d).all()


def _grow_arena(n, vocab, seed, lead_ws=True):
    """Answers whose vocabulary grows along the arena (key k first appears near k * n / vocab),
    with whitespace pads and hesitant forms: new keys keep arriving in every round of tiles."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    top = np.maximum(1, (i * vocab) // n + 1)
    key = (rng.random(n) * top).astype(np.int64)
    lpad = rng.integers(0, 3, n) if lead_ws else np.zeros(n, np.int64)
    rpad = rng.integers(0, 3, n)
    hes = rng.random(n) < 0.05
    names = [b"k%d" % k for k in range(vocab)]
    wsb = [bytes([c]) for c in b" \t\n\r\f\v"]
    w = rng.integers(0, 6, (n, 4))
    parts = [b"".join(wsb[w[a, q]] for q in range(lpad[a])) + (b"wait, " if hes[a] else b"") + names[key[a]] +
             b"".join(wsb[w[a, 2 + q]] for q in range(rpad[a])) for a in range(n)]
    lens = np.fromiter((len(x) for x in parts), np.int64, n)
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    return np.frombuffer(b"".join(parts), np.uint8).copy(), offs


@pytest.mark.parametrize("n,vocab", [(1 << 18, 3000), (1 << 21, 100), (1 << 21, 60000)])
def test_intern_growing_vocabulary(ctx, n, vocab):
    """Keys first seen in late rounds of tiles: dense ids come from the round counts (final
    slices) or the flagged-slice remap; both must equal the oracle's first-seen order."""
    import torch
    arena, offs = _grow_arena(n, vocab, seed=n + vocab)
    ta = torch.from_numpy(arena).cuda()
    to = torch.from_numpy(offs.view(np.int64)).cuda()
    ids, hes, first, nu = ctx.canon_intern(ta, to, ("wait", "hmm"))
    ctx.sync()
    oid, ohes, onu = O.canon_intern_arena(arena, offs, ("wait", "hmm"))
    assert nu == onu
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oid)
    assert np.array_equal(hes.cpu().numpy(), ohes)
    f = first.cpu().numpy()[:nu]
    first_seen = np.full(nu, -1, np.int64)
    _, idx = np.unique(oid, return_index=True)
    first_seen[:] = idx
    assert np.array_equal(f.astype(np.int64), first_seen)


def test_intern_synthetic_arena_large(ctx):
    """Config K's arena at 2^24 answers (16K tiles, ~110 rounds): every id and flag."""
    import torch
    from paper_2412_20993_b200 import GenParams, synth
    n = 1 << 24
    sid = ctx.gen_sc(GenParams(seed=20993 + 8, conv_hi=64), n // (64 * 32), 64, 32).view(-1)
    ta, to = synth.answer_arena_torch(sid, 12)
    got, hes, first, nu = ctx.canon_intern(ta, to)
    ctx.sync()
    oid, ohes, onu = O.canon_intern_arena(ta.cpu().numpy(), to.cpu().numpy().view(np.uint64))
    assert nu == onu
    assert np.array_equal(got.cpu().numpy().view(np.uint32), oid)
    assert np.array_equal(hes.cpu().numpy(), ohes)


def _gang_inputs(N, seed, frac_term=0.1, sorted_arrival=True):
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(1e-3, N)
    arrival = np.cumsum(gaps) if sorted_arrival else rng.random(N) * N * 1e-3
    if not sorted_arrival:
        arrival[rng.integers(0, N, N // 10)] = arrival[0]  # duplicate arrivals -> id tie-break
    now = float(arrival.max()) + 1.0
    last = np.minimum(now, arrival + rng.exponential(0.5, N))
    cnt = rng.integers(0, 5, N).astype(np.uint32)
    sums = (rng.integers(32, 512, N) * cnt).astype(np.int64)
    cap = rng.integers(1, 64, N).astype(np.int32)
    knob = np.minimum(cap, rng.integers(0, 64, N)).astype(np.int32)
    term = (rng.random(N) < frac_term).astype(np.uint8)
    return dict(arrival=arrival, last_service=last, iter_tok_sum=sums, iter_count=cnt, knob=knob, cap=cap,
                terminated=term), now


def _to_dev(soa):
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() if v.dtype != np.uint16 else
            torch.from_numpy(np.ascontiguousarray(v).view(np.int16)).cuda() for k, v in soa.items()}


@pytest.mark.parametrize("N,order,limit,sorted_arrival", [(1, 1, 1.0, True), (1000, 1, 0.7, True),
                                                          (100000, 1, 0.5, True), (50000, 0, 0.5, True),
                                                          (70000, 1, 0.9, False), (5000, 0, 100.0, False),
                                                          (4096, 1, 0.5, True), (4097, 1, 0.5, False),
                                                          (8193, 0, 0.5, False), (1 << 22, 1, 0.5, True)])
def test_gang_parity(ctx, N, order, limit, sorted_arrival):
    from paper_2412_20993_b200 import InterPolicy
    soa, now = _gang_inputs(N, N + order, sorted_arrival=sorted_arrival)
    got, esc, _ = ctx.gang_priority(_to_dev(soa), InterPolicy(order=order, starvation_limit=limit, prior_tokens=128.0),
                                    now, want_escalated=True)
    ctx.sync()
    ref, resc = O.gang_order(soa, order, limit, 128.0, now)
    assert np.array_equal(esc.cpu().numpy(), resc)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("N,sorted_arrival,mode", [(5000, True, None), (100000, True, None), (100000, False, None),
                                                   (70001, True, "checked"), (70001, False, "full"), (1, True, None)])
def test_gang_explicit_program_ids(ctx, monkeypatch, N, sorted_arrival, mode):
    """cdx_prog_soa.program_id: the last tie-break is the program id, not the
    position.  Shuffled sparse ids with runs of equal arrivals (and identical keys) must come
    out in (escalated, key, arrival, id) order on every path (fast, checked, full)."""
    import torch
    from paper_2412_20993_b200 import InterPolicy
    if mode:
        monkeypatch.setenv("CDX_GANG_MODE", mode)
    soa, now = _gang_inputs(N, 77 + N, sorted_arrival=sorted_arrival)
    rng = np.random.default_rng(N)
    if N > 1:
        soa["arrival"] = np.sort(soa["arrival"]) if sorted_arrival else soa["arrival"]
        soa["arrival"][1::3] = soa["arrival"][0::3][: len(soa["arrival"][1::3])]  # equal-arrival pairs
        if sorted_arrival:
            soa["arrival"] = np.maximum.accumulate(soa["arrival"])
        soa["iter_tok_sum"][::2] = 0
        soa["iter_count"][::2] = 0  # prior estimate: many identical SJF keys
    ids = rng.permutation(np.arange(N, dtype=np.uint64) * 7 + 3).astype(np.uint32)
    soa["program_id"] = ids
    dev = _to_dev(soa)
    got, esc, _ = ctx.gang_priority(dev, InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), now,
                                    want_escalated=True)
    ctx.sync()
    ref, resc = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(esc.cpu().numpy(), resc)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("N,off", [(1 << 16, 1), (70001, 3), (4096, 2), (1 << 20, 0)])
def test_gang_flag_bytes_and_alignment(ctx, N, off):
    """The live count reads the terminated flags a word at a time when the tile is full and the
    flags are 4-byte aligned, a byte at a time otherwise: any non-zero byte is terminated
    (oracle/cdx_oracle.c's `if (terminated[i]) continue`), whatever the pointer's alignment."""
    import torch
    from paper_2412_20993_b200 import InterPolicy
    soa, now = _gang_inputs(N, 900 + off)
    rng = np.random.default_rng(off)
    soa["terminated"] = (soa["terminated"] * rng.integers(1, 256, N)).astype(np.uint8)
    dev = _to_dev(soa)
    store = torch.zeros(N + 8, dtype=torch.uint8, device="cuda")
    store[off:off + N] = dev["terminated"]
    dev["terminated"] = store[off:off + N]
    got, _, _ = ctx.gang_priority(dev, InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), now)
    ctx.sync()
    ref, _ = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("ps", ["1", "0"])
@pytest.mark.parametrize("case", ["identical", "all_escalated", "one_digit", "upper_half_ties", "short_runs"])
def test_gang_degenerate_keys(ctx, case, ps, monkeypatch):
    """Keys that agree on most or all radix digits (skipped passes, single-digit sorts,
    ties resolved purely by arrival then program id), on the one-launch persistent order
    (CDX_GANG_PS=1, the default) and on the multi-launch onesweep path (CDX_GANG_PS=0)."""
    from paper_2412_20993_b200 import InterPolicy
    monkeypatch.setenv("CDX_GANG_PS", ps)
    N = 20000
    soa, now = _gang_inputs(N, 3, frac_term=0.0)
    if case == "identical":
        for k in ("arrival", "last_service"):
            soa[k][:] = 1.0
        soa["iter_tok_sum"][:] = 640
        soa["iter_count"][:] = 5
        soa["cap"][:] = 10
        soa["knob"][:] = 3
        now = 1.5
    elif case == "all_escalated":
        soa["last_service"][:] = 0.0
        now = float(soa["arrival"].max()) + 10.0
    elif case == "upper_half_ties":  # equal upper 32 bits, shuffled lower bits: the 8-digit fallback
        soa["iter_count"][:] = 1
        soa["iter_tok_sum"][:] = (1 << 40) + np.random.default_rng(9).integers(0, 1000, N)
        soa["cap"][:] = 2
        soa["knob"][:] = 1
        soa["last_service"][:] = soa["arrival"]
        now = float(soa["arrival"].max()) + 0.1
    elif case == "short_runs":  # pairs/triples of keys sharing upper halves, fixed up in place
        base = np.random.default_rng(10).integers(1 << 30, 1 << 31, N // 3 + 1)
        soa["iter_count"][:] = 1
        soa["iter_tok_sum"][:] = (np.repeat(base, 3)[:N] << 12) + np.random.default_rng(11).integers(0, 64, N)
        soa["cap"][:] = 2
        soa["knob"][:] = 1
        soa["last_service"][:] = soa["arrival"]
        now = float(soa["arrival"].max()) + 0.1
    else:  # sjf keys that differ only in their lowest mantissa byte
        soa["iter_count"][:] = 1
        soa["iter_tok_sum"][:] = 1 << 20
        soa["cap"][:] = 2
        soa["knob"][:] = 1
        soa["arrival"][:] = np.sort(soa["arrival"])
        soa["last_service"][:] = soa["arrival"]
        now = float(soa["arrival"].max()) + 0.1
    pol = InterPolicy(order=1, starvation_limit=1.0, prior_tokens=128.0)
    got, _, _ = ctx.gang_priority(_to_dev(soa), pol, now)
    ctx.sync()
    ref, _ = O.gang_order(soa, 1, 1.0, 128.0, now)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("ps", ["1", "0"])
@pytest.mark.parametrize("N,frac_term,sorted_arrival", [(2, 0.0, True), (33, 0.5, True), (8192, 0.1, True),
                                                        (8193, 0.0, True), (50000, 1.0, True), (1212121, 0.3, True),
                                                        (3000001, 0.1, True), (30000, 0.2, False)])
def test_gang_one_launch_and_multi_launch(ctx, monkeypatch, ps, N, frac_term, sorted_arrival):
    """The persistent one-launch order (key build, 4 radix passes with grid-wide digit
    offsets, run fix-up: gang_order_persistent) and the multi-launch onesweep path it
    replaces, on tile and CTA-range boundaries, all-terminated traces, several tiles per CTA
    and unsorted arrivals (which send both to the host-checked path)."""
    from paper_2412_20993_b200 import InterPolicy
    monkeypatch.setenv("CDX_GANG_PS", ps)
    soa, now = _gang_inputs(N, 4242 + N, frac_term=frac_term, sorted_arrival=sorted_arrival)
    got, esc, _ = ctx.gang_priority(_to_dev(soa), InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0),
                                    now, want_escalated=True)
    ctx.sync()
    ref, resc = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(esc.cpu().numpy(), resc)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("N", [5000, 300000])
def test_gang_range_radix_option(ctx, N, monkeypatch):
    """CDX_RADIX=ranges (reduce-then-scan range passes instead of onesweep look-back) on the
    host-driven full sort: the documented alternative must give the same order."""
    from paper_2412_20993_b200 import InterPolicy
    monkeypatch.setenv("CDX_GANG_MODE", "full")
    monkeypatch.setenv("CDX_RADIX", "ranges")
    soa, now = _gang_inputs(N, 91, sorted_arrival=False)
    got, _, _ = ctx.gang_priority(_to_dev(soa), InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), now)
    ctx.sync()
    ref, _ = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("mode", ["full", "checked"])
@pytest.mark.parametrize("N,sorted_arrival", [(5000, True), (300000, True), (70000, False)])
def test_gang_pinned_modes(ctx, N, sorted_arrival, mode, monkeypatch):
    """The host-driven paths on their own: `checked` (pre-sort when arrivals are unsorted,
    upper-half sort + run fix-up) and `full` (8 digits), the fallbacks of the one-sync path."""
    from paper_2412_20993_b200 import InterPolicy
    monkeypatch.setenv("CDX_GANG_MODE", mode)
    soa, now = _gang_inputs(N, 77, sorted_arrival=sorted_arrival)
    got, _, _ = ctx.gang_priority(_to_dev(soa), InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), now)
    ctx.sync()
    ref, _ = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)


def test_gang_merge_equals_single_sort(ctx):
    """Per-rank sorted runs merged on the device == the one-shot global order (the
    multi-GPU path: each rank sorts its shard, allgathers keys, merges)."""
    import torch
    from paper_2412_20993_b200 import InterPolicy
    N, ranks = 40000, 4
    soa, now = _gang_inputs(N, 5)
    pol = InterPolicy(order=1, starvation_limit=0.6, prior_tokens=128.0)
    ref, _ = O.gang_order(soa, 1, 0.6, 128.0, now)
    stride = N // ranks + 7  # padded receive layout of the allgather
    keys = torch.full((ranks * stride, 3), -1, dtype=torch.int64, device="cuda")
    lens = []
    for r in range(ranks):
        sl = slice(r * N // ranks, (r + 1) * N // ranks)
        part = {k: v[sl] for k, v in soa.items()}
        o, _, k = ctx.gang_priority(_to_dev(part), pol, now, id_base=sl.start, want_keys=True)
        keys[r * stride: r * stride + k.shape[0]] = k
        lens.append(k.shape[0])
    total = torch.zeros((1,), dtype=torch.int64, device="cuda")
    out = ctx.gang_merge(keys, torch.tensor(lens, dtype=torch.int64, device="cuda"), stride, total=total)
    ctx.sync()
    assert int(total) == len(ref) == sum(lens)
    assert np.array_equal(out[: len(ref)].cpu().numpy().view(np.uint32), ref)


def test_gang_errors(ctx):
    from paper_2412_20993_b200 import CdxInvalidArgument, InterPolicy
    soa, now = _gang_inputs(10, 1)
    with pytest.raises(CdxInvalidArgument, match="starvation_limit"):
        ctx.gang_priority(_to_dev(soa), InterPolicy(order=1, starvation_limit=0.0), now)
    soa["arrival"][3] = -1.0
    with pytest.raises(CdxInvalidArgument, match="finite and >= 0"):
        ctx.gang_priority(_to_dev(soa), InterPolicy(order=1, starvation_limit=1.0), now)


@pytest.mark.parametrize("trial", range(24))
def test_gang_persistent_fuzz(ctx, trial):
    """Randomised traces through the one-launch order: sizes around tile (8192) and CTA-range
    boundaries, real-valued estimates (low halves differ: the run fix-up), integer-valued ones
    (low halves equal: fix-up skipped), FIFO and SJF, few to all escalated, duplicate keys,
    explicit program ids; every result against the oracle."""
    from paper_2412_20993_b200 import InterPolicy
    rng = np.random.default_rng(1000 + trial)
    N = int(rng.choice([1, 2, 7, 8191, 8192, 8193, 20000, 148 * 8192 + 5, 300001, 1 << 20]))
    order = int(rng.integers(0, 2))
    limit = float(rng.choice([0.05, 0.5, 5.0, 1e9]))
    arrival = np.cumsum(rng.exponential(1e-3, N))
    if rng.random() < 0.3:
        arrival = np.round(arrival, 2)  # runs of equal arrivals: the id decides
    now = float(arrival[-1]) + float(rng.uniform(0.0, 2.0))
    last = np.minimum(now, arrival + rng.exponential(limit, N))
    cnt = rng.integers(0, 6, N).astype(np.uint32)
    if rng.random() < 0.5:
        sums = (rng.integers(1, 2000, N) * cnt).astype(np.int64)  # integer means
    else:
        sums = (rng.integers(0, 5000, N) * (cnt + (rng.random(N) < 0.5))).astype(np.int64)  # real means
    cap = rng.integers(1, 64, N).astype(np.int32)
    knob = np.minimum(cap, rng.integers(0, 64, N)).astype(np.int32)
    term = (rng.random(N) < float(rng.choice([0.0, 0.2, 0.9]))).astype(np.uint8)
    soa = dict(arrival=arrival, last_service=last, iter_tok_sum=sums, iter_count=cnt, knob=knob, cap=cap,
               terminated=term)
    if rng.random() < 0.3 and N > 1:
        soa["program_id"] = (np.arange(N, dtype=np.uint64) * 3 + 11).astype(np.uint32)  # increasing ids
    prior = float(rng.choice([128.0, 1.5, 1e6]))
    got, esc, _ = ctx.gang_priority(_to_dev(soa), InterPolicy(order=order, starvation_limit=limit, prior_tokens=prior),
                                    now, want_escalated=True)
    ctx.sync()
    ref, resc = O.gang_order(soa, order, limit, prior, now)
    assert np.array_equal(esc.cpu().numpy(), resc)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)
