"""Repeated calls do not leak device memory: every kernel family is called many times with
shapes that vary (so scratch buffers grow, tables are cached, descriptors are re-encoded),
and after the first round the free device memory stays put.  Also re-checks one result per
round so a stale cache (tensor maps, occupancy, composition tables) would show."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _round(ctx, i):
    import torch
    from paper_2412_20993_b200 import AllocPolicy, GenParams, InterPolicy, ProbeConfig, Threshold
    R, P, S = 300 + 37 * (i % 3), 64 if i % 2 else 40, (16, 31, 32, 8)[i % 4]
    ids = ctx.gen_sc(GenParams(seed=i, conv_hi=P), R, P, S)
    h, m = ctx.sc_certaindex(ids, [Threshold(0, 0.7, 0)])
    ctx.allocate_scan(m, R, P, AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64))
    cids, hes = ctx.gen_cot(GenParams(seed=i, conv_hi=64, hesitation_prob=0.1), 500 + i, 64)
    ctx.cot_exit(cids, hes, ProbeConfig(64, 3, 0.9, 4096))
    rw, rid = ctx.gen_reward(GenParams(seed=i, conv_hi=8), 200, 8, (64, 48, 32)[i % 3])
    agg = torch.zeros(200, dtype=torch.uint8, device="cuda")
    ctx.reward_certaindex(rw, rid, agg)
    n = 5000 + 100 * i
    soa = {"arrival": torch.arange(n, dtype=torch.float64, device="cuda") * 1e-3,
           "last_service": torch.zeros(n, dtype=torch.float64, device="cuda"),
           "iter_tok_sum": torch.full((n,), 640, dtype=torch.int64, device="cuda"),
           "iter_count": torch.full((n,), 5, dtype=torch.int32, device="cuda"),
           "knob": torch.ones(n, dtype=torch.int32, device="cuda"),
           "cap": torch.full((n,), 9, dtype=torch.int32, device="cuda"),
           "terminated": torch.zeros(n, dtype=torch.uint8, device="cuda")}
    ctx.gang_priority(soa, InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), float(n))
    text = "\n".join(f'{{"program_id": "p{k % 7}", "step_index": {k // 7 + 1}, "token_offset": {64 * (k // 7 + 1)}, '
                     f'"answer": "a{k % 3}"}}' for k in range(200 + i)).encode()
    t = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    ctx.jsonl_parse(t, 300 + i)
    ctx.sync()
    # spot check: this round's SC result against the oracle
    _, oh32, _ = O.sc_certaindex(O.gen_sc(O.gen_params(seed=i, conv_hi=P), R, P, S), [(0, 0.7, 0)])
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))


def test_no_device_memory_growth(ctx):
    import torch
    for i in range(8):  # warm: scratch buffers reach their high-water marks
        _round(ctx, i)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for i in range(8, 48):
        _round(ctx, i)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 >= free0 - (64 << 20), (free0, free1)  # no growth beyond 64 MB of allocator slack


def test_streams_own_and_foreign(ctx):
    """The context's own non-blocking stream (cdx_ctx_use_own_stream) and a foreign torch
    stream give the same results; work on one stream is ordered before cdx_sync returns."""
    import torch
    from paper_2412_20993_b200 import GenParams, Threshold
    R, P, S = 700, 64, 32
    ids = ctx.gen_sc(GenParams(seed=5, conv_hi=P), R, P, S)
    ctx.sync()
    outs = []
    for mode in ("own", "foreign"):
        if mode == "own":
            assert ctx.lib.cdx_ctx_use_own_stream(ctx.h) == 0
            h = torch.empty((R, P), dtype=torch.float32, device="cuda")
            m = torch.empty((R, 2), dtype=torch.int32, device="cuda")
            import ctypes as C
            from paper_2412_20993_b200 import c_thresholds
            arr, n = c_thresholds([Threshold(0, 0.7, 0)])
            assert ctx.lib.cdx_sc_certaindex(ctx.h, C.c_void_p(ids.data_ptr()), R, P, S, arr, n,
                                             C.c_void_p(h.data_ptr()), C.c_void_p(m.data_ptr())) == 0
            assert ctx.lib.cdx_sync(ctx.h) == 0
        else:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                h, m = ctx.sc_certaindex(ids, [Threshold(0, 0.7, 0)])
            ctx.sync()
        outs.append((h.cpu().numpy().copy(), m.cpu().numpy().copy()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1], outs[1][1])
    _, oh32, om = O.sc_certaindex(O.gen_sc(O.gen_params(seed=5, conv_hi=P), R, P, S), [(0, 0.7, 0)])
    assert np.array_equal(outs[0][0].view(np.uint32), oh32.view(np.uint32))
