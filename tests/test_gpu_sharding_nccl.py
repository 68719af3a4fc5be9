"""The sharded path's collectives over a real NCCL communicator on the B200 (world size 1:
this harness reaches one GPU; the multi-rank exchange is covered by the gloo tests and by the
two-thread C++ test over the C-ABI, tests/cpp/shard_world2.cpp).  Two drivers: torch.distributed
collectives over the device building blocks (samples, bounds, merge of the received runs),
and a context that owns its NCCL communicator (cdx_ctx_create_comm, the C-ABI sharded
entries).  Both must reproduce the single-GPU results."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sc_decide_and_gang_order_through_nccl(ctx, nccl):
    from paper_2412_20993_b200 import AllocPolicy, GenParams, InterPolicy, Threshold
    from paper_2412_20993_b200.sharding import Sharded
    sh = Sharded(ctx, force_collectives=True)
    assert sh.nccl and sh.world == 1
    R, P, S = 3000, 64, 32
    ids = ctx.gen_sc(GenParams(seed=41, conv_hi=64), R, P, S)
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=64, tokens_per_unit=64 * S)
    res = sh.sc_decide(ids, [Threshold(0, 0.7, 0)], pol, r0=0)
    ctx.sync()
    _, _, om = O.sc_certaindex(O.gen_sc(O.gen_params(seed=41, conv_hi=64), R, P, S), [(0, 0.7, 0)])
    ref = O.allocate_scan(om, R, P, 2, 5, 64, 1, 64 * S)
    assert np.array_equal(res["offsets"].cpu().numpy(), ref["offsets"])
    assert int(res["shard_totals"][0]) == int((ref["granted"].astype(np.int64) * 64 * S).sum())
    # gang order: padded allgather of the sorted key run + device merge
    N = 20000
    rng = np.random.default_rng(3)
    arrival = np.cumsum(rng.exponential(1e-3, N))
    now = float(arrival[-1]) + 1e-3
    cnt = rng.integers(0, 5, N).astype(np.uint32)
    soa = dict(arrival=arrival, last_service=np.maximum(now - rng.exponential(0.2, N), 0.0),
               iter_tok_sum=(rng.integers(1, 500, N) * cnt).astype(np.int64), iter_count=cnt,
               cap=rng.integers(1, 30, N).astype(np.int32), terminated=(rng.random(N) < 0.2).astype(np.uint8))
    soa["knob"] = np.minimum(soa["cap"], rng.integers(0, 30, N)).astype(np.int32)
    dev = {k: (torch.from_numpy(v.view(np.int16)) if v.dtype == np.uint16 else torch.from_numpy(v)).cuda()
           for k, v in soa.items()}
    order = sh.gang_order(dev, InterPolicy(order=1, starvation_limit=0.15, prior_tokens=128.0), now, 0)
    ctx.sync()
    gref, _ = O.gang_order(soa, 1, 0.15, 128.0, now)
    assert np.array_equal(order.cpu().numpy().view(np.uint32), gref)


def _gang_inputs(N, seed):
    rng = np.random.default_rng(seed)
    arrival = np.cumsum(rng.exponential(1e-3, N))
    now = float(arrival[-1]) + 1e-3
    cnt = rng.integers(0, 5, N).astype(np.uint32)
    soa = dict(arrival=arrival, last_service=np.maximum(now - rng.exponential(0.2, N), 0.0),
               iter_tok_sum=(rng.integers(1, 500, N) * cnt).astype(np.int64), iter_count=cnt,
               cap=rng.integers(1, 30, N).astype(np.int32), terminated=(rng.random(N) < 0.2).astype(np.uint8))
    soa["knob"] = np.minimum(soa["cap"], rng.integers(0, 30, N)).astype(np.int32)
    return soa, now


def test_context_owned_nccl_communicator_world1():
    """cdx_ctx_create_comm with an NCCL unique id: the context creates and owns the NCCL
    communicator; cdx_allocate_scan_sharded / cdx_gang_priority_sharded run their allgathers
    and grouped send/recv through it and equal the 1-GPU results."""
    from paper_2412_20993_b200 import AllocPolicy, Context, GenParams, InterPolicy, Threshold, nccl_unique_id
    from paper_2412_20993_b200.sharding import Sharded
    cx = Context.with_nccl(0, 0, 1, nccl_unique_id())
    assert cx.world == 1
    R, P, S = 5000, 64, 32
    ids = cx.gen_sc(GenParams(seed=43, conv_hi=64), R, P, S)
    _, meets = cx.sc_certaindex(ids, [Threshold(0, 0.7, 0)])
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=64, tokens_per_unit=64 * S)
    res = cx.allocate_scan_sharded(meets, R, P, pol)
    cx.sync()
    _, _, om = O.sc_certaindex(O.gen_sc(O.gen_params(seed=43, conv_hi=64), R, P, S), [(0, 0.7, 0)])
    ref = O.allocate_scan(om, R, P, 2, 5, 64, 1, 64 * S)
    assert np.array_equal(res["offsets"].cpu().numpy(), ref["offsets"])
    nk = int(res["scalars"][0])
    assert nk == ref["n_kept"]
    assert np.array_equal(res["kept"][:nk].cpu().numpy().view(np.uint32), ref["kept"][:nk])
    assert int(res["scalars"][1]) == ref["tokens_saved"]
    info = res["shard_info"].cpu().numpy()
    assert info[0, 0] == R and info[0, 2] == nk
    for N, seed in ((30000, 5), (1, 6), (257, 7)):
        soa, now = _gang_inputs(N, seed)
        dev = {k: torch.from_numpy(v).cuda() for k, v in soa.items()}
        order = cx.gang_priority_sharded(dev, InterPolicy(order=1, starvation_limit=0.15, prior_tokens=128.0), now)
        cx.sync()
        gref, _ = O.gang_order(soa, 1, 0.15, 128.0, now)
        assert np.array_equal(order.cpu().numpy().view(np.uint32), gref)
        # the Sharded facade takes the context's own communicator
        sh = Sharded(cx)
        assert sh.native
        o2 = sh.gang_order(dev, InterPolicy(order=1, starvation_limit=0.15, prior_tokens=128.0), now, 0)
        assert np.array_equal(o2.cpu().numpy().view(np.uint32), gref)
    cx.close()
