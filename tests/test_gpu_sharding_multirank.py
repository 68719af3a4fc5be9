"""The sharded path with the real B200 kernels at world size 2: two processes share the one
reachable GPU and exchange over gloo (NCCL refuses two ranks on one device), so every
kernel of the multi-rank flow runs for real: each rank generates its request shard on the
device, K2 + K5 with the budget-total allgather and the device rebase, K6 on its program
shard with the padded key-run allgather and the device merge.  The concatenated / merged
results must equal the single-process oracle.  Then bench.py itself runs at --gpus 2
under torchrun the same way, and must print its JSON line."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu

R, P, S = 5000, 64, 32
N_PROG = 30000
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _soa():
    rng = np.random.default_rng(8)
    arrival = np.cumsum(rng.exponential(1e-3, N_PROG))
    now = float(arrival.max()) + 1e-3
    cnt = rng.integers(0, 5, N_PROG).astype(np.uint32)
    cap = rng.integers(1, 40, N_PROG).astype(np.int32)
    soa = dict(arrival=arrival, last_service=np.maximum(now - rng.exponential(0.2, N_PROG), 0.0),
               iter_tok_sum=(rng.integers(1, 500, N_PROG) * cnt).astype(np.int64), iter_count=cnt, cap=cap,
               knob=np.minimum(cap, rng.integers(0, 40, N_PROG)).astype(np.int32),
               terminated=(rng.random(N_PROG) < 0.2).astype(np.uint8))
    return soa, now


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_20993_b200 import AllocPolicy, Context, GenParams, InterPolicy, Threshold
        from paper_2412_20993_b200.sharding import Sharded, shard_range
        cx = Context(0)
        sh = Sharded(cx)
        assert not sh.nccl and sh.world == world
        r0, n = shard_range(R, rank, world)
        ids = cx.gen_sc(GenParams(seed=77, conv_hi=P), n, P, S, r0=r0)
        pol = AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S)
        res = sh.sc_decide(ids, [Threshold(0, 0.7, 0)], pol, r0)
        soa, now = _soa()
        g0, gn = shard_range(N_PROG, rank, world)
        part = {k: (torch.from_numpy(np.ascontiguousarray(v[g0:g0 + gn])) if v.dtype != np.uint16 else
                    torch.from_numpy(np.ascontiguousarray(v[g0:g0 + gn]).view(np.int16))).cuda()
                for k, v in soa.items()}
        order = sh.gang_order(part, InterPolicy(order=1, starvation_limit=0.15, prior_tokens=128.0), now, g0)
        cx.sync()
        nk = int(res["scalars"][0])
        q.put((rank, res["offsets"].cpu().numpy(), res["kept"][:nk].cpu().numpy().view(np.uint32),
               res["exit_knob"].cpu().numpy(), order.cpu().numpy().view(np.uint32)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        item = q.get(timeout=240)
        got[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ids = O.gen_sc(O.gen_params(seed=77, conv_hi=P), R, P, S)
    _, _, meets = O.sc_certaindex(ids, [(0, 0.7, 0)])
    ref = O.allocate_scan(meets, R, P, 2, 5, P, 1, 64 * S)
    assert np.array_equal(np.concatenate([got[r][0] for r in range(world)]), ref["offsets"])
    assert np.array_equal(np.concatenate([got[r][1] for r in range(world)]), ref["kept"])
    assert np.array_equal(np.concatenate([got[r][2] for r in range(world)]), ref["exit_knob"])
    soa, now = _soa()
    gref, _ = O.gang_order(soa, 1, 0.15, 128.0, now)
    for r in range(world):
        assert np.array_equal(got[r][3], gref)


@pytest.mark.parametrize("config", ["C", "E", "G"])
def test_bench_two_ranks_prints_its_line(config):
    env = dict(os.environ, CDX_BENCH_BACKEND="gloo", CDX_BENCH_SHARE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--config", config,
           "--steps", "2", "--warmup", "3", "--no-others", "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=280)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["scaling"] == ("strong" if config in ("E", "G") else "weak")
