"""Multi-rank exchange through the C-ABI with a caller-supplied communicator (SURVEY.md §8(b),
§8(e)): tests/cpp/shard_world2.cpp runs `world` ranks as host threads, one context each
(cdx_ctx_create_comm with allgather / alltoallv callbacks staging through host memory), on
the one reachable B200.  Rank q scores requests / programs of its contiguous shard; the global
token offsets, kept indices, totals (cdx_allocate_scan_sharded) and the global gang order
(cdx_gang_priority_sharded, the distributed sample sort) must equal the single-process oracle."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "bin", "shard_world2")
R, P, S = 6000, 64, 32


def _gang(d, N, seed, order):
    rng = np.random.default_rng(seed)
    arrival = np.cumsum(rng.exponential(1e-3, N))
    arrival[0:-1:5] = arrival[1::5]  # arrival ties: the program-id tie-break crosses ranks
    now = float(arrival[-1]) + 1e-3
    cnt = rng.integers(0, 5, N).astype(np.uint32)
    cap = rng.integers(1, 30, N).astype(np.int32)
    soa = dict(arrival=arrival, last_service=np.maximum(now - rng.exponential(0.2, N), 0.0),
               iter_tok_sum=(rng.integers(1, 500, N) * cnt).astype(np.int64), iter_count=cnt, cap=cap,
               knob=np.minimum(cap, rng.integers(0, 30, N)).astype(np.int32),
               terminated=(rng.random(N) < 0.25).astype(np.uint8))
    for k, v in soa.items():
        np.ascontiguousarray(v).tofile(os.path.join(d, f"gang_{k}.bin"))
    np.array([now, 0.15, 128.0, float(order)]).tofile(os.path.join(d, "gang_params.bin"))
    return soa, now


@pytest.mark.parametrize("world,N,seed,order", [(2, 50000, 1, 1), (3, 20011, 2, 1), (4, 7, 3, 0), (2, 1, 4, 1),
                                                 (5, 100000, 5, 0)])
def test_sharded_cabi_equals_single_process(world, N, seed, order):
    with tempfile.TemporaryDirectory() as d:
        soa, now = _gang(d, N, seed, order)
        r = subprocess.run([EXE, d, str(world)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr

        def ld(q, name, dt):
            return np.fromfile(os.path.join(d, f"rank{q}_{name}.bin"), dtype=dt)
        ids = O.gen_sc(O.gen_params(seed=91, conv_hi=64), R, P, S)
        _, _, meets = O.sc_certaindex(ids, [(0, 0.7, 0)])
        ref = O.allocate_scan(meets, R, P, 2, 5, 64, 1, 64 * S)
        assert np.array_equal(np.concatenate([ld(q, "offsets", np.int64) for q in range(world)]), ref["offsets"])
        assert np.array_equal(np.concatenate([ld(q, "exit", np.int32) for q in range(world)]), ref["exit_knob"])
        assert np.array_equal(np.concatenate([ld(q, "kept", np.uint32) for q in range(world)]),
                              ref["kept"][: ref["n_kept"]])
        budget = int((ref["granted"].astype(np.int64) * 64 * S).sum())
        for q in range(world):
            sc = ld(q, "scalars", np.int64)
            assert sc[1] == ref["tokens_saved"] and sc[2] == budget
            info = ld(q, "info", np.uint64).reshape(world, 4)
            assert [int(x) for x in info[:, 0]] == [R * (k + 1) // world - R * k // world for k in range(world)]
        gref, _ = O.gang_order(soa, order, 0.15, 128.0, now)
        for q in range(world):
            assert np.array_equal(ld(q, "order", np.uint32), gref), q
