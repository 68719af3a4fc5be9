"""The batched C++ API (include/cdx/batch.hpp) driven by a C++ host (tests/cpp/batch_pipeline.cpp):
SC (K2 -> K5 -> aggregation, also replayed as a CUDA graph), CoT (K3 + epsilon stop),
MCTS/Rebase (K4 -> aggregation) and JSONL ingestion, each output compared bit for bit with
the oracle restatement on the same device-generated traces."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "bin", "batch_pipeline")


def _gp(seed, conv_hi, hes=0.0):
    return O.gen_params(seed=seed, conv_hi=conv_hi, hesitation_prob=hes)


def test_pipeline_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    if not os.path.exists(EXE):
        pytest.fail(f"{EXE} not built")
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([EXE, d], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "no usable sm_100 device" in r.stdout


@pytest.mark.gpu
def test_batch_pipeline_matches_oracle():
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([EXE, d], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr

        def ld(name, dt):
            return np.fromfile(os.path.join(d, name + ".bin"), dtype=dt)

        # SC
        R, P, S = 4096, 64, 32
        ids = O.gen_sc(_gp(31, 64), R, P, S)
        _, h32, meets = O.sc_certaindex(ids, [(0, 0.7, 0)])
        ref = O.allocate_scan(meets, R, P, 2, 5, 64, 1, 64 * S)
        assert np.array_equal(ld("sc_hcert", np.uint32), h32.view(np.uint32).ravel())
        assert np.array_equal(ld("sc_meets", np.uint32), meets.ravel())
        assert np.array_equal(ld("sc_exit", np.int32), ref["exit_knob"])
        assert np.array_equal(ld("sc_offsets", np.int64), ref["offsets"])
        ans = O.sc_aggregate(ids, ref["exit_knob"])
        assert np.array_equal(ld("sc_answer", np.uint32), ans)
        assert ld("sc_scalars", np.int64)[0] == ref["n_kept"]
        assert np.array_equal(ld("sc_exit_graph", np.int32), ref["exit_knob"])
        assert np.array_equal(ld("sc_answer_graph", np.uint32), ans)
        _, _, _, m32, mmeets = O.sc_certaindex_ex(ids, [(0, 0.7, 0), (4, 0.6, 0)])
        assert np.array_equal(ld("sc_majority", np.uint32), m32.view(np.uint32).ravel())
        assert np.array_equal(ld("sc_meets_majority", np.uint32), mmeets.ravel())
        # CoT
        cids, hes = O.gen_cot(_gp(32, 64, 0.05), 8192, 64)
        cref = O.cot_exit(cids, hes, O.probe_cfg(64, 3, 0.9, 4096))
        assert np.array_equal(ld("cot_exit", np.int32), cref["exit_step"])
        assert np.array_equal(ld("cot_reason", np.uint8), cref["reason"])
        assert np.array_equal(ld("cot_final", np.uint32), cref["final_id"])
        estep, _ = O.cot_eps_stop(cids, hes, 3, 0.5)
        assert np.array_equal(ld("cot_eps", np.int32), estep)
        # MCTS / Rebase
        G, T, W = 2048, 16, 64
        rw, rid = O.gen_reward(_gp(33, 16), G, T, W)
        agg = (np.arange(G) % 2).astype(np.uint8)
        _, R32, H32 = O.reward_certaindex(rw, rid, agg)
        assert np.array_equal(ld("rw_R", np.uint32), R32.view(np.uint32).ravel())
        assert np.array_equal(ld("rw_H", np.uint32), H32.view(np.uint32).ravel())
        mh = ld("rw_meets", np.uint32)
        step = np.array([(int(m) & -int(m)).bit_length() - 1 if m else T - 1 for m in mh], np.int32)
        assert np.array_equal(ld("rw_answer", np.uint32), O.reward_aggregate(rw, rid, agg, step))
        assert ld("rw_inexact", np.uint64)[0] == 0
        # JSONL
        nr, npg = ld("jl_counts", np.uint64)
        assert (nr, npg) == (3, 2)
        assert ld("jl_program", np.uint32)[:3].tolist() == [0, 1, 0]
        assert ld("jl_step", np.int32)[:3].tolist() == [1, 1, 2]
        assert ld("jl_tok", np.int64)[:3].tolist() == [64, 64, 128]
        assert ld("jl_hes", np.uint8)[:3].tolist() == [0, 1, 0]
        ao = ld("jl_answer_off", np.uint64)
        aa = ld("jl_answer_arena", np.uint8).tobytes()
        assert [aa[ao[i]:ao[i + 1]] for i in range(3)] == [b" 12 ", b"wait, 7", b"12"]
