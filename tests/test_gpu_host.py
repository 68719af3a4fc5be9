"""GPU: the end-to-end host-buffer entry cdx_sc_decide_host (chunked H2D + K2 + K5 + D2H)
equals the oracle, including global budget offsets across chunks."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,P,S", [(1, 32, 16), (5000, 64, 32), (70000, 64, 32), (3000, 20, 7)])
def test_sc_decide_host(ctx, R, P, S):
    from paper_2412_20993_b200 import AllocPolicy, Threshold, c_policy, c_thresholds
    ids = O.gen_sc(O.gen_params(seed=R, conv_hi=P), R, P, S)
    ex = np.empty(R, np.int32)
    why = np.empty(R, np.uint8)
    off = np.empty(R, np.int64)
    hc = np.empty((R, P), np.float32)
    saved = C.c_int64(0)
    arr, n = c_thresholds([Threshold(0, 0.7, 0)])
    pol = c_policy(AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S))
    st = ctx.lib.cdx_sc_decide_host(ctx.h, ids.ctypes.data, R, P, S, arr, n, C.byref(pol), ex.ctypes.data,
                                    why.ctypes.data, off.ctypes.data, hc.ctypes.data, C.byref(saved))
    ctx._check(st)
    _, oh32, om = O.sc_certaindex(ids, [(0, 0.7, 0)])
    ref = O.allocate_scan(om, R, P, 2, 5, P, 1, 64 * S)
    assert np.array_equal(hc.view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(ex, ref["exit_knob"]) and np.array_equal(why, ref["reason"])
    assert np.array_equal(off, ref["offsets"])
    assert saved.value == ref["tokens_saved"]
