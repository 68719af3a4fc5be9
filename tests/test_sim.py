"""The sim module's SPEC examples through cdx::sim (include/cdx/sim.hpp),
a host event loop whose every scheduling decision is scheduler::next_batch -> K6 on the
B200: Fig. 5's 6.5 ms (gang) vs 9 ms (interleaved), deadlines, SJF by estimated remaining
work, attainment with horizon truncation."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "bin", "sim_cases")

SPEC = {
    "deadline 1 1 240": "240",      # SPEC.md:510 (Table 2 SC/MATH)
    "deadline 1.5 2 60": "180",
    "deadline 1 3 300": "900",
    "fig5 gang": "6.5",
    "fig5 interleaved": "9",
    "zero programs": "0 0",
    "single program": "7 7",        # gang on/off identical
    "sjf": "90 20 40",              # short programs overtake (est x remaining knob)
    "attainment": "0.9 0.3 1",
    "attainment empty": "EXC attainment: empty report",
}


def _run():
    if not os.path.exists(EXE):
        pytest.fail(f"{EXE} not built")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return dict(l.split(" | ", 1) for l in r.stdout.splitlines())


def test_sim_host_arithmetic_and_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    got = _run()
    for k in ("deadline 1 1 240", "deadline 1.5 2 60", "deadline 1 3 300", "zero programs", "attainment empty"):
        assert got[k] == SPEC[k]
    assert "no usable sm_100 device" in got["fig5 gang"]


@pytest.mark.gpu
def test_sim_spec_examples():
    got = _run()
    assert {k: got[k] for k in SPEC} == SPEC


def _poisson_restated(n, rate, seed):
    """SimConfig::arrival_rate restated: gaps -log1p(-u)/rate, u = 53-bit uniform of the
    reference's derive_seed(seed, i, 0) (rng.hpp:25-34, through the oracle's copy)."""
    import math
    from oracle import oracle as O
    t, out = 0.0, []
    for i in range(n):
        u = (O.lib().cdxo_derive_seed(seed, i, 0) >> 11) * 2.0 ** -53
        t += -math.log1p(-u) / rate
        out.append(t)
    return out


@pytest.mark.gpu
def test_sim_knob_programs_poisson_and_allocate():
    """Knob-unit SC programs (signals from the reference API on the B200) under Poisson
    arrivals, allocate at detect / recheck points.  SPEC properties: safety
    (knob <= cap), determinism, throughput ceiling, early-exit savings at equal accuracy on a
    zero-residual-noise workload, threshold monotonicity, the
    token-to-accuracy curve."""
    got = _run()
    want = _poisson_restated(6, 250.0, 99)
    assert [float(x) for x in got["poisson"].split()] == pytest.approx(want, rel=1e-8, abs=0)

    def parse(k):
        v = got[k].split()
        return dict(tokens=float(v[0]), acc=float(v[1]), units=int(v[2]), dec=int(v[3]), cert=int(v[4]),
                    maxknob=int(v[5]), lat=float(v[6]), makespan=float(v[7]), tput=float(v[8]), trunc=int(v[9]))
    even, static, kstep, k07 = (parse(k) for k in ("knob even", "knob static", "knob kstep", "knob kstep tau0.7"))
    NP, CAP, S = 48, 16, 8
    for r in (even, static, kstep, k07):
        assert r["maxknob"] <= CAP and r["trunc"] == 0                  # safety
        assert r["tput"] <= 16 * 64000.0 * (1 + 1e-12)                   # throughput ceiling
        assert r["tokens"] == r["units"] * S * 64                        # every unit issues S requests
    assert got["knob kstep repeat"] == got["knob kstep"]                 # determinism
    assert even["units"] == NP * CAP and even["cert"] == 0 and even["dec"] == NP
    # tau = 1: stop only on a unanimous row; residual noise 0 -> every converged row is unanimous "S"
    assert kstep["acc"] == even["acc"] and static["acc"] == even["acc"]
    assert kstep["tokens"] < static["tokens"] < even["tokens"]
    assert kstep["cert"] > 0 and kstep["lat"] < even["lat"]
    assert k07["tokens"] <= kstep["tokens"]
    assert got["knob monotone"] == "0"
    pts = [tuple(map(float, p.split(":"))) for p in got["curve"].split()]
    assert len(pts) == 2 and pts[0][0] < pts[1][0]
    assert pts[1][0] == 2 * pts[0][0]                                     # even allocation: cap 16 = 2 x cap 8
