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
    assert _run() == SPEC
