"""CPU: the majority-fraction restatement (oracle/cdx_oracle.c cdxo_majority_fraction,
cdxo_sc_certaindex_ex) pinned to the reference's own plurality vote.

The reference has no majority-fraction function; north_star (2) names the signal and the
reference's SC aggregation defines it: ProgramDriver::aggregate_prefix -> weighted_plurality
(runtime.cpp:317-334) returns the first-seen answer of largest weight.  The restated fraction
must equal (occurrences of the reference's winner among the trimmed answers) / n, bit for bit,
on random rows with many ties, and its thresholds follow combined_meets_thresholds
(metrics.cpp:159-171) exactly as the entropy signal's do.
"""
import numpy as np
import pytest

from oracle import oracle as O

SC = 0
VOC = O.vocab(5)  # "S", "D1".."D4", and their hesitant forms


@pytest.mark.parametrize("seed", range(4))
def test_majority_restatement_pinned_to_reference_vote(seed):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    R, P, S = 24, 6, (16, 32, 7, 3)[seed]
    ids = rng.integers(0, (2, 5, 3, 4)[seed], size=(R, P, S)).astype(np.uint32)
    _, _, m64, m32, _ = O.sc_certaindex_ex(ids, [])
    for r in range(R):
        for p in range(P):
            row = ids[r, p].tolist()
            win = O.ref_aggregate(SC, row, None, [], S, VOC)
            want = float(row.count(win)) / float(S)
            assert m64[r, p] == want
            assert m32[r, p] == np.float32(want)


def test_majority_fraction_examples():
    assert O.majority_fraction([3]) == 1.0
    assert O.majority_fraction([1, 2]) == 2 / 3
    assert O.majority_fraction([2, 2, 1]) == 0.4  # tie: the first-seen winner, same share
    assert O.majority_fraction([1] * 32) == 1 / 32


def test_majority_thresholds_and_entropy_and():
    """Thresholds on the majority signal AND the entropy signal, inclusive compares."""
    ids = np.array([[[0, 0, 0, 1], [0, 1, 2, 3], [0, 0, 1, 1]]], np.uint32)  # maj 0.75, 0.25, 0.5
    _, _, m64, _, meets = O.sc_certaindex_ex(ids, [(4, 0.5, 0)])
    assert list(m64[0]) == [0.75, 0.25, 0.5]
    assert int(meets[0, 0]) == 0b101
    _, _, _, _, meets = O.sc_certaindex_ex(ids, [(4, 0.5, 0), (4, 0.5, 1)])
    assert int(meets[0, 0]) == 0b100
    h64, _, _, _, meets = O.sc_certaindex_ex(ids, [(4, 0.5, 0), (0, 0.5, 0)])
    want = sum(1 << p for p in range(3) if m64[0, p] >= 0.5 and h64[0, p] >= 0.5)
    assert int(meets[0, 0]) == want
    _, _, _, _, meets = O.sc_certaindex_ex(ids, [(4, float("nan"), 0)])
    assert int(meets[0, 0]) == 0
