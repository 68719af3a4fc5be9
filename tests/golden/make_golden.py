"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref/libcdxref.so, the
reference's own C++ sources compiled here) — the fixtures that pin the C restatement
(oracle/cdx_oracle.c) and, through it, the CUDA path.

Run in the dev container (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs /root/reference.
"""
import itertools
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def spec_examples():
    """SPEC.md examples (metrics :46-93, probe :157-186, runtime :346-348) as computed by
    the reference functions."""
    ex = {}
    ex["cluster_exact"] = [
        {"in": a, "out": O.ref_cluster_exact(a)}
        for a in (["7", "7", "7"], ["a", "b", "c"], ["12", " 12", "13"], ["\t x\n", "x", " y", "y ", "x\v"])]
    ex["entropy"] = [{"sizes": s, "H": O.ref_entropy(s)[0], "Hc": O.ref_entropy(s)[1]}
                     for s in ([4], [1, 1, 1, 1], [2, 2], [3, 1, 1], [1], [2, 1], [5, 3, 2, 1, 1])]
    ex["reward"] = [{"r": r, "agg_max": m, "out": O.ref_certaindex_reward(r, m)}
                    for r, m in (([0.9], 0), ([0.9], 1), ([0.2, 0.9], 1), ([0.2, 0.4, 0.6], 0), ([0.2, 0.6], 0))]
    errs = []
    for r in ([1.5], [-0.1, 0.5], []):
        try:
            O.ref_certaindex_reward(r, 0)
            errs.append({"r": r, "error": None})
        except O.RefError as e:
            errs.append({"r": r, "error": str(e)})
    ex["reward_errors"] = errs
    th = [(0, 0.99, 0), (1, 0.4, 0)]
    ex["meets"] = [{"signals": {"0": 0.995, "1": 0.5}, "th": th, "out": O.ref_meets({0: 0.995, 1: 0.5}, th)},
                   {"signals": {"0": 0.995, "1": 0.3}, "th": th, "out": O.ref_meets({0: 0.995, 1: 0.3}, th)},
                   {"signals": {"0": 0.5}, "th": [], "out": O.ref_meets({0: 0.5}, [])}]
    try:
        O.ref_meets({0: 0.5}, [(1, 0.4, 0)])
        ex["meets_absent_error"] = None
    except O.RefError as e:
        ex["meets_absent_error"] = str(e)
    mk = ["wait", "hmm"]
    ex["hesitation"] = [{"a": a, "m": m, "out": O.ref_flag_hesitation(a, m)}
                        for a, m in (("42", mk), ("wait, let me check", mk), ("Hmm 42", mk), ("WAIT", ["WAIT"]),
                                     ("abc", [""]), ("xHMMx", ["hmm"]))]
    recs = lambda answers, hes=None: [(i + 1, (i + 1) * 64, a, bool(hes and hes[i])) for i, a in enumerate(answers)]
    ex["consistency"] = [
        {"recs": recs(["x", "x", "x"]), "k": 3, "w": 3, "out": O.ref_consistency(recs(["x", "x", "x"]), 3, 3)},
        {"recs": recs(["x", "y", "x"]), "k": 3, "w": 3, "out": O.ref_consistency(recs(["x", "y", "x"]), 3, 3)},
        {"recs": recs(["x", "x", "x"], [0, 1, 0]), "k": 3, "w": 2,
         "out": O.ref_consistency(recs(["x", "x", "x"], [0, 1, 0]), 3, 2)},
        {"recs": recs(["x", "y"]), "k": 2, "w": 3, "out": O.ref_consistency(recs(["x", "y"]), 2, 3)},
    ]
    se = []
    for answers, hes, w, tau, mt in ((["a", "a"], None, 2, 1.0, 10 ** 6), (["a", "b"], None, 2, 1.0, 128),
                                     (["a", "a", "b", "a", "a"], None, 5, 0.6, 10 ** 6),
                                     (["a", "b", "c"], [0, 0, 1], 2, 0.5, 192)):
        se.append({"recs": recs(answers, hes), "w": w, "tau": tau, "max_tokens": mt,
                   "out": O.ref_should_exit(recs(answers, hes), 64, w, tau, mt)})
    ex["should_exit"] = se
    fa = []
    for answers, hes, term, reason in ((["a", "b", "7"], None, 3, 0), (["a", "b"], [0, 1], 2, 1), (["x"], None, 1, 1),
                                       (["a", "b"], [1, 1], 2, 1)):
        fa.append({"recs": recs(answers, hes), "terminated_at": term, "reason": reason,
                   "out": O.ref_final_answer(recs(answers, hes), term, reason)})
    ex["final_answer"] = fa
    jl = []
    for text in ('{"program_id":"p","step_index":1,"token_offset":64,"answer":"a"}\n'
                 '{"program_id":"p","step_index":2,"token_offset":64,"answer":"a"}\n',
                 '{"program_id":"p","step_index":1,"token_offset":64,"answer":"a","hesitant":true}\n\n'
                 '{"program_id":"q","step_index":1,"token_offset":10,"answer":"b"}\n'):
        try:
            jl.append({"text": text, "lines": O.ref_read_trace_jsonl(text), "error": None})
        except O.RefError as e:
            jl.append({"text": text, "lines": None, "error": str(e)})
    ex["jsonl"] = jl
    ent, rew, ln = O.ref_driver_signals(2, 123, 20, 5, 1, 6)
    ex["driver_mcts"] = {"entropy": ent, "reward": rew, "mean_len": ln}
    ent, rew, ln = O.ref_driver_signals(0, 77, 20, 3, 1, 6)
    ex["driver_sc"] = {"entropy": ent, "reward": rew, "mean_len": ln}
    ex["mix64"] = [[x, O.ref().ref_mix64(x)] for x in (0, 1, 20993, 2 ** 63 + 5)]
    ex["derive_seed"] = [[a, b, c, O.ref().ref_derive_seed(a, b, c)] for a, b, c in ((20993, 1, 2), (7, 0, 0x757))]
    return ex


def partitions(n, mx=None):
    mx = n if mx is None else mx
    if n == 0:
        yield []
        return
    for k in range(min(n, mx), 0, -1):
        for rest in partitions(n - k, k):
            yield [k] + rest


def entropy_suite():
    """H and H~ for every clustering shape of n <= 12, in every distinct cluster order,
    straight from metrics::semantic_entropy / certaindex_entropy."""
    out = []
    for n in range(1, 13):
        for part in partitions(n):
            for perm in sorted(set(itertools.permutations(part))):
                H, Hc = O.ref_entropy(list(perm))
                out.append([list(perm), H.hex(), Hc.hex()])
    return out


def sc_rows():
    """A seeded SC trace (configs A-like) with the reference's per-row H~ and meets bits."""
    g = O.gen_params(seed=11, conv_hi=32)
    ids = O.gen_sc(g, 24, 32, 16)
    ths = [(0, 0.7, 0)]
    h, meets = O.ref_sc_batch(ids, 5, ths, nthreads=1)
    return {"seed": 11, "R": 24, "P": 32, "S": 16, "conv_hi": 32, "tau": 0.7,
            "ids_sha": __import__("hashlib").sha256(ids.tobytes()).hexdigest(),
            "hcert": [float(x).hex() for x in h.ravel()], "meets": meets.ravel().tolist()}


def cot_rows():
    g = O.gen_params(seed=5, conv_hi=64, hesitation_prob=0.1)
    ids, hes = O.gen_cot(g, 40, 64)
    r = O.ref_cot_batch(ids, hes, 5, 64, 3, 0.9, 4096, nthreads=1)
    return {"seed": 5, "R": 40, "P": 64, "hes_prob": 0.1, "w": 3, "tau": 0.9, "max_tokens": 4096,
            "ids_sha": __import__("hashlib").sha256(ids.tobytes() + hes.tobytes()).hexdigest(),
            **{k: v.ravel().tolist() for k, v in r.items() if k != "ck"},
            "ck": [float(x).hex() for x in r["ck"].ravel()]}


def reward_rows():
    g = O.gen_params(seed=9, conv_hi=16)
    rw, ids = O.gen_reward(g, 12, 8, 16)
    agg = (np.arange(12) % 2).astype(np.uint8)
    R, H = O.ref_reward_batch(rw, ids, agg, nthreads=1)
    return {"seed": 9, "G": 12, "T": 8, "W": 16, "conv_hi": 16,
            "R": [float(x).hex() for x in R.ravel()], "H": [float(x).hex() for x in H.ravel()]}


def main():
    if not O.ref_available():
        raise SystemExit("reference library unavailable; run in the dev container")
    data = {"spec": spec_examples(), "entropy_suite": entropy_suite(), "sc": sc_rows(), "cot": cot_rows(),
            "reward": reward_rows()}
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(data, f, indent=0, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
