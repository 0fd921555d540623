"""Regenerates tests/golden/*.json from the REFERENCE's own code (oracle/_ref, compiled in place
from /root/reference/proj by oracle/Makefile) plus the SPEC's worked examples.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; the GPU box never reads /root/reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def reference_vectors():
    po.build(ref=True)
    R = po.ref_lib()
    g = {"source": "oracle/_ref/libember_ref.so built from /root/reference/proj/src/ordering.cpp + "
                   "include/ember/{common,ordering}.h (unmodified, compiled in place)"}
    # RNG streams, common.h:51-117
    rng = {}
    for seed in (0, 1, 42, 210108358, 2**63 + 5):
        nxt = np.zeros(8, np.uint64)
        R.ref_rng_next(seed, 8, nxt)
        ub = {}
        for n in (1, 2, 7, 1000, 5378385, 2**32 + 3, 2**63 + 1):
            out = np.zeros(8, np.uint64)
            R.ref_rng_uniform_below(seed, n, 8, out)
            ub[str(n)] = [int(x) for x in out]
        uni = np.zeros(8, np.float32)
        R.ref_rng_uniform(seed, -0.1, 0.1, 8, uni)
        sh = np.zeros(10, np.uint32)
        R.ref_rng_shuffle_iota(seed, 10, sh)
        rng[str(seed)] = {"next": [int(x) for x in nxt], "uniform_below": ub,
                          "uniform_m0p1_0p1_bits": [int(x) for x in uni.view(np.uint32)],
                          "shuffle10": [int(x) for x in sh]}
    g["rng"] = rng
    g["splitmix64"] = {str(x): int(R.ref_splitmix64(x)) for x in (0, 1, 12345, 2**64 - 1)}
    g["mix_seed"] = {f"{a},{b}": int(R.ref_mix_seed(a, b)) for a, b in ((0, 0x0e11), (1, 2), (210108358, 7))}
    g["mix_seed3"] = {f"{a},{b},{c}": int(R.ref_mix_seed3(a, b, c)) for a, b, c in ((99, 4, 2), (1, 2, 3))}
    # Ordering plans, ordering.cpp:185-401
    plans = []
    cases = [(0, 4, 2, 42), (0, 6, 3, 7), (0, 16, 4, 0), (0, 16, 8, 3), (0, 16, 16, 0), (0, 32, 8, 1),
             (0, 5, 3, 11), (0, 7, 2, 5), (1, 4, 2, 0), (1, 6, 3, 0), (2, 4, 2, 0), (2, 7, 3, 0), (3, 4, 2, 17),
             (3, 8, 4, 5), (0, 1, 1, 0), (0, 2, 2, 9), (0, 64, 16, 123)]
    for kind, p, c, seed in cases:
        pl = po.ref_plan(kind, p, c, seed)
        plans.append({"kind": kind, "p": p, "c": c, "seed": seed, "seq": pl["seq"].reshape(-1).tolist(),
                      "swap_count": pl["swap_count"], "admissions": pl["admissions"].tolist(),
                      "swaps": pl["swaps"].reshape(-1).tolist(), "bucket_state": pl["bucket_state"].tolist()})
    g["plans"] = plans
    # closed forms (ordering.cpp:163-183)
    g["lower_bound"] = {f"{p},{c}": int(R.ref_lower_bound_swaps(p, c)) for p, c in
                        ((4, 2), (6, 3), (128, 32), (16, 4), (32, 8), (1, 1), (4, 4))}
    g["elim_formula"] = {f"{p},{c}": int(R.ref_elimination_swap_formula(p, c)) for p, c in
                         ((4, 2), (6, 3), (16, 4), (32, 8), (64, 16), (128, 32))}
    io = np.zeros(3, np.uint64)
    R.ref_simulate_io(0, 32, 8, 3, 68_800_000_000 // 32, io)
    g["simulate_io_elim_32_8_3"] = [int(x) for x in io]
    return g


def spec_known_answers():
    """SPEC.md worked examples (file:line cited per entry)."""
    return {
        "score_dot_11": {"line": "SPEC.md:145", "s": [1, 2], "d": [3, 4], "expect": 11.0},
        "adagrad_one": {"line": "SPEC.md:173", "theta": 0.0, "acc": 0.0, "g": 2.0, "lr": 0.1, "eps": 1e-10,
                        "expect_theta": -0.1, "expect_acc": 4.0},
        "adagrad_two": {"line": "SPEC.md:174", "g": 1.0, "lr": 0.1, "expect_theta": -0.1 * (1 + 2 ** -0.5),
                        "tol": 1e-6},
        "loss_zero_negatives": {"line": "SPEC.md:163", "expect": 0.0},
        "loss_all_zero_scores": {"line": "SPEC.md:164", "per_side": "log(1+n)"},
        "eval_mrr": {"line": "SPEC.md:467", "ranks": [1, 2, 4], "mrr": 0.5833333333333334, "hits1": 1 / 3,
                     "hits10": 1.0},
        "eval_tie": {"line": "SPEC.md:459", "pos": 0.5, "negs": [0.5, 0.5, 0.1, -1.0], "rank": 3},
        "lower_bound": {"line": "SPEC.md:259-261", "4,2": 5, "128,32": 247},
        "elimination": {"line": "SPEC.md:234-235", "4,2": 5, "6,3": 7},
        "hilbert_4_2_misses": {"line": "SPEC.md:243", "expect": 9},
    }


if __name__ == "__main__":
    with open(os.path.join(OUT, "reference_rng_ordering.json"), "w") as f:
        json.dump(reference_vectors(), f)
    with open(os.path.join(OUT, "spec_known_answers.json"), "w") as f:
        json.dump(spec_known_answers(), f, indent=1)
    print("wrote golden fixtures to", OUT)
