"""Regenerates tests/golden/reference_cases.npz from the REFERENCE LIBRARY itself
(oracle/_ref/libla_ref.so, compiled from /root/reference/proj/src by oracle/Makefile):
f64 forward (out, g) and backward (dq, dk, dv) of la::forward_* / la::backward_* on
inputs drawn with the reference's own make_tensor (mt19937_64, seeded; q, k row-normalised
by la::normalize_qk, verify.cpp:83). Inputs are not stored: tests regenerate them from
the seeds with oracle.seeded, which is pinned bitwise to make_tensor.

    python tests/golden/make_golden.py      # in the authoring container (needs the reference)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

FM, SM = O.FEATURE_MAJOR, O.SEQUENCE_MAJOR
# (name, G, N, D, causal, a, b, seed, fault)
CASES = [
    ("causal_small", 1, 3, 2, True, 1.0, 1.0, 3, 0),
    ("causal_g2", 2, 37, 8, True, 1.0, 1.0, 11, 0),
    ("full_g2", 2, 37, 8, False, 1.0, 1.0, 13, 0),
    ("causal_coeffs", 1, 129, 16, True, 0.5, 2.0, 17, 0),
    ("full_coeffs", 3, 64, 32, False, 2.0, 0.25, 19, 0),
    ("causal_d64", 1, 130, 64, True, 1.0, 1.0, 23, 0),
    ("fault_offby1", 2, 40, 8, True, 1.0, 1.0, 29, 2),
    ("fault_flipbeta", 2, 40, 8, True, 1.0, 1.0, 31, 1),
    ("fault_dropv", 2, 40, 8, False, 1.0, 1.0, 37, 3),
]


def inputs(G, N, D, seed):
    q = O.normalize_rows(O.seeded(G, N, D, seed + 1, SM))
    k = O.normalize_rows(O.seeded(G, N, D, seed + 2, SM))
    v = O.seeded(G, N, D, seed + 3, FM)
    w = O.seeded(G, N, D, seed + 4, FM)
    return q, k, v, w


def main():
    assert O.ref_lib() is not None, "needs oracle/_ref/libla_ref.so (built from /root/reference)"
    out = {}
    for name, G, N, D, causal, a, b, seed, fault in CASES:
        q, k, v, w = inputs(G, N, D, seed)
        o, g = O.ref_forward(q, k, v, a, b, causal=causal, fault=fault)
        dq, dk, dv = O.ref_backward(q, k, v, o, w, g, a, b, causal=causal, fault=fault)
        out[name + "/meta"] = np.array([G, N, D, int(causal), a, b, seed, fault], np.float64)
        for key, val in (("out", o), ("g", g), ("dq", dq), ("dk", dk), ("dv", dv)):
            out[f"{name}/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **out)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
