"""Shared helpers for the parity tests: seeded inputs exactly as the reference
bench builds them (bench.cpp:75-97), rounding to the device dtype, and the
comparison metrics named in BASELINE.json."""
import numpy as np

from oracle import oracle as O

FM, SM = O.FEATURE_MAJOR, O.SEQUENCE_MAJOR


def bench_inputs(G, N, D, seed=0, normalize=True, need_omega=True):
    """q seed+1, k seed+2 (SequenceMajor, row-normalised), v seed+3, omega seed+4 (FeatureMajor)."""
    q = O.seeded(G, N, D, seed + 1, SM)
    k = O.seeded(G, N, D, seed + 2, SM)
    if normalize:
        q, k = O.normalize_rows(q), O.normalize_rows(k)
    v = O.seeded(G, N, D, seed + 3, FM)
    w = O.seeded(G, N, D, seed + 4, FM) if need_omega else None
    return q, k, v, w


def fast_inputs(G, N, D, seed=0):
    """Large-shape stand-in with the same distribution (U(-1,1), unit q/k rows),
    drawn with numpy for speed; used where the mt19937_64 fill would dominate."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (G, N, D))
    k = rng.uniform(-1, 1, (G, N, D))
    q /= np.linalg.norm(q, axis=2, keepdims=True)
    k /= np.linalg.norm(k, axis=2, keepdims=True)
    v = rng.uniform(-1, 1, (G, N, D))
    w = rng.uniform(-1, 1, (G, N, D))
    return q, k, v, w


def round_to(x, dtype):
    import torch
    t = torch.as_tensor(np.asarray(x, np.float64)).to(getattr(torch, {"f32": "float32", "bf16": "bfloat16",
                                                                       "f16": "float16"}[dtype]))
    return t, t.double().numpy()


def rel_err(x, y):
    """max|x - y| / max|y| (the fp32 <= 1e-5 relative bar)."""
    return float(np.max(np.abs(np.asarray(x) - np.asarray(y))) / max(np.max(np.abs(np.asarray(y))), 1e-30))


def max_abs(x, y):
    return float(np.max(np.abs(np.asarray(x) - np.asarray(y))))
