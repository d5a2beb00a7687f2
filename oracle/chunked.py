"""TEST INFRASTRUCTURE ONLY — float64 chunked restatement of the reference's
causal / non-causal forward and backward, for parity checks at full sequence
length (N up to 1M rows per group) where the loop-for-loop C restatement
(oracle.c) would take minutes per group.

It computes the same quantities as the reference kernels, reorganised into
row chunks so numpy's BLAS does the contractions:

    forward_kernels.hpp:22-56  (constant_causal_core, denominator_causal_core)
        sigma_i = sum_{n<=i} v_n ; z_i = sum_{n<=i} k_n ; g_i = a(i+1) + b q_i.z_i
    forward_kernels.hpp:63-128 (linear_causal_core)
        S_i = sum_{n<=i} k_n^T v_n ; o_i = (a sigma_i + b q_i S_i) / g_i
    forward_kernels.hpp:133-206 (the *_full_core variants): totals over all N, g_i = aN + b q_i.z
    backward_kernels.hpp:21-57  (grad_q_causal_core)   dq_i = b (w_i S_i^T - s_i z_i)
    backward_kernels.hpp:61-130 (grad_k_alpha/beta)    dk_i = b (v_i R_i^T - u_i)
    backward_kernels.hpp:134-168 (grad_v_causal_core)  dv_i = a c_i + b k_i R_i
        with w_i = omega_i / g_i, s_i = o_i.w_i, R_i = sum_{t>=i} q_t^T w_t,
        u_i = sum_{t>=i} s_t q_t, c_i = sum_{t>=i} w_t  (backward.cpp:74-91 for w)
    backward_kernels.hpp:173-288 (grad_*_full_core): the same with full sums.

Every prefix state is accumulated in the FORWARD direction in float64 (no
"total minus suffix" shortcut), so it is a cancellation-free checker. It is
pinned against the C restatement and the reference library at small sizes by
tests/test_oracle.py::test_chunked_oracle_matches_restatement.

Arrays are logical per-group (N, D) float64. ``carry`` optionally injects the
state of rows preceding this sequence shard: (S, z, sigma, row_offset) for the
forward / dq, and (R, u, c) for the backward suffix.
"""
from __future__ import annotations

import numpy as np

CHUNK = 512


def forward(q, k, v, a=1.0, b=1.0, causal=True, prefix=None, row0=0):
    """One group. Returns (o (N, D), g (N,)) in float64."""
    q, k, v = (np.asarray(x, np.float64) for x in (q, k, v))
    N, D = q.shape
    if not causal:
        S = k.T @ v
        z = k.sum(0)
        sig = v.sum(0)
        g = a * N + b * (q @ z)
        return (a * sig[None, :] + b * (q @ S)) / g[:, None], g
    S = np.zeros((D, D)) if prefix is None else np.array(prefix[0], np.float64)
    z = np.zeros(D) if prefix is None else np.array(prefix[1], np.float64)
    sig = np.zeros(D) if prefix is None else np.array(prefix[2], np.float64)
    o = np.empty((N, D))
    g = np.empty(N)
    for s0 in range(0, N, CHUNK):
        s1 = min(N, s0 + CHUNK)
        qc, kc, vc = q[s0:s1], k[s0:s1], v[s0:s1]
        P = np.tril(a + b * (qc @ kc.T))
        f = P @ vc + a * sig[None, :] + b * (qc @ S)
        gc = P.sum(1) + a * (row0 + s0) + b * (qc @ z)
        o[s0:s1] = f / gc[:, None]
        g[s0:s1] = gc
        S += kc.T @ vc
        z += kc.sum(0)
        sig += vc.sum(0)
    return o, g


def backward(q, k, v, o, omega, g, a=1.0, b=1.0, causal=True, prefix=None, suffix=None):
    """One group. Returns (dq, dk, dv), each (N, D) float64."""
    q, k, v, o, omega = (np.asarray(x, np.float64) for x in (q, k, v, o, omega))
    g = np.asarray(g, np.float64)
    N, D = q.shape
    w = omega / g[:, None]
    s = (o * w).sum(1)
    if not causal:
        S, z = k.T @ v, k.sum(0)
        R, u, c = q.T @ w, q.T @ s, w.sum(0)
        dq = b * (w @ S.T - s[:, None] * z[None, :])
        dk = b * (v @ R.T - u[None, :])
        dv = a * c[None, :] + b * (k @ R)
        return dq, dk, dv
    dq = np.empty((N, D))
    dk = np.empty((N, D))
    dv = np.empty((N, D))
    S = np.zeros((D, D)) if prefix is None else np.array(prefix[0], np.float64)
    z = np.zeros(D) if prefix is None else np.array(prefix[1], np.float64)
    for s0 in range(0, N, CHUNK):
        s1 = min(N, s0 + CHUNK)
        kc, vc, wc, sc = k[s0:s1], v[s0:s1], w[s0:s1], s[s0:s1]
        dS = b * np.tril(wc @ vc.T - sc[:, None])
        dq[s0:s1] = dS @ kc + b * (wc @ S.T - sc[:, None] * z[None, :])
        S += kc.T @ vc
        z += kc.sum(0)
    R = np.zeros((D, D)) if suffix is None else np.array(suffix[0], np.float64)
    u = np.zeros(D) if suffix is None else np.array(suffix[1], np.float64)
    c = np.zeros(D) if suffix is None else np.array(suffix[2], np.float64)
    last = ((N - 1) // CHUNK) * CHUNK
    for s0 in range(last, -1, -CHUNK):
        s1 = min(N, s0 + CHUNK)
        qc, kc, vc, wc, sc = q[s0:s1], k[s0:s1], v[s0:s1], w[s0:s1], s[s0:s1]
        P = np.tril(a + b * (qc @ kc.T))
        dS = b * np.tril(wc @ vc.T - sc[:, None])
        dk[s0:s1] = dS.T @ qc + b * (vc @ R.T - u[None, :])
        dv[s0:s1] = P.T @ wc + a * c[None, :] + b * (kc @ R)
        R += qc.T @ wc
        u += qc.T @ sc
        c += wc.sum(0)
    return dq, dk, dv


def shard_totals_forward(k, v):
    """(S, z, sigma) over a shard's rows (the forward's all-gathered record)."""
    k, v = np.asarray(k, np.float64), np.asarray(v, np.float64)
    return k.T @ v, k.sum(0), v.sum(0)


def shard_totals_backward(q, o, omega, g):
    """(R, u, c) over a shard's rows (the backward's all-gathered record)."""
    q, o, omega = (np.asarray(x, np.float64) for x in (q, o, omega))
    w = omega / np.asarray(g, np.float64)[:, None]
    s = (o * w).sum(1)
    return q.T @ w, q.T @ s, w.sum(0)
