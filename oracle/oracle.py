"""TEST INFRASTRUCTURE ONLY — Python access to the CPU oracle.

Two checkers live here, both loaded with ctypes:

* ``liboracle.so``: the plain-C restatement of the reference kernels
  (oracle.c; forward_kernels.hpp / backward_kernels.hpp loop for loop).
* ``_ref/libla_ref.so``: the unmodified reference library compiled from
  /root/reference/proj/src (oracle/Makefile) plus a C shim. Optional: present
  when it was built in the authoring container and shipped with the snapshot.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) import this module. The product (paper_2510_21956_b200) never does.

Tensors are handled as *logical* float arrays of shape (G, N, D); ``to_flat`` /
``from_flat`` convert to the reference storage layouts (tensor.hpp:12-15):
FeatureMajor (0) = g*N*D + j*N + i, SequenceMajor (1) = g*N*D + i*D + j.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FEATURE_MAJOR, SEQUENCE_MAJOR = 0, 1
FAULTS = {"none": 0, "beta-k-sign": 1, "causal-off-by-one": 2, "drop-v-a-term": 3}


class OracleDegenerate(Exception):
    def __init__(self, group, position):
        super().__init__(f"degenerate attention denominator at group {group}, position {position}")
        self.group, self.position = int(group), int(position)


def to_flat(x, layout):
    x = np.asarray(x)
    return np.ascontiguousarray(x.transpose(0, 2, 1) if layout == FEATURE_MAJOR else x).reshape(-1)


def from_flat(flat, G, N, D, layout):
    flat = np.asarray(flat)
    if layout == FEATURE_MAJOR:
        return flat.reshape(G, D, N).transpose(0, 2, 1)
    return flat.reshape(G, N, D)


_i64p = C.POINTER(C.c_int64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


_lib = None
_ref = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _lib = C.CDLL(path)
    return _lib


def ref_lib():
    """The reference library itself, or None when it was not built/shipped."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libla_ref.so")
        if not os.path.exists(path) and os.path.isdir("/root/reference/proj/src"):
            build()
        if not os.path.exists(path):
            return None
        _ref = C.CDLL(path)
    return _ref


# --------------------------------------------------------------------------- fixtures
def seeded(G, N, D, seed, layout=SEQUENCE_MAJOR, lo=-1.0, hi=1.0):
    """make_tensor(SeededUniform) (tensor.cpp:43-77) as a logical (G,N,D) array."""
    flat = np.empty(G * N * D, np.float64)
    lib().oracle_fill_uniform(_p(flat), C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_int(layout),
                              C.c_uint64(seed), C.c_double(lo), C.c_double(hi))
    return from_flat(flat, G, N, D, layout).copy()


def normalize_rows(x):
    """normalize_qk row normalisation (plan.cpp:95-117) on a logical array."""
    x = np.array(x, np.float64, copy=True)
    G, N, D = x.shape
    flat = to_flat(x, SEQUENCE_MAJOR)
    lib().oracle_normalize_rows(_p(flat), C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_int(1))
    return from_flat(flat, G, N, D, SEQUENCE_MAJOR).copy()


# --------------------------------------------------------------------------- kernels
def forward(q, k, v, a=1.0, b=1.0, causal=True, fault=0, dtype=np.float64,
            lq=SEQUENCE_MAJOR, lk=SEQUENCE_MAJOR, lv=FEATURE_MAJOR):
    """run_forward<T> restated. Returns logical (out, g) arrays in ``dtype``."""
    G, N, D = q.shape
    qf, kf, vf = (to_flat(np.asarray(x, dtype), l) for x, l in ((q, lq), (k, lk), (v, lv)))
    out = np.zeros(G * N * D, dtype)
    g = np.zeros(G * N, dtype)
    bg, bp = C.c_int64(-1), C.c_int64(-1)
    fn = lib().oracle_forward_f64 if dtype == np.float64 else lib().oracle_forward_f32
    st = fn(_p(qf), lq, _p(kf), lk, _p(vf), lv, C.c_int64(G), C.c_int64(N), C.c_int64(D),
            C.c_double(a), C.c_double(b), C.c_int(int(causal)), C.c_int(fault), _p(out), _p(g),
            C.byref(bg), C.byref(bp))
    if st:
        raise OracleDegenerate(bg.value, bp.value)
    return from_flat(out, G, N, D, FEATURE_MAJOR).copy(), g.reshape(G, N)


def backward(q, k, v, o, omega, g, a=1.0, b=1.0, causal=True, fault=0, dtype=np.float64,
             lq=SEQUENCE_MAJOR, lk=SEQUENCE_MAJOR, lv=FEATURE_MAJOR, lo=FEATURE_MAJOR,
             lw=FEATURE_MAJOR):
    """run_backward<T> restated. Returns logical (dq, dk, dv)."""
    G, N, D = q.shape
    fl = [to_flat(np.asarray(x, dtype), l) for x, l in ((q, lq), (k, lk), (v, lv), (o, lo),
                                                        (omega, lw))]
    gf = np.ascontiguousarray(np.asarray(g, dtype).reshape(-1))
    dq = np.zeros(G * N * D, dtype)
    dk = np.zeros(G * N * D, dtype)
    dv = np.zeros(G * N * D, dtype)
    fn = lib().oracle_backward_f64 if dtype == np.float64 else lib().oracle_backward_f32
    fn(_p(fl[0]), lq, _p(fl[1]), lk, _p(fl[2]), lv, _p(fl[3]), lo, _p(fl[4]), lw, _p(gf),
       C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_double(a), C.c_double(b),
       C.c_int(int(causal)), C.c_int(fault), _p(dq), _p(dk), _p(dv))
    return (from_flat(dq, G, N, D, SEQUENCE_MAJOR).copy(), from_flat(dk, G, N, D, FEATURE_MAJOR).copy(),
            from_flat(dv, G, N, D, FEATURE_MAJOR).copy())


def quadratic(q, k, v, a=1.0, b=1.0, causal=True):
    """quadratic_la (reference.cpp:67-106): O(N^2 D) ground truth."""
    G, N, D = q.shape
    qf, kf, vf = (to_flat(np.asarray(x, np.float64), SEQUENCE_MAJOR) for x in (q, k, v))
    out = np.zeros(G * N * D)
    g = np.zeros(G * N)
    bg, bp = C.c_int64(-1), C.c_int64(-1)
    st = lib().oracle_quadratic(_p(qf), 1, _p(kf), 1, _p(vf), 1, C.c_int64(G), C.c_int64(N),
                                C.c_int64(D), C.c_double(a), C.c_double(b), C.c_int(int(causal)),
                                _p(out), _p(g), C.byref(bg), C.byref(bp))
    if st:
        raise OracleDegenerate(bg.value, bp.value)
    return out.reshape(G, N, D), g.reshape(G, N)


def fwd_bwd_f32_threads(q, k, v, omega, a=1.0, b=1.0, causal=True, threads=1):
    """CPU-baseline port: f32 fwd+bwd over groups on `threads` host threads.
    Inputs are flat canonical-layout float32 arrays (q,k SeqMajor; v,omega FeatMajor)."""
    G, N, D = q.shape[0], q.shape[1], q.shape[2]
    q, k, v, omega = (np.ascontiguousarray(x, np.float32) for x in (q, k, v, omega))
    out = np.empty(G * N * D, np.float32)
    g = np.empty(G * N, np.float32)
    dq, dk, dv = (np.empty(G * N * D, np.float32) for _ in range(3))
    st = lib().oracle_fwd_bwd_f32_threads(_p(q), _p(k), _p(v), _p(omega), C.c_int64(G), C.c_int64(N),
                                          C.c_int64(D), C.c_double(a), C.c_double(b),
                                          C.c_int(int(causal)), C.c_int(threads), _p(out), _p(g),
                                          _p(dq), _p(dk), _p(dv))
    if st:
        raise OracleDegenerate(-1, -1)
    return out, g, dq, dk, dv


# --------------------------------------------------------------------------- reference lib
def ref_seeded(G, N, D, seed, layout):
    r = ref_lib()
    flat = np.empty(G * N * D)
    r.ref_make_tensor(_p(flat), C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_int(layout),
                      C.c_uint64(seed))
    return from_flat(flat, G, N, D, layout).copy()


def ref_forward(q, k, v, a=1.0, b=1.0, causal=True, fault=0, L=0, workers=2,
                lq=SEQUENCE_MAJOR, lk=SEQUENCE_MAJOR, lv=FEATURE_MAJOR):
    """la::forward_causal / forward_full (f64 public API) of the reference itself."""
    G, N, D = q.shape
    fl = [to_flat(np.asarray(x, np.float64), l) for x, l in ((q, lq), (k, lk), (v, lv))]
    out = np.zeros(G * N * D)
    g = np.zeros(G * N)
    bg, bp = C.c_int64(-1), C.c_int64(-1)
    st = ref_lib().ref_forward_f64(C.c_int(int(causal)), _p(fl[0]), lq, _p(fl[1]), lk, _p(fl[2]), lv,
                                   C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_double(a),
                                   C.c_double(b), C.c_int(fault), C.c_int64(L), C.c_int(workers),
                                   _p(out), _p(g), C.byref(bg), C.byref(bp))
    if st == 6:
        raise OracleDegenerate(bg.value, bp.value)
    if st:
        raise RuntimeError(f"reference forward failed with status {st}")
    return from_flat(out, G, N, D, FEATURE_MAJOR).copy(), g.reshape(G, N)


def ref_backward(q, k, v, o, omega, g, a=1.0, b=1.0, causal=True, fault=0, L=0, workers=2,
                 lq=SEQUENCE_MAJOR, lk=SEQUENCE_MAJOR, lv=FEATURE_MAJOR, lw=FEATURE_MAJOR):
    G, N, D = q.shape
    fl = [to_flat(np.asarray(x, np.float64), l) for x, l in ((q, lq), (k, lk), (v, lv),
                                                              (o, FEATURE_MAJOR), (omega, lw))]
    gf = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    dq, dk, dv = (np.zeros(G * N * D) for _ in range(3))
    st = ref_lib().ref_backward_f64(C.c_int(int(causal)), _p(fl[0]), lq, _p(fl[1]), lk, _p(fl[2]),
                                    lv, _p(fl[3]), _p(fl[4]), lw, _p(gf), C.c_int64(G),
                                    C.c_int64(N), C.c_int64(D), C.c_double(a), C.c_double(b),
                                    C.c_int(fault), C.c_int64(L), C.c_int(workers), _p(dq),
                                    _p(dk), _p(dv))
    if st:
        raise RuntimeError(f"reference backward failed with status {st}")
    return (from_flat(dq, G, N, D, SEQUENCE_MAJOR).copy(), from_flat(dk, G, N, D, FEATURE_MAJOR).copy(),
            from_flat(dv, G, N, D, FEATURE_MAJOR).copy())


def ref_finite_diff(q, k, v, omega, a=1.0, b=1.0, causal=True, h=1e-6):
    G, N, D = q.shape
    fl = [to_flat(np.asarray(x, np.float64), SEQUENCE_MAJOR) for x in (q, k, v, omega)]
    dq, dk, dv = (np.zeros(G * N * D) for _ in range(3))
    st = ref_lib().ref_finite_diff(C.c_int(int(causal)), _p(fl[0]), 1, _p(fl[1]), 1, _p(fl[2]), 1,
                                   _p(fl[3]), 1, C.c_int64(G), C.c_int64(N), C.c_int64(D),
                                   C.c_double(a), C.c_double(b), C.c_double(h), _p(dq), _p(dk),
                                   _p(dv))
    if st:
        raise RuntimeError(f"reference finite_diff failed with status {st}")
    return tuple(from_flat(x, G, N, D, SEQUENCE_MAJOR).copy() for x in (dq, dk, dv))


def ref_fwd_bwd_f32(q, k, v, omega, a=1.0, b=1.0, causal=True, workers=1, outs=None):
    """The reference's own timed fast path: run_forward<float> then run_backward<float>
    on flat canonical-layout float32 inputs (bench.cpp:137-139, 176-179). ``outs`` =
    (out, g, dq, dk, dv) preallocated float32 buffers (reused across timed steps, as the
    reference bench reuses its own, bench.cpp:111-191)."""
    r = ref_lib()
    G, N, D = q.shape
    q, k, v, omega = (np.ascontiguousarray(x, np.float32) for x in (q, k, v, omega))
    if outs is None:
        outs = (np.empty(G * N * D, np.float32), np.empty(G * N, np.float32),
                *(np.empty(G * N * D, np.float32) for _ in range(3)))
    out, g = outs[0], outs[1]
    st = r.ref_run_forward_f32(C.c_int(int(causal)), _p(q), _p(k), _p(v), C.c_int64(G), C.c_int64(N),
                               C.c_int64(D), C.c_double(a), C.c_double(b), C.c_int(workers), _p(out),
                               _p(g))
    if st:
        raise RuntimeError(f"reference run_forward<float> failed with status {st}")
    dq, dk, dv = outs[2], outs[3], outs[4]
    st = r.ref_run_backward_f32(C.c_int(int(causal)), _p(q), _p(k), _p(v), _p(out), _p(omega), _p(g),
                                C.c_int64(G), C.c_int64(N), C.c_int64(D), C.c_double(a),
                                C.c_double(b), C.c_int(workers), _p(dq), _p(dk), _p(dv))
    if st:
        raise RuntimeError(f"reference run_backward<float> failed with status {st}")
    return out, g, dq, dk, dv


# --------------------------------------------------------------------------- prologue + term passes
# numpy restatements (logical (G, N, D) arrays, f64) of the reference's API calls
# either side of the hot path; pinned against the reference library in tests/test_oracle.py.
def relayout_flat(x, layout):
    """relayout (tensor.cpp:101-119): the flat buffer of logical x in ``layout``."""
    return to_flat(np.asarray(x, np.float64), layout)


def omega_hat(omega, g):
    """make_omega_hat (backward.cpp:74-91): omega_ij / g_i."""
    G, N, _ = omega.shape
    return np.asarray(omega, np.float64) / np.asarray(g, np.float64).reshape(G, N, 1)


def constant_term(v, a):
    """constant_causal_core (forward_kernels.hpp:22-34): f_ij = running sum of a*v_nj."""
    return np.cumsum(a * np.asarray(v, np.float64), axis=1)


def linear_term(q, k, v, b, f):
    """linear_causal_core with g_vec = null (forward_kernels.hpp:63-128, forward.cpp:109-131):
    state[j][m] += b*k_im*v_ij, then f_ij += sum_m q_im * state[j][m]."""
    q, k, v = (np.asarray(x, np.float64) for x in (q, k, v))
    G, N, D = q.shape
    f = np.array(f, np.float64, copy=True)
    for g in range(G):
        st = np.zeros((D, D))
        for i in range(N):
            st += np.outer(v[g, i], b * k[g, i])
            f[g, i] += st @ q[g, i]
    return f


def alpha_term(q, v, wh, b):
    """grad_k_alpha_core at unit g (backward_kernels.hpp:61-91, backward.cpp:103-128):
    suffix alpha[r][j] += b*q_ir*wh_ij; dk_ir = sum_j alpha[r][j]*v_ij (assign)."""
    q, v, wh = (np.asarray(x, np.float64) for x in (q, v, wh))
    G, N, D = q.shape
    dk = np.zeros((G, N, D))
    for g in range(G):
        al = np.zeros((D, D))
        for i in range(N - 1, -1, -1):
            al += np.outer(b * q[g, i], wh[g, i])
            dk[g, i] = al @ v[g, i]
    return dk


def beta_term(q, o, wh, b, dk):
    """grad_k_beta_core at unit g (backward_kernels.hpp:95-130, backward.cpp:130-153):
    suffix beta[r][j] += b*q_ir*o_ij*wh_ij; dk_ir -= sum_j beta[r][j]."""
    q, o, wh = (np.asarray(x, np.float64) for x in (q, o, wh))
    G, N, D = q.shape
    dk = np.array(dk, np.float64, copy=True)
    for g in range(G):
        be = np.zeros((D, D))
        for i in range(N - 1, -1, -1):
            be += np.outer(b * q[g, i], o[g, i] * wh[g, i])
            dk[g, i] -= be.sum(axis=1)
    return dk


def ref_term_pass(kind, x, y, z, a, b, acc, lx=SEQUENCE_MAJOR, ly=FEATURE_MAJOR, lz=FEATURE_MAJOR, L=0):
    """The reference's own term pass (kind 0 constant, 1 linear, 2 alpha, 3 beta) on a
    logical f64 accumulator; returns the logical result."""
    G, N, D = x.shape
    fl = [to_flat(np.asarray(t if t is not None else x, np.float64), l) for t, l in ((x, lx), (y, ly), (z, lz))]
    accf = np.array(to_flat(np.asarray(acc, np.float64), FEATURE_MAJOR), copy=True)  # never alias the caller
    st = ref_lib().ref_term_pass(C.c_int(kind), _p(fl[0]), lx, _p(fl[1]), ly, _p(fl[2]), lz, C.c_int64(G),
                                 C.c_int64(N), C.c_int64(D), C.c_double(a), C.c_double(b), C.c_int64(L), _p(accf))
    if st:
        raise RuntimeError(f"reference term pass failed with status {st}")
    return from_flat(accf, G, N, D, FEATURE_MAJOR).copy()


def ref_omega_hat(omega, g, lw=FEATURE_MAJOR):
    G, N, D = omega.shape
    wf = to_flat(np.asarray(omega, np.float64), lw)
    gf = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    out = np.zeros(G * N * D)
    st = ref_lib().ref_make_omega_hat(_p(wf), lw, _p(gf), C.c_int64(G), C.c_int64(N), C.c_int64(D), _p(out))
    if st:
        raise RuntimeError(f"reference make_omega_hat failed with status {st}")
    return from_flat(out, G, N, D, FEATURE_MAJOR).copy()


def ref_normalize_qk(q, k, lq=SEQUENCE_MAJOR, lk=SEQUENCE_MAJOR):
    G, N, D = q.shape
    qf, kf = to_flat(np.asarray(q, np.float64), lq), to_flat(np.asarray(k, np.float64), lk)
    qo, ko = np.zeros(G * N * D), np.zeros(G * N * D)
    st = ref_lib().ref_normalize_qk(_p(qf), lq, _p(kf), lk, C.c_int64(G), C.c_int64(N), C.c_int64(D),
                                    _p(qo), _p(ko))
    if st:
        raise RuntimeError(f"reference normalize_qk failed with status {st}")
    return from_flat(qo, G, N, D, lq).copy(), from_flat(ko, G, N, D, lk).copy()


def ref_prefix_advance(k_rows, v_rows, a, b):
    """make_prefix_state + prefix_advance over the rows; returns (x1, x2, y1, y2)."""
    k_rows, v_rows = np.ascontiguousarray(k_rows, np.float64), np.ascontiguousarray(v_rows, np.float64)
    R, D = k_rows.shape
    st_ = np.zeros(D + D * D + 1 + D)
    st = ref_lib().ref_prefix_advance(_p(k_rows), _p(v_rows), C.c_int64(R), C.c_int64(D), C.c_double(a),
                                      C.c_double(b), _p(st_))
    if st:
        raise RuntimeError(f"reference prefix_advance failed with status {st}")
    return st_[:D], st_[D:D + D * D].reshape(D, D), st_[D + D * D], st_[D + D * D + 1:]
