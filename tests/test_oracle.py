"""The CPU oracle (oracle/oracle.c) pinned against the reference's own goldens
and, when oracle/_ref/libla_ref.so is present, against the reference library
itself (compiled from /root/reference sources by oracle/Makefile)."""
import numpy as np
import pytest

from oracle import oracle as O

FM, SM = O.FEATURE_MAJOR, O.SEQUENCE_MAJOR


def test_seed3_forward_goldens():
    # tests/test_forward.cpp:115-134 (== test_reference.cpp:119-140)
    q = O.seeded(1, 3, 2, 3, SM)
    k = O.seeded(1, 3, 2, 4, SM)
    v = O.seeded(1, 3, 2, 5, FM)
    out, g = O.forward(q, k, v, 1.0, 1.0, causal=True)
    golden_o = np.array([[0.34612980794285586, -0.92301077838464207],
                         [-0.13319984306864124, -0.24065510636744042],
                         [-0.37239006181521767, -0.43676585673830626]])
    golden_g = np.array([1.1233087720476638, 2.4344381472035654, 3.6168703758830461])
    assert np.max(np.abs(g[0] - golden_g)) <= 1e-12
    assert np.max(np.abs(out[0] - golden_o)) <= 1e-12


def test_seed11_backward_fd_goldens():
    # tests/test_backward.cpp:74-113: analytic backward vs frozen FD goldens
    q = O.seeded(1, 4, 3, 11, SM)
    k = O.seeded(1, 4, 3, 12, SM)
    v = O.seeded(1, 4, 3, 13, FM)
    w = O.seeded(1, 4, 3, 14, FM)
    out, g = O.forward(q, k, v)
    dq, dk, dv = O.backward(q, k, v, out, w, g)
    gq = np.array([[0.0, 0.0, 0.0], [0.2610970160077386, 0.2013241874321281, 0.21024364305066712],
                   [-0.13182186642257676, -0.28236676963278029, 0.22961200862869902],
                   [-0.091971119497991083, 0.080342248132136973, 0.12996088871730649]])
    gk = np.array([[-0.14090294364610401, 0.16918765327611496, 0.095115568587988975],
                   [0.12103498014948144, -0.38476471603265949, -0.20953733026463084],
                   [0.2273959877618914, 0.13656927555505405, 0.059613165848126926],
                   [0.16058720514466884, -0.098595440367610365, -0.17331046453517018]])
    gv = np.array([[0.42000940503328366, -0.78945868081659043, -0.31639909331415694],
                   [0.36274863224328158, -0.25156616106913887, 0.41217273516469533],
                   [0.1195796959230222, -0.029249696442690265, 0.066468620774084997],
                   [0.00075433592705564934, -0.0089216108389855719, -0.0039506778404252429]])
    for got, gold in ((dq[0], gq), (dk[0], gk), (dv[0], gv)):
        assert np.all(np.abs(got - gold) <= 1e-7 + 1e-5 * np.abs(gold))


def test_single_token_and_zero_query_known_answers():
    # test_forward.cpp:86-113
    q = O.seeded(1, 1, 3, 61, SM)
    k = O.seeded(1, 1, 3, 62, SM)
    v = O.seeded(1, 1, 3, 63, FM)
    out, g = O.forward(q, k, v)
    assert np.max(np.abs(out - v)) <= 1e-15
    assert abs(g[0, 0] - (1.0 + float(q[0, 0] @ k[0, 0]))) <= 1e-14
    q0 = np.zeros((1, 7, 3))
    k = O.seeded(1, 7, 3, 64, SM)
    v = O.seeded(1, 7, 3, 65, FM)
    out, g = O.forward(q0, k, v, 1.0, 0.7)
    assert np.allclose(g[0], np.arange(1, 8), rtol=1e-13)
    means = np.cumsum(v[0], axis=0) / np.arange(1, 8)[:, None]
    assert np.allclose(out[0], means, rtol=1e-12)


def test_degenerate_position_reported():
    # test_forward.cpp:334-348
    q = np.array([[[1.0, 0.0], [-1.0, 0.0]]])
    k = np.array([[[1.0, 0.0], [1.0, 0.0]]])
    v = O.seeded(1, 2, 2, 88, FM)
    with pytest.raises(O.OracleDegenerate) as e:
        O.forward(q, k, v)
    assert (e.value.group, e.value.position) == (0, 1)


@pytest.mark.parametrize("causal", [True, False])
def test_fast_matches_quadratic(causal):
    rng = np.random.default_rng(7)
    for _ in range(10):
        G, N, D = 2, int(rng.integers(1, 30)), int(rng.integers(1, 12))
        q = O.normalize_rows(O.seeded(G, N, D, int(rng.integers(1 << 30)), SM))
        k = O.normalize_rows(O.seeded(G, N, D, int(rng.integers(1 << 30)), SM))
        v = O.seeded(G, N, D, int(rng.integers(1 << 30)), FM)
        out, g = O.forward(q, k, v, 1.0, 0.5, causal=causal)
        qo, qg = O.quadratic(q, k, v, 1.0, 0.5, causal=causal)
        assert np.max(np.abs(out - qo)) <= 1e-10
        assert np.max(np.abs(g - qg)) <= 1e-10


def test_faults_change_results():
    q = O.normalize_rows(O.seeded(1, 8, 4, 1, SM))
    k = O.normalize_rows(O.seeded(1, 8, 4, 2, SM))
    v = O.seeded(1, 8, 4, 3, FM)
    w = O.seeded(1, 8, 4, 4, FM)
    out, g = O.forward(q, k, v)
    bad, _ = O.forward(q, k, v, fault=2)
    assert np.max(np.abs(bad - out)) > 1e-3
    base = O.backward(q, k, v, out, w, g)
    flip = O.backward(q, k, v, out, w, g, fault=1)
    drop = O.backward(q, k, v, out, w, g, fault=3)
    assert np.max(np.abs(flip[1] - base[1])) > 1e-3 and np.array_equal(flip[2], base[2])
    assert np.max(np.abs(drop[2] - base[2])) > 1e-3 and np.array_equal(drop[1], base[1])


ref = pytest.mark.skipif(O.ref_lib() is None, reason="reference library not built/shipped")


@ref
def test_fill_matches_reference_make_tensor():
    for layout in (FM, SM):
        assert np.array_equal(O.ref_seeded(2, 5, 3, 1234, layout), O.seeded(2, 5, 3, 1234, layout))


@ref
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("fault", [0, 1, 2, 3])
def test_restatement_bitwise_equals_reference_f64(causal, fault):
    G, N, D = 2, 37, 9
    q = O.normalize_rows(O.seeded(G, N, D, 11, SM))
    k = O.normalize_rows(O.seeded(G, N, D, 12, SM))
    v = O.seeded(G, N, D, 13, FM)
    w = O.seeded(G, N, D, 14, FM)
    out, g = O.forward(q, k, v, 0.7, 1.3, causal=causal, fault=fault)
    rout, rg = O.ref_forward(q, k, v, 0.7, 1.3, causal=causal, fault=fault, L=3, workers=3)
    assert np.array_equal(out, rout) and np.array_equal(g, rg)
    got = O.backward(q, k, v, out, w, g, 0.7, 1.3, causal=causal, fault=fault)
    exp = O.ref_backward(q, k, v, out, w, g, 0.7, 1.3, causal=causal, fault=fault, L=3, workers=2)
    for a_, b_ in zip(got, exp):
        assert np.array_equal(a_, b_)


@ref
def test_restatement_bitwise_equals_reference_f32_fast_path():
    G, N, D = 3, 64, 16
    q = O.normalize_rows(O.seeded(G, N, D, 1, SM)).astype(np.float32)
    k = O.normalize_rows(O.seeded(G, N, D, 2, SM)).astype(np.float32)
    v = O.seeded(G, N, D, 3, FM).astype(np.float32)
    w = O.seeded(G, N, D, 4, FM).astype(np.float32)
    flat = lambda x, l: O.to_flat(x, l)
    r = O.ref_fwd_bwd_f32(flat(q, SM).reshape(G, N, D), flat(k, SM).reshape(G, N, D),
                          flat(v, FM).reshape(G, N, D), flat(w, FM).reshape(G, N, D), workers=2)
    p = O.fwd_bwd_f32_threads(flat(q, SM).reshape(G, N, D), flat(k, SM).reshape(G, N, D),
                              flat(v, FM).reshape(G, N, D), flat(w, FM).reshape(G, N, D), threads=2)
    for a_, b_ in zip(r, p):
        assert np.array_equal(a_, b_)


@ref
def test_finite_difference_goldens_from_reference():
    q = O.seeded(1, 4, 3, 11, SM)
    k = O.seeded(1, 4, 3, 12, SM)
    v = O.seeded(1, 4, 3, 13, FM)
    w = O.seeded(1, 4, 3, 14, FM)
    fd = O.ref_finite_diff(q, k, v, w, h=1e-6)
    out, g = O.forward(q, k, v)
    an = O.backward(q, k, v, out, w, g)
    for a_, f_ in zip(an, fd):
        assert np.all(np.abs(a_ - f_) <= 1e-7 + 1e-5 * np.abs(f_))


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("N,D,a,b", [(1300, 24, 1.0, 1.0), (515, 16, 0.7, 1.3), (3, 2, 1.0, 1.0)])
def test_chunked_oracle_matches_restatement(causal, N, D, a, b):
    """oracle/chunked.py (BLAS-chunked f64, used for full-N parity) equals the loop-for-loop
    restatement, chunk tails included (CHUNK = 512), and its sequence-shard carries
    reproduce the unsharded result ('Sequence shards')."""
    from oracle import chunked as CH
    q = O.normalize_rows(O.seeded(1, N, D, 31, SM))
    k = O.normalize_rows(O.seeded(1, N, D, 32, SM))
    v = O.seeded(1, N, D, 33, FM)
    w = O.seeded(1, N, D, 34, FM)
    out, g = O.forward(q, k, v, a, b, causal=causal)
    dq, dk, dv = O.backward(q, k, v, out, w, g, a, b, causal=causal)
    co, cg = CH.forward(q[0], k[0], v[0], a, b, causal)
    assert np.max(np.abs(co - out[0])) <= 1e-11 and np.max(np.abs(cg - g[0])) <= 1e-10
    cq, ck, cv = CH.backward(q[0], k[0], v[0], out[0], w[0], g[0], a, b, causal)
    for x, y in ((cq, dq[0]), (ck, dk[0]), (cv, dv[0])):
        assert np.max(np.abs(x - y)) <= 1e-10 * max(1.0, np.max(np.abs(y)))
    if causal and N > 8:
        cut = N // 3
        pre = CH.shard_totals_forward(k[0, :cut], v[0, :cut])
        o2, g2 = CH.forward(q[0, cut:], k[0, cut:], v[0, cut:], a, b, True, prefix=pre, row0=cut)
        assert np.max(np.abs(o2 - out[0, cut:])) <= 1e-11
        suf = CH.shard_totals_backward(q[0, cut:], out[0, cut:], w[0, cut:], g[0, cut:])
        q1, k1, v1 = CH.backward(q[0, :cut], k[0, :cut], v[0, :cut], out[0, :cut], w[0, :cut], g[0, :cut],
                                 a, b, True, suffix=suf)
        for x, y in ((q1, dq[0, :cut]), (k1, dk[0, :cut]), (v1, dv[0, :cut])):
            assert np.max(np.abs(x - y)) <= 1e-10 * max(1.0, np.max(np.abs(y)))
