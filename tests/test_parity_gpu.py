"""GPU parity: the CUDA library (through the reference-mirroring API over the
C-ABI) against the CPU oracle on identical inputs.

Tolerances (BASELINE.json north_star): fp32 <= 1e-5 relative (max|x-y|/max|y|)
against the f64 oracle on the fp32 inputs; bf16 <= 2e-2 max-abs against the f64
oracle on the bf16-rounded inputs."""
import numpy as np
import pytest

import paper_2510_21956_b200 as la
from oracle import oracle as O
from tests._util import FM, SM, bench_inputs, fast_inputs, max_abs, rel_err, round_to

pytestmark = pytest.mark.gpu

FP32_REL = 1e-5
BF16_ABS = 2e-2


def dev(x, dtype, layout, cuda):
    t, r = round_to(x, dtype)
    return la.HeadTensor.from_logical(t.to(cuda), la.Layout(layout)), r


def run_dev(q, k, v, w, dtype, cuda, causal=True, a=1.0, b=1.0, impl="auto", fault=la.Fault.None_,
            lq=SM, lk=SM, lv=FM, lw=FM, impl_bwd=None):
    qt, qr = dev(q, dtype, lq, cuda)
    kt, kr = dev(k, dtype, lk, cuda)
    vt, vr = dev(v, dtype, lv, cuda)
    c = la.LinearKernelCoeffs(a, b)
    fwd = la.forward_causal if causal else la.forward_full
    bwd = la.backward_causal if causal else la.backward_full
    art = fwd(qt, kt, vt, c, None, fault, impl=impl)
    res = {"out": art.out.logical(), "g": art.g.cpu().numpy().reshape(q.shape[0], q.shape[1]),
           "rounded": (qr, kr, vr)}
    if w is not None:
        wt, wr = dev(w, dtype, lw, cuda)
        gr = bwd(art, wt, c, None, fault, impl=impl_bwd or impl)
        res.update(dq=gr.dq.logical(), dk=gr.dk.logical(), dv=gr.dv.logical(), w=wr)
    return res


def oracle_all(res, causal, a=1.0, b=1.0, fault=0, dtype=np.float64):
    qr, kr, vr = res["rounded"]
    out, g = O.forward(qr, kr, vr, a, b, causal=causal, fault=fault, dtype=dtype)
    ref = {"out": out, "g": g}
    if "w" in res:
        # the backward consumes the device forward's o and g, as the reference's
        # backward consumes its own ForwardArtifacts
        dq, dk, dv = O.backward(qr, kr, vr, res["out"], res["w"], res["g"], a, b, causal=causal,
                                fault=fault, dtype=dtype)
        ref.update(dq=dq, dk=dk, dv=dv)
    return ref


@pytest.mark.parametrize("causal", [True, False])
def test_config1_fp32_parity(cuda, causal):
    # BASELINE config 1: fp32 B=1 H=4 N=2048 D=64 a=b=1, reference inputs (bench.cpp:75-97)
    q, k, v, w = bench_inputs(4, 2048, 64)
    res = run_dev(q, k, v, w, "f32", cuda, causal=causal)
    ref = oracle_all(res, causal)
    for key in ("out", "g", "dq", "dk", "dv"):
        assert rel_err(res[key], ref[key]) <= FP32_REL, key


def test_seed3_forward_goldens_on_gpu(cuda):
    q = O.seeded(1, 3, 2, 3, SM)
    k = O.seeded(1, 3, 2, 4, SM)
    v = O.seeded(1, 3, 2, 5, FM)
    res = run_dev(q, k, v, None, "f32", cuda)
    golden_o = np.array([[0.34612980794285586, -0.92301077838464207],
                         [-0.13319984306864124, -0.24065510636744042],
                         [-0.37239006181521767, -0.43676585673830626]])
    golden_g = np.array([1.1233087720476638, 2.4344381472035654, 3.6168703758830461])
    assert rel_err(res["out"][0], golden_o) <= FP32_REL
    assert rel_err(res["g"][0], golden_g) <= FP32_REL


def test_seed11_backward_goldens_on_gpu(cuda):
    q = O.seeded(1, 4, 3, 11, SM)
    k = O.seeded(1, 4, 3, 12, SM)
    v = O.seeded(1, 4, 3, 13, FM)
    w = O.seeded(1, 4, 3, 14, FM)
    res = run_dev(q, k, v, w, "f32", cuda)
    gq = np.array([[0.0, 0.0, 0.0], [0.2610970160077386, 0.2013241874321281, 0.21024364305066712],
                   [-0.13182186642257676, -0.28236676963278029, 0.22961200862869902],
                   [-0.091971119497991083, 0.080342248132136973, 0.12996088871730649]])
    gv = np.array([[0.42000940503328366, -0.78945868081659043, -0.31639909331415694],
                   [0.36274863224328158, -0.25156616106913887, 0.41217273516469533],
                   [0.1195796959230222, -0.029249696442690265, 0.066468620774084997],
                   [0.00075433592705564934, -0.0089216108389855719, -0.0039506778404252429]])
    assert max_abs(res["dq"][0], gq) <= 1e-5
    assert max_abs(res["dv"][0], gv) <= 1e-5


def test_randomized_shapes_fp32_mixed_layouts(cuda):
    # test_forward.cpp:284-317: random N, D, both masks, coefficient table, mixed layouts
    rng = np.random.default_rng(777)
    table = [(1.0, 1.0), (1.0, 0.5), (0.3, 1.0)]
    for case in range(24):
        N, D = int(rng.integers(1, 200)), int(rng.integers(1, 40))
        G = int(rng.integers(1, 3))
        causal = bool(case % 2)
        a, b = table[case % 3]
        q = O.normalize_rows(O.seeded(G, N, D, int(rng.integers(1 << 40)), SM))
        k = O.normalize_rows(O.seeded(G, N, D, int(rng.integers(1 << 40)), FM))
        v = O.seeded(G, N, D, int(rng.integers(1 << 40)), FM)
        w = O.seeded(G, N, D, int(rng.integers(1 << 40)), SM)
        try:
            _, qg = O.quadratic(q, k, v, a, b, causal=causal)
        except O.OracleDegenerate:
            continue
        if np.min(np.abs(qg)) < 0.25:
            continue
        res = run_dev(q, k, v, w, "f32", cuda, causal=causal, a=a, b=b, lk=FM, lw=SM)
        ref = oracle_all(res, causal, a, b)
        for key in ("out", "g", "dq", "dk", "dv"):
            assert rel_err(res[key], ref[key]) <= FP32_REL, (case, key, N, D)


@pytest.mark.parametrize("fault", [1, 2, 3])
def test_fault_variants_match_oracle(cuda, fault):
    # Fault mutations are honoured on the device (fault.hpp:7-15, acceptance.cpp:195-217)
    q, k, v, w = bench_inputs(2, 96, 16, seed=5)
    res = run_dev(q, k, v, w, "f32", cuda, fault=la.Fault(fault))
    ref = oracle_all(res, True, fault=fault)
    clean = oracle_all(run_dev(q, k, v, w, "f32", cuda), True)
    for key in ("out", "dq", "dk", "dv"):
        assert rel_err(res[key], ref[key]) <= FP32_REL, key
    changed = {1: "dk", 2: "out", 3: "dv"}[fault]
    assert max_abs(res[changed], clean[changed]) > 1e-3


def test_degenerate_denominator_reported(cuda):
    import torch
    q = np.array([[[1.0, 0.0], [-1.0, 0.0]]])
    k = np.array([[[1.0, 0.0], [1.0, 0.0]]])
    v = O.seeded(1, 2, 2, 88, FM)
    with pytest.raises(la.DegenerateDenominator) as e:
        run_dev(q, k, v, None, "f32", cuda)
    assert (e.value.group(), e.value.position()) == (0, 1)
    # lexicographically first offender across groups (pool.hpp:36-42)
    q2 = np.concatenate([np.array([[[1.0, 0.0], [1.0, 0.0], [1.0, 0.0]]]),
                         np.array([[[1.0, 0.0], [-1.0, 0.0], [-1.0, 0.0]]])])
    k2 = np.ones((2, 3, 2)) * np.array([1.0, 0.0])
    v2 = O.seeded(2, 3, 2, 89, FM)
    with pytest.raises(la.DegenerateDenominator) as e:
        run_dev(q2, k2, v2, None, "f32", cuda)
    assert (e.value.group(), e.value.position()) == (1, 1)
    torch.cuda.synchronize()


def test_host_buffer_api_matches_device_api(cuda):
    q, k, v, w = bench_inputs(2, 300, 32, seed=9)
    c = la.LinearKernelCoeffs()
    hq = la.HeadTensor.from_logical(q, la.Layout.SequenceMajor)
    hk = la.HeadTensor.from_logical(k, la.Layout.SequenceMajor)
    hv = la.HeadTensor.from_logical(v, la.Layout.FeatureMajor)
    hw = la.HeadTensor.from_logical(w, la.Layout.FeatureMajor)
    art = la.forward_causal(hq, hk, hv, c, dtype="f32")
    gr = la.backward_causal(art, hw, c, dtype="f32")
    res = run_dev(q, k, v, w, "f32", cuda)
    assert np.array_equal(art.out.logical(), res["out"])
    assert np.array_equal(gr.dk.logical(), res["dk"])


@pytest.mark.parametrize("impl", ["simt", "auto"])
def test_bf16_causal_d128_parity(cuda, impl):
    # north-star dtype/head-dim at a size the f64 oracle finishes in seconds
    q, k, v, w = fast_inputs(2, 4096, 128, seed=1)
    res = run_dev(q, k, v, w, "bf16", cuda, impl=impl)
    ref = oracle_all(res, True)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("D", [32, 64, 96, 128, 192, 256])
def test_bf16_noncausal_head_dim_sweep(cuda, D):
    # BASELINE config 4 shape family (non-causal, D sweep) at reduced N; D = 64 / 192 / 256
    # run la_full.cu, D = 128 the la_sm100 kernels, D = 32 / 96 those on a zero-padded copy
    q, k, v, w = fast_inputs(2, 2048, D, seed=D)
    res = run_dev(q, k, v, w, "bf16", cuda, causal=False)
    ref = oracle_all(res, False)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, (D, key)
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("ctas", [5, 3])
def test_noncausal_d64_paired_chunks_odd_segments(cuda, ctas):
    """D = 64 applies chunks in pairs (block-diagonal W, la_full.cu apply_pairs): segments of
    7 and 4 chunks (ctas = 5) or 11 and 10 (ctas = 3) cover odd tails and several pairs."""
    from paper_2510_21956_b200 import _abi
    q, k, v, w = fast_inputs(2, 2048, 64, seed=11 + ctas)
    _abi.set_tuning(full_ctas_fwd=ctas)
    try:
        res = run_dev(q, k, v, w, "bf16", cuda, causal=False)
    finally:
        _abi.set_tuning()
    ref = oracle_all(res, False)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("D,a,b", [(256, 1.0, 1.0), (64, 0.5, 2.0), (192, 2.0, 0.25)])
def test_noncausal_full_tc_path_runs_and_matches(cuda, D, a, b):
    """Non-causal D = 64 / 192 / 256 runs the tcgen05 kernels of la_full.cu (profile scopes:
    totals, forward apply, dQ / dK / dV applies), fp16 here, unequal coefficients."""
    from paper_2510_21956_b200 import _abi
    q, k, v, w = fast_inputs(3, 1024, D, seed=D + 1)
    L = _abi.lib()
    L.la_profile_enable(1)
    _abi.profile_read()
    res = run_dev(q, k, v, w, "f16", cuda, causal=False, a=a, b=b)
    names = {r["name"] for r in _abi.profile_read()}
    L.la_profile_enable(0)
    assert {"la_fwd_full_kv", "la_bwd_full_r", "la_fwd_full_apply", "la_bwd_full_dq", "la_bwd_full_dk",
            "la_bwd_full_dv"} <= names, names
    ref = oracle_all(res, False, a=a, b=b)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, (D, key)


def test_north_star_sampled_groups_full_n(cuda):
    # BASELINE config 2 at full N=65536, D=128, bf16: two groups checked against
    # the oracle (groups are independent, forward_kernels.hpp:221-235)
    q, k, v, w = fast_inputs(2, 65536, 128, seed=3)
    res = run_dev(q, k, v, w, "bf16", cuda)
    ref = oracle_all(res, True, dtype=np.float32)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key


def test_bitwise_deterministic(cuda):
    q, k, v, w = fast_inputs(3, 1000, 128, seed=4)
    r1 = run_dev(q, k, v, w, "bf16", cuda)
    r2 = run_dev(q, k, v, w, "bf16", cuda)
    for key in ("out", "g", "dq", "dk", "dv"):
        assert np.array_equal(r1[key], r2[key]), key


def test_prefix_extensional(cuda):
    # test_forward.cpp:256-282: rows of a causal run on a prefix match the full run
    q, k, v, w = fast_inputs(2, 2048, 128, seed=6)
    full = run_dev(q, k, v, None, "f32", cuda)
    pre = run_dev(q[:, :700], k[:, :700], v[:, :700], None, "f32", cuda)
    assert rel_err(pre["out"], full["out"][:, :700]) <= FP32_REL
    assert rel_err(pre["g"], full["g"][:, :700]) <= FP32_REL


def test_backward_linear_in_cotangent(cuda):
    # test_backward.cpp:230-261 as a size-independent property
    q, k, v, w1 = fast_inputs(2, 4096, 64, seed=8)
    w2 = np.random.default_rng(9).uniform(-1, 1, w1.shape)
    r1 = run_dev(q, k, v, w1, "f32", cuda)
    r2 = run_dev(q, k, v, w2, "f32", cuda)
    rs = run_dev(q, k, v, w1 + w2, "f32", cuda)
    for key in ("dq", "dk", "dv"):
        assert rel_err(r1[key] + r2[key], rs[key]) <= 1e-5, key


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("N", [128, 4096])
def test_tcgen05_forward_parity(cuda, dtype, N):
    # the sm_100a chunked forward (forced), multi-segment carries at N=4096
    q, k, v, _ = fast_inputs(3, N, 128, seed=N + len(dtype))
    res = run_dev(q, k, v, None, dtype, cuda, impl="tcgen05")
    ref = oracle_all(res, True)
    assert max_abs(res["out"], ref["out"]) <= BF16_ABS
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("N", [128, 1024, 8192])
def test_tcgen05_backward_parity(cuda, dtype, N):
    # the sm_100a fused reverse-sweep backward (forced), multi-segment carries at N>=1024
    q, k, v, w = fast_inputs(2, N, 128, seed=N + 7 * len(dtype))
    res = run_dev(q, k, v, w, dtype, cuda, impl="tcgen05")
    ref = oracle_all(res, True)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key


def test_backward_with_saved_forward_state_matches_recompute(cuda):
    # la_backward_saved (prefix states from the forward) vs la_backward (recomputed)
    import torch
    q, k, v, w = fast_inputs(4, 8192, 128, seed=21)
    res = run_dev(q, k, v, w, "bf16", cuda)          # API uses the saved-state path
    ref = oracle_all(res, True)
    qt, _ = dev(q, "bf16", SM, cuda)
    kt, _ = dev(k, "bf16", SM, cuda)
    vt, _ = dev(v, "bf16", FM, cuda)
    wt, _ = dev(w, "bf16", FM, cuda)
    art = la.forward_causal(qt, kt, vt)
    art.saved = None                                  # force the recompute path
    gr = la.backward_causal(art, wt)
    for key, t in (("dq", gr.dq), ("dk", gr.dk), ("dv", gr.dv)):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
        assert max_abs(t.logical(), res[key]) <= 1e-2, key
    torch.cuda.synchronize()


# (bf16, 69, 8192): blocks of 5 groups (P = 29 segments each) and a ragged last block of
# 4 (P = 37): the last block needs more saved-state / workspace bytes than a full one
@pytest.mark.parametrize("dtype,G,N,D", [("bf16", 10, 1024, 128), ("f32", 3, 300, 64), ("bf16", 69, 8192, 128)])
def test_host_step_pipeline_matches_oracle(cuda, dtype, G, N, D):
    # la_host_step: forward + backward over host buffers, groups pipelined in blocks
    # (ragged last block at G=10) through the H2D / compute / D2H streams
    import ctypes as C

    import torch
    from paper_2510_21956_b200 import _abi
    q, k, v, w = fast_inputs(G, N, D, seed=G + N)
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    hq = torch.as_tensor(q).to(tdt).contiguous().pin_memory()                     # SequenceMajor
    hk = torch.as_tensor(k).to(tdt).contiguous().pin_memory()
    hv = torch.as_tensor(v).to(tdt).transpose(1, 2).contiguous().pin_memory()     # FeatureMajor
    hw = torch.as_tensor(w).to(tdt).transpose(1, 2).contiguous().pin_memory()
    hout = torch.empty((G, D, N), dtype=tdt).pin_memory()
    hg = torch.empty((G, N), dtype=torch.float32).pin_memory()
    hdq = torch.empty((G, N, D), dtype=tdt).pin_memory()
    hdk = torch.empty((G, D, N), dtype=tdt).pin_memory()
    hdv = torch.empty((G, D, N), dtype=tdt).pin_memory()
    L = _abi.lib()
    p = _abi.make_problem(G, N, D, dtype)
    err = _abi.ErrorInfo()
    st = L.la_host_step(C.byref(p), hq.data_ptr(), SM, hk.data_ptr(), SM, hv.data_ptr(), FM, hw.data_ptr(), FM,
                        hout.data_ptr(), hg.data_ptr(), hdq.data_ptr(), hdk.data_ptr(), hdv.data_ptr(),
                        C.byref(err))
    assert st == 0, err.message
    rq, rk = hq.double().numpy(), hk.double().numpy()
    rv, rw = hv.double().transpose(1, 2).numpy(), hw.double().transpose(1, 2).numpy()
    out = hout.double().transpose(1, 2).numpy()
    g = hg.double().numpy()
    ro, rg = O.forward(rq, rk, rv)
    dq, dk, dv = O.backward(rq, rk, rv, out, rw, g)
    got = {"out": out, "dq": hdq.double().numpy(), "dk": hdk.double().transpose(1, 2).numpy(),
           "dv": hdv.double().transpose(1, 2).numpy()}
    ref = {"out": ro, "dq": dq, "dk": dk, "dv": dv}
    for key in got:
        if dtype == "f32":
            assert rel_err(got[key], ref[key]) <= FP32_REL, key
        else:
            assert max_abs(got[key], ref[key]) <= BF16_ABS, key
    assert rel_err(g, rg) <= (1e-5 if dtype == "f32" else 1e-3)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("N", [128, 4096])
def test_tcgen05_noncausal_forward_parity(cuda, dtype, N):
    # the sm_100a non-causal forward (forced): aggregate totals + apply pass
    q, k, v, _ = fast_inputs(3, N, 128, seed=N + 3 * len(dtype))
    res = run_dev(q, k, v, None, dtype, cuda, causal=False, impl="tcgen05")
    ref = oracle_all(res, False)
    assert max_abs(res["out"], ref["out"]) <= BF16_ABS
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("N", [128, 4096])
def test_tcgen05_noncausal_backward_parity(cuda, dtype, N):
    # the sm_100a non-causal backward (forced): totals + independent chunk pass
    q, k, v, w = fast_inputs(2, N, 128, seed=N + 5 * len(dtype))
    res = run_dev(q, k, v, w, dtype, cuda, causal=False, impl="tcgen05")
    ref = oracle_all(res, False)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("D", [32, 64, 96])
def test_bf16_small_head_dim_padded_tcgen05(cuda, causal, D):
    # D < 128 runs the tensor-core kernels on a zero-padded copy (exact algebra: padded
    # key features add nothing to S or z, padded value features are dropped)
    q, k, v, w = fast_inputs(2, 2048, D, seed=D + causal)
    res = run_dev(q, k, v, w, "bf16", cuda, causal=causal)
    ref = oracle_all(res, causal)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, (D, key)
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("causal,D", [(True, 128), (False, 128), (False, 64), (False, 256)])
def test_f16_key_sum_beyond_half_range(cuda, causal, D):
    # every key is e_0, so z_0 = N = 131072 > 65504 (the fp16 maximum): the q.z term
    # must not overflow on the fp16 tensor-core paths (la_sm100 D = 128, la_full D = 64 / 256)
    G, N = 1, 131072
    rng = np.random.default_rng(11)
    q = O.normalize_rows(rng.uniform(-1, 1, (G, N, D)))
    k = np.zeros((G, N, D))
    k[..., 0] = 1.0
    v = rng.uniform(-1, 1, (G, N, D))
    w = rng.uniform(-1, 1, (G, N, D))
    res = run_dev(q, k, v, w, "f16", cuda, causal=causal)
    ref = oracle_all(res, causal, dtype=np.float32)
    for key in ("out", "g", "dq", "dk", "dv"):
        assert np.isfinite(res[key]).all(), key
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("G,N", [(3, 4096), (5, 1280), (64, 2048), (200, 256)])
def test_segment_partition_matches_oracle(cuda, G, N):
    """Segment counts from 1 (G = 200 >= 148 SMs) to many (G = 3): carries across
    segment boundaries, bf16 fwd+bwd against the oracle on sampled groups."""
    import torch
    q, k, v, w = fast_inputs(G, N, 128, seed=G + N)
    t = [torch.as_tensor(x).to(torch.bfloat16) for x in (q, k, v, w)]
    L = la.Layout
    hq = la.HeadTensor.from_logical(t[0].to(cuda), L.SequenceMajor)
    hk = la.HeadTensor.from_logical(t[1].to(cuda), L.SequenceMajor)
    hv = la.HeadTensor.from_logical(t[2].to(cuda), L.FeatureMajor)
    hw = la.HeadTensor.from_logical(t[3].to(cuda), L.FeatureMajor)
    art = la.forward_causal(hq, hk, hv)
    gr = la.backward_causal(art, hw)
    torch.cuda.synchronize()
    o_dev = art.out.logical()
    g_dev = art.g.cpu().numpy().reshape(G, N)
    dq_d, dk_d, dv_d = gr.dq.logical(), gr.dk.logical(), gr.dv.logical()
    for gi in sorted({0, G // 2, G - 1}):
        rq, rk, rv, rw = (x[gi:gi + 1].double().numpy() for x in t)
        out, g = O.forward(rq, rk, rv)
        assert max_abs(o_dev[gi:gi + 1], out) <= 2e-2
        dq, dk, dv = O.backward(rq, rk, rv, o_dev[gi:gi + 1], rw, g_dev[gi:gi + 1])
        for a_, b_ in ((dq_d, dq), (dk_d, dk), (dv_d, dv)):
            assert max_abs(a_[gi:gi + 1], b_) <= 2e-2


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("a,b", [(0.5, 2.0), (1.0, 0.0), (2.0, 0.25)])
def test_tcgen05_kernel_coefficients(cuda, causal, a, b):
    """f(x) = a + b x with b = 0 (pure prefix / full averaging) and unequal a, b on the
    tensor-core kernels, forward and backward."""
    q, k, v, w = fast_inputs(2, 512, 128, seed=int(10 * a + 100 * b))
    res = run_dev(q, k, v, w, "bf16", cuda, causal=causal, a=a, b=b, impl="tcgen05")
    ref = oracle_all(res, causal, a=a, b=b)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("N,D", [(1000, 128), (130, 128), (4095, 64), (777, 256)])
def test_unaligned_sequence_length_on_fast_path(cuda, causal, N, D):
    """N not a multiple of 128: rows zero-padded in device scratch, tensor-core / GEMM
    kernels (not the CUDA-core sweep), results against the oracle."""
    from paper_2510_21956_b200 import _abi
    q, k, v, w = fast_inputs(2, N, D, seed=N + D)
    L = _abi.lib()
    L.la_profile_enable(1)
    _abi.profile_read()
    res = run_dev(q, k, v, w, "bf16", cuda, causal=causal)
    names = {r["name"] for r in _abi.profile_read()}
    L.la_profile_enable(0)
    assert not any(n.startswith("k_fwd_rows") or n.startswith("k_bwd_rows") for n in names), names
    ref = oracle_all(res, causal)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("G,N", [(1, 128), (1, 64), (3, 1), (1, 129), (5, 192)])
def test_small_and_edge_shapes_bf16(cuda, causal, G, N):
    """Single chunks, one row, one group, N just past a chunk boundary: whatever path
    takes them (tensor core, padded, CUDA cores) matches the oracle."""
    q, k, v, w = fast_inputs(G, N, 128, seed=G * 1000 + N)
    res = run_dev(q, k, v, w, "bf16", cuda, causal=causal)
    ref = oracle_all(res, causal)
    for key in ("out", "dq", "dk", "dv"):
        assert max_abs(res[key], ref[key]) <= BF16_ABS, key
    assert rel_err(res["g"], ref["g"]) <= 1e-3


def test_step_is_cuda_graph_capturable(cuda):
    """la_forward_save + la_backward_saved capture into a CUDA graph (no host syncs, no
    pageable copies on the path) and a replay reproduces the eager step bitwise."""
    import ctypes as C
    import torch
    from paper_2510_21956_b200 import _abi
    L = _abi.lib()
    G, N, D = 4, 2048, 128
    q, k, v, w = fast_inputs(G, N, D, seed=5)
    tq, tk = (torch.as_tensor(x).to(torch.bfloat16).to(cuda).contiguous() for x in (q, k))
    tv, tw = (torch.as_tensor(x.transpose(0, 2, 1)).to(torch.bfloat16).to(cuda).contiguous() for x in (v, w))
    p = _abi.make_problem(G, N, D, "bf16")
    out = torch.empty((G, D, N), device=cuda, dtype=torch.bfloat16)
    g = torch.empty((G, N), device=cuda, dtype=torch.float32)
    dq, dk, dv = torch.empty_like(tq), torch.empty_like(tv), torch.empty_like(tv)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)

    def step():
        s = torch.cuda.current_stream().cuda_stream
        assert L.la_forward_save(C.byref(p), tq.data_ptr(), 1, tk.data_ptr(), 1, tv.data_ptr(), 0, out.data_ptr(),
                                 g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), s, None) == 0
        assert L.la_backward_saved(C.byref(p), tq.data_ptr(), 1, tk.data_ptr(), 1, tv.data_ptr(), 0,
                                   out.data_ptr(), tw.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(),
                                   dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), s,
                                   None) == 0

    step()
    torch.cuda.synchronize()
    ref = [x.clone() for x in (out, g, dq, dk, dv)]
    for x in (out, g, dq, dk, dv):
        x.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    graph.replay()
    torch.cuda.synchronize()
    for a_, b_ in zip((out, g, dq, dk, dv), ref):
        assert torch.equal(a_, b_)


def test_saved_state_mismatch_reported(cuda):
    """la_backward_saved validates the saved-state header on the device (no host read):
    a buffer that does not come from la_forward_save of this problem is reported as
    MissingForwardState (backward.cpp:15-20's error class), synchronously with err."""
    import ctypes as C
    import torch
    from paper_2510_21956_b200 import _abi
    L = _abi.lib()
    G, N, D = 2, 2048, 128
    q, k, v, w = fast_inputs(G, N, D, seed=12)
    tq, tk = (torch.as_tensor(x).to(torch.bfloat16).to(cuda).contiguous() for x in (q, k))
    tv, tw = (torch.as_tensor(x.transpose(0, 2, 1)).to(torch.bfloat16).to(cuda).contiguous() for x in (v, w))
    p = _abi.make_problem(G, N, D, "bf16")
    p2 = _abi.make_problem(G, N // 2, D, "bf16")
    out = torch.empty((G, D, N), device=cuda, dtype=torch.bfloat16)
    g = torch.empty((G, N), device=cuda, dtype=torch.float32)
    dq, dk, dv = torch.empty_like(tq), torch.empty_like(tv), torch.empty_like(tv)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    s = torch.cuda.current_stream().cuda_stream
    err = _abi.ErrorInfo()

    def bwd():
        return L.la_backward_saved(C.byref(p), tq.data_ptr(), 1, tk.data_ptr(), 1, tv.data_ptr(), 0, out.data_ptr(),
                                   tw.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(),
                                   dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), s, C.byref(err))

    assert L.la_forward_save(C.byref(p), tq.data_ptr(), 1, tk.data_ptr(), 1, tv.data_ptr(), 0, out.data_ptr(),
                             g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), s, C.byref(err)) == 0
    assert bwd() == 0
    sv.zero_()                                          # not a saved state
    assert bwd() == 5 and b"la_forward_save" in err.message
    # states of another problem (half the rows) in a large-enough buffer
    assert L.la_forward_save(C.byref(p2), tq.data_ptr(), 1, tk.data_ptr(), 1, tv.data_ptr(), 0, out.data_ptr(),
                             g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), s, C.byref(err)) == 0
    assert bwd() == 5
