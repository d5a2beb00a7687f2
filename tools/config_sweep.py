"""Device time of one fwd+bwd for each BASELINE.json config on one GPU (CUDA events,
warm-up first, inputs resident in HBM), with the path that ran (tcgen05 or SIMT) and the
HBM-roofline fraction of the step's algorithmic bytes. Config 5 (N = 1M, sequence-sharded
over 8 GPUs) is measured as one rank's shard: 131072 rows with a carried-in prefix state.
Usage: python tools/config_sweep.py > gpurun_out/configs.jsonl"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_21956_b200 import _abi  # noqa: E402

L = _abi.lib()
dev = torch.device("cuda")
HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json"))).get("hbm_gbs", 6530.6)
TD = {"f32": torch.float32, "bf16": torch.bfloat16}


def run(name, B, H, N, D, dtype, causal, shard=False, reps=5):
    G = B * H
    p = _abi.make_problem(G, N, D, dtype, causal=causal)
    e = 4 if dtype == "f32" else 2
    td = TD[dtype]

    def unit(shape):
        x = torch.rand(shape, device=dev) * 2 - 1
        return (x / x.norm(dim=-1, keepdim=True)).to(td)
    q, k = unit((G, N, D)), unit((G, N, D))
    v = (torch.rand((G, D, N), device=dev) * 2 - 1).to(td)
    w = (torch.rand((G, D, N), device=dev) * 2 - 1).to(td)
    out = torch.empty((G, D, N), device=dev, dtype=td)
    g = torch.empty((G, N), device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(v), torch.empty_like(v)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    st = torch.cuda.current_stream().cuda_stream
    sh = None
    if shard:  # rank 7 of 8: carried-in prefix state of the 7 earlier shards (synthetic)
        nf = L.la_shard_state_floats(C.byref(p))
        carry = torch.rand(nf, device=dev) * 0.01
        sh = _abi.Shard()
        sh.row_offset = 7 * N
        sh.carry_in = carry.data_ptr()
        sh.carry_suffix = None

    def step():
        if shard:
            # as la_sharded_forward / _backward run it (la_dist.cu): the forward's states saved
            s1 = L.la_forward_sharded_save(C.byref(p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(),
                                           0, out.data_ptr(), g.data_ptr(), sv.data_ptr(), sv.numel(),
                                           wsf.data_ptr(), wsf.numel(), st, None)
            s2 = L.la_backward_sharded_saved(C.byref(p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1,
                                             v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(),
                                             sv.data_ptr(), sv.numel(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                             wsb.data_ptr(), wsb.numel(), st, None)
        else:
            s1 = L.la_forward_save(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(),
                                   g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), st, None)
            s2 = L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(),
                                     w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(),
                                     dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), st, None)
        assert s1 == 0 and s2 == 0, (s1, s2)
    for _ in range(3):
        step()
    L.la_profile_enable(1)
    _abi.profile_read()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for _ in range(reps):
        step()
    t1.record()
    torch.cuda.synchronize()
    L.la_profile_enable(0)
    kern = sorted({r["name"] for r in _abi.profile_read()})
    ms = t0.elapsed_time(t1) / reps
    alg = G * N * (12 * D * e + 8)  # fwd 4De+4 + bwd 8De+4 per row
    gbs = alg / (ms / 1e3) / 1e9
    print(json.dumps({"config": name, "B": B, "H": H, "N": N, "D": D, "dtype": dtype, "causal": causal,
                      "ms_fwd_bwd": round(ms, 4), "tokens_per_s": B * N / (ms / 1e3),
                      "alg_GB": round(alg / 1e9, 3), "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 3),
                      "kernels": kern}), flush=True)
    del q, k, v, w, out, g, dq, dk, dv, wsf, wsb, sv
    torch.cuda.empty_cache()


run("1: causal fp32 B1 H4 N2048 D64", 1, 4, 2048, 64, "f32", True)
run("2: causal bf16 B4 H16 N65536 D128 (north star)", 4, 16, 65536, 128, "bf16", True)
run("3: causal bf16 B8 H16 N4096 D128 (1.4B-LM layer, 1 GPU)", 8, 16, 4096, 128, "bf16", True)
run("3: same, one of 8 batch x head shards (16 groups)", 1, 16, 4096, 128, "bf16", True)
for D in (64, 128, 256):
    run(f"4: non-causal bf16 B2 H32 N32768 D{D}", 2, 32, 32768, D, "bf16", False, reps=2)
run("5: causal bf16 B1 H16 N=1M, one of 8 sequence shards (131072 rows, carried prefix)", 1, 16, 131072, 128, "bf16",
    True, shard=True)
