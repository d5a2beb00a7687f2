"""Benchmark: causal linear-attention fwd+bwd (f(x) = a + b*x) on B200.

Default workload = BASELINE.json configs[1], the north star:
B=4 H=16 N=65536 D=128, bf16, causal, a=b=1, one fwd+bwd per step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python bench.py --config 3|5 ...   (the sharded BASELINE configs, see run_sharded_arm)

Our arm: inputs resident in HBM (each input tensor is 1.07 GB, far above the
126 MB L2, so no flush is needed between steps); K steps timed with CUDA events
on the launching stream between barriers; max over ranks. N>1 ranks each run
their own batch x head shard (weak scaling, no collective on the data path).
`e2e` repeats the step through the host-buffer C-ABI (la_host_step: pinned host ->
HBM -> host every step). `cpu_baseline` times the reference's own CPU path
(oracle/_ref, compiled from the reference sources; else the oracle port) on a
bounded sample (8 heads x 16384 rows); `--impl reference` runs that CPU path on the
FULL workload every step (same config object as this arm).

`roofline` is the dominant phase (the backward: W_hat / R aggregate + reverse sweep)
against its algorithmic bytes 8 D e + 4 per row; `phases` holds both phases,
`kernels` each kernel's in-region time and ncu DRAM bytes (profiles/ncu_traffic.json).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "causal LA fwd+bwd tokens/s at N=64K D=128"
UNIT = "tokens/s"
CFG = dict(batch=4, heads=16, seq_len=65536, dim=128, dtype="bf16", causal=True, a=1.0, b=1.0)
# CPU sample for the reference arm / cpu_baseline: 8 heads x 16384 rows of the same
# shape family (f32 fast path, as the reference bench times it, bench.cpp:111-191).
CPU_SAMPLE = dict(groups=8, seq_len=16384, dim=128)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML (SM clock, max SM clock, clock-event reasons) from a thread every
    ~2 ms while the timed region runs; one sample is always taken on entry and exit,
    so even a short region is covered."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, period_s=0.002):
        self.index, self.period, self.rows, self.h, self.nv = index, period_s, [], None, None
        self.stop = threading.Event()

    def _handle(self):
        import pynvml as nv
        import torch
        nv.nvmlInit()
        self.nv = nv
        try:  # match the CUDA device to its NVML handle by UUID (CUDA_VISIBLE_DEVICES safe)
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            for i in range(nv.nvmlDeviceGetCount()):
                h = nv.nvmlDeviceGetHandleByIndex(i)
                u = nv.nvmlDeviceGetUUID(h)
                u = u.decode() if isinstance(u, bytes) else u
                if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                    return h
        except Exception:
            pass
        return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((sm, mx, rs))

    def _loop(self):
        while not self.stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            self.h = self._handle()
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        # the entry/exit samples bracket the region; the load samples are the inner ones
        inner = self.rows[1:-1] or self.rows
        reasons = sorted({n for _, _, r in self.rows for bit, n in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _, _ in inner),
                "sm_max_mhz": max(m for _, m, _ in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


# ----------------------------------------------------------------------------- CPU arms
def cpu_inputs(seed=0):
    import numpy as np
    G, N, D = CPU_SAMPLE["groups"], CPU_SAMPLE["seq_len"], CPU_SAMPLE["dim"]
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (G, N, D)).astype(np.float32)
    k = rng.uniform(-1, 1, (G, N, D)).astype(np.float32)
    q /= np.linalg.norm(q, axis=2, keepdims=True)
    k /= np.linalg.norm(k, axis=2, keepdims=True)
    # canonical reference layouts: q,k SequenceMajor; v, omega FeatureMajor ([g][j][i])
    v = rng.uniform(-1, 1, (G, D, N)).astype(np.float32)
    w = rng.uniform(-1, 1, (G, D, N)).astype(np.float32)
    return q, k, v, w


def cpu_runner():
    """(kind, fn) timing one fwd+bwd of the CPU sample with all host threads."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    q, k, v, w = cpu_inputs()
    shp = lambda x: x.reshape(CPU_SAMPLE["groups"], CPU_SAMPLE["seq_len"], CPU_SAMPLE["dim"])
    if O.ref_lib() is not None:
        def fn():
            O.ref_fwd_bwd_f32(q, k, shp(v), shp(w), workers=cores)
        return "reference", cores, fn
    def fn():
        O.fwd_bwd_f32_threads(q, k, shp(v), shp(w), threads=cores)
    return "port", min(cores, CPU_SAMPLE["groups"]), fn


def cpu_sample_desc(kind):
    s = CPU_SAMPLE
    src = ("reference la_core detail::run_forward<float> + run_backward<float> (oracle/_ref, built from "
           "/root/reference/proj/src)" if kind == "reference" else "oracle/oracle.c f32 port")
    return (f"{src}; {s['groups']} heads x N={s['seq_len']} x D={s['dim']} f32 causal, U(-1,1) with "
            f"row-normalised q,k; tokens/s scaled to the config as (heads_sample*N_sample/H)/t, "
            f"valid because cost is linear in N and in heads (acceptance.cpp:118)")


def cpu_tokens_per_s(t):
    return CPU_SAMPLE["groups"] * CPU_SAMPLE["seq_len"] / CFG["heads"] / t


def full_cpu_inputs(seed=0):
    """The whole north-star workload in the reference's f32 layouts (bench.cpp:75-97
    distribution: U(-1,1), q/k rows normalised; q, k SequenceMajor, v, omega FeatureMajor)."""
    import numpy as np
    G, N, D = CFG["batch"] * CFG["heads"], CFG["seq_len"], CFG["dim"]
    rng = np.random.default_rng(seed)

    def uni(shape):
        x = rng.random(shape, dtype=np.float32)
        x *= 2
        x -= 1
        return x

    q, k = uni((G, N, D)), uni((G, N, D))
    for x in (q, k):
        x /= np.linalg.norm(x, axis=2, keepdims=True)
    return q, k, uni((G, D, N)), uni((G, D, N))


def our_config(world=1, kernel="auto", graph=False):
    """The `config` object of the default arm; the reference arm reports the same one."""
    wl = ("causal LA fwd+bwd B=4 H=16 N=65536 D=128 a=b=1 per GPU (BASELINE configs[1])" if CFG["causal"] else
          f"non-causal LA fwd+bwd B=2 H=32 N=32768 D={CFG['dim']} a=b=1 (BASELINE configs[3])")
    return {"workload": wl,
            "global_batch": CFG["batch"] * world, "seq_len": CFG["seq_len"], "heads": CFG["heads"],
            "dim": CFG["dim"], "parallelism": f"batch_head{world}",
            "l2": "inputs 1.07 GB each >> 126 MB L2; no flush", "kernel_impl": kernel, "cuda_graph": bool(graph)}


def run_reference_arm(args):
    """The reference's own CPU implementation of the path (oracle/_ref: la_core built from
    /root/reference/proj/src, else the C port) on the FULL workload every step: G = 64
    heads x N = 65536 x D = 128, run_forward<float> + run_backward<float> with all host
    threads, exactly the calls bench.cpp:137-139 / 176-179 time."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    G, N, D = CFG["batch"] * CFG["heads"], CFG["seq_len"], CFG["dim"]
    q, k, v, w = full_cpu_inputs()
    outs = (np.empty(G * N * D, np.float32), np.empty(G * N, np.float32),
            *(np.empty(G * N * D, np.float32) for _ in range(3)))
    for x in outs:  # first touch outside the timed steps
        x.fill(0)
    v3, w3 = v.reshape(G, N, D), w.reshape(G, N, D)  # flat FeatureMajor buffers, shape only
    if O.ref_lib() is not None:
        kind = "reference"

        def fn():
            O.ref_fwd_bwd_f32(q, k, v3, w3, workers=cores, outs=outs)
    else:
        kind, cores = "port", min(cores, G)

        def fn():
            O.fwd_bwd_f32_threads(q, k, v3, w3, threads=cores)
    # one full fwd+bwd takes ~16-20 s on 16 cores: at most one warm-up step (it only pages in
    # the buffers), and the timed steps stop once --ref-budget-s is spent (at least 2), so the
    # arm ends within a few minutes; `steps` / `warmup` report what actually ran
    warm = min(args.warmup, 1)
    for _ in range(warm):
        fn()
    times = []
    t_start = time.perf_counter()
    for i in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if i + 1 >= 2 and time.perf_counter() - t_start > args.ref_budget_s:
            break
    t = sum(times) / len(times)
    val = CFG["batch"] * N / t
    src = ("reference la_core detail::run_forward<float> + run_backward<float> (oracle/_ref, built from "
           "/root/reference/proj/src)" if kind == "reference" else "oracle/oracle.c f32 port")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (U(-1,1), unit-norm q/k rows)", "config": our_config(),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{src}; the full workload every step (G=64 x N=65536 x D=128, f32, "
                                       f"causal, canonical layouts), {cores} worker threads"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
ALG_BYTES = {  # algorithmic bytes per processed row (D, element bytes e), SURVEY §8(d)
    "fwd": lambda D, e: 4 * D * e + 4,
    "bwd": lambda D, e: 8 * D * e + 4,
}


def run_our_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_21956_b200 as la  # noqa: F401  (loads the CUDA library)
    from paper_2510_21956_b200 import _abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _abi.lib()
    B, H, N, D = CFG["batch"], CFG["heads"], CFG["seq_len"], CFG["dim"]
    G = B * H
    e = 2
    p = _abi.make_problem(G, N, D, CFG["dtype"], CFG["a"], CFG["b"], CFG["causal"], impl=args.kernel)

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def unit_rows(shape):
        x = torch.rand(shape, device=dev, generator=gen, dtype=torch.float32) * 2 - 1
        return (x / x.norm(dim=-1, keepdim=True)).to(torch.bfloat16)

    def uni(shape):
        return (torch.rand(shape, device=dev, generator=gen, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)

    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    q = unit_rows((G, N, D))       # SequenceMajor
    k = unit_rows((G, N, D))       # SequenceMajor
    v = uni((G, D, N))             # FeatureMajor
    w = uni((G, D, N))             # FeatureMajor (cotangent dO)
    out = torch.empty((G, D, N), device=dev, dtype=torch.bfloat16)
    g = torch.empty((G, N), device=dev, dtype=torch.float32)
    dq = torch.empty((G, N, D), device=dev, dtype=torch.bfloat16)
    dk = torch.empty((G, D, N), device=dev, dtype=torch.bfloat16)
    dv = torch.empty((G, D, N), device=dev, dtype=torch.bfloat16)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    # per-(group, segment) prefix states saved by the forward for the backward
    # (the analogue of keeping (out, g) in ForwardArtifacts)
    saved = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    FMj, SMj = 0, 1

    def step():
        sp = torch.cuda.current_stream(dev).cuda_stream  # the capture stream under --graph
        st = L.la_forward_save(C.byref(p), q.data_ptr(), SMj, k.data_ptr(), SMj, v.data_ptr(), FMj,
                               out.data_ptr(), g.data_ptr(), saved.data_ptr(), saved.numel(), wsf.data_ptr(),
                               wsf.numel(), sp, None)
        assert st == 0, _abi.STATUS_NAMES[st]
        st = L.la_backward_saved(C.byref(p), q.data_ptr(), SMj, k.data_ptr(), SMj, v.data_ptr(), FMj,
                                 out.data_ptr(), w.data_ptr(), FMj, g.data_ptr(), saved.data_ptr(), saved.numel(),
                                 dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), sp,
                                 None)
        assert st == 0, _abi.STATUS_NAMES[st]

    for _ in range(args.warmup):
        step()
    launches_per_graph = 0
    if args.graph:
        # one step captured in a CUDA graph and replayed in the timed region; event records
        # inside a graph carry no timing, so the per-kernel times come from eager steps run
        # right after the timed region (`kernels_source` in the line)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        c0 = L.la_launch_count()
        with torch.cuda.graph(graph):
            step()
        launches_per_graph = L.la_launch_count() - c0  # replays do not pass through the host API
        eager_step, step = step, graph.replay
        for _ in range(2):
            step()
    err = _abi.ErrorInfo()
    st = L.la_query_status(wsf.data_ptr(), sp, C.byref(err))
    assert st == 0, f"forward status {_abi.STATUS_NAMES[st]}: {err.message}"
    torch.cuda.synchronize()

    # ---- timed region
    if not args.graph:
        L.la_profile_enable(1)
        _abi.profile_read()
    launches0 = L.la_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.la_launch_count() - launches0 + launches_per_graph * args.steps
    # ---- peak HBM: everything the step touches is allocated through torch
    # (inputs, outputs, workspaces, saved segment states); the library itself allocates
    # nothing on this path, which the driver-level free-memory delta cross-checks.
    T_ = G * N * D * e
    retained = 4 * T_ + 4 * T_ + 4 * G * N  # q, k, v, dO in; o, dq, dk, dv out; g
    transient = wsf.numel() + wsb.numel() + saved.numel()
    memory = {"peak_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
              "driver_delta_bytes": int(free0 - torch.cuda.mem_get_info(dev)[0]),
              "retained_bytes": int(retained), "transient_bytes": int(transient),
              "minimal_retained_bytes": int(8 * T_ + 4 * G * N),
              "note": "retained = q,k,v,dO,o,g,dq,dk,dv; transient = fwd/bwd workspaces + per-segment "
                      "saved prefix states (O(G*P*D^2), independent of N)"}
    prof_steps = args.steps
    if args.graph:
        for _ in range(2):
            eager_step()
        torch.cuda.synchronize()
        L.la_profile_enable(1)
        _abi.profile_read()
        prof_steps = 5
        for _ in range(prof_steps):
            eager_step()
        torch.cuda.synchronize()
    L.la_profile_enable(0)
    prof = _abi.profile_read()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    tokens_step = B * N * world
    value = tokens_step / (ms / 1e3)

    # ---- roofline per phase from the in-region events. The algorithmic bytes of SURVEY
    # 8(d) belong to a phase, not to one kernel: the forward (aggregate + sweep) reads
    # Q, K, V and writes O, g (4 D e + 4 per row); the backward (W_hat / R aggregate +
    # sweep) reads Q, K, V, O, dO, g and writes dQ, dK, dV (8 D e + 4 per row). The
    # dominant phase is the `roofline` object; `traffic` is the ncu DRAM bytes of the
    # same kernels (profiles/ncu_traffic.json, one --set full capture per kernel).
    hbm, tf, src = peaks()
    per = {}
    for r in prof:
        per.setdefault(r["name"], []).append(r["ms"])
    kstats = {n: {"ms": sum(v_) / len(v_), "launches_per_step": len(v_) / prof_steps,
                  "share": sum(v_) / prof_steps / ms} for n, v_ in per.items()}
    ncu = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        ncu = {k_: v_ for k_, v_ in json.load(open(tpath)).items() if not k_.startswith("_")}
    for n, st_ in kstats.items():
        st_["ncu_dram_bytes"] = ncu.get(n)
    phases = {}
    for ph, prefix in (("forward", "la_fwd"), ("backward", "la_bwd")):
        names = sorted(n for n in kstats if n.startswith(prefix))
        if not names:
            continue
        pms = sum(kstats[n]["ms"] * kstats[n]["launches_per_step"] for n in names)
        alg = G * N * ALG_BYTES["fwd" if ph == "forward" else "bwd"](D, e)
        traffic = sum(ncu[n] for n in names) if all(n in ncu for n in names) else None
        ach = alg / (pms / 1e3) / 1e9
        phases[ph] = {"bound": "hbm", "kernel": " + ".join(names) + f" ({ph} phase)", "achieved": ach,
                      "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": traffic, "peak_source": src,
                      "alg_bytes_per_launch": alg, "kernel_ms": pms,
                      "traffic_over_alg": traffic / alg if traffic else None}
    roof = max(phases.values(), key=lambda r_: r_["kernel_ms"]) if phases else None
    step_bytes = G * N * (ALG_BYTES["fwd"](D, e) + ALG_BYTES["bwd"](D, e))
    step_gbs = step_bytes / (ms / 1e3) / 1e9
    flops = G * N * 14 * D * D
    clocks = clk.summary()

    # ---- e2e through the host-buffer C-ABI (pinned host memory, copies every step)
    e2e = None
    if not args.no_e2e:
        pin = dict(device="cpu", dtype=torch.bfloat16, pin_memory=True)
        hq, hk, hv, hw = (x.cpu().pin_memory() for x in (q, k, v, w))
        hout, hdq, hdk, hdv = (torch.empty(x.shape, **pin) for x in (out, dq, dk, dv))
        hg = torch.empty((G, N), dtype=torch.float32, pin_memory=True)

        def e2e_step():  # one training step through the host-buffer C-ABI (la_host_step)
            st = L.la_host_step(C.byref(p), hq.data_ptr(), SMj, hk.data_ptr(), SMj, hv.data_ptr(), FMj,
                                hw.data_ptr(), FMj, hout.data_ptr(), hg.data_ptr(), hdq.data_ptr(),
                                hdk.data_ptr(), hdv.data_ptr(), C.byref(err))
            assert st == 0, err.message

        e2e_step()
        if world > 1:
            dist.barrier()
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        et = (time.perf_counter() - te) / args.e2e_steps
        if world > 1:
            tt = torch.tensor([et], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        T = G * N * D * e
        e2e = {"value": tokens_step / et, "unit": UNIT, "h2d_bytes_per_step": 4 * T,
               "d2h_bytes_per_step": 4 * T + 4 * G * N, "ms_per_step": et * 1e3,
               "api": "la_host_step: forward + backward over pinned host buffers (q, k, v, dO in; "
                      "o, g, dq, dk, dv out), group blocks pipelined over H2D / compute / D2H streams"}
        L.la_host_release()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind, cores, fn = cpu_runner()
        fn()
        ts = []
        for _ in range(3):
            t_ = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t_)
        cpu = {"value": cpu_tokens_per_s(statistics.median(ts)), "unit": UNIT, "cores": cores,
               "kind": kind, "sample": cpu_sample_desc(kind)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (U(-1,1), unit-norm q/k rows)",
                "config": our_config(world, args.kernel, args.graph),
                "roofline": roof, "phases": phases,
                "step_roofline": {"alg_bytes": step_bytes, "achieved_gbs": step_gbs, "frac_hbm": step_gbs / hbm,
                                  "alg_tflops": flops / (ms / 1e3) / 1e12,
                                  "frac_bf16": flops / (ms / 1e3) / 1e12 / tf},
                "library": L.la_version().decode(),
                "kernels": kstats, "kernels_source": "eager steps after the graph-replayed timed region"
                if args.graph else "timed region", "memory": memory, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- sharded configs
SHARDED = {
    # BASELINE configs[2]: 1.4B-LM attention layer, batch x head sharded (no collective)
    "3": dict(batch=8, heads=16, seq_len=4096, mode="batch_head",
              metric="causal LA fwd+bwd tokens/s, B=8 H=16 N=4096 D=128 (batch x head sharded)"),
    # BASELINE configs[4]: long context, sequence-sharded with an all-gather scan of shard states
    "5": dict(batch=1, heads=16, seq_len=1 << 20, mode="sequence",
              metric="causal LA fwd+bwd tokens/s, B=1 H=16 N=1M D=128 (sequence sharded)"),
}


def run_sharded_arm(args):
    """Config 3: the B*H = 128 groups split over ranks (strong scaling of one layer, no
    collective). Config 5: every rank owns N / world consecutive rows of all 16 heads;
    one step = shard totals -> NCCL all-gather -> exclusive prefix -> carried forward,
    then backward shard totals -> all-gather -> exclusive suffix -> carried backward,
    all inside the C-ABI's la_sharded_forward / la_sharded_backward (csrc/la_dist.cu;
    sharding.DistStep is the ctypes wrapper). Same timing rules as the default arm."""
    import torch
    import torch.distributed as dist

    from paper_2510_21956_b200 import _abi
    from paper_2510_21956_b200 import sharding as S

    cfg = SHARDED[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _abi.lib()
    D, G_all, N_all = 128, cfg["batch"] * cfg["heads"], cfg["seq_len"]
    if cfg["mode"] == "batch_head":
        g0, g1 = S.batch_head_range(G_all, rank, world)
        G, N, row0 = g1 - g0, N_all, 0
    else:
        sh = S.SequenceShard(N_all, rank, world)
        G, N, row0 = G_all, sh.row1 - sh.row0, sh.row0
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)

    def unit_rows(shape):
        x = torch.rand(shape, device=dev, generator=gen) * 2 - 1
        return (x / x.norm(dim=-1, keepdim=True)).to(torch.bfloat16)

    q, k = unit_rows((G, N, D)), unit_rows((G, N, D))
    v = (torch.rand((G, D, N), device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand((G, D, N), device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
    # the C-ABI multi-GPU entry points: shard totals, ncclAllGather and the prefix / suffix
    # combine run inside la_sharded_forward / la_sharded_backward (la_dist.cu)
    if world > 1:
        comm = S.nccl_comm(rank, world)
    else:  # one rank: the library's single-shard exchange (a record copy), no communicator
        comm = None
    dstep = S.DistStep(G, N, D, cfg["mode"], rank, world, row_offset=row0, comm=comm)
    out, g = torch.empty_like(v), torch.empty(G * N, device=dev)
    saved = torch.empty(dstep.saved_bytes, dtype=torch.uint8, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(v), torch.empty_like(v)

    def step():  # the forward's saved segment states feed the backward (no K/V re-read)
        dstep.forward(q, k, v, out=out, g=g, saved=saved, check=False)
        dstep.backward(q, k, v, out, w, g, saved, dq=dq, dk=dk, dv=dv, check=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    per_graph = 0
    if args.graph:  # small shards are launch-bound: replay one captured step (no host gaps)
        graph = torch.cuda.CUDAGraph()
        c0 = L.la_launch_count()
        with torch.cuda.graph(graph):
            step()
        per_graph = L.la_launch_count() - c0  # replays do not pass through the host API
        step = graph.replay
        for _ in range(2):
            step()
        torch.cuda.synchronize()
    launches0 = L.la_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.la_launch_count() - launches0 + per_graph * args.steps
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    tokens = cfg["batch"] * N_all  # the whole job's tokens per step
    hbm, tf, src = peaks()
    alg = G_all * N_all * 3080 / max(1, world)  # per-rank algorithmic bytes
    if rank == 0:
        print(json.dumps({
            "metric": cfg["metric"], "value": tokens / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (U(-1,1), unit-norm q/k rows)",
            "config": {"workload": f"BASELINE config {args.config}", "global_batch": cfg["batch"],
                       "seq_len": N_all, "heads": cfg["heads"], "dim": D,
                       "parallelism": f"{cfg['mode']}{world}", "l2": "inputs > L2 at world <= 8; no flush",
                       "cuda_graph": bool(args.graph)},
            "step_roofline": {"alg_bytes_per_rank": alg, "achieved_gbs": alg / (ms / 1e3) / 1e9,
                              "frac_hbm": alg / (ms / 1e3) / 1e9 / hbm},
            "e2e": None, "cpu_baseline": None, "gpu_launches": int(launches), "clocks": clk.summary()}),
            flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: stop timing full-workload CPU steps after this many seconds")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true", help="replay the step as a captured CUDA graph")
    ap.add_argument("--config", default="2", choices=["2", "3", "4", "5"],
                    help="2 = the north star (default); 3 / 5 = the sharded BASELINE configs; "
                         "4 = the non-causal head-dim sweep (one D per run, --dim)")
    ap.add_argument("--dim", type=int, default=128, choices=[64, 128, 256], help="config 4 head dim")
    args = ap.parse_args()
    if args.config == "4":  # BASELINE configs[3]: same single-GPU arm, non-causal B2 H32 N32768
        global METRIC
        CFG.update(batch=2, heads=32, seq_len=32768, dim=args.dim, causal=False)
        METRIC = f"non-causal LA fwd+bwd tokens/s, B=2 H=32 N=32768 D={args.dim}"
        args.no_cpu_baseline = True  # the CPU sample above is the causal D=128 path
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.config in ("3", "5"):
        run_sharded_arm(args)
    else:
        run_our_arm(args)


if __name__ == "__main__":
    main()
