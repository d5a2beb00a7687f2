"""Benchmark records in the reference's CSV schema, the log-log slope fit, and a
device sweep driver.

    reference (proj/src/bench.cpp)             here
    BenchRecord (bench.hpp:26-41)              BenchRecord
    kCsvHeader / emit_csv (:405-421)           CSV_HEADER / emit_csv
    read_csv (:459-503)                        read_csv
    fit_slope (:365-403)                       fit_slope
    run_sweep (:279-363)                       run_sweep (device timing, CUDA events)

The reference's parser accepts impl in {fast, quad, softmax, recurrent} and precision
in {f32, f64}. Device records are impl "fast" (the factorised kernel). fp32 device
records are written in exactly that schema; bf16 / fp16 records carry their precision
name in the same 13 columns, which makes such a file a side file the reference parser
rejects by design (bench.cpp:443-449).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

CSV_HEADER = "impl,pass,mask,B,H,N,D,L,workers,precision,wall_time_s,peak_transient_scalars,checksum"


class IoError(RuntimeError):
    """la::IoError (error.hpp:72)."""


class InsufficientData(RuntimeError):
    """la::InsufficientData (error.hpp:67)."""


@dataclass
class BenchRecord:
    impl: str = "fast"
    pass_: str = "fwd"
    mask: str = "causal"
    batch: int = 0
    heads: int = 0
    seq_len: int = 0
    dim: int = 0
    reduction_blocks: int = 0
    workers: int = 0
    precision: str = "f32"
    wall_time_s: float = 0.0
    peak_transient_scalars: int = 0
    checksum: float = 0.0


def _g9(x: float) -> str:
    return "%.9g" % x


def emit_csv(records, out) -> None:
    """emit_csv (bench.cpp:408-421): header line, then one row per record, %.9g floats."""
    out.write(CSV_HEADER + "\n")
    for r in records:
        out.write(",".join([r.impl, r.pass_, r.mask, str(r.batch), str(r.heads), str(r.seq_len), str(r.dim),
                            str(r.reduction_blocks), str(r.workers), r.precision, _g9(r.wall_time_s),
                            str(r.peak_transient_scalars), _g9(r.checksum)]) + "\n")


def read_csv(text: str, precisions=("f32", "f64")):
    """read_csv (bench.cpp:459-503) with the same rejections; ``precisions`` widens the
    accepted set for device side files."""
    lines = text.split("\n")
    if not lines or lines[0] == "" and len(lines) == 1:
        raise IoError("empty CSV input")
    if lines[0] != CSV_HEADER:
        raise IoError("unexpected CSV header: " + lines[0])
    recs = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 13:
            raise IoError("malformed CSV row: " + line)
        if f[0] not in ("fast", "quad", "softmax", "recurrent"):
            raise IoError("unknown impl in CSV: " + f[0])
        if f[1] not in ("fwd", "bwd"):
            raise IoError("unknown pass in CSV: " + f[1])
        if f[2] not in ("causal", "none"):
            raise IoError("unknown mask in CSV: " + f[2])
        if f[9] not in precisions:
            raise IoError("unknown precision in CSV: " + f[9])
        recs.append(BenchRecord(f[0], f[1], f[2], int(f[3]), int(f[4]), int(f[5]), int(f[6]), int(f[7]),
                                int(f[8]), f[9], float(f[10]), int(f[11]), float(f[12])))
    return recs


@dataclass
class SlopeFit:
    slope: float = 0.0
    intercept: float = 0.0
    r2: float = 0.0
    points: list = None


def fit_slope(records, axis: str) -> SlopeFit:
    """fit_slope (bench.cpp:365-403): least squares of log(wall_time_s) on log(N or D)."""
    pts, distinct = [], []
    for r in records:
        x = r.seq_len if axis == "N" else r.dim
        if x <= 0 or r.wall_time_s <= 0.0:
            continue
        pts.append((math.log(float(x)), math.log(r.wall_time_s)))
        if x not in distinct:
            distinct.append(x)
    if len(pts) < 3 or len(distinct) < 3:
        raise InsufficientData("slope fitting needs at least 3 points with distinct axis values")
    n = float(len(pts))
    sx = sy = sxx = sxy = 0.0
    for x, y in pts:
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    slope = (n * sxy - sx * sy) / (n * sxx - sx * sx)
    intercept = (sy - slope * sx) / n
    mean_y = sy / n
    ss_res = sum((y - (intercept + slope * x)) ** 2 for x, y in pts)
    ss_tot = sum((y - mean_y) ** 2 for _, y in pts)
    r2 = max(0.0, 1.0 - ss_res / ss_tot) if ss_tot > 0.0 else (1.0 if ss_res == 0.0 else 0.0)
    return SlopeFit(slope, intercept, r2, pts)


def run_sweep(batch=4, heads=16, seq_lens=(1024, 2048, 4096, 8192), dims=(128,), causal=True,
              precision="bf16", forward_pass=True, backward_pass=True, repeats=5, seed=0, device="cuda"):
    """run_sweep (bench.cpp:279-363) on the device: one record per (N, D, pass), the median
    of ``repeats`` CUDA-event timings after one warm-up; checksum = sum of the pass's
    outputs (bench.cpp:162, 187); peak_transient_scalars = workspace (+ saved states) / 4."""
    import torch

    from . import _abi
    L = _abi.lib()
    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[precision]
    recs = []
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for D in dims:
        for N in seq_lens:
            G = batch * heads
            p = _abi.make_problem(G, N, D, precision, 1.0, 1.0, causal)

            def unit_rows(shape):
                x = torch.rand(shape, device=device, generator=gen) * 2 - 1
                return (x / x.norm(dim=-1, keepdim=True)).to(dt)

            q, k = unit_rows((G, N, D)), unit_rows((G, N, D))
            v = (torch.rand((G, D, N), device=device, generator=gen) * 2 - 1).to(dt)
            w = (torch.rand((G, D, N), device=device, generator=gen) * 2 - 1).to(dt)
            out = torch.empty((G, D, N), device=device, dtype=dt)
            g = torch.empty((G, N), device=device, dtype=torch.float32)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(v), torch.empty_like(v)
            wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=device, dtype=torch.uint8)
            wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=device, dtype=torch.uint8)
            sv = torch.empty(max(1, L.la_saved_state_bytes(C.byref(p))), device=device, dtype=torch.uint8)
            sp = torch.cuda.current_stream().cuda_stream
            err = _abi.ErrorInfo()

            def fwd():
                st = L.la_forward_save(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0,
                                       out.data_ptr(), g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(),
                                       wsf.numel(), sp, C.byref(err))
                assert st == 0, err.message

            def bwd():
                st = L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0,
                                         out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(),
                                         dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(),
                                         sp, C.byref(err))
                assert st == 0, err.message

            def timed(fn):
                fn()
                ts = []
                for _ in range(repeats):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    a.record()
                    fn()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b) / 1e3)
                return float(np.median(ts))

            Lb = next(c for c in range(max(1, D // 32), 0, -1) if D % c == 0)  # default_plan (plan.cpp:28-38)
            mask = "causal" if causal else "none"
            fwd()
            if forward_pass:
                t = timed(fwd)
                recs.append(BenchRecord("fast", "fwd", mask, batch, heads, N, D, Lb, 1, precision, t,
                                        (wsf.numel() + sv.numel()) // 4, float(out.double().sum())))
            if backward_pass:
                t = timed(bwd)
                recs.append(BenchRecord("fast", "bwd", mask, batch, heads, N, D, Lb, 1, precision, t,
                                        wsb.numel() // 4,
                                        float(dq.double().sum() + dk.double().sum() + dv.double().sum())))
            del q, k, v, w, out, g, dq, dk, dv, wsf, wsb, sv
            torch.cuda.empty_cache()
    return recs
