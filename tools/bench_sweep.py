"""Device sweeps in the reference's CSV schema with the reference's slope criteria
(bench.cpp:279-503, SPEC N-slope ~1, D-slope ~2 on the CPU).

    python tools/bench_sweep.py --axis N --out gpurun_out/sweep_N.csv
    python tools/bench_sweep.py --axis D --dims 32,64,128 --out gpurun_out/sweep_D.csv

Prints one JSON line per pass with the fitted slope / r2 (our restatement of
fit_slope), and writes the CSV (a side file when --precision is not f32/f64).
On the GPU the kernels are HBM-bound: bytes and time grow ~linearly in N and in D,
so the D-slope is ~1 here where the reference's CPU path (compute-bound) gives ~2."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_21956_b200 import bench_csv as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--axis", choices=["N", "D"], default="N")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq-lens", default="4096,8192,16384,32768,65536")
    ap.add_argument("--dims", default="128")
    ap.add_argument("--mask", choices=["causal", "none"], default="causal")
    ap.add_argument("--precision", default="bf16", choices=["f32", "bf16", "f16"])
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/sweep.csv")
    a = ap.parse_args()
    Ns = [int(x) for x in a.seq_lens.split(",")]
    Ds = [int(x) for x in a.dims.split(",")]
    if a.axis == "D" and len(Ds) < 3:
        Ds = [32, 64, 128]
    if a.axis == "D":
        Ns = Ns[:1]
    recs = B.run_sweep(a.batch, a.heads, Ns, Ds, a.mask == "causal", a.precision, repeats=a.repeats)
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    with open(a.out, "w") as f:
        B.emit_csv(recs, f)
    for ps in ("fwd", "bwd"):
        sel = [r for r in recs if r.pass_ == ps]
        fit = B.fit_slope(sel, a.axis)
        print(json.dumps({"pass": ps, "axis": a.axis, "slope": fit.slope, "r2": fit.r2, "precision": a.precision,
                          "points": [(r.seq_len if a.axis == "N" else r.dim, r.wall_time_s) for r in sel],
                          "csv": a.out}), flush=True)


if __name__ == "__main__":
    main()
