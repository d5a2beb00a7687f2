"""CSV schema and slope fit (bench.cpp:365-503) restated in paper_2510_21956_b200/bench_csv.py,
pinned against the reference's own read_csv_file / fit_slope (oracle/_ref), and a
device sweep whose CSV the reference parses (GPU)."""
import ctypes as C
import io
import math

import pytest

from oracle import oracle as O
from paper_2510_21956_b200 import bench_csv as B

needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="reference library not built")


def _recs():
    out = []
    for i, n in enumerate((1024, 2048, 4096, 8192)):
        for ps, f in (("fwd", 1.0), ("bwd", 4.6)):
            out.append(B.BenchRecord("fast", ps, "causal", 4, 16, n, 128, 4, 8, "f32",
                                     f * 1e-3 * n / 1024 * (1 + 0.01 * i), 12345 + i, 0.125 * i - 3.5))
    return out


def _ref_fit(path, axis, ps):
    r = O.ref_lib()
    r.ref_csv_fit.argtypes = [C.c_char_p, C.c_int, C.c_char_p] + [C.c_void_p] * 4
    n, sl, ic, r2 = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
    st = r.ref_csv_fit(path.encode(), 0 if axis == "N" else 1, ps.encode(), C.byref(n), C.byref(sl), C.byref(ic),
                       C.byref(r2))
    return st, n.value, sl.value, ic.value, r2.value


@needs_ref
def test_header_and_fit_match_reference(tmp_path):
    r = O.ref_lib()
    r.ref_csv_header.restype = C.c_char_p
    assert r.ref_csv_header().decode() == B.CSV_HEADER  # test_bench.cpp:94-98
    recs = _recs()
    path = tmp_path / "s.csv"
    with open(path, "w") as f:
        B.emit_csv(recs, f)
    for ps in ("fwd", "bwd"):
        st, n, sl, ic, r2 = _ref_fit(str(path), "N", ps)
        assert st == 0 and n == len(recs)
        fit = B.fit_slope(B.read_csv(path.read_text()), "N") if ps == "" else \
            B.fit_slope([x for x in B.read_csv(path.read_text()) if x.pass_ == ps], "N")
        assert math.isclose(fit.slope, sl, rel_tol=1e-12) and math.isclose(fit.intercept, ic, rel_tol=1e-12, abs_tol=1e-12)
        assert math.isclose(fit.r2, r2, rel_tol=1e-12, abs_tol=1e-12)


@needs_ref
def test_rejections_match_reference(tmp_path):
    bad = B.CSV_HEADER + "\nfast,fwd,causal,4,16,1024,128,4,8,bf16,0.1,1,0.5\n"
    p = tmp_path / "b.csv"
    p.write_text(bad)
    assert _ref_fit(str(p), "N", "")[0] == 10  # IoError: unknown precision
    with pytest.raises(B.IoError):
        B.read_csv(bad)
    assert len(B.read_csv(bad, precisions=("f32", "f64", "bf16"))) == 1  # device side file
    with pytest.raises(B.InsufficientData):
        B.fit_slope(B.read_csv(bad, precisions=("bf16",)), "N")
    with pytest.raises(B.IoError):
        B.read_csv("impl,pass\n")


@pytest.mark.gpu
def test_device_sweep_csv_parses_and_scales_linearly_in_n(cuda, tmp_path):
    # fp32 records (SIMT path) are in the reference schema: its own parser reads them
    recs = B.run_sweep(1, 4, (1024, 2048, 4096), (64,), True, "f32", repeats=2)
    path = tmp_path / "dev.csv"
    with open(path, "w") as f:
        B.emit_csv(recs, f)
    assert len(B.read_csv(path.read_text())) == 6
    if O.ref_lib() is not None:
        st, n, _, _, _ = _ref_fit(str(path), "N", "bwd")
        assert st == 0 and n == 6
    assert all(math.isfinite(r.checksum) for r in recs)
    # bf16 tensor-core records: time linear in N once the grid is full (the O(N) criterion)
    recs = B.run_sweep(4, 16, (16384, 32768, 65536), (128,), True, "bf16", repeats=3)
    for ps in ("fwd", "bwd"):
        fit = B.fit_slope([r for r in recs if r.pass_ == ps], "N")
        assert 0.7 < fit.slope < 1.3, (ps, fit.slope)
