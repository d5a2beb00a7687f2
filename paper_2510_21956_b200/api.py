"""Host-side mirror of the reference library's public API (proj/include/la/*.hpp)
over the sm_100a C-ABI (include/la_cuda.h).

Same names, argument meaning and error behaviour as the reference so callers and
tests port line for line:

    reference (C++)                          here
    la::forward_causal(q,k,v,c,plan,fault)   forward_causal(q,k,v,c,plan,fault)   forward.cpp:133
    la::forward_full(...)                    forward_full(...)                    forward.cpp:139
    la::backward_causal(art,omega,c,plan)    backward_causal(art,omega,c,plan)    backward.cpp:93
    la::backward_full(...)                   backward_full(...)                   backward.cpp:98
    la::default_plan / validate_plan         default_plan / validate_plan         plan.cpp:24-62
    la::Error hierarchy                      Error, InvalidShape, ...             error.hpp:10-75
    la::normalize_qk / relayout              normalize_qk / relayout              plan.cpp:95, tensor.cpp:101
    la::make_omega_hat                       make_omega_hat                       backward.cpp:74
    la::constant_term_pass / linear_term_pass  (same names, TermAccumulator)      forward.cpp:97-131
    la::alpha_term_pass / beta_term_pass     (same names)                         backward.cpp:103-153
    la::make_prefix_state / prefix_advance   (same names, host, O(D^2))           forward.cpp:50-83

Tensors are HeadTensor objects holding a flat buffer in a declared layout.
A buffer that is a CUDA ``torch.Tensor`` runs through the device entry points
(la_forward / la_backward, inputs already in HBM); a numpy buffer runs through
the host entry points (la_host_forward / la_host_backward: copy in, compute,
copy out). Either way the arithmetic is the CUDA library's; nothing here
computes attention on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi


# ----------------------------------------------------------------------------- errors
class Error(RuntimeError):
    """la::Error (error.hpp:10-14)."""


class InvalidShape(Error):
    pass


class ShapeMismatch(Error):
    pass


class InvalidArgument(Error):
    pass


class InvalidPlan(Error):
    pass


class MissingForwardState(Error):
    pass


class CudaError(Error):
    pass


class Unsupported(Error):
    pass


class WorkspaceError(Error):
    pass


class DegenerateDenominator(Error):
    """la::DegenerateDenominator(group, position) (error.hpp:31-47)."""

    def __init__(self, group, position, message=None):
        super().__init__(message or f"degenerate attention denominator at group {group}, "
                                    f"position {position}")
        self._group, self._position = int(group), int(position)

    def group(self):
        return self._group

    def position(self):
        return self._position


_STATUS_EXC = {1: InvalidShape, 2: ShapeMismatch, 3: InvalidArgument, 4: InvalidPlan,
               5: MissingForwardState, 7: CudaError, 8: Unsupported, 9: WorkspaceError}


def _raise(status, err):
    if status == _abi.LA_OK:
        return
    msg = err.message.decode(errors="replace") if err is not None else _abi.STATUS_NAMES[status]
    if status == 6:
        raise DegenerateDenominator(err.group, err.position, msg)
    raise _STATUS_EXC.get(status, Error)(msg)


# ----------------------------------------------------------------------------- data model
class Layout(enum.IntEnum):
    """la::Layout (tensor.hpp:12-15)."""
    FeatureMajor = 0
    SequenceMajor = 1


class Fault(enum.IntEnum):
    """la::Fault (fault.hpp:7-15)."""
    None_ = 0
    FlipBetaKSign = 1
    CausalPrefixOffByOne = 2
    DropGradVConstantTerm = 3


@dataclass
class Shape:
    """la::Shape (tensor.hpp:20-27)."""
    batch: int
    heads: int
    seq_len: int
    dim: int

    def groups(self):
        return self.batch * self.heads


@dataclass
class LinearKernelCoeffs:
    """la::LinearKernelCoeffs, f(x) = a + b*x (tensor.hpp:30-35)."""
    a: float = 1.0
    b: float = 1.0

    def valid(self):
        return self.a != 0.0 or self.b != 0.0


BlockPlan = _abi.BlockPlan


def default_plan(shape: Shape, workers: int = 1) -> BlockPlan:
    """la::default_plan (plan.cpp:24-47)."""
    if shape.batch <= 0 or shape.heads <= 0 or shape.seq_len <= 0 or shape.dim <= 0:
        raise InvalidShape("default_plan requires a valid shape")
    plan = BlockPlan()
    _abi.lib().la_default_plan(shape.groups(), shape.dim, max(1, int(workers)), C.byref(plan))
    return plan


def validate_plan(plan: BlockPlan, groups: int, dim: int) -> None:
    """la::validate_plan (plan.cpp:49-62): raises InvalidPlan."""
    err = _abi.ErrorInfo()
    _raise(_abi.lib().la_validate_plan(C.byref(plan), groups, dim, C.byref(err)), err)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


class HeadTensor:
    """A (groups, seq_len, dim) stack stored flat in a declared layout (tensor.hpp:55-98).

    ``data`` is a 1-D numpy array (host) or a 1-D CUDA torch.Tensor (device).
    """

    def __init__(self, groups, seq_len, dim, layout, data):
        self._g, self._n, self._d = int(groups), int(seq_len), int(dim)
        self._layout = Layout(layout)
        self.data = data

    @staticmethod
    def from_logical(x, layout=Layout.SequenceMajor, dtype=np.float64):
        """Wrap a logical (G, N, D) array (numpy or torch) stored in ``layout``."""
        G, N, D = x.shape
        if _is_torch(x):
            flat = (x.transpose(1, 2) if layout == Layout.FeatureMajor else x).contiguous().reshape(-1)
        else:
            x = np.asarray(x, dtype)
            flat = np.ascontiguousarray(x.transpose(0, 2, 1) if layout == Layout.FeatureMajor else x).reshape(-1)
        return HeadTensor(G, N, D, layout, flat)

    def groups(self):
        return self._g

    def seq_len(self):
        return self._n

    def dim(self):
        return self._d

    def layout(self):
        return self._layout

    def empty(self):
        return self.data is None

    def size(self):
        return self._g * self._n * self._d

    def same_shape(self, other):
        return (self._g, self._n, self._d) == (other._g, other._n, other._d)

    def logical(self):
        """(G, N, D) view of the stored values (numpy float64 for host tensors)."""
        d = self.data
        if _is_torch(d):
            d = d.float().cpu().numpy()
        d = np.asarray(d, np.float64)
        if self._layout == Layout.FeatureMajor:
            return d.reshape(self._g, self._d, self._n).transpose(0, 2, 1)
        return d.reshape(self._g, self._n, self._d)

    def at(self, g, i, j):
        return float(self.logical()[g, i, j])


@dataclass
class ForwardArtifacts:
    """la::ForwardArtifacts (forward.hpp:35-41): out is FeatureMajor, g is (G*N,)."""
    out: HeadTensor = None
    g: object = None
    q: HeadTensor = None
    k: HeadTensor = None
    v: HeadTensor = None
    saved: object = None  # device path: per-segment prefix states (la_forward_save)


@dataclass
class Gradients:
    """la::Gradients (gradients.hpp:8-12): dq SequenceMajor, dk/dv FeatureMajor."""
    dq: HeadTensor = None
    dk: HeadTensor = None
    dv: HeadTensor = None


# ----------------------------------------------------------------------------- dtype plumbing
_TORCH_DT = {"f32": "float32", "bf16": "bfloat16", "f16": "float16"}


def _dtype_of_torch(t):
    import torch
    return {torch.float32: "f32", torch.bfloat16: "bf16", torch.float16: "f16"}[t.dtype]


def _host_buffer(x, dtype):
    """Host staging buffer of ``x`` (numpy, flat) in the device dtype; returns (keepalive, ptr)."""
    if dtype == "f32":
        arr = np.ascontiguousarray(np.asarray(x, np.float32))
        return arr, arr.ctypes.data
    import torch
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float32))).to(getattr(torch, _TORCH_DT[dtype]))
    return t, t.data_ptr()


def _host_out(n, dtype):
    if dtype == "f32":
        arr = np.empty(n, np.float32)
        return arr, arr.ctypes.data
    import torch
    t = torch.empty(n, dtype=getattr(torch, _TORCH_DT[dtype]))
    return t, t.data_ptr()


def _to_np(buf):
    if isinstance(buf, np.ndarray):
        return buf
    return buf.float().numpy()


def _stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


# ----------------------------------------------------------------------------- entry points
def _check_forward_inputs(q, k, v, c, plan):
    """check_forward_inputs (forward.cpp:13-25)."""
    if q is None or k is None or v is None or q.empty() or k.empty() or v.empty():
        raise InvalidShape("forward requires non-empty Q, K, V")
    if not q.same_shape(k) or not q.same_shape(v):
        raise ShapeMismatch("Q, K, V shapes must agree")
    if not c.valid():
        raise InvalidArgument("kernel coefficients (a, b) must not both be zero")
    validate_plan(plan, q.groups(), q.dim())


def _problem(q, c, plan, causal, fault, dtype, impl):
    p = _abi.make_problem(q.groups(), q.seq_len(), q.dim(), dtype, c.a, c.b, causal, int(fault), impl,
                          plan)
    return p


def _run_forward(q, k, v, c, plan, causal, fault, dtype, impl):
    _check_forward_inputs(q, k, v, c, plan)
    L = _abi.lib()
    G, N, D = q.groups(), q.seq_len(), q.dim()
    err = _abi.ErrorInfo()
    if _is_torch(q.data):
        import torch
        dtype = _dtype_of_torch(q.data)
        p = _problem(q, c, plan, causal, fault, dtype, impl)
        dev = q.data.device
        out = torch.empty(G * N * D, dtype=q.data.dtype, device=dev)
        g = torch.empty(G * N, dtype=torch.float32, device=dev)
        ws = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        saved = torch.empty(L.la_saved_state_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        st = L.la_forward_save(C.byref(p), q.data.data_ptr(), int(q.layout()), k.data.data_ptr(),
                               int(k.layout()), v.data.data_ptr(), int(v.layout()), out.data_ptr(),
                               g.data_ptr(), saved.data_ptr(), saved.numel(), ws.data_ptr(), ws.numel(),
                               _stream_ptr(), C.byref(err))
        _raise(st, err)
    else:
        dtype = dtype or "f32"
        p = _problem(q, c, plan, causal, fault, dtype, impl)
        bufs = [_host_buffer(t.data, dtype) for t in (q, k, v)]
        outb, outp = _host_out(G * N * D, dtype)
        g = np.empty(G * N, np.float32)
        st = L.la_host_forward(C.byref(p), bufs[0][1], int(q.layout()), bufs[1][1], int(k.layout()),
                               bufs[2][1], int(v.layout()), outp, g.ctypes.data, C.byref(err))
        _raise(st, err)
        out = _to_np(outb)
    art = ForwardArtifacts()
    art.out = HeadTensor(G, N, D, Layout.FeatureMajor, out)
    art.g = g
    art.q, art.k, art.v = q, k, v
    art.saved = saved if _is_torch(q.data) else None
    return art


def forward_causal(q, k, v, c=LinearKernelCoeffs(), plan=None, fault=Fault.None_, *, dtype=None,
                   impl="auto"):
    """la::forward_causal (forward.cpp:133-137)."""
    plan = plan if plan is not None else default_plan(Shape(1, q.groups(), q.seq_len(), q.dim()))
    return _run_forward(q, k, v, c, plan, True, fault, dtype, impl)


def forward_full(q, k, v, c=LinearKernelCoeffs(), plan=None, fault=Fault.None_, *, dtype=None,
                 impl="auto"):
    """la::forward_full (forward.cpp:139-142)."""
    plan = plan if plan is not None else default_plan(Shape(1, q.groups(), q.seq_len(), q.dim()))
    return _run_forward(q, k, v, c, plan, False, fault, dtype, impl)


def _check_backward_inputs(art, omega, c, plan):
    """check_backward_inputs (backward.cpp:13-28)."""
    if art is None or any(t is None or t.empty() for t in (art.out, art.q, art.k, art.v)):
        raise MissingForwardState("backward requires the forward artifacts (Q, K, V, O)")
    if art.g is None or len(art.g) != art.out.groups() * art.out.seq_len():
        raise MissingForwardState("backward requires the retained denominator vector g")
    if omega is None or omega.empty() or not omega.same_shape(art.out):
        raise ShapeMismatch("cotangent shape must match the forward output")
    if not c.valid():
        raise InvalidArgument("kernel coefficients (a, b) must not both be zero")
    validate_plan(plan, art.out.groups(), art.out.dim())


def _run_backward(art, omega, c, plan, causal, fault, dtype, impl):
    _check_backward_inputs(art, omega, c, plan)
    if art.out.layout() != Layout.FeatureMajor:
        raise InvalidArgument("forward output must be FeatureMajor (forward.cpp:37)")
    L = _abi.lib()
    q, k, v, o = art.q, art.k, art.v, art.out
    G, N, D = q.groups(), q.seq_len(), q.dim()
    err = _abi.ErrorInfo()
    if _is_torch(q.data):
        import torch
        dtype = _dtype_of_torch(q.data)
        p = _problem(q, c, plan, causal, fault, dtype, impl)
        dev = q.data.device
        dq, dk, dv = (torch.empty(G * N * D, dtype=q.data.dtype, device=dev) for _ in range(3))
        ws = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        g = art.g if _is_torch(art.g) else torch.as_tensor(np.asarray(art.g, np.float32), device=dev)
        if art.saved is not None:  # per-segment prefixes (causal) or the K/V totals (non-causal)
            st = L.la_backward_saved(C.byref(p), q.data.data_ptr(), int(q.layout()), k.data.data_ptr(),
                                     int(k.layout()), v.data.data_ptr(), int(v.layout()), o.data.data_ptr(),
                                     omega.data.data_ptr(), int(omega.layout()), g.data_ptr(),
                                     art.saved.data_ptr(), art.saved.numel(), dq.data_ptr(), dk.data_ptr(),
                                     dv.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(), C.byref(err))
        else:
            st = L.la_backward(C.byref(p), q.data.data_ptr(), int(q.layout()), k.data.data_ptr(),
                               int(k.layout()), v.data.data_ptr(), int(v.layout()), o.data.data_ptr(),
                               omega.data.data_ptr(), int(omega.layout()), g.data_ptr(), dq.data_ptr(),
                               dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(),
                               C.byref(err))
        _raise(st, err)
    else:
        dtype = dtype or "f32"
        p = _problem(q, c, plan, causal, fault, dtype, impl)
        bufs = [_host_buffer(t.data, dtype) for t in (q, k, v, o, omega)]
        g = np.ascontiguousarray(np.asarray(art.g, np.float32))
        outs = [_host_out(G * N * D, dtype) for _ in range(3)]
        st = L.la_host_backward(C.byref(p), bufs[0][1], int(q.layout()), bufs[1][1], int(k.layout()),
                                bufs[2][1], int(v.layout()), bufs[3][1], bufs[4][1], int(omega.layout()),
                                g.ctypes.data, outs[0][1], outs[1][1], outs[2][1], C.byref(err))
        _raise(st, err)
        dq, dk, dv = (_to_np(o_[0]) for o_ in outs)
    grads = Gradients()
    grads.dq = HeadTensor(G, N, D, Layout.SequenceMajor, dq)
    grads.dk = HeadTensor(G, N, D, Layout.FeatureMajor, dk)
    grads.dv = HeadTensor(G, N, D, Layout.FeatureMajor, dv)
    return grads


def _plan_for_art(art, plan):
    if plan is not None:
        return plan
    if art is None or art.out is None or art.out.empty():
        raise MissingForwardState("backward requires the forward artifacts (Q, K, V, O)")
    return default_plan(Shape(1, art.out.groups(), art.out.seq_len(), art.out.dim()))


def backward_causal(art, omega, c=LinearKernelCoeffs(), plan=None, fault=Fault.None_, *, dtype=None,
                    impl="auto"):
    """la::backward_causal (backward.cpp:93-96)."""
    return _run_backward(art, omega, c, _plan_for_art(art, plan), True, fault, dtype, impl)


def backward_full(art, omega, c=LinearKernelCoeffs(), plan=None, fault=Fault.None_, *, dtype=None,
                  impl="auto"):
    """la::backward_full (backward.cpp:98-101)."""
    return _run_backward(art, omega, c, _plan_for_art(art, plan), False, fault, dtype, impl)


def max_abs_diff(x: HeadTensor, y: HeadTensor) -> float:
    """la::max_abs_diff (tensor.cpp:121-135); layouts may differ."""
    if not x.same_shape(y):
        raise ShapeMismatch("max_abs_diff requires identical shapes")
    return float(np.max(np.abs(x.logical() - y.logical())))


def launch_count() -> int:
    return int(_abi.lib().la_launch_count())


# ----------------------------------------------------------------------------- prologue + diagnostics
# The reference's API calls either side of the hot path, on
# the device through la_normalize_qk / la_relayout / la_make_omega_hat / la_*_term_pass.
# They take device (CUDA torch) HeadTensors; accumulators are fp32 on the device.
def _device_tensor(t, what):
    if t is None or t.empty():
        raise InvalidShape(what)
    if not _is_torch(t.data) or not t.data.is_cuda:
        raise InvalidArgument("device entry point: tensor data must be a CUDA torch.Tensor")
    return t


def _simple_problem(t, c=None, plan=None):
    c = c or LinearKernelCoeffs()
    return _abi.make_problem(t.groups(), t.seq_len(), t.dim(), _dtype_of_torch(t.data), c.a, c.b, True, 0,
                             "auto", plan)


def normalize_qk(q: HeadTensor, k: HeadTensor):
    """la::normalize_qk (plan.cpp:95-117): unit-norm rows, zero rows kept, layouts kept."""
    import torch
    _device_tensor(q, "normalize_qk requires non-empty Q and K")
    _device_tensor(k, "normalize_qk requires non-empty Q and K")
    if not q.same_shape(k) or q.data.dtype != k.data.dtype:
        raise ShapeMismatch("Q and K shapes must agree")
    qo, ko = torch.empty_like(q.data), torch.empty_like(k.data)
    err = _abi.ErrorInfo()
    p = _simple_problem(q)
    _raise(_abi.lib().la_normalize_qk(C.byref(p), q.data.data_ptr(), int(q.layout()), k.data.data_ptr(),
                                      int(k.layout()), qo.data_ptr(), ko.data_ptr(), _stream_ptr(),
                                      C.byref(err)), err)
    return (HeadTensor(q.groups(), q.seq_len(), q.dim(), q.layout(), qo),
            HeadTensor(k.groups(), k.seq_len(), k.dim(), k.layout(), ko))


def relayout(t: HeadTensor, target) -> HeadTensor:
    """la::relayout (tensor.cpp:101-119): same values in ``target`` layout (shared when equal)."""
    import torch
    _device_tensor(t, "relayout of an empty tensor")
    if Layout(target) == t.layout():
        return t
    y = torch.empty_like(t.data)
    err = _abi.ErrorInfo()
    p = _simple_problem(t)
    _raise(_abi.lib().la_relayout(C.byref(p), t.data.data_ptr(), int(t.layout()), y.data_ptr(), int(target),
                                  _stream_ptr(), C.byref(err)), err)
    return HeadTensor(t.groups(), t.seq_len(), t.dim(), Layout(target), y)


def make_omega_hat(omega: HeadTensor, g) -> HeadTensor:
    """la::make_omega_hat (backward.cpp:74-91): omega / g per row, FeatureMajor."""
    import torch
    _device_tensor(omega, "make_omega_hat requires a non-empty cotangent")
    if g is None or len(g) != omega.groups() * omega.seq_len():
        raise MissingForwardState("denominator vector length must equal groups*seq_len")
    g = g if _is_torch(g) else torch.as_tensor(np.asarray(g, np.float32), device=omega.data.device)
    g = g.to(torch.float32).contiguous()
    out = torch.empty_like(omega.data)
    err = _abi.ErrorInfo()
    p = _simple_problem(omega)
    _raise(_abi.lib().la_make_omega_hat(C.byref(p), omega.data.data_ptr(), int(omega.layout()), g.data_ptr(),
                                        out.data_ptr(), _stream_ptr(), C.byref(err)), err)
    return HeadTensor(omega.groups(), omega.seq_len(), omega.dim(), Layout.FeatureMajor, out)


@dataclass
class TermAccumulator:
    """la::TermAccumulator (forward.hpp:44-50): FeatureMajor (G, D, N) numerator, fp32 on the device."""
    groups: int = 0
    seq_len: int = 0
    dim: int = 0
    data: object = None

    def logical(self):
        return self.data.double().cpu().numpy().reshape(self.groups, self.dim, self.seq_len).transpose(0, 2, 1)


def make_accumulator(groups, seq_len, dim, device="cuda") -> TermAccumulator:
    """la::make_accumulator (forward.cpp:85-95): zero-initialised."""
    import torch
    if groups <= 0 or seq_len <= 0 or dim <= 0:
        raise InvalidShape("accumulator dimensions must be strictly positive")
    return TermAccumulator(groups, seq_len, dim, torch.zeros(groups * dim * seq_len, dtype=torch.float32,
                                                             device=device))


def _check_acc(acc, t):
    if acc.groups != t.groups() or acc.seq_len != t.seq_len() or acc.dim != t.dim():
        raise ShapeMismatch("accumulator shape must match the inputs")


def constant_term_pass(v: HeadTensor, c: LinearKernelCoeffs, f: TermAccumulator) -> None:
    """la::constant_term_pass (forward.cpp:97-107): f = a * prefix sum of V (overwrites)."""
    _device_tensor(v, "constant_term_pass requires a non-empty V")
    if f.groups != v.groups() or f.seq_len != v.seq_len() or f.dim != v.dim():
        raise ShapeMismatch("accumulator shape must match V")
    err = _abi.ErrorInfo()
    p = _simple_problem(v, c)
    _raise(_abi.lib().la_constant_term_pass(C.byref(p), v.data.data_ptr(), int(v.layout()), f.data.data_ptr(),
                                            _stream_ptr(), C.byref(err)), err)


def linear_term_pass(q, k, v, c: LinearKernelCoeffs, plan, f: TermAccumulator) -> None:
    """la::linear_term_pass (forward.cpp:109-131): f += q . (b-weighted causal K^T V state)."""
    for t in (q, k, v):
        _device_tensor(t, "forward requires non-empty Q, K, V")
    _check_forward_inputs(q, k, v, c, plan)
    _check_acc(f, q)
    err = _abi.ErrorInfo()
    p = _simple_problem(q, c, plan)
    _raise(_abi.lib().la_linear_term_pass(C.byref(p), q.data.data_ptr(), int(q.layout()), k.data.data_ptr(),
                                          int(k.layout()), v.data.data_ptr(), int(v.layout()),
                                          f.data.data_ptr(), _stream_ptr(), C.byref(err)), err)


def _check_pass_inputs(a_, b_, omega_hat, plan, dk):
    """check_pass_inputs (backward.cpp:58-72)."""
    for t in (a_, b_, omega_hat):
        _device_tensor(t, "term passes require non-empty inputs")
    if not a_.same_shape(b_) or not a_.same_shape(omega_hat):
        raise ShapeMismatch("term pass input shapes must agree")
    _check_acc(dk, a_)
    validate_plan(plan, a_.groups(), a_.dim())


def alpha_term_pass(q, v, omega_hat, plan, dk: TermAccumulator, b: float = 1.0) -> None:
    """la::alpha_term_pass (backward.cpp:103-128): dk = sum_j alphaK_rj v_ij (assigns)."""
    _check_pass_inputs(q, v, omega_hat, plan, dk)
    err = _abi.ErrorInfo()
    p = _simple_problem(q, LinearKernelCoeffs(1.0, b), plan)
    _raise(_abi.lib().la_alpha_term_pass(C.byref(p), q.data.data_ptr(), int(q.layout()), v.data.data_ptr(),
                                         int(v.layout()), omega_hat.data.data_ptr(), int(omega_hat.layout()),
                                         dk.data.data_ptr(), _stream_ptr(), C.byref(err)), err)


def beta_term_pass(q, o, omega_hat, plan, dk: TermAccumulator, b: float = 1.0) -> None:
    """la::beta_term_pass (backward.cpp:130-153): dk -= sum_j betaK_rj."""
    _check_pass_inputs(q, o, omega_hat, plan, dk)
    err = _abi.ErrorInfo()
    p = _simple_problem(q, LinearKernelCoeffs(1.0, b), plan)
    _raise(_abi.lib().la_beta_term_pass(C.byref(p), q.data.data_ptr(), int(q.layout()), o.data.data_ptr(),
                                        int(o.layout()), omega_hat.data.data_ptr(), int(omega_hat.layout()),
                                        dk.data.data_ptr(), _stream_ptr(), C.byref(err)), err)


@dataclass
class PrefixState:
    """la::PrefixState (forward.hpp:13-25): x1 = a*sum v, x2[j][m] = b*sum k_m v_j, y1 = a*i, y2 = b*sum k.
    The same quantities as a device state record (S^T scaled by b, sigma by a, z by b, count by a)."""
    dim: int = 0
    x1: np.ndarray = None
    x2: np.ndarray = None
    y1: float = 0.0
    y2: np.ndarray = None


def make_prefix_state(dim: int) -> PrefixState:
    """la::make_prefix_state (forward.cpp:50-61)."""
    if dim <= 0:
        raise InvalidShape("prefix state dimension must be strictly positive")
    return PrefixState(dim, np.zeros(dim), np.zeros((dim, dim)), 0.0, np.zeros(dim))


def prefix_advance(state: PrefixState, k_row, v_row, c: LinearKernelCoeffs) -> PrefixState:
    """la::prefix_advance (forward.cpp:63-83): pure one-row update (host, O(D^2), f64 like the reference)."""
    k_row, v_row = np.asarray(k_row, np.float64), np.asarray(v_row, np.float64)
    if k_row.shape != (state.dim,) or v_row.shape != (state.dim,):
        raise ShapeMismatch("prefix_advance rows must match the state dimension")
    x2 = state.x2.copy()
    for j in range(state.dim):  # the reference's accumulation order, row j then column m
        x2[j] += c.b * k_row * v_row[j]
    return PrefixState(state.dim, state.x1 + c.a * v_row, x2, state.y1 + c.a, state.y2 + c.b * k_row)
