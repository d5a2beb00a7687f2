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
        if art.saved is not None and causal:
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
