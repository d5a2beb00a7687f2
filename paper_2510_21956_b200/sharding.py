"""Multi-GPU partitioning of the linear-attention path (one process per GPU).

Two modes:

* batch x head sharding: groups are independent (forward_kernels.hpp:221-235),
  so rank r simply owns a contiguous range of the G = B*H groups. No collective.
* sequence sharding: rank r owns rows [r*N/P, (r+1)*N/P) of every group. The
  causal forward needs the exclusive prefix of the per-shard totals
  (S = sum k^T v, z = sum k, sigma = sum v); the backward needs the same prefix
  (for dQ) and the exclusive suffix of (R = sum q^T w_hat, u = sum s q,
  c = sum w_hat) (for dK/dV). One all-gather of the per-shard state records
  per pass (G * (D*D + 2D + 1) fp32, ~1 MB for 16 heads at D=128) over NCCL, then
  a local prefix/suffix sum; the kernels take the result as their carry.

The product entry points are the C-ABI's la_sharded_forward / la_sharded_backward
(``DistStep``): the shard totals, the all-gather (ncclAllGather on a communicator made
by la_nccl_comm_init, or a caller-supplied all-gather) and the prefix / suffix combine
all run inside the library. The step-by-step functions below (an ``ops`` object over
the lower-level C-ABI calls, CudaOps) are kept for tests, which substitute a CPU double
to check the exchange logic over the gloo backend.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _abi


def batch_head_range(groups: int, rank: int, world: int):
    """Contiguous [g0, g1) of the G groups owned by `rank` (balanced to within one group)."""
    g0 = groups * rank // world
    g1 = groups * (rank + 1) // world
    return g0, g1


@dataclass
class SequenceShard:
    """Rows [row0, row1) of an N-row sequence owned by `rank` of `world`."""
    n_total: int
    rank: int
    world: int
    align: int = 128

    @property
    def row0(self):
        per = -(-self.n_total // self.world)
        per = -(-per // self.align) * self.align
        return min(self.n_total, self.rank * per)

    @property
    def row1(self):
        per = -(-self.n_total // self.world)
        per = -(-per // self.align) * self.align
        return min(self.n_total, (self.rank + 1) * per)


def exclusive_prefix(gathered, rank):
    """sum_{t < rank} gathered[t] (gathered: [world, ...])."""
    if rank == 0:
        return gathered[0] * 0
    return gathered[:rank].sum(dim=0)


def exclusive_suffix(gathered, rank):
    """sum_{t > rank} gathered[t]."""
    if rank == gathered.shape[0] - 1:
        return gathered[0] * 0
    return gathered[rank + 1:].sum(dim=0)


def all_gather_states(state, group=None):
    """[world, ...] stack of every rank's state record (one collective)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    flat = state.contiguous().reshape(-1)
    out = torch.empty(world * flat.numel(), dtype=state.dtype, device=state.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    return out.view((world,) + tuple(state.shape))


def sequence_sharded_forward(ops, shard: SequenceShard, q, k, v, group=None):
    """Causal forward of this rank's rows. Returns (out, g, carry_prefix)."""
    state = ops.forward_shard_state(k, v)
    carry = exclusive_prefix(all_gather_states(state, group), shard.rank)
    out, g = ops.forward_with_carry(q, k, v, carry, shard.row0)
    return out, g, carry


def sequence_sharded_backward(ops, shard: SequenceShard, q, k, v, o, omega, g, carry_prefix, group=None):
    """Causal backward of this rank's rows given the forward's carry. Returns (dq, dk, dv)."""
    bstate = ops.backward_shard_state(q, o, omega, g)
    carry_suffix = exclusive_suffix(all_gather_states(bstate, group), shard.rank)
    return ops.backward_with_carry(q, k, v, o, omega, g, carry_prefix, carry_suffix, shard.row0)


class CudaOps:
    """Device ops over the C-ABI for one shard: tensors are flat CUDA torch
    buffers in the canonical layouts (q, k SequenceMajor; v, o, omega FeatureMajor)."""

    def __init__(self, groups, rows, dim, dtype="bf16", a=1.0, b=1.0, impl="auto"):
        self.G, self.N, self.D = groups, rows, dim
        self.p = _abi.make_problem(groups, rows, dim, dtype, a, b, True, impl=impl)
        self.L = _abi.lib()

    def _stream(self):
        import torch
        return torch.cuda.current_stream().cuda_stream

    def _empty_state(self, like):
        import torch
        n = self.L.la_shard_state_floats(C.byref(self.p))
        return torch.zeros(n, dtype=torch.float32, device=like.device)

    def _scratch(self, like):
        import torch
        return torch.empty(self.L.la_shard_state_workspace_bytes(C.byref(self.p)), dtype=torch.uint8,
                           device=like.device)

    def forward_shard_state(self, k, v):
        st, ws = self._empty_state(k), self._scratch(k)
        rc = self.L.la_forward_shard_state(C.byref(self.p), k.data_ptr(), 1, v.data_ptr(), 0, st.data_ptr(),
                                           ws.data_ptr(), ws.numel(), self._stream())
        assert rc == 0, _abi.STATUS_NAMES[rc]
        return st

    def backward_shard_state(self, q, o, omega, g):
        st, ws = self._empty_state(q), self._scratch(q)
        rc = self.L.la_backward_shard_state(C.byref(self.p), q.data_ptr(), 1, o.data_ptr(), omega.data_ptr(), 0,
                                            g.data_ptr(), st.data_ptr(), ws.data_ptr(), ws.numel(), self._stream())
        assert rc == 0, _abi.STATUS_NAMES[rc]
        return st

    def forward_with_carry(self, q, k, v, carry, row0, save=False):
        """Carried forward of this shard; with save=True also returns the per-segment
        saved states (la_forward_sharded_save) for backward_with_carry."""
        import torch
        from .api import _raise
        out = torch.empty_like(v)
        g = torch.empty(self.G * self.N, dtype=torch.float32, device=q.device)
        ws = torch.empty(self.L.la_forward_workspace_bytes(C.byref(self.p)), dtype=torch.uint8, device=q.device)
        sh = _abi.Shard(row0, carry.data_ptr(), None)
        err = _abi.ErrorInfo()
        if save:
            saved = torch.empty(self.L.la_saved_state_bytes(C.byref(self.p)), dtype=torch.uint8, device=q.device)
            rc = self.L.la_forward_sharded_save(C.byref(self.p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1,
                                                v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), saved.data_ptr(),
                                                saved.numel(), ws.data_ptr(), ws.numel(), self._stream(),
                                                C.byref(err))
            _raise(rc, err)
            return out, g, saved
        rc = self.L.la_forward_sharded(C.byref(self.p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1,
                                       v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), ws.data_ptr(), ws.numel(),
                                       self._stream(), C.byref(err))
        _raise(rc, err)
        return out, g

    def backward_with_carry(self, q, k, v, o, omega, g, carry_prefix, carry_suffix, row0, saved=None):
        import torch
        from .api import _raise
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        ws = torch.empty(self.L.la_backward_workspace_bytes(C.byref(self.p)), dtype=torch.uint8, device=q.device)
        sh = _abi.Shard(row0, carry_prefix.data_ptr(), carry_suffix.data_ptr())
        err = _abi.ErrorInfo()
        if saved is not None:
            rc = self.L.la_backward_sharded_saved(C.byref(self.p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1,
                                                  v.data_ptr(), 0, o.data_ptr(), omega.data_ptr(), 0, g.data_ptr(),
                                                  saved.data_ptr(), saved.numel(), dq.data_ptr(), dk.data_ptr(),
                                                  dv.data_ptr(), ws.data_ptr(), ws.numel(), self._stream(),
                                                  C.byref(err))
        else:
            rc = self.L.la_backward_sharded(C.byref(self.p), C.byref(sh), q.data_ptr(), 1, k.data_ptr(), 1,
                                            v.data_ptr(), 0, o.data_ptr(), omega.data_ptr(), 0, g.data_ptr(),
                                            dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(),
                                            self._stream(), C.byref(err))
        _raise(rc, err)
        return dq, dk, dv


# ---------------------------------------------------------------------------- C-ABI entry points
def nccl_comm(rank, world, group=None):
    """An ncclComm_t over the `world` processes of `group` (la_nccl_comm_init; the unique id
    travels over the existing torch.distributed group)."""
    import torch.distributed as dist
    L = _abi.lib()
    obj = [None]
    if rank == 0:
        buf = C.create_string_buffer(128)
        rc = L.la_nccl_get_unique_id(buf)
        assert rc == 0, _abi.STATUS_NAMES[rc]
        obj[0] = buf.raw
    dist.broadcast_object_list(obj, src=0, group=group)
    comm = C.c_void_p()
    rc = L.la_nccl_comm_init(C.byref(comm), world, C.create_string_buffer(obj[0], 128), rank)
    assert rc == 0, _abi.STATUS_NAMES[rc]
    return comm


def host_allgather(group=None):
    """An la_allgather_fn over a CPU torch.distributed group (gloo): device -> host copy,
    all_gather_into_tensor, host -> device. For running several ranks on one device
    (NCCL refuses two ranks on the same GPU); not a product path."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rt = C.CDLL("libcudart.so.12")
    rt.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    rt.cudaStreamSynchronize.argtypes = [C.c_void_p]

    def fn(send, recv, count, ctx, stream):
        world = dist.get_world_size(group)
        host = np.empty(count, dtype=np.float32)
        if rt.cudaStreamSynchronize(stream) != 0:
            return 1
        if rt.cudaMemcpy(host.ctypes.data, send, count * 4, 2) != 0:
            return 1
        out = torch.empty(world * count, dtype=torch.float32)
        dist.all_gather_into_tensor(out, torch.from_numpy(host), group=group)
        return 1 if rt.cudaMemcpy(recv, out.numpy().ctypes.data, world * count * 4, 1) != 0 else 0

    return _abi.ALLGATHER_FN(fn)


class DistStep:
    """Forward + backward of this rank's shard through la_sharded_forward /
    la_sharded_backward. mode: "batch_head" (rank owns whole groups; p = its local
    groups) or "sequence" (rank owns rows [row_offset, row_offset + rows) of every
    group). Tensors are flat CUDA buffers in the canonical layouts (q, k SequenceMajor;
    v, o, omega FeatureMajor)."""

    def __init__(self, groups, rows, dim, mode, rank, nranks, row_offset=0, dtype="bf16", a=1.0, b=1.0,
                 comm=None, allgather=None, impl="auto"):
        self.L = _abi.lib()
        self.G, self.N, self.D = groups, rows, dim
        self.p = _abi.make_problem(groups, rows, dim, dtype, a, b, True, impl=impl)
        self.d = _abi.Dist()
        self.d.mode = _abi.SHARD_SEQUENCE if mode == "sequence" else _abi.SHARD_BATCH_HEAD
        self.d.rank, self.d.nranks, self.d.row_offset = rank, nranks, row_offset
        self.d.nccl_comm = comm.value if isinstance(comm, C.c_void_p) else comm
        if allgather is not None:
            self.d.allgather = allgather
        self._keep = allgather  # the callback must outlive the calls
        self.saved_bytes = self.L.la_dist_saved_bytes(C.byref(self.p), C.byref(self.d))
        self.ws_bytes = self.L.la_dist_workspace_bytes(C.byref(self.p), C.byref(self.d))
        self._ws = None

    def _workspace(self, dev):
        import torch
        if self._ws is None:
            self._ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        return self._ws

    @staticmethod
    def _stream():
        import torch
        return torch.cuda.current_stream().cuda_stream

    def forward(self, q, k, v, out=None, g=None, saved=None, check=True):
        """check=False keeps the call asynchronous (no degenerate-denominator readback)."""
        import torch
        from .api import _raise
        out = torch.empty_like(v) if out is None else out
        g = torch.empty(self.G * self.N, dtype=torch.float32, device=q.device) if g is None else g
        saved = torch.empty(self.saved_bytes, dtype=torch.uint8, device=q.device) if saved is None else saved
        ws = self._workspace(q.device)
        err = _abi.ErrorInfo()
        rc = self.L.la_sharded_forward(C.byref(self.p), C.byref(self.d), q.data_ptr(), 1, k.data_ptr(), 1,
                                       v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), saved.data_ptr(), saved.numel(),
                                       ws.data_ptr(), ws.numel(), self._stream(), C.byref(err) if check else None)
        _raise(rc, err)
        return out, g, saved

    def backward(self, q, k, v, o, omega, g, saved, dq=None, dk=None, dv=None, check=True):
        import torch
        from .api import _raise
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k if k.shape == v.shape else v) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
        ws = self._workspace(q.device)
        err = _abi.ErrorInfo()
        rc = self.L.la_sharded_backward(C.byref(self.p), C.byref(self.d), q.data_ptr(), 1, k.data_ptr(), 1,
                                        v.data_ptr(), 0, o.data_ptr(), omega.data_ptr(), 0, g.data_ptr(),
                                        saved.data_ptr(), saved.numel(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                        ws.data_ptr(), ws.numel(), self._stream(), C.byref(err) if check else None)
        _raise(rc, err)
        return dq, dk, dv
