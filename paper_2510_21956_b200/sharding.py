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

The device work goes through an ``ops`` object (CudaOps: the C-ABI in
include/la_cuda.h). Tests substitute a CPU double to check the exchange logic
over the gloo backend.
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

    def forward_shard_state(self, k, v):
        st = self._empty_state(k)
        rc = self.L.la_forward_shard_state(C.byref(self.p), k.data_ptr(), 1, v.data_ptr(), 0, st.data_ptr(),
                                           self._stream())
        assert rc == 0, _abi.STATUS_NAMES[rc]
        return st

    def backward_shard_state(self, q, o, omega, g):
        st = self._empty_state(q)
        rc = self.L.la_backward_shard_state(C.byref(self.p), q.data_ptr(), 1, o.data_ptr(), omega.data_ptr(), 0,
                                            g.data_ptr(), st.data_ptr(), self._stream())
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
