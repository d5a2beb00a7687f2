"""Multi-GPU partitioning (paper_2510_21956_b200/sharding.py).

* CPU, world_size 2 over gloo: the sequence-sharding exchange (all-gather of shard
  states, exclusive prefix / suffix, row offsets) with a float64 CPU double of the
  device ops, checked against the unsharded oracle.
* GPU (-m gpu): the same exchange through the C-ABI carries (la_forward_sharded /
  la_backward_sharded), shards simulated sequentially on one device.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2510_21956_b200 import sharding as S
from tests._util import fast_inputs, max_abs, rel_err


# ---------------------------------------------------------------------------- CPU double
class CpuOps:
    """float64 torch restatement of the four shard ops on logical (G, rows, D) tensors."""

    def __init__(self, a=1.0, b=1.0):
        self.a, self.b = a, b

    @staticmethod
    def _rec(X, va, vb, count):
        G, D = X.shape[0], X.shape[1]
        sz = (D * D + 2 * D + 1 + 3) // 4 * 4
        r = torch.zeros(G, sz, dtype=torch.float64)
        r[:, :D * D] = X.reshape(G, -1)
        r[:, D * D:D * D + D] = va
        r[:, D * D + D:D * D + 2 * D] = vb
        r[:, D * D + 2 * D] = count
        return r

    @staticmethod
    def _unrec(r, D):
        G = r.shape[0]
        return r[:, :D * D].reshape(G, D, D), r[:, D * D:D * D + D], r[:, D * D + D:D * D + 2 * D]

    def forward_shard_state(self, k, v):
        return self._rec(torch.einsum("gtm,gtj->gmj", k, v), k.sum(1), v.sum(1), k.shape[1])

    def forward_with_carry(self, q, k, v, carry, row0):
        a, b = self.a, self.b
        D = q.shape[2]
        Sc, zc, sc = self._unrec(carry, D)
        Scum = Sc[:, None] + torch.cumsum(torch.einsum("gtm,gtj->gtmj", k, v), 1)
        zcum = zc[:, None] + torch.cumsum(k, 1)
        scum = sc[:, None] + torch.cumsum(v, 1)
        idx = torch.arange(q.shape[1], dtype=torch.float64)
        g = a * (row0 + idx + 1)[None] + b * torch.einsum("gim,gim->gi", q, zcum)
        f = a * scum + b * torch.einsum("gim,gimj->gij", q, Scum)
        return f / g[..., None], g

    def backward_shard_state(self, q, o, omega, g):
        wh = omega / g[..., None]
        s = (o * wh).sum(-1)
        return self._rec(torch.einsum("gim,gij->gmj", q, wh), torch.einsum("gi,gim->gm", s, q), wh.sum(1),
                         q.shape[1])

    def backward_with_carry(self, q, k, v, o, omega, g, carry_prefix, carry_suffix, row0):
        a, b = self.a, self.b
        D = q.shape[2]
        Sc, zc, _ = self._unrec(carry_prefix, D)
        Rc, uc, cc = self._unrec(carry_suffix, D)
        wh = omega / g[..., None]
        s = (o * wh).sum(-1)
        Scum = Sc[:, None] + torch.cumsum(torch.einsum("gtm,gtj->gtmj", k, v), 1)
        zcum = zc[:, None] + torch.cumsum(k, 1)
        rev = lambda x: torch.flip(torch.cumsum(torch.flip(x, [1]), 1), [1])
        Rcum = Rc[:, None] + rev(torch.einsum("gim,gij->gimj", q, wh))
        ucum = uc[:, None] + rev(s[..., None] * q)
        ccum = cc[:, None] + rev(wh)
        dq = b * (torch.einsum("gij,gimj->gim", wh, Scum) - s[..., None] * zcum)
        dk = b * (torch.einsum("gij,gimj->gim", v, Rcum) - ucum)
        dv = a * ccum + b * torch.einsum("gim,gimj->gij", k, Rcum)
        return dq, dk, dv


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _worker(rank, world, port, q, k, v, w, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = q.shape[1]
        sh = S.SequenceShard(N, rank, world, align=8)
        sl = slice(sh.row0, sh.row1)
        ops = CpuOps()
        qs, ks, vs, ws_ = (torch.as_tensor(x[:, sl]) for x in (q, k, v, w))
        out, g, carry = S.sequence_sharded_forward(ops, sh, qs, ks, vs)
        dq, dk, dv = S.sequence_sharded_backward(ops, sh, qs, ks, vs, out, ws_, g, carry)
        results[rank] = tuple(x.numpy() for x in (out, g, dq, dk, dv))
    finally:
        dist.destroy_process_group()


def test_sequence_sharding_exchange_gloo_world2():
    import torch.multiprocessing as mp
    G, N, D = 2, 40, 6
    q = O.normalize_rows(O.seeded(G, N, D, 1, O.SEQUENCE_MAJOR))
    k = O.normalize_rows(O.seeded(G, N, D, 2, O.SEQUENCE_MAJOR))
    v = O.seeded(G, N, D, 3, O.FEATURE_MAJOR)
    w = O.seeded(G, N, D, 4, O.FEATURE_MAJOR)
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q, k, v, w, results), nprocs=2, join=True)
    out = np.concatenate([results[r][0] for r in range(2)], 1)
    g = np.concatenate([results[r][1] for r in range(2)], 1)
    ro, rg = O.forward(q, k, v)
    assert max_abs(out, ro) < 1e-12 and max_abs(g, rg) < 1e-12
    dq = np.concatenate([results[r][2] for r in range(2)], 1)
    dk = np.concatenate([results[r][3] for r in range(2)], 1)
    dv = np.concatenate([results[r][4] for r in range(2)], 1)
    rq, rk, rv = O.backward(q, k, v, ro, w, rg)
    assert max_abs(dq, rq) < 1e-12 and max_abs(dk, rk) < 1e-12 and max_abs(dv, rv) < 1e-12


def test_batch_head_ranges_cover_groups():
    for G in (1, 7, 64, 128):
        for world in (1, 2, 4, 8):
            rs = [S.batch_head_range(G, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == G
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_sequence_shards_partition_rows():
    for N in (1024, 4096, 1 << 20):
        for world in (1, 2, 4, 8):
            sh = [S.SequenceShard(N, r, world) for r in range(world)]
            assert sh[0].row0 == 0 and sh[-1].row1 == N
            assert all(sh[i].row1 == sh[i + 1].row0 for i in range(world - 1))
            assert all(x.row0 % 128 == 0 for x in sh)


# ---------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("impl,save", [("auto", False), ("auto", True), ("simt", False)])
@pytest.mark.parametrize("world", [2, 4])
def test_sequence_sharding_carries_on_device(cuda, impl, save, world):
    """P shards run one after another on one GPU through the C-ABI carries (save: the
    carried forward's segment states feed the carried backward)."""
    G, N, D = 4, 2048, 128
    q, k, v, w = fast_inputs(G, N, D, seed=world)
    tb = lambda x: torch.as_tensor(x).to(torch.bfloat16)
    qb, kb, vb, wb = (tb(x) for x in (q, k, v, w))
    rq, rk, rv, rw = (x.double().numpy() for x in (qb, kb, vb, wb))
    shards = [S.SequenceShard(N, r, world) for r in range(world)]
    opss, ins, fstates = [], [], []
    for sh in shards:
        rows = sh.row1 - sh.row0
        ops = S.CudaOps(G, rows, D, "bf16", impl=impl)
        sl = slice(sh.row0, sh.row1)
        qs = qb[:, sl].contiguous().to(cuda)
        ks = kb[:, sl].contiguous().to(cuda)
        vs = vb[:, sl].transpose(1, 2).contiguous().to(cuda)   # FeatureMajor shard
        ws_ = wb[:, sl].transpose(1, 2).contiguous().to(cuda)
        opss.append(ops)
        ins.append((qs, ks, vs, ws_))
        fstates.append(ops.forward_shard_state(ks, vs))
    gathered = torch.stack(fstates)
    outs, gs, carries, saves = [], [], [], []
    for r, sh in enumerate(shards):
        carry = S.exclusive_prefix(gathered, r)
        qs, ks, vs, _ = ins[r]
        if save:
            out, g, sv = opss[r].forward_with_carry(qs, ks, vs, carry, sh.row0, save=True)
            saves.append(sv)
        else:
            out, g = opss[r].forward_with_carry(qs, ks, vs, carry, sh.row0)
            saves.append(None)
        outs.append(out)
        gs.append(g)
        carries.append(carry)
    out = torch.cat([o.view(G, D, -1) for o in outs], 2).transpose(1, 2).double().cpu().numpy()
    g = torch.cat([x.view(G, -1) for x in gs], 1).cpu().numpy()
    ro, rg = O.forward(rq, rk, rv)
    assert max_abs(out, ro) <= 2e-2
    assert rel_err(g, rg) <= 1e-3
    bstates = [opss[r].backward_shard_state(ins[r][0], outs[r], ins[r][3], gs[r]) for r in range(world)]
    bg = torch.stack(bstates)
    grads = []
    for r, sh in enumerate(shards):
        qs, ks, vs, ws_ = ins[r]
        grads.append(opss[r].backward_with_carry(qs, ks, vs, outs[r], ws_, gs[r], carries[r],
                                                 S.exclusive_suffix(bg, r), sh.row0, saved=saves[r]))
    dq = torch.cat([x[0].view(G, -1, D) for x in grads], 1).double().cpu().numpy()
    dk = torch.cat([x[1].view(G, D, -1) for x in grads], 2).transpose(1, 2).double().cpu().numpy()
    dv = torch.cat([x[2].view(G, D, -1) for x in grads], 2).transpose(1, 2).double().cpu().numpy()
    oq, ok_, ov = O.backward(rq, rk, rv, out, rw, g)
    assert max_abs(dq, oq) <= 2e-2 and max_abs(dk, ok_) <= 2e-2 and max_abs(dv, ov) <= 2e-2


@pytest.mark.gpu
def test_shard_states_tensor_core_match_simt(cuda):
    """la_forward_shard_state / la_backward_shard_state: the tcgen05 totals (aggregate
    kernels + unit sums) equal the CUDA-core totals (same records, fp32)."""
    G, N, D = 3, 1024, 128
    q, k, v, w = fast_inputs(G, N, D, seed=11)
    tb = lambda x: torch.as_tensor(x).to(torch.bfloat16).to(cuda)
    qs, ks = tb(q), tb(k)
    vs, ws_ = tb(v.transpose(0, 2, 1)), tb(w.transpose(0, 2, 1))
    tc, si = S.CudaOps(G, N, D, "bf16", impl="auto"), S.CudaOps(G, N, D, "bf16", impl="simt")
    f_tc, f_si = tc.forward_shard_state(ks, vs), si.forward_shard_state(ks, vs)
    out, g = tc.forward_with_carry(qs, ks, vs, torch.zeros_like(f_tc), 0)
    b_tc, b_si = tc.backward_shard_state(qs, out, ws_, g), si.backward_shard_state(qs, out, ws_, g)
    torch.cuda.synchronize()
    SZ = f_tc.numel() // G
    for name, a_, b_ in (("fwd", f_tc, f_si), ("bwd", b_tc, b_si)):
        a_, b_ = a_.double().cpu().numpy().reshape(G, SZ), b_.double().cpu().numpy().reshape(G, SZ)
        d = np.abs(a_ - b_)
        where = np.unravel_index(np.argmax(d), d.shape)
        # the tensor-core sums take W_hat in bf16 (the MMA operand): 2e-2 of the record scale
        assert d.max() <= 2e-2 * max(1.0, np.abs(b_[:, :-4]).max()), (name, d.max(), where, a_[where], b_[where])
