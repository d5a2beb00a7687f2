"""Multi-GPU C-ABI entry points: la_sharded_forward / la_sharded_backward (la_dist.cu).

* CPU: the entry points exist, size their buffers, and reject bad sharding
  descriptions without touching a device.
* GPU, world size 2 over gloo: two processes share cuda:0 (NCCL refuses two ranks on
  one GPU, so the library's caller-supplied all-gather carries the exchange), each runs
  its shard through the C-ABI -- shard totals, all-gather, prefix / suffix combine and
  the carried tensor-core sweeps all inside the library -- and the concatenated shards
  match the f64 oracle within the bf16 bar.
* GPU, NCCL: the same entry points with a real ncclComm_t (la_nccl_comm_init) at one
  rank, both modes, equal to the single-GPU call.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2510_21956_b200 import _abi
from paper_2510_21956_b200 import sharding as S
from tests._util import fast_inputs, max_abs


def _dist(mode, rank, nranks, row_offset=0):
    d = _abi.Dist()
    d.mode, d.rank, d.nranks, d.row_offset = mode, rank, nranks, row_offset
    return d


def test_dist_sizes_and_validation():
    L = _abi.lib()
    p = _abi.make_problem(16, 131072, 128, "bf16")
    bh = _dist(_abi.SHARD_BATCH_HEAD, 0, 8)
    sq = _dist(_abi.SHARD_SEQUENCE, 3, 8, 3 * 131072)
    # batch x head: exactly the single-GPU workspace; sequence: + state, gathered, carry, scratch
    wb = L.la_dist_workspace_bytes(C.byref(p), C.byref(bh))
    ws = L.la_dist_workspace_bytes(C.byref(p), C.byref(sq))
    rec = L.la_shard_state_floats(C.byref(p)) * 4
    assert wb >= max(L.la_forward_workspace_bytes(C.byref(p)), L.la_backward_workspace_bytes(C.byref(p)))
    assert ws >= wb + (2 + 8) * rec + L.la_shard_state_workspace_bytes(C.byref(p))
    assert L.la_dist_saved_bytes(C.byref(p), C.byref(sq)) >= L.la_saved_state_bytes(C.byref(p)) + rec
    # invalid descriptions fail synchronously, before any device work
    err = _abi.ErrorInfo()
    bad = _dist(_abi.SHARD_SEQUENCE, 8, 8)
    rc = L.la_sharded_forward(C.byref(p), C.byref(bad), 1, 1, 1, 1, 1, 0, 1, 1, 1, 1 << 40, 1, 1 << 40, None,
                              C.byref(err))
    assert _abi.STATUS_NAMES[rc] == "InvalidArgument"
    rc = L.la_sharded_forward(C.byref(p), C.byref(sq), 1, 1, 1, 1, 1, 0, 1, 1, 1, 16, 1, 1 << 40, None,
                              C.byref(err))
    assert _abi.STATUS_NAMES[rc] == "WorkspaceError"
    rc = L.la_sharded_backward(C.byref(p), C.byref(sq), 1, 1, 1, 1, 1, 0, 1, 1, 0, 1, None, 0, 1, 1, 1, 1,
                               1 << 40, None, C.byref(err))
    assert _abi.STATUS_NAMES[rc] == "MissingForwardState"


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _inputs(G, N, D, seed):
    q, k, v, w = fast_inputs(G, N, D, seed=seed)
    tb = lambda x: torch.as_tensor(x).to(torch.bfloat16)
    return tuple(tb(x) for x in (q, k, v, w))


def _worker(rank, world, port, mode, G, N, D, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda:0")
        qb, kb, vb, wb = _inputs(G, N, D, 7)
        if mode == "sequence":
            sh = S.SequenceShard(N, rank, world)
            sl, gs, rows, row0 = slice(sh.row0, sh.row1), slice(0, G), sh.row1 - sh.row0, sh.row0
        else:
            g0, g1 = S.batch_head_range(G, rank, world)
            sl, gs, rows, row0 = slice(0, N), slice(g0, g1), N, 0
        ng = gs.stop - gs.start
        qs = qb[gs, sl].contiguous().to(dev)
        ks = kb[gs, sl].contiguous().to(dev)
        vs = vb[gs, sl].transpose(1, 2).contiguous().to(dev)
        ws_ = wb[gs, sl].transpose(1, 2).contiguous().to(dev)
        step = S.DistStep(ng, rows, D, mode, rank, world, row_offset=row0, allgather=S.host_allgather())
        out, g, saved = step.forward(qs, ks, vs)
        dq, dk, dv = step.backward(qs, ks, vs, out, ws_, g, saved)
        torch.cuda.synchronize()
        f = lambda x, shape: x.view(shape).float().cpu().numpy()
        results[rank] = (f(out, (ng, D, rows)), f(g, (ng, rows)), f(dq, (ng, rows, D)), f(dk, (ng, D, rows)),
                         f(dv, (ng, D, rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["sequence", "batch_head"])
def test_sharded_entry_points_world2_one_gpu(cuda, mode):
    import torch.multiprocessing as mp
    G, N, D, world = 4, 8192, 128, 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), mode, G, N, D, results), nprocs=world, join=True)
    ax = {"sequence": (2, 1, 1, 2, 2), "batch_head": (0, 0, 0, 0, 0)}[mode]
    out, g, dq, dk, dv = (np.concatenate([results[r][i] for r in range(world)], ax[i]) for i in range(5))
    qb, kb, vb, wb = _inputs(G, N, D, 7)
    rq, rk, rv, rw = (x.double().numpy() for x in (qb, kb, vb, wb))
    for grp in (0, G - 1):  # f64 oracle on two groups
        sl = slice(grp, grp + 1)
        ro, rg = O.forward(rq[sl], rk[sl], rv[sl])
        o_dev = out[sl].transpose(0, 2, 1).astype(np.float64)
        assert max_abs(o_dev, ro) <= 2e-2
        assert np.max(np.abs(g[sl] - rg) / np.abs(rg)) <= 1e-3
        oq, ok_, ov = O.backward(rq[sl], rk[sl], rv[sl], o_dev, rw[sl], g[sl].astype(np.float64))
        assert max_abs(dq[sl], oq) <= 2e-2
        assert max_abs(dk[sl].transpose(0, 2, 1), ok_) <= 2e-2
        assert max_abs(dv[sl].transpose(0, 2, 1), ov) <= 2e-2


def _nccl_worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda:0")
        G, N, D = 4, 4096, 128
        qb, kb, vb, wb = _inputs(G, N, D, 3)
        qs, ks = qb.contiguous().to(dev), kb.contiguous().to(dev)
        vs, ws_ = vb.transpose(1, 2).contiguous().to(dev), wb.transpose(1, 2).contiguous().to(dev)
        comm = S.nccl_comm(rank, world)
        res = {}
        for mode in ("sequence", "batch_head"):
            step = S.DistStep(G, N, D, mode, rank, world, comm=comm)
            out, g, saved = step.forward(qs, ks, vs)
            grads = step.backward(qs, ks, vs, out, ws_, g, saved)
            res[mode] = [x.float().cpu().numpy() for x in (out, g, *grads)]
        # the single-GPU entry points on the same data
        p = _abi.make_problem(G, N, D, "bf16")
        L = _abi.lib()
        out, g = torch.empty_like(vs), torch.empty(G * N, device=dev)
        sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        wf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        wk = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
        assert L.la_forward_save(C.byref(p), qs.data_ptr(), 1, ks.data_ptr(), 1, vs.data_ptr(), 0, out.data_ptr(),
                                 g.data_ptr(), sv.data_ptr(), sv.numel(), wf.data_ptr(), wf.numel(), None, None) == 0
        dq, dk, dv = torch.empty_like(qs), torch.empty_like(vs), torch.empty_like(vs)
        assert L.la_backward_saved(C.byref(p), qs.data_ptr(), 1, ks.data_ptr(), 1, vs.data_ptr(), 0, out.data_ptr(),
                                   ws_.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(),
                                   dk.data_ptr(), dv.data_ptr(), wk.data_ptr(), wk.numel(), None, None) == 0
        torch.cuda.synchronize()
        res["single"] = [x.float().cpu().numpy() for x in (out, g, dq, dk, dv)]
        results[rank] = res
        _abi.lib().la_nccl_comm_destroy(comm)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_entry_points_nccl_one_rank(cuda):
    """ncclAllGather inside la_sharded_forward / _backward (one rank): bitwise the
    single-GPU call for both modes (a one-rank exchange gives a zero carry)."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, _free_port(), results), nprocs=1, join=True)
    res = results[0]
    for mode in ("sequence", "batch_head"):
        for a_, b_ in zip(res[mode], res["single"]):
            assert np.array_equal(a_, b_), mode
