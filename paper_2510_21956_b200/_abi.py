"""ctypes binding of include/la_cuda.h (libla_cuda.so, built in-tree).

The product path is this library; there is no CPU fallback. If the shared
object is missing the import fails loudly (run ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LA_CUDA_LIB") or os.path.join(PKG, "libla_cuda.so")  # override: A/B builds

# enums (la_cuda.h)
LA_OK = 0
STATUS_NAMES = {0: "ok", 1: "InvalidShape", 2: "ShapeMismatch", 3: "InvalidArgument", 4: "InvalidPlan",
                5: "MissingForwardState", 6: "DegenerateDenominator", 7: "CudaError", 8: "Unsupported",
                9: "WorkspaceError"}
FEATURE_MAJOR, SEQUENCE_MAJOR = 0, 1
DTYPES = {"f32": 0, "bf16": 1, "f16": 2}
IMPLS = {"auto": 0, "simt": 1, "tcgen05": 2}

EXPORTS = [
    "la_version", "la_status_name", "la_forward_workspace_bytes", "la_backward_workspace_bytes",
    "la_shard_state_floats", "la_validate_plan", "la_default_plan", "la_launch_count", "la_forward",
    "la_backward", "la_forward_sharded", "la_backward_sharded", "la_forward_shard_state",
    "la_backward_shard_state", "la_combine_shard_states", "la_query_status", "la_host_forward",
    "la_host_backward", "la_host_step", "la_host_release", "la_profile_enable", "la_profile_read",
    "la_saved_state_bytes", "la_forward_save", "la_backward_saved",
    "la_normalize_qk", "la_relayout", "la_make_omega_hat", "la_constant_term_pass", "la_linear_term_pass",
    "la_alpha_term_pass", "la_beta_term_pass", "la_forward_sharded_save", "la_backward_sharded_saved",
    "la_set_tuning", "la_get_tuning", "la_shard_state_workspace_bytes", "la_dist_saved_bytes",
    "la_dist_workspace_bytes", "la_sharded_forward", "la_sharded_backward", "la_nccl_get_unique_id",
    "la_nccl_comm_init", "la_nccl_comm_destroy",
]


class BlockPlan(C.Structure):
    """la_block_plan == la::BlockPlan (plan.hpp:15-21)."""
    _fields_ = [("groups", C.c_int64), ("reduction_blocks", C.c_int64), ("lanes", C.c_int64),
                ("workers", C.c_int32), ("deterministic", C.c_int32)]


class Problem(C.Structure):
    _fields_ = [("groups", C.c_int64), ("seq_len", C.c_int64), ("dim", C.c_int64), ("dtype", C.c_int),
                ("a", C.c_double), ("b", C.c_double), ("causal", C.c_int32), ("fault", C.c_int),
                ("impl", C.c_int), ("plan", BlockPlan)]


class ErrorInfo(C.Structure):
    _fields_ = [("code", C.c_int), ("group", C.c_int64), ("position", C.c_int64),
                ("message", C.c_char * 256)]


class Tuning(C.Structure):
    """la_tuning: measurement overrides of the schedule rules (0 = built-in rule)."""
    _fields_ = [(n, C.c_int32) for n in ("segments", "agg_split", "full_ctas_fwd", "full_ctas_bwd", "prefetch",
                                         "host_blocks", "simt_seg_rows", "bwd_pair")]


class Shard(C.Structure):
    _fields_ = [("row_offset", C.c_int64), ("carry_in", C.c_void_p), ("carry_suffix", C.c_void_p)]


SHARD_BATCH_HEAD, SHARD_SEQUENCE = 0, 1
# int (*)(const float* send, float* recv, size_t count, void* ctx, void* stream)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class Dist(C.Structure):
    """la_dist: the multi-GPU entry points' sharding description."""
    _fields_ = [("mode", C.c_int), ("rank", C.c_int32), ("nranks", C.c_int32), ("row_offset", C.c_int64),
                ("nccl_comm", C.c_void_p), ("allgather", ALLGATHER_FN), ("allgather_ctx", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first "
                              "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        vp, i64, sz = C.c_void_p, C.c_int64, C.c_size_t
        P, E = C.POINTER(Problem), C.POINTER(ErrorInfo)
        L.la_version.restype = C.c_char_p
        L.la_status_name.restype = C.c_char_p
        L.la_forward_workspace_bytes.restype = sz
        L.la_forward_workspace_bytes.argtypes = [P]
        L.la_backward_workspace_bytes.restype = sz
        L.la_backward_workspace_bytes.argtypes = [P]
        L.la_shard_state_floats.restype = sz
        L.la_shard_state_floats.argtypes = [P]
        L.la_validate_plan.argtypes = [C.POINTER(BlockPlan), i64, i64, E]
        L.la_default_plan.argtypes = [i64, i64, C.c_int32, C.POINTER(BlockPlan)]
        L.la_launch_count.restype = C.c_uint64
        L.la_profile_enable.argtypes = [C.c_int32]
        L.la_profile_read.argtypes = [C.c_char_p, sz]
        L.la_profile_read.restype = C.c_int32
        L.la_forward.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, sz, vp, E]
        L.la_backward.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, vp, vp,
                                  vp, vp, vp, sz, vp, E]
        L.la_forward_sharded.argtypes = [P, C.POINTER(Shard), vp, C.c_int, vp, C.c_int, vp, C.c_int,
                                         vp, vp, vp, sz, vp, E]
        L.la_backward_sharded.argtypes = [P, C.POINTER(Shard), vp, C.c_int, vp, C.c_int, vp, C.c_int,
                                          vp, vp, C.c_int, vp, vp, vp, vp, vp, sz, vp, E]
        L.la_shard_state_workspace_bytes.restype = sz
        L.la_shard_state_workspace_bytes.argtypes = [P]
        L.la_forward_shard_state.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, vp, sz, vp]
        L.la_backward_shard_state.argtypes = [P, vp, C.c_int, vp, vp, C.c_int, vp, vp, vp, sz, vp]
        Dp = C.POINTER(Dist)
        L.la_dist_saved_bytes.restype = sz
        L.la_dist_saved_bytes.argtypes = [P, Dp]
        L.la_dist_workspace_bytes.restype = sz
        L.la_dist_workspace_bytes.argtypes = [P, Dp]
        L.la_sharded_forward.argtypes = [P, Dp, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, sz, vp, sz,
                                         vp, E]
        L.la_sharded_backward.argtypes = [P, Dp, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, vp, vp,
                                          sz, vp, vp, vp, vp, sz, vp, E]
        L.la_nccl_get_unique_id.argtypes = [C.c_char_p]
        L.la_nccl_comm_init.argtypes = [C.POINTER(vp), C.c_int32, C.c_char_p, C.c_int32]
        L.la_nccl_comm_destroy.argtypes = [vp]
        L.la_combine_shard_states.argtypes = [P, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp]
        L.la_query_status.argtypes = [vp, vp, E]
        L.la_saved_state_bytes.restype = sz
        L.la_saved_state_bytes.argtypes = [P]
        L.la_forward_save.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, sz, vp, sz, vp, E]
        L.la_backward_saved.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, vp, vp, sz,
                                        vp, vp, vp, vp, sz, vp, E]
        L.la_host_forward.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, E]
        L.la_host_step.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp,
                                   vp, E]
        L.la_host_backward.argtypes = [P, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, vp,
                                       vp, vp, vp, E]
        ci = C.c_int
        L.la_forward_sharded_save.argtypes = [P, C.POINTER(Shard), vp, ci, vp, ci, vp, ci, vp, vp, vp, sz, vp, sz,
                                              vp, E]
        L.la_backward_sharded_saved.argtypes = [P, C.POINTER(Shard), vp, ci, vp, ci, vp, ci, vp, vp, ci, vp, vp,
                                                sz, vp, vp, vp, vp, sz, vp, E]
        L.la_normalize_qk.argtypes = [P, vp, ci, vp, ci, vp, vp, vp, E]
        L.la_relayout.argtypes = [P, vp, ci, vp, ci, vp, E]
        L.la_make_omega_hat.argtypes = [P, vp, ci, vp, vp, vp, E]
        L.la_constant_term_pass.argtypes = [P, vp, ci, vp, vp, E]
        L.la_linear_term_pass.argtypes = [P, vp, ci, vp, ci, vp, ci, vp, vp, E]
        L.la_alpha_term_pass.argtypes = [P, vp, ci, vp, ci, vp, ci, vp, vp, E]
        L.la_beta_term_pass.argtypes = [P, vp, ci, vp, ci, vp, ci, vp, vp, E]
        L.la_set_tuning.argtypes = [C.POINTER(Tuning)]
        L.la_set_tuning.restype = None
        L.la_get_tuning.argtypes = [C.POINTER(Tuning)]
        L.la_get_tuning.restype = None
        _lib = L
    return _lib


def set_tuning(**fields):
    """la_set_tuning with the named overrides (no arguments: the built-in rules)."""
    t = Tuning()
    for k, v in fields.items():
        setattr(t, k, int(v))
    lib().la_set_tuning(C.byref(t) if fields else None)


def profile_read():
    """Per-kernel device times recorded since the last read (la_profile_read)."""
    import json
    buf = C.create_string_buffer(1 << 20)
    lib().la_profile_read(buf, len(buf))
    return json.loads(buf.value.decode())


def make_problem(G, N, D, dtype="f32", a=1.0, b=1.0, causal=True, fault=0, impl="auto", plan=None):
    p = Problem()
    p.groups, p.seq_len, p.dim = G, N, D
    p.dtype = DTYPES[dtype]
    p.a, p.b = float(a), float(b)
    p.causal = 1 if causal else 0
    p.fault = int(fault)
    p.impl = IMPLS[impl]
    if plan is None:
        bp = BlockPlan()
        lib().la_default_plan(G, D, 1, C.byref(bp))
        p.plan = bp
    else:
        p.plan = plan
    return p
