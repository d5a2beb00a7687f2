// Multi-GPU entry points (include/la_cuda.h: la_sharded_forward / la_sharded_backward).
//
// The reference runs every group on one machine (run_forward / run_backward,
// forward_kernels.hpp:210-259, backward_kernels.hpp:292-396); groups are independent
// (forward_kernels.hpp:221-235) and, within a group, the causal sweep only couples rows
// through the running states. So one process per GPU shards either
//   * whole groups (batch x head): the local call is the single-GPU call, no collective;
//   * rows of every group (sequence): each rank reduces its rows to one state record per
//     group (forward: S = sum k^T v, z, sigma, rows; backward: R = sum q^T w_hat, u, c),
//     the records are all-gathered (ncclAllGather, ~1 MB at 16 heads, D = 128) and the
//     exclusive prefix (forward) / suffix (backward) becomes the local sweep's carry.
// NCCL is loaded with dlopen at first use, so the library loads (and the single-GPU
// path runs) on hosts without it; a caller-supplied all-gather can replace it.
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/la_cuda.h"
#include "internal.h"

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's NCCL if one is loaded already (e.g. torch's), else the system's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    if (api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather) api.handle = h;
  });
  return api.handle ? &api : nullptr;
}

la_status fail(la_error_info* err, la_status code, const char* msg) {
  if (err) {
    err->code = code;
    err->group = err->position = -1;
    std::snprintf(err->message, sizeof(err->message), "%s", msg);
  }
  return code;
}

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

bool dist_ok(const la_dist* d) {
  return d && (d->mode == LA_SHARD_BATCH_HEAD || d->mode == LA_SHARD_SEQUENCE) && d->nranks >= 1 &&
         d->rank >= 0 && d->rank < d->nranks && d->row_offset >= 0;
}

// Workspace carving for the sequence mode: [pass workspace | state | gathered | carry | scratch].
struct DistWs {
  char* pass;
  size_t pass_bytes;
  float* state;
  float* gathered;
  float* carry;
  void* scratch;
  size_t scratch_bytes;
};
size_t rec_bytes(const la_problem* p) { return la_shard_state_floats(p) * sizeof(float); }
size_t pass_bytes(const la_problem* p) {
  return a256(std::max(la_forward_workspace_bytes(p), la_backward_workspace_bytes(p)));
}
DistWs carve(const la_problem* p, const la_dist* d, void* ws) {
  DistWs w;
  char* c = (char*)ws;
  w.pass = c;
  w.pass_bytes = pass_bytes(p);
  c += w.pass_bytes;
  w.state = (float*)c;
  c += a256(rec_bytes(p));
  w.gathered = (float*)c;
  c += a256(rec_bytes(p) * (size_t)d->nranks);
  w.carry = (float*)c;
  c += a256(rec_bytes(p));
  w.scratch = c;
  w.scratch_bytes = la_shard_state_workspace_bytes(p);
  return w;
}

la_status all_gather(const la_dist* d, const float* send, float* recv, size_t count, void* stream,
                     la_error_info* err) {
  struct Range {
    Range() { nvtxRangePushA("sharded.all_gather"); }
    ~Range() { nvtxRangePop(); }
  } range;
  if (d->nccl_comm) {
    const NcclApi* api = nccl();
    if (!api) return fail(err, LA_ERR_UNSUPPORTED, "libnccl.so.2 not found");
    const ncclResult_t r = api->all_gather(send, recv, count, ncclFloat32, (ncclComm_t)d->nccl_comm,
                                           (cudaStream_t)stream);
    if (r != ncclSuccess) {
      char msg[200];
      std::snprintf(msg, sizeof(msg), "ncclAllGather failed: %s", api->error_string ? api->error_string(r) : "?");
      return fail(err, LA_ERR_CUDA, msg);
    }
    return LA_OK;
  }
  if (d->allgather) {
    if (d->allgather(send, recv, count, d->allgather_ctx, stream) != 0)
      return fail(err, LA_ERR_CUDA, "all-gather callback failed");
    return LA_OK;
  }
  if (d->nranks == 1)  // a single shard gathers its own record
    return cudaMemcpyAsync(recv, send, count * sizeof(float), cudaMemcpyDeviceToDevice, (cudaStream_t)stream) ==
                   cudaSuccess
               ? LA_OK
               : fail(err, LA_ERR_CUDA, "record copy failed");
  return fail(err, LA_ERR_INVALID_ARGUMENT, "sequence sharding over several ranks needs nccl_comm or allgather");
}

}  // namespace

extern "C" {

size_t la_dist_saved_bytes(const la_problem* p, const la_dist* d) {
  (void)d;
  if (!p) return 0;
  return a256(la_saved_state_bytes(p)) + a256(rec_bytes(p));  // + the forward carry
}

size_t la_dist_workspace_bytes(const la_problem* p, const la_dist* d) {
  if (!p || !dist_ok(d)) return 0;
  if (d->mode == LA_SHARD_BATCH_HEAD) return pass_bytes(p);
  return pass_bytes(p) + a256(rec_bytes(p)) * (size_t)(2 + d->nranks) + la_shard_state_workspace_bytes(p);
}

la_status la_sharded_forward(const la_problem* p, const la_dist* d, const void* q, la_layout lq, const void* k,
                             la_layout lk, const void* v, la_layout lv, void* out, float* g, void* saved,
                             size_t saved_bytes, void* workspace, size_t ws_bytes, void* stream,
                             la_error_info* err) {
  if (!p) return fail(err, LA_ERR_INVALID_ARGUMENT, "null problem");
  if (!dist_ok(d)) return fail(err, LA_ERR_INVALID_ARGUMENT, "invalid la_dist (mode, rank, nranks, row_offset)");
  if (!saved || saved_bytes < la_dist_saved_bytes(p, d))
    return fail(err, LA_ERR_WORKSPACE, "saved buffer smaller than la_dist_saved_bytes");
  if (!workspace || ws_bytes < la_dist_workspace_bytes(p, d))
    return fail(err, LA_ERR_WORKSPACE, "workspace smaller than la_dist_workspace_bytes");
  const size_t sv = la_saved_state_bytes(p);
  if (d->mode == LA_SHARD_BATCH_HEAD)
    return la_forward_save(p, q, lq, k, lk, v, lv, out, g, saved, sv, workspace, pass_bytes(p), stream, err);
  if (!p->causal) return fail(err, LA_ERR_UNSUPPORTED, "sequence sharding is defined for the causal mask");
  if (d->nranks == 1) {  // the whole sequence: nothing to exchange, a zero carry
    const la_shard sh{d->row_offset, nullptr, nullptr};
    cudaMemsetAsync((char*)saved + a256(sv), 0, rec_bytes(p), (cudaStream_t)stream);
    return la_forward_sharded_save(p, &sh, q, lq, k, lk, v, lv, out, g, saved, sv, workspace, pass_bytes(p), stream,
                                   err);
  }
  DistWs w = carve(p, d, workspace);
  float* carry = (float*)((char*)saved + a256(sv));
  la_status s = la_forward_shard_state(p, k, lk, v, lv, w.state, w.scratch, w.scratch_bytes, stream);
  if (s != LA_OK) return fail(err, s, "forward shard totals failed");
  const size_t n = la_shard_state_floats(p);
  if ((s = all_gather(d, w.state, w.gathered, n, stream, err)) != LA_OK) return s;
  s = la_combine_shard_states(p, w.gathered, d->nranks, d->rank, 0, carry, stream);
  if (s != LA_OK) return fail(err, s, "prefix combine failed");
  const la_shard sh{d->row_offset, carry, nullptr};
  return la_forward_sharded_save(p, &sh, q, lq, k, lk, v, lv, out, g, saved, sv, w.pass, w.pass_bytes, stream, err);
}

la_status la_sharded_backward(const la_problem* p, const la_dist* d, const void* q, la_layout lq, const void* k,
                              la_layout lk, const void* v, la_layout lv, const void* o, const void* omega,
                              la_layout lw, const float* g, const void* saved, size_t saved_bytes, void* dq,
                              void* dk, void* dv, void* workspace, size_t ws_bytes, void* stream,
                              la_error_info* err) {
  if (!p) return fail(err, LA_ERR_INVALID_ARGUMENT, "null problem");
  if (!dist_ok(d)) return fail(err, LA_ERR_INVALID_ARGUMENT, "invalid la_dist (mode, rank, nranks, row_offset)");
  if (!saved || saved_bytes < la_dist_saved_bytes(p, d))
    return fail(err, LA_ERR_MISSING_FORWARD_STATE, "backward requires the la_sharded_forward artifacts");
  if (!workspace || ws_bytes < la_dist_workspace_bytes(p, d))
    return fail(err, LA_ERR_WORKSPACE, "workspace smaller than la_dist_workspace_bytes");
  const size_t sv = la_saved_state_bytes(p);
  if (d->mode == LA_SHARD_BATCH_HEAD)
    return la_backward_saved(p, q, lq, k, lk, v, lv, o, omega, lw, g, saved, sv, dq, dk, dv, workspace,
                             pass_bytes(p), stream, err);
  if (!p->causal) return fail(err, LA_ERR_UNSUPPORTED, "sequence sharding is defined for the causal mask");
  if (d->nranks == 1) {
    const la_shard sh{d->row_offset, nullptr, nullptr};
    return la_backward_sharded_saved(p, &sh, q, lq, k, lk, v, lv, o, omega, lw, g, saved, sv, dq, dk, dv, workspace,
                                     pass_bytes(p), stream, err);
  }
  DistWs w = carve(p, d, workspace);
  const float* carry_prefix = (const float*)((const char*)saved + a256(sv));
  la_status s = la_backward_shard_state(p, q, lq, o, omega, lw, g, w.state, w.scratch, w.scratch_bytes, stream);
  if (s != LA_OK) return fail(err, s, "backward shard totals failed");
  const size_t n = la_shard_state_floats(p);
  if ((s = all_gather(d, w.state, w.gathered, n, stream, err)) != LA_OK) return s;
  s = la_combine_shard_states(p, w.gathered, d->nranks, d->rank, 1, w.carry, stream);
  if (s != LA_OK) return fail(err, s, "suffix combine failed");
  const la_shard sh{d->row_offset, carry_prefix, w.carry};
  return la_backward_sharded_saved(p, &sh, q, lq, k, lk, v, lv, o, omega, lw, g, saved, sv, dq, dk, dv, w.pass,
                                   w.pass_bytes, stream, err);
}

la_status la_nccl_get_unique_id(char* id) {
  const NcclApi* api = nccl();
  if (!api) return LA_ERR_UNSUPPORTED;
  if (!id) return LA_ERR_INVALID_ARGUMENT;
  ncclUniqueId u;
  if (api->get_unique_id(&u) != ncclSuccess) return LA_ERR_CUDA;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return LA_OK;
}

la_status la_nccl_comm_init(void** comm, int32_t nranks, const char* id, int32_t rank) {
  const NcclApi* api = nccl();
  if (!api) return LA_ERR_UNSUPPORTED;
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return LA_ERR_INVALID_ARGUMENT;
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  if (api->comm_init_rank(&c, nranks, u, rank) != ncclSuccess) return LA_ERR_CUDA;
  *comm = c;
  return LA_OK;
}

la_status la_nccl_comm_destroy(void* comm) {
  const NcclApi* api = nccl();
  if (!api) return LA_ERR_UNSUPPORTED;
  if (!comm) return LA_ERR_INVALID_ARGUMENT;
  return api->comm_destroy((ncclComm_t)comm) == ncclSuccess ? LA_OK : LA_ERR_CUDA;
}

}  // extern "C"
