// sm_100a tensor-core backward: chunked causal linear attention, f(x) = a + b*x.
//
// Replaces backward_kernels.hpp run_backward<T> (causal, D = 128): its four
// barrier-separated CPU sweeps (dQ prefix, dK alpha/beta suffix, dV suffix)
// become ONE reverse sweep per (group, segment) over chunks of C = 64 rows.
// With w_hat = omega / g and s_i = o_i . w_hat_i (backward_kernels.hpp:33-38):
//   dPt = W_hat V^T, T1 = Q K^T                          (M=64, lanes i)
//   dS  = b tril(dPt - s 1^T),  P = tril(a + b T1)       -> bf16 smem
//   dQ  = dS K + W_hat (b S_prev)^T - b s z_prev^T        (M=64, two lane halves)
//   dK^T = Q^T dS^T + (b R_next) V^T - b u_next           (M=128, lanes m)
//   dV^T = W_hat^T P + (b R_next)^T K^T + a c_next        (M=128, lanes j)
//   R += Q^T W_hat (suffix state, lanes m);  S -= K^T V (prefix state by
//   negated MMA from the segment-end prefix, lanes m); u, z, c on CUDA cores.
// The reference's beta^K state collapses to the D-vector u and beta^V aliases
// alpha^K = b R. TMEM holds exactly 512 columns:
//   [0,64) dPt (lanes 0-15,32-47,..) + T1 (other half), [64,128) dQ halves,
//   [128,192) dK^T, [192,256) dV^T, [256,384) R, [384,512) S.
// Segment carries: an aggregate pass (R, u, c and S, z per segment) + scan.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"
#include "bwd_tiles.cuh"

namespace lab {

using namespace sm100;

__device__ unsigned long long g_trace_b[4][64][10];
__device__ __forceinline__ void traceb(int role, int n, int ev) {
#ifndef LA_TRACE_G
#define LA_TRACE_G 0  // traced group (blockIdx.y) of segment 0
#endif
#ifdef LA_TRACE  // compiled out by default: the kernels are I-cache sensitive
  if (blockIdx.x == 0 && blockIdx.y == LA_TRACE_G && n < 64) g_trace_b[role][n][ev] = clock64();
#endif
}

namespace {

constexpr int kCB = 64;   // chunk rows
constexpr int kD = 128;   // head dim
constexpr int kT64 = 16384;  // a 64x128 or 128x64 16-bit tile
constexpr int kStage = 4 * kT64;  // Q, K, V^T, Omega^T
constexpr int kBPrefetch = 0;     // L2 prefetch distance (chunks); 0 = the chunk itself, before the slot wait (la_sm100.cu)
constexpr uint32_t kDP = 0, kDQ = 64, kDK = 128, kDV = 192, kR = 256, kS = 384;
constexpr uint32_t kHalf = 16u << 16;  // TMEM lane offset of the upper M=64 half

struct BwdParams {
  const void* o;         // O^T  [G][D][N]
  const float* g;        // [G][N]
  void* dq;              // [G][N][D]
  void* dk;              // [G][D][N]
  void* dv;              // [G][D][N]
  float* stS;            // per-segment S records (agg: out; main: inclusive prefix)
  float* stR;            // per-segment R records (agg: out; main: exclusive suffix)
  int64_t N;
  int64_t seg_len;
  int P;
  float a, b;
  int dbg;     // debug bitmask (LA_BWD_DEBUG): 1 skip dS K, 2 skip W_hat S^T
  int skipS;   // aggregate pass: S records come from the forward (la_backward_saved)
  int p0;      // aggregate pass: first unit of the grid
  int A;       // aggregate units per segment (records are per unit: [G][P * A])
  const float* carry_pre;  // sequence-shard carries (or null)
  const float* carry_suf;
  float* cmb;  // per (g, segment) combined [S inclusive prefix | R exclusive suffix]
  int pf;      // chunks prefetched into L2 ahead of the ring
  int store_w = 0;  // W_hat pass: store W_hat^T (into dv) and s (into dq rows) for the sweep
  int r_unit0 = 0;  // aggregate pass: units below this only produce W_hat^T / s (their R records
                    // would feed no segment: segment 0 in the causal sweep)
  const float* ck = nullptr;  // exact prefix (S, z) records the sweep reloads (internal.h, kCkC0):
  int ck_K = 0;               //   ck_unit == 0: [G][ck_K] at global rows C0 * 2^k (the forward's)
  int64_t row_offset = 0;     // global index of row 0 (sequence shards)
  int64_t ck_unit = 0;        //   ck_unit > 0: [G][P][A] at the segment's unit boundaries, built by
                              //   the sweep's prologue from the aggregate's unit sums (la_backward)
  int cmb_ready = 0;          // cmb (and the unit-boundary prefixes) already formed by seg_scan
};

// Half-tile variant: rows j = jbase + 16 rr + jg (rr < 4); the partial s of this
// half goes to s_half, and rs[rr] returns this thread's partial row sum of W_hat
// (its 8 columns of row j).
template <bool kBF16>
__device__ __forceinline__ void what_pass_half(uint8_t* w_t, const uint4 (&o4)[4], const float4 (&g8)[2],
                                               float* s_half, int et, int jbase, float (&rs)[4]) {
  const int lane = et & 31, w = et >> 5;
  const int jg = lane & 15, ig = 2 * w + (lane >> 4);
  float ginv[8] = {1.f / g8[0].x, 1.f / g8[0].y, 1.f / g8[0].z, 1.f / g8[0].w,
                   1.f / g8[1].x, 1.f / g8[1].y, 1.f / g8[1].z, 1.f / g8[1].w};
  float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int j = jbase + 16 * rr + jg;
    uint4* p = (uint4*)(w_t + sw128_off(j, 8 * ig, 128));
    const uint4 wv = *p;
    const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
    const uint32_t oa[4] = {o4[rr].x, o4[rr].y, o4[rr].z, o4[rr].w};
    uint32_t res[4];
    float rsum = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float2 wf = unpack2<kBF16>(wa[u]);
      const float2 of = unpack2<kBF16>(oa[u]);
      const float w0 = wf.x * ginv[2 * u], w1 = wf.y * ginv[2 * u + 1];
      sp[2 * u] += of.x * w0;
      sp[2 * u + 1] += of.y * w1;
      rsum += w0 + w1;
      res[u] = pack2<kBF16>(w0, w1);
    }
    rs[rr] = rsum;
    *p = make_uint4(res[0], res[1], res[2], res[3]);
  }
  // Reduce-scatter of the 8 partial sums over the 16 lanes sharing ig: each exchange
  // step halves the values a lane keeps (8 shuffles instead of 32). Afterwards lanes
  // jg and jg^1 hold the full sum of value (jg >> 1).
  const bool b3 = (jg & 8) != 0, b2 = (jg & 4) != 0, b1 = (jg & 2) != 0;
  float s4[4], s2v[2], s1v;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float mine = b3 ? sp[4 + k] : sp[k], other = b3 ? sp[k] : sp[4 + k];
    s4[k] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float mine = b2 ? s4[2 + k] : s4[k], other = b2 ? s4[k] : s4[2 + k];
    s2v[k] = mine + __shfl_xor_sync(0xffffffffu, other, 4);
  }
  {
    const float mine = b1 ? s2v[1] : s2v[0], other = b1 ? s2v[0] : s2v[1];
    s1v = mine + __shfl_xor_sync(0xffffffffu, other, 2);
  }
  s1v += __shfl_xor_sync(0xffffffffu, s1v, 1);
  if ((jg & 1) == 0) s_half[8 * ig + (jg >> 1)] = s1v;
}

template <bool kBF16>
__device__ __forceinline__ void what_prefetch_half(const BwdParams& prm, int64_t grp, int64_t row0, int et,
                                                   int jbase, uint4 (&o4)[4], float4 (&g8)[2]) {
  const int lane = et & 31, w = et >> 5;
  const int jg = lane & 15, ig = 2 * w + (lane >> 4);
  const uint16_t* o = (const uint16_t*)prm.o;
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
    o4[rr] = __ldg((const uint4*)(o + (grp * kD + jbase + 16 * rr + jg) * prm.N + row0 + 8 * ig));
  const float* gp = prm.g + grp * prm.N + row0 + 8 * ig;
  g8[0] = __ldg((const float4*)gp);
  g8[1] = __ldg((const float4*)(gp + 4));
}

// Prefetch of this thread's O^T slice (8 rows j x 8 columns i) and g for a chunk.
template <bool kBF16>
__device__ __forceinline__ void what_prefetch(const BwdParams& prm, int64_t grp, int64_t row0, int et,
                                              uint4 (&o8)[8], float4 (&g8)[2]) {
  const int lane = et & 31, w = et >> 5;
  const int jg = lane & 15, ig = 2 * w + (lane >> 4);
  const uint16_t* o = (const uint16_t*)prm.o;
#pragma unroll
  for (int rr = 0; rr < 8; ++rr)
    o8[rr] = __ldg((const uint4*)(o + (grp * kD + 16 * rr + jg) * prm.N + row0 + 8 * ig));
  const float* gp = prm.g + grp * prm.N + row0 + 8 * ig;
  g8[0] = __ldg((const float4*)gp);
  g8[1] = __ldg((const float4*)(gp + 4));
}

// ================================================================ aggregates
// Per (g, segment): S = sum k^T v, z = sum k (stS record); R = sum q^T w_hat,
// u = sum s q, c = sum w_hat (stR record). Record layout of internal.h.
template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    k_bwd_agg_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW,
                 BwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bars = (uint64_t*)(smem + 2 * kStage);
  uint64_t* full = bars;       // [2]
  uint64_t* empty = bars + 2;  // [2]
  uint64_t* w_ready = bars + 4;
  uint64_t* done = bars + 5;
  uint32_t* tslot = (uint32_t*)(bars + 8);
  float* s_s = (float*)(bars + 16);  // [64]

  const int p = blockIdx.x + prm.p0;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = (int)((s1 - s0) / kCB);
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmW);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 128);
    }
    mbar_init(w_ready, 128);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;  // [0,128) R, [128,256) S
  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c & 1;
        if (c >= 2) mbar_wait(&empty[s], ((c >> 1) & 1) ^ 1);
        const int64_t row0 = s0 + (int64_t)c * kCB;
        uint8_t* st = smem + s * kStage;
        mbar_expect_tx(&full[s], prm.skipS ? 2 * kT64 : kStage);
        tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * prm.N + row0), 0);
        if (!prm.skipS) {
          tma_load_3d(st + kT64, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 0);
          tma_load_3d(st + 2 * kT64, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        }
        tma_load_3d(st + 3 * kT64, &tmW, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t f = kBF16 ? 1 : 0;
    const uint32_t id_R = idesc_f16(128, 128, f, 1, 0);  // A = Q^T (MN), B = W_hat (K-major rows j)
    const uint32_t id_S = idesc_f16(128, 128, f, 1, 0);  // A = K^T (MN), B = V (K-major rows j)
    for (int c = 0; c < nc; ++c) {
      const int s = c & 1;
      const uint32_t st = smem_u32(smem + s * kStage);
      mbar_wait(&full[s], (c >> 1) & 1);
      tc_fence_after();
      if (!prm.skipS && elect_one()) {
        for (int ks = 0; ks < 4; ++ks)
          mma_ss(tmem + 128, mn(st + kT64, ks, 8192), kd(st + 2 * kT64, ks, 128), id_S,
                 (c > 0 || ks > 0) ? 1u : 0u);
      }
      __syncwarp();
      mbar_wait(w_ready, c & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 4; ++ks)
          mma_ss(tmem, mn(st, ks, 8192), kd(st + 3 * kT64, ks, 128), id_R, (c > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (c == nc - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    const int et = (int)threadIdx.x - 64;
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    float u = 0.f, z = 0.f, cc = 0.f;
    uint4 o8[8];
    float4 g8[2];
    if (nc > 0) what_prefetch<kBF16>(prm, grp, s0, et, o8, g8);
    for (int c = 0; c < nc; ++c) {
      const int s = c & 1;
      uint8_t* st = smem + s * kStage;
      named_bar(1, 128);  // previous chunk's s_s readers are done
      mbar_wait(&full[s], (c >> 1) & 1);
      what_pass<kBF16>(st + 3 * kT64, o8, g8, s_s, et);
      if (c + 1 < nc) what_prefetch<kBF16>(prm, grp, s0 + (int64_t)(c + 1) * kCB, et, o8, g8);
      fence_proxy_async();
      mbar_arrive(w_ready);
      named_bar(1, 128);  // s_s and W_hat complete
      // u_m += sum_i q_im s_i ; z_m += sum_t k_tm   (m = r) ; c_j += sum_i w_hat_ji (j = r)
#pragma unroll 8
      for (int i = 0; i < kCB; ++i) {
        u += h2f<kBF16>(*(const uint16_t*)(st + sw128_off(i, r, kCB))) * s_s[i];
        if (!prm.skipS) z += h2f<kBF16>(*(const uint16_t*)(st + kT64 + sw128_off(i, r, kCB)));
      }
#pragma unroll
      for (int i8 = 0; i8 < kCB; i8 += 8) {
        const uint4 v4 = *(const uint4*)(st + 3 * kT64 + sw128_off(r, i8, 128));
        const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f2 = unpack2<kBF16>(w4[q]);
          cc += f2.x + f2.y;
        }
      }
      pin(u);  // the stage's loads have returned before it is released
      pin(z);
      pin(cc);
      mbar_arrive(&empty[s]);
    }
    float* rS = prm.stS + (grp * prm.P + p) * state_floats(kD);
    float* rR = prm.stR + (grp * prm.P + p) * state_floats(kD);
    const uint32_t lb = (qd * 32u) << 16;
    if (nc > 0) {
      mbar_wait(done, 0);
      tc_fence_after();
    }
    for (int j0 = 0; j0 < kD; j0 += 32) {
      uint32_t xr[32], xs[32];
      if (nc > 0) {
        tmem_ld32(tmem + lb + j0, xr);
        tmem_ld32(tmem + lb + 128 + j0, xs);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) xr[q] = xs[q] = 0u;
      }
#pragma unroll
      for (int q = 0; q < 32; q += 4) {
        *(float4*)(rR + r * kD + j0 + q) = make_float4(__uint_as_float(xr[q]), __uint_as_float(xr[q + 1]),
                                                      __uint_as_float(xr[q + 2]), __uint_as_float(xr[q + 3]));
        if (!prm.skipS)
          *(float4*)(rS + r * kD + j0 + q) = make_float4(__uint_as_float(xs[q]), __uint_as_float(xs[q + 1]),
                                                        __uint_as_float(xs[q + 2]), __uint_as_float(xs[q + 3]));
      }
    }
    if (!prm.skipS) rS[kD * kD + r] = z;
    rR[kD * kD + r] = u;
    rR[kD * kD + kD + r] = cc;
    if (r == 0) {
      if (!prm.skipS) rS[kD * kD + 2 * kD] = (float)(s1 - s0);
      rR[kD * kD + 2 * kD] = (float)(s1 - s0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

// ================================================================ W_hat pass + R aggregate
// Runs over every unit of rows before the reverse sweep: W_hat = Omega^T / g and
// s_i = sum_j o_ji w_hat_ji per 64-row chunk, stored for the sweep (W_hat^T by TMA
// into the dV output, s as the first 256 bytes of the chunk's dQ rows: both are
// overwritten by the sweep after it has read them), and per unit R^T = sum W_hat^T Q,
// c = sum_i w_hat (a ones panel appended to Q as extra N columns of the same MMA) and
// u = Q^T s (a second small MMA against two bf16 rows s_hi, s_lo). The only CUDA-core
// work is the W_hat / s pass, spread over 256 threads. Stage: Q [64 i][128 m]
// (2 panels) | ones panel | W_hat^T [128 j][64 i] | s rows | O^T [128 j][64 i] (by TMA).
constexpr int kAStages = 3;
constexpr int kAStage = 2 * 8192 + 8192 + kT64 + 2048 + kT64;  // 58 KB
constexpr int kAOffOnes = 16384, kAOffW = 24576, kAOffS = 24576 + kT64, kAOffO = kAOffS + 2048;
constexpr size_t kAggRSmem = kAStages * kAStage + 128 + 4 * 2 * kCB * 4 + 1024;

// 320 threads (warps 0-9); its CTA-wide barriers are named barrier 2 over those 320.
template <bool kBF16>
__device__ __forceinline__ void bwd_aggR_body(const CUtensorMap& tmQ, const CUtensorMap& tmW,
                                              const CUtensorMap& tmO, const CUtensorMap& tmWo,
                                              const BwdParams& prm, const int p, const int64_t grp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bars = (uint64_t*)(smem + kAStages * kAStage);
  uint64_t* full = bars;                 // [4]
  uint64_t* empty = bars + kAStages;     // [4]
  uint64_t* w_ready = bars + 2 * kAStages;
  uint64_t* done = bars + 2 * kAStages + 1;
  uint32_t* tslot = (uint32_t*)(bars + 2 * kAStages + 2);
  float* s_part = (float*)(bars + 16);   // [2 parity][2 halves][64]

  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = (int)((s1 - s0) / kCB);
  const bool needR = p >= prm.r_unit0;
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmW);
    tma_prefetch(&tmO);
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // MMA commit + the W_hat^T store having read the stage
    }
    mbar_init(w_ready, 256);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  if (warp >= 2) {  // constant ones panels and the zero rows 2..15 of every s-rows tile
    const uint32_t one2 = kBF16 ? 0x3F803F80u : 0x3C003C00u;
    const int t = (int)threadIdx.x - 64;
    for (int s = 0; s < kAStages; ++s) {
      uint4* op = (uint4*)(smem + s * kAStage + kAOffOnes);
      for (int e = t; e < 8192 / 16; e += 256) op[e] = make_uint4(one2, one2, one2, one2);
      uint4* sp = (uint4*)(smem + s * kAStage + kAOffS);
      for (int e = t; e < 2048 / 16; e += 256) sp[e] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async();
  }
  tc_fence_before();
  named_bar(2, 320);
  tc_fence_after();
  const uint32_t tmem = *tslot;  // [0,144) R^T | c, [160,176) U
  if (warp == 0) {
    if (elect_one()) {
      auto l2_prefetch = [&](int c) {
        const int64_t row0 = s0 + (int64_t)c * kCB;
        if (needR) tma_prefetch_l2_3d(&tmQ, 0, (int)(grp * prm.N + row0), 0);
        tma_prefetch_l2_3d(&tmW, 0, (int)(grp * kD), (int)(row0 / 64));
        tma_prefetch_l2_3d(&tmO, 0, (int)(grp * kD), (int)(row0 / 64));
      };
      for (int c = 0; c < prm.pf && c < nc; ++c) l2_prefetch(c);
      for (int c = 0; c < nc; ++c) {
        const int s = c % kAStages;
        if (c + prm.pf < nc) l2_prefetch(c + prm.pf);
        if (c >= kAStages) mbar_wait(&empty[s], ((c / kAStages) & 1) ^ 1);
        const int64_t row0 = s0 + (int64_t)c * kCB;
        uint8_t* st = smem + s * kAStage;
        mbar_expect_tx(&full[s], (needR ? 3 : 2) * kT64);
        if (needR) tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kAOffW, &tmW, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        tma_load_3d(st + kAOffO, &tmO, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t f = kBF16 ? 1 : 0;
    const uint32_t id_RT = idesc_f16(128, 144, f, 0, 1);  // A = W_hat^T (K-major), B = [Q | 1] (MN-major)
    const uint32_t id_U = idesc_f16(128, 16, f, 1, 0);    // A = Q^T (MN-major), B = s rows (K-major)
    for (int c = 0; c < nc; ++c) {
      const int s = c % kAStages;
      const uint32_t st = smem_u32(smem + s * kAStage);
      mbar_wait(w_ready, c & 1);
      tc_fence_after();
      if (elect_one()) {
        if (needR) {
          for (int ks = 0; ks < 4; ++ks)
            mma_ss(tmem, kd(st + kAOffW, ks, 128), mn(st, ks, 8192), id_RT, (c > 0 || ks > 0) ? 1u : 0u);
          for (int ks = 0; ks < 4; ++ks)
            mma_ss(tmem + 160, mn(st, ks, 8192), kd(st + kAOffS, ks, 16), id_U, (c > 0 || ks > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
          if (c == nc - 1) mma_commit(done);
        } else {
          mbar_arrive(&empty[s]);  // no MMA reads this stage
        }
      }
      __syncwarp();
    }
  } else {
    const int et = (int)threadIdx.x - 64;        // 0..255
    const int half = et >> 7, eh = et & 127;
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    const int jg = eh & 15, ig = 2 * (eh >> 5) + ((eh & 31) >> 4);  // what_pass_half's mapping
    float4 g8[2];
    auto g_prefetch = [&](int c) {
      const float* gp = prm.g + grp * prm.N + s0 + (int64_t)c * kCB + 8 * ig;
      g8[0] = __ldg((const float4*)gp);
      g8[1] = __ldg((const float4*)(gp + 4));
    };
    if (nc > 0) g_prefetch(0);
    for (int c = 0; c < nc; ++c) {
      const int s = c % kAStages;
      uint8_t* st = smem + s * kAStage;
      float* sp = s_part + (c & 1) * 2 * kCB;
      mbar_wait(&full[s], (c / kAStages) & 1);
      uint4 o4[4];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        o4[rr] = *(const uint4*)(st + kAOffO + sw128_off(64 * half + 16 * rr + jg, 8 * ig, 128));
      const float4 gc[2] = {g8[0], g8[1]};
      if (c + 1 < nc) g_prefetch(c + 1);
      float rs_unused[4];
      what_pass_half<kBF16>(st + kAOffW, o4, gc, sp + half * kCB, eh, 64 * half, rs_unused);
      fence_proxy_async();
      named_bar(1, 256);  // W_hat^T and both halves' partial s of chunk c are complete
      const int64_t row0 = s0 + (int64_t)c * kCB;
      if (prm.store_w && et == 0) {
        tma_store_3d(&tmWo, st + kAOffW, 0, (int)(grp * kD), (int)(row0 / 64));
        tma_store_commit();
      }
      if (et < kCB) {     // s rows (hi, lo) of the U = Q^T s MMA
        const float si = sp[et] + sp[kCB + et];
        if (prm.store_w) ((float*)((uint16_t*)prm.dq + (grp * prm.N + row0) * kD))[et] = si;
        uint16_t hv, lv;
        if (kBF16) {
          const __nv_bfloat16 h = __float2bfloat16_rn(si);
          hv = __bfloat16_as_ushort(h);
          lv = __bfloat16_as_ushort(__float2bfloat16_rn(si - __bfloat162float(h)));
        } else {
          const __half h = __float2half_rn(si);
          hv = __half_as_ushort(h);
          lv = __half_as_ushort(__float2half_rn(si - __half2float(h)));
        }
        *(uint16_t*)(st + kAOffS + sw128_off(0, et, 16)) = hv;
        *(uint16_t*)(st + kAOffS + sw128_off(1, et, 16)) = lv;
      }
      fence_proxy_async();
      mbar_arrive(w_ready);
      if (et == 0) {  // the previous chunk's W_hat^T store has read its stage
        tma_store_wait_read1();
        if (c >= 1) mbar_arrive(&empty[(c - 1) % kAStages]);
      }
    }
    if (et == 0) tma_store_wait0();
    if (half == 0 && needR) {  // records: R (X[m][j]), u, c, count
      float* rR = prm.stR + (grp * prm.P + p) * state_floats(kD);
      const uint32_t lb = (qd * 32u) << 16;
      if (nc > 0) {
        mbar_wait(done, 0);
        tc_fence_after();
        for (int m0 = 0; m0 < kD; m0 += 32) {  // lane r = j of R^T: column j of X
          uint32_t x[32];
          tmem_ld32(tmem + lb + m0, x);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 32; ++u) rR[(m0 + u) * kD + r] = __uint_as_float(x[u]);
        }
        uint32_t cc, c1, u0, u1;
        tmem_ld2(tmem + lb + 128, cc, c1);
        tmem_ld2(tmem + lb + 160, u0, u1);
        tmem_ld_wait();
        rR[kD * kD + r] = __uint_as_float(u0) + __uint_as_float(u1);  // u_m (lane r = m of U)
        rR[kD * kD + kD + r] = __uint_as_float(cc);                   // c_j
      } else {
        for (int m = 0; m < kD; ++m) rR[m * kD + r] = 0.f;
        rR[kD * kD + r] = 0.f;
        rR[kD * kD + kD + r] = 0.f;
      }
      if (r == 0) rR[kD * kD + 2 * kD] = (float)(s1 - s0);
    }
  }
  tc_fence_before();
  named_bar(2, 320);
  if (warp == 1) tmem_dealloc<256>(tmem);
}

template <bool kBF16>
__global__ void __launch_bounds__(320, 1)
    k_bwd_aggR_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmWo,
                  BwdParams prm) {
  bwd_aggR_body<kBF16>(tmQ, tmW, tmO, tmWo, prm, blockIdx.x + prm.p0, blockIdx.y);
}


// ================================================================ main reverse sweep
// Inputs per 64-row chunk (reverse order): Q, K, V^T and the W_hat^T / s written by the
// aggregate pass (W_hat^T in the dV buffer, s in the chunk's first dQ row), all by
// TMA. Warp roles (512 threads): 0 TMA producer; 1 MMA issuer + TMEM owner; 2-3 idle
// (warpgroup 0 hands its registers to the epilogue warpgroups with setmaxnreg);
// 4-7 WG-A: dV^T drain, bR -> sR (j < 64), E1 columns 32..63; 8-11 WG-B: dK^T drain,
// bR -> sR (j >= 64), dQ drain, bS -> sS; 12-15 WG-C: dc, s, E1 columns 0..31, z, du.
// E1: dPt -> dS (lower TMEM lane half), T1 -> P (upper half).
// MMA order per chunk n: dK^T / dV^T, R +=, dQ, then T1 / dPt and S -= of chunk n+1:
// the chain from one chunk's dK^T / dV^T to the next is the drains and E_R in
// parallel with E1.
constexpr int kBwdThreads = 512;
template <bool kBF16>
__device__ __forceinline__ void bwd_main_body(const CUtensorMap& tmQ, const CUtensorMap& tmK,
                                              const CUtensorMap& tmV, const CUtensorMap& tmW,
                                              const BwdParams& prm, const int p, const int64_t grp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sP = smem + 2 * kStage;         // P  [64 rows i][64 t]     8 KB
  uint8_t* sdS = sP + 8192;                // dS [64 rows i][64 t]     8 KB
  uint8_t* sR = sdS + 8192;                // b R  [128 rows m][128 j] 32 KB
  uint8_t* sS = sR + 32768;                // b S  [128 rows m][128 j] 32 KB
  uint64_t* bars = (uint64_t*)(sS + 32768);
  uint64_t* full = bars;        // [2]
  uint64_t* empty = bars + 2;   // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* dpt_full = bars + 6;
  uint64_t* dpt_empty = bars + 7;
  uint64_t* sS_ready = bars + 8;
  uint64_t* ps_ready = bars + 9;
  uint64_t* sR_ready = bars + 10;
  uint64_t* gkv_full = bars + 11;   // dK^T, dV^T accumulators complete
  uint64_t* gkv_empty = bars + 12;  // ... drained (WG-A dV^T, WG-B dK^T)
  uint64_t* r_full = bars + 13;
  uint32_t* tslot = (uint32_t*)(bars + 16);
  uint64_t* gq_full = bars + 17;    // dQ accumulator complete
  uint64_t* gq_empty = bars + 18;   // ... drained (WG-B)
  float* s_s = (float*)(bars + 20);   // [2 stages][64]  s of the staged chunk (TMA)
  float* du_s = s_s + 2 * kCB;        // [4][128]  du per chunk (WG-C -> WG-B's dK^T drain)
  float* zbuf = du_s + 4 * kD;        // [4][128]  z_prev per chunk (WG-C -> WG-B's dQ drain)
  float* dcp = zbuf + 4 * kD;         // [4][128]  dc per chunk (WG-C -> WG-A's dV^T drain)
  float* s_ring = dcp + 4 * kD;       // [4][64]   s per chunk (WG-C -> WG-B's dQ drain)
  uint8_t* dkscr = (uint8_t*)(s_ring + 4 * kCB);  // [4 warps][2 KB] dK^T store staging

  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = (int)((s1 - s0) / kCB);
  auto row_of = [&](int m) -> int64_t { return s0 + (int64_t)(nc - 1 - m) * kCB; };  // reverse sweep
  // the forward's exact prefix at chunk m's first row when that row is an interior checkpoint
  auto ck_record = [&](int m) -> const float* {
    if (!prm.ck || m >= nc - 1) return nullptr;
    if (prm.ck_unit > 0) {
      const int64_t off = row_of(m) - s0;
      if (off % prm.ck_unit) return nullptr;
      return prm.ck + ((grp * prm.P + p) * prm.A + off / prm.ck_unit) * state_floats(kD);
    }
    const int k = ck_index(prm.row_offset + row_of(m), prm.ck_K);
    return k < 0 ? nullptr : prm.ck + (grp * prm.ck_K + k) * state_floats(kD);
  };
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) traceb(0, 63, 8);
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmW);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 128);
    }
    mbar_init(s_full, 1);
    mbar_init(dpt_full, 1);
    mbar_init(dpt_empty, 256);
    mbar_init(sS_ready, 256);
    mbar_init(ps_ready, 256);
    mbar_init(sR_ready, 256);
    mbar_init(gkv_full, 1);
    mbar_init(gkv_empty, 256);
    mbar_init(gq_full, 1);
    mbar_init(gq_empty, 128);
    mbar_init(r_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  {  // carries: S inclusive prefix at s1 (saved by the forward, or carry + segment sums
     // 0..p) and R exclusive suffix after s1 (carry + segment sums p+1..P-1)
    const int64_t SZ = state_floats(kD);
    const int U = prm.P * prm.A;
    float* cS = prm.cmb + (grp * prm.P + p) * 2 * SZ;
    if (warp >= 4) {
      const int ct = (int)threadIdx.x - 128, cn = kBwdThreads - 128;
      if (prm.skipS)
        combine_records(cS, prm.stS + (grp * prm.P + p) * SZ, prm.stS, 0, 0, SZ, ct, cn);
      else if (!prm.cmb_ready)
        combine_records(cS, prm.carry_pre ? prm.carry_pre + grp * SZ : nullptr, prm.stS + grp * U * SZ, 0,
                        (p + 1) * prm.A, SZ, ct, cn);
      if (!prm.cmb_ready)
        combine_records(cS + SZ, prm.carry_suf ? prm.carry_suf + grp * SZ : nullptr, prm.stR + grp * U * SZ,
                        (p + 1) * prm.A, U, SZ, ct, cn);
      if (!prm.skipS && prm.ck_unit > 0 && !prm.cmb_ready) {  // exclusive prefix at each unit boundary of the segment
        float* ck = const_cast<float*>(prm.ck) + (grp * prm.P + p) * prm.A * SZ;
        combine_records(ck, prm.carry_pre ? prm.carry_pre + grp * SZ : nullptr, prm.stS + grp * U * SZ, 0,
                        p * prm.A, SZ, ct, cn);
        for (int j = 1; j < prm.A; ++j)  // each thread re-reads only the elements it wrote
          combine_records(ck + j * SZ, ck + (j - 1) * SZ, prm.stS + grp * U * SZ, p * prm.A + j - 1,
                          p * prm.A + j, SZ, ct, cn);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // Carries (R_next, S_end, u, c, z) are written into TMEM by WG-B before any role
  // starts: the first S -= K^T V must see S_end.
  if (warp >= 8 && warp < 12) {
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    const uint32_t lb = (qd * 32u) << 16;
    const float* recS = prm.cmb + (grp * prm.P + p) * 2 * state_floats(kD);  // inclusive prefix at s1
    const float* recR = recS + state_floats(kD);                             // exclusive suffix after s1
    for (int j0 = 0; j0 < kD; j0 += 32) {
      uint32_t xr[32], xs[32];
#pragma unroll
      for (int q = 0; q < 32; q += 4) {
        const float4 fr = *(const float4*)(recR + r * kD + j0 + q);
        const float4 fs = *(const float4*)(recS + r * kD + j0 + q);
        xr[q] = __float_as_uint(fr.x); xr[q + 1] = __float_as_uint(fr.y);
        xr[q + 2] = __float_as_uint(fr.z); xr[q + 3] = __float_as_uint(fr.w);
        xs[q] = __float_as_uint(fs.x); xs[q + 1] = __float_as_uint(fs.y);
        xs[q + 2] = __float_as_uint(fs.z); xs[q + 3] = __float_as_uint(fs.w);
      }
      tmem_st32(tmem + lb + kR + j0, xr);
      tmem_st32(tmem + lb + kS + j0, xs);
    }
    tmem_st_wait();
    zbuf[3 * kD + r] = recS[kD * kD + r];  // z at the segment end (read as chunk "-1")
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) traceb(0, 63, 9);

  if (warp < 4) {
#ifndef LA_BWD_REG_LO
#define LA_BWD_REG_LO 96
#define LA_BWD_REG_HI 136
#endif
  regs_dec<LA_BWD_REG_LO>();
#ifdef LA_TRACE
  if (warp == 2 && lane_id() == 0) {  // observer: when each chunk's stage lands
    for (int n = 0; n < nc && n < 64; ++n) {
      mbar_wait(&full[n & 1], (n >> 1) & 1);
      traceb(2, n, 4);
    }
  }
#endif
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (reverse)
    if (elect_one()) {
      auto l2_prefetch = [&](int n) {  // Q, K, V^T, W_hat^T of chunk n into L2
        const int64_t row0 = row_of(n);
        tma_prefetch_l2_3d(&tmQ, 0, (int)(grp * prm.N + row0), 0);
        tma_prefetch_l2_3d(&tmK, 0, (int)(grp * prm.N + row0), 0);
        tma_prefetch_l2_3d(&tmV, 0, (int)(grp * kD), (int)(row0 / 64));
        tma_prefetch_l2_3d(&tmW, 0, (int)(grp * kD), (int)(row0 / 64));
      };
      for (int n = 0; n < prm.pf && n < nc; ++n) l2_prefetch(n);
      for (int n = 0; n < nc; ++n) {
        const int s = n & 1;
        if (n + prm.pf < nc) l2_prefetch(n + prm.pf);
        if (n >= 2) mbar_wait(&empty[s], ((n >> 1) & 1) ^ 1);
        traceb(0, n, 4);
        const int64_t row0 = row_of(n);
        uint8_t* st = smem + s * kStage;
        mbar_expect_tx(&full[s], kStage + kCB * 4);
        tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kT64, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + 2 * kT64, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        tma_load_3d(st + 3 * kT64, &tmW, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        bulk_load(s_s + s * kCB, (const uint16_t*)prm.dq + (grp * prm.N + row0) * kD, kCB * 4, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t f = kBF16 ? 1 : 0;
    const uint32_t id_T1 = idesc_f16(64, 64, f, 0, 0);
    const uint32_t id_dPt = idesc_f16(64, 64, f, 1, 1);
    const uint32_t id_Sneg = idesc_f16(128, 128, f, 1, 0, 1);
    const uint32_t id_dQ1 = idesc_f16(64, 64, f, 0, 1);
    const uint32_t id_dQ2 = idesc_f16(64, 64, f, 1, 0);
    const uint32_t id_dK1 = idesc_f16(128, 64, f, 1, 1);
    const uint32_t id_dK2 = idesc_f16(128, 64, f, 0, 1);
    const uint32_t id_dV1 = idesc_f16(128, 64, f, 0, 1);
    const uint32_t id_dV2 = idesc_f16(128, 64, f, 1, 0);
    const uint32_t id_R = idesc_f16(128, 128, f, 1, 0);
    const uint32_t aP = smem_u32(sP), adS = smem_u32(sdS), aR = smem_u32(sR), aS = smem_u32(sS);
    for (int n = -1; n < nc; ++n) {
      const uint32_t aQ = smem_u32(smem + (n & 1) * kStage), aK = aQ + kT64, aV = aQ + 2 * kT64,
                     aW = aQ + 3 * kT64;
      const uint32_t bQ = smem_u32(smem + ((n + 1) & 1) * kStage), bK = bQ + kT64, bV = bQ + 2 * kT64,
                     bW = bQ + 3 * kT64;  // chunk n+1
      if (n >= 0) {
        if (lane_id() == 0) traceb(0, n, 0);
        mbar_wait(ps_ready, n & 1);
        mbar_wait(sR_ready, n & 1);
        if (n >= 1) mbar_wait(gkv_empty, (n - 1) & 1);
        if (lane_id() == 0) traceb(0, n, 1);
        tc_fence_after();
        if (elect_one()) {
          for (int ks = 0; ks < 4; ++ks)  // dK^T = Q^T dS^T
            mma_ss(tmem + kDK, mn(aQ, ks, 8192), mn(adS, ks, 8192), id_dK1, ks > 0);
          for (int ks = 0; ks < 8; ++ks)  //      + (b R) V^T
            mma_ss(tmem + kDK, kd(aR, ks, 128), mn(aV, ks, 8192), id_dK2, 1);
          for (int ks = 0; ks < 4; ++ks)  // dV^T = W_hat^T P
            mma_ss(tmem + kDV, kd(aW, ks, 128), mn(aP, ks, 8192), id_dV1, ks > 0);
          for (int ks = 0; ks < 8; ++ks)  //      + (b R)^T K^T
            mma_ss(tmem + kDV, mn(aR, ks, 16384), kd(aK, ks, 64), id_dV2, 1);
          mma_commit(gkv_full);
          for (int ks = 0; ks < 4; ++ks)  // R += Q^T W_hat
            mma_ss(tmem + kR, mn(aQ, ks, 8192), kd(aW, ks, 128), id_R, 1);
          mma_commit(r_full);
        }
        __syncwarp();
      }
      if (n >= 0) {
        mbar_wait(sS_ready, n & 1);
        if (n >= 1) mbar_wait(gq_empty, (n - 1) & 1);
        if (lane_id() == 0) traceb(0, n, 3);
        tc_fence_after();
        if (elect_one()) {
          for (int h = 0; h < 2; ++h) {  // dQ[:, 64h:64h+64]
            const uint32_t d = tmem + kDQ + (h ? kHalf : 0u);
            for (int ks = 0; ks < 4; ++ks)  // dS K
              mma_ss(d, kd(adS, ks, 64), mn(aK + h * 8192, ks, 8192), id_dQ1, ks > 0);
            for (int ks = 0; ks < 8; ++ks)  // W_hat (b S)^T
              mma_ss(d, mn(aW, ks, 8192), kd(aS + h * 8192, ks, 128), id_dQ2, 1);
          }
          mma_commit(gq_full);
          mma_commit(&empty[n & 1]);
        }
        __syncwarp();
        if (lane_id() == 0) traceb(0, n, 5);
      }
      if (n + 1 < nc) {  // T1 and dPt of chunk n+1 (E1(n) has read the previous ones)
        mbar_wait(&full[(n + 1) & 1], ((n + 1) >> 1) & 1);
        if (n >= 0) mbar_wait(dpt_empty, n & 1);
        if (lane_id() == 0) traceb(0, n + 1, 2);
        tc_fence_after();
        if (elect_one()) {
          for (int ks = 0; ks < 8; ++ks)  // T1 = Q K^T -> upper lane half
            mma_ss(tmem + kDP + kHalf, kd(bQ, ks, 64), kd(bK, ks, 64), id_T1, ks > 0);
          for (int ks = 0; ks < 8; ++ks)  // dPt = W_hat V^T -> lower lane half
            mma_ss(tmem + kDP, mn(bW, ks, 8192), mn(bV, ks, 8192), id_dPt, ks > 0);
          mma_commit(dpt_full);
        }
        __syncwarp();
        if (lane_id() == 0) traceb(0, n + 1, 6);
      }
      if (n + 1 < nc) {  // S -= K^T V of chunk n+1 (E_S(n) has read S: sS_ready above)
        tc_fence_after();
        if (elect_one()) {
          for (int ks = 0; ks < 4; ++ks)
            mma_ss(tmem + kS, mn(bK, ks, 8192), kd(bV, ks, 128), id_Sneg, 1);
          mma_commit(s_full);
        }
        __syncwarp();
      }
    }
  }
  } else {
  regs_inc<LA_BWD_REG_HI>();
  const uint32_t qd = warp & 3;
  const int l = (int)lane_id();
  const int r = (int)(qd * 32) + l;            // lane of the M=128 accumulators (j or m)
  const int ih = (int)(qd * 16) + (l & 15);    // half-lane row i of M=64 accumulators
  const bool upper = l >= 16;                  // lanes 16..31 of a quadrant: upper half
  const uint32_t lb = (qd * 32u) << 16;
  const float a = prm.a, b = prm.b;
  const float* recR = prm.cmb + (grp * prm.P + p) * 2 * state_floats(kD) + state_floats(kD);
  // b R_next -> sR for columns [jb, jb + 64) (R complete after the previous chunk's R +=)
  auto er_half = [&](int n, int jb) {
    if (n >= 1) mbar_wait(r_full, (n - 1) & 1);
    tc_fence_after();
#pragma unroll 1
    for (int j0 = jb; j0 < jb + 64; j0 += 32) {
      uint32_t x[32];
      tmem_ld32(tmem + lb + kR + j0, x);
      tmem_ld_wait();
#pragma unroll
      for (int w8 = 0; w8 < 4; ++w8) {
        uint4 v;
        v.x = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 0]), b * __uint_as_float(x[8 * w8 + 1]));
        v.y = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 2]), b * __uint_as_float(x[8 * w8 + 3]));
        v.z = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 4]), b * __uint_as_float(x[8 * w8 + 5]));
        v.w = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 6]), b * __uint_as_float(x[8 * w8 + 7]));
        *(uint4*)(sR + sw128_off(r, j0 + 8 * w8, 128)) = v;
      }
    }
    fence_proxy_async();
    tc_fence_before();
    mbar_arrive(sR_ready);
  };
  // E1 for columns [t0, t0 + 32) of chunk n: P = a + b T1 (upper lanes), dS = b dPt - b s
  // (lower lanes), one FFMA per element, no divergence
  auto e1_half = [&](int n, int t0) {
    mbar_wait(dpt_full, n & 1);
    if (n >= 1) mbar_wait(gq_full, (n - 1) & 1);  // dK^T/dV^T(n-1) and dQ(n-1) have read sP / sdS
    tc_fence_after();
    if (threadIdx.x == 384) traceb(3, n, 4);
    const float si = s_s[(n & 1) * kCB + ih];
    const float alpha = upper ? a : -b * si;
    uint8_t* dst = upper ? sP : sdS;
    uint32_t x[32];
    tmem_ld32(tmem + lb + kDP + t0, x);
    tmem_ld_wait();
    if (threadIdx.x == 384) traceb(3, n, 5);
#pragma unroll
    for (int w8 = 0; w8 < 4; ++w8) {
      uint32_t pk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = t0 + 8 * w8 + 2 * q;
        const float x0 = __uint_as_float(x[8 * w8 + 2 * q]), x1 = __uint_as_float(x[8 * w8 + 2 * q + 1]);
        const float v0 = t <= ih ? fmaf(b, x0, alpha) : 0.f;
        const float v1 = t + 1 <= ih ? fmaf(b, x1, alpha) : 0.f;
        pk[q] = pack2<kBF16>(v0, v1);
      }
      *(uint4*)(dst + sw128_off(ih, t0 + 8 * w8, kCB)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (threadIdx.x == 384) traceb(3, n, 6);
    fence_proxy_async();
    if (threadIdx.x == 384) traceb(3, n, 7);
    tc_fence_before();
    mbar_arrive(dpt_empty);
    mbar_arrive(ps_ready);
  };
  if (warp < 8) {
    // ------------------------------------------------------------ WG-A (warps 4..7)
    // Iteration n: dV^T drain of chunk n-1 (then c += dc(n-1)); bR -> sR for j < 64 and
    // E1 columns 32..63 of chunk n.
    const int et = (int)threadIdx.x - 128;
    float cj = recR[kD * kD + kD + r];  // c_next (j = r)
    auto dv_out = [&](int m) {  // dV^T of chunk m (lanes j): acc + a c_next
      mbar_wait(gkv_full, m & 1);
      if (et == 0) traceb(1, m, 0);
      tc_fence_after();
      const float ac = a * cj;
      uint4 vt[8];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lb + kDV + c0, x);
        tmem_ld_wait();
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          uint32_t k4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            k4[q] = pack2<kBF16>(__uint_as_float(x[8 * w4 + 2 * q]) + ac, __uint_as_float(x[8 * w4 + 2 * q + 1]) + ac);
          vt[c0 / 8 + w4] = make_uint4(k4[0], k4[1], k4[2], k4[3]);
        }
      }
      tc_fence_before();
      uint16_t* dvb = (uint16_t*)prm.dv + (grp * kD + qd * 32) * prm.N + row_of(m);
      warp_store_rows_2k(sP + qd * 2048, vt, [&](int seg) { return dvb + seg * prm.N; });
      mbar_arrive(gkv_empty);  // after the staging: WG-C's E1(m+1) rewrites these sP rows
      cj += dcp[(m & 3) * kD + r];
    };
    // One call site per phase (the kernel's code must stay small for the I-cache):
    // iteration n = nc only drains dV^T(nc-1).
    for (int n = 0; n <= nc; ++n) {
      if (n >= 1) dv_out(n - 1);
      if (n == nc) break;
      er_half(n, 0);
      if (et == 0) traceb(1, n, 1);
      e1_half(n, 32);  // after dv_out: this warp's sP rows were its staging scratch
      if (et == 0) traceb(1, n, 2);
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ WG-B (warps 8..11)
    // Iteration n: dK^T drain of chunk n-1, bR -> sR for j >= 64 of chunk n, dQ drain
    // of chunk n-1, bS -> sS (E_S) of chunk n.
    const int eb = (int)threadIdx.x - 256;
    float u = recR[kD * kD + r];  // u_next (m = r)
    auto dk_out = [&](int m) {  // dK^T (lanes m): acc - b u_next
      mbar_wait(gkv_full, m & 1);
      if (m >= 1) u += du_s[((m - 1) & 3) * kD + r];  // suffix sum through chunk m-1
      tc_fence_after();
      const float bu = b * u;
      uint4 vt[8];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lb + kDK + c0, x);
        tmem_ld_wait();
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          uint32_t k4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            k4[q] = pack2<kBF16>(__uint_as_float(x[8 * w4 + 2 * q]) - bu, __uint_as_float(x[8 * w4 + 2 * q + 1]) - bu);
          vt[c0 / 8 + w4] = make_uint4(k4[0], k4[1], k4[2], k4[3]);
        }
      }
      tc_fence_before();
      mbar_arrive(gkv_empty);
      uint16_t* dkb = (uint16_t*)prm.dk + (grp * kD + qd * 32) * prm.N + row_of(m);
      warp_store_rows_2k(dkscr + qd * 2048, vt, [&](int seg) { return dkb + seg * prm.N; });
    };
    auto dq_out = [&](int m) {  // dQ (half lanes): acc - b s_i z_prev
      mbar_wait(gq_full, m & 1);
      if (eb == 0) traceb(2, m, 0);
      tc_fence_after();
      const float* zq = zbuf + (m & 3) * kD;
      const int m0 = upper ? 64 : 0;
      const float bs = b * s_ring[(m & 3) * kCB + ih];
      uint4 vt[8];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lb + kDQ + c0, x);
        tmem_ld_wait();
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          uint32_t q4[4];
          const float4 za = *(const float4*)(zq + m0 + c0 + 8 * w4);
          const float4 zb = *(const float4*)(zq + m0 + c0 + 8 * w4 + 4);
          const float z8[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            q4[q] = pack2<kBF16>(__uint_as_float(x[8 * w4 + 2 * q]) - bs * z8[2 * q],
                                 __uint_as_float(x[8 * w4 + 2 * q + 1]) - bs * z8[2 * q + 1]);
          vt[c0 / 8 + w4] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
        }
      }
      tc_fence_before();
      // scratch: this warp's 4 KB of sS (E_S of the next chunk waits for gq_empty)
      uint8_t* scr_lo = sS + qd * 4096;
      uint16_t* dqb = (uint16_t*)prm.dq + (grp * prm.N + row_of(m) + qd * 16) * kD;
      warp_store_rows(scr_lo, scr_lo + 2048, vt, [&](int seg) { return dqb + (seg & 15) * kD + (seg >> 4) * 64; });
      mbar_arrive(gq_empty);
    };
    for (int n = 0; n <= nc; ++n) {
      if (n >= 1) dk_out(n - 1);
      if (n < nc) er_half(n, 64);
      if (n >= 1) dq_out(n - 1);
      if (n == nc) break;
      // ---- E_S: b S_prev -> sS (after every warp's dQ staging in sS: gq_empty). At a
      //      checkpoint row the forward's exact prefix replaces the rebuilt one, in TMEM
      //      too, so the later subtractions start from it (internal.h, kCkC0).
      mbar_wait(s_full, n & 1);
      if (n >= 1) mbar_wait(gq_empty, (n - 1) & 1);
      if (eb == 0) traceb(2, n, 1);
      tc_fence_after();
      if (const float* ck = ck_record(n)) {  // out of line: the loop below is I-cache sensitive
#pragma unroll 1
        for (int j0 = 0; j0 < kD; j0 += 32) {
          uint32_t x[32];
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            const float4 f4 = *(const float4*)(ck + r * kD + j0 + q);
            x[q] = __float_as_uint(f4.x); x[q + 1] = __float_as_uint(f4.y);
            x[q + 2] = __float_as_uint(f4.z); x[q + 3] = __float_as_uint(f4.w);
          }
          tmem_st32(tmem + lb + kS + j0, x);
        }
        tmem_st_wait();
      }
#pragma unroll 1
      for (int j0 = 0; j0 < kD; j0 += 64) {  // two loads in flight per wait
        uint32_t x[64];
        tmem_ld32(tmem + lb + kS + j0, *reinterpret_cast<uint32_t(*)[32]>(x));
        tmem_ld32(tmem + lb + kS + j0 + 32, *reinterpret_cast<uint32_t(*)[32]>(x + 32));
        tmem_ld_wait();
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) {
          uint4 v;
          v.x = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 0]), b * __uint_as_float(x[8 * w8 + 1]));
          v.y = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 2]), b * __uint_as_float(x[8 * w8 + 3]));
          v.z = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 4]), b * __uint_as_float(x[8 * w8 + 5]));
          v.w = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 6]), b * __uint_as_float(x[8 * w8 + 7]));
          *(uint4*)(sS + sw128_off(r, j0 + 8 * w8, 128)) = v;
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(sS_ready);
      if (eb == 0) traceb(2, n, 2);
    }
  } else {
    // ------------------------------------------------------------ WG-C (warps 12..15)
    // Chunk n: dc_j = sum_i w_hat_ji (-> dcp for WG-A), s (-> s_ring for WG-B), E1
    // columns 0..31, z_prev(n) = z_prev(n-1) - sum_t k_t, du_m = sum_i q_im s_i.
    const int ec = (int)threadIdx.x - 384;
    const int mg = ec >> 3, tg = ec & 7;  // column sums: columns 8 mg.., rows tg + 8 k
    for (int n = 0; n < nc; ++n) {
      const int s = n & 1;
      uint8_t* st = smem + s * kStage;
      mbar_wait(&full[s], (n >> 1) & 1);
      if (ec == 0) traceb(3, n, 3);
      {  // row j = r of W_hat^T: 8 conflict-free 16-byte chunks
        const uint8_t* w_t = st + 3 * kT64;
        uint4 wv[8];
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) wv[c8] = *(const uint4*)(w_t + sw128_off(r, 8 * c8, 128));
        float dc = 0.f;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint32_t w4[4] = {wv[c8].x, wv[c8].y, wv[c8].z, wv[c8].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f2 = unpack2<kBF16>(w4[q]);
            dc += f2.x + f2.y;
          }
        }
        dcp[(n & 3) * kD + r] = dc;
        if (ec < kCB) s_ring[(n & 3) * kCB + ec] = s_s[s * kCB + ec];
      }
      if (n >= 1) mbar_wait(gkv_empty, (n - 1) & 1);  // WG-A's dV^T staging in sP is done
      if (ec == 0) traceb(3, n, 0);
      e1_half(n, 0);
      if (ec == 0) traceb(3, n, 1);
      // ---- z_prev(n) -> zbuf[n & 3]
      {
        const uint8_t* k_t = st + kT64;
        float zs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint4 kv[kCB / 8];
#pragma unroll
        for (int k8 = 0; k8 < kCB / 8; ++k8) kv[k8] = *(const uint4*)(k_t + sw128_off(tg + 8 * k8, 8 * mg, kCB));
#pragma unroll
        for (int k8 = 0; k8 < kCB / 8; ++k8) {
          const uint32_t xx[4] = {kv[k8].x, kv[k8].y, kv[k8].z, kv[k8].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f2 = unpack2<kBF16>(xx[q]);
            zs[2 * q] += f2.x;
            zs[2 * q + 1] += f2.y;
          }
        }
        const int m = 8 * mg + tg;
        const float zn = zbuf[((n - 1) & 3) * kD + m] - reduce_scatter8(zs, tg);
        const float* ck = ck_record(n);
        zbuf[(n & 3) * kD + m] = ck ? ck[kD * kD + m] : zn;
      }
      mbar_arrive(sS_ready);  // publishes z(n), s(n) for dq_out(n) (dQ(n) waits sS_ready)
      // ---- du_m = sum_i q_im s_i of this chunk -> du_s[n & 3] (read by dk_out(n + 1))
      {
        const uint8_t* q_t = st;
        const float* sc = s_s + s * kCB;
        float du[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint4 qv[kCB / 8];  // all loads first: smem latency is long under the MMA traffic
        float wv[kCB / 8];
#pragma unroll
        for (int k8 = 0; k8 < kCB / 8; ++k8) {
          qv[k8] = *(const uint4*)(q_t + sw128_off(tg + 8 * k8, 8 * mg, kCB));
          wv[k8] = sc[tg + 8 * k8];
        }
#pragma unroll
        for (int k8 = 0; k8 < kCB / 8; ++k8) {
          const uint32_t xx[4] = {qv[k8].x, qv[k8].y, qv[k8].z, qv[k8].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f2 = unpack2<kBF16>(xx[q]);
            du[2 * q] += wv[k8] * f2.x;
            du[2 * q + 1] += wv[k8] * f2.y;
          }
        }
        du_s[(n & 3) * kD + 8 * mg + tg] = reduce_scatter8(du, tg);
      }
      mbar_arrive(&empty[s]);
      if (ec == 0) traceb(3, n, 2);
    }
  }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) traceb(0, 63, 7);
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <bool kBF16>
__global__ void __launch_bounds__(kBwdThreads, 1)
    k_bwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW,
             BwdParams prm) {
  bwd_main_body<kBF16>(tmQ, tmK, tmV, tmW, prm, blockIdx.x, blockIdx.y);
}

// ================================================================ non-causal backward
// backward_full (backward_kernels.hpp:173-288): with the totals S, z (keys/values) and
// R = sum q^T w_hat, u = sum s q, c = sum w_hat over all N, every 64-row chunk is
// independent:
//   dQ   = W_hat (b S)^T - b s z^T          (M=64 halves; bS a constant smem operand)
//   dK^T = (b R) V^T - b u                  (bR constant)
//   dV^T = (b R)^T K^T + a c
// Stage: K [64 t][128 m] | V^T | Omega^T (-> W_hat in place) | O^T. Two epilogue
// warpgroups share the W_hat / s pass (rows j 0..63 / 64..127); WG-A drains dV^T, WG-B
// dQ and dK^T. TMEM: [dQ | dK^T | dV^T] x 2 buffers.
struct BwdFullParams {
  const float* totS;  // per group: S (X[m][j]), z, sigma, count
  const float* totR;  // per group: R (X[m][j]), u, c, count
  const void* o;
  const float* g;
  void* dq;
  void* dk;
  void* dv;
  int64_t N;
  int64_t seg_len;
  float a, b;
};

constexpr int kFStageB = 4 * kT64;  // K, V^T, Omega^T, O^T
constexpr size_t kBwdFullSmem = 2 * kFStageB + 2 * 32768 + 128 + 4 * kCB * 2 * 4 + 1024;

template <bool kBF16>
__global__ void __launch_bounds__(320, 1)
    k_bwd_full_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
                  BwdFullParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sR = smem + 2 * kFStageB;       // b R [128 rows m][128 j]
  uint8_t* sS = sR + 32768;                // b S [128 rows m][128 j]
  uint64_t* bars = (uint64_t*)(sS + 32768);
  uint64_t* full = bars;         // [2]
  uint64_t* empty = bars + 2;    // [2]
  uint64_t* w_ready = bars + 4;  // [2] by chunk parity
  uint64_t* acc_full = bars + 6; // [2]
  uint64_t* acc_empty = bars + 8;// [2]
  uint32_t* tslot = (uint32_t*)(bars + 10);
  float* s_s = (float*)(bars + 16);  // [4][2][64]

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = s1 > s0 ? (int)((s1 - s0) / kCB) : 0;
  auto row_of = [&](int m) -> int64_t { return s0 + (int64_t)m * kCB; };
  const uint32_t warp = warp_id();
  const float* tS = prm.totS + grp * state_floats(kD);
  const float* tR = prm.totR + grp * state_floats(kD);
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmW);
    tma_prefetch(&tmO);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1 + 256);
      mbar_init(&w_ready[b], 256);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  if (warp >= 2) {  // constants bR, bS -> smem (row m = r, bf16, K-major over j)
    const int t = (int)threadIdx.x - 64;
    const int r = t & 127;
    const float* src = t < 128 ? tR : tS;
    uint8_t* dst = t < 128 ? sR : sS;
    const float b = prm.b;
#pragma unroll 4  // 8 loads in flight: the row of each lane is 512 B away from its neighbour's
    for (int j0 = 0; j0 < kD; j0 += 8) {
      const float4 x0 = *(const float4*)(src + r * kD + j0), x1 = *(const float4*)(src + r * kD + j0 + 4);
      *(uint4*)(dst + sw128_off(r, j0, 128)) =
          make_uint4(pack2<kBF16>(b * x0.x, b * x0.y), pack2<kBF16>(b * x0.z, b * x0.w),
                     pack2<kBF16>(b * x1.x, b * x1.y), pack2<kBF16>(b * x1.z, b * x1.w));
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (elect_one()) {
      for (int n = 0; n < nc; ++n) {
        const int s = n & 1;
        if (n >= 2) mbar_wait(&empty[s], ((n >> 1) & 1) ^ 1);
        const int64_t row0 = row_of(n);
        uint8_t* st = smem + s * kFStageB;
        mbar_expect_tx(&full[s], kFStageB);
        tma_load_3d(st, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kT64, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        tma_load_3d(st + 2 * kT64, &tmW, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
        tma_load_3d(st + 3 * kT64, &tmO, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t f = kBF16 ? 1 : 0;
    const uint32_t id_dQ2 = idesc_f16(64, 64, f, 1, 0);
    const uint32_t id_dK2 = idesc_f16(128, 64, f, 0, 1);
    const uint32_t id_dV2 = idesc_f16(128, 64, f, 1, 0);
    const uint32_t aR = smem_u32(sR), aS = smem_u32(sS);
    for (int n = 0; n < nc; ++n) {
      const int s = n & 1, bb = n & 1;
      const uint32_t aK = smem_u32(smem + s * kFStageB), aV = aK + kT64, aW = aK + 2 * kT64;
      mbar_wait(&w_ready[s], (n >> 1) & 1);
      if (n >= 2) mbar_wait(&acc_empty[bb], ((n - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t base = tmem + bb * 192;
        for (int h = 0; h < 2; ++h)  // dQ[:, 64h:64h+64] = W_hat (b S)^T
          for (int ks = 0; ks < 8; ++ks)
            mma_ss(base + (h ? kHalf : 0u), mn(aW, ks, 8192), kd(aS + h * 8192, ks, 128), id_dQ2, ks > 0);
        for (int ks = 0; ks < 8; ++ks)  // dK^T = (b R) V^T
          mma_ss(base + 64, kd(aR, ks, 128), mn(aV, ks, 8192), id_dK2, ks > 0);
        for (int ks = 0; ks < 8; ++ks)  // dV^T = (b R)^T K^T
          mma_ss(base + 128, mn(aR, ks, 16384), kd(aK, ks, 64), id_dV2, ks > 0);
        mma_commit(&acc_full[bb]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    const bool is_a = warp < 6;
    const uint32_t qd = warp & 3;
    const int l = (int)lane_id();
    const int r = (int)(qd * 32) + l;              // j (WG-A: dV^T) / m (WG-B: dK^T)
    const int ih = (int)(qd * 16) + (l & 15);
    const bool upper = l >= 16;
    const uint32_t lb = (qd * 32u) << 16;
    const int et = (int)threadIdx.x - (is_a ? 64 : 192);
    const int jbase = is_a ? 0 : 64;
    const float a = prm.a, b = prm.b;
    const float ac = a * tR[kD * kD + kD + r];     // WG-A: a c_j
    const float bu = b * tR[kD * kD + r];          // WG-B: b u_m
    uint4 o4[4];
    float4 g8[2];
    auto e0 = [&](int m) {  // W_hat / partial s of chunk m (rows jbase..jbase+63), O^T from the stage
      const int sm = m & 1;
      mbar_wait(&full[sm], (m >> 1) & 1);
      uint8_t* st = smem + sm * kFStageB;
      const int jg = et & 15, ig = 2 * (et >> 5) + ((et & 31) >> 4);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        o4[rr] = *(const uint4*)(st + 3 * kT64 + sw128_off(jbase + 16 * rr + jg, 8 * ig, 128));
      const float* gp = prm.g + grp * prm.N + row_of(m) + 8 * ig;
      g8[0] = __ldg((const float4*)gp);
      g8[1] = __ldg((const float4*)(gp + 4));
      float rs_unused[4];
      what_pass_half<kBF16>(st + 2 * kT64, o4, g8, s_s + (m & 3) * 2 * kCB + (jbase ? kCB : 0), et, jbase,
                            rs_unused);
      fence_proxy_async();
      mbar_arrive(&w_ready[sm]);
      mbar_arrive(&empty[sm]);
    };
    if (nc > 0) e0(0);
    for (int n = 0; n < nc; ++n) {
      if (n + 1 < nc) e0(n + 1);
      const int bb = n & 1;
      const int64_t row0 = row_of(n);
      mbar_wait(&acc_full[bb], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + bb * 192;
      uint32_t x0[32], x1[32];
      uint4 vt[8];
      if (is_a) {  // dV^T (lanes j) + a c_j
        tmem_ld32(base + lb + 128, x0);
        tmem_ld32(base + lb + 128 + 32, x1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&acc_empty[bb]);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          vt[w] = make_uint4(pack2<kBF16>(__uint_as_float(x0[8 * w]) + ac, __uint_as_float(x0[8 * w + 1]) + ac),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 2]) + ac, __uint_as_float(x0[8 * w + 3]) + ac),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 4]) + ac, __uint_as_float(x0[8 * w + 5]) + ac),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 6]) + ac, __uint_as_float(x0[8 * w + 7]) + ac));
          vt[4 + w] = make_uint4(pack2<kBF16>(__uint_as_float(x1[8 * w]) + ac, __uint_as_float(x1[8 * w + 1]) + ac),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 2]) + ac, __uint_as_float(x1[8 * w + 3]) + ac),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 4]) + ac, __uint_as_float(x1[8 * w + 5]) + ac),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 6]) + ac, __uint_as_float(x1[8 * w + 7]) + ac));
        }
        uint4* dst = (uint4*)((uint16_t*)prm.dv + (grp * kD + r) * prm.N + row0);
#pragma unroll
        for (int w = 0; w < 8; ++w) dst[w] = vt[w];
      } else {  // dQ (half lanes) - b s_i z_m, then dK^T (lanes m) - b u_m
        const float* sA = s_s + (n & 3) * 2 * kCB;
        const float bsi = b * (sA[ih] + sA[kCB + ih]);
        const float* zq = tS + kD * kD + (upper ? 64 : 0);
        tmem_ld32(base + lb, x0);
        tmem_ld32(base + lb + 32, x1);
        tmem_ld_wait();
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float4 za = *(const float4*)(zq + 8 * w), zb = *(const float4*)(zq + 8 * w + 4);
          vt[w] = make_uint4(pack2<kBF16>(__uint_as_float(x0[8 * w]) - bsi * za.x, __uint_as_float(x0[8 * w + 1]) - bsi * za.y),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 2]) - bsi * za.z, __uint_as_float(x0[8 * w + 3]) - bsi * za.w),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 4]) - bsi * zb.x, __uint_as_float(x0[8 * w + 5]) - bsi * zb.y),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 6]) - bsi * zb.z, __uint_as_float(x0[8 * w + 7]) - bsi * zb.w));
          const float4 zc = *(const float4*)(zq + 32 + 8 * w), zd = *(const float4*)(zq + 32 + 8 * w + 4);
          vt[4 + w] = make_uint4(pack2<kBF16>(__uint_as_float(x1[8 * w]) - bsi * zc.x, __uint_as_float(x1[8 * w + 1]) - bsi * zc.y),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 2]) - bsi * zc.z, __uint_as_float(x1[8 * w + 3]) - bsi * zc.w),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 4]) - bsi * zd.x, __uint_as_float(x1[8 * w + 5]) - bsi * zd.y),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 6]) - bsi * zd.z, __uint_as_float(x1[8 * w + 7]) - bsi * zd.w));
        }
        uint4* dqr = (uint4*)((uint16_t*)prm.dq + (grp * prm.N + row0 + ih) * kD + (upper ? 64 : 0));
#pragma unroll
        for (int w = 0; w < 8; ++w) dqr[w] = vt[w];
        tmem_ld32(base + lb + 64, x0);
        tmem_ld32(base + lb + 64 + 32, x1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&acc_empty[bb]);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          vt[w] = make_uint4(pack2<kBF16>(__uint_as_float(x0[8 * w]) - bu, __uint_as_float(x0[8 * w + 1]) - bu),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 2]) - bu, __uint_as_float(x0[8 * w + 3]) - bu),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 4]) - bu, __uint_as_float(x0[8 * w + 5]) - bu),
                             pack2<kBF16>(__uint_as_float(x0[8 * w + 6]) - bu, __uint_as_float(x0[8 * w + 7]) - bu));
          vt[4 + w] = make_uint4(pack2<kBF16>(__uint_as_float(x1[8 * w]) - bu, __uint_as_float(x1[8 * w + 1]) - bu),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 2]) - bu, __uint_as_float(x1[8 * w + 3]) - bu),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 4]) - bu, __uint_as_float(x1[8 * w + 5]) - bu),
                                 pack2<kBF16>(__uint_as_float(x1[8 * w + 6]) - bu, __uint_as_float(x1[8 * w + 7]) - bu));
        }
        uint4* dkr = (uint4*)((uint16_t*)prm.dk + (grp * kD + r) * prm.N + row0);
#pragma unroll
        for (int w = 0; w < 8; ++w) dkr[w] = vt[w];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

constexpr size_t kAggSmemB = 2 * kStage + 512 + 1024;
constexpr size_t kMainSmemB = 2 * kStage + 2 * 8192 + 2 * 32768 + 160 + (6 * kCB + 16 * kD) * 4 + 8192 + 1024;
static_assert(kMainSmemB <= 232448, "backward smem");

int tcb_segments(int64_t G, int64_t N) { return tc_segments(G, N); }

}  // namespace

bool tc_backward_supported(const Launch& L, const Tensors& t) {
  return (L.dtype == LA_BF16 || L.dtype == LA_F16) && L.D == kD && L.fault == LA_FAULT_NONE &&
         (L.causal || (L.carry_prefix == nullptr && L.carry_suffix == nullptr && L.row_offset == 0)) &&
         L.N % 128 == 0 && t.lq == LA_SEQUENCE_MAJOR && t.lk == LA_SEQUENCE_MAJOR &&
         t.lv == LA_FEATURE_MAJOR && t.lw == LA_FEATURE_MAJOR && t.lo == LA_FEATURE_MAJOR &&
         L.G * L.N < (1ll << 31) && L.G * kD < (1ll << 31);
}

size_t tc_backward_ws_floats(int64_t G, int64_t N, int64_t D) {
  if (D != kD || N % 128) return 0;
  const int P = tcb_segments(G, N);
  const int64_t seg = ((N / 128 + P - 1) / P) * 128;
  const int A = std::max(std::max(agg_split(G, seg, P > 1 ? P - 1 : 1), agg_split(G, seg, P)), bwd_agg_split(seg, P, false));  // the larger of the two
  // S, R unit sums + combined records, then the unit-boundary prefixes of the recomputing
  // sweep
  const size_t causal = (size_t)((2 * A + 2) * G * P) + (size_t)(G * P * A);
  const int Af = agg_split(G, seg, P);
  const size_t full = (size_t)(tc_kv_units(G, N) * G + Af * P * G + 2 * G);  // non-causal unit sums + totals
  return (causal > full ? causal : full) * state_floats(kD);
}

// Non-causal backward: totals (S, z from K, V; R, u, c from Q, dO, O, g), then one
// independent pass over 64-row chunks.
static cudaError_t tc_backward_full(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                                    Workspace ws) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N, SZ = state_floats(kD);
  const int P = tcb_segments(G, N);
  const int64_t seg = ((N / 128 + P - 1) / P) * 128;
  const int A = agg_split(G, seg, P);
  const int Ukv = tc_kv_units(G, N);
  float* unitsS = ws.base;
  float* totS = unitsS + G * Ukv * SZ;
  float* unitsR = totS + G * SZ;
  float* totR = unitsR + G * P * A * SZ;
  cudaError_t e = cudaSuccess;
  if (L.saved_in)  // the forward's K/V totals (la_forward_save)
    totS = const_cast<float*>(L.saved_in) + kSavedHeader;
  else
    e = tc_kv_totals(L, t, unitsS, totS);
  if (e != cudaSuccess) return e;
  CUtensorMap mQ, mK, mV, mW, mO;
  if (!make_tma_map(&mO, t.o, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mQ, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mK, t.k, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mW, t.w, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  BwdParams pa{t.o, t.g, dq, dk, dv, unitsS, unitsR, N, seg / A, P * A, L.a, L.b, 0, 1, 0, A, nullptr, nullptr,
               nullptr, 0};
  auto aggR = bf ? k_bwd_aggR_tc<true> : k_bwd_aggR_tc<false>;
  cudaFuncSetAttribute(aggR, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggRSmem);
  {
    ProfScope ps("la_bwd_agg", L.stream);
    aggR<<<dim3(A * P, G), 320, kAggRSmem, L.stream>>>(mQ, mW, mO, mW, pa);
  }
  e = tc_sum_units(unitsR, G, P * A, totR, L.stream);
  if (e != cudaSuccess) return e;
  const int64_t c64 = N / kCB;
  // independent chunks: ~4 waves of CTAs balance the tail against the per-CTA setup
  // of the constant bS / bR operands (G = 64: 1.19 ms at 1.3 waves -> 0.85 ms at 3.9)
  int64_t P2 = (4 * 148 + G / 2) / G;
  if (tuning().full_ctas_bwd > 0) P2 = tuning().full_ctas_bwd;  // measurement override
  if (P2 > c64) P2 = c64;
  if (P2 < 1) P2 = 1;
  const int64_t seg2 = ((c64 + P2 - 1) / P2) * kCB;
  P2 = (N + seg2 - 1) / seg2;
  BwdFullParams prm{totS, totR, t.o, t.g, dq, dk, dv, N, seg2, L.a, L.b};
  auto main_k = bf ? k_bwd_full_tc<true> : k_bwd_full_tc<false>;
  cudaFuncSetAttribute(main_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdFullSmem);
  {
    ProfScope ps("la_bwd_full", L.stream);
    main_k<<<dim3((unsigned)P2, (unsigned)G), 320, kBwdFullSmem, L.stream>>>(mK, mV, mW, mO, prm);
  }
  note_launch(2);
  return cudaGetLastError();
}

// Sequence-shard totals on the tensor core (the inputs of the NCCL all-gather scan,
// la_sharded_forward / sharding.py): forward (S, z, sigma, rows) = the non-causal K/V
// totals; backward (R, u, c, rows) = the R aggregate units summed per group. The unit
// records go to caller scratch (tc_shard_state_scratch_floats), no allocation.
size_t tc_shard_state_scratch_floats(int64_t G, int64_t N) {
  const int P = tcb_segments(G, N);
  const int64_t seg = ((N / 128 + P - 1) / P) * 128;
  const int A = agg_split(G, seg, P);
  const size_t f = (size_t)G * tc_kv_units(G, N), b = (size_t)G * P * A;
  return (f > b ? f : b) * state_floats(kD);
}

cudaError_t tc_forward_shard_state(const Launch& L, const Tensors& t, float* out, float* units) {
  return tc_kv_totals(L, t, units, out);
}

cudaError_t tc_backward_shard_state(const Launch& L, const Tensors& t, float* out, float* units) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int P = tcb_segments(G, N);
  const int64_t seg = ((N / 128 + P - 1) / P) * 128;
  const int A = agg_split(G, seg, P);
  CUtensorMap mQ, mW, mO;
  if (!make_tma_map(&mO, t.o, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mQ, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mW, t.w, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  BwdParams pa{t.o, t.g, nullptr, nullptr, nullptr, nullptr, units, N, seg / A, P * A, L.a, L.b, 0, 1, 0, A,
               nullptr, nullptr, nullptr, 0};
  auto aggR = bf ? k_bwd_aggR_tc<true> : k_bwd_aggR_tc<false>;
  cudaFuncSetAttribute(aggR, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggRSmem);
  {
    ProfScope ps("la_bwd_shard_state", L.stream);
    aggR<<<dim3(A * P, G), 320, kAggRSmem, L.stream>>>(mQ, mW, mO, mW, pa);
  }
  note_launch(1);
  return tc_sum_units(units, G, P * A, out, L.stream);
}

cudaError_t tc_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws) {
  if (!L.causal) return tc_backward_full(L, t, dq, dk, dv, ws);
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int P = tcb_segments(G, N);
  const int64_t c128 = N / 128;
  const int64_t seg = ((c128 + P - 1) / P) * 128;
  const int64_t SZ = state_floats(kD);
  // S records: the paired forward's saved end states when they match this
  // segmentation (no K/V re-read), else computed by the aggregate pass.
  const float* sv = L.saved_in;
  const bool use_saved = sv != nullptr;  // validated by the ABI layer
  if (use_saved && bwd_pair_rule(G) && G % 2 == 0) return tc_backward_pair(L, t, dq, dk, dv);
  const int A = bwd_agg_split(seg, P, sv != nullptr);  // the W_hat pass covers every segment
  float* stS = ws.base;
  float* stR = stS + G * P * A * SZ;
  float* cmb = stR + G * P * A * SZ;
  CUtensorMap mQ, mK, mV, mW, mO, mWh;
  if (!make_tma_map(&mO, t.o, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mQ, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mK, t.k, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mW, t.w, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mWh, dv, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))  // W_hat^T staged in dV
    return cudaErrorInvalidValue;
  // The W_hat pass + R aggregate runs over every unit of seg / A rows (the sweep
  // reads W_hat^T and s from it; the R sums of segments 1..P-1 feed the earlier
  // segments' suffix). Without the forward's saved S records a second aggregate
  // sums S per unit for the inclusive prefix. The main kernel's prologue sums the
  // unit records.
  BwdParams prm{t.o, t.g, dq, dk, dv, use_saved ? const_cast<float*>(sv + kSavedHeader) : stS, stR, N, seg, P,
                L.a, L.b, 0, use_saved ? 1 : 0, 0, A, L.carry_prefix, L.carry_suffix, cmb,
                tuning().prefetch > 0 ? tuning().prefetch : kBPrefetch};
  prm.row_offset = L.row_offset;
  if (use_saved) {  // checkpoints follow the G * P segment records (la_sm100.cu, tc_forward)
    prm.ck = sv + kSavedHeader + G * P * SZ;
    prm.ck_K = ck_count(N);
  } else if (A > 1) {  // unit-boundary prefixes from the S aggregate (after cmb)
    prm.ck = cmb + G * P * 2 * SZ;
    prm.ck_unit = seg / A;
  }
  BwdParams pa = prm;  // aggregate launch: unit geometry
  pa.stS = stS;
  pa.seg_len = seg / A;
  pa.P = P * A;
  pa.p0 = 0;
  pa.store_w = 1;
  pa.r_unit0 = A;  // segment 0 R records would feed no sweep: its units only write W_hat^T / s
  auto agg = bf ? k_bwd_agg_tc<true> : k_bwd_agg_tc<false>;
  auto main_k = bf ? k_bwd_tc<true> : k_bwd_tc<false>;
  cudaFuncSetAttribute(agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggSmemB);
  cudaFuncSetAttribute(main_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMainSmemB);
  int launches = 2;
  if (!use_saved) {
    ProfScope ps("la_bwd_agg_s", L.stream);
    agg<<<dim3(A * P, G), 192, kAggSmemB, L.stream>>>(mQ, mK, mV, mW, pa);
    launches += 1;
  }
  {
    auto aggR = bf ? k_bwd_aggR_tc<true> : k_bwd_aggR_tc<false>;
    cudaFuncSetAttribute(aggR, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggRSmem);
    ProfScope ps("la_bwd_agg", L.stream);
    aggR<<<dim3(A * P, G), 320, kAggRSmem, L.stream>>>(mQ, mW, mO, mWh, pa);
  }
  if (P > 1 && (P - 1) * A > kScanMinRecords) {  // many unit records: one scan launch, not a chain per CTA
    const int U = P * A;
    cudaError_t e = seg_scan(stR, G, U, A, SZ, L.carry_suffix, cmb + SZ, 2 * SZ, 2, nullptr, L.stream, "la_bwd_scan");
    if (e == cudaSuccess && !use_saved)
      e = seg_scan(stS, G, U, A, SZ, L.carry_prefix, cmb, 2 * SZ, 1, A > 1 ? const_cast<float*>(prm.ck) : nullptr,
                   L.stream, "la_bwd_scan_s");
    if (e != cudaSuccess) return e;
    prm.cmb_ready = 1;
    launches += 1 + (use_saved ? 0 : 1);
  }
  {
    ProfScope ps("la_bwd_causal", L.stream);
    main_k<<<dim3(P, G), kBwdThreads, kMainSmemB, L.stream>>>(mQ, mK, mV, mWh, prm);
  }
  note_launch(launches);
  return cudaGetLastError();
}

}  // namespace lab

extern "C" int la_internal_trace_read_bwd(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lab::g_trace_b, sizeof(lab::g_trace_b));
}
