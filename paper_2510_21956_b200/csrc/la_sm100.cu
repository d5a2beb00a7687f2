// sm_100a tensor-core path: chunked causal linear attention, f(x) = a + b*x.
//
// Forward (replaces forward_kernels.hpp run_forward<T>, causal, D = 128):
//   the sequence of each group g is cut into P segments; a segment is walked in
//   chunks of C = 128 rows with the running state S^T = sum v k^T (fp32, TMEM),
//   z = sum k and sigma = sum v (fp32). Per chunk (rows i, t in the chunk):
//     T1  = Q K^T                                  tcgen05, TMEM   (lanes i)
//     P'  = tril(a + b T1) -> bf16 smem; g_i = rowsum(P') + a*row0 + b q_i.z
//     O^T = V^T P'^T + bf16(b S^T) Q^T             tcgen05, TMEM   (lanes j)
//     S^T += V^T K                                 tcgen05, TMEM   (lanes j)
//     o_ij = (O^T[j][i] + a sigma_j) / g_i -> bf16 -> TMA store (FeatureMajor)
//   Warp roles: warp 0 TMA producer, warp 1 MMA issuer (+TMEM owner), warps 2-5
//   the TMEM<->register epilogue. Q/K/V tiles arrive by TMA (128B swizzle) in a
//   2-stage ring. Segment carries come from an aggregate pass (S, z, sigma per
//   segment via the same tcgen05 state MMA) and an exclusive scan.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace lab {

using namespace sm100;

// Pipeline tracing (diagnostics): CTA (0,0) records clock64 stamps per role,
// chunk and event; read back with la_internal_trace_read (not part of the ABI).
__device__ unsigned long long g_trace[4][64][8];
__device__ __forceinline__ void trace(int role, int c, int ev) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && c < 64) g_trace[role][c][ev] = clock64();
}

namespace {

constexpr int kC = 128;          // chunk rows
constexpr int kD = 128;          // head dim handled here
constexpr int kTile = kC * kD * 2;  // 32 KB: one 128x128 16-bit tile (2 SW128 panels)
constexpr int kPanel = 128 * 128;   // bytes per 64-column panel of 128 rows

// TMEM columns (forward main)


// A (rows x 128) 16-bit tile of a row-major [R][inner] matrix as two SW128 panels.
bool make_map(CUtensorMap* m, const void* base, bool bf16, uint64_t rows, uint64_t inner) {
  return make_tma_map(m, base, bf16, rows, inner, 128, 2);
}

// K-major SW128 descriptor for k-step ks (16 elements) of a 128-row tile.
__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int ks) {
  return sdesc_sw128(tile + (ks >> 2) * kPanel + (ks & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor for k-step ks: K rows of 128 B, MN panels kPanel apart.
__device__ __forceinline__ uint64_t mndesc(uint32_t tile, int ks) {
  return sdesc_sw128(tile + ks * 2048, kPanel, 1024);
}

struct FwdParams {
  const float* states;  // per (g, segment) exclusive-prefix records, or null (no carry)
  float* gout;          // G*N
  unsigned long long* flag;
  int64_t N, G;
  int64_t seg_len;      // rows per segment (multiple of kC)
  int P;
  int64_t row_offset;
  float a, b;
  float* st_out;        // per-(group, segment) end state (S, z, sigma, rows) for the backward, or null
};

// ================================================================ forward main
// Chunks of C = 64 rows, 3-stage TMA ring. Warp roles (320 threads):
// 0 TMA producer; 1 MMA issuer + TMEM owner; 2-5 "WG-A" (S^T -> bf16 operand,
// T1 -> P', g, z); 6-9 "WG-B" (O^T -> o -> TMA store, sigma).
// TMEM: [0,64) T1 (M=64: lanes 0-15 of each quadrant), [64,192) O^T x2,
// [192,320) S^T, [320,448) bf16(b S^T) x2.
constexpr int kCF = 64;                 // forward chunk rows
constexpr int kFT = 16384;              // 64x128 / 128x64 16-bit tile
constexpr int kFStages = 3;
constexpr int kFStage = 3 * kFT;        // Q, K, V^T
constexpr uint32_t kF_T1 = 0, kF_OT = 64, kF_ST = 192, kF_SB = 320;

__device__ __forceinline__ uint64_t kd64(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile + (ks >> 2) * rows * 128 + (ks & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mn64(uint32_t tile, int ks, uint32_t panel) {
  return sdesc_sw128(tile + ks * 2048, panel, 1024);
}

template <bool kBF16>
__global__ void __launch_bounds__(320, 1)
    k_fwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
             FwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sP = smem + kFStages * kFStage;   // [2][8K]   P' (rows i, cols t)
  uint8_t* sO = sP + 2 * 8192;               // [2][16K]  O^T staging (rows j, cols i)
  uint64_t* bars = (uint64_t*)(sO + 2 * kFT);
  uint64_t* full = bars;            // [3]
  uint64_t* empty = bars + 3;       // [3]
  uint64_t* t1_full = bars + 6;
  uint64_t* t1_empty = bars + 7;
  uint64_t* sb_ready = bars + 8;
  uint64_t* st_full = bars + 9;
  uint64_t* p_ready = bars + 10;
  uint64_t* o_full = bars + 11;     // [2]
  uint64_t* ot_empty = bars + 13;   // [2]
  uint64_t* a2b = bars + 15;        // [4]
  uint32_t* tslot = (uint32_t*)(bars + 19);
  float* ginv_s = (float*)(bars + 20);  // [4][64]
  float* zq = ginv_s + 4 * kCF;         // [128]

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = (int)((s1 - s0) / kCF);
  const uint32_t warp = warp_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmO);
    for (int s = 0; s < kFStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 128 + 128);
    }
    mbar_init(t1_full, 1);
    mbar_init(t1_empty, 128);
    mbar_init(sb_ready, 128);
    mbar_init(st_full, 1);
    mbar_init(p_ready, 128);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&ot_empty[b], 128);
    }
    for (int b = 0; b < 4; ++b) mbar_init(&a2b[b], 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const float* st_in = prm.states ? prm.states + (grp * prm.P + p) * state_floats(kD) : nullptr;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c % kFStages;
        if (lane_id() == 0) trace(3, c, 0);
        if (c >= kFStages) mbar_wait(&empty[s], ((c / kFStages) & 1) ^ 1);
        trace(3, c, 1);
        const int64_t row0 = s0 + (int64_t)c * kCF;
        uint8_t* st = smem + s * kFStage;
        mbar_expect_tx(&full[s], kFStage);
        tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kFT, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + 2 * kFT, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Per chunk: M3(c) S^T update, M1(c+1) next T1, M2(c) O^T.
    constexpr uint32_t fmt = kBF16 ? 1 : 0;
    const uint32_t id_T1 = idesc_f16(64, 64, fmt, 0, 0);
    const uint32_t id_ST = idesc_f16(128, 128, fmt, 0, 1);
    const uint32_t id_OT = idesc_f16(128, 64, fmt, 0, 0);
    const uint32_t a0 = smem_u32(smem), aP = smem_u32(sP);
    if (nc > 0) {
      mbar_wait(&full[0], 0);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + kF_T1, kd64(a0, ks, 64), kd64(a0 + kFT, ks, 64), id_T1, ks > 0);
        mma_commit(t1_full);
      }
      __syncwarp();
    }
    for (int c = 0; c < nc; ++c) {
      const int s = c % kFStages, b = c & 1;
      const uint32_t aQ = a0 + s * kFStage, aK = aQ + kFT, aV = aQ + 2 * kFT;
      if (lane_id() == 0) trace(0, c, 0);
      mbar_wait(sb_ready, c & 1);
      if (lane_id() == 0) trace(0, c, 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 4; ++ks)  // S^T += V^T K  (A: V^T rows j, K-major; B: K (N=m, K=t) MN-major)
          mma_ss(tmem + kF_ST, kd64(aV, ks, 128), mn64(aK, ks, 8192), id_ST, 1);
        mma_commit(st_full);
      }
      __syncwarp();
      if (c + 1 < nc) {
        const int sn = (c + 1) % kFStages;
        const uint32_t aQn = a0 + sn * kFStage;
        mbar_wait(&full[sn], ((c + 1) / kFStages) & 1);
        if (lane_id() == 0) trace(0, c, 2);
        mbar_wait(t1_empty, c & 1);
        if (lane_id() == 0) trace(0, c, 3);
        tc_fence_after();
        if (elect_one()) {
          for (int ks = 0; ks < 8; ++ks)  // T1(c+1) = Q K^T (M=64)
            mma_ss(tmem + kF_T1, kd64(aQn, ks, 64), kd64(aQn + kFT, ks, 64), id_T1, ks > 0);
          mma_commit(t1_full);
        }
        __syncwarp();
      }
      mbar_wait(p_ready, c & 1);
      if (lane_id() == 0) trace(0, c, 4);
      if (c >= 2) mbar_wait(&ot_empty[b], ((c - 2) >> 1) & 1);
      if (lane_id() == 0) trace(0, c, 5);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem + kF_OT + b * 64;
        for (int ks = 0; ks < 4; ++ks)  // O^T = V^T P'^T
          mma_ss(d, kd64(aV, ks, 128), kd64(aP + b * 8192, ks, 64), id_OT, ks > 0);
        for (int ks = 0; ks < 8; ++ks)  // O^T += bf16(b S^T) Q^T  (A from TMEM)
          mma_ts(d, tmem + kF_SB + b * 64 + ks * 8, kd64(aQ, ks, 64), id_OT, 1);
        mma_commit(&o_full[b]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ WG-A (warps 2..5)
    const uint32_t qd = warp & 3;
    const int l = (int)lane_id();
    const int r = (int)(qd * 32) + l;              // full-lane row (j of S^T)
    const int ih = (int)(qd * 16) + (l & 15);      // row i of the M=64 T1
    const bool lower = l < 16;
    const uint32_t lane_base = (qd * 32u) << 16;
    const int et = (int)threadIdx.x - 64;          // 0..127
    const float a = prm.a, b = prm.b;
    for (int m0 = 0; m0 < kD; m0 += 32) {  // carry-in S^T row r = S[:, r]
      uint32_t v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = st_in ? __float_as_uint(st_in[(m0 + u) * kD + r]) : 0u;
      tmem_st32(tmem + lane_base + kF_ST + m0, v);
    }
    tmem_st_wait();
    zq[r] = st_in ? st_in[kD * kD + r] : 0.f;
    tc_fence_before();
    named_bar(1, 128);
    tc_fence_after();

    for (int c = 0; c < nc; ++c) {
      const int s = c % kFStages, bb = c & 1;
      const int64_t row0 = s0 + (int64_t)c * kCF;
      const uint8_t* q_t = smem + s * kFStage;
      const uint8_t* k_t = q_t + kFT;
      // ---- E2: S^T -> bf16(b S^T) in TMEM buffer bb
      if (et == 0) trace(1, c, 0);
      if (c >= 1) mbar_wait(st_full, (c - 1) & 1);
      if (et == 0) trace(1, c, 1);
      tc_fence_after();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t x0[32], x1[32], pk[32];
        tmem_ld32(tmem + lane_base + kF_ST + half * 64, x0);
        tmem_ld32(tmem + lane_base + kF_ST + half * 64 + 32, x1);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          pk[u] = pack2<kBF16>(b * __uint_as_float(x0[2 * u]), b * __uint_as_float(x0[2 * u + 1]));
          pk[16 + u] = pack2<kBF16>(b * __uint_as_float(x1[2 * u]), b * __uint_as_float(x1[2 * u + 1]));
        }
        tmem_st32(tmem + lane_base + kF_SB + bb * 64 + half * 32, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(sb_ready);
      if (et == 0) trace(1, c, 2);

      // ---- E1: T1 -> P' (registers, lower lanes); q.z_prev (upper lanes)
      mbar_wait(&full[s], (c / kFStages) & 1);
      mbar_wait(t1_full, c & 1);
      if (et == 0) trace(1, c, 3);
      tc_fence_after();
      uint32_t pk[32];
      float rowsum = 0.f;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t x[32];
        tmem_ld32(tmem + lane_base + kF_T1 + cc * 32, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int t0 = cc * 32 + 2 * u;
          const float p0 = t0 <= ih ? a + b * __uint_as_float(x[2 * u]) : 0.f;
          const float p1 = t0 + 1 <= ih ? a + b * __uint_as_float(x[2 * u + 1]) : 0.f;
          rowsum += p0 + p1;
          pk[cc * 16 + u] = pack2<kBF16>(p0, p1);
        }
      }
      tc_fence_before();
      mbar_arrive(t1_empty);
      if (et == 0) trace(1, c, 7);
      float qz = 0.f;
      if (!lower) {
#pragma unroll 4
        for (int m8 = 0; m8 < kD; m8 += 8) {
          const uint4 v4 = *(const uint4*)(q_t + sw128_off(ih, m8, kCF));
          const float4 za = *(const float4*)(zq + m8), zb = *(const float4*)(zq + m8 + 4);
          const float2 f0 = unpack2<kBF16>(v4.x), f1 = unpack2<kBF16>(v4.y);
          const float2 f2 = unpack2<kBF16>(v4.z), f3 = unpack2<kBF16>(v4.w);
          qz += f0.x * za.x + f0.y * za.y + f1.x * za.z + f1.y * za.w + f2.x * zb.x + f2.y * zb.y +
                f3.x * zb.z + f3.y * zb.w;
        }
      }
      qz = __shfl_xor_sync(0xffffffffu, qz, 16);  // lower lane i receives q_i . z from lane i + 16
      if (lower) {
        const float gi = rowsum + a * (float)(prm.row_offset + row0) + b * qz;
        if (fabsf(gi) < kEpsF32) flag_degenerate(prm.flag, grp, prm.row_offset + row0 + ih);
        ginv_s[(c & 3) * kCF + ih] = 1.f / gi;
        prm.gout[grp * prm.N + row0 + ih] = gi;
      }
      if (et == 0) trace(2, c, 6);
      named_bar(1, 128);  // zq reads done, ginv(c) written
      if (et == 0) trace(2, c, 7);
      mbar_arrive(&a2b[c & 3]);
      {  // z_m += sum_t K[t][m]: thread (mg, tg) sums rows [8 tg, 8 tg + 8) of columns [8 mg, 8 mg + 8)
        const int mg = et >> 3, tg = et & 7;
        float zs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int t = 8 * tg; t < 8 * tg + 8; ++t) {
          const uint4 v4 = *(const uint4*)(k_t + sw128_off(t, 8 * mg, kCF));
          const float2 f0 = unpack2<kBF16>(v4.x), f1 = unpack2<kBF16>(v4.y);
          const float2 f2 = unpack2<kBF16>(v4.z), f3 = unpack2<kBF16>(v4.w);
          zs[0] += f0.x; zs[1] += f0.y; zs[2] += f1.x; zs[3] += f1.y;
          zs[4] += f2.x; zs[5] += f2.y; zs[6] += f3.x; zs[7] += f3.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          zs[u] += __shfl_xor_sync(0xffffffffu, zs[u], 1);
          zs[u] += __shfl_xor_sync(0xffffffffu, zs[u], 2);
          zs[u] += __shfl_xor_sync(0xffffffffu, zs[u], 4);
        }
        if (tg == 0) {
          const float4 za = *(const float4*)(zq + 8 * mg), zb = *(const float4*)(zq + 8 * mg + 4);
          *(float4*)(zq + 8 * mg) = make_float4(za.x + zs[0], za.y + zs[1], za.z + zs[2], za.w + zs[3]);
          *(float4*)(zq + 8 * mg + 4) = make_float4(zb.x + zs[4], zb.y + zs[5], zb.z + zs[6], zb.w + zs[7]);
        }
      }
      mbar_arrive(&empty[s]);  // WG-A is done with Q(c), K(c)
      if (et == 0) trace(1, c, 4);
      if (c >= 2) mbar_wait(&o_full[bb], ((c - 2) >> 1) & 1);  // M2(c-2) drained sP[bb]
      if (et == 0) trace(1, c, 5);
      if (lower) {
        uint8_t* pp = sP + bb * 8192;
#pragma unroll
        for (int w = 0; w < 8; ++w)
          *(uint4*)(pp + sw128_off(ih, 8 * w, kCF)) = make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
      }
      fence_proxy_async();
      named_bar(1, 128);  // P' complete; zq updates visible
      mbar_arrive(p_ready);
      if (et == 0) trace(1, c, 6);
    }
    if (prm.st_out && nc > 0) {  // final state for the backward (S, z)
      mbar_wait(st_full, (nc - 1) & 1);
      tc_fence_after();
      float* so = prm.st_out + (grp * prm.P + p) * state_floats(kD);
      for (int m0 = 0; m0 < kD; m0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lane_base + kF_ST + m0, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) so[(m0 + u) * kD + r] = __uint_as_float(x[u]);
      }
      so[kD * kD + r] = zq[r];
      if (r == 0) so[kD * kD + 2 * kD] = (float)(prm.row_offset + s1);
    }
  } else {
    // ------------------------------------------------------------ WG-B (warps 6..9)
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());     // j of O^T
    const uint32_t lane_base = (qd * 32u) << 16;
    const int eb = (int)threadIdx.x - 192;        // 0..127
    const float a = prm.a;
    float sigma = st_in ? st_in[kD * kD + kD + r] : 0.f;
    for (int c = 0; c < nc; ++c) {
      const int s = c % kFStages, bb = c & 1;
      const int64_t row0 = s0 + (int64_t)c * kCF;
      const uint8_t* v_t = smem + s * kFStage + 2 * kFT;
      if (eb == 0) trace(2, c, 0);
      mbar_wait(&o_full[bb], (c >> 1) & 1);
      if (eb == 0) trace(2, c, 1);
      mbar_wait(&a2b[c & 3], (c >> 2) & 1);
      if (eb == 0) trace(2, c, 2);
      tc_fence_after();
      const float asig = a * sigma;
      const float* gv = ginv_s + (c & 3) * kCF;
      uint32_t pk[32];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t x[32];
        tmem_ld32(tmem + lane_base + kF_OT + bb * 64 + cc * 32, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int i0 = cc * 32 + 2 * u;
          pk[cc * 16 + u] = pack2<kBF16>((__uint_as_float(x[2 * u]) + asig) * gv[i0],
                                         (__uint_as_float(x[2 * u + 1]) + asig) * gv[i0 + 1]);
        }
      }
      tc_fence_before();
      mbar_arrive(&ot_empty[bb]);
      if (eb == 0) trace(2, c, 3);
      // sigma_j += sum_t V^T[j][t]   (j = r), for the next chunk
      float vs = 0.f;
#pragma unroll
      for (int t8 = 0; t8 < kCF; t8 += 8) {
        const uint4 v4 = *(const uint4*)(v_t + sw128_off(r, t8, kD));
        const float2 f0 = unpack2<kBF16>(v4.x), f1 = unpack2<kBF16>(v4.y);
        const float2 f2 = unpack2<kBF16>(v4.z), f3 = unpack2<kBF16>(v4.w);
        vs += f0.x + f0.y + f1.x + f1.y + f2.x + f2.y + f3.x + f3.y;
      }
      sigma += vs;
      mbar_arrive(&empty[s]);  // WG-B is done with V(c)
      // staging buffer bb: the store issued two chunks ago must have left it
      if (eb == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      named_bar(2, 128);
      uint8_t* so = sO + bb * kFT;
#pragma unroll
      for (int w = 0; w < 8; ++w)
        *(uint4*)(so + sw128_off(r, 8 * w, kD)) = make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
      fence_proxy_async();
      named_bar(2, 128);
      if (eb == 0) {
        tma_store_3d(&tmO, so, 0, (int)(grp * kD), (int)(row0 / 64));
        tma_store_commit();
        trace(2, c, 4);
      }
    }
    if (eb == 0) tma_store_wait0();
    if (prm.st_out && nc > 0) prm.st_out[(grp * prm.P + p) * state_floats(kD) + kD * kD + kD + r] = sigma;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ================================================================ segment aggregates
// Per (g, segment): S = sum_t k_t^T v_t (stored X[m][j]), z = sum k, sigma = sum v,
// count; the record layout of la_simt.cu's k_seg_sums (internal.h).
template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    k_fwd_agg_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                 float* states, int64_t N, int64_t seg_len, int P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;                  // [2][32K]
  uint8_t* sV = smem + 2 * kTile;      // [2][32K]
  uint64_t* bars = (uint64_t*)(smem + 4 * kTile);
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  uint64_t* done = bars + 4;
  uint32_t* tslot = (uint32_t*)(bars + 8);
  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * seg_len;
  const int64_t s1 = lmin(N, s0 + seg_len);
  const int nc = (int)((s1 - s0) / kC);
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 128);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c & 1;
        if (c >= 2) mbar_wait(&empty[s], ((c >> 1) & 1) ^ 1);
        const int64_t row0 = s0 + (int64_t)c * kC;
        mbar_expect_tx(&full[s], 2 * kTile);
        tma_load_3d(sK + s * kTile, &tmK, &full[s], 0, (int)(grp * N + row0), 0);
        tma_load_3d(sV + s * kTile, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    const uint32_t id_kmn = idesc_f16(128, 128, kBF16 ? 1 : 0, 0, 1);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    for (int c = 0; c < nc; ++c) {
      const int s = c & 1;
      mbar_wait(&full[s], (c >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem, kdesc(aV + s * kTile, ks), mndesc(aK + s * kTile, ks), id_kmn,
                 (c > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (c == nc - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    float zs = 0.f, vs = 0.f;
    for (int c = 0; c < nc; ++c) {
      const int s = c & 1;
      mbar_wait(&full[s], (c >> 1) & 1);
      const uint8_t* k_t = sK + s * kTile;
      const uint8_t* v_t = sV + s * kTile;
#pragma unroll 4
      for (int t8 = 0; t8 < kC; t8 += 8) {
        const uint4 v4 = *(const uint4*)(v_t + sw128_off(r, t8, kD));
        const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 f = unpack2<kBF16>(w4[u]);
          vs += f.x + f.y;
        }
      }
#pragma unroll 8
      for (int t = 0; t < kC; ++t) {
        const uint16_t h = *(const uint16_t*)(k_t + sw128_off(t, r, kC));
        zs += kBF16 ? __bfloat162float(__ushort_as_bfloat16(h)) : __half2float(__ushort_as_half(h));
      }
      mbar_arrive(&empty[s]);
    }
    float* st = states + (grp * P + p) * state_floats(kD);
    if (nc > 0) {
      mbar_wait(done, 0);
      tc_fence_after();
      const uint32_t lane_base = (qd * 32u) << 16;
      for (int m0 = 0; m0 < kD; m0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lane_base + m0, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) st[(m0 + u) * kD + r] = __uint_as_float(x[u]);  // X[m][j=r]
      }
    } else {
      for (int m = 0; m < kD; ++m) st[m * kD + r] = 0.f;
    }
    st[kD * kD + r] = zs;
    st[kD * kD + kD + r] = vs;
    if (r == 0) st[kD * kD + 2 * kD] = (float)(s1 - s0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
}

constexpr size_t kFwdSmem = kFStages * kFStage + 2 * 8192 + 2 * kFT + 256 + (4 * kCF + kD) * 4 + 1024;
constexpr size_t kAggSmem = 4 * kTile + 128 + 1024;

__global__ void k_scan_fwd(float* states, int P, int64_t SZ, const float* carry) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (e >= SZ) return;
  float* base = states + grp * P * SZ + e;
  float run = carry ? carry[grp * SZ + e] : 0.f;
  for (int q = 0; q < P; ++q) {
    const float t = base[q * SZ];
    base[q * SZ] = run;
    run += t;
  }
}

}  // namespace

int tc_segments(int64_t G, int64_t N) {
  const char* e = getenv("LA_SEGMENTS");
  if (e) return (int)lmax(1, atoi(e));
  return choose_segments(G, N);
}

bool tc_forward_supported(const Launch& L, const Tensors& t) {
  return (L.dtype == LA_BF16 || L.dtype == LA_F16) && L.D == kD && L.causal && L.fault == LA_FAULT_NONE &&
         L.N % kC == 0 && t.lq == LA_SEQUENCE_MAJOR && t.lk == LA_SEQUENCE_MAJOR &&
         t.lv == LA_FEATURE_MAJOR && L.G * L.N < (1ll << 31) && L.G * kD < (1ll << 31);
}

size_t tc_forward_ws_floats(int64_t G, int64_t N, int64_t D) {
  if (D != kD || N % kC) return 0;
  const int P = tc_segments(G, N);
  return P > 1 ? (size_t)(G * P * state_floats(kD)) : 0;
}

size_t tc_saved_floats(int64_t G, int64_t N, int64_t D) {
  if (D != kD || N % kC) return kSavedHeader;
  return (size_t)(kSavedHeader + G * tc_segments(G, N) * state_floats(kD));
}

// One CTA per (group, segment). P = 1 walks whole sequences (no carries, no
// aggregate pass); P > 1 takes exclusive-prefix carries from k_fwd_agg_tc + scan.
cudaError_t tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int64_t SZ = state_floats(kD);
  const int P = tc_segments(G, N);
  const int64_t chunks = N / kC;
  const int64_t seg = ((chunks + P - 1) / P) * kC;
  CUtensorMap mK, mV, mQ64, mK64, mV64, mO64;
  if (!make_map(&mK, t.k, bf, (uint64_t)(G * N), kD) || !make_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N) ||
      !make_tma_map(&mQ64, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mK64, t.k, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mV64, t.v, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mO64, out, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  auto main_k = bf ? k_fwd_tc<true> : k_fwd_tc<false>;
  cudaFuncSetAttribute(main_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwdSmem);
  float* saved = L.saved_out ? L.saved_out + kSavedHeader : nullptr;
  const float* states = L.carry_prefix;
  int launches = 1;
  if (P > 1) {
    float* st = ws.base;
    auto agg = bf ? k_fwd_agg_tc<true> : k_fwd_agg_tc<false>;
    cudaFuncSetAttribute(agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggSmem);
    {
      ProfScope ps("la_fwd_agg", L.stream);
      agg<<<dim3(P, G), 192, kAggSmem, L.stream>>>(mK, mV, st, N, seg, P);
    }
    {
      ProfScope ps("la_fwd_scan", L.stream);
      k_scan_fwd<<<dim3((unsigned)((SZ + 255) / 256), (unsigned)G), 256, 0, L.stream>>>(st, P, SZ,
                                                                                      L.carry_prefix);
    }
    states = st;
    launches += 2;
  }
  if (L.saved_out) {
    const float hdr[kSavedHeader] = {kSavedMagic, (float)G, (float)N, (float)kD, (float)P, (float)seg};
    cudaMemcpyAsync(L.saved_out, hdr, sizeof(hdr), cudaMemcpyHostToDevice, L.stream);
  }
  FwdParams prm{states, g, ws.flag, N, G, seg, P, L.row_offset, L.a, L.b, saved};
  {
    ProfScope ps("la_fwd_causal", L.stream);
    main_k<<<dim3(P, G), 320, kFwdSmem, L.stream>>>(mQ64, mK64, mV64, mO64, prm);
  }
  note_launch(launches);
  return cudaGetLastError();
}

}  // namespace lab

extern "C" int la_internal_trace_read(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lab::g_trace, sizeof(lab::g_trace));
}
