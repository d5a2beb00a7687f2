// sm_100a causal backward as a CTA PAIR per group: one 2-CTA cluster sweeps a whole
// group in reverse (C = 64-row chunks), the work split by the state it needs:
//
//   KV CTA (cluster rank 0): dK^T = Q^T dS^T + (b R_next) V^T - b u_next
//                            dV^T = W_hat^T P + (b R_next)^T K^T + a c_next
//                            R += Q^T W_hat   (suffix state, fp32 in TMEM)
//   Q  CTA (cluster rank 1): W_hat = Omega / g, s = rowsum(O .* W_hat)   (the W_hat pass)
//                            dQ = dS K + W_hat (b S_prev)^T - b s z_prev^T
//                            S -= K^T V       (prefix state rebuilt from the forward's
//                                              saved segment-end prefix, exact reloads at
//                                              checkpoints)
//
// with dS = b tril(W_hat V^T - s 1^T) (both CTAs form it: the M=64 MMA is cheaper than a
// DSMEM hand-off) and P = tril(a + b Q K^T). This is backward_kernels.hpp run_backward<T>
// (:292-396): grad_q_causal_core (:21-57) on the Q CTA, grad_k_alpha/beta_core and
// grad_v_causal_core (:59-168) on the KV CTA, with the reference's per-row w_hat / s
// prologue (:33-38) fused into the Q CTA. The Q CTA pushes each chunk's W_hat^T tile
// and s into the KV CTA's shared memory with st.async (DSMEM, counted on the KV CTA's
// mbarrier), so the whole backward reads Q, K, V, O, Omega, g once and writes dQ, dK,
// dV once: the algorithmic 8 D e + 4 bytes per row, in ONE launch.
//
// Why a pair: the single-CTA sweep (la_sm100_bwd.cu) holds both states, five
// accumulators and both bf16 state operands in one SM (TMEM exactly full, two 64 KB
// stages), so every chunk serialises MMAs -> drains -> state conversions. Split over
// two SMs each CTA double-buffers its accumulators and keeps a deeper TMA ring, and
// the R / S state chains run concurrently on separate tensor pipes.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"
#include "bwd_tiles.cuh"

namespace lab {

using namespace sm100;

// clock64 pipeline trace of cluster 0, chunks [kTrW0, kTrW0 + 64): [rank][role][chunk][event].
// Compiled in only with -DLA_TRACE (the kernel is I-cache sensitive); read by
// la_internal_trace_read_pair.
__device__ unsigned long long g_trace_p[2][5][64][4];
#ifndef LA_PAIR_CLUSTER
#define LA_PAIR_CLUSTER 4
#endif
#ifndef LA_TRACE_W0
#define LA_TRACE_W0 256
#endif
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trp(uint32_t rank, int role, int n, int ev) {
#ifdef LA_TRACE
  if (blockIdx.y == 0 && (blockIdx.x % (LA_PAIR_CLUSTER / 2)) == 0 && n >= LA_TRACE_W0 && n < LA_TRACE_W0 + 64 && (threadIdx.x & 31) == 0)
    g_trace_p[rank][role][n - LA_TRACE_W0][ev] = globaltimer_ns();
#endif
}

namespace {

constexpr int kCB = 64;
constexpr int kD = 128;
constexpr int kT64 = 16384;            // a 64 x 128 or 128 x 64 16-bit tile
constexpr uint32_t kHalf = 16u << 16;  // TMEM lane offset of the upper M=64 half

// ---- KV CTA (rank 0) shared memory
constexpr int kKvStages = 2;
constexpr int kKvStage = 3 * kT64;                 // Q | K | V^T
#ifndef LA_PAIR_WSLOTS
#define LA_PAIR_WSLOTS 2
#endif
constexpr int kWSlots = LA_PAIR_WSLOTS;             // W_hat^T tiles written by the Q CTA
constexpr int kPSBufs = kWSlots > 2 ? 1 : 2;       // P / dS buffers (smem: a third W slot or a second P / dS)
constexpr int kKvOffW = kKvStages * kKvStage;      // 96 KB
#ifndef LA_KV_PREFETCH
#define LA_KV_PREFETCH 2
#endif
constexpr int kKvPrefetch = LA_KV_PREFETCH;        // chunks the KV CTA prefetches into L2 ahead
constexpr int kKvOffP = kKvOffW + kWSlots * kT64;  // x kPSBufs: P [64 i][64 t] | dS [64 i][64 t]
constexpr int kKvOffR = kKvOffP + kPSBufs * 16384; // b R [128 m][128 j]
constexpr int kKvOffStg = kKvOffR + 32768;         // 8 warps x 2 KB drain staging
constexpr int kKvEnd = kKvOffStg + 16384;
// ---- Q CTA (rank 1) shared memory
constexpr int kQStages = 3;
constexpr int kQStage = 4 * kT64;                  // K | V^T | Omega^T (-> W_hat^T in place) | O^T
constexpr int kQOffdS = kQStages * kQStage;        // dS [64 i][64 t]
constexpr int kQOffStg = kQOffdS + 8192;           // 4 warps x 4 KB drain staging
constexpr int kQOffOnes = kQOffStg + 16384;        // [16][64] bf16 ones: B of z = K^T 1
constexpr int kQEnd = kQOffOnes + 2048;
constexpr int kDataEnd = kQEnd > kKvEnd ? kQEnd : kKvEnd;
// ---- small area at the same offset in both CTAs: mbarriers, then float rings
constexpr int kNumBars = 32;
constexpr int kFloats = 1280;
constexpr size_t kPairSmem = 1024 + kDataEnd + kNumBars * 8 + kFloats * 4;
static_assert(kPairSmem <= 232448, "pair smem");
constexpr uint32_t kWBytes = kT64 + kCB * 4;
// mbarrier slots. Cross-CTA (fixed in both layouts): the KV CTA's wfull[kWSlots], the Q
// CTA's kvfree[kWSlots] and empty[kQStages] (the KV CTA acknowledges each push there).
constexpr int kBarWfull = 0, kBarKvfree = 3, kBarQempty = 6;
// KV CTA
constexpr int kBarKFull = 8, kBarKEmpty = 10, kBarWempty = 12, kBarTdFull = 15, kBarTdEmpty = 17,
              kBarKPs = 19, kBarSR = 21, kBarRFull = 22, kBarDkvFull = 23, kBarDkvEmpty = 25;
// Q CTA
constexpr int kBarQFull = 9, kBarWReady = 12, kBarSFull = 15, kBarSS = 16, kBarDptFull = 17, kBarQPs = 19,
              kBarDqFull = 20, kBarDqEmpty = 22;
static_assert(kBarQempty + kQStages <= kBarQFull && kBarDkvEmpty + 2 < 31 && kBarDqEmpty + 2 < 31 &&
              kWSlots <= 3, "barrier map");
// Cluster of kCl CTAs = kCl / 2 pairs: ranks [0, kCl/2) are the KV CTAs of groups
// blockIdx.y * kCl/2 + rank, ranks [kCl/2, kCl) their Q CTAs (peer = rank ^ kCl/2), so
// neighbouring SMs run the same role.
constexpr int kCl = LA_PAIR_CLUSTER;  // per chunk pushed to the KV CTA: W_hat^T + s

struct PairParams {
  const void* o;   // O^T [G][D][N]
  const float* g;  // [G][N]
  void* dq;        // [G][N][D]
  void* dk;        // [G][D][N]
  void* dv;        // [G][D][N]
  int64_t N;
  float a, b;
  const float* seg_rec;  // the forward's saved inclusive prefix at each segment end [G][Pf]
  int Pf;
  int64_t segf;
  const float* ck;  // the forward's exact prefix checkpoints [G][ck_K] (internal.h, kCkC0)
  int ck_K;
  int64_t row_offset;     // global index of row 0 (sequence shards)
  const float* carry_suf; // [G] exclusive suffix (R, u, c) after the last row, or null
};

// b * X (a 128 x 128 fp32 state in TMEM, lane r = row) -> bf16 SW128 K-major smem operand.
// The next 32 columns' tcgen05.ld is in flight while the current ones are converted.
template <bool kBF16>
__device__ __forceinline__ void cvt32_store(const uint32_t (&x)[32], uint8_t* dst, int r, int j0, float b) {
#pragma unroll
  for (int w8 = 0; w8 < 4; ++w8) {
    uint4 v;
    v.x = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 0]), b * __uint_as_float(x[8 * w8 + 1]));
    v.y = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 2]), b * __uint_as_float(x[8 * w8 + 3]));
    v.z = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 4]), b * __uint_as_float(x[8 * w8 + 5]));
    v.w = pack2<kBF16>(b * __uint_as_float(x[8 * w8 + 6]), b * __uint_as_float(x[8 * w8 + 7]));
    *(uint4*)(dst + sw128_off(r, j0 + 8 * w8, 128)) = v;
  }
}
// The epilogue helpers below are out of line: the two CTAs of a pair run different roles,
// and shared call sites keep each role's hot code small (instruction-cache bound otherwise).
template <bool kBF16>
__device__ __noinline__ void state_to_smem(uint32_t taddr, uint8_t* dst, int r, float b) {
  uint32_t xa[32], xb[32];
  tmem_ld32(taddr, xa);
  tmem_ld_wait();
  tmem_ld32(taddr + 32, xb);
  cvt32_store<kBF16>(xa, dst, r, 0, b);
  tmem_ld_wait();
  tmem_ld32(taddr + 64, xa);
  cvt32_store<kBF16>(xb, dst, r, 32, b);
  tmem_ld_wait();
  tmem_ld32(taddr + 96, xb);
  cvt32_store<kBF16>(xa, dst, r, 64, b);
  tmem_ld_wait();
  cvt32_store<kBF16>(xb, dst, r, 96, b);
}

// E1 for 32 columns [t0, t0 + 32) of an M=64 accumulator half: row ih gets
// t <= ih ? b x + alpha : 0 in bf16 (P = a + b T1 with alpha = a; dS = b dPt - b s with
// alpha = -b s). The TMEM load is warp-collective; lanes with !act only take part in it.
template <bool kBF16>
__device__ __noinline__ void e1_cols(uint32_t taddr, uint8_t* dst, int ih, int t0, float b, float alpha, bool act) {
  uint32_t x[32];
  tmem_ld32(taddr, x);
  tmem_ld_wait();
  if (!act) return;
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
}

// Drain 64 columns of an M=128 accumulator (lane = feature row) + bias -> bf16, arrive on
// `empty` once TMEM is read, then the warp's 32 rows x 128 B go out as coalesced
// FeatureMajor rows (row seg at dst + seg * N) through a 2 KB transpose scratch.
template <bool kBF16>
__device__ __noinline__ void drain64_fm(uint32_t taddr, float bias, uint64_t* empty, uint8_t* scratch, uint16_t* dst,
                                        int64_t N) {
  uint4 vt[8];
#pragma unroll
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t x[32];
    tmem_ld32(taddr + c0, x);
    tmem_ld_wait();
#pragma unroll
    for (int w4 = 0; w4 < 4; ++w4) {
      uint32_t k4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        k4[q] = pack2<kBF16>(__uint_as_float(x[8 * w4 + 2 * q]) + bias, __uint_as_float(x[8 * w4 + 2 * q + 1]) + bias);
      vt[c0 / 8 + w4] = make_uint4(k4[0], k4[1], k4[2], k4[3]);
    }
  }
  tc_fence_before();
  mbar_arrive(empty);
  warp_store_rows_2k(scratch, vt, [&](int seg) { return dst + seg * N; });
}

// ================================================================ KV CTA
template <bool kBF16>
__device__ __forceinline__ void kv_role(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                        const PairParams& prm, const int64_t grp, const int nc, uint8_t* smem,
                                        uint64_t* bars, float* fl, const uint32_t tmem) {
  uint64_t* wfull = bars + kBarWfull;     // [kWSlots] W_hat^T + s of the chunk pushed by the Q CTA
  uint64_t* full = bars + kBarKFull;      // [2]
  uint64_t* empty = bars + kBarKEmpty;    // [2]
  uint64_t* wempty = bars + kBarWempty;   // [kWSlots] W slot consumed (MMAs + WG-C)
  uint64_t* td_full = bars + kBarTdFull;  // [2] T1 / dPt accumulators
  uint64_t* td_empty = bars + kBarTdEmpty;  // [2]
  uint64_t* ps_ready = bars + kBarKPs;    // [2] P, dS of buffer n & 1 in smem (per buffer: E1(n + 1)
                                          // may finish before the MMA waits for E1(n))
  uint64_t* sR_ready = bars + kBarSR;     // b R_next in smem
  uint64_t* r_full = bars + kBarRFull;    // R += of the chunk retired
  uint64_t* dkv_full = bars + kBarDkvFull;    // [2]
  uint64_t* dkv_empty = bars + kBarDkvEmpty;  // [2]
  float* s_w = fl;          // [kWSlots][64] s of the chunk in each W slot (pushed)
  float* du_s = fl + 192;   // [4][128] du per chunk (WG-C -> WG-B's dK^T drain)
  float* dcp = fl + 704;    // [4][128] dc per chunk (WG-C -> WG-A's dV^T drain)
  uint8_t* sW = smem + kKvOffW;
  uint8_t* sPdS = smem + kKvOffP;  // buffer b: P at b * 16 KB, dS 8 KB after it
  uint8_t* sR = smem + kKvOffR;
  uint8_t* stg = smem + kKvOffStg;
  // TMEM: T1 / dPt x2 (dPt lower lane half, T1 upper), dK^T x2, dV^T x2, R
  auto kTD = [](int s) -> uint32_t { return 64u * s; };
  auto kDK = [](int s) -> uint32_t { return 128u + 64u * s; };
  auto kDV = [](int s) -> uint32_t { return 256u + 64u * s; };
  constexpr uint32_t kR = 384;
  const int64_t N = prm.N;
  auto row_of = [&](int n) -> int64_t { return (int64_t)(nc - 1 - n) * kCB; };
  const uint32_t warp = warp_id();
  const float* recR = prm.carry_suf ? prm.carry_suf + grp * state_floats(kD) : nullptr;

  if (warp < 4) {
    regs_dec<96>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (reverse)
      if (elect_one()) {
        #pragma unroll 1
        for (int n = 0; n < nc; ++n) {
          const int s = n & 1;
          if (n >= 2) mbar_wait_h(&empty[s], ((n >> 1) & 1) ^ 1);
          const int64_t row0 = row_of(n);
          uint8_t* st = smem + s * kKvStage;
          mbar_expect_tx(&full[s], kKvStage);
          tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * N + row0), 0);
          tma_load_3d(st + kT64, &tmK, &full[s], 0, (int)(grp * N + row0), 0);
          tma_load_3d(st + 2 * kT64, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
          if (n + kKvPrefetch < nc) {  // L2 prefetch ahead of the 2-stage ring (DRAM latency)
            const int64_t rp = row_of(n + kKvPrefetch);
            tma_prefetch_l2_3d(&tmQ, 0, (int)(grp * N + rp), 0);
            tma_prefetch_l2_3d(&tmK, 0, (int)(grp * N + rp), 0);
            tma_prefetch_l2_3d(&tmV, 0, (int)(grp * kD), (int)(rp / 64));
          }
        }
      }
    } else if (warp == 2) {
      // ---------------------------------------------------------- W slot arming: each use of
      // a slot expects the Q CTA's push (it may land before or after the arming)
      if (elect_one()) {
#pragma unroll 1
        for (int n = 0; n < nc; ++n) {
          const int w = n % kWSlots;
          if (n >= kWSlots) mbar_wait_h(&wempty[w], ((n / kWSlots) & 1) ^ 1);
          mbar_expect_tx(&wfull[w], kWBytes);
        }
      }
    } else if (warp == 3) {
      // ---------------------------------------------------------- hand-offs to the Q CTA
      // (1) a landed push has read the Q CTA's stage: part of that stage's empty barrier;
      // (2) a consumed W slot may be overwritten. (2) follows (1) for every chunk, so the
      // Q CTA cannot push chunk n + kWSlots before this warp has seen chunk n land (no
      // waiter here can fall two phases behind).
      if (elect_one()) {
        const uint32_t peer = cluster_ctarank() ^ (kCl / 2);
        const uint32_t qempty = mapa(smem_u32(bars + kBarQempty), peer), qfree = mapa(smem_u32(bars + kBarKvfree), peer);
#pragma unroll 1
        for (int n = 0; n < nc; ++n) {
          const int w = n % kWSlots;
          mbar_wait_cluster(&wfull[w], (n / kWSlots) & 1);
          mbar_arrive_remote(qempty + 8u * (n % kQStages));
          trp(0, 4, n, 0);
          mbar_wait_h(&wempty[w], (n / kWSlots) & 1);
          trp(0, 4, n, 1);
          mbar_arrive_remote(qfree + 8u * w);
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t f = kBF16 ? 1 : 0;
      const uint32_t id_T1 = idesc_f16(64, 64, f, 0, 0);
      const uint32_t id_dPt = idesc_f16(64, 64, f, 1, 1);
      const uint32_t id_dK1 = idesc_f16(128, 64, f, 1, 1);
      const uint32_t id_dK2 = idesc_f16(128, 64, f, 0, 1);
      const uint32_t id_dV1 = idesc_f16(128, 64, f, 0, 1);
      const uint32_t id_dV2 = idesc_f16(128, 64, f, 1, 0);
      const uint32_t id_R = idesc_f16(128, 128, f, 1, 0);
      const uint32_t aPdS = smem_u32(sPdS), aR = smem_u32(sR);
      auto issue_td = [&](int n) {  // T1 = Q K^T (upper lanes), dPt = W_hat V^T (lower lanes)
        const int s = n & 1, w = n % kWSlots;
        const uint32_t bQ = smem_u32(smem + s * kKvStage), bK = bQ + kT64, bV = bQ + 2 * kT64,
                       bW = smem_u32(sW + w * kT64);
        trp(0, 0, n, 2);
        mbar_wait_h(&full[s], (n >> 1) & 1);
        mbar_wait_cluster(&wfull[w], (n / kWSlots) & 1);
        if (n >= 2) mbar_wait_h(&td_empty[s], ((n >> 1) & 1) ^ 1);
        trp(0, 0, n, 3);
        fence_proxy_async();  // the st.async-written W_hat^T is read by the tensor core
        tc_fence_after();
        if (elect_one()) {
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            mma_ss(tmem + kTD(s) + kHalf, kd(bQ, ks, 64), kd(bK, ks, 64), id_T1, ks > 0);
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            mma_ss(tmem + kTD(s), mn(bW, ks, 8192), mn(bV, ks, 8192), id_dPt, ks > 0);
          mma_commit(&td_full[s]);
        }
        __syncwarp();
      };
      auto td_ready = [&](int n) -> bool {  // the inputs of issue_td(n) are there (non-blocking)
        const int s = n & 1;
        return mbar_test(&full[s], (n >> 1) & 1) && mbar_test_cluster(&wfull[n % kWSlots], (n / kWSlots) & 1) &&
               (n < 2 || mbar_test(&td_empty[s], ((n >> 1) & 1) ^ 1));
      };
      if (nc > 0) issue_td(0);
      #pragma unroll 1
      for (int n = 0; n < nc; ++n) {
        const int s = n & 1, w = n % kWSlots;
        const uint32_t aQ = smem_u32(smem + s * kKvStage), aK = aQ + kT64, aV = aQ + 2 * kT64,
                       aW = smem_u32(sW + w * kT64), aP = aPdS + (s % kPSBufs) * 16384, adS = aP + 8192;
        trp(0, 0, n, 0);
        mbar_wait_h(sR_ready, n & 1);  // E_R(n) has read R: R += of chunk n may go now
        tc_fence_after();
        if (elect_one()) {
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // R += Q^T W_hat (E_R(n + 1) then overlaps dK / dV(n))
            mma_ss(tmem + kR, mn(aQ, ks, 8192), kd(aW, ks, 128), id_R, 1);
          mma_commit(r_full);
        }
        __syncwarp();
        const bool td_early = n + 1 < nc && td_ready(n + 1);
        if (td_early) issue_td(n + 1);
        mbar_wait_h(&ps_ready[s], (n >> 1) & 1);
        if (n >= 2) mbar_wait_h(&dkv_empty[s], ((n >> 1) & 1) ^ 1);
        trp(0, 0, n, 1);
        tc_fence_after();
        if (elect_one()) {
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // dK^T = Q^T dS^T
            mma_ss(tmem + kDK(s), mn(aQ, ks, 8192), mn(adS, ks, 8192), id_dK1, ks > 0);
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks)  //      + (b R) V^T
            mma_ss(tmem + kDK(s), kd(aR, ks, 128), mn(aV, ks, 8192), id_dK2, 1);
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // dV^T = W_hat^T P
            mma_ss(tmem + kDV(s), kd(aW, ks, 128), mn(aP, ks, 8192), id_dV1, ks > 0);
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks)  //      + (b R)^T K^T
            mma_ss(tmem + kDV(s), mn(aR, ks, 16384), kd(aK, ks, 64), id_dV2, 1);
          mma_commit(&dkv_full[s]);
          mma_commit(&empty[s]);
          mma_commit(&wempty[w]);
        }
        __syncwarp();
        if (n + 1 < nc && !td_early) issue_td(n + 1);
      }
    }
    return;
  }
  regs_inc<136>();
  const uint32_t qd = warp & 3;
  const int l = (int)lane_id();
  const int r = (int)(qd * 32) + l;          // lane of the M=128 accumulators (j or m)
  const int ih = (int)(qd * 16) + (l & 15);  // row i of the M=64 accumulators
  const bool upper = l >= 16;                // lanes 16..31 of a quadrant: the T1 half
  const uint32_t lb = (qd * 32u) << 16;
  const float a = prm.a, b = prm.b;
  // E1 for columns [t0, t0 + 32) of chunk n: P = a + b T1 (upper lanes), dS = b dPt - b s
  // (lower lanes) -> sP / sdS
  auto e1 = [&](int n, int t0) {
    const int s = n & 1, w = n % kWSlots;
    if (t0) trp(0, 1, n, 0);
    mbar_wait_cluster(&wfull[w], (n / kWSlots) & 1);  // s of the chunk (pushed)
    mbar_wait_h(&td_full[s], (n >> 1) & 1);
    if (n >= kPSBufs)  // dK / dV(n - kPSBufs) has read this P / dS buffer
      mbar_wait_h(&dkv_full[(n - kPSBufs) & 1], ((n - kPSBufs) >> 1) & 1);
    if (t0) trp(0, 1, n, 1);
    tc_fence_after();
    const float si = s_w[w * kCB + ih];
    e1_cols<kBF16>(tmem + lb + kTD(s) + t0, sPdS + (s % kPSBufs) * 16384 + (upper ? 0 : 8192), ih, t0, b,
                   upper ? a : -b * si, true);
    fence_proxy_async();
    tc_fence_before();
    mbar_arrive(&td_empty[s]);
    mbar_arrive(&ps_ready[s]);
  };
  if (warp < 8) {
    // ------------------------------------------------------------ WG-A: E1 columns 32..63,
    // dV^T drain (+ a c_next)
    float cj = recR ? recR[kD * kD + kD + r] : 0.f;  // c_next (j = r)
    auto dv_out = [&](int m) {
      const int s = m & 1;
      mbar_wait_h(&dkv_full[s], (m >> 1) & 1);
      trp(0, 1, m, 2);
      tc_fence_after();
      drain64_fm<kBF16>(tmem + lb + kDV(s), a * cj, &dkv_empty[s], stg + qd * 2048,
                        (uint16_t*)prm.dv + (grp * kD + qd * 32) * N + row_of(m), N);
      cj += dcp[(m & 3) * kD + r];
      trp(0, 1, m, 3);
    };
    #pragma unroll 1
    for (int n = 0; n <= nc; ++n) {
      if (n < nc) e1(n, 32);
      if (n >= 1) dv_out(n - 1);
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ WG-B: E_R (b R -> sR),
    // dK^T drain (- b u_next)
    float u = recR ? recR[kD * kD + r] : 0.f;  // u_next (m = r)
    auto er = [&](int n) {  // b R_next(n) -> sR: TMEM read + convert while dK / dV(n-1) still
                            // read sR, the stores once they are done
      trp(0, 2, n, 0);
      if (n >= 1) mbar_wait_h(r_full, (n - 1) & 1);
      trp(0, 2, n, 1);
      tc_fence_after();
      uint32_t pk[64];
#pragma unroll
      for (int j0 = 0; j0 < 4; ++j0) {
        uint32_t x[32];
        tmem_ld32(tmem + lb + kR + 32 * j0, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u)
          pk[16 * j0 + u] = pack2<kBF16>(b * __uint_as_float(x[2 * u]), b * __uint_as_float(x[2 * u + 1]));
      }
      if (n >= 1) mbar_wait_h(&dkv_full[(n - 1) & 1], ((n - 1) >> 1) & 1);
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8)
        *(uint4*)(sR + sw128_off(r, 8 * c8, 128)) = make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(sR_ready);
      trp(0, 2, n, 2);
    };
    auto dk_out = [&](int m) {
      const int s = m & 1;
      mbar_wait_h(&dkv_full[s], (m >> 1) & 1);
      if (m >= 1) u += du_s[((m - 1) & 3) * kD + r];  // suffix sum through chunk m-1
      tc_fence_after();
      drain64_fm<kBF16>(tmem + lb + kDK(s), -b * u, &dkv_empty[s], stg + (4 + qd) * 2048,
                        (uint16_t*)prm.dk + (grp * kD + qd * 32) * N + row_of(m), N);
      trp(0, 2, m, 3);
    };
    #pragma unroll 1
    for (int n = 0; n <= nc; ++n) {
      if (n < nc) er(n);
      if (n >= 1) dk_out(n - 1);
    }
  } else {
    // ------------------------------------------------------------ WG-C: dc (row sums of
    // W_hat^T), E1 columns 0..31, du_m = sum_i q_im s_i
    const int ec = (int)threadIdx.x - 384;
    const int mg = ec >> 3, tg = ec & 7;
    #pragma unroll 1
    for (int n = 0; n < nc; ++n) {
      const int s = n & 1, w = n % kWSlots;
      trp(0, 3, n, 0);
      mbar_wait_cluster(&wfull[w], (n / kWSlots) & 1);
      trp(0, 3, n, 1);
      {  // row j = r of W_hat^T: 8 conflict-free 16-byte chunks
        const uint8_t* w_t = sW + w * kT64;
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
      }
      e1(n, 0);
      trp(0, 3, n, 2);
      mbar_wait_h(&full[s], (n >> 1) & 1);
      {
        const uint8_t* q_t = smem + s * kKvStage;
        const float* sc = s_w + w * kCB;
        float du[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint4 qv[kCB / 8];
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
      mbar_arrive(&wempty[w]);
      trp(0, 3, n, 3);
    }
  }
}

// ================================================================ Q CTA
template <bool kBF16>
__device__ __forceinline__ void q_role(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmW,
                                       const CUtensorMap& tmO,
                                       const PairParams& prm, const int64_t grp, const int nc, uint8_t* smem,
                                       uint64_t* bars, float* fl, const uint32_t tmem) {
  uint64_t* kvfree = bars + kBarKvfree;   // [kWSlots] the KV CTA's W slot may be overwritten
  uint64_t* full = bars + kBarQFull;      // [kQStages]
  uint64_t* empty = bars + kBarQempty;    // [kQStages] MMA commit + WG-C + the KV CTA's push ack
  uint64_t* w_ready = bars + kBarWReady;  // [kQStages] W_hat^T / s of the stage written (local)
  uint64_t* s_full = bars + kBarSFull;    // S -= K^T V retired
  uint64_t* sS_ready = bars + kBarSS;     // bf16 b S_prev in TMEM (and TMEM S read)
  uint64_t* dpt_full = bars + kBarDptFull;  // [2] dPt in TMEM lane half n & 1
  uint64_t* ps_ready = bars + kBarQPs;    // dS in smem
  uint64_t* dq_full = bars + kBarDqFull;  // [2]
  uint64_t* dq_empty = bars + kBarDqEmpty;  // [2]
  float* s_loc = fl + 128;         // [3][64] s per stage (E0 -> E1, drains)
  float* zbuf = fl + 320;          // [4][128] z_prev per chunk; slot 3 = z at the end first
  float* s_ring = fl + 832;        // [4][64] s per chunk for the dQ drain
  float* g_ring = fl + 1088;       // [3][64] g of the stage's rows (bulk-loaded)
  uint8_t* sdS = smem + kQOffdS;
  uint8_t* stg = smem + kQOffStg;
  // TMEM: dPt (M=64, buffer n & 1 in lane half n & 1), dQ^T x2 (M=128 lanes m, 64 columns i),
  // S (fp32), bf16 b S x2 (the A operand of dQ^T += (b S) W_hat^T, packed pairs)
  constexpr uint32_t kDP = 0, kS = 256;
  auto kDQ = [](int b) -> uint32_t { return 64u + 64u * b; };
  auto kBS = [](int b) -> uint32_t { return 384u + 64u * b; };
  auto kZC = [](int b) -> uint32_t { return 192u + 16u * b; };  // column sums K^T 1 of chunk n, x2
  const int64_t N = prm.N;
  const int64_t SZ = state_floats(kD);
  auto row_of = [&](int n) -> int64_t { return (int64_t)(nc - 1 - n) * kCB; };
  // exact exclusive prefix (S, z) at chunk n's first row: a forward segment boundary or
  // a checkpoint row (internal.h, kCkC0)
  auto ck_record = [&](int n) -> const float* {
    if (n >= nc - 1) return nullptr;
    const uint32_t r0 = (uint32_t)(nc - 1 - n) * kCB;  // N < 2^31
    if (r0 % (uint32_t)prm.segf == 0) {  // a forward segment end (segf a multiple of 128)
      const uint32_t p = r0 / (uint32_t)prm.segf - 1;
      if (p < (uint32_t)prm.Pf - 1) return prm.seg_rec + (grp * prm.Pf + p) * SZ;
    }
    const uint64_t gr = (uint64_t)prm.row_offset + r0;  // checkpoint rows kCkC0 * 2^k
    if (gr % kCkC0 || ((gr / kCkC0) & (gr / kCkC0 - 1))) return nullptr;
    const int k = __ffsll((long long)(gr / kCkC0)) - 1;
    return k < prm.ck_K ? prm.ck + (grp * prm.ck_K + k) * SZ : nullptr;
  };
  const uint32_t warp = warp_id();

  if (warp < 4) {
    regs_dec<96>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (reverse)
      if (elect_one()) {
        #pragma unroll 1
        for (int n = 0; n < nc; ++n) {
          const int s = n % kQStages;
          trp(1, 4, n, 0);
          if (n >= kQStages) mbar_wait_h(&empty[s], ((n / kQStages) & 1) ^ 1);
          trp(1, 4, n, 1);
          const int64_t row0 = row_of(n);
          uint8_t* st = smem + s * kQStage;
          mbar_expect_tx(&full[s], kQStage + kCB * 4);
          tma_load_3d(st, &tmK, &full[s], 0, (int)(grp * N + row0), 0);
          tma_load_3d(st + kT64, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
          tma_load_3d(st + 2 * kT64, &tmW, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
          tma_load_3d(st + 3 * kT64, &tmO, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
          bulk_load(g_ring + s * kCB, prm.g + grp * N + row0, kCB * 4, &full[s]);
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t f = kBF16 ? 1 : 0;
      const uint32_t id_dPt = idesc_f16(64, 64, f, 1, 1);
      const uint32_t id_Sneg = idesc_f16(128, 128, f, 1, 0, 1);
      const uint32_t id_dQ1 = idesc_f16(128, 64, f, 1, 0);  // A = K^T (MN-major), B = dS (K-major)
      const uint32_t id_dQ2 = idesc_f16(128, 64, f, 0, 1);  // A = b S (TMEM), B = W_hat^T (MN-major)
      const uint32_t id_Z = idesc_f16(128, 16, f, 1, 0);    // A = K^T (MN-major), B = ones (K-major)
      const uint32_t adS = smem_u32(sdS), aOnes = smem_u32(smem + kQOffOnes);
      auto issue_s = [&](int n) {  // S -= K^T V and the column sums K^T 1 of chunk n
        const int s = n % kQStages;
        const uint32_t bK = smem_u32(smem + s * kQStage), bV = bK + kT64;
        tc_fence_after();
        if (elect_one()) {
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks) mma_ss(tmem + kS, mn(bK, ks, 8192), kd(bV, ks, 128), id_Sneg, 1);
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // column sums of K (z_prev update, read by E_S)
            mma_ss(tmem + kZC(n & 1), mn(bK, ks, 8192), kd(aOnes, ks, 16), id_Z, ks > 0);
          mma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dpt = [&](int n) {  // dPt = W_hat V^T of chunk n (lane half n & 1)
        const int s = n % kQStages;
        const uint32_t bV = smem_u32(smem + s * kQStage) + kT64, bW = bV + kT64;
        mbar_wait_h(&w_ready[s], (n / kQStages) & 1);
        trp(1, 0, n, 3);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + kDP + ((n & 1) ? kHalf : 0u);
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks) mma_ss(d, mn(bW, ks, 8192), mn(bV, ks, 8192), id_dPt, ks > 0);
          mma_commit(&dpt_full[n & 1]);
        }
        __syncwarp();
      };
      if (nc > 0) {
        mbar_wait_h(&full[0], 0);
        issue_s(0);
        issue_dpt(0);
      }
      #pragma unroll 1
      for (int n = 0; n < nc; ++n) {
        const int s = n % kQStages, bb = n & 1;
        const uint32_t aK = smem_u32(smem + s * kQStage), aW = aK + 2 * kT64;
        trp(1, 0, n, 0);
        mbar_wait_h(sS_ready, n & 1);  // E_S(n) has read S: S -= of chunk n + 1 may go now
        const int s1 = (n + 1) % kQStages;
        bool s_early = false;
        if (n + 1 < nc && mbar_test(&full[s1], ((n + 1) / kQStages) & 1)) {
          issue_s(n + 1);
          s_early = true;
        }
        mbar_wait_h(ps_ready, n & 1);
        if (n >= 2) mbar_wait_h(&dq_empty[bb], ((n >> 1) & 1) ^ 1);
        trp(1, 0, n, 1);
        tc_fence_after();
        if (elect_one()) {
          #pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // dQ^T = K^T dS^T
            mma_ss(tmem + kDQ(bb), mn(aK, ks, 8192), kd(adS, ks, 64), id_dQ1, ks > 0);
          #pragma unroll
          for (int ks = 0; ks < 8; ++ks)  //      + (b S) W_hat^T   (A from TMEM)
            mma_ts(tmem + kDQ(bb), tmem + kBS(bb) + ks * 8, mn(aW, ks, 8192), id_dQ2, 1);
          mma_commit(&dq_full[bb]);
          mma_commit(&empty[s]);
        }
        __syncwarp();
        if (n + 1 < nc) {
          trp(1, 0, n + 1, 2);
          if (!s_early) {
            mbar_wait_h(&full[s1], ((n + 1) / kQStages) & 1);
            issue_s(n + 1);
          }
          issue_dpt(n + 1);
        }
      }
    }
    return;
  }
  regs_inc<136>();
  const uint32_t qd = warp & 3;
  const int l = (int)lane_id();
  const int r = (int)(qd * 32) + l;
  const int ih = (int)(qd * 16) + (l & 15);
  const bool upper = l >= 16;
  const uint32_t lb = (qd * 32u) << 16;
  const float b = prm.b;
  if (warp < 8) {
    // ------------------------------------------------------------ WG-A: the W_hat pass (E0)
    // W_hat^T = Omega^T / g in place (bf16), s_i = sum_j o_ji w_hat_ji; each 16-byte piece
    // also goes to the KV CTA's W slot by st.async. 128 threads: rows j = 16 rr + jg,
    // columns i in [8 ig, 8 ig + 8) (conflict-free, see what_pass).
    const int et = (int)threadIdx.x - 128;
    const int jg = et & 15, ig = et >> 4;
    const uint32_t peer = cluster_ctarank() ^ (kCl / 2);
    const uint32_t kv_w = mapa(smem_u32(smem + kKvOffW), peer), kv_s = mapa(smem_u32(fl), peer);
    const uint32_t kv_bar = mapa(smem_u32(bars + kBarWfull), peer);
    #pragma unroll 1
    for (int n = 0; n < nc; ++n) {
      const int s = n % kQStages, w = n % kWSlots;
      trp(1, 1, n, 0);
      mbar_wait_h(&full[s], (n / kQStages) & 1);
      trp(1, 1, n, 1);
      if (n >= kWSlots) mbar_wait_cluster(&kvfree[w], ((n / kWSlots) & 1) ^ 1);
      trp(1, 1, n, 2);
      uint8_t* w_t = smem + s * kQStage + 2 * kT64;
      const uint8_t* o_t = w_t + kT64;
      const float4 g0 = *(const float4*)(g_ring + s * kCB + 8 * ig), g1 = *(const float4*)(g_ring + s * kCB + 8 * ig + 4);
      const float ginv[8] = {__frcp_rn(g0.x), __frcp_rn(g0.y), __frcp_rn(g0.z), __frcp_rn(g0.w),
                             __frcp_rn(g1.x), __frcp_rn(g1.y), __frcp_rn(g1.z), __frcp_rn(g1.w)};
      const uint32_t kvb = kv_bar + 8u * w;
      float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const uint32_t off = sw128_off(16 * rr + jg, 8 * ig, 128);
        uint4* p = (uint4*)(w_t + off);
        const uint4 wv = *p;
        const uint4 ov = *(const uint4*)(o_t + off);
        const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t oa[4] = {ov.x, ov.y, ov.z, ov.w};
        uint32_t res[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 wf = unpack2<kBF16>(wa[u]);
          const float2 of = unpack2<kBF16>(oa[u]);
          const float w0 = wf.x * ginv[2 * u], w1 = wf.y * ginv[2 * u + 1];
          sp[2 * u] += of.x * w0;
          sp[2 * u + 1] += of.y * w1;
          res[u] = pack2<kBF16>(w0, w1);
        }
        *p = make_uint4(res[0], res[1], res[2], res[3]);
      }
      trp(1, 4, n, 2);
      // s_i for this thread's 8 columns: sum over the 16 lanes sharing ig
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) sp[u] += __shfl_xor_sync(0xffffffffu, sp[u], off);
      }
      if (jg == 0) {
        const float4 s0 = make_float4(sp[0], sp[1], sp[2], sp[3]), s1 = make_float4(sp[4], sp[5], sp[6], sp[7]);
        *(float4*)(s_loc + s * kCB + 8 * ig) = s0;
        *(float4*)(s_loc + s * kCB + 8 * ig + 4) = s1;
      }
      trp(1, 4, n, 3);
      fence_proxy_async();
      mbar_arrive(&w_ready[s]);
      named_bar(1, 128);  // W_hat^T and s of the chunk complete -> one bulk DSMEM push
      if (et == 0) {
        bulk_s2s(kv_w + w * kT64, w_t, kT64, kvb);
        bulk_s2s(kv_s + (uint32_t)(w * kCB) * 4u, s_loc + s * kCB, kCB * 4, kvb);
      }
      trp(1, 1, n, 3);
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ WG-B: E_S (bf16 b S_prev ->
    // TMEM), E1 (dS -> smem): the two inputs of dQ^T(n); z_prev per chunk
    float zr = prm.seg_rec[(grp * prm.Pf + prm.Pf - 1) * SZ + kD * kD + r];  // z at N
    auto e1 = [&](int n) {
      const int s = n % kQStages, bb = n & 1;
      mbar_wait_h(&w_ready[s], (n / kQStages) & 1);  // s of the chunk
      mbar_wait_h(&dpt_full[bb], (n >> 1) & 1);
      if (n >= 1) mbar_wait_h(&dq_full[(n - 1) & 1], ((n - 1) >> 1) & 1);  // dQ(n-1) has read sdS
      tc_fence_after();
      const bool act = upper == (bb != 0);  // this lane holds row ih of buffer bb
      const float nbs = -b * s_loc[s * kCB + ih];
      e1_cols<kBF16>(tmem + lb + kDP, sdS, ih, 0, b, nbs, act);
      e1_cols<kBF16>(tmem + lb + kDP + 32, sdS, ih, 32, b, nbs, act);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ps_ready);
    };
    #pragma unroll 1
    for (int n = 0; n < nc; ++n) {
      trp(1, 2, n, 0);
      mbar_wait_h(s_full, n & 1);
      trp(1, 2, n, 1);
      if (n >= 2) mbar_wait_h(&dq_full[n & 1], ((n - 2) >> 1) & 1);  // dQ(n-2) has read b S buffer n & 1
      trp(1, 2, n, 2);
      tc_fence_after();
      const float* ck = ck_record(n);
      {  // z_prev(n) = z_prev(n-1) - sum_t k_t (lane r = m), or the exact reload
        uint32_t c0, c1;
        tmem_ld2(tmem + lb + kZC(n & 1), c0, c1);
        tmem_ld_wait();
        zr = ck ? ck[kD * kD + r] : zr - __uint_as_float(c0);
        zbuf[(n & 3) * kD + r] = zr;
      }
      if (ck) {  // the exact prefix replaces the rebuilt one, in TMEM too
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
      for (int half = 0; half < 2; ++half) {
        uint32_t x0[32], x1[32], pk[32];
        tmem_ld32(tmem + lb + kS + half * 64, x0);
        tmem_ld32(tmem + lb + kS + half * 64 + 32, x1);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          pk[u] = pack2<kBF16>(b * __uint_as_float(x0[2 * u]), b * __uint_as_float(x0[2 * u + 1]));
          pk[16 + u] = pack2<kBF16>(b * __uint_as_float(x1[2 * u]), b * __uint_as_float(x1[2 * u + 1]));
        }
        tmem_st32(tmem + lb + kBS(n & 1) + half * 32, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(sS_ready);
      trp(1, 2, n, 3);
      e1(n);
    }
  } else {
    // ------------------------------------------------------------ WG-C: s ring, dQ drain
    // (- b s_i z_prev)
    const int ec = (int)threadIdx.x - 384;
    auto zs = [&](int n) {  // s(n) -> s_ring for the drain; the stage's s_loc is free again
      const int s = n % kQStages;
      mbar_wait_h(&w_ready[s], (n / kQStages) & 1);  // s of the chunk (E0)
      if (ec < kCB) s_ring[(n & 3) * kCB + ec] = s_loc[s * kCB + ec];
      mbar_arrive(&empty[s]);
    };
    auto dq_out = [&](int m) {  // dQ^T (lanes m) - b s_i z_m -> dQ rows (SequenceMajor)
      const int bb = m & 1;
      mbar_wait_h(&dq_full[bb], (m >> 1) & 1);
      tc_fence_after();
      const float bz = b * zbuf[(m & 3) * kD + r];
      const float4* si4 = (const float4*)(s_ring + (m & 3) * kCB);
      uint8_t* scr = stg + qd * 4096;  // [64 i][32 m] bf16 of this warp's feature slice
#pragma unroll 1
      for (int c0 = 0; c0 < kCB; c0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lb + kDQ(bb) + c0, x);
        tmem_ld_wait();
        if (c0 + 32 == kCB) {
          tc_fence_before();
          mbar_arrive(&dq_empty[bb]);
        }
        float si[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 f4 = si4[c0 / 4 + q];
          si[4 * q] = f4.x; si[4 * q + 1] = f4.y; si[4 * q + 2] = f4.z; si[4 * q + 3] = f4.w;
        }
        // lanes l, l ^ 1 trade columns: even lanes write (m, m + 1) of row i, odd lanes of row i + 1
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          const float v0 = __uint_as_float(x[q]) - bz * si[q];
          const float v1 = __uint_as_float(x[q + 1]) - bz * si[q + 1];
          const bool odd = (l & 1) != 0;
          const float give = odd ? v0 : v1, keep = odd ? v1 : v0;
          const float got = __shfl_xor_sync(0xffffffffu, give, 1);
          const uint32_t w2 = odd ? pack2<kBF16>(got, keep) : pack2<kBF16>(keep, got);
          const int row = c0 + q + (odd ? 1 : 0);
          *(uint32_t*)(scr + row * 64 + (l & ~1) * 2) = w2;
        }
      }
      __syncwarp();
      uint8_t* dqb = (uint8_t*)prm.dq + ((grp * N + row_of(m)) * kD + qd * 32) * 2;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // 256 16-byte pieces: row c >> 2, piece c & 3
        const int c = k * 32 + l;
        *(uint4*)(dqb + (c >> 2) * (kD * 2) + (c & 3) * 16) = *(const uint4*)(scr + (c >> 2) * 64 + (c & 3) * 16);
      }
      __syncwarp();
    };
    #pragma unroll 1
    for (int n = 0; n <= nc; ++n) {
      if (n < nc) {
        trp(1, 3, n, 1);
        zs(n);
        trp(1, 3, n, 2);
      }
      named_bar(2, 128);  // z_prev / s written by other WG-C threads than the ones draining them
      if (n >= 1) {
        dq_out(n - 1);
        trp(1, 3, n - 1, 3);
      }
    }
  }
}

template <bool kBF16>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(512, 1)
    k_bwd_pair_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmO, PairParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bars = (uint64_t*)(smem + kDataEnd);
  float* fl = (float*)(bars + kNumBars);
  uint32_t* tslot = (uint32_t*)(bars + kNumBars - 1);
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank >= kCl / 2 ? 1u : 0u;  // 0: KV CTA, 1: Q CTA
  const int64_t grp = (int64_t)blockIdx.y * (kCl / 2) + (crank % (kCl / 2));
  const int nc = (int)(prm.N / kCB);
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    if (rank == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      for (int i = 0; i < kWSlots; ++i) {
        mbar_init(bars + kBarWfull + i, 1);          // the expect_tx arrival + the pushed bytes
        mbar_init(bars + kBarWempty + i, 1 + 128);   // MMA commit + WG-C
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(bars + kBarKFull + i, 1);
        mbar_init(bars + kBarKEmpty + i, 1 + 128);   // MMA commit + WG-C
        mbar_init(bars + kBarTdFull + i, 1);
        mbar_init(bars + kBarTdEmpty + i, 256);      // WG-A + WG-C
        mbar_init(bars + kBarDkvFull + i, 1);
        mbar_init(bars + kBarDkvEmpty + i, 256);     // WG-A + WG-B
        mbar_init(bars + kBarKPs + i, 256);          // WG-A + WG-C
      }
      mbar_init(bars + kBarSR, 128);
      mbar_init(bars + kBarRFull, 1);
    } else {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmW);
      tma_prefetch(&tmO);
      for (int i = 0; i < kWSlots; ++i) mbar_init(bars + kBarKvfree + i, 1);  // remote arrive
      for (int i = 0; i < 2; ++i) {
        mbar_init(bars + kBarDptFull + i, 1);
        mbar_init(bars + kBarDqFull + i, 1);
        mbar_init(bars + kBarDqEmpty + i, 128);
      }
      for (int i = 0; i < kQStages; ++i) {
        mbar_init(bars + kBarQFull + i, 1);
        mbar_init(bars + kBarQempty + i, 1 + 128 + 1);  // MMA commit + WG-C + the push ack
        mbar_init(bars + kBarWReady + i, 128);          // WG-A
      }
      mbar_init(bars + kBarSFull, 1);
      mbar_init(bars + kBarSS, 128);
      mbar_init(bars + kBarQPs, 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  // initial states in TMEM: R_next (KV: the suffix carry or 0), S at N (Q: the forward's
  // saved inclusive prefix at the last segment end); z at N as chunk "-1"
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp >= 8 && warp < 12) {
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    const uint32_t lb = (qd * 32u) << 16;
    const int64_t SZ = state_floats(kD);
    const float* rec = rank == 0 ? (prm.carry_suf ? prm.carry_suf + grp * SZ : nullptr)
                                 : prm.seg_rec + (grp * prm.Pf + prm.Pf - 1) * SZ;
    const uint32_t col = rank == 0 ? 384u : 256u;
    for (int j0 = 0; j0 < kD; j0 += 32) {
      uint32_t x[32];
#pragma unroll
      for (int q = 0; q < 32; q += 4) {
        const float4 f4 = rec ? *(const float4*)(rec + r * kD + j0 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[q] = __float_as_uint(f4.x); x[q + 1] = __float_as_uint(f4.y);
        x[q + 2] = __float_as_uint(f4.z); x[q + 3] = __float_as_uint(f4.w);
      }
      tmem_st32(tmem + lb + col + j0, x);
    }
    tmem_st_wait();
    if (rank == 1) {  // the constant ones tile of z = K^T 1 (16 rows x 64 bf16, any swizzle)
      const uint32_t one2 = kBF16 ? 0x3F803F80u : 0x3C003C00u;
      uint4* op = (uint4*)(smem + kQOffOnes);
      op[threadIdx.x - 256] = make_uint4(one2, one2, one2, one2);
      fence_proxy_async();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / st.async
  if (rank == 0)
    kv_role<kBF16>(tmQ, tmK, tmV, prm, grp, nc, smem, bars, fl, tmem);
  else
    q_role<kBF16>(tmK, tmV, tmW, tmO, prm, grp, nc, smem, bars, fl, tmem);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still write into its shared memory
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

// Used for the causal tensor-core backward with the forward's saved states when the
// pairs fill the GPU in one wave (bwd_pair_rule, internal.h).
cudaError_t tc_backward_pair(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int Pf = tc_segments(G, N);
  const int64_t segf = ((N / 128 + Pf - 1) / Pf) * 128;
  CUtensorMap mQ, mK, mV, mW, mO;
  if (!make_tma_map(&mO, t.o, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mQ, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mK, t.k, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mW, t.w, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  PairParams prm{t.o, t.g, dq, dk, dv, N, L.a, L.b, L.saved_in + kSavedHeader, Pf, segf,
                 L.saved_in + kSavedHeader + G * Pf * state_floats(kD), ck_count(N), L.row_offset,
                 L.carry_suffix};
  auto k = bf ? k_bwd_pair_tc<true> : k_bwd_pair_tc<false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPairSmem);
  {
    ProfScope ps("la_bwd_pair", L.stream);
    k<<<dim3(kCl, (unsigned)(G / (kCl / 2))), 512, kPairSmem, L.stream>>>(mQ, mK, mV, mW, mO, prm);
  }
  note_launch(1);
  return cudaGetLastError();
}

}  // namespace lab

extern "C" int la_internal_trace_read_pair(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lab::g_trace_p, sizeof(lab::g_trace_p));
}
