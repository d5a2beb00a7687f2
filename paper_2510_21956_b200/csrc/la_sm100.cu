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
#ifdef LA_TRACE  // compiled out by default: the kernels are I-cache sensitive
  if (blockIdx.x == 0 && blockIdx.y == 0 && c < 64) g_trace[role][c][ev] = clock64();
#endif
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
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * kPanel + (ks & 3) * 32) >> 4);
}
// MN-major SW128 descriptor for k-step ks: K rows of 128 B, MN panels kPanel apart.
__device__ __forceinline__ uint64_t mndesc(uint32_t tile, int ks) {
  return sdesc_sw128(tile, kPanel, 1024) + (uint64_t)((ks * 2048) >> 4);
}

struct FwdParams {
  const float* agg;     // per (g, unit) raw sums (A units per segment, segments 0..P-2)
  int A;                // units per segment
  const float* carry;   // per-group carry-in (sequence sharding), or null
  float* cmb;           // per (g, segment) scratch: exclusive prefix combined in the prologue
  float* gout;          // G*N
  unsigned long long* flag;
  int64_t N, G;
  int64_t seg_len;      // rows per segment (multiple of kC)
  int P;
  int64_t row_offset;
  float a, b;
  float* st_out;        // per-(group, segment) end state (S, z, sigma, rows) for the backward, or null
  void* out;            // o, FeatureMajor [G][D][N]
  int pf;               // chunks prefetched into L2 ahead of the ring
  float* ck_out;        // [G][ck_K] prefix checkpoints at global rows C0 * 2^k (internal.h), or null
  int ck_K;
  int cmb_ready = 0;    // cmb already holds every segment's prefix (seg_scan, many unit records)
};

// ================================================================ forward main
// Chunks of C = 64 rows, 3-stage TMA ring (+ L2 prefetch ahead of it). Warp roles
// (448 threads): 0 TMA producer; 1 MMA issuer + TMEM owner; 2-5 "WG-A" (T1 -> P',
// g); 6-9 "WG-B" (sigma, O^T -> o); 10-13 "WG-S" (S^T -> bf16 operand, z, z rows).
// Per chunk c the tensor core computes
//   T1  = Q [K ; z_hi ; z_lo]^T   (M=64, N=80: columns 64, 65 give q_i . z_prev)
//   S^T += V^T K                  (the running state, fp32 in TMEM)
//   O^T = V^T P'^T + bf16(b S^T) Q^T   (bf16 S^T is an A operand read from TMEM)
// so the CUDA-core passes are the TMEM epilogues, z (column sums of K, written as
// the two bf16 rows z_hi, z_lo under the next chunk's K tile) and sigma (row sums of V^T).
// Stage: Q [64][128] | K as two 80-row panels (64 key rows + 16 rows for z) | V^T.
// TMEM: [0,80) T1 (M=64: lanes 0-15 of each quadrant), [128,256) O^T x2,
// [256,384) S^T, [384,512) bf16(b S^T) x2.
constexpr int kCF = 64;                  // forward chunk rows
constexpr int kFT = 16384;               // 64x128 / 128x64 16-bit tile
constexpr int kKPanel = 80 * 128;        // K-tile panel: 64 key rows + 16 z rows
constexpr int kFStages = 3;
constexpr int kFPrefetch = 0;            // L2 prefetch distance (chunks). 0: each chunk is prefetched
                                         // into L2 just before the producer waits for its ring slot
                                         // (sweep 0.76 -> 0.72 ms, bwd aggregate 0.69 -> 0.64 ms
                                         // against no prefetch); >= 1 costs extra DRAM re-reads
constexpr int kFStage = kFT + 2 * kKPanel + kFT;  // Q, K(+z), V^T  = 52 KB
constexpr int kOffK = kFT, kOffV = kFT + 2 * kKPanel;
constexpr uint32_t kF_T1 = 0, kF_OT = 128, kF_ST = 256, kF_SB = 384;
constexpr uint32_t kHalfLanes = 16u << 16;  // TMEM lane offset of the upper M=64 half

// z (a sum of up to N keys) is handed to the tensor core as two 16-bit rows; fp16
// would overflow at |z| > 65504, so fp16 rows carry z / 256 and g multiplies back.
template <bool kBF16>
__host__ __device__ constexpr float z_row_scale() { return kBF16 ? 1.f : 1.f / 256.f; }

template <bool kBF16>
__device__ __forceinline__ float h2f_fwd(uint16_t h) {
  return kBF16 ? __bfloat162float(__ushort_as_bfloat16(h)) : __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ uint64_t kd64(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * rows * 128 + (ks & 3) * 32) >> 4);
}
__device__ __forceinline__ uint64_t mn64(uint32_t tile, int ks, uint32_t panel) {
  return sdesc_sw128(tile, panel, 1024) + (uint64_t)((ks * 2048) >> 4);
}

template <bool kBF16>
__global__ void __launch_bounds__(448, 1)
    k_fwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
             FwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sP = smem + kFStages * kFStage;   // [2][8K]   P' (rows i, cols t)
  uint8_t* sO = sP + 2 * 8192;               // [2][16K]  o^T staging (rows j, cols i) for TMA stores
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
  uint64_t* zrow_ready = bars + 19; // z rows of the next chunk's stage written
  uint32_t* tslot = (uint32_t*)(bars + 20);
  float* ginv_s = (float*)(bars + 22);  // [4][64] (16-byte aligned: read as float4), then [128] z exchange

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
      mbar_init(&empty[s], 1 + 2 * 128);  // M2 commit, WG-B (V), WG-S (K)
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
    mbar_init(zrow_ready, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  // exclusive prefix of this segment: carry + sum of the earlier segments' sums
  const bool has_in = p > 0 || prm.carry != nullptr;
  float* st_in = has_in ? prm.cmb + (grp * prm.P + p) * state_floats(kD) : nullptr;
  if (has_in && !prm.cmb_ready && warp >= 2 && warp < 10)
    combine_records(st_in, prm.carry ? prm.carry + grp * state_floats(kD) : nullptr,
                    prm.agg + grp * prm.P * prm.A * state_floats(kD), 0, p * prm.A, state_floats(kD),
                    (int)threadIdx.x - 64, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      auto l2_prefetch = [&](int c) {
        const int64_t row0 = s0 + (int64_t)c * kCF;
        tma_prefetch_l2_3d(&tmQ, 0, (int)(grp * prm.N + row0), 0);
        tma_prefetch_l2_3d(&tmK, 0, (int)(grp * prm.N + row0), 0);
        tma_prefetch_l2_3d(&tmK, 0, (int)(grp * prm.N + row0), 1);
        tma_prefetch_l2_3d(&tmV, 0, (int)(grp * kD), (int)(row0 / 64));
      };
      for (int c = 0; c < prm.pf && c < nc; ++c) l2_prefetch(c);
      for (int c = 0; c < nc; ++c) {
        const int s = c % kFStages;
        if (c + prm.pf < nc) l2_prefetch(c + prm.pf);
        if (lane_id() == 0) trace(3, c, 0);
        if (c >= kFStages) mbar_wait(&empty[s], ((c / kFStages) & 1) ^ 1);
        trace(3, c, 1);
        const int64_t row0 = s0 + (int64_t)c * kCF;
        uint8_t* st = smem + s * kFStage;
        mbar_expect_tx(&full[s], 3 * kFT);  // Q 16K + K 2 x 8K + V^T 16K
        tma_load_3d(st, &tmQ, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kOffK, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + kOffK + kKPanel, &tmK, &full[s], 0, (int)(grp * prm.N + row0), 1);
        tma_load_3d(st + kOffV, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Per chunk: M3(c) = S^T and Z^T updates, M2(c) = O^T, then M1(c+1) = next T1.
    constexpr uint32_t fmt = kBF16 ? 1 : 0;
    const uint32_t id_T1 = idesc_f16(64, 40, fmt, 0, 0);
    const uint32_t id_ST = idesc_f16(128, 128, fmt, 0, 1);
    const uint32_t id_OT = idesc_f16(128, 64, fmt, 0, 0);
    const uint32_t a0 = smem_u32(smem), aP = smem_u32(sP);
    auto issue_t1 = [&](int c) {  // T1(c) = Q [K ; z rows]^T
      const uint32_t aQ = a0 + (c % kFStages) * kFStage;
      mbar_wait(&full[c % kFStages], (c / kFStages) & 1);
      mbar_wait(zrow_ready, c & 1);
      if (c >= 1) mbar_wait(t1_empty, (c - 1) & 1);
      tc_fence_after();
      if (elect_one()) {  // key rows 0..39 -> lower lane half, rows 40..79 (incl. z) -> upper half
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + kF_T1, kd64(aQ, ks, 64), kd64(aQ + kOffK, ks, 80), id_T1, ks > 0);
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + kF_T1 + kHalfLanes, kd64(aQ, ks, 64), kd64(aQ + kOffK + 40 * 128, ks, 80), id_T1, ks > 0);
        mma_commit(t1_full);
      }
      __syncwarp();
    };
    if (nc > 0) issue_t1(0);
    for (int c = 0; c < nc; ++c) {
      const int s = c % kFStages, b = c & 1;
      const uint32_t aQ = a0 + s * kFStage, aK = aQ + kOffK, aV = aQ + kOffV;
      if (lane_id() == 0) trace(0, c, 0);
      mbar_wait(sb_ready, c & 1);
      if (lane_id() == 0) trace(0, c, 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 4; ++ks)  // S^T += V^T K  (A: V^T rows j, K-major; B: K (N=m, K=t) MN-major)
          mma_ss(tmem + kF_ST, kd64(aV, ks, 128), mn64(aK, ks, kKPanel), id_ST, 1);
        mma_commit(st_full);
      }
      __syncwarp();
      if (c + 1 < nc) issue_t1(c + 1);
      if (lane_id() == 0) trace(0, c, 2);
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
    // Per chunk: T1 -> P' (registers), g = rowsum(P') + a (row) + b q.z_prev -> 1/g for
    // WG-B, P' -> smem.
    const uint32_t qd = warp & 3;
    const int l = (int)lane_id();
    const int ih = (int)(qd * 16) + (l & 15);      // row i of the M=64 T1
    const bool lower = l < 16;
    const uint32_t lane_base = (qd * 32u) << 16;
    const int et = (int)threadIdx.x - 64;          // 0..127
    const float a = prm.a, b = prm.b;
    for (int c = 0; c < nc; ++c) {
      const int bb = c & 1;
      const int64_t row0 = s0 + (int64_t)c * kCF;
      mbar_wait(t1_full, c & 1);
      if (et == 0) trace(1, c, 3);
      tc_fence_after();
      // lower lanes hold T1 columns t = 0..39 of row ih, upper lanes t = 40..79 (t = 64, 65:
      // q . z_hi, q . z_lo); each half builds its part of P' and of the row sum
      uint32_t pk[20];
      float rs0 = 0.f, rs1 = 0.f, qz;
      {
        uint32_t x[40];
        tmem_ld32(tmem + lane_base + kF_T1, *(uint32_t(*)[32])x);
        tmem_ld8(tmem + lane_base + kF_T1 + 32, *(uint32_t(*)[8])(x + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(t1_empty);
        const int tb = lower ? 0 : 40;
        qz = lower ? 0.f : (__uint_as_float(x[24]) + __uint_as_float(x[25])) * (1.f / z_row_scale<kBF16>());
#pragma unroll
        for (int u = 0; u < 20; ++u) {
          const int t0 = tb + 2 * u;
          const float p0 = t0 <= ih ? a + b * __uint_as_float(x[2 * u]) : 0.f;  // t >= 64 never passes
          const float p1 = t0 + 1 <= ih ? a + b * __uint_as_float(x[2 * u + 1]) : 0.f;
          rs0 += p0;
          rs1 += p1;
          pk[u] = pack2<kBF16>(p0, p1);
        }
      }
      const float rs = (rs0 + rs1) + __shfl_xor_sync(0xffffffffu, rs0 + rs1, 16);
      qz += __shfl_xor_sync(0xffffffffu, qz, 16);
      if (et == 0) trace(1, c, 7);
      if (lower) {
        const float gi = rs + a * (float)(prm.row_offset + row0) + b * qz;
        if (fabsf(gi) < kEpsF32) flag_degenerate(prm.flag, grp, prm.row_offset + row0 + ih);
        ginv_s[(c & 3) * kCF + ih] = 1.f / gi;
        prm.gout[grp * prm.N + row0 + ih] = gi;
      }
      mbar_arrive(&a2b[c & 3]);
      if (et == 0) trace(1, c, 4);
      if (c >= 2) mbar_wait(&o_full[bb], ((c - 2) >> 1) & 1);  // M2(c-2) drained sP[bb]
      if (et == 0) trace(1, c, 5);
      {  // P' row ih: lower lanes columns 0..39 (5 chunks), upper lanes 40..63 (3 chunks)
        uint8_t* pp = sP + bb * 8192;
        const int w0 = lower ? 0 : 5, nw = lower ? 5 : 3;
#pragma unroll
        for (int w = 0; w < 5; ++w)
          if (w < nw)
            *(uint4*)(pp + sw128_off(ih, 8 * (w0 + w), kCF)) =
                make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
      }
      fence_proxy_async();
      mbar_arrive(p_ready);
      if (et == 0) trace(1, c, 6);
    }
  } else if (warp >= 10) {
    // ------------------------------------------------------------ WG-S (warps 10..13)
    // Per chunk: E2 (S^T -> bf16(b S^T) TMEM operand), then the z rows (z_hi, z_lo of
    // z after this chunk, from the Z^T accumulator) into the next chunk's K tile.
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());      // j of S^T; m of Z^T
    const uint32_t lane_base = (qd * 32u) << 16;
    const int es = (int)threadIdx.x - 320;         // 0..127
    const float b = prm.b;
    // z_hi / z_lo of feature m = r into rows 64, 65 of the K-tile panel holding column m
    auto put_zrows = [&](int c, float z) {
      z *= z_row_scale<kBF16>();
      uint8_t* kt = smem + (c % kFStages) * kFStage + kOffK + (r >> 6) * kKPanel;
      const __nv_bfloat16 h = __float2bfloat16_rn(z);
      const float lo = z - __bfloat162float(h);
      uint16_t hv, lv;
      if (kBF16) {
        hv = __bfloat16_as_ushort(h);
        lv = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
      } else {
        const __half hh = __float2half_rn(z);
        hv = __half_as_ushort(hh);
        lv = __half_as_ushort(__float2half_rn(z - __half2float(hh)));
      }
      *(uint16_t*)(kt + sw128_off(64, r & 63, 80)) = hv;
      *(uint16_t*)(kt + sw128_off(65, r & 63, 80)) = lv;
      if (c < kFStages) {  // rows 66..79 stay zero (first use of the stage)
        for (int rr = 66; rr < 80; ++rr) *(uint16_t*)(kt + sw128_off(rr, r & 63, 80)) = 0;
      }
      fence_proxy_async();
      mbar_arrive(zrow_ready);
    };
    float zr = st_in ? st_in[kD * kD + r] : 0.f;  // z_m (m = r) before the current chunk
    float* zx = (float*)(ginv_s + 4 * kCF);        // [128] column-sum exchange
    for (int m0 = 0; m0 < kD; m0 += 32) {  // carry-in S^T row r = S[:, r]
      uint32_t v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = st_in ? __float_as_uint(st_in[(m0 + u) * kD + r]) : 0u;
      tmem_st32(tmem + lane_base + kF_ST + m0, v);
    }
    tmem_st_wait();
    if (nc > 0) put_zrows(0, zr);
    const int mg = es >> 3, tg = es & 7;
    for (int c = 0; c < nc; ++c) {
      const int s = c % kFStages, bb = c & 1;
      // ---- E2: S^T (after chunk c-1) -> bf16(b S^T) in TMEM buffer bb
      if (es == 0) trace(1, c, 0);
      if (c >= 1) mbar_wait(st_full, (c - 1) & 1);
      tc_fence_after();
      // exact prefix at this chunk's first row when it is a checkpoint row (internal.h);
      // kept out of the conversion loop below, which is I-cache sensitive
      if (prm.ck_out && c >= 1) {
        const int k = ck_index(prm.row_offset + s0 + (int64_t)c * kCF, prm.ck_K);
        if (k >= 0) {
          float* ck = prm.ck_out + (grp * prm.ck_K + k) * state_floats(kD);
          ck[kD * kD + r] = zr;
          if (r == 0) ck[kD * kD + 2 * kD] = (float)(prm.row_offset + s0 + (int64_t)c * kCF);
#pragma unroll 1
          for (int m0 = 0; m0 < kD; m0 += 32) {  // record X[m][j] = S[m][j]; S^T row j = r here
            uint32_t x[32];
            tmem_ld32(tmem + lane_base + kF_ST + m0, x);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) ck[(m0 + u) * kD + r] = __uint_as_float(x[u]);
          }
        }
      }
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
      if (es == 0) trace(1, c, 1);
      // ---- z after chunk c (column sums of K(c), CUDA cores) -> z rows of chunk c + 1.
      //      Thread (mg, tg) sums rows tg + 8 u of columns [8 mg, 8 mg + 8): a quarter-warp
      //      reads 8 consecutive rows (distinct swizzle chunks, no bank conflicts).
      if (c + 1 < nc) {
        mbar_wait(&full[s], (c / kFStages) & 1);
        const uint8_t* kt = smem + s * kFStage + kOffK + (mg >> 3) * kKPanel;
        float zs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int t = tg; t < kCF; t += 8) {
          const uint4 v4 = *(const uint4*)(kt + sw128_off(t, 8 * (mg & 7), 80));
          const float2 f0 = unpack2<kBF16>(v4.x), f1 = unpack2<kBF16>(v4.y);
          const float2 f2 = unpack2<kBF16>(v4.z), f3 = unpack2<kBF16>(v4.w);
          zs[0] += f0.x; zs[1] += f0.y; zs[2] += f1.x; zs[3] += f1.y;
          zs[4] += f2.x; zs[5] += f2.y; zs[6] += f3.x; zs[7] += f3.y;
        }
        zx[8 * mg + tg] = reduce_scatter8(zs, tg);
        mbar_arrive(&empty[s]);  // WG-S is done with K(c)
        named_bar(3, 128);
        zr += zx[r];
        named_bar(3, 128);  // zx is reused next chunk
        if (es == 0) trace(1, c, 2);
        mbar_wait(&full[(c + 1) % kFStages], ((c + 1) / kFStages) & 1);
        put_zrows(c + 1, zr);
      } else {
        mbar_arrive(&empty[s]);  // last chunk: K(c) is summed below, the stage is not reloaded
      }
    }
    if (prm.st_out && nc > 0) {  // final state for the backward (S, z)
      mbar_wait(st_full, (nc - 1) & 1);
      tc_fence_after();
      if (nc >= 1) {  // z after the last chunk
        const int s = (nc - 1) % kFStages;
        const uint8_t* kt = smem + s * kFStage + kOffK + (r >> 6) * kKPanel;
        float zs = 0.f;
        for (int t = 0; t < kCF; ++t) zs += h2f_fwd<kBF16>(*(const uint16_t*)(kt + sw128_off(t, r & 63, 80)));
        zr += zs;
      }
      float* so = prm.st_out + (grp * prm.P + p) * state_floats(kD);
      for (int m0 = 0; m0 < kD; m0 += 32) {
        uint32_t x[32];
        tmem_ld32(tmem + lane_base + kF_ST + m0, x);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) so[(m0 + u) * kD + r] = __uint_as_float(x[u]);
      }
      so[kD * kD + r] = zr;
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
      const uint8_t* v_t = smem + s * kFStage + kOffV;
      if (eb == 0) trace(2, c, 0);
      // sigma_j += sum_t V^T[j][t] (j = r) as soon as V(c) lands; a * sigma_prev feeds
      // this chunk's outputs.
      mbar_wait(&full[s], (c / kFStages) & 1);
      float vs = 0.f;
#pragma unroll
      for (int t8 = 0; t8 < kCF; t8 += 8) {
        const uint4 v4 = *(const uint4*)(v_t + sw128_off(r, t8, kD));
        const float2 f0 = unpack2<kBF16>(v4.x), f1 = unpack2<kBF16>(v4.y);
        const float2 f2 = unpack2<kBF16>(v4.z), f3 = unpack2<kBF16>(v4.w);
        vs += ((f0.x + f0.y) + (f1.x + f1.y)) + ((f2.x + f2.y) + (f3.x + f3.y));
      }
      pin(vs);                 // the V(c) loads have returned before the stage is released
      mbar_arrive(&empty[s]);  // WG-B is done with V(c)
      const float asig = a * sigma;
      sigma += vs;
      mbar_wait(&o_full[bb], (c >> 1) & 1);
      if (eb == 0) trace(2, c, 1);
      mbar_wait(&a2b[c & 3], (c >> 2) & 1);
      if (eb == 0) trace(2, c, 2);
      tc_fence_after();
      const float* gv = ginv_s + (c & 3) * kCF;
      uint32_t pk[32];
      {
        uint32_t x0[32], x1[32];
        tmem_ld32(tmem + lane_base + kF_OT + bb * 64, x0);
        tmem_ld32(tmem + lane_base + kF_OT + bb * 64 + 32, x1);
        float gr[64];
#pragma unroll
        for (int u = 0; u < 16; ++u) *(float4*)(gr + 4 * u) = *(const float4*)(gv + 4 * u);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&ot_empty[bb]);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          pk[u] = pack2<kBF16>((__uint_as_float(x0[2 * u]) + asig) * gr[2 * u],
                               (__uint_as_float(x0[2 * u + 1]) + asig) * gr[2 * u + 1]);
          pk[16 + u] = pack2<kBF16>((__uint_as_float(x1[2 * u]) + asig) * gr[32 + 2 * u],
                                    (__uint_as_float(x1[2 * u + 1]) + asig) * gr[32 + 2 * u + 1]);
        }
      }
      if (eb == 0) trace(2, c, 3);
      // o^T row j = r, columns [row0, row0 + 64): one 128-byte line per thread
      // o^T rows j, columns [row0, row0 + 64) -> staging buffer bb -> one TMA store
      if (eb == 0) tma_store_wait_read1();  // the store issued two chunks ago has left buffer bb
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
      }
      if (eb == 0) trace(2, c, 4);
    }
    if (eb == 0) tma_store_wait0();
    if (prm.st_out && nc > 0) prm.st_out[(grp * prm.P + p) * state_floats(kD) + kD * kD + kD + r] = sigma;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ================================================================ segment aggregates
// Per (g, unit): S = sum_t k_t^T v_t (stored X[m][j]), z = sum k, sigma = sum v,
// count; the record layout of la_simt.cu's k_seg_sums (internal.h). Everything is on
// the tensor core: S^T|sigma = V^T [K | 1] (a constant ones panel appended to the K
// tile gives N = 144, column 128 = sigma) and Z = K^T 1 (M=128 lanes m, N=16 against
// a constant ones tile), so the epilogue warps only read TMEM once per unit.
// Stage: K [128 t][128 m] (2 panels) | ones panel | V^T [128 j][128 t] (2 panels).
constexpr int kAggStage = 2 * kTile + kPanel;  // 80 KB
constexpr int kAggOffOnes = kTile, kAggOffV = kTile + kPanel;

template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    k_fwd_agg_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                 float* states, int64_t N, int64_t seg_len, int P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sOnesZ = smem + 2 * kAggStage;   // [16 rows][128 t] ones (K-major B of the Z MMA)
  uint64_t* bars = (uint64_t*)(sOnesZ + 4096);
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  uint64_t* done = bars + 4;
  uint32_t* tslot = (uint32_t*)(bars + 8);
  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * seg_len;
  const int64_t s1 = lmin(N, s0 + seg_len);
  const int nc = s1 > s0 ? (int)((s1 - s0) / kC) : 0;
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  if (warp >= 2) {  // constant ones: the N-augmentation panel of each stage and the Z tile
    const uint32_t one2 = kBF16 ? 0x3F803F80u : 0x3C003C00u;
    const int t = (int)threadIdx.x - 64;
    for (int st = 0; st < 2; ++st) {
      uint4* op = (uint4*)(smem + st * kAggStage + kAggOffOnes);
      for (int e = t; e < kPanel / 16; e += 128) op[e] = make_uint4(one2, one2, one2, one2);
    }
    for (int e = t; e < 4096 / 16; e += 128) ((uint4*)sOnesZ)[e] = make_uint4(one2, one2, one2, one2);
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;  // [0,144) S^T | sigma, [160,176) Z
  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c & 1;
        const int64_t row0 = s0 + (int64_t)c * kC;
        tma_prefetch_l2_3d(&tmK, 0, (int)(grp * N + row0), 0);  // before the slot wait (kFPrefetch)
        tma_prefetch_l2_3d(&tmV, 0, (int)(grp * kD), (int)(row0 / 64));
        if (c >= 2) mbar_wait(&empty[s], ((c >> 1) & 1) ^ 1);
        uint8_t* st = smem + s * kAggStage;
        mbar_expect_tx(&full[s], 2 * kTile);
        tma_load_3d(st, &tmK, &full[s], 0, (int)(grp * N + row0), 0);
        tma_load_3d(st + kAggOffV, &tmV, &full[s], 0, (int)(grp * kD), (int)(row0 / 64));
      }
    }
  } else if (warp == 1) {
    const uint32_t id_S = idesc_f16(128, 144, kBF16 ? 1 : 0, 0, 1);  // A = V^T (K-major), B = [K | 1] (MN-major)
    const uint32_t id_Z = idesc_f16(128, 16, kBF16 ? 1 : 0, 1, 0);   // A = K^T (MN-major), B = ones (K-major)
    const uint32_t aZ = smem_u32(sOnesZ);
    for (int c = 0; c < nc; ++c) {
      const int s = c & 1;
      const uint32_t aK = smem_u32(smem + s * kAggStage), aV = aK + kAggOffV;
      mbar_wait(&full[s], (c >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem, kdesc(aV, ks), mndesc(aK, ks), id_S, (c > 0 || ks > 0) ? 1u : 0u);
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + 160, mndesc(aK, ks),
                 sdesc_sw128(aZ, 16, 1024) + (uint64_t)(((ks >> 2) * 16 * 128 + (ks & 3) * 32) >> 4), id_Z,
                 (c > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (c == nc - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
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
      uint32_t sg, s2_, zz, z2;
      tmem_ld2(tmem + lane_base + 128, sg, s2_);
      tmem_ld2(tmem + lane_base + 160, zz, z2);
      tmem_ld_wait();
      st[kD * kD + r] = __uint_as_float(zz);        // z_m (lane r = m of Z)
      st[kD * kD + kD + r] = __uint_as_float(sg);   // sigma_j (lane r = j of S^T)
    } else {
      for (int m = 0; m < kD; ++m) st[m * kD + r] = 0.f;
      st[kD * kD + r] = 0.f;
      st[kD * kD + kD + r] = 0.f;
    }
    if (r == 0) st[kD * kD + 2 * kD] = (float)(s1 > s0 ? s1 - s0 : 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

constexpr size_t kFwdSmem = kFStages * kFStage + 2 * 8192 + 2 * kFT + 256 + (4 * kCF + kD) * 4 + 1024;
constexpr size_t kAggSmem = 2 * kAggStage + 4096 + 128 + 1024;

// ================================================================ non-causal forward
// forward_full (forward_kernels.hpp:133-206): with the totals S = sum k^T v, z = sum k,
// sigma = sum v over all N (aggregate pass + k_sum_units),
//   O^T = bf16(b S^T) Q^T        (bf16 S^T is a constant A operand in TMEM)
//   g   = a N + b Q [z_hi; z_lo]^T   (M=64, N=16 against two bf16 rows of z)
//   o   = (O^T + a sigma) / g  -> staging -> TMA store.
// One CTA per (group, segment) of 64-row chunks; 4-stage Q ring; 192 threads:
// 0 TMA producer, 1 MMA issuer + TMEM owner, 2-5 epilogue.
constexpr int kQStages = 4;
constexpr uint32_t kFF_SB = 0, kFF_OT = 64, kFF_GZ = 192;  // TMEM: bf16 S^T | O^T x2 | q.z x2
constexpr size_t kFwdFullSmem = kQStages * kFT + 4096 + 2 * kFT + 128 + 2 * kCF * 4 + 1024;

__global__ void k_sum_units(const float* recs, int U, int64_t SZ, float* tot) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (e >= SZ) return;
  const float* r = recs + grp * U * SZ + e;
  float acc = 0.f;
  if (e <= (int64_t)kD * kD + 2 * kD)  // record padding: never written by the units, kept zero
    for (int u = 0; u < U; ++u) acc += r[u * SZ];
  tot[grp * SZ + e] = acc;
}

struct FwdFullParams {
  const float* tot;     // per-group totals (S, z, sigma, count)
  float* gout;
  unsigned long long* flag;
  int64_t N, n_total, seg_len;
  float a, b;
};

template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    k_fwd_full_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
                  FwdFullParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sZ = smem + kQStages * kFT;   // [16 rows][128 m] z_hi, z_lo, zeros (K-major, 2 panels)
  uint8_t* sO = sZ + 4096;               // [2][16K] o^T staging
  uint64_t* bars = (uint64_t*)(sO + 2 * kFT);
  uint64_t* full = bars;                 // [4]
  uint64_t* empty = bars + 4;            // [4]
  uint64_t* o_full = bars + 8;           // [2]
  uint64_t* ot_empty = bars + 10;        // [2]
  uint32_t* tslot = (uint32_t*)(bars + 12);
  float* ginv_s = (float*)(bars + 16);   // [2][64]

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = s1 > s0 ? (int)((s1 - s0) / kCF) : 0;
  const uint32_t warp = warp_id();
  const float* tot = prm.tot + grp * state_floats(kD);
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&ot_empty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp >= 2) {  // constants: bf16(b S^T) into TMEM, z rows into smem
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());
    const uint32_t lb = (qd * 32u) << 16;
    const float b = prm.b;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      uint32_t pk[32];
#pragma unroll
      for (int u = 0; u < 32; ++u)
        pk[u] = pack2<kBF16>(b * tot[(half * 64 + 2 * u) * kD + r], b * tot[(half * 64 + 2 * u + 1) * kD + r]);
      tmem_st32(tmem + lb + kFF_SB + half * 32, pk);
    }
    tmem_st_wait();
    const float z = tot[kD * kD + r] * z_row_scale<kBF16>();
    uint16_t hv, lv;
    if (kBF16) {
      const __nv_bfloat16 h = __float2bfloat16_rn(z);
      hv = __bfloat16_as_ushort(h);
      lv = __bfloat16_as_ushort(__float2bfloat16_rn(z - __bfloat162float(h)));
    } else {
      const __half h = __float2half_rn(z);
      hv = __half_as_ushort(h);
      lv = __half_as_ushort(__float2half_rn(z - __half2float(h)));
    }
    uint8_t* zp = sZ + (r >> 6) * 2048;
    *(uint16_t*)(zp + sw128_off(0, r & 63, 16)) = hv;
    *(uint16_t*)(zp + sw128_off(1, r & 63, 16)) = lv;
    for (int rr = 2; rr < 16; ++rr) *(uint16_t*)(zp + sw128_off(rr, r & 63, 16)) = 0;
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c % kQStages;
        tma_prefetch_l2_3d(&tmQ, 0, (int)(grp * prm.N + s0 + (int64_t)c * kCF), 0);  // before the slot wait
        if (c >= kQStages) mbar_wait(&empty[s], ((c / kQStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], kFT);
        tma_load_3d(smem + s * kFT, &tmQ, &full[s], 0, (int)(grp * prm.N + s0 + (int64_t)c * kCF), 0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t fmt = kBF16 ? 1 : 0;
    const uint32_t id_OT = idesc_f16(128, 64, fmt, 0, 0);
    const uint32_t id_GZ = idesc_f16(64, 16, fmt, 0, 0);
    const uint32_t aZ = smem_u32(sZ);
    for (int c = 0; c < nc; ++c) {
      const int s = c % kQStages, b = c & 1;
      const uint32_t aQ = smem_u32(smem + s * kFT);
      mbar_wait(&full[s], (c / kQStages) & 1);
      if (c >= 2) mbar_wait(&ot_empty[b], ((c - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < 8; ++ks)  // O^T = bf16(b S^T) Q^T  (A from TMEM)
          mma_ts(tmem + kFF_OT + b * 64, tmem + kFF_SB + ks * 8, kd64(aQ, ks, 64), id_OT, ks > 0);
        for (int ks = 0; ks < 8; ++ks)  // q . [z_hi, z_lo]
          mma_ss(tmem + kFF_GZ + b * 16, kd64(aQ, ks, 64), kd64(aZ, ks, 16), id_GZ, ks > 0);
        mma_commit(&o_full[b]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    const uint32_t qd = warp & 3;
    const int l = (int)lane_id();
    const int r = (int)(qd * 32) + l;              // j of O^T
    const int ih = (int)(qd * 16) + (l & 15);      // row i of the M=64 q.z accumulator
    const bool lower = l < 16;
    const uint32_t lb = (qd * 32u) << 16;
    const int et = (int)threadIdx.x - 64;
    const float a = prm.a, b = prm.b;
    const float asig = a * tot[kD * kD + kD + r];
    const float an = a * (float)prm.n_total;
    for (int c = 0; c < nc; ++c) {
      const int bb = c & 1;
      const int64_t row0 = s0 + (int64_t)c * kCF;
      mbar_wait(&o_full[bb], (c >> 1) & 1);
      tc_fence_after();
      uint32_t x0[32], x1[32], zh, zl;
      tmem_ld32(tmem + lb + kFF_OT + bb * 64, x0);
      tmem_ld32(tmem + lb + kFF_OT + bb * 64 + 32, x1);
      tmem_ld2(tmem + lb + kFF_GZ + bb * 16, zh, zl);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&ot_empty[bb]);
      if (lower) {
        const float gi = an + b * (__uint_as_float(zh) + __uint_as_float(zl)) * (1.f / z_row_scale<kBF16>());
        if (fabsf(gi) < kEpsF32) flag_degenerate(prm.flag, grp, row0 + ih);
        ginv_s[bb * kCF + ih] = 1.f / gi;
        prm.gout[grp * prm.N + row0 + ih] = gi;
      }
      if (et == 0) tma_store_wait_read1();  // the store issued two chunks ago has left buffer bb
      named_bar(1, 128);                     // ginv of chunk c complete; staging bb free
      const float* gv = ginv_s + bb * kCF;
      uint8_t* so = sO + bb * kFT;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t p0[4], p1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i0 = 8 * w + 2 * q;
          p0[q] = pack2<kBF16>((__uint_as_float(x0[i0]) + asig) * gv[i0], (__uint_as_float(x0[i0 + 1]) + asig) * gv[i0 + 1]);
          p1[q] = pack2<kBF16>((__uint_as_float(x1[i0]) + asig) * gv[32 + i0],
                               (__uint_as_float(x1[i0 + 1]) + asig) * gv[32 + i0 + 1]);
        }
        *(uint4*)(so + sw128_off(r, 8 * w, kD)) = make_uint4(p0[0], p0[1], p0[2], p0[3]);
        *(uint4*)(so + sw128_off(r, 32 + 8 * w, kD)) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
      }
      fence_proxy_async();
      named_bar(1, 128);
      if (et == 0) {
        tma_store_3d(&tmO, so, 0, (int)(grp * kD), (int)(row0 / 64));
        tma_store_commit();
      }
    }
    if (et == 0) tma_store_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

}  // namespace

int tc_segments(int64_t G, int64_t N) {
  if (const int e = tuning().segments) return (int)lmax(1, e);
  return choose_segments(G, N);
}

bool tc_forward_supported(const Launch& L, const Tensors& t) {
  return (L.dtype == LA_BF16 || L.dtype == LA_F16) && L.D == kD && L.fault == LA_FAULT_NONE &&
         (L.causal || (L.carry_prefix == nullptr && L.row_offset == 0)) &&
         L.N % kC == 0 && t.lq == LA_SEQUENCE_MAJOR && t.lk == LA_SEQUENCE_MAJOR &&
         t.lv == LA_FEATURE_MAJOR && L.G * L.N < (1ll << 31) && L.G * kD < (1ll << 31);
}

static int fwd_agg_split(int64_t G, int64_t N, int P) {
  const int64_t seg = ((N / kC + P - 1) / P) * kC;
  return agg_split(G, seg, P - 1);
}

size_t tc_forward_ws_floats(int64_t G, int64_t N, int64_t D) {
  if (D != kD || N % kC) return 0;
  const int P = tc_segments(G, N);
  const int64_t seg = ((N / kC + P - 1) / P) * kC;
  const int Af = agg_split(G, seg, P);  // non-causal: every segment is aggregated
  const int A = fwd_agg_split(G, N, P);
  const size_t causal = (size_t)((A + 1) * G * P), full = (size_t)(Af * G * P + G);
  return (causal > full ? causal : full) * state_floats(kD);  // unit sums + combined prefixes / totals
}

// Non-causal forward: aggregate every segment, sum the unit records per group, then
// the apply pass over 64-row chunks.
static cudaError_t tc_forward_full(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N, SZ = state_floats(kD);
  const int P = tc_segments(G, N);
  const int64_t seg = ((N / kC + P - 1) / P) * kC;
  const int A = agg_split(G, seg, P);
  float* units = ws.base;
  // with a saved-state buffer the totals land there (header P = -1 marks "totals") and
  // the non-causal backward reuses them instead of re-reading K and V
  float* tot = L.saved_out ? L.saved_out + kSavedHeader : ws.base + G * P * A * SZ;
  if (L.saved_out) {
    write_saved_header(L.saved_out, (double)G, (double)N, (double)kD, -1, 0, L.stream);
  }
  CUtensorMap mK, mV, mQ64, mO64;
  if (!make_map(&mK, t.k, bf, (uint64_t)(G * N), kD) || !make_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N) ||
      !make_tma_map(&mQ64, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mO64, out, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  auto agg = bf ? k_fwd_agg_tc<true> : k_fwd_agg_tc<false>;
  cudaFuncSetAttribute(agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggSmem);
  {
    ProfScope ps("la_fwd_agg", L.stream);
    agg<<<dim3(A * P, G), 192, kAggSmem, L.stream>>>(mK, mV, units, N, seg / A, P * A);
  }
  {
    ProfScope ps("la_fwd_sum", L.stream);
    k_sum_units<<<dim3((unsigned)((SZ + 255) / 256), (unsigned)G), 256, 0, L.stream>>>(units, P * A, SZ, tot);
  }
  // apply pass: segments of whole 64-row chunks, about two CTAs per SM
  const int64_t c64 = N / kCF;
  // independent chunks: ~7 waves (G = 64: 0.24 ms at 2 waves -> 0.19 ms)
  int64_t P2 = (7 * 148 + G / 2) / G;
  if (tuning().full_ctas_fwd > 0) P2 = tuning().full_ctas_fwd;  // measurement override
  if (P2 > c64) P2 = c64;
  if (P2 < 1) P2 = 1;
  const int64_t seg2 = ((c64 + P2 - 1) / P2) * kCF;
  P2 = (N + seg2 - 1) / seg2;
  auto main_k = bf ? k_fwd_full_tc<true> : k_fwd_full_tc<false>;
  cudaFuncSetAttribute(main_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwdFullSmem);
  FwdFullParams prm{tot, g, ws.flag, N, L.n_total > 0 ? L.n_total : N, seg2, L.a, L.b};
  {
    ProfScope ps("la_fwd_full", L.stream);
    main_k<<<dim3((unsigned)P2, (unsigned)G), 192, kFwdFullSmem, L.stream>>>(mQ64, mO64, prm);
  }
  note_launch(3);
  return cudaGetLastError();
}

size_t tc_saved_floats(int64_t G, int64_t N, int64_t D) {
  if (D != kD && D <= 256) return (size_t)(kSavedHeader + G * state_floats(D));  // la_full.cu: K/V totals
  if (D != kD || N % kC) return kSavedHeader;
  return (size_t)(kSavedHeader + G * (tc_segments(G, N) + ck_count(N)) * state_floats(kD));
}

// One CTA per (group, segment). P = 1 walks whole sequences (no carries, no
// aggregate pass); P > 1 takes exclusive-prefix carries from k_fwd_agg_tc + scan.
int tc_kv_units(int64_t G, int64_t N) {
  const int P = tc_segments(G, N);
  const int64_t seg = ((N / kC + P - 1) / P) * kC;
  return P * agg_split(G, seg, P);
}

cudaError_t tc_sum_units(const float* recs, int64_t G, int U, float* tot, cudaStream_t st) {
  const int64_t SZ = state_floats(kD);
  k_sum_units<<<dim3((unsigned)((SZ + 255) / 256), (unsigned)G), 256, 0, st>>>(recs, U, SZ, tot);
  note_launch(1);
  return cudaGetLastError();
}

// Totals over the whole sequence of S = sum k^T v, z, sigma (count) per group.
cudaError_t tc_kv_totals(const Launch& L, const Tensors& t, float* units, float* tot) {
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int P = tc_segments(G, N);
  const int64_t seg = ((N / kC + P - 1) / P) * kC;
  const int A = agg_split(G, seg, P);
  CUtensorMap mK, mV;
  if (!make_map(&mK, t.k, bf, (uint64_t)(G * N), kD) || !make_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N))
    return cudaErrorInvalidValue;
  auto agg = bf ? k_fwd_agg_tc<true> : k_fwd_agg_tc<false>;
  cudaFuncSetAttribute(agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggSmem);
  {
    ProfScope ps("la_kv_agg", L.stream);
    agg<<<dim3(A * P, G), 192, kAggSmem, L.stream>>>(mK, mV, units, N, seg / A, P * A);
  }
  note_launch(1);
  return tc_sum_units(units, G, P * A, tot, L.stream);
}

// Segment carries from aggregate unit records in one launch, for when the sweep CTAs would
// each sum many records in their prologue (small N per segment, many segments: the sum is a
// latency chain of dependent loads there). Per group g and element e of a state record
// (recs: [G][U] records of SZ floats, A units per segment, P = U / A segments):
//   kExclPrefix:   out[g][p] = base[g] + sum_{u <  p A}     recs[g][u]   (the forward's carry)
//   kInclPrefix:   out[g][p] = base[g] + sum_{u < (p+1) A}   recs[g][u]   (S at the segment end)
//   kExclSuffix:   out[g][p] = base[g] + sum_{u >= (p+1) A}  recs[g][u]   (R after the segment)
// with out[g][p] at out + (g P + p) * ostride; unit_pre[g][u] (optional) = the exclusive prefix
// before unit u. One thread per float4 of a record: the loads of successive units are
// independent, only the adds chain.
__global__ void k_seg_scan(const float* recs, int U, int A, int64_t SZ, const float* base, float* out,
                           int64_t ostride, int mode, float* unit_pre) {
  const int64_t e = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  const int64_t g = blockIdx.y;
  if (e >= SZ) return;
  const int P = U / A;
  const float* rg = recs + g * U * SZ + e;
  float4 acc = base ? *(const float4*)(base + g * SZ + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  auto add = [&](const float4 v) { acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; };
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  // units in blocks of 8: the 8 loads are issued together, only the adds chain
  if (mode == 2) {
    *(float4*)(out + (g * P + P - 1) * ostride + e) = acc;
    for (int u1 = U - 1; u1 >= A; u1 -= 8) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = u1 - k >= A ? *(const float4*)(rg + (int64_t)(u1 - k) * SZ) : zero;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int u = u1 - k;
        if (u >= A) {
          add(v[k]);
          if (u % A == 0) *(float4*)(out + (g * P + u / A - 1) * ostride + e) = acc;
        }
      }
    }
    return;
  }
  // mode 0 never reads the last segment's units (the forward aggregates segments 0..P-2)
  const int u_read = mode == 0 ? (P - 1) * A : U;
  for (int u0 = 0; u0 < U; u0 += 8) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = u0 + k < u_read ? *(const float4*)(rg + (int64_t)(u0 + k) * SZ) : zero;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int u = u0 + k;
      if (u < U) {
        if (mode == 0 && u % A == 0) *(float4*)(out + (g * P + u / A) * ostride + e) = acc;
        if (unit_pre) *(float4*)(unit_pre + (g * U + u) * SZ + e) = acc;
        if (u < u_read) add(v[k]);
        if (mode == 1 && (u + 1) % A == 0) *(float4*)(out + (g * P + (u + 1) / A - 1) * ostride + e) = acc;
      }
    }
  }
}

cudaError_t seg_scan(const float* recs, int64_t G, int U, int A, int64_t SZ, const float* base, float* out,
                     int64_t ostride, int mode, float* unit_pre, cudaStream_t st, const char* name) {
  const dim3 grid((unsigned)((SZ / 4 + 127) / 128), (unsigned)G);
  ProfScope ps(name, st);
  k_seg_scan<<<grid, 128, 0, st>>>(recs, U, A, SZ, base, out, ostride, mode, unit_pre);
  note_launch(1);
  return cudaGetLastError();
}

cudaError_t tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  if (!L.causal) return tc_forward_full(L, t, out, g, ws);
  const bool bf = L.dtype == LA_BF16;
  const int64_t G = L.G, N = L.N;
  const int64_t SZ = state_floats(kD);
  const int P = tc_segments(G, N);
  const int64_t chunks = N / kC;
  const int64_t seg = ((chunks + P - 1) / P) * kC;
  CUtensorMap mK, mV, mQ64, mK64, mV64, mO64;
  if (!make_map(&mK, t.k, bf, (uint64_t)(G * N), kD) || !make_map(&mV, t.v, bf, (uint64_t)(G * kD), (uint64_t)N) ||
      !make_tma_map(&mQ64, t.q, bf, (uint64_t)(G * N), kD, 64, 2) ||
      !make_tma_map(&mK64, t.k, bf, (uint64_t)(G * N), kD, 64, 1) ||
      !make_tma_map(&mV64, t.v, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1) ||
      !make_tma_map(&mO64, out, bf, (uint64_t)(G * kD), (uint64_t)N, 128, 1))
    return cudaErrorInvalidValue;
  auto main_k = bf ? k_fwd_tc<true> : k_fwd_tc<false>;
  cudaFuncSetAttribute(main_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwdSmem);
  float* saved = L.saved_out ? L.saved_out + kSavedHeader : nullptr;
  const int A = fwd_agg_split(G, N, P);
  float* agg_st = ws.base;
  float* cmb = ws.base + G * P * A * SZ;
  int launches = 1;
  if (P > 1) {  // only segments 0..P-2 feed a later segment's prefix
    auto agg = bf ? k_fwd_agg_tc<true> : k_fwd_agg_tc<false>;
    cudaFuncSetAttribute(agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAggSmem);
    ProfScope ps("la_fwd_agg", L.stream);
    agg<<<dim3(A * (P - 1), G), 192, kAggSmem, L.stream>>>(mK, mV, agg_st, N, seg / A, P * A);
    launches += 1;
  }
  const int ckK = ck_count(N);
  if (L.saved_out) {
    write_saved_header(L.saved_out, (double)G, (double)N, (double)kD, (double)P, (double)seg, L.stream, ckK);
  }
  FwdParams prm{agg_st, A, L.carry_prefix, cmb, g, ws.flag, N, G, seg, P, L.row_offset, L.a, L.b, saved, out,
                tuning().prefetch > 0 ? tuning().prefetch : kFPrefetch, saved ? saved + G * P * SZ : nullptr, ckK};
  if (P > 1 && (P - 1) * A > kScanMinRecords) {  // many unit records: one scan launch, not a chain per CTA
    cudaError_t e = seg_scan(agg_st, G, P * A, A, SZ, L.carry_prefix, cmb, SZ, 0, nullptr, L.stream, "la_fwd_scan");
    if (e != cudaSuccess) return e;
    prm.cmb_ready = 1;
    launches += 1;
  }
  {
    ProfScope ps("la_fwd_causal", L.stream);
    main_k<<<dim3(P, G), 448, kFwdSmem, L.stream>>>(mQ64, mK64, mV64, mO64, prm);
  }
  note_launch(launches);
  return cudaGetLastError();
}

}  // namespace lab

extern "C" int la_internal_trace_read(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lab::g_trace, sizeof(lab::g_trace));
}
