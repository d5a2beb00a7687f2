// fp32 inputs on the sm_100a tensor core: 3xTF32 chunked linear attention.
//
// The reference's timed path is run_forward<float> / run_backward<float>
// (forward_kernels.hpp:210-259, backward_kernels.hpp:292-396; bench.cpp:137-139,
// 176-179). One TF32 product misses the 1e-5 relative bar (4.6e-4), so
// every product here is split: x = hi + lo with hi = x with its 13 low mantissa bits
// cleared (exactly a TF32 value) and lo = x - hi (exact in fp32), and
//   X Y ~= X_lo Y_hi + X_hi Y_lo + X_hi Y_hi      (small terms first, fp32 accumulation)
// which leaves ~2^-22 relative per product (SURVEY App. B measured 3e-7 end to end).
//
// One generic kernel covers the forward and the three backward gradients, all of the
// form (rows x_i, k_t, y_t in R^D; i, t over a group's N rows)
//   o_i = sum_{t in T(i)} (alpha_i + alpha'_t + beta x_i . k_t) y_t  [ / g_i ]
//   g_i = sum_{t in T(i)} (alpha_i + alpha'_t + beta x_i . k_t)
// with T(i) = {t <= i} (causal), {t >= i} (anticausal) or all t (full):
//   forward  (forward_kernels.hpp:22-128):  x = q, k = k, y = v, alpha = a, normalised
//   dQ       (backward_kernels.hpp:21-57):  x = w_hat, k = v, y = k, alpha_i = -b s_i
//   dK       (backward_kernels.hpp:61-130): x = v, k = w_hat, y = q, alpha'_t = -b s_t, anti
//   dV       (backward_kernels.hpp:134-168): x = k, k = q, y = w_hat, alpha = a, anti
// (w_hat = omega / g, s_i = o_i . w_hat_i, backward_kernels.hpp:33-38), and the
// non-causal *_full_core variants (forward_kernels.hpp:133-206, backward_kernels.hpp:
// 173-288) with T(i) = all rows.
//
// Chunked form, C = 64 rows per chunk, one CTA per (group, segment), state carried in
// TMEM: S^T[e][d] = sum_t y_te k_td (fp32 master), its beta-scaled TF32 split
// (hi, lo) as the A operand of the inter-chunk product, z = sum k, sigma = sum y,
// sigma' = sum alpha'_t y_t, count, sum alpha'. Per chunk (M = 64 rows i, 128 lanes e):
//   T1 = X K^T (M=64, N=64),  O^T = (beta S)^T X^T  (A from TMEM)
//   P'[i][t] = mask(alpha_i + alpha'_t + beta T1)  -> smem (hi / lo),  g_i
//   O^T += Y^T P'^T,  dS^T = Y^T K (fresh accumulator; S += dS on the CUDA cores, one
//   round-to-nearest add per chunk instead of a tensor-core accumulation per k-step)
// Tiles: every operand is a 64-row x 128-feature fp32 tile (32 KB) loaded by TMA with
// the 128B swizzle; D < 128 reads as zeros (TMA out-of-bounds fill) and stores clip.
// SequenceMajor tiles are K-major over features, FeatureMajor tiles K-major over rows,
// so each operand's UMMA major-ness follows its layout (TF32 takes both).
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace lab {

using namespace sm100;

namespace {

constexpr int kC = 64;                // chunk rows
constexpr int kT = 128;               // tile feature width (D padded)
constexpr uint32_t kTile = 32768;     // 64 x 128 fp32
constexpr int kThreads = 256;
constexpr int64_t kSZ = kT * kT + 3 * kT + 4;  // record: S^T[e][d] | z | sigma | sigma' | count, sum alpha'
constexpr uint32_t cT1 = 0, cO = 64, cS = 128, cSh = 256, cSl = 384;  // TMEM columns
constexpr uint32_t kSmem = 6 * kTile + 8192 + 1024;
enum { kCausal = 0, kAnti = 1, kFull = 2 };
enum { kSweep = 0, kAgg = 1 };

struct F32Params {
  int64_t N;
  int D;
  int seg_chunks;  // chunks per CTA
  int P;           // records per group
  int dir;
  int mode;
  int lx, lk, ly, lo;  // LA_FEATURE_MAJOR / LA_SEQUENCE_MAJOR of X, K, Y and the output
  float alpha_c, alpha_s;
  const float* alpha_v;  // alpha_i = alpha_c + alpha_s * alpha_v[i]
  float alphk_s;
  const float* alphk_v;  // alpha'_t = alphk_s * alphk_v[t] (null: 0)
  float beta;
  int shift;    // Fault::CausalPrefixOffByOne: the beta window of row i ends at i + 1
  float* recs;  // [G][U][kSZ] aggregate-unit records (A units per segment, U = P * A)
  int A, U;        // units per segment, unit records per group
  int unit_chunks; // chunks per aggregate unit
  int u0;          // first unit of the aggregate grid
  int normalize;
  int scanned;  // records hold the scanned carries (k_f32_scan ran)
  float* g;  // [G][N] (normalize)
  unsigned long long* flag;
};

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
#ifndef LA_F32_WRITE_HI
#define LA_F32_WRITE_HI 0
#endif
constexpr bool kWriteHi = LA_F32_WRITE_HI;  // 1: clear the low bits of the hi tiles in smem explicitly
__device__ __forceinline__ void h4_w(uint8_t* hi, int v, float4 x) {
  x.x = __uint_as_float(tf32_hi(x.x)); x.y = __uint_as_float(tf32_hi(x.y));
  x.z = __uint_as_float(tf32_hi(x.z)); x.w = __uint_as_float(tf32_hi(x.w));
  ((float4*)hi)[v] = x;
}

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N, uint32_t a_major, uint32_t b_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_major << 15) | (b_major << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
// K-major tile: `rows` rows of 128 B per 32-element panel (k-step = 8 elements = 32 B).
__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * rows * 128 + (ks & 3) * 32) >> 4);
}
// MN-major tile: 32-bit MN-major operands take only the 128B swizzle with 32-byte
// atoms (descriptor layout type 1, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): K rows of
// 128 B in groups of 4 (SBO = 512 B), 8 rows per k-step, 32-element MN panels `panel`
// bytes apart (LBO).
__device__ __forceinline__ uint64_t mdesc(uint32_t tile, int ks, uint32_t panel) {
  uint64_t d = 0;
  const uint32_t a = tile + ks * 1024;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((panel >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((512u >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
// Operand views of the two tile layouts. A tile holds 64 chunk rows x 128 features:
//   SequenceMajor: [feature panel (4)][row (64)][32 features]
//   FeatureMajor:  [row panel (2)][feature (128)][32 rows]
// desc_rows_k: operand with MN = chunk rows, K = features (SequenceMajor: K-major,
// 16-byte swizzle; FeatureMajor: MN-major, 32-byte swizzle); desc_feat_k: MN = features,
// K = chunk rows (SequenceMajor: MN-major, 32-byte; FeatureMajor: K-major, 16-byte).
__device__ __forceinline__ uint64_t desc_rows_k(uint32_t tile, int ks, int lay) {
  return lay == LA_SEQUENCE_MAJOR ? kdesc(tile, ks, kC) : mdesc(tile, ks, 16384);
}
__device__ __forceinline__ uint64_t desc_feat_k(uint32_t tile, int ks, int lay) {
  return lay == LA_SEQUENCE_MAJOR ? mdesc(tile, ks, 8192) : kdesc(tile, ks, kT);
}
// Physical position of 16-byte chunk c of 128-byte tile row `row`: 128B swizzle with
// 16-byte atoms (chunk ^ row % 8) or with 32-byte atoms (32-byte granule ^ row % 4).
__device__ __forceinline__ uint32_t chunk_pos(uint32_t c, uint32_t row, bool swz32) {
  return swz32 ? ((((c >> 1) ^ (row & 3)) << 1) | (c & 1)) : (c ^ (row & 7));
}
// Byte offset of element (row r < 64, feature f < 128) in a tile of layout `lay`.
__device__ __forceinline__ uint32_t tile_off(int lay, uint32_t r, uint32_t f, bool swz32) {
  if (lay == LA_SEQUENCE_MAJOR) {
    const uint32_t c = f & 31;
    return (f >> 5) * 8192u + r * 128u + (chunk_pos(c >> 2, r, swz32) << 4) + ((c & 3) << 2);
  }
  const uint32_t c = r & 31;
  return (r >> 5) * 16384u + f * 128u + (chunk_pos(c >> 2, f, swz32) << 4) + ((c & 3) << 2);
}
// In-place change of a 32 KB tile's swizzle (256 rows of 128 B, one row per thread):
// the K tile feeds T1 as rows-by-features and dS as features-by-rows, and the two
// operand forms need different swizzles for 32-bit data.
__device__ __forceinline__ void reswizzle(uint8_t* tile, bool from32, int tid) {
  uint8_t* row = tile + tid * 128;
  uint4 v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = *(const uint4*)(row + (chunk_pos(c, tid, from32) << 4));
#pragma unroll
  for (int c = 0; c < 8; ++c) *(uint4*)(row + (chunk_pos(c, tid, !from32) << 4)) = v[c];
}

// The generic sweep / aggregate. Grid (segments, groups), 256 threads, 1 CTA per SM.
__global__ void __launch_bounds__(kThreads, 1)
    k_f32_sweep(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mK,
                const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mO, F32Params prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* tX = smem;  // X (hi, in place), later P' hi
  uint8_t* tK = smem + kTile;  // K (hi), later the output staging tile
  uint8_t* tY = smem + 2 * kTile;
  uint8_t* lX = smem + 3 * kTile;  // lo parts (P' lo in lX)
  uint8_t* lK = smem + 4 * kTile;
  uint8_t* lY = smem + 5 * kTile;
  float* vz = (float*)(smem + 6 * kTile);  // [128] z (sum k) before the chunk
  float* vs = vz + kT;                     // [128] sigma (sum y)
  float* vsp = vs + kT;                    // [128] sigma' (sum alpha' y)
  float* cks = vsp + kT;                   // [128] chunk column sums of k
  float* cys = cks + kT;                   // [128] ... of y
  float* cysp = cys + kT;                  // [128] ... of alpha' y
  float* va = cysp + kT;                   // [64] alpha_i of the chunk rows
  float* vap = va + kC;                    // [64] alpha'_t
  float* xz = vap + kC;                    // [64] x_i . z
  float* gs = xz + kC;                     // [64] g_i
  float* psum = gs + kC;                   // [2][64] row-sum partials of P'
  float* scal = psum + 2 * kC;             // [4] count, sum alpha', chunk sum alpha'
  uint64_t* bars = (uint64_t*)(scal + 8);  // full, mma1, mma2
  uint32_t* tslot = (uint32_t*)(bars + 4);

  const int tid = threadIdx.x, warp = tid >> 5, l = tid & 31;
  const int qd = warp & 3, half = warp >> 2;
  const int64_t grp = blockIdx.y;
  const int p = blockIdx.x;  // sweep: segment; aggregate: unit u0 + p
  const int64_t Nc = prm.N / kC;
  const bool agg_mode = prm.mode == kAgg;
  const int64_t span = agg_mode ? prm.unit_chunks : prm.seg_chunks;
  const int64_t c_lo = lmin(Nc, (int64_t)(agg_mode ? prm.u0 + p : p) * span), c_hi = lmin(Nc, c_lo + span);
  const int nch = (int)(c_hi - c_lo);
  const bool agg = prm.mode == kAgg, full = prm.dir == kFull;
  const bool needX = !agg, needKY = agg || !full;
  const uint32_t lb = (uint32_t)(qd * 32) << 16;
  const int e = qd * 32 + l;  // TMEM lane of the M = 128 accumulators (output feature)
  const float beta = prm.beta;
  const float* recs = prm.recs + grp * prm.U * kSZ;

  if (tid == 0) {
    tma_prefetch(&mX);
    tma_prefetch(&mK);
    tma_prefetch(&mY);
    tma_prefetch(&mO);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // ---- carry: this segment's record after k_f32_scan (exclusive prefix for causal,
  //      exclusive suffix for anticausal, the totals in record 0 for full); zero in agg
  //      mode and when the pass has a single segment
  const int cslot = full ? 0 : prm.dir == kCausal ? p * prm.A : (p + 1) * prm.A - 1;
  const float* crec = (!agg && prm.scanned) ? recs + cslot * kSZ : nullptr;
  for (int j0 = 0; j0 < 64; j0 += 32) {
    const int d0 = half * 64 + j0;
    float acc[32];
    if (crec) {
      const float4* src = (const float4*)(crec + (int64_t)e * kT + d0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 f = __ldg(src + c);
        acc[4 * c] = f.x; acc[4 * c + 1] = f.y; acc[4 * c + 2] = f.z; acc[4 * c + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.f;
    }
    uint32_t x[32], h[32], lo[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      x[c] = __float_as_uint(acc[c]);
      const float bs = beta * acc[c];
      h[c] = tf32_hi(bs);
      lo[c] = __float_as_uint(bs - __uint_as_float(h[c]));
    }
    tmem_st32(tmem + lb + cS + d0, x);
    tmem_st32(tmem + lb + cSh + d0, h);
    tmem_st32(tmem + lb + cSl + d0, lo);
  }
  if (tid < kT) {
    const float* r = crec ? crec + kT * kT : nullptr;
    vz[tid] = r ? r[tid] : 0.f;
    vs[tid] = r ? r[kT + tid] : 0.f;
    vsp[tid] = r ? r[2 * kT + tid] : 0.f;
  }
  if (tid == 0) {
    scal[0] = crec ? crec[kT * kT + 3 * kT] : 0.f;
    scal[1] = crec ? crec[kT * kT + 3 * kT + 1] : 0.f;
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t aX = smem_u32(tX), aK = smem_u32(tK), aY = smem_u32(tY);
  const uint32_t bX = smem_u32(lX), bK = smem_u32(lK), bY = smem_u32(lY);
  const uint32_t ax = prm.lx == LA_SEQUENCE_MAJOR ? 0u : 1u;      // X as MN = rows operand
  const uint32_t ak = prm.lk == LA_SEQUENCE_MAJOR ? 0u : 1u;      // K as MN = rows operand
  const uint32_t ay = prm.ly == LA_SEQUENCE_MAJOR ? 1u : 0u;      // Y as MN = features operand
  const uint32_t akf = prm.lk == LA_SEQUENCE_MAJOR ? 1u : 0u;     // K as MN = features operand
  const uint32_t id_T1 = idesc_tf32(64, 64, ax, ak);
  const uint32_t id_Oi = idesc_tf32(128, 64, 0, ax);              // A = S^T (TMEM), B = X^T
  const uint32_t id_Oa = idesc_tf32(128, 64, ay, 0);              // A = Y^T, B = P'^T (K-major)
  const uint32_t id_dS = idesc_tf32(128, 128, ay, akf);           // A = Y^T, B = K

  auto load_tile = [&](const CUtensorMap* m, uint8_t* dst, int lay, int64_t r0) {
    if (lay == LA_SEQUENCE_MAJOR) {
      for (int pnl = 0; pnl < 4; ++pnl)
        tma_load_3d(dst + pnl * 8192, m, &bars[0], pnl * 32, (int)(grp * prm.N + r0), 0);
    } else {
      for (int pnl = 0; pnl < 2; ++pnl) tma_load_3d(dst + pnl * 16384, m, &bars[0], (int)(r0 + 32 * pnl), 0, (int)grp);
    }
  };

  auto prefetch_tile = [&](const CUtensorMap* mp, int lay, int64_t r0) {
    if (lay == LA_SEQUENCE_MAJOR) {
      for (int pnl = 0; pnl < 4; ++pnl) tma_prefetch_l2_3d(mp, pnl * 32, (int)(grp * prm.N + r0), 0);
    } else {
      for (int pnl = 0; pnl < 2; ++pnl) tma_prefetch_l2_3d(mp, (int)(r0 + 32 * pnl), 0, (int)grp);
    }
  };
  for (int m = 0; m < nch; ++m) {
    const int64_t c = prm.dir == kAnti ? c_hi - 1 - m : c_lo + m;
    const int64_t r0 = c * kC;
    // ------------------------------------------------ loads
    if (tid == 0) {
      tma_store_wait_read0();  // the previous chunk's output staging (tK) has been read
      uint32_t bytes = 0;
      if (needX) bytes += kTile;
      if (needKY) bytes += 2 * kTile;
      mbar_expect_tx(&bars[0], bytes);
      if (needX) load_tile(&mX, tX, prm.lx, r0);
      if (needKY) {
        load_tile(&mK, tK, prm.lk, r0);
        load_tile(&mY, tY, prm.ly, r0);
      }
      if (m + 1 < nch) {  // the next chunk's tiles into L2 while this one computes (one smem stage)
        const int64_t rn = (prm.dir == kAnti ? c_hi - 2 - m : c_lo + m + 1) * kC;
        if (needX) prefetch_tile(&mX, prm.lx, rn);
        if (needKY) {
          prefetch_tile(&mK, prm.lk, rn);
          prefetch_tile(&mY, prm.ly, rn);
        }
      }
    }
    if (tid < kC) {
      const int64_t gi = grp * prm.N + r0 + tid;
      va[tid] = prm.alpha_c + (prm.alpha_v ? prm.alpha_s * __ldg(prm.alpha_v + gi) : 0.f);
    } else if (tid < 2 * kC) {
      const int64_t gi = grp * prm.N + r0 + tid - kC;
      vap[tid - kC] = prm.alphk_v ? prm.alphk_s * __ldg(prm.alphk_v + gi) : 0.f;
    }
    mbar_wait(&bars[0], m & 1);
    __syncthreads();  // va / vap visible
    // ------------------------------------------------ CUDA-core sums on the raw tiles
    if (needX && prm.normalize) {  // x_i . z: 4 threads per row, 32 features (8 x 16 B) each
      const int r = tid >> 2, f0 = (tid & 3) * 32;
      float a = 0.f;
      if (prm.lx == LA_SEQUENCE_MAJOR) {
        const uint8_t* row = tX + (f0 >> 5) * 8192 + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = *(const float4*)(row + (chunk_pos(c, r, false) << 4));
          const float4 z = *(const float4*)(vz + f0 + 4 * c);
          a += x.x * z.x + x.y * z.y + x.z * z.z + x.w * z.w;
        }
      } else {
#pragma unroll 8
        for (int f = 0; f < 32; ++f) a += *(const float*)(tX + tile_off(prm.lx, r, f0 + f, true)) * vz[f0 + f];
      }
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      if ((tid & 3) == 0) xz[r] = a;
    }
    if (needKY) {  // column sums over the chunk rows: feature f, half h of the rows
      const int f = tid & 127, h = tid >> 7;
      // sums of `tile` over rows [32 h, 32 h + 32) for feature f, weighted by w (or 1)
      auto colsum = [&](const uint8_t* tile, int lay, bool swz32, float& s1, float& sw, bool weighted) {
        s1 = 0.f;
        sw = 0.f;
        if (lay == LA_SEQUENCE_MAJOR) {  // a warp reads 32 consecutive features of one row
          const uint8_t* base = tile + (f >> 5) * 8192 + ((f & 3) << 2);
#pragma unroll 8
          for (int r = 32 * h; r < 32 * h + 32; ++r) {
            const float x = *(const float*)(base + r * 128 + (chunk_pos((f & 31) >> 2, r, swz32) << 4));
            s1 += x;
            if (weighted) sw += vap[r] * x;
          }
        } else {  // this thread's own 128-byte tile row (feature f, rows of panel h)
          const uint8_t* row = tile + h * 16384 + f * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = *(const float4*)(row + (chunk_pos(c, f, swz32) << 4));
            s1 += (x.x + x.y) + (x.z + x.w);
            if (weighted) {
              const float* w = vap + 32 * h + 4 * c;
              sw += w[0] * x.x + w[1] * x.y + w[2] * x.z + w[3] * x.w;
            }
          }
        }
      };
      float sk, dummy, sy, syp;
      colsum(tK, prm.lk, prm.lk == LA_FEATURE_MAJOR, sk, dummy, false);
      colsum(tY, prm.ly, prm.ly == LA_SEQUENCE_MAJOR, sy, syp, prm.alphk_v != nullptr);
      if (h == 1) {
        cks[f] = sk;
        cys[f] = sy;
        cysp[f] = syp;
      }
      __syncthreads();
      if (h == 0) {
        cks[f] += sk;
        cys[f] += sy;
        cysp[f] += syp;
      }
    }
    if (tid == 0) {
      float ca = 0.f;
      for (int r = 0; r < kC; ++r) ca += vap[r];
      scal[2] = ca;
    }
    __syncthreads();
    // ------------------------------------------------ TF32 split in place (hi) + lo tiles
    auto split = [&](uint8_t* hi, uint8_t* lo) {
      const float4* h4 = (const float4*)hi;
      float4* l4 = (float4*)lo;
#pragma unroll 4
      for (int v = tid; v < (int)(kTile / 16); v += kThreads) {
        const float4 x = h4[v];
        float4 b;
        b.x = x.x - __uint_as_float(tf32_hi(x.x));
        b.y = x.y - __uint_as_float(tf32_hi(x.y));
        b.z = x.z - __uint_as_float(tf32_hi(x.z));
        b.w = x.w - __uint_as_float(tf32_hi(x.w));
        if (kWriteHi) h4_w(hi, v, x);
        l4[v] = b;
      }
    };
    if (needX) split(tX, lX);
    if (needKY) {
      split(tK, lK);
      split(tY, lY);
    }
    if (agg) {  // K only feeds dS: its features-by-rows swizzle now
      __syncthreads();
      reswizzle(tK, prm.lk == LA_FEATURE_MAJOR, tid);
      reswizzle(lK, prm.lk == LA_FEATURE_MAJOR, tid);
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // ------------------------------------------------ MMA group 1: T1 = X K^T, O^T = (b S)^T X^T
    if (!agg && tid == 0) {
      if (!full) {
        for (int ks = 0; ks < 16; ++ks)
          mma_tf32(tmem + cT1, desc_rows_k(bX, ks, prm.lx), desc_rows_k(aK, ks, prm.lk), id_T1, ks > 0);
        for (int ks = 0; ks < 16; ++ks)
          mma_tf32(tmem + cT1, desc_rows_k(aX, ks, prm.lx), desc_rows_k(bK, ks, prm.lk), id_T1, 1);
        for (int ks = 0; ks < 16; ++ks)
          mma_tf32(tmem + cT1, desc_rows_k(aX, ks, prm.lx), desc_rows_k(aK, ks, prm.lk), id_T1, 1);
      }
      for (int ks = 0; ks < 16; ++ks)
        mma_tf32_ts(tmem + cO, tmem + cSl + 8 * ks, desc_rows_k(aX, ks, prm.lx), id_Oi, ks > 0);
      for (int ks = 0; ks < 16; ++ks)
        mma_tf32_ts(tmem + cO, tmem + cSh + 8 * ks, desc_rows_k(bX, ks, prm.lx), id_Oi, 1);
      for (int ks = 0; ks < 16; ++ks)
        mma_tf32_ts(tmem + cO, tmem + cSh + 8 * ks, desc_rows_k(aX, ks, prm.lx), id_Oi, 1);
      mma_commit(&bars[1]);
    }
    // ------------------------------------------------ E1: P' (hi -> tX, lo -> lX) and g
    if (!agg) {
      mbar_wait(&bars[1], m & 1);
      tc_fence_after();
      const float cnt = scal[0], ca = scal[1];
      if (!full) {
        uint32_t x[32];
        tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + cT1 + 32 * half, x);  // M = 64: rows in lanes 0..15
        tmem_ld_wait();
        const int i = qd * 16 + (l & 15);
        if (l < 16) {
          const float ai = va[i];
          float rs = 0.f;
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            float pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = 32 * half + 4 * c8 + u;
              const bool on = prm.dir == kCausal ? t <= i : t >= i;
              const bool on_b = prm.shift ? t <= i + 1 : on;
              const float bt = beta * __uint_as_float(x[4 * c8 + u]);
              pv[u] = (on ? ai + vap[t] : 0.f) + (on_b ? bt : 0.f);
              rs += on ? ai + vap[t] + bt : 0.f;
            }
            float4 a, b;
            a.x = __uint_as_float(tf32_hi(pv[0])); b.x = pv[0] - a.x;
            a.y = __uint_as_float(tf32_hi(pv[1])); b.y = pv[1] - a.y;
            a.z = __uint_as_float(tf32_hi(pv[2])); b.z = pv[2] - a.z;
            a.w = __uint_as_float(tf32_hi(pv[3])); b.w = pv[3] - a.w;
            const uint32_t off = half * 8192u + i * 128u + (((uint32_t)c8 ^ (i & 7)) << 4);  // K-major [t panel][i][32 t]
            *(float4*)(tX + off) = a;
            *(float4*)(lX + off) = b;
          }
          psum[half * kC + i] = rs;
        }
      }
      if (!full) {  // T1 has read K: switch it to the swizzle of its dS operand form
        reswizzle(tK, prm.lk == LA_FEATURE_MAJOR, tid);
        reswizzle(lK, prm.lk == LA_FEATURE_MAJOR, tid);
      }
      __syncthreads();
      if (tid < kC && prm.normalize) {
        const int i = tid;
        float gi = va[i] * cnt + ca + beta * xz[i];
        if (!full) gi += psum[i] + psum[kC + i];
        gs[i] = 1.f / gi;  // the drain multiplies (<= 1 ulp from the reference's divide)
        const int64_t row = r0 + i;
        prm.g[grp * prm.N + row] = gi;
        if (!(fabsf(gi) >= kEpsF32)) flag_degenerate(prm.flag, grp, row);
      }
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
    }
    // ------------------------------------------------ MMA group 2: O^T += Y^T P'^T, dS^T = Y^T K
    if (tid == 0 && needKY) {
      if (!agg) {
        const uint32_t pH = aX, pL = bX;
        for (int ks = 0; ks < 8; ++ks)
          mma_tf32(tmem + cO, desc_feat_k(bY, ks, prm.ly), kdesc(pH, ks, kC), id_Oa, 1);
        for (int ks = 0; ks < 8; ++ks)
          mma_tf32(tmem + cO, desc_feat_k(aY, ks, prm.ly), kdesc(pL, ks, kC), id_Oa, 1);
        for (int ks = 0; ks < 8; ++ks)
          mma_tf32(tmem + cO, desc_feat_k(aY, ks, prm.ly), kdesc(pH, ks, kC), id_Oa, 1);
      }
      for (int ks = 0; ks < 8; ++ks)
        mma_tf32(tmem + cSl, desc_feat_k(bY, ks, prm.ly), desc_feat_k(aK, ks, prm.lk), id_dS, ks > 0);
      for (int ks = 0; ks < 8; ++ks)
        mma_tf32(tmem + cSl, desc_feat_k(aY, ks, prm.ly), desc_feat_k(bK, ks, prm.lk), id_dS, 1);
      for (int ks = 0; ks < 8; ++ks)
        mma_tf32(tmem + cSl, desc_feat_k(aY, ks, prm.ly), desc_feat_k(aK, ks, prm.lk), id_dS, 1);
      mma_commit(&bars[2]);
    }
    if (needKY) mbar_wait(&bars[2], m & 1);
    tc_fence_after();
    // ------------------------------------------------ E2: output drain -> staging (tK) -> TMA store
    if (!agg) {
      uint32_t x[32];
      tmem_ld32(tmem + lb + cO + 32 * half, x);
      tmem_ld_wait();
      const float se = vs[e], spe = vsp[e];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = 32 * half + k;
        float o = __uint_as_float(x[k]) + va[i] * se + spe;
        if (prm.normalize) o *= gs[i];
        x[k] = __float_as_uint(o);
      }
      if (prm.lo == LA_FEATURE_MAJOR) {  // [i panel][e][32 i]: this thread's 32 rows are one 128 B row
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8)
          *(uint4*)(tK + half * 16384u + e * 128u + (((uint32_t)c8 ^ (e & 7)) << 4)) =
              make_uint4(x[4 * c8], x[4 * c8 + 1], x[4 * c8 + 2], x[4 * c8 + 3]);
      } else {  // [e panel][i][32 e]
#pragma unroll
        for (int k = 0; k < 32; ++k) *(uint32_t*)(tK + tile_off(LA_SEQUENCE_MAJOR, 32 * half + k, e, false)) = x[k];
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        if (prm.lo == LA_FEATURE_MAJOR) {
          for (int pnl = 0; pnl < 2; ++pnl) tma_store_3d(&mO, tK + pnl * 16384, (int)(r0 + 32 * pnl), 0, (int)grp);
        } else {
          for (int pnl = 0; pnl < 4; ++pnl) tma_store_3d(&mO, tK + pnl * 8192, pnl * 32, (int)(grp * prm.N + r0), 0);
        }
        tma_store_commit();
      }
    }
    // ------------------------------------------------ state update: S += dS (RN), split, vectors
    if (needKY) {
      for (int j0 = 0; j0 < 64; j0 += 32) {
        const uint32_t col = half * 64 + j0;
        uint32_t s[32], d[32];
        tmem_ld32(tmem + lb + cS + col, s);
        tmem_ld32(tmem + lb + cSl + col, d);
        tmem_ld_wait();
        uint32_t h[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float sn = __uint_as_float(s[k]) + __uint_as_float(d[k]);
          s[k] = __float_as_uint(sn);
          const float bs = beta * sn;
          h[k] = tf32_hi(bs);
          d[k] = __float_as_uint(bs - __uint_as_float(h[k]));
        }
        tmem_st32(tmem + lb + cS + col, s);
        if (!agg) {
          tmem_st32(tmem + lb + cSh + col, h);
          tmem_st32(tmem + lb + cSl + col, d);
        }
      }
      if (tid < kT) {
        vz[tid] += cks[tid];
        vs[tid] += cys[tid];
        vsp[tid] += cysp[tid];
      }
      if (tid == 0) {
        scal[0] += (float)kC;
        scal[1] += scal[2];
      }
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  // ---- aggregate: write this segment's record
  if (agg) {
    float* rec = prm.recs + (grp * prm.U + prm.u0 + p) * kSZ;
    for (int j0 = 0; j0 < 64; j0 += 32) {
      const uint32_t col = half * 64 + j0;
      uint32_t s[32];
      tmem_ld32(tmem + lb + cS + col, s);
      tmem_ld_wait();
      float4* dst = (float4*)(rec + (int64_t)e * kT + col);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        dst[c] = make_float4(__uint_as_float(s[4 * c]), __uint_as_float(s[4 * c + 1]), __uint_as_float(s[4 * c + 2]),
                             __uint_as_float(s[4 * c + 3]));
    }
    if (tid < kT) {
      rec[kT * kT + tid] = vz[tid];
      rec[kT * kT + kT + tid] = vs[tid];
      rec[kT * kT + 2 * kT + tid] = vsp[tid];
    }
    if (tid == 0) {
      rec[kT * kT + 3 * kT] = scal[0];
      rec[kT * kT + 3 * kT + 1] = scal[1];
    }
  }
  if (tid == 0) tma_store_wait0();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// w_hat = omega / g (FeatureMajor, into `wh`), s_i = sum_j o_ij w_hat_ij (make_omega_hat
// backward.cpp:74-91; backward_kernels.hpp:33-38). Thread per row i, loop over j.
__global__ void k_f32_what(const float* o, const float* w, int lw, const float* g, float* wh, float* s, int64_t N,
                           int D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (i >= N) return;
  const float gi = g[grp * N + i];
  const Strides sw = strides_of(lw, N, D);
  const float* wg = w + grp * N * D;
  float acc = 0.f;
  for (int j = 0; j < D; ++j) {
    const int64_t ix = (grp * D + j) * N + i;
    const float wv = wg[i * sw.is + j * sw.js] / gi;
    wh[ix] = wv;
    acc += o[ix] * wv;
  }
  s[grp * N + i] = acc;
}

// Unit records [u0, u1) -> carries, in place, per element (coalesced over the record):
// causal: exclusive prefix (segment p reads slot p * A); anticausal: exclusive suffix
// (slot (p + 1) * A - 1); full: the totals in slot 0.
__global__ void k_f32_scan(float* recs, int U, int u0, int u1, int dir) {
  const int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (el >= kSZ) return;
  float* r = recs + (int64_t)blockIdx.y * U * kSZ + el;
  float run = 0.f;
  if (dir == kFull) {
    for (int q = u0; q < u1; ++q) run += r[q * kSZ];
    r[0] = run;
  } else if (dir == kCausal) {
    for (int q = u0; q < u1; ++q) {
      const float t = r[q * kSZ];
      r[q * kSZ] = run;
      run += t;
    }
    if (u1 < U) r[u1 * kSZ] = run;
  } else {
    for (int q = u1 - 1; q >= u0; --q) {
      const float t = r[q * kSZ];
      r[q * kSZ] = run;
      run += t;
    }
    if (u0 > 0) r[(u0 - 1) * kSZ] = run;
  }
}

// fp32 TMA maps: SequenceMajor [G*N][D] as {D, G*N, 1} with {32, 64, 1} boxes (one
// 32-feature panel per load); FeatureMajor [G][D][N] as {N, D, G} with {32, 128, 1}
// boxes (one 32-row panel). D < 128 reads as zeros / stores clip.
bool f32_map(CUtensorMap* m, const void* base, int lay, int64_t G, int64_t N, int64_t D, bool swz32) {
  cuuint64_t dims[3];
  cuuint64_t strides[2];
  cuuint32_t box[3];
  if (lay == LA_SEQUENCE_MAJOR) {
    dims[0] = (cuuint64_t)D; dims[1] = (cuuint64_t)(G * N); dims[2] = 1;
    strides[0] = (cuuint64_t)D * 4; strides[1] = (cuuint64_t)(G * N * D) * 4;
    box[0] = 32; box[1] = kC; box[2] = 1;
  } else {
    dims[0] = (cuuint64_t)N; dims[1] = (cuuint64_t)D; dims[2] = (cuuint64_t)G;
    strides[0] = (cuuint64_t)N * 4; strides[1] = (cuuint64_t)(D * N) * 4;
    box[0] = 32; box[1] = kT; box[2] = 1;
  }
  cuuint32_t es[3] = {1, 1, 1};
  return tma_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swz32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int f32_segments(int64_t G, int64_t N) {
  const int64_t nc = N / kC;
  int64_t P = G >= 148 ? 1 : 148 / G;
  if (const int s = tuning().segments) P = s;
  P = std::max<int64_t>(1, std::min<int64_t>(P, nc));
  const int64_t seg = (nc + P - 1) / P;
  return (int)((nc + seg - 1) / seg);  // no empty trailing segment
}

// Aggregate units per segment: split the aggregated segments so the aggregate grid fills
// the SMs (units must tile the segment's chunks).
int f32_units(int64_t G, int P, int seg, int dir) {
  const int64_t segs = dir == kFull ? P : P - 1;
  if (segs <= 0) return 1;
  int best = 1;
  for (int a = 1; a <= 16; ++a) {
    if (seg % a) continue;
    if (G * segs * a <= 148) best = a;
  }
  return best;
}

size_t f32_unit_slots(int64_t G, int64_t N) {
  const int P = f32_segments(G, N);
  const int seg = (int)((N / kC + P - 1) / P);
  const int a = std::max(f32_units(G, P, seg, kCausal), f32_units(G, P, seg, kFull));
  return (size_t)(G * P * a);
}

struct Operand {
  const void* ptr;
  int lay;
};

// One instance of the generic pass: the aggregate over P segments, then the sweep (or,
// non-causal, the apply pass over every chunk with the totals).
cudaError_t f32_pass(const Launch& L, Operand X, Operand K, Operand Y, void* out, int lo, int dir, float alpha_c,
                     float alpha_s, const float* alpha_v, float alphk_s, const float* alphk_v, bool normalize,
                     int shift, float* g, unsigned long long* flag, float* recs, const char* name) {
  const int64_t G = L.G, N = L.N;
  const int D = (int)L.D;
  CUtensorMap mX, mK, mY, mO;
  // load swizzles: the T1-time operand forms (X, K rows-by-features; Y features-by-rows)
  if (!f32_map(&mX, X.ptr, X.lay, G, N, D, X.lay == LA_FEATURE_MAJOR) ||
      !f32_map(&mK, K.ptr, K.lay, G, N, D, K.lay == LA_FEATURE_MAJOR) ||
      !f32_map(&mY, Y.ptr, Y.lay, G, N, D, Y.lay == LA_SEQUENCE_MAJOR) || !f32_map(&mO, out, lo, G, N, D, false))
    return cudaErrorInvalidValue;
  const int P = f32_segments(G, N);
  const int64_t nc = N / kC;
  const int seg = (int)((nc + P - 1) / P);
  const int A = f32_units(G, P, seg, dir);
  F32Params prm{N, D, seg, P, dir, kAgg, X.lay, K.lay, Y.lay, lo, alpha_c, alpha_s, alpha_v, alphk_s, alphk_v, L.b,
                shift, recs, A, P * A, seg / A, 0, normalize ? 1 : 0, 0, g, flag};
  cudaFuncSetAttribute(k_f32_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  if (P > 1 || dir == kFull) {
    // only the segments whose sums some sweep needs: causal 0..P-2, anticausal 1..P-1
    const int s0 = dir == kAnti ? 1 : 0, s1 = dir == kCausal ? P - 1 : P;
    prm.u0 = s0 * A;
    {
      ProfScope ps("la_f32_agg", L.stream);
      k_f32_sweep<<<dim3((unsigned)((s1 - s0) * A), (unsigned)G), kThreads, kSmem, L.stream>>>(mX, mK, mY, mO, prm);
    }
    k_f32_scan<<<dim3((unsigned)((kSZ + 255) / 256), (unsigned)G), 256, 0, L.stream>>>(recs, P * A, s0 * A, s1 * A,
                                                                                     dir);
    note_launch(2);
    prm.scanned = 1;
  }
  prm.mode = kSweep;
  {
    ProfScope ps(name, L.stream);
    k_f32_sweep<<<dim3(P, (unsigned)G), kThreads, kSmem, L.stream>>>(mX, mK, mY, mO, prm);
    note_launch(1);
  }
  return cudaGetLastError();
}

}  // namespace

bool f32tc_supported(const Launch& L, const Tensors& t) {
  (void)t;
  return L.dtype == LA_F32 && L.D % 4 == 0 && L.D <= kT && L.N % kC == 0 && L.carry_prefix == nullptr &&
         L.carry_suffix == nullptr && L.row_offset == 0 && L.n_total == L.N && L.G * L.N < (1ll << 31) &&
         L.G < 65536;
}

size_t f32tc_ws_floats(int64_t G, int64_t N, int64_t D) {
  (void)D;
  if (N % kC) return 0;
  return f32_unit_slots(G, N) * kSZ + (size_t)(G * N);  // unit records + s
}

cudaError_t f32tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const int dir = L.causal ? kCausal : kFull;
  const int shift = L.causal && L.fault == LA_FAULT_CAUSAL_PREFIX_OFF_BY_ONE ? 1 : 0;
  cudaError_t e = f32_pass(L, {t.q, t.lq}, {t.k, t.lk}, {t.v, t.lv}, out, LA_FEATURE_MAJOR, dir, L.a, 0.f, nullptr,
                           0.f, nullptr, true, shift, g, ws.flag, ws.base,
                           L.causal ? "la_f32_fwd_causal" : "la_f32_fwd_full");
  if (e != cudaSuccess || !shift) return e;
  return offbyone_fix(L, t, out, g);
}

// Backward: w_hat (into the dV buffer) and s, then dQ, dK and dV as three instances of
// the generic pass; dV last, over its own w_hat input (each chunk is loaded before its
// output tile is stored, and segments are disjoint).
cudaError_t f32tc_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws) {
  const int64_t G = L.G, N = L.N;
  const int D = (int)L.D;
  float* recs = ws.base;
  float* s = ws.base + f32_unit_slots(G, N) * kSZ;
  {
    ProfScope ps("la_f32_what", L.stream);
    k_f32_what<<<dim3((unsigned)((N + 255) / 256), (unsigned)G), 256, 0, L.stream>>>(
        (const float*)t.o, (const float*)t.w, t.lw, t.g, (float*)dv, s, N, D);
    note_launch(1);
  }
  const int fwd = L.causal ? kCausal : kFull, rev = L.causal ? kAnti : kFull;
  const float b = L.b;
  const float kbeta = L.fault == LA_FAULT_FLIP_BETA_K_SIGN ? b : -b;              // backward_kernels.hpp:104, 224
  const float va = L.fault == LA_FAULT_DROP_GRAD_V_CONSTANT_TERM ? 0.f : L.a;      // backward_kernels.hpp:144, 262
  cudaError_t e;
  // dq_i = sum_{t<=i} (b w_i.v_t - b s_i) k_t
  e = f32_pass(L, {dv, LA_FEATURE_MAJOR}, {t.v, t.lv}, {t.k, t.lk}, dq, LA_SEQUENCE_MAJOR, fwd, 0.f, -b, s, 0.f,
               nullptr, false, 0, nullptr, ws.flag, recs, "la_f32_bwd_dq");
  if (e != cudaSuccess) return e;
  // dk_i = sum_{t>=i} (b v_i.w_t - b s_t) q_t
  e = f32_pass(L, {t.v, t.lv}, {dv, LA_FEATURE_MAJOR}, {t.q, t.lq}, dk, LA_FEATURE_MAJOR, rev, 0.f, 0.f, nullptr,
               kbeta, s, false, 0, nullptr, ws.flag, recs, "la_f32_bwd_dk");
  if (e != cudaSuccess) return e;
  // dv_i = sum_{t>=i} (a + b k_i.q_t) w_t
  return f32_pass(L, {t.k, t.lk}, {t.q, t.lq}, {dv, LA_FEATURE_MAJOR}, dv, LA_FEATURE_MAJOR, rev, va, 0.f, nullptr,
                  0.f, nullptr, false, 0, nullptr, ws.flag, recs, "la_f32_bwd_dv");
}

}  // namespace lab
