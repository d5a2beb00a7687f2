// Generic 16-bit (bf16 / fp16) tensor-core sweep: the causal and non-causal forward
// and the dQ / dK / dV gradients for every shape the specialised kernels
// (la_sm100.cu, la_sm100_bwd.cu, la_full.cu) do not take:
//   * any head dimension D <= 256 (D % 8 == 0) natively -- no zero-padded copies;
//     D > 128 runs the output features in two halves of 128;
//   * any layout of q, k, v, omega (each operand's UMMA major-ness follows its
//     layout, tensor.cpp:35-41 index maps);
//   * the three Fault mutations (fault.hpp:7-15; forward_kernels.hpp:86-106,
//     backward_kernels.hpp:104, 123-127, 144, 165, 224, 262).
// Same formulation as the fp32 path (la_f32tc.cu): with rows x_i, k_t, y_t,
//   o_i = sum_{t in T(i)} (alpha_i + alpha'_t + beta x_i . k_t) y_t  [ / g_i ]
// over T(i) = {t <= i} / {t >= i} / all t, one kernel instance per output:
//   forward x=q k=k y=v alpha=a (normalised); dQ x=w_hat k=v y=k alpha_i=-b s_i;
//   dK x=v k=w_hat y=q alpha'_t=-b s_t (anti); dV x=k k=q y=w_hat alpha=a (anti).
// Chunk C = 64 rows, one CTA per (group, segment), two-stage TMA ring, fp32 state
// S^T[e][d] accumulated by the tensor core in TMEM and its bf16/fp16 copy b*S^T as the
// A operand of the inter-chunk product (read from TMEM).
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace lab {

using namespace sm100;

namespace {

constexpr int kC = 64;          // chunk rows
constexpr int kE = 128;         // output features per pass (TMEM lanes)
constexpr int kThreads = 256;
enum { kCausal = 0, kAnti = 1, kFull = 2 };
enum { kSweep = 0, kAgg = 1 };

template <int kDK>
struct G16 {
  static constexpr uint32_t kXT = kDK * 128;  // X / K tile: 64 rows x kDK 16-bit features
  static constexpr uint32_t kYT = kE * 128;   // Y tile: 64 rows x 128 features
  static constexpr uint32_t kStage = 2 * kXT + kYT;
  static constexpr uint32_t kPT = 8192;       // P' 64 x 64
  static constexpr uint32_t kOT = kE * 128;   // output staging
  static constexpr int64_t kSZ = (int64_t)kE * kDK + kDK + 2 * kE + 4;  // S^T[e][d] | z | sigma | sigma' | cnt, ca
  static constexpr uint32_t kSmem = 2 * kStage + kPT + kOT + 8192 + 1024;
  static constexpr uint32_t cT1 = 0, cO = 64, cS = 128, cSb = 128 + kDK;  // TMEM columns
};

struct G16Params {
  int64_t N;
  int D;         // features of x and k (<= kDK)
  int e0;        // first output feature of this pass (y / out columns e0 .. e0 + 127)
  int DY;        // features of y / out
  int seg_chunks, P;
  int dir, mode;
  int lx, lk, ly, lo;
  float alpha_c, alpha_s;
  const float* alpha_v;
  float alphk_s;
  const float* alphk_v;
  float beta;
  int shift;     // Fault::CausalPrefixOffByOne: the beta window of row i ends at i + 1
  float* recs;   // [G][U][kSZ]
  int A, U, unit_chunks, u0;
  int normalize, scanned;
  float* g;
  unsigned long long* flag;
  float n_total;  // non-causal normaliser length when rows were zero-padded (0: the row count)
};

// K-major tile: `rows` rows of 128 B per 64-element panel (k-step = 16 elements = 32 B).
__device__ __forceinline__ uint64_t kd16(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * rows * 128 + (ks & 3) * 32) >> 4);
}
// MN-major tile: K rows of 128 B (16 per k-step), 64-element MN panels `panel` bytes apart.
__device__ __forceinline__ uint64_t mn16(uint32_t tile, int ks, uint32_t panel) {
  return sdesc_sw128(tile, panel, 1024) + (uint64_t)((ks * 2048) >> 4);
}
// Tiles: SequenceMajor [feature panel][64 rows][64 features]; FeatureMajor [features][64 rows].
// rows-by-features operand (MN = chunk rows, K = features) and features-by-rows (MN =
// features, K = chunk rows) views.
__device__ __forceinline__ uint64_t d_rows(uint32_t tile, int ks, int lay) {
  return lay == LA_SEQUENCE_MAJOR ? kd16(tile, ks, kC) : mn16(tile, ks, 8192);
}
__device__ __forceinline__ uint64_t d_feat(uint32_t tile, int ks, int lay, uint32_t feats) {
  return lay == LA_SEQUENCE_MAJOR ? mn16(tile, ks, 8192) : kd16(tile, ks, feats);
}
// Byte offset of element (row r < 64, feature f) in a 16-bit tile of layout `lay`.
__device__ __forceinline__ uint32_t off16(int lay, uint32_t r, uint32_t f) {
  if (lay == LA_SEQUENCE_MAJOR) return sw128_off(r, f, kC);
  return f * 128u + ((((r >> 3) ^ (f & 7))) << 4) + ((r & 7) << 1);
}

template <bool kBF16, int kDK>
__global__ void __launch_bounds__(kThreads, 1)
    k_g16_sweep(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mK,
                const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mO, G16Params prm) {
  using Gm = G16<kDK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sP = smem + 2 * Gm::kStage;
  uint8_t* sO = sP + Gm::kPT;
  float* vz = (float*)(sO + Gm::kOT);  // [kDK] z before the chunk
  float* cks = vz + kDK;               // [kDK] chunk sums of k
  float* vs = cks + kDK;               // [128] sigma
  float* vsp = vs + kE;                // [128] sigma'
  float* cys = vsp + kE;               // [128] chunk sums of y
  float* cysp = cys + kE;              // [128] ... of alpha' y
  float* va = cysp + kE;               // [64]
  float* vap = va + kC;                // [64]
  float* xz = vap + kC;                // [64]
  float* gs = xz + kC;                 // [64] 1 / g
  float* psum = gs + kC;               // [2][64]
  float* scal = psum + 2 * kC;         // count, sum alpha', chunk sum alpha'
  uint64_t* bars = (uint64_t*)(scal + 8);  // full[2], mma1, mma2
  uint32_t* tslot = (uint32_t*)(bars + 4);

  const int tid = threadIdx.x, warp = tid >> 5, l = tid & 31;
  const int qd = warp & 3, half = warp >> 2;
  const int64_t grp = blockIdx.y;
  const int p = blockIdx.x;
  const int64_t Nc = prm.N / kC;
  const bool agg = prm.mode == kAgg, full = prm.dir == kFull;
  const int64_t span = agg ? prm.unit_chunks : prm.seg_chunks;
  const int64_t c_lo = lmin(Nc, (int64_t)(agg ? prm.u0 + p : p) * span), c_hi = lmin(Nc, c_lo + span);
  const int nch = (int)(c_hi - c_lo);
  const bool needX = !agg, needKY = agg || !full;
  const uint32_t lb = (uint32_t)(qd * 32) << 16;
  const int e = qd * 32 + l;
  const float beta = prm.beta;
  const float* recs = prm.recs + grp * prm.U * Gm::kSZ;
  constexpr uint32_t fmt = kBF16 ? 1 : 0;

  if (tid == 0) {
    tma_prefetch(&mX);
    tma_prefetch(&mK);
    tma_prefetch(&mY);
    tma_prefetch(&mO);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  auto chunk_of = [&](int m) -> int64_t { return prm.dir == kAnti ? c_hi - 1 - m : c_lo + m; };
  auto load_chunk = [&](int m) {
    const int s = m & 1;
    uint8_t* st = smem + s * Gm::kStage;
    const int64_t r0 = chunk_of(m) * kC;
    uint32_t bytes = 0;
    if (needX) bytes += Gm::kXT;
    if (needKY) bytes += Gm::kXT + Gm::kYT;
    mbar_expect_tx(&bars[s], bytes);
    auto load = [&](const CUtensorMap* mp, uint8_t* dst, int lay, int feats, int f0) {
      if (lay == LA_SEQUENCE_MAJOR) {
        for (int pnl = 0; pnl < feats / 64; ++pnl)
          tma_load_3d(dst + pnl * 8192, mp, &bars[s], f0 + pnl * 64, (int)(grp * prm.N + r0), 0);
      } else {
        tma_load_3d(dst, mp, &bars[s], (int)r0, f0, (int)grp);
      }
    };
    if (needX) load(&mX, st, prm.lx, kDK, 0);
    if (needKY) {
      load(&mK, st + Gm::kXT, prm.lk, kDK, 0);
      load(&mY, st + 2 * Gm::kXT, prm.ly, kE, prm.e0);
    }
  };
  if (tid == 0 && nch > 0) {
    load_chunk(0);
    if (nch > 1) load_chunk(1);
  }

  // ---- carry (after the scan of the unit records), or zero
  const int cslot = full ? 0 : prm.dir == kCausal ? p * prm.A : (p + 1) * prm.A - 1;
  const float* crec = (!agg && prm.scanned) ? recs + cslot * Gm::kSZ : nullptr;
  auto write_bS = [&](const float* src_or_null, bool from_tmem) {
    // this thread: lane e, features [half * kDK / 2, + kDK / 2) of S^T -> fp32 S (unless
    // from_tmem) and the 16-bit copy of b * S^T, packed in pairs
    for (int j0 = 0; j0 < kDK / 2; j0 += 32) {
      const int d0 = half * (kDK / 2) + j0;
      uint32_t x[32];
      if (from_tmem) {
        tmem_ld32(tmem + lb + Gm::cS + d0, x);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          float4 f = src_or_null ? __ldg((const float4*)(src_or_null + (int64_t)e * kDK + d0 + c))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
          x[c] = __float_as_uint(f.x); x[c + 1] = __float_as_uint(f.y);
          x[c + 2] = __float_as_uint(f.z); x[c + 3] = __float_as_uint(f.w);
        }
        tmem_st32(tmem + lb + Gm::cS + d0, x);
      }
      uint32_t h[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        h[c] = pack2<kBF16>(beta * __uint_as_float(x[2 * c]), beta * __uint_as_float(x[2 * c + 1]));
      tmem_st16(tmem + lb + Gm::cSb + d0 / 2, h);
    }
  };
  write_bS(crec, false);
  if (tid < kDK) {
    vz[tid] = crec ? crec[kE * kDK + tid] : 0.f;
  }
  if (tid < kE) {
    vs[tid] = crec ? crec[kE * kDK + kDK + tid] : 0.f;
    vsp[tid] = crec ? crec[kE * kDK + kDK + kE + tid] : 0.f;
  }
  if (tid == 0) {
    scal[0] = crec ? crec[kE * kDK + kDK + 2 * kE] : 0.f;
    scal[1] = crec ? crec[kE * kDK + kDK + 2 * kE + 1] : 0.f;
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t ax = prm.lx == LA_SEQUENCE_MAJOR ? 0u : 1u;
  const uint32_t ak = prm.lk == LA_SEQUENCE_MAJOR ? 0u : 1u;
  const uint32_t ay = prm.ly == LA_SEQUENCE_MAJOR ? 1u : 0u;
  const uint32_t akf = prm.lk == LA_SEQUENCE_MAJOR ? 1u : 0u;
  const uint32_t id_T1 = idesc_f16(64, 64, fmt, ax, ak);
  const uint32_t id_Oi = idesc_f16(kE, 64, fmt, 0, ax);
  const uint32_t id_Oa = idesc_f16(kE, 64, fmt, ay, 0);
  const uint32_t id_S = idesc_f16(kE, kDK, fmt, ay, akf);
  const uint32_t aP = smem_u32(sP);

  for (int m = 0; m < nch; ++m) {
    const int s = m & 1;
    uint8_t* st = smem + s * Gm::kStage;
    uint8_t *tX = st, *tK = st + Gm::kXT, *tY = st + 2 * Gm::kXT;
    const uint32_t aX = smem_u32(tX), aK = smem_u32(tK), aY = smem_u32(tY);
    const int64_t r0 = chunk_of(m) * kC;
    if (tid < kC) {
      const int64_t gi = grp * prm.N + r0 + tid;
      va[tid] = prm.alpha_c + (prm.alpha_v ? prm.alpha_s * __ldg(prm.alpha_v + gi) : 0.f);
    } else if (tid < 2 * kC) {
      const int64_t gi = grp * prm.N + r0 + tid - kC;
      vap[tid - kC] = prm.alphk_v ? prm.alphk_s * __ldg(prm.alphk_v + gi) : 0.f;
    }
    mbar_wait(&bars[s], (m >> 1) & 1);
    __syncthreads();
    // ------------------------------------------------ CUDA-core sums
    if (needX && prm.normalize) {  // x_i . z, 4 threads per row
      const int r = tid >> 2;
      float a = 0.f;
      for (int f = (tid & 3); f < prm.D; f += 4) {
        const uint16_t hv = *(const uint16_t*)(tX + off16(prm.lx, r, f));
        a += (kBF16 ? __bfloat162float(__ushort_as_bfloat16(hv)) : __half2float(__ushort_as_half(hv))) * vz[f];
      }
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      if ((tid & 3) == 0) xz[r] = a;
    }
    if (needKY) {
      auto h2f = [](uint16_t hv) {
        return kBF16 ? __bfloat162float(__ushort_as_bfloat16(hv)) : __half2float(__ushort_as_half(hv));
      };
      for (int f = tid; f < kDK; f += kThreads) {  // k column sums
        float sk = 0.f;
        if (prm.lk == LA_FEATURE_MAJOR) {
          const uint8_t* row = tK + f * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = *(const uint4*)(row + ((c ^ (f & 7)) << 4));
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 t2 = unpack2<kBF16>(w4[q]);
              sk += t2.x + t2.y;
            }
          }
        } else {
          for (int r = 0; r < kC; ++r) sk += h2f(*(const uint16_t*)(tK + off16(prm.lk, r, f)));
        }
        cks[f] = sk;
      }
      if (tid < kE) {  // y column sums (plain and alpha'-weighted)
        const int f = tid;
        float sy = 0.f, syp = 0.f;
        if (prm.ly == LA_FEATURE_MAJOR) {
          const uint8_t* row = tY + f * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = *(const uint4*)(row + ((c ^ (f & 7)) << 4));
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 t2 = unpack2<kBF16>(w4[q]);
              sy += t2.x + t2.y;
              syp += vap[8 * c + 2 * q] * t2.x + vap[8 * c + 2 * q + 1] * t2.y;
            }
          }
        } else {
          for (int r = 0; r < kC; ++r) {
            const float y = h2f(*(const uint16_t*)(tY + off16(prm.ly, r, f)));
            sy += y;
            syp += vap[r] * y;
          }
        }
        cys[f] = sy;
        cysp[f] = syp;
      }
    }
    if (tid == 0) {
      float ca = 0.f;
      for (int r = 0; r < kC; ++r) ca += vap[r];
      scal[2] = ca;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // ------------------------------------------------ MMA group 1: T1 = X K^T, O^T = (b S)^T X^T
    if (!agg && tid == 0) {
      if (!full)
        for (int ks = 0; ks < kDK / 16; ++ks)
          mma_ss(tmem + Gm::cT1, d_rows(aX, ks, prm.lx), d_rows(aK, ks, prm.lk), id_T1, ks > 0);
      for (int ks = 0; ks < kDK / 16; ++ks)
        mma_ts(tmem + Gm::cO, tmem + Gm::cSb + 8 * ks, d_rows(aX, ks, prm.lx), id_Oi, ks > 0);
      mma_commit(&bars[2]);
    }
    // ------------------------------------------------ E1: P' -> sP, g
    if (!agg) {
      mbar_wait(&bars[2], m & 1);
      tc_fence_after();
      if (!full) {
        uint32_t x[32];
        tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + Gm::cT1 + 32 * half, x);
        tmem_ld_wait();
        const int i = qd * 16 + (l & 15);
        if (l < 16) {
          const float ai = va[i];
          float rs = 0.f;
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t pk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float pv2[2];
#pragma unroll
              for (int w = 0; w < 2; ++w) {
                const int t = 32 * half + 8 * c8 + 2 * u + w;
                const float bt = beta * __uint_as_float(x[8 * c8 + 2 * u + w]);
                const bool on = prm.dir == kCausal ? t <= i : t >= i;
                const bool on_b = prm.shift ? t <= i + 1 : on;
                pv2[w] = (on ? ai + vap[t] : 0.f) + (on_b ? bt : 0.f);
                rs += on ? ai + vap[t] + bt : 0.f;
              }
              pk[u] = pack2<kBF16>(pv2[0], pv2[1]);
            }
            *(uint4*)(sP + sw128_off(i, 32 * half + 8 * c8, kC)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          psum[half * kC + i] = rs;
        }
      }
      __syncthreads();
      if (tid < kC && prm.normalize) {
        const int i = tid;
        const float cnt = (full && prm.n_total > 0.f) ? prm.n_total : scal[0];
        float gi = va[i] * cnt + scal[1] + beta * xz[i];
        if (!full) gi += psum[i] + psum[kC + i];
        gs[i] = 1.f / gi;
        const int64_t row = r0 + i;
        if (prm.e0 == 0) {
          prm.g[grp * prm.N + row] = gi;
          if (!(fabsf(gi) >= kEpsF32)) flag_degenerate(prm.flag, grp, row);
        }
      }
      if (tid == 0) tma_store_wait_read0();  // the previous chunk's output staging is free
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
    }
    // ------------------------------------------------ MMA group 2: O^T += Y^T P'^T, S^T += Y^T K
    if (tid == 0 && needKY) {
      if (!agg)
        for (int ks = 0; ks < 4; ++ks)
          mma_ss(tmem + Gm::cO, d_feat(aY, ks, prm.ly, kE), kd16(aP, ks, kC), id_Oa, 1);
      for (int ks = 0; ks < 4; ++ks)
        mma_ss(tmem + Gm::cS, d_feat(aY, ks, prm.ly, kE), d_feat(aK, ks, prm.lk, kDK), id_S, 1);
      mma_commit(&bars[3]);
    }
    if (needKY) mbar_wait(&bars[3], m & 1);
    tc_fence_after();
    // ------------------------------------------------ E2: output -> staging -> TMA store
    if (!agg) {
      uint32_t x[32];
      tmem_ld32(tmem + lb + Gm::cO + 32 * half, x);
      tmem_ld_wait();
      const float se = vs[e], spe = vsp[e];
      float o[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = 32 * half + k;
        o[k] = __uint_as_float(x[k]) + va[i] * se + spe;
        if (prm.normalize) o[k] *= gs[i];
      }
      if (prm.lo == LA_FEATURE_MAJOR) {  // [e][64 rows]: this thread's 32 rows = 64 bytes of row e
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 v;
          v.x = pack2<kBF16>(o[8 * c], o[8 * c + 1]);
          v.y = pack2<kBF16>(o[8 * c + 2], o[8 * c + 3]);
          v.z = pack2<kBF16>(o[8 * c + 4], o[8 * c + 5]);
          v.w = pack2<kBF16>(o[8 * c + 6], o[8 * c + 7]);
          *(uint4*)(sO + e * 128 + (((uint32_t)(4 * half + c) ^ (e & 7)) << 4)) = v;
        }
      } else {  // [e panel][64 rows][64 e]
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float ov = o[k];
          *(uint16_t*)(sO + sw128_off(32 * half + k, e, kC)) =
              kBF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(ov)) : __half_as_ushort(__float2half_rn(ov));
        }
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        if (prm.lo == LA_FEATURE_MAJOR) {
          tma_store_3d(&mO, sO, (int)r0, prm.e0, (int)grp);
        } else {
          for (int pnl = 0; pnl < 2; ++pnl) tma_store_3d(&mO, sO + pnl * 8192, prm.e0 + pnl * 64, (int)(grp * prm.N + r0), 0);
        }
        tma_store_commit();
      }
    }
    // ------------------------------------------------ state: b S -> 16-bit copy, vectors
    if (needKY) {
      if (!agg) write_bS(nullptr, true);
      for (int f = tid; f < kDK; f += kThreads) vz[f] += cks[f];
      if (tid < kE) {
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
    if (tid == 0 && m + 2 < nch) load_chunk(m + 2);  // this stage is free again
  }
  if (agg) {  // the unit's record
    float* rec = prm.recs + (grp * prm.U + prm.u0 + p) * Gm::kSZ;
    for (int j0 = 0; j0 < kDK / 2; j0 += 32) {
      const int d0 = half * (kDK / 2) + j0;
      uint32_t x[32];
      tmem_ld32(tmem + lb + Gm::cS + d0, x);
      tmem_ld_wait();
      float4* dst = (float4*)(rec + (int64_t)e * kDK + d0);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        dst[c] = make_float4(__uint_as_float(x[4 * c]), __uint_as_float(x[4 * c + 1]), __uint_as_float(x[4 * c + 2]),
                             __uint_as_float(x[4 * c + 3]));
    }
    for (int f = tid; f < kDK; f += kThreads) rec[kE * kDK + f] = vz[f];
    if (tid < kE) {
      rec[kE * kDK + kDK + tid] = vs[tid];
      rec[kE * kDK + kDK + kE + tid] = vsp[tid];
    }
    if (tid == 0) {
      rec[kE * kDK + kDK + 2 * kE] = scal[0];
      rec[kE * kDK + kDK + 2 * kE + 1] = scal[1];
    }
  }
  if (tid == 0) tma_store_wait0();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Unit records [u0, u1) -> carries, per element (la_f32tc.cu's k_f32_scan, record size SZ).
__global__ void k_g16_scan(float* recs, int64_t SZ, int U, int u0, int u1, int dir) {
  const int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (el >= SZ) return;
  float* r = recs + (int64_t)blockIdx.y * U * SZ + el;
  float run = 0.f;
  if (dir == kFull) {
    for (int q = u0; q < u1; ++q) run += r[q * SZ];
    r[0] = run;
  } else if (dir == kCausal) {
    for (int q = u0; q < u1; ++q) {
      const float t = r[q * SZ];
      r[q * SZ] = run;
      run += t;
    }
    if (u1 < U) r[u1 * SZ] = run;
  } else {
    for (int q = u1 - 1; q >= u0; --q) {
      const float t = r[q * SZ];
      r[q * SZ] = run;
      run += t;
    }
    if (u0 > 0) r[(u0 - 1) * SZ] = run;
  }
}

// 16-bit TMA maps (128B swizzle): SequenceMajor [G*N][D] as {D, G*N, 1}, box {64, 64, 1};
// FeatureMajor [G][D][N] as {N, D, G}, box {64, feats, 1}. Features beyond D read as
// zeros / stores clip.
bool g16_map(CUtensorMap* m, const void* base, bool bf16, int lay, int64_t G, int64_t N, int64_t D, int feats) {
  cuuint64_t dims[3];
  cuuint64_t strides[2];
  cuuint32_t box[3];
  if (lay == LA_SEQUENCE_MAJOR) {
    dims[0] = (cuuint64_t)D; dims[1] = (cuuint64_t)(G * N); dims[2] = 1;
    strides[0] = (cuuint64_t)D * 2; strides[1] = (cuuint64_t)(G * N * D) * 2;
    box[0] = 64; box[1] = kC; box[2] = 1;
  } else {
    dims[0] = (cuuint64_t)N; dims[1] = (cuuint64_t)D; dims[2] = (cuuint64_t)G;
    strides[0] = (cuuint64_t)N * 2; strides[1] = (cuuint64_t)(D * N) * 2;
    box[0] = 64; box[1] = (cuuint32_t)feats; box[2] = 1;
  }
  cuuint32_t es[3] = {1, 1, 1};
  return tma_encode_fn()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                         const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g16_segments(int64_t G, int64_t N) {
  const int64_t nc = N / kC;
  int64_t P = G >= 148 ? 1 : 148 / G;
  if (const int s = tuning().segments) P = s;
  P = std::max<int64_t>(1, std::min<int64_t>(P, nc));
  const int64_t seg = (nc + P - 1) / P;
  return (int)((nc + seg - 1) / seg);
}
int g16_units(int64_t G, int P, int seg, int dir) {
  const int64_t segs = dir == kFull ? P : P - 1;
  if (segs <= 0) return 1;
  int best = 1;
  for (int a = 1; a <= 16; ++a) {
    if (seg % a) continue;
    if (G * segs * a <= 148) best = a;
  }
  return best;
}
size_t g16_unit_slots(int64_t G, int64_t N) {
  const int P = g16_segments(G, N);
  const int seg = (int)((N / kC + P - 1) / P);
  return (size_t)(G * P * std::max(g16_units(G, P, seg, kCausal), g16_units(G, P, seg, kFull)));
}
int dk_of(int64_t D) { return D <= 128 ? 128 : 256; }
int64_t sz_of(int64_t D) { return dk_of(D) == 128 ? G16<128>::kSZ : G16<256>::kSZ; }

struct Operand {
  const void* ptr;
  int lay;
};

template <bool kBF16, int kDK>
cudaError_t g16_pass_t(const Launch& L, Operand X, Operand K, Operand Y, void* out, int lo, int dir, float alpha_c,
                       float alpha_s, const float* alpha_v, float alphk_s, const float* alphk_v, bool normalize,
                       int shift, float* g, unsigned long long* flag, float* recs, const char* name) {
  using Gm = G16<kDK>;
  const int64_t G = L.G, N = L.N, D = L.D;
  const int P = g16_segments(G, N);
  const int64_t nc = N / kC;
  const int seg = (int)((nc + P - 1) / P);
  const int A = g16_units(G, P, seg, dir);
  auto kern = k_g16_sweep<kBF16, kDK>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::kSmem);
  for (int e0 = 0; e0 < D; e0 += kE) {  // output features in halves of 128 (D > 128)
    CUtensorMap mX, mK, mY, mO;
    if (!g16_map(&mX, X.ptr, kBF16, X.lay, G, N, D, kDK) || !g16_map(&mK, K.ptr, kBF16, K.lay, G, N, D, kDK) ||
        !g16_map(&mY, Y.ptr, kBF16, Y.lay, G, N, D, kE) || !g16_map(&mO, out, kBF16, lo, G, N, D, kE))
      return cudaErrorInvalidValue;
    G16Params prm{N, (int)D, e0, (int)D, seg, P, dir, kAgg, X.lay, K.lay, Y.lay, lo, alpha_c, alpha_s, alpha_v,
                  alphk_s, alphk_v, L.b, shift, recs, A, P * A, seg / A, 0, normalize ? 1 : 0, 0, g, flag,
                  L.n_total != L.N ? (float)L.n_total : 0.f};
    if (P > 1 || dir == kFull) {
      const int s0 = dir == kAnti ? 1 : 0, s1 = dir == kCausal ? P - 1 : P;
      prm.u0 = s0 * A;
      {
        ProfScope ps("la_g16_agg", L.stream);
        kern<<<dim3((unsigned)((s1 - s0) * A), (unsigned)G), kThreads, Gm::kSmem, L.stream>>>(mX, mK, mY, mO, prm);
      }
      k_g16_scan<<<dim3((unsigned)((Gm::kSZ + 255) / 256), (unsigned)G), 256, 0, L.stream>>>(
          recs, Gm::kSZ, P * A, s0 * A, s1 * A, dir);
      note_launch(2);
      prm.scanned = 1;
    }
    prm.mode = kSweep;
    {
      ProfScope ps(name, L.stream);
      kern<<<dim3((unsigned)P, (unsigned)G), kThreads, Gm::kSmem, L.stream>>>(mX, mK, mY, mO, prm);
      note_launch(1);
    }
  }
  return cudaGetLastError();
}

cudaError_t g16_pass(const Launch& L, Operand X, Operand K, Operand Y, void* out, int lo, int dir, float alpha_c,
                     float alpha_s, const float* alpha_v, float alphk_s, const float* alphk_v, bool normalize,
                     int shift, float* g, unsigned long long* flag, float* recs, const char* name) {
  const bool bf = L.dtype == LA_BF16;
  if (dk_of(L.D) == 128)
    return bf ? g16_pass_t<true, 128>(L, X, K, Y, out, lo, dir, alpha_c, alpha_s, alpha_v, alphk_s, alphk_v,
                                      normalize, shift, g, flag, recs, name)
              : g16_pass_t<false, 128>(L, X, K, Y, out, lo, dir, alpha_c, alpha_s, alpha_v, alphk_s, alphk_v,
                                       normalize, shift, g, flag, recs, name);
  return bf ? g16_pass_t<true, 256>(L, X, K, Y, out, lo, dir, alpha_c, alpha_s, alpha_v, alphk_s, alphk_v,
                                    normalize, shift, g, flag, recs, name)
            : g16_pass_t<false, 256>(L, X, K, Y, out, lo, dir, alpha_c, alpha_s, alpha_v, alphk_s, alphk_v,
                                     normalize, shift, g, flag, recs, name);
}

__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }

// w_hat = omega / g (FeatureMajor, into `wh`, the element type of the problem) and
// s_i = sum_j o_ij w_hat_ij from the rounded w_hat (make_omega_hat backward.cpp:74-91,
// backward_kernels.hpp:33-38). omega in either layout, o FeatureMajor.
template <typename T>
__global__ void k_g16_what(const T* o, const T* w, int lw, const float* g, T* wh, float* s, int64_t N, int D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (i >= N) return;
  const float gi = g[grp * N + i];
  const Strides sw = strides_of(lw, N, D);
  const T* wg = w + grp * N * D;
  float acc = 0.f;
  for (int j = 0; j < D; ++j) {
    const int64_t ix = (grp * D + j) * N + i;
    const T wv = cvt<T>(ld(wg + i * sw.is + j * sw.js) / gi);
    wh[ix] = wv;
    acc += ld(o + ix) * to_f(wv);
  }
  s[grp * N + i] = acc;
}

// Fault::CausalPrefixOffByOne across chunk boundaries: the kernel's beta window of a
// chunk's last row i stops at the chunk; add b (x_i . k_{i+1}) y_{i+1} / g_i
// (forward_kernels.hpp:86-106, rows i < n - 1). One block per boundary row.
template <typename T>
__global__ void k_offbyone_fix(const T* q, int lq, const T* k, int lk, const T* v, int lv, T* out, const float* g,
                               int64_t N, int D, float b) {
  const int64_t grp = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * kC + kC - 1;
  if (i + 1 >= N) return;
  __shared__ float red[32];
  const Strides sq = strides_of(lq, N, D), sk = strides_of(lk, N, D), sv = strides_of(lv, N, D);
  const T* qg = q + grp * N * D;
  const T* kg = k + grp * N * D;
  const T* vg = v + grp * N * D;
  float part = 0.f;
  for (int m = threadIdx.x; m < D; m += blockDim.x) part += ld(qg + i * sq.is + m * sq.js) * ld(kg + (i + 1) * sk.is + m * sk.js);
  for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  float dot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) dot += red[w];
  const float sc = b * dot / g[grp * N + i];
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    T* slot = out + (grp * D + j) * N + i;
    *slot = cvt<T>(ld(slot) + sc * ld(vg + (i + 1) * sv.is + j * sv.js));
  }
}

}  // namespace

// Fault::CausalPrefixOffByOne chunk-boundary fix-up for the generic paths (all dtypes).
cudaError_t offbyone_fix(const Launch& L, const Tensors& t, void* out, const float* g) {
  const dim3 grid((unsigned)(L.N / kC), (unsigned)L.G);
  if (L.dtype == LA_BF16)
    k_offbyone_fix<__nv_bfloat16><<<grid, 128, 0, L.stream>>>(
        (const __nv_bfloat16*)t.q, t.lq, (const __nv_bfloat16*)t.k, t.lk, (const __nv_bfloat16*)t.v, t.lv,
        (__nv_bfloat16*)out, g, L.N, (int)L.D, L.b);
  else if (L.dtype == LA_F16)
    k_offbyone_fix<__half><<<grid, 128, 0, L.stream>>>((const __half*)t.q, t.lq, (const __half*)t.k, t.lk,
                                                        (const __half*)t.v, t.lv, (__half*)out, g, L.N, (int)L.D,
                                                        L.b);
  else
    k_offbyone_fix<float><<<grid, 128, 0, L.stream>>>((const float*)t.q, t.lq, (const float*)t.k, t.lk,
                                                       (const float*)t.v, t.lv, (float*)out, g, L.N, (int)L.D, L.b);
  note_launch(1);
  return cudaGetLastError();
}

bool g16_supported(const Launch& L, const Tensors& t) {
  (void)t;
  return (L.dtype == LA_BF16 || L.dtype == LA_F16) && L.D % 8 == 0 && L.D <= 256 && L.N % kC == 0 &&
         L.carry_prefix == nullptr && L.carry_suffix == nullptr && L.row_offset == 0 && L.G * L.N < (1ll << 31) &&
         L.G < 65536;
}

size_t g16_ws_floats(int64_t G, int64_t N, int64_t D) {
  if (N % kC) return 0;
  return g16_unit_slots(G, N) * (size_t)sz_of(D) + (size_t)(G * N);
}

cudaError_t g16_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const int dir = L.causal ? kCausal : kFull;
  const int shift = L.causal && L.fault == LA_FAULT_CAUSAL_PREFIX_OFF_BY_ONE ? 1 : 0;
  cudaError_t e = g16_pass(L, {t.q, t.lq}, {t.k, t.lk}, {t.v, t.lv}, out, LA_FEATURE_MAJOR, dir, L.a, 0.f, nullptr,
                           0.f, nullptr, true, shift, g, ws.flag, ws.base,
                           L.causal ? "la_g16_fwd_causal" : "la_g16_fwd_full");
  if (e != cudaSuccess || !shift) return e;
  return offbyone_fix(L, t, out, g);
}

// Backward: w_hat (into the dV buffer) and s, then dQ, dK and dV (dV last, over its own
// w_hat input). Faults: FlipBetaKSign adds the dK beta term, DropGradVConstantTerm
// drops dV's a-weighted term (backward_kernels.hpp:104, 144, 224, 262).
cudaError_t g16_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws) {
  const int64_t G = L.G, N = L.N;
  const int D = (int)L.D;
  float* recs = ws.base;
  float* s = ws.base + g16_unit_slots(G, N) * (size_t)sz_of(D);
  {
    ProfScope ps("la_g16_what", L.stream);
    const dim3 grid((unsigned)((N + 255) / 256), (unsigned)G);
    if (L.dtype == LA_BF16)
      k_g16_what<__nv_bfloat16><<<grid, 256, 0, L.stream>>>((const __nv_bfloat16*)t.o, (const __nv_bfloat16*)t.w,
                                                            t.lw, t.g, (__nv_bfloat16*)dv, s, N, D);
    else
      k_g16_what<__half><<<grid, 256, 0, L.stream>>>((const __half*)t.o, (const __half*)t.w, t.lw, t.g, (__half*)dv,
                                                     s, N, D);
    note_launch(1);
  }
  const int fwd = L.causal ? kCausal : kFull, rev = L.causal ? kAnti : kFull;
  const float b = L.b;
  const float kbeta = L.fault == LA_FAULT_FLIP_BETA_K_SIGN ? b : -b;
  const float va = L.fault == LA_FAULT_DROP_GRAD_V_CONSTANT_TERM ? 0.f : L.a;
  cudaError_t e;
  e = g16_pass(L, {dv, LA_FEATURE_MAJOR}, {t.v, t.lv}, {t.k, t.lk}, dq, LA_SEQUENCE_MAJOR, fwd, 0.f, -b, s, 0.f,
               nullptr, false, 0, nullptr, ws.flag, recs, "la_g16_bwd_dq");
  if (e != cudaSuccess) return e;
  e = g16_pass(L, {t.v, t.lv}, {dv, LA_FEATURE_MAJOR}, {t.q, t.lq}, dk, LA_FEATURE_MAJOR, rev, 0.f, 0.f, nullptr,
               kbeta, s, false, 0, nullptr, ws.flag, recs, "la_g16_bwd_dk");
  if (e != cudaSuccess) return e;
  return g16_pass(L, {t.k, t.lk}, {t.q, t.lq}, {dv, LA_FEATURE_MAJOR}, dv, LA_FEATURE_MAJOR, rev, va, 0.f, nullptr,
                  0.f, nullptr, false, 0, nullptr, ws.flag, recs, "la_g16_bwd_dv");
}

}  // namespace lab
