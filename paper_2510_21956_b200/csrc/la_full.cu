// sm_100a tensor-core non-causal linear attention for head dims D = 64, 192, 256
// (forward_full / backward_full: forward_kernels.hpp:133-206, backward_kernels.hpp:173-288;
// D = 128 keeps the kernels of la_sm100.cu / la_sm100_bwd.cu).
//
// Without the mask the algebra is two kinds of contraction:
//   totals over rows  T = X^T Y      k_full_totals: S = K^T V, z = sum k, sigma = sum v (forward)
//                                                    R = Q^T W_hat, u = Q^T s, c = sum w_hat (backward)
//   apply per row     Out^T = W Y^T  k_full_apply:  O^T  = (b S)^T Q^T,  o = (O^T + a sigma) / g
//                                                    dQ^T = (b S) W_hat^T - b z s^T
//                                                    dK^T = (b R) V^T - b u 1^T
//                                                    dV^T = (b R)^T K^T + a c 1^T
// with w_hat_i = omega_i / g_i, s_i = o_i . w_hat_i and g_i = a N + b q_i . z.
//
// Layout: every accumulator has the output features on the 128 TMEM lanes (M = 128, in
// NH = ceil(D / 128) halves; D = 64 and the second half of D = 192 leave lanes unused) and
// rows on the columns. The constant W (D x D) is built once per CTA from the fp32 totals,
// converted to bf16 / fp16 and stored in TMEM as the MMA's A operand; the row tiles arrive
// by TMA (128B swizzle) and serve as the B operand K-major (Q, K: SequenceMajor) or
// MN-major (V^T, Omega^T: FeatureMajor) without any transpose. Warp roles (192 threads):
// 0 TMA producer, 1 MMA issuer + TMEM owner, 2-5 CUDA-core work (g, W_hat, s, the
// vector sums) and the epilogue (TMEM -> registers -> swizzled staging -> TMA store).
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace lab {

using namespace sm100;

namespace {

template <int D>
struct FG {
  static constexpr int NH = (D + 127) / 128;     // 128-lane halves of the feature dimension
  static constexpr int CR = 64;                  // rows per chunk (MMA N of the apply pass)
  // D = 64 needs few TMEM columns and little shared memory: two CTAs per SM (the passes
  // are latency-bound with one: 4 CUDA-core warps, half of the 128 lanes used).
  // D = 128 (backward only): W takes 64 TMEM columns and the two accumulators 128, so two
  // CTAs fit an SM's 512 columns (dQ pass 0.263 -> 0.192 ms at config 4)
  static constexpr bool k128 = D == 128;
  static constexpr int kCtas = D <= 64 ? 3 : k128 ? 2 : 1;
  // totals CTAs per SM: at D = 64 four (4 x 128 TMEM columns; R pass 0.193 -> 0.173 ms). The
  // apply passes stay at three: at four they spill and lose more than the totals gain.
  static constexpr int kCtasTot = D <= 64 ? 4 : kCtas;
  // D = 128: a 2-stage ring (100 KB) lets two totals CTAs share an SM (R pass 0.324 -> 0.279 ms)
  static constexpr int kTotStages = D <= 64 || D == 128 ? 2 : 0;  // 0: the stage-size rule of k_full_totals
  static constexpr int kAccBufs = D <= 64 ? 1 : 2;           // apply accumulators (D = 64: CTAs overlap)
  static constexpr uint32_t kTmemTot = D <= 64 ? 128 : k128 ? 256 : 512;  // totals: NH x 256-column blocks
  static constexpr uint32_t kTmemApp = D <= 64 ? 128 : k128 ? 256 : 512;  // apply: W + kAccBufs x NH x CR
  static constexpr uint32_t kAccApp = D <= 64 ? 64 : k128 ? 64 : 256;
  static constexpr int KS = D / 16;              // MMA k-steps over the feature dimension
  static constexpr int T = CR * D * 2;           // one [CR][D] or [D][CR] 16-bit tile
  static constexpr int64_t SZ = (D * D + 2 * D + 1 + 3) & ~3;  // state_floats(D)
};

// K-major SW128 tile of `rows` 128-byte rows per 64-element panel: k-step ks.
__device__ __forceinline__ uint64_t kmaj(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * rows * 128 + (ks & 3) * 32) >> 4);
}
// MN-major SW128 tile (K rows of 128 B, 64-element MN panels `panel` bytes apart): k-step ks.
__device__ __forceinline__ uint64_t mnmaj(uint32_t tile, int ks, uint32_t panel) {
  return sdesc_sw128(tile, panel, 1024) + (uint64_t)((ks * 2048) >> 4);
}

// Column sums of a [CR][D] K-major tile (optionally weighted per row): thread (mg, tg) =
// (et >> 3, et & 7) sums rows tg + 8 k of the 8 columns of group cg = mg + 16 q with 16-byte
// loads (a quarter-warp reads 8 rows of one 16-byte column chunk: distinct swizzle chunks),
// then a reduce-scatter over the 8 tg lanes leaves column 8 cg + tg in lane tg.
template <int D, bool kBF16, bool kW>
__device__ __forceinline__ void col_sums(const uint8_t* xt, const float* w, float (&ucol)[(D + 127) / 128], int et) {
  constexpr int CR = FG<D>::CR;
  const int mg = et >> 3, tg = et & 7;
#pragma unroll
  for (int q = 0; q < (D + 127) / 128; ++q) {
    const int cg = mg + 16 * q;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (cg < D / 8) {
#pragma unroll
      for (int k = 0; k < CR / 8; ++k) {
        const int i = tg + 8 * k;
        const uint4 v4 = *(const uint4*)(xt + sw128_off(i, 8 * cg, CR));
        const float wi = kW ? w[i] : 1.f;
        const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float2 f2 = unpack2<kBF16>(vv[h]);
          acc[2 * h] += wi * f2.x;
          acc[2 * h + 1] += wi * f2.y;
        }
      }
    }
    const float tot = reduce_scatter8(acc, tg);  // whole warp: the shuffles need every lane
    if (cg < D / 8) ucol[q] += tot;
  }
}

// ================================================================ totals over row units
struct TotParams {
  const float* g;   // [G][N] (QW)
  float* s_out;     // [G][N] s_i (QW), consumed by the dQ apply
  float* recs;      // [G][U] records
  int64_t N, unit_rows;
  int U;
};

// kQW = false: X = K [rows][D] (SequenceMajor), Y^T = V^T [D][rows]: S[m][j], z, sigma.
// kQW = true:  X = Q, Y^T = W_hat^T = Omega^T / g (scaled in place), third tile O^T:
//              R[m][j], u = sum s_i q_i, c = sum w_hat; s_i = o_i . w_hat_i -> s_out.
template <int D, bool kBF16, bool kQW>
__global__ void __launch_bounds__(192, FG<D>::kCtasTot)
    k_full_totals(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                  const __grid_constant__ CUtensorMap tmO, TotParams prm) {
  using F = FG<D>;
  constexpr int CR = F::CR, T = F::T, NT = kQW ? 3 : 2;
  constexpr int STAGE = (NT * T + CR * 4 + 1023) & ~1023;  // tiles + g of the chunk (QW), 1 KB aligned
  constexpr int NS = F::kTotStages ? F::kTotStages : (STAGE <= 56 * 1024) ? 3 : 2;
  constexpr int RPT = (D + 127) / 128;  // feature rows per CUDA-core thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  float* sv = (float*)(smem + NS * STAGE);          // [CR] s of the chunk
  uint64_t* bars = (uint64_t*)(sv + 6 * CR);
  uint64_t* full = bars;            // [NS]
  uint64_t* empty = bars + 4;       // [NS]
  uint64_t* wready = bars + 8;      // [NS] (QW: W_hat^T written)
  uint64_t* done = bars + 12;
  uint32_t* tslot = (uint32_t*)(bars + 14);

  const int u = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t r0 = (int64_t)u * prm.unit_rows;
  const int64_t r1 = lmin(prm.N, r0 + prm.unit_rows);
  const int nc = r1 > r0 ? (int)((r1 - r0) / CR) : 0;
  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmY);
    if (kQW) tma_prefetch(&tmO);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 128);
      mbar_init(&wready[s], 128);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<F::kTmemTot>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c % NS;
        const int64_t row0 = r0 + (int64_t)c * CR;
        if (!kQW || D <= 64) {  // into L2 before the slot wait (measured: helps the K/V pass at
                                // every D, the Q/W/O pass only at D = 64)
          tma_prefetch_l2_3d(&tmX, 0, (int)(grp * prm.N + row0), 0);
          tma_prefetch_l2_3d(&tmY, 0, (int)(grp * D), (int)(row0 / 64));
          if (kQW) tma_prefetch_l2_3d(&tmO, 0, (int)(grp * D), (int)(row0 / 64));
        }
        if (c >= NS) mbar_wait(&empty[s], ((c / NS) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE;
        mbar_expect_tx(&full[s], NT * T + (kQW ? CR * 4 : 0));
        tma_load_3d(st, &tmX, &full[s], 0, (int)(grp * prm.N + row0), 0);
        tma_load_3d(st + T, &tmY, &full[s], 0, (int)(grp * D), (int)(row0 / 64));
        if (kQW) {
          tma_load_3d(st + 2 * T, &tmO, &full[s], 0, (int)(grp * D), (int)(row0 / 64));
          bulk_load(st + NT * T, prm.g + grp * prm.N + row0, CR * 4, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // T[m][j] (+)= sum_rows X[i][m] Y[i][j]: A = X^T (MN-major over m), B = Y (K-major: the
    // Y^T tile's rows are j with the rows i contiguous); one M = 128 accumulator per half of m
    constexpr uint32_t fmt = kBF16 ? 1 : 0;
    const uint32_t id_T = idesc_f16(128, D, fmt, 1, 0);
    for (int c = 0; c < nc; ++c) {
      const int s = c % NS;
      const uint32_t aX = smem_u32(smem + s * STAGE), aY = aX + T;
      mbar_wait(&full[s], (c / NS) & 1);
      if (kQW) mbar_wait(&wready[s], (c / NS) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int h = 0; h < F::NH; ++h)
          for (int ks = 0; ks < CR / 16; ++ks)
            mma_ss(tmem + h * 256, mnmaj(aX + h * 2 * CR * 128, ks, CR * 128), kmaj(aY, ks, D), id_T,
                   (c > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (c == nc - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ CUDA cores (128 threads)
    // Y^T tile [D rows j][CR = 64 columns i]: thread (jg, ig) = (et & 15, et >> 4) owns the
    // 16-byte column chunk ig (columns 8 ig .. 8 ig + 7) of rows j = jg + 16 rr (every lane
    // busy for any D; a quarter-warp reads 8 consecutive rows: distinct swizzle chunks).
    // Row sums (sigma / c) stay per thread until the unit ends; column sums of X (z / u)
    // go through col_sums.
    static_assert(CR == 64, "the (jg, ig) tiling covers 64 columns");
    constexpr int RR = D / 16;
    const int et = (int)threadIdx.x - 64;
    const uint32_t qd = warp & 3;
    const int r = (int)(qd * 32 + lane_id());  // TMEM lane of this thread's warp quadrant
    const int jg = et & 15, ig = et >> 4;
    float crow[RR];  // sigma_j or c_j partials of this thread's 8 columns, rows jg + 16 rr
#pragma unroll
    for (int q = 0; q < RR; ++q) crow[q] = 0.f;
    float ucol[(D + 127) / 128] = {};  // z or u: column sums in col_sums' (mg, tg) layout
    for (int c = 0; c < nc; ++c) {
      const int s = c % NS;
      uint8_t* st = smem + s * STAGE;
      mbar_wait(&full[s], (c / NS) & 1);
      const uint8_t* xt = st;  // [CR][D] K-major panels of CR rows
      uint8_t* yt = st + T;    // [D][CR] panels of D rows (64 row-elements each)
      if (kQW) {
        // W_hat^T = Omega^T / g in place; c_j += w_hat; s_i = sum_j o_ij w_hat_ij
        const float* gg = (const float*)(st + NT * T);
        const float4 g0 = *(const float4*)(gg + 8 * ig), g1 = *(const float4*)(gg + 8 * ig + 4);
        const float gi[8] = {__frcp_rn(g0.x), __frcp_rn(g0.y), __frcp_rn(g0.z), __frcp_rn(g0.w),
                             __frcp_rn(g1.x), __frcp_rn(g1.y), __frcp_rn(g1.z), __frcp_rn(g1.w)};
        const uint8_t* ot = st + 2 * T;
        float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const uint32_t off = sw128_off(jg + 16 * rr, 8 * ig, D);
          uint4 w4 = *(const uint4*)(yt + off);
          const uint4 o4 = *(const uint4*)(ot + off);
          uint32_t* wp = (uint32_t*)&w4;
          const uint32_t* op = (const uint32_t*)&o4;
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2) {
            const float2 w2 = unpack2<kBF16>(wp[h2]), o2 = unpack2<kBF16>(op[h2]);
            const float w0 = w2.x * gi[2 * h2], w1 = w2.y * gi[2 * h2 + 1];
            crow[rr] += w0 + w1;
            sp[2 * h2] += o2.x * w0;
            sp[2 * h2 + 1] += o2.y * w1;
            wp[h2] = pack2<kBF16>(w0, w1);
          }
          *(uint4*)(yt + off) = w4;
        }
        // s_i: sum over the 16 jg lanes of each column chunk
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) sp[k] += __shfl_xor_sync(0xffffffffu, sp[k], o);
        if (jg == 0) {
          *(float4*)(sv + 8 * ig) = make_float4(sp[0], sp[1], sp[2], sp[3]);
          *(float4*)(sv + 8 * ig + 4) = make_float4(sp[4], sp[5], sp[6], sp[7]);
        }
        fence_proxy_async();
        mbar_arrive(&wready[s]);
        named_bar(1, 128);  // s of the chunk complete
        if (et < CR) prm.s_out[grp * prm.N + r0 + (int64_t)c * CR + et] = sv[et];
        col_sums<D, kBF16, true>(xt, sv, ucol, et);  // u_m += sum_i s_i q_im
        named_bar(1, 128);  // sv is rewritten by the next chunk
      } else {
        col_sums<D, kBF16, false>(xt, nullptr, ucol, et);  // z_m: column sums of K
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {  // sigma_j: rows of V^T
          const uint4 v4 = *(const uint4*)(yt + sw128_off(jg + 16 * rr, 8 * ig, D));
          const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2) {
            const float2 v2 = unpack2<kBF16>(vv[h2]);
            crow[rr] += v2.x + v2.y;
          }
        }
      }
      // The stage is refilled by TMA (async proxy) once this arrival completes the phase, and
      // the arrive does not wait for this thread's outstanding shared loads: at D = 64 the last
      // 16 rows of V^T were still being read when the next chunk landed (sigma_48..63 differed
      // run to run, scratch/det_probe_c4.py). The proxy fence retires the generic reads first.
      fence_proxy_async();
      mbar_arrive(&empty[s]);
    }
    // row sums: the 8 ig partials of each row j -> vrow (shared scratch: the stages are idle
    // once the unit's MMAs have retired)
    if (nc > 0) mbar_wait(done, 0);
    named_bar(1, 128);  // every CUDA-core thread is done reading the stages
    float* red = (float*)smem;  // [8 ig][D]
#pragma unroll
    for (int rr = 0; rr < RR; ++rr) red[ig * D + jg + 16 * rr] = crow[rr];
    named_bar(1, 128);
    // ---- the unit's record: X[m][j] (lanes m), vA (z | u), vB (sigma | c), rows
    float* rec = prm.recs + (grp * prm.U + u) * F::SZ;
    if (nc > 0) {
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < F::NH; ++h) {
        const int m = 128 * h + r;
#pragma unroll 1
        for (int j0 = 0; j0 < D; j0 += 32) {
          uint32_t x[32];
          tmem_ld32(tmem + ((qd * 32u) << 16) + h * 256 + j0, x);
          tmem_ld_wait();
          if (m < D) {
#pragma unroll
            for (int k = 0; k < 32; k += 4)
              *(float4*)(rec + (int64_t)m * D + j0 + k) =
                  make_float4(__uint_as_float(x[k]), __uint_as_float(x[k + 1]), __uint_as_float(x[k + 2]),
                              __uint_as_float(x[k + 3]));
          }
        }
      }
    } else {
      for (int e = et; e < D * D; e += 128) rec[e] = 0.f;
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int f = et + 128 * q;
      if (f < D) {  // sigma | c: the 8 column-chunk partials of row f
        float v = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) v += red[k * D + f];
        rec[D * D + D + f] = v;
      }
      const int cg = (et >> 3) + 16 * q;  // z / u: col_sums' layout
      if (cg < D / 8) rec[D * D + 8 * cg + (et & 7)] = ucol[q];
    }
    if (et == 0) rec[D * D + 2 * D] = (float)(r1 > r0 ? r1 - r0 : 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<F::kTmemTot>(tmem);
}

// Per-group totals: tot[g] = sum_u recs[g][u] (elements D*D + 2D + 1; padding zero).
__global__ void k_full_sum(const float* recs, int U, int64_t SZ, int64_t used, float* tot) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (e >= SZ) return;
  float acc = 0.f;
  if (e < used)
    for (int u = 0; u < U; ++u) acc += recs[(grp * U + u) * SZ + e];
  tot[grp * SZ + e] = acc;
}

// ================================================================ apply passes
enum ApplyMode { kFwd = 0, kDQ = 1, kDK = 2, kDV = 3 };

struct ApplyParams {
  const float* tot;     // per-group fp32 totals record: S (kFwd, kDQ) or R (kDK, kDV)
  const float* totS;    // kDQ: z comes from the S record (same as tot); kFwd: S record
  const float* g;       // [G][N]: kDQ (w_hat = omega / g)
  const float* s;       // [G][N]: kDQ
  float* gout;          // kFwd: g_i
  unsigned long long* flag;
  int64_t N, n_total, seg_len;
  float a, b;
};

// Out^T = W Y^T per chunk of CR rows, W = the constant D x D operand in TMEM:
//   kFwd: W[j][m] = b S[m][j],  Y = Q  (K-major),          o^T = (acc + a sigma_j) / g_i
//   kDQ:  W[m][j] = b S[m][j],  Y^T = Omega^T / g (MN-major), dQ = acc - b z_m s_i (transposed store)
//   kDK:  W[m][j] = b R[m][j],  Y^T = V^T (MN-major),       dK^T = acc - b u_m
//   kDV:  W[j][m] = b R[m][j],  Y = K (K-major),            dV^T = acc + a c_j
template <int D>
constexpr int apply_wgs(int mode) { return mode == 1 ? FG<D>::NH : 1; }  // kDQ: a warpgroup per half
// D = 64: chunks are applied in pairs, with W block-diagonal in TMEM ([W 0; 0 W], K = 128) so
// that one M = 128 MMA writes chunk c to lanes 0..63 and chunk c + 1 to lanes 64..127 and
// every epilogue lane has a row to drain (a single chunk would leave lanes 64..127 empty).
#ifndef LA_D64_PAIR
#define LA_D64_PAIR 1
#endif
// Measured: the passes with a CUDA-core pre-pass (kFwd 0.119 -> 0.099 ms, kDQ 0.204 -> 0.159 ms
// at config 4) gain; dK^T (0.102 -> 0.110) does not, so kDK / kDV stay one chunk per MMA.
template <int D>
constexpr bool apply_pairs(int mode) { return LA_D64_PAIR && D == 64 && (mode == 0 || mode == 1); }
template <int D>
constexpr int apply_stages(int mode) { return apply_pairs<D>(mode) ? 4 : 3; }
template <int D>
constexpr int apply_slots(int mode) { return apply_pairs<D>(mode) ? 4 : 2; }  // staging tiles; 1/g, s slots

template <int D, bool kBF16, int kMode>
__global__ void __launch_bounds__(64 + 128 * apply_wgs<D>(kMode), FG<D>::kCtas)
    k_full_apply(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmOut,
                 ApplyParams prm) {
  using F = FG<D>;
  constexpr int CR = F::CR, T = F::T, NH = F::NH;
  constexpr bool kSeqIn = kMode == kFwd || kMode == kDV;  // Y tile [CR][D] (else [D][CR])
  constexpr bool kPre = kMode == kFwd || kMode == kDQ;    // CUDA-core pass over the tile first
  constexpr int STAGE = (T + (kMode == kDQ ? 2 * CR * 4 : 0) + 1023) & ~1023;  // + g, s of the chunk
  constexpr bool kPair = apply_pairs<D>(kMode);
  constexpr int NS = apply_stages<D>(kMode), kSl = apply_slots<D>(kMode);
  constexpr int RPT = (D + 127) / 128;
  constexpr int kWG = apply_wgs<D>(kMode), kCT = 128 * kWG;  // compute warpgroups (kDQ: one per half)
  constexpr uint32_t kAcc = F::kAccApp;  // accumulators: 2 buffers x NH halves x CR columns after W
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* stg = smem + NS * STAGE;              // [kSl][T] output staging
  float* zf = (float*)(stg + kSl * T);           // [D] z (kFwd)
  float* ginv = zf + D;                          // [kSl][CR] 1 / g_i (kFwd, kDQ)
  float* sbuf = ginv + kSl * CR;                 // [kSl][CR] s_i (kDQ)
  float* part = sbuf + kSl * CR;                 // [4][CR] (kFwd: partial q.z)
  uint64_t* bars = (uint64_t*)(part + 4 * CR);
  uint64_t* full = bars;        // [NS]
  uint64_t* empty = bars + 4;   // [NS]
  uint64_t* pre = bars + 8;     // [NS] CUDA-core pass done (kDQ: W_hat^T ready)
  uint64_t* acc_full = bars + 12;   // [2]
  uint64_t* acc_empty = bars + 14;  // [2]
  uint32_t* tslot = (uint32_t*)(bars + 16);

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * prm.seg_len;
  const int64_t s1 = lmin(prm.N, s0 + prm.seg_len);
  const int nc = s1 > s0 ? (int)((s1 - s0) / CR) : 0;
  const uint32_t warp = warp_id();
  const float* tot = prm.tot + grp * F::SZ;
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmY);
    tma_prefetch(&tmOut);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + (kPre ? kCT : 0));
      mbar_init(&pre[s], kCT);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kCT);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<F::kTmemApp>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int et = (int)threadIdx.x - 64;
  const int wg = kWG > 1 ? (et >> 7) : 0;  // compute warpgroup: feature half h = wg (+ kWG ...)
  const uint32_t qd = warp & 3;
  const int r = (int)(qd * 32 + lane_id());
  const uint32_t lb = (qd * 32u) << 16;
  if (warp >= 2) {
    // W (bf16 / fp16) into TMEM columns [h * D / 2, (h + 1) * D / 2): lane = output feature
    // f = 128 h + r, column c = input features (2c, 2c + 1)
    constexpr bool kTrans = kMode == kFwd || kMode == kDV;  // W[f][k] = b X[k][f]
    const float b = prm.b;
#pragma unroll 1
    for (int h = wg; h < NH; h += kWG) {
      const int f = kPair ? (r & 63) : 128 * h + r;
#pragma unroll 1
      for (int k0 = 0; k0 < D; k0 += 64) {
        uint32_t pk[32];
        if (kTrans) {  // W[f][k] = b X[k][f]: lanes f read consecutive addresses
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            float w0 = 0.f, w1 = 0.f;
            if (f < D) {
              const int k = k0 + 2 * c;
              w0 = b * tot[(int64_t)k * D + f];
              w1 = b * tot[(int64_t)(k + 1) * D + f];
            }
            pk[c] = pack2<kBF16>(w0, w1);
          }
        } else {  // W[f][k] = b X[f][k]: row f of the record, 16-byte loads (the scalar ones
                  // were 14 % of the D = 256 dQ pass)
#pragma unroll
          for (int c4 = 0; c4 < 16; ++c4) {
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (f < D) w = *(const float4*)(tot + (int64_t)f * D + k0 + 4 * c4);
            pk[2 * c4] = pack2<kBF16>(b * w.x, b * w.y);
            pk[2 * c4 + 1] = pack2<kBF16>(b * w.z, b * w.w);
          }
        }
        if (kPair) {  // block-diagonal: lanes 0..63 take K 0..63, lanes 64..127 take K 64..127
          uint32_t zr[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) zr[c] = 0u;
          tmem_st32(tmem + lb, r < 64 ? pk : zr);
          tmem_st32(tmem + lb + 32, r < 64 ? zr : pk);
        } else {
          tmem_st32(tmem + lb + h * (D / 2) + k0 / 2, pk);
        }
      }
    }
    tmem_st_wait();
    if (kMode == kFwd)
      for (int m = et; m < D; m += kCT) zf[m] = tot[D * D + m];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (elect_one()) {
      for (int c = 0; c < nc; ++c) {
        const int s = c % NS;
        const int64_t row0 = s0 + (int64_t)c * CR;
        if (c >= NS) mbar_wait(&empty[s], ((c / NS) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE;
        mbar_expect_tx(&full[s], T + (kMode == kDQ ? 2 * CR * 4 : 0));
        if (kSeqIn)
          tma_load_3d(st, &tmY, &full[s], 0, (int)(grp * prm.N + row0), 0);
        else
          tma_load_3d(st, &tmY, &full[s], 0, (int)(grp * D), (int)(row0 / 64));
        if (kMode == kDQ) {
          bulk_load(st + T, prm.g + grp * prm.N + row0, CR * 4, &full[s]);
          bulk_load(st + T + CR * 4, prm.s + grp * prm.N + row0, CR * 4, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t fmt = kBF16 ? 1 : 0;
    const uint32_t id = idesc_f16(128, CR, fmt, 0, kSeqIn ? 0 : 1);
    if (kPair) {
      for (int c = 0; c < nc; c += 2) {  // chunks c, c1 (c1 = c for an odd last chunk)
        const int c1 = c + 1 < nc ? c + 1 : c, sa = c % NS, sb = c1 % NS;
        const uint32_t aY0 = smem_u32(smem + sa * STAGE), aY1 = smem_u32(smem + sb * STAGE);
        mbar_wait(&full[sa], (c / NS) & 1);
        if (kMode == kDQ) mbar_wait(&pre[sa], (c / NS) & 1);
        mbar_wait(&full[sb], (c1 / NS) & 1);
        if (kMode == kDQ) mbar_wait(&pre[sb], (c1 / NS) & 1);
        if (c >= 2) mbar_wait(&acc_empty[0], ((c / 2) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < 2 * F::KS; ++ks) {
            const uint32_t aY = ks < F::KS ? aY0 : aY1;
            const int kk = ks % F::KS;
            mma_ts(tmem + kAcc, tmem + ks * 8, kSeqIn ? kmaj(aY, kk, CR) : mnmaj(aY, kk, D * 128), id, ks > 0);
          }
          mma_commit(&acc_full[0]);
          mma_commit(&empty[sa]);
          if (c1 != c) mma_commit(&empty[sb]);
        }
        __syncwarp();
      }
    } else
    for (int c = 0; c < nc; ++c) {
      const int s = c % NS, bb = c % F::kAccBufs;
      const uint32_t aY = smem_u32(smem + s * STAGE);
      mbar_wait(&full[s], (c / NS) & 1);
      if (kMode == kDQ) mbar_wait(&pre[s], (c / NS) & 1);
      if (c >= F::kAccBufs) mbar_wait(&acc_empty[bb], ((c / F::kAccBufs) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int h = 0; h < NH; ++h)
          for (int ks = 0; ks < F::KS; ++ks)
            mma_ts(tmem + kAcc + (bb * NH + h) * CR, tmem + h * (D / 2) + ks * 8,
                   kSeqIn ? kmaj(aY, ks, CR) : mnmaj(aY, ks, D * 128), id, ks > 0);
        mma_commit(&acc_full[bb]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ CUDA cores + epilogue
    const float a = prm.a, b = prm.b;
    float bias[RPT];  // per output feature of this thread's lanes: a sigma_j, -b u_m, a c_j, b z_m
#pragma unroll
    for (int h = 0; h < RPT; ++h) {
      const int f = kPair ? (r & 63) : 128 * h + r;
      float x = 0.f;
      if (f < D) {
        if (kMode == kFwd) x = a * tot[D * D + D + f];
        if (kMode == kDK) x = -b * tot[D * D + f];
        if (kMode == kDV) x = a * tot[D * D + D + f];
        if (kMode == kDQ) x = b * tot[D * D + f];
      }
      bias[h] = x;
    }
    // pass over chunk c's tile before its MMA / epilogue
    auto pre_pass = [&](int c) {
      const int s = c % NS;
      uint8_t* st = smem + s * STAGE;
      mbar_wait(&full[s], (c / NS) & 1);
      const int64_t row0 = s0 + (int64_t)c * CR;
      if (kMode == kFwd) {  // g_i = a N + b q_i . z; kCT / CR threads per row
        constexpr int TPR = kCT / CR;
        const int i = et / TPR, part_k = et % TPR;
        float acc = 0.f;
#pragma unroll
        for (int m8 = part_k * (D / TPR); m8 < (part_k + 1) * (D / TPR); m8 += 8) {
          const uint4 q4 = *(const uint4*)(st + sw128_off(i, m8, CR));
          const float4 za = *(const float4*)(zf + m8), zb = *(const float4*)(zf + m8 + 4);
          const float z8[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
          const uint32_t* qp = (const uint32_t*)&q4;
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2) {
            const float2 q2 = unpack2<kBF16>(qp[h2]);
            acc += q2.x * z8[2 * h2] + q2.y * z8[2 * h2 + 1];
          }
        }
#pragma unroll
        for (int o = 1; o < TPR; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (part_k == 0) {
          const float gi = a * (float)prm.n_total + b * acc;
          if (fabsf(gi) < kEpsF32) flag_degenerate(prm.flag, grp, row0 + i);
          ginv[(c % kSl) * CR + i] = __frcp_rn(gi);
          prm.gout[grp * prm.N + row0 + i] = gi;
        }
        fence_proxy_async();     // the Q tile reads retire before the refill (see k_full_totals)
        mbar_arrive(&empty[s]);  // Q tile no longer read by the CUDA cores
      } else {  // kDQ: W_hat^T = Omega^T / g in place; keep 1/g, s for the epilogue
        const float* gg = (const float*)(st + T);
        const float* ss = gg + CR;
        if (et < CR) {
          ginv[(c % kSl) * CR + et] = __frcp_rn(gg[et]);
          sbuf[(c % kSl) * CR + et] = ss[et];
        }
        named_bar(1, kCT);
        // (jg, ig) tiling: rows j = jg + 16 rr (rr = wg mod kWG), the 16-byte column chunk ig
        const float* gi = ginv + (c % kSl) * CR;
        const int e = et & 127, jg = e & 15, ig = e >> 4;
        const float4 ga = *(const float4*)(gi + 8 * ig), gb = *(const float4*)(gi + 8 * ig + 4);
        const float g8[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
#pragma unroll
        for (int rr = wg; rr < D / 16; rr += kWG) {
          const uint32_t off = sw128_off(jg + 16 * rr, 8 * ig, D);
          uint4 w4 = *(const uint4*)(st + off);
          uint32_t* wp = (uint32_t*)&w4;
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2) {
            const float2 w2 = unpack2<kBF16>(wp[h2]);
            wp[h2] = pack2<kBF16>(w2.x * g8[2 * h2], w2.y * g8[2 * h2 + 1]);
          }
          *(uint4*)(st + off) = w4;
        }
        fence_proxy_async();
        mbar_arrive(&pre[s]);
        mbar_arrive(&empty[s]);
      }
    };
    // kPair: c is the first chunk of a pair; lanes 64..127 hold chunk c + 1
    auto epilogue = [&](int c) {
      const int bb = kPair ? 0 : c % F::kAccBufs;
      const int gi2 = kPair ? c / 2 : c;  // MMA group
      const int cc = kPair ? c + (r >> 6) : c;  // this lane's chunk
      const int sb = cc % kSl;  // 1/g, s slot of the chunk
      const int tb = kPair ? (gi2 & 1) * 2 + (r >> 6) : (c & 1);  // staging tile
      const int64_t row0 = s0 + (int64_t)c * CR;
      mbar_wait(&acc_full[bb], (gi2 / F::kAccBufs) & 1);
      tc_fence_after();
      if (et == 0) tma_store_wait_read1();  // the store group that used these staging tiles
      named_bar(1, kCT);
      uint8_t* so = stg + tb * T;
#pragma unroll 1
      for (int h = wg; h < NH; h += kWG) {
        const int f = kPair ? (r & 63) : 128 * h + r;
        const float bh = h == 0 ? bias[0] : bias[RPT - 1];
#pragma unroll 1
        for (int c0 = 0; c0 < CR; c0 += 32) {
          uint32_t x[32];
          tmem_ld32(tmem + lb + kAcc + (bb * NH + h) * CR + c0, x);
          tmem_ld_wait();
          if (f < D && cc < nc) {
            if (kMode == kDQ) {  // dQ[i][f]: SequenceMajor staging [CR][D]; lanes f, f ^ 1 trade
              float sv[32];  // s_i of the 32 rows, 16-byte shared loads (not 32 scalar ones)
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 s4 = *(const float4*)(sbuf + sb * CR + c0 + 4 * q);
                sv[4 * q] = s4.x; sv[4 * q + 1] = s4.y; sv[4 * q + 2] = s4.z; sv[4 * q + 3] = s4.w;
              }
              // even lanes store (f, f+1) of row i, odd lanes (f-1, f) of row i + 4: rows whose
              // indices differ in bit 2 take disjoint 16-byte chunk sets under the 128-byte
              // swizzle, so the warp's 32 stores hit 32 distinct banks (rows i, i + 1 collide)
              const bool odd = (lane_id() & 1) != 0;
#pragma unroll
              for (int kk = 0; kk < 16; ++kk) {
                const int k = (kk & 3) + ((kk >> 2) << 3);  // 0..3, 8..11, 16..19, 24..27
                const float v0 = __uint_as_float(x[k]) - bh * sv[k], v1 = __uint_as_float(x[k + 4]) - bh * sv[k + 4];
                const float got = __shfl_xor_sync(0xffffffffu, odd ? v0 : v1, 1);
                const uint32_t w2 = odd ? pack2<kBF16>(got, v1) : pack2<kBF16>(v0, got);
                *(uint32_t*)(so + sw128_off(c0 + k + (odd ? 4 : 0), f & ~1, CR)) = w2;
              }
            } else {  // FeatureMajor staging [D][CR]: row f
              const float* gv = ginv + sb * CR + c0;
#pragma unroll
              for (int k8 = 0; k8 < 32; k8 += 8) {
                uint32_t pk[4];
                float g8[8];
                if (kMode == kFwd) {
                  const float4 ga = *(const float4*)(gv + k8), gb = *(const float4*)(gv + k8 + 4);
                  g8[0] = ga.x; g8[1] = ga.y; g8[2] = ga.z; g8[3] = ga.w;
                  g8[4] = gb.x; g8[5] = gb.y; g8[6] = gb.z; g8[7] = gb.w;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float v0 = __uint_as_float(x[k8 + 2 * q]) + bh;
                  float v1 = __uint_as_float(x[k8 + 2 * q + 1]) + bh;
                  if (kMode == kFwd) {
                    v0 *= g8[2 * q];
                    v1 *= g8[2 * q + 1];
                  }
                  pk[q] = pack2<kBF16>(v0, v1);
                }
                *(uint4*)(so + sw128_off(f, c0 + k8, D)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[bb]);
      fence_proxy_async();
      named_bar(1, kCT);
      if (et == 0) {
#pragma unroll 1
        for (int k = 0; k < (kPair ? 2 : 1) && c + k < nc; ++k) {
          const uint8_t* sk = kPair ? stg + ((gi2 & 1) * 2 + k) * T : so;
          if (kMode == kDQ)
            tma_store_3d(&tmOut, sk, 0, (int)(grp * prm.N + row0 + k * CR), 0);
          else
            tma_store_3d(&tmOut, sk, 0, (int)(grp * D), (int)((row0 + k * CR) / 64));
        }
        tma_store_commit();
      }
    };
    if (kPair) {
      for (int c = 0; c < nc; c += 2) {
        if (kPre) {
          pre_pass(c);
          if (c + 1 < nc) pre_pass(c + 1);
        }
        if (c >= 2) epilogue(c - 2);
      }
      if (nc > 0) epilogue((nc - 1) & ~1);
    } else {
      for (int c = 0; c <= nc; ++c) {
        if (kPre && c < nc) pre_pass(c);
        if (c >= 1) epilogue(c - 1);
      }
    }
    if (et == 0) tma_store_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<F::kTmemApp>(tmem);
}

template <int D>
constexpr size_t totals_smem(bool qw) {
  using F = FG<D>;
  const int stage = ((qw ? 3 : 2) * F::T + F::CR * 4 + 1023) & ~1023;
  const int ns = F::kTotStages ? F::kTotStages : stage <= 56 * 1024 ? 3 : 2;  // as k_full_totals
  return (size_t)ns * stage + 6 * F::CR * 4 + 16 * 8 + 1024;
}
template <int D>
constexpr size_t apply_smem(int mode) {
  using F = FG<D>;
  const int stage = (F::T + (mode == kDQ ? 2 * F::CR * 4 : 0) + 1023) & ~1023;
  const int sl = apply_slots<D>(mode);
  return (size_t)apply_stages<D>(mode) * stage + sl * F::T + (D + (2 * sl + 4) * F::CR) * 4 + 17 * 8 + 1024;
}

// CTAs of a kernel resident per SM: its __launch_bounds__ minimum and the 228 KB of shared
// memory (1 KB of it reserved per CTA).
constexpr int ctas_per_sm(int launch_min, size_t smem) {
  const int by_smem = (int)(233472 / (smem + 1024));
  return by_smem < launch_min ? (by_smem < 1 ? 1 : by_smem) : launch_min;
}
// Pieces per group for G groups of `chunks` chunks over `slots` resident CTAs: minimises
// waves x (chunks per piece + 2), the 2 standing for a CTA's fixed cost (prologue, ring
// fill, records). A grid of 1.3 waves (576 CTAs on 444 slots) costs as much as 2 full ones.
inline int64_t pieces(int64_t G, int64_t chunks, int64_t slots, int64_t cap) {
  int64_t best = 1, best_cost = INT64_MAX;
  for (int64_t u = 1; u <= std::min(chunks, cap); ++u) {
    const int64_t waves = (G * u + slots - 1) / slots, per = (chunks + u - 1) / u;
    const int64_t cost = waves * (per + 2);
    if (cost < best_cost) best = u, best_cost = cost;
  }
  return best;
}

// geometry of the totals units and the apply segments
template <int D>
struct Plan {
  int U;
  int64_t unit_rows;
  int P;
  int64_t seg_rows;
  Plan(int64_t G, int64_t N) {
    using F = FG<D>;
    const int64_t CR = F::CR, chunks = std::max<int64_t>(1, N / CR);  // sizing queries: any N
    const int tot_ctas =
        std::min(ctas_per_sm(F::kCtasTot, totals_smem<D>(false)), ctas_per_sm(F::kCtasTot, totals_smem<D>(true)));
    const int app_ctas = std::min(ctas_per_sm(F::kCtas, apply_smem<D>(kFwd)), ctas_per_sm(F::kCtas, apply_smem<D>(kDQ)));
    const int64_t u = pieces(G, chunks, 148 * tot_ctas, 64);
    unit_rows = ((chunks + u - 1) / u) * CR;
    U = (int)((N + unit_rows - 1) / unit_rows);
    int64_t p2 = pieces(G, chunks, 148 * app_ctas, 64);
    if (tuning().full_ctas_fwd > 0) p2 = std::min<int64_t>(chunks, tuning().full_ctas_fwd);
    seg_rows = ((chunks + p2 - 1) / p2) * CR;
    P = (int)((N + seg_rows - 1) / seg_rows);
  }
};

bool maps_seq(CUtensorMap* m, const void* base, bool bf, int64_t G, int64_t N, int D, int CR) {
  return make_tma_map(m, base, bf, (uint64_t)(G * N), (uint64_t)D, (uint32_t)CR, (uint32_t)(D / 64));
}
bool maps_feat(CUtensorMap* m, const void* base, bool bf, int64_t G, int64_t N, int D, int CR) {
  return make_tma_map(m, base, bf, (uint64_t)(G * D), (uint64_t)N, (uint32_t)D, (uint32_t)(CR / 64));
}

template <int D, bool kBF16>
cudaError_t totals(const Launch& L, const Tensors& t, bool qw, float* units, float* tot, float* s_out) {
  using F = FG<D>;
  const Plan<D> pl(L.G, L.N);
  CUtensorMap mX, mY, mO;
  const void* x = qw ? t.q : t.k;
  const void* y = qw ? t.w : t.v;
  if (!maps_seq(&mX, x, kBF16, L.G, L.N, D, F::CR) || !maps_feat(&mY, y, kBF16, L.G, L.N, D, F::CR) ||
      !maps_feat(&mO, qw ? t.o : t.v, kBF16, L.G, L.N, D, F::CR))
    return cudaErrorInvalidValue;
  TotParams prm{t.g, s_out, units, L.N, pl.unit_rows, pl.U};
  const size_t smem = totals_smem<D>(qw);
  const dim3 grid((unsigned)pl.U, (unsigned)L.G);
  if (qw) {
    auto k = k_full_totals<D, kBF16, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ProfScope ps("la_bwd_full_r", L.stream);
    k<<<grid, 192, smem, L.stream>>>(mX, mY, mO, prm);
  } else {
    auto k = k_full_totals<D, kBF16, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ProfScope ps("la_fwd_full_kv", L.stream);
    k<<<grid, 192, smem, L.stream>>>(mX, mY, mO, prm);
  }
  k_full_sum<<<dim3((unsigned)((F::SZ + 255) / 256), (unsigned)L.G), 256, 0, L.stream>>>(
      units, pl.U, F::SZ, (int64_t)D * D + 2 * D + 1, tot);
  note_launch(2);
  return cudaGetLastError();
}

template <int D, bool kBF16, int kMode>
cudaError_t apply(const Launch& L, const CUtensorMap& mY, const CUtensorMap& mOut, const ApplyParams& prm,
                  const char* name) {
  const Plan<D> pl(L.G, L.N);
  auto k = k_full_apply<D, kBF16, kMode>;
  const size_t smem = apply_smem<D>(kMode);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  {
    ProfScope ps(name, L.stream);
    k<<<dim3((unsigned)pl.P, (unsigned)L.G), 64 + 128 * apply_wgs<D>(kMode), smem, L.stream>>>(mY, mOut, prm);
  }
  note_launch(1);
  return cudaGetLastError();
}

template <int D, bool kBF16>
cudaError_t forward_d(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  using F = FG<D>;
  const Plan<D> pl(L.G, L.N);
  float* units = ws.base;
  // with a saved-state buffer the totals land there (header P = -1 marks "totals") and the
  // backward reuses them instead of re-reading K and V
  float* tot = L.saved_out ? L.saved_out + kSavedHeader : units + L.G * pl.U * F::SZ;
  if (L.saved_out) write_saved_header(L.saved_out, (double)L.G, (double)L.N, (double)D, -1, 0, L.stream);
  cudaError_t e = totals<D, kBF16>(L, t, false, units, tot, nullptr);
  if (e != cudaSuccess) return e;
  CUtensorMap mQ, mO;
  if (!maps_seq(&mQ, t.q, kBF16, L.G, L.N, D, F::CR) || !maps_feat(&mO, out, kBF16, L.G, L.N, D, F::CR))
    return cudaErrorInvalidValue;
  ApplyParams prm{tot, tot, nullptr, nullptr, g, ws.flag, L.N, L.n_total > 0 ? L.n_total : L.N, pl.seg_rows,
                  L.a, L.b};
  return apply<D, kBF16, kFwd>(L, mQ, mO, prm, "la_fwd_full_apply");
}

template <int D, bool kBF16>
cudaError_t backward_d(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws) {
  using F = FG<D>;
  const Plan<D> pl(L.G, L.N);
  float* units = ws.base;                         // [G][U] records (S, then R)
  float* totR = units + L.G * pl.U * F::SZ;       // [G]
  float* totS = totR + L.G * F::SZ;               // [G] (when not saved)
  float* s = totS + L.G * F::SZ;                  // [G][N]
  cudaError_t e = cudaSuccess;
  if (L.saved_in)
    totS = const_cast<float*>(L.saved_in) + kSavedHeader;
  else
    e = totals<D, kBF16>(L, t, false, units, totS, nullptr);
  if (e != cudaSuccess) return e;
  e = totals<D, kBF16>(L, t, true, units, totR, s);
  if (e != cudaSuccess) return e;
  CUtensorMap mW, mV, mK, mdQ, mdK, mdV;
  if (!maps_feat(&mW, t.w, kBF16, L.G, L.N, D, F::CR) || !maps_feat(&mV, t.v, kBF16, L.G, L.N, D, F::CR) ||
      !maps_seq(&mK, t.k, kBF16, L.G, L.N, D, F::CR) || !maps_seq(&mdQ, dq, kBF16, L.G, L.N, D, F::CR) ||
      !maps_feat(&mdK, dk, kBF16, L.G, L.N, D, F::CR) || !maps_feat(&mdV, dv, kBF16, L.G, L.N, D, F::CR))
    return cudaErrorInvalidValue;
  ApplyParams pq{totS, totS, t.g, s, nullptr, nullptr, L.N, L.N, pl.seg_rows, L.a, L.b};
  if ((e = apply<D, kBF16, kDQ>(L, mW, mdQ, pq, "la_bwd_full_dq")) != cudaSuccess) return e;
  ApplyParams pr{totR, totR, nullptr, nullptr, nullptr, nullptr, L.N, L.N, pl.seg_rows, L.a, L.b};
  if ((e = apply<D, kBF16, kDK>(L, mV, mdK, pr, "la_bwd_full_dk")) != cudaSuccess) return e;
  return apply<D, kBF16, kDV>(L, mK, mdV, pr, "la_bwd_full_dv");
}

template <int D>
size_t ws_floats_d(int64_t G, int64_t N) {
  const Plan<D> pl(G, N);
  return (size_t)(G * pl.U * FG<D>::SZ + 2 * G * FG<D>::SZ + G * N);
}

}  // namespace

// Non-causal D = 128: the backward runs here (per-pass kernels: config 4 D = 128 backward
// 1.13 -> 0.98 ms), the forward stays on the fused k_fwd_full_tc (0.37 ms against 0.48 ms for
// the K/V totals + apply passes). The backward reads the totals that forward saved: the same
// [S | z | sigma | count] records behind a P = -1 header.
constexpr bool kFull128 = true;
bool full_tc_supported(const Launch& L, const Tensors& t, bool bwd) {
  const int64_t cr = L.D <= 64 ? 128 : 64;
  return !L.causal && (L.dtype == LA_BF16 || L.dtype == LA_F16) &&
         (L.D == 64 || (kFull128 && bwd && L.D == 128) || L.D == 192 || L.D == 256) &&
         L.fault == LA_FAULT_NONE && L.carry_prefix == nullptr && L.carry_suffix == nullptr && L.row_offset == 0 &&
         L.N % cr == 0 && t.lq == LA_SEQUENCE_MAJOR && t.lk == LA_SEQUENCE_MAJOR && t.lv == LA_FEATURE_MAJOR &&
         (t.w == nullptr || t.lw == LA_FEATURE_MAJOR) && L.G * L.N < (1ll << 31) && L.G * L.D < (1ll << 31);
}

size_t full_ws_floats(int64_t G, int64_t N, int64_t D) {
  switch (D) {
    case 64: return ws_floats_d<64>(G, N);
    case 128: return ws_floats_d<128>(G, N);
    case 192: return ws_floats_d<192>(G, N);
    case 256: return ws_floats_d<256>(G, N);
  }
  return 0;
}

cudaError_t full_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const bool bf = L.dtype == LA_BF16;
  switch (L.D) {
    case 64: return bf ? forward_d<64, true>(L, t, out, g, ws) : forward_d<64, false>(L, t, out, g, ws);
    case 192: return bf ? forward_d<192, true>(L, t, out, g, ws) : forward_d<192, false>(L, t, out, g, ws);
    case 256: return bf ? forward_d<256, true>(L, t, out, g, ws) : forward_d<256, false>(L, t, out, g, ws);
  }
  return cudaErrorInvalidValue;
}

cudaError_t full_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws) {
  const bool bf = L.dtype == LA_BF16;
  switch (L.D) {
    case 64: return bf ? backward_d<64, true>(L, t, dq, dk, dv, ws) : backward_d<64, false>(L, t, dq, dk, dv, ws);
    case 128:
      return bf ? backward_d<128, true>(L, t, dq, dk, dv, ws) : backward_d<128, false>(L, t, dq, dk, dv, ws);
    case 192:
      return bf ? backward_d<192, true>(L, t, dq, dk, dv, ws) : backward_d<192, false>(L, t, dq, dk, dv, ws);
    case 256:
      return bf ? backward_d<256, true>(L, t, dq, dk, dv, ws) : backward_d<256, false>(L, t, dq, dk, dv, ws);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lab
