// Tile helpers shared by the tensor-core backward kernels (la_sm100_bwd.cu, la_bwd_pair.cu):
// UMMA smem descriptors for the SW128 tiles, per-warp transposed row stores, the W_hat pass.
#pragma once
#include "sm100.cuh"

namespace lab {
namespace {

using namespace sm100;

// descriptors ---------------------------------------------------------------
// K-major tile with `rows` rows and 64-column panels `rows*128` bytes apart.
// The tile's base descriptor plus the k-step's byte offset (>> 4) in the start-address
// field: the base is common to a whole MMA chain, so each MMA costs one add (small hot code).
__device__ __forceinline__ uint64_t kd(uint32_t tile, int ks, uint32_t rows) {
  return sdesc_sw128(tile, 16, 1024) + (uint64_t)(((ks >> 2) * rows * 128 + (ks & 3) * 32) >> 4);
}
// MN-major tile: K rows of 128 B (16 per k-step), MN panels `panel` bytes apart.
__device__ __forceinline__ uint64_t mn(uint32_t tile, int ks, uint32_t panel) {
  return sdesc_sw128(tile, panel, 1024) + (uint64_t)((ks * 2048) >> 4);
}

// Per-warp transpose of 32 row segments (128 B each) through a 4 KB smem scratch
// (XOR-swizzled 16 B chunks), then coalesced 128 B-row global stores: lane L holds
// segment L in v[8]; dst(seg) gives the segment's global address.
// Same with one 2 KB scratch: lanes 0-15, then lanes 16-31.
template <typename DstFn>
__device__ __forceinline__ void warp_store_rows_2k(uint8_t* scratch, const uint4 (&v)[8], DstFn dst) {
  const int lane = (int)lane_id();
  auto slot = [&](int seg, int ch) -> uint4* {
    return (uint4*)(scratch + (seg & 15) * 128 + ((ch ^ (seg & 7)) << 4));
  };
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if ((lane >> 4) == h) {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) *slot(lane, ch) = v[ch];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int seg = 16 * h + 4 * k + (lane >> 3), ch = lane & 7;
      *(uint4*)((uint8_t*)dst(seg) + ch * 16) = *slot(seg, ch);
    }
    __syncwarp();
  }
}

template <typename DstFn>
__device__ __forceinline__ void warp_store_rows(uint8_t* scratch_lo, uint8_t* scratch_hi,
                                                const uint4 (&v)[8], DstFn dst) {
  const int lane = (int)lane_id();
  auto slot = [&](int seg, int ch) -> uint4* {
    uint8_t* base = seg < 16 ? scratch_lo : scratch_hi;
    return (uint4*)(base + (seg & 15) * 128 + ((ch ^ (seg & 7)) << 4));
  };
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) *slot(lane, ch) = v[ch];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int seg = 4 * k + (lane >> 3), ch = lane & 7;
    *(uint4*)((uint8_t*)dst(seg) + ch * 16) = *slot(seg, ch);
  }
  __syncwarp();
}

template <bool kBF16>
__device__ __forceinline__ float h2f(uint16_t h) {
  return kBF16 ? __bfloat162float(__ushort_as_bfloat16(h)) : __half2float(__ushort_as_half(h));
}

// Epilogue step E0: W_hat = omega / g in place (bf16) and s_i = sum_j o_ij w_hat_ij.
// 128 threads: lane = jg + 16 * (ig & 1), warp w -> ig = 2 w + lane / 16, each thread
// owns rows j = 16 rr + jg (rr < 8) and columns i in [8 ig, 8 ig + 8) of the 128 x 64
// tile; the 8 lanes of a quarter-warp touch 8 distinct swizzle rows (no bank conflicts).
template <bool kBF16>
__device__ __forceinline__ void what_pass(uint8_t* w_t, const uint4 (&o8)[8], const float4 (&g8)[2],
                                          float* s_s, int et) {
  const int lane = et & 31, w = et >> 5;
  const int jg = lane & 15, ig = 2 * w + (lane >> 4);
  float ginv[8] = {1.f / g8[0].x, 1.f / g8[0].y, 1.f / g8[0].z, 1.f / g8[0].w,
                   1.f / g8[1].x, 1.f / g8[1].y, 1.f / g8[1].z, 1.f / g8[1].w};
  float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const int j = 16 * rr + jg;
    uint4* p = (uint4*)(w_t + sw128_off(j, 8 * ig, 128));
    const uint4 wv = *p;
    const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
    const uint32_t oa[4] = {o8[rr].x, o8[rr].y, o8[rr].z, o8[rr].w};
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
#pragma unroll
  for (int u = 0; u < 8; ++u) {
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) sp[u] += __shfl_xor_sync(0xffffffffu, sp[u], off);
  }
  if (jg == 0) {
    *(float4*)(s_s + 8 * ig) = make_float4(sp[0], sp[1], sp[2], sp[3]);
    *(float4*)(s_s + 8 * ig + 4) = make_float4(sp[4], sp[5], sp[6], sp[7]);
  }
}

}  // namespace
}  // namespace lab
