// kvq_append.cu -- K1, quantize-on-append: bf16 K/V rows -> per-(token, head)
// fp32 scale + INT8 / FP8-E4M3 codes written into the paged pool
// (kvq_quant_append).  Rounding contract: DESIGN.md §3.
#include "kvq_common.cuh"

#include <algorithm>

namespace kvq {

// ---------------------------------------------------------------------------
// K1: quantize-on-append.  CTA = 16 consecutive tokens x 4 kv heads; an
// 8-lane group owns one (token pair 2p/2p+1, head): its 4 rows (K and V of
// both tokens, 16 elements per lane) are loaded up front with LDG.128 and
// their amax reduced over the 8 lanes.  Each lane then performs ONE of the
// group's 8 IEEE divisions (the scale or the inverse of one row) and the
// results are shuffled to where they are needed.  INT8 codes come from the
// exact round-to-nearest-even of an fp32 add of 1.5 * 2^23 (|y| <= 127 lands
// in the low mantissa byte) and byte permutes; rows holding NaN / inf, or
// whose inverse overflows (subnormal amax), take the F2I path instead, so the
// contract of DESIGN.md §3 holds bit for bit.  Output:
//   * whole page (slots blk*16 + 0..15: chunked prefill): the page image is
//     built in shared memory (st.shared, base + immediate offsets) and
//     written by one TMA bulk store per (block, head);
//   * otherwise (scattered tokens): direct global stores, V as interleaved
//     16-byte chunks when the pair's two slots are adjacent, else byte-wise.
// ---------------------------------------------------------------------------
constexpr int K1_THREADS = 256;
constexpr int K1_HEADS = 4;


__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ void bf16x16(const uint4 lo, const uint4 hi, float (&x)[16]) {
  const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[2 * i] = __uint_as_float(w[i] << 16);
    x[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
// INT8 codes of 16 values (contract).  FAST: no NaN / inf in
// the row and a finite inverse, so y = x * inv is finite with |y| <= 127 (1 + 2^-24):
// y + 1.5 * 2^23 rounds to the integer rint_even(y) (ulp 1, RN-even), which the
// clamp to +-127 cannot change, and its low byte is the code.
template <bool FAST>
__device__ __forceinline__ void int8x16(const float (&x)[16], float inv, uint32_t (&codes)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (FAST) {
      uint32_t r[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) r[e] = __float_as_uint(__fadd_rn(__fmul_rn(x[4 * i + e], inv), 12582912.0f));
      codes[i] = __byte_perm(__byte_perm(r[0], r[1], 0x0040), __byte_perm(r[2], r[3], 0x0040), 0x5410);
    } else {
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = max(-127, min(127, __float2int_rn(__fmul_rn(x[4 * i + e], inv))));  // NaN -> 0
        word |= ((uint32_t)(c & 0xff)) << (8 * e);
      }
      codes[i] = word;
    }
  }
}
__device__ __forceinline__ void e4m3x16(const float (&x)[16], float inv, uint32_t (&codes)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) y[e] = __fmul_rn(x[4 * i + e], inv);
    uint16_t l, h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(l) : "f"(y[1]), "f"(y[0]));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(y[3]), "f"(y[2]));
    codes[i] = (uint32_t)l | ((uint32_t)h << 16);
  }
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int KVD>
__global__ void __launch_bounds__(K1_THREADS, 3) quant_append_kernel(  // 80 regs, no spills
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int64_t k_stride,
    int64_t v_stride, const int32_t* __restrict__ slots, int T, int Hkv,
    uint8_t* __restrict__ pool, int64_t num_blocks) {
  // A K2 launched behind this kernel with programmatic serialization may start
  // its prologue now; it waits (griddepcontrol.wait) before reading any page.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ __align__(128) uint8_t img[K1_HEADS][PAGE];
  const int t0 = blockIdx.x * 16, h0 = blockIdx.y * K1_HEADS;
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 3, j = threadIdx.x & 7;  // lane j of the group owns d [16j, 16j+16)
  const int hh = grp >> 3, pp = grp & 7;                  // head h0+hh, tokens t0+2pp, t0+2pp+1
  const int h = h0 + hh;
  // Row loads first (they do not depend on the slots), then the slot loads.
  uint4 raw[2][2][2];  // [token][K|V][lo|hi 16 B]
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = t0 + 2 * pp + i;
    const bool in = t < T && h < Hkv;
#pragma unroll
    for (int kv = 0; kv < 2; ++kv) {
      const __nv_bfloat16* src = (kv ? v + (int64_t)t * v_stride : k + (int64_t)t * k_stride) + h * HD + 16 * j;
      raw[i][kv][0] = in ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0, 0, 0, 0);
      raw[i][kv][1] = in ? __ldg(reinterpret_cast<const uint4*>(src + 8)) : make_uint4(0, 0, 0, 0);
    }
  }
  int slot[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = t0 + 2 * pp + i;
    slot[i] = t < T ? __ldg(slots + t) : -1;
  }
  // Whole-page test: 16 in-range tokens with slots blk*16 + 0..15.
  int my_slot = -1;
  if (threadIdx.x < 16 && t0 + threadIdx.x < T) my_slot = __ldg(slots + t0 + threadIdx.x);
  const int first = t0 < T ? __ldg(slots + t0) : -1;
  const bool mine_ok = threadIdx.x >= 16 ||
                       (my_slot >= 0 && my_slot == first + (int)threadIdx.x && (first & 15) == 0 &&
                        (first >> 4) < num_blocks);
  const bool whole = __syncthreads_and(mine_ok);

  // ---- per-row amax over the 8 lanes (NaN-propagating for INT8: flags NaN rows)
  const float qmax = KVD == KVQ_FP8_E4M3 ? 448.0f : 127.0f;
  float am[4];  // row rr = 2 * token + kv
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    float x[16];
    bf16x16(raw[rr >> 1][rr & 1][0], raw[rr >> 1][rr & 1][1], x);
    float a = 0.0f;
#pragma unroll
    for (int e = 0; e < 16; ++e) a = KVD == KVQ_INT8 ? max_nan(a, fabsf(x[e])) : fmaxf(a, fabsf(x[e]));
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const float b = __shfl_xor_sync(FULL, a, o);
      a = KVD == KVQ_INT8 ? max_nan(a, b) : fmaxf(a, b);
    }
    am[rr] = a;
  }
  bool nanrow[4] = {false, false, false, false};
  if (KVD == KVQ_INT8 && __any_sync(FULL, am[0] != am[0] || am[1] != am[1] || am[2] != am[2] || am[3] != am[3])) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {  // rare: NaN-ignoring amax of the rows that hold NaN
      nanrow[rr] = am[rr] != am[rr];
      float x[16];
      bf16x16(raw[rr >> 1][rr & 1][0], raw[rr >> 1][rr & 1][1], x);
      float a = 0.0f;
#pragma unroll
      for (int e = 0; e < 16; ++e) a = fmaxf(a, fabsf(x[e]));
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) a = fmaxf(a, __shfl_xor_sync(FULL, a, o));
      if (nanrow[rr]) am[rr] = a;
    }
  }
  // ---- one IEEE division per lane: lane j -> row j & 3, scale (j >= 4) or inverse (j < 4)
  float dv;
  {
    const int rr = j & 3;
    const float a = rr == 0 ? am[0] : rr == 1 ? am[1] : rr == 2 ? am[2] : am[3];
    const bool is_scale = j >= 4;
    dv = __fdiv_rn(is_scale ? a : qmax, is_scale ? qmax : a);
    if (!is_scale && !(a > 0.0f)) dv = 0.0f;
  }
  float inv[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) inv[rr] = __shfl_sync(FULL, dv, (lane & ~7) | rr);

  // ---- codes: [token][K|V][4 words]
  uint32_t code[2][2][4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    float x[16];
    bf16x16(raw[rr >> 1][rr & 1][0], raw[rr >> 1][rr & 1][1], x);
    if constexpr (KVD == KVQ_FP8_E4M3) {
      e4m3x16(x, inv[rr], code[rr >> 1][rr & 1]);
    } else {
      const bool fast = !nanrow[rr] && am[rr] < INFINITY && inv[rr] < INFINITY;  // uniform per group
      if (fast) int8x16<true>(x, inv[rr], code[rr >> 1][rr & 1]);
      else int8x16<false>(x, inv[rr], code[rr >> 1][rr & 1]);
    }
  }
  // V codes of the token pair interleaved: bytes (d, t0), (d, t1) for d = 16j .. 16j+15
  // form logical pair-row bytes [32j, 32j+32) = two 16-byte chunks.
  uint32_t il[8];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    il[2 * w] = __byte_perm(code[0][1][w], code[1][1][w], 0x5140);
    il[2 * w + 1] = __byte_perm(code[0][1][w], code[1][1][w], 0x7362);
  }
  const int rs = j & 3, ts = rs >> 1;  // the scale this lane holds (j >= 4): row rs, token ts

  if (whole) {
    // ---- page image in shared memory; K word w of token tok sits at
    //      p*256 + 16c + (2*half + hi)*4 + 64*(w ^ (p & 1)), p = tok & 7 (p & 1 == i here)
    const uint32_t img_s = smem_u32(img[hh]);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int tok = 2 * pp + i, p = tok & 7;
      const uint32_t kb = img_s + p * 256 + 16 * (j & 3) + (2 * (j >> 2) + (tok >> 3)) * 4;
#pragma unroll
      for (int w = 0; w < 4; ++w) sts32(kb + 64 * (w ^ i), code[i][0][w]);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half)
      sts128(img_s + v_code_off(2 * pp, 16 * j + 8 * half),
             make_uint4(il[4 * half], il[4 * half + 1], il[4 * half + 2], il[4 * half + 3]));
    if (j >= 4) sts32(img_s + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * (2 * pp + ts), __float_as_uint(dv));
    // generic-proxy smem writes -> visible to the bulk copy (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int nh = min(K1_HEADS, Hkv - h0);
    if (threadIdx.x < nh) {
      uint8_t* dst = pool + ((int64_t)(first >> 4) * Hkv + h0 + threadIdx.x) * PAGE;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"(smem_u32(img[threadIdx.x])), "n"(PAGE)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // Only the shared-memory reads must finish before the CTA exits (and its
      // smem is reused); the global writes complete with the grid.
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    return;
  }

  // ---- scattered tokens: direct global stores
  bool live[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    live[i] = slot[i] >= 0 && (slot[i] >> 4) < num_blocks && h < Hkv;
    if (slot[i] >= 0 && (slot[i] >> 4) >= num_blocks && j == 0 && hh == 0) flag_dev_err(KVQ_DERR_SLOT);
  }
  const bool pair_adj = live[0] && live[1] && (slot[0] & 1) == 0 && slot[1] == slot[0] + 1;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (!live[i]) continue;
    const int tok = slot[i] & 15;
    uint8_t* page = pool + ((int64_t)(slot[i] >> 4) * Hkv + h) * PAGE;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      *reinterpret_cast<uint32_t*>(page + k_code_off(tok, 16 * j + 4 * w)) = code[i][0][w];
    if (!pair_adj) {  // lone token: V bytes at 2d + (tok & 1)
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          page[v_code_off(tok, 16 * j + 4 * w + e)] = (uint8_t)(code[i][1][w] >> (8 * e));
    }
    if (j >= 4 && ts == i)
      *reinterpret_cast<float*>(page + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * tok) = dv;
  }
  if (pair_adj) {
    const int tok = slot[0] & 15;  // even
    uint8_t* page = pool + ((int64_t)(slot[0] >> 4) * Hkv + h) * PAGE;
#pragma unroll
    for (int half = 0; half < 2; ++half)
      *reinterpret_cast<uint4*>(page + v_code_off(tok, 16 * j + 8 * half)) =
          make_uint4(il[4 * half], il[4 * half + 1], il[4 * half + 2], il[4 * half + 3]);
  }
}

// ---------------------------------------------------------------------------
// K1 tile loop (large appends: chunked prefill).  Same tile work and rounding
// as quant_append_kernel, but a persistent grid (2 CTAs per SM) walks the
// (16-token, 4-head) tiles, and the NEXT tile's rows and slots are loaded into
// registers before the current tile is quantized and stored, so every warp
// keeps a tile of loads in flight through its compute and store phases (the
// one-shot kernel ran 2.4 waves of short CTAs, each exposing its whole load
// latency).  No CTA-wide barrier: every warp decides "whole page" itself from
// the tile's 16 slots (L1 hits), and the page image of one head is built by
// its own pair of warps, which meet at a named barrier before one of them
// issues the TMA bulk store; images are double-buffered, so the store of tile
// n reads its buffer while tile n + 1 fills the other.
// ---------------------------------------------------------------------------
constexpr int K1L_CTAS = 2;

struct TileRows {
  uint4 raw[2][2][2];  // [token][K|V][lo|hi 16 B]
  int slot[2];         // slots of this group's two tokens
  int s16;             // lanes 0..15: slot of tile token `lane` (whole-page test)
};

__device__ __forceinline__ void load_tile(const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                                          int64_t k_stride, int64_t v_stride, const int32_t* __restrict__ slots,
                                          int T, int Hkv, int t0, int h, int pp, int j, int lane, TileRows& r) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = t0 + 2 * pp + i;
    const bool in = t < T && h < Hkv;
#pragma unroll
    for (int kv = 0; kv < 2; ++kv) {
      const __nv_bfloat16* src = (kv ? v + (int64_t)t * v_stride : k + (int64_t)t * k_stride) + h * HD + 16 * j;
      r.raw[i][kv][0] = in ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0, 0, 0, 0);
      r.raw[i][kv][1] = in ? __ldg(reinterpret_cast<const uint4*>(src + 8)) : make_uint4(0, 0, 0, 0);
    }
    r.slot[i] = t < T ? __ldg(slots + t) : -1;
  }
  r.s16 = (lane < 16 && t0 + lane < T) ? __ldg(slots + t0 + lane) : -1;
}

template <int KVD>
__global__ void __launch_bounds__(K1_THREADS, K1L_CTAS) quant_append_loop_kernel(
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int64_t k_stride,
    int64_t v_stride, const int32_t* __restrict__ slots, int T, int Hkv,
    uint8_t* __restrict__ pool, int64_t num_blocks, int HG, int ntiles) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ __align__(128) uint8_t img[2][K1_HEADS][PAGE];
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 3, j = threadIdx.x & 7;
  const int hh = grp >> 3, pp = grp & 7;
  const bool issuer = (threadIdx.x & 63) == 0;  // one thread of the warp pair that builds head hh's image
  const float qmax = KVD == KVQ_FP8_E4M3 ? 448.0f : 127.0f;
  int buf = 0;
  TileRows cur;
  int tile = blockIdx.x;
  if (tile < ntiles) {
    const int tt = tile / HG;
    load_tile(k, v, k_stride, v_stride, slots, T, Hkv, tt * 16, (tile - tt * HG) * K1_HEADS + hh, pp, j, lane, cur);
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const int tt = tile / HG, h = (tile - tt * HG) * K1_HEADS + hh;
    TileRows nxt;
    const int next = tile + gridDim.x;
    if (next < ntiles) {  // in flight while this tile is quantized and stored
      const int nt = next / HG;
      load_tile(k, v, k_stride, v_stride, slots, T, Hkv, nt * 16, (next - nt * HG) * K1_HEADS + hh, pp, j, lane,
                nxt);
    }
    // Whole-page test (every warp alike): 16 in-range tokens with slots blk*16 + 0..15.
    const int first = __shfl_sync(FULL, cur.s16, 0);
    const bool whole = __all_sync(FULL, lane >= 16 || (cur.s16 >= 0 && cur.s16 == first + lane &&
                                                       (first & 15) == 0 && (first >> 4) < num_blocks));
    // ---- per-row amax over the 8 lanes (NaN-propagating for INT8: flags NaN rows)
    float am[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      float x[16];
      bf16x16(cur.raw[rr >> 1][rr & 1][0], cur.raw[rr >> 1][rr & 1][1], x);
      float a = 0.0f;
#pragma unroll
      for (int e = 0; e < 16; ++e) a = KVD == KVQ_INT8 ? max_nan(a, fabsf(x[e])) : fmaxf(a, fabsf(x[e]));
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const float b = __shfl_xor_sync(FULL, a, o);
        a = KVD == KVQ_INT8 ? max_nan(a, b) : fmaxf(a, b);
      }
      am[rr] = a;
    }
    bool nanrow[4] = {false, false, false, false};
    if (KVD == KVQ_INT8 &&
        __any_sync(FULL, am[0] != am[0] || am[1] != am[1] || am[2] != am[2] || am[3] != am[3])) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {  // rare: NaN-ignoring amax of the rows that hold NaN
        nanrow[rr] = am[rr] != am[rr];
        float x[16];
        bf16x16(cur.raw[rr >> 1][rr & 1][0], cur.raw[rr >> 1][rr & 1][1], x);
        float a = 0.0f;
#pragma unroll
        for (int e = 0; e < 16; ++e) a = fmaxf(a, fabsf(x[e]));
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) a = fmaxf(a, __shfl_xor_sync(FULL, a, o));
        if (nanrow[rr]) am[rr] = a;
      }
    }
    // ---- one IEEE division per lane: lane j -> row j & 3, scale (j >= 4) or inverse (j < 4)
    float dv;
    {
      const int rr = j & 3;
      const float a = rr == 0 ? am[0] : rr == 1 ? am[1] : rr == 2 ? am[2] : am[3];
      const bool is_scale = j >= 4;
      dv = __fdiv_rn(is_scale ? a : qmax, is_scale ? qmax : a);
      if (!is_scale && !(a > 0.0f)) dv = 0.0f;
    }
    float inv[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) inv[rr] = __shfl_sync(FULL, dv, (lane & ~7) | rr);
    uint32_t code[2][2][4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      float x[16];
      bf16x16(cur.raw[rr >> 1][rr & 1][0], cur.raw[rr >> 1][rr & 1][1], x);
      if constexpr (KVD == KVQ_FP8_E4M3) {
        e4m3x16(x, inv[rr], code[rr >> 1][rr & 1]);
      } else {
        const bool fast = !nanrow[rr] && am[rr] < INFINITY && inv[rr] < INFINITY;  // uniform per group
        if (fast) int8x16<true>(x, inv[rr], code[rr >> 1][rr & 1]);
        else int8x16<false>(x, inv[rr], code[rr >> 1][rr & 1]);
      }
    }
    uint32_t il[8];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      il[2 * w] = __byte_perm(code[0][1][w], code[1][1][w], 0x5140);
      il[2 * w + 1] = __byte_perm(code[0][1][w], code[1][1][w], 0x7362);
    }
    const int rs = j & 3, ts = rs >> 1;
    if (whole) {
      const uint32_t img_s = smem_u32(img[buf][hh]);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int tok = 2 * pp + i, p = tok & 7;
        const uint32_t kb = img_s + p * 256 + 16 * (j & 3) + (2 * (j >> 2) + (tok >> 3)) * 4;
#pragma unroll
        for (int w = 0; w < 4; ++w) sts32(kb + 64 * (w ^ i), code[i][0][w]);
      }
#pragma unroll
      for (int half = 0; half < 2; ++half)
        sts128(img_s + v_code_off(2 * pp, 16 * j + 8 * half),
               make_uint4(il[4 * half], il[4 * half + 1], il[4 * half + 2], il[4 * half + 3]));
      if (j >= 4) sts32(img_s + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * (2 * pp + ts), __float_as_uint(dv));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // The issuer first waits until every earlier store has read its image (the
      // one from this buffer was issued two whole tiles ago); past the barrier
      // the pair may refill the other buffer.
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync %0, 64;" ::"r"(1 + hh) : "memory");
      if (issuer && h < Hkv) {
        uint8_t* dst = pool + ((int64_t)(first >> 4) * Hkv + h) * PAGE;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(img_s), "n"(PAGE)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      buf ^= 1;
    } else {
      bool live[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        live[i] = cur.slot[i] >= 0 && (cur.slot[i] >> 4) < num_blocks && h < Hkv;
        if (cur.slot[i] >= 0 && (cur.slot[i] >> 4) >= num_blocks && j == 0 && hh == 0) flag_dev_err(KVQ_DERR_SLOT);
      }
      const bool pair_adj = live[0] && live[1] && (cur.slot[0] & 1) == 0 && cur.slot[1] == cur.slot[0] + 1;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (!live[i]) continue;
        const int tok = cur.slot[i] & 15;
        uint8_t* page = pool + ((int64_t)(cur.slot[i] >> 4) * Hkv + h) * PAGE;
#pragma unroll
        for (int w = 0; w < 4; ++w)
          *reinterpret_cast<uint32_t*>(page + k_code_off(tok, 16 * j + 4 * w)) = code[i][0][w];
        if (!pair_adj) {
#pragma unroll
          for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              page[v_code_off(tok, 16 * j + 4 * w + e)] = (uint8_t)(code[i][1][w] >> (8 * e));
        }
        if (j >= 4 && ts == i)
          *reinterpret_cast<float*>(page + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * tok) = dv;
      }
      if (pair_adj) {
        const int tok = cur.slot[0] & 15;
        uint8_t* page = pool + ((int64_t)(cur.slot[0] >> 4) * Hkv + h) * PAGE;
#pragma unroll
        for (int half = 0; half < 2; ++half)
          *reinterpret_cast<uint4*>(page + v_code_off(tok, 16 * j + 8 * half)) =
              make_uint4(il[4 * half], il[4 * half + 1], il[4 * half + 2], il[4 * half + 3]);
      }
    }
    cur = nxt;
  }
  // the images must stay valid until the bulk copies have read them
  if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// K1r: the decode-shaped append (a few tokens, each in a different page).
// One warp per (token, head): lane l quantizes K and V elements [4l, 4l+4)
// (one LDG.64 each), so the per-warp chain is ~100 instructions and a
// B = 256 x 8-head step spreads over 256 CTAs instead of 32.  Same rounding
// as quantize16 (the amax is an exact max, independent of the lane split).
// ---------------------------------------------------------------------------
constexpr int K1R_WARPS = 8;
// Up to this many (token, head) rows a launch takes the one-warp-per-row kernel.
constexpr int64_t K1_ROWS_MAX = 8192;

template <int KVD>
__global__ void __launch_bounds__(K1R_WARPS * 32) quant_append_rows_kernel(
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int64_t k_stride,
    int64_t v_stride, const int32_t* __restrict__ slots, int T, int Hkv,
    uint8_t* __restrict__ pool, int64_t num_blocks) {
  // A K2 launched behind this kernel with programmatic serialization may start
  // its prologue now; it waits (griddepcontrol.wait) before reading any page.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row = blockIdx.x * K1R_WARPS + (threadIdx.x >> 5);  // t * Hkv + h
  const int lane = threadIdx.x & 31;
  if (row >= T * Hkv) return;  // whole warps only
  const int t = row / Hkv, h = row - t * Hkv;
  const uint2 kw = __ldg(reinterpret_cast<const uint2*>(k + (int64_t)t * k_stride + h * HD + 4 * lane));
  const uint2 vw = __ldg(reinterpret_cast<const uint2*>(v + (int64_t)t * v_stride + h * HD + 4 * lane));
  const int slot = __ldg(slots + t);
  float xk[4], xv[4];
  xk[0] = __uint_as_float(kw.x << 16), xk[1] = __uint_as_float(kw.x & 0xffff0000u);
  xk[2] = __uint_as_float(kw.y << 16), xk[3] = __uint_as_float(kw.y & 0xffff0000u);
  xv[0] = __uint_as_float(vw.x << 16), xv[1] = __uint_as_float(vw.x & 0xffff0000u);
  xv[2] = __uint_as_float(vw.y << 16), xv[3] = __uint_as_float(vw.y & 0xffff0000u);
  float ak = fmaxf(fmaxf(fabsf(xk[0]), fabsf(xk[1])), fmaxf(fabsf(xk[2]), fabsf(xk[3])));
  float av = fmaxf(fmaxf(fabsf(xv[0]), fabsf(xv[1])), fmaxf(fabsf(xv[2]), fabsf(xv[3])));
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    ak = fmaxf(ak, __shfl_xor_sync(FULL, ak, o));
    av = fmaxf(av, __shfl_xor_sync(FULL, av, o));
  }
  if (slot < 0 || (slot >> 4) >= num_blocks) {
    if (slot >= 0 && lane == 0) flag_dev_err(KVQ_DERR_SLOT);
    return;
  }
  const float qmax = KVD == KVQ_FP8_E4M3 ? 448.0f : 127.0f;
  const float ik = ak > 0.0f ? __fdiv_rn(qmax, ak) : 0.0f;
  const float iv = av > 0.0f ? __fdiv_rn(qmax, av) : 0.0f;
  const uint32_t ck = quant_codes4<KVD>(xk, ik), cv = quant_codes4<KVD>(xv, iv);
  const int tok = slot & 15;
  uint8_t* page = pool + ((int64_t)(slot >> 4) * Hkv + h) * PAGE;
  *reinterpret_cast<uint32_t*>(page + k_code_off(tok, 4 * lane)) = ck;
#pragma unroll
  for (int e = 0; e < 4; ++e) page[v_code_off(tok, 4 * lane + e)] = (uint8_t)(cv >> (8 * e));
  if (lane < 2) {
    const float a = lane ? av : ak;
    *reinterpret_cast<float*>(page + (lane ? VS_OFF : KS_OFF) + 4 * tok) = __fdiv_rn(a, qmax);
  }
}

unsigned read_and_clear_dev_err_append() { return read_and_clear_dev_err_tu(); }

}  // namespace kvq

using namespace kvq_abi;

extern "C" {

int kvq_quant_append(const void* k, const void* v, int64_t k_token_stride, int64_t v_token_stride,
                     const int32_t* slot_mapping, int32_t T, int32_t Hkv, int32_t kv_dtype,
                     void* pool, int64_t num_blocks, void* stream) {
  if (T < 0 || Hkv <= 0 || num_blocks <= 0) return fail(KVQ_EINVAL, "quant_append: bad sizes");
  if (T == 0) return KVQ_OK;
  if (!k || !v || !slot_mapping || !pool) return fail(KVQ_EINVAL, "quant_append: null pointer");
  if (!aligned(k, 8) || !aligned(v, 8) || !aligned(pool, 16) || (k_token_stride % 4) || (v_token_stride % 4))
    return fail(KVQ_EINVAL, "quant_append: k/v rows must be 8-byte aligned, pool 16-byte aligned");
  if (kv_dtype != KVQ_INT8 && kv_dtype != KVQ_FP8_E4M3)
    return fail(KVQ_EUNSUPPORTED, "quant_append: unknown kv dtype");
  if (int rc = check_device()) return rc;
  if (Hkv > 65535) return fail(KVQ_EINVAL, "quant_append: Hkv too large");
  auto st = static_cast<cudaStream_t>(stream);
  // Same (max-shared) L1/smem carveout as K2 so a decode step never pays an
  // SM reconfiguration between the append and the attention kernel.
  static const bool carve = [] {
    const void* fns[] = {(const void*)kvq::quant_append_kernel<KVQ_INT8>,
                         (const void*)kvq::quant_append_kernel<KVQ_FP8_E4M3>,
                         (const void*)kvq::quant_append_loop_kernel<KVQ_INT8>,
                         (const void*)kvq::quant_append_loop_kernel<KVQ_FP8_E4M3>,
                         (const void*)kvq::quant_append_rows_kernel<KVQ_INT8>,
                         (const void*)kvq::quant_append_rows_kernel<KVQ_FP8_E4M3>};
    for (const void* f : fns)
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    return true;
  }();
  (void)carve;
  const auto kp = static_cast<const __nv_bfloat16*>(k);
  const auto vp = static_cast<const __nv_bfloat16*>(v);
  auto* pp = static_cast<uint8_t*>(pool);
  const bool rows16 = aligned(k, 16) && aligned(v, 16) && (k_token_stride % 8) == 0 && (v_token_stride % 8) == 0;
  if ((int64_t)T * Hkv <= kvq::K1_ROWS_MAX || !rows16) {
    // Decode-shaped batch (latency-bound), or rows only 8-byte aligned (the tile
    // kernels load 16 bytes per lane): one warp per (token, head).
    const unsigned nblk = (unsigned)((T * Hkv + kvq::K1R_WARPS - 1) / kvq::K1R_WARPS);
    if (kv_dtype == KVQ_INT8)
      kvq::quant_append_rows_kernel<KVQ_INT8><<<nblk, kvq::K1R_WARPS * 32, 0, st>>>(
          kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks);
    else
      kvq::quant_append_rows_kernel<KVQ_FP8_E4M3><<<nblk, kvq::K1R_WARPS * 32, 0, st>>>(
          kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks);
    return check_launch("quant_append");
  }
  const int HG = (Hkv + kvq::K1_HEADS - 1) / kvq::K1_HEADS;
  const int64_t ntiles = (int64_t)((T + 15) / 16) * HG;
  if (ntiles > INT32_MAX) return fail(KVQ_EINVAL, "quant_append: too many tokens");
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * kvq::K1L_CTAS);
  if (kv_dtype == KVQ_INT8)
    kvq::quant_append_loop_kernel<KVQ_INT8><<<grid, kvq::K1_THREADS, 0, st>>>(
        kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks, HG, (int)ntiles);
  else
    kvq::quant_append_loop_kernel<KVQ_FP8_E4M3><<<grid, kvq::K1_THREADS, 0, st>>>(
        kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks, HG, (int)ntiles);
  return check_launch("quant_append");
}

}  // extern "C"
