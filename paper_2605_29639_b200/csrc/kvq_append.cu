// kvq_append.cu -- K1, quantize-on-append: bf16 K/V rows -> per-(token, head)
// fp32 scale + INT8 / FP8-E4M3 codes written into the paged pool
// (kvq_quant_append).  Rounding contract: DESIGN.md §3.
#include "kvq_common.cuh"

#include <cudaTypedefs.h>

#include <algorithm>

namespace kvq {

// ---------------------------------------------------------------------------
// K1 quantizer math, per 8-lane group.  The group owns one (token pair, head):
// its 4 rows (K and V of both tokens; lane j holds elements [16j, 16j+16) of
// each) are in registers.  Each row's amax is reduced over the 8 lanes; each
// lane then performs ONE of the group's 8 IEEE divisions (the scale or the
// inverse of one row) and the results are shuffled to where they are needed.
// INT8 codes come from the exact round-to-nearest-even of an fp32 add of
// 1.5 * 2^23 (|y| <= 127 lands in the low mantissa byte) and byte permutes;
// rows holding NaN / inf, or whose inverse overflows (subnormal amax), take the
// F2I path instead, so the contract of DESIGN.md §3 holds bit for bit.
// ---------------------------------------------------------------------------
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

struct GroupCodes {
  uint32_t kc[2][4];  // K codes of the pair's tokens 0 / 1 (this lane's 16 values)
  uint32_t il[8];     // V codes of the pair, token-interleaved: bytes (d, t0), (d, t1), d = 16j .. 16j+15
  float dv;           // this lane's division: row j & 3 (= 2 * token + kv), scale (j >= 4) or inverse
};

template <int KVD>
__device__ __forceinline__ void quant_group(const uint4 (&raw)[2][2][2], int lane, int j, GroupCodes& g) {
  const float qmax = KVD == KVQ_FP8_E4M3 ? 448.0f : 127.0f;
  // ---- per-row amax over the 8 lanes (NaN-propagating for INT8: flags NaN rows)
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
  // ---- one IEEE division per lane
  {
    const int rr = j & 3;
    const float a = rr == 0 ? am[0] : rr == 1 ? am[1] : rr == 2 ? am[2] : am[3];
    const bool is_scale = j >= 4;
    g.dv = __fdiv_rn(is_scale ? a : qmax, is_scale ? qmax : a);
    if (!is_scale && !(a > 0.0f)) g.dv = 0.0f;
  }
  float inv[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) inv[rr] = __shfl_sync(FULL, g.dv, (lane & ~7) | rr);
  uint32_t vc[2][4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    float x[16];
    bf16x16(raw[rr >> 1][rr & 1][0], raw[rr >> 1][rr & 1][1], x);
    uint32_t(&c)[4] = (rr & 1) ? vc[rr >> 1] : g.kc[rr >> 1];
    if constexpr (KVD == KVQ_FP8_E4M3) {
      e4m3x16(x, inv[rr], c);
    } else {
      const bool fast = !nanrow[rr] && am[rr] < INFINITY && inv[rr] < INFINITY;  // uniform per group
      if (fast) int8x16<true>(x, inv[rr], c);
      else int8x16<false>(x, inv[rr], c);
    }
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    g.il[2 * w] = __byte_perm(vc[0][w], vc[1][w], 0x5140);
    g.il[2 * w + 1] = __byte_perm(vc[0][w], vc[1][w], 0x7362);
  }
}

// Page image of one head in shared memory (a whole block: tokens 2pp, 2pp + 1
// of this group).  K word w of token tok sits at
// p*256 + 16c + (2*half + hi)*4 + 64*(w ^ (p & 1)), p = tok & 7 (p & 1 == i here).
__device__ __forceinline__ void write_image(uint32_t img_s, int pp, int j, const GroupCodes& g) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int tok = 2 * pp + i, p = tok & 7;
    const uint32_t kb = img_s + p * 256 + 16 * (j & 3) + (2 * (j >> 2) + (tok >> 3)) * 4;
#pragma unroll
    for (int w = 0; w < 4; ++w) sts32(kb + 64 * (w ^ i), g.kc[i][w]);
  }
#pragma unroll
  for (int half = 0; half < 2; ++half)
    sts128(img_s + v_code_off(2 * pp, 16 * j + 8 * half),
           make_uint4(g.il[4 * half], g.il[4 * half + 1], g.il[4 * half + 2], g.il[4 * half + 3]));
  const int rs = j & 3, ts = rs >> 1;
  if (j >= 4) sts32(img_s + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * (2 * pp + ts), __float_as_uint(g.dv));
}

// Scattered tokens (not one whole block): direct global stores, V as
// interleaved 16-byte chunks when the pair's two slots are adjacent, else byte-wise.
__device__ __forceinline__ void store_scattered(uint8_t* __restrict__ pool, int64_t num_blocks, int Hkv, int h,
                                                const int (&slot)[2], int j, bool flag_lane, const GroupCodes& g) {
  bool live[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    live[i] = slot[i] >= 0 && (slot[i] >> 4) < num_blocks && h < Hkv;
    if (slot[i] >= 0 && (slot[i] >> 4) >= num_blocks && flag_lane) flag_dev_err(KVQ_DERR_SLOT);
  }
  const bool pair_adj = live[0] && live[1] && (slot[0] & 1) == 0 && slot[1] == slot[0] + 1;
  const int rs = j & 3, ts = rs >> 1;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (!live[i]) continue;
    const int tok = slot[i] & 15;
    uint8_t* page = pool + ((int64_t)(slot[i] >> 4) * Hkv + h) * PAGE;
#pragma unroll
    for (int w = 0; w < 4; ++w) *reinterpret_cast<uint32_t*>(page + k_code_off(tok, 16 * j + 4 * w)) = g.kc[i][w];
    if (!pair_adj) {  // lone token: V bytes at 2d + (tok & 1)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t vw = __byte_perm(g.il[2 * w], g.il[2 * w + 1], i ? 0x7531 : 0x6420);
#pragma unroll
        for (int e = 0; e < 4; ++e) page[v_code_off(tok, 16 * j + 4 * w + e)] = (uint8_t)(vw >> (8 * e));
      }
    }
    if (j >= 4 && ts == i) *reinterpret_cast<float*>(page + ((rs & 1) ? VS_OFF : KS_OFF) + 4 * tok) = g.dv;
  }
  if (pair_adj) {
    const int tok = slot[0] & 15;  // even
    uint8_t* page = pool + ((int64_t)(slot[0] >> 4) * Hkv + h) * PAGE;
#pragma unroll
    for (int half = 0; half < 2; ++half)
      *reinterpret_cast<uint4*>(page + v_code_off(tok, 16 * j + 8 * half)) =
          make_uint4(g.il[4 * half], g.il[4 * half + 1], g.il[4 * half + 2], g.il[4 * half + 3]);
  }
}

// ---------------------------------------------------------------------------
// K1 tile kernel (large appends: chunked prefill, T * Hkv > K1_ROWS_MAX).
// Work unit = 16 consecutive tokens x 1 kv head (one page when the 16 slots
// are one whole block).  Persistent grid, 2 CTAs per SM, 9 warps:
//   * warp 0, the producer: one thread issues, per unit, two TMA tensor loads
//     (cp.async.bulk.tensor.2d over the [T][Hkv * 128] bf16 K and V views,
//     box 16 tokens x 128 = 4 KB each; tokens past T are zero-filled) into a
//     ring of K1T_STAGES 8 KB stages; the stage's mbarrier counts the bytes;
//   * warps 1..8, four teams of 2 consumers: team i & 3 quantizes the CTA's
//     i-th unit.  An 8-lane group owns one token pair and reads its 4 rows (K
//     and V of both tokens) from the stage, two LDS.128 per row; each warp
//     releases the stage (one mbarrier arrive) as soon as its rows are in
//     registers;
//   * whole page: the team builds the page image in shared memory (double-
//     buffered), meets at a named barrier, and one thread issues a 4224-byte
//     TMA bulk store; otherwise direct global stores.
// The ring keeps up to 8 x 8 KB of row loads in flight per CTA whatever the
// consumers are doing.  Designs measured before it (profiles/r2/k1_*):
// register prefetch of one tile per warp (0.47 of the copy peak, LDG
// long-scoreboard stalls); per-row 512-byte cp.async.bulk copies (32 per unit:
// the producer's serialized issue loop, ~86 cycles per copy, was the
// bottleneck); 2-head units (7.1 per CTA on C5, so 1 CTA in 7 ran an 8th unit
// after the others were done: a 2-3 us tail in the per-CTA timeline).
// ---------------------------------------------------------------------------
constexpr int K1T_STAGES = 8;
constexpr int K1T_STAGE = 2 * 16 * HD * 2;       // K|V x 16 tokens x 256 B
constexpr int K1T_TEAMS = 4;                     // of 2 warps
constexpr int K1T_THREADS = 32 + K1T_TEAMS * 64;
constexpr int K1T_IMG = K1T_TEAMS * 2 * PAGE;    // [team][buf] page images
constexpr int K1T_SMEM = K1T_STAGES * K1T_STAGE + K1T_IMG + 2 * K1T_STAGES * 8 + 128;  // + alignment slack

// TMA tensor load of one box into shared memory, completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

struct UnitSlots {
  int slot[2];  // slots of this group's two tokens
  int s16;      // lanes 0..15: slot of unit token `lane` (whole-page test)
};
__device__ __forceinline__ void load_slots(const int32_t* __restrict__ slots, int T, int t0, int pp, int lane,
                                           UnitSlots& s) {
#pragma unroll
  for (int i = 0; i < 2; ++i) s.slot[i] = t0 + 2 * pp + i < T ? __ldg(slots + t0 + 2 * pp + i) : -1;
  s.s16 = (lane < 16 && t0 + lane < T) ? __ldg(slots + t0 + lane) : -1;
}

template <int KVD>
__global__ void __launch_bounds__(K1T_THREADS, 2) quant_append_tile_kernel(
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
    const int32_t* __restrict__ slots, int T, int Hkv, uint8_t* __restrict__ pool, int64_t num_blocks,
    int nunits, unsigned long long* span) {
  // A K2 launched behind this kernel with programmatic serialization may start
  // its prologue now; it waits (griddepcontrol.wait) before reading any page.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (span && threadIdx.x == 0) atomicMin(span, global_ns());
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* const smem = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);  // TMA boxes: 128-byte aligned
  uint8_t* const stage = smem;
  uint8_t* const imgs = smem + K1T_STAGES * K1T_STAGE;
  uint64_t* const full = reinterpret_cast<uint64_t*>(imgs + K1T_IMG);
  uint64_t* const empty = full + K1T_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
    for (int s = 0; s < K1T_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // one arrive per consumer warp of the team
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // ---- producer
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();  // the rows are read once
    int i = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
      const int s = i % K1T_STAGES, r = i / K1T_STAGES;
      if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
      const int tt = u / Hkv, h = u - tt * Hkv;
      mbar_arrive_expect_tx(&full[s], K1T_STAGE);  // full boxes, OOB elements included
      tma_load_2d(stage + s * K1T_STAGE, &tmk, h * HD, tt * 16, &full[s], pol);
      tma_load_2d(stage + s * K1T_STAGE + K1T_STAGE / 2, &tmv, h * HD, tt * 16, &full[s], pol);
    }
    return;
  }

  // ---- consumers
  const int ct = threadIdx.x - 32, team = ct >> 6, tt_ = ct & 63;
  const int pp = tt_ >> 3, j = lane & 7;  // tokens 2pp, 2pp + 1 of the unit; lane j of the group
  const bool issuer = tt_ == 0;
  uint8_t* const my_img = imgs + team * 2 * PAGE;  // + buf * PAGE
  int buf = 0, i = team;
  int u = blockIdx.x + team * gridDim.x;
  UnitSlots cur;
  if (u < nunits) load_slots(slots, T, (u / Hkv) * 16, pp, lane, cur);
  for (; u < nunits; u += K1T_TEAMS * gridDim.x, i += K1T_TEAMS) {
    const int tt = u / Hkv, h = u - tt * Hkv;
    UnitSlots nxt;
    const int un = u + K1T_TEAMS * gridDim.x;
    if (un < nunits) load_slots(slots, T, (un / Hkv) * 16, pp, lane, nxt);  // in flight through this unit
    const int s = i % K1T_STAGES;
    mbar_wait(&full[s], (i / K1T_STAGES) & 1);
    uint4 raw[2][2][2];  // [token][K|V][lo|hi 16 B]; tokens past T were zero-filled by the TMA
    const uint8_t* sb = stage + s * K1T_STAGE + 32 * j;
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
      for (int kv = 0; kv < 2; ++kv) {
        const uint8_t* rp = sb + kv * (K1T_STAGE / 2) + (2 * pp + i2) * (HD * 2);
        raw[i2][kv][0] = lds128(rp);
        raw[i2][kv][1] = lds128(rp + 16);
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // Whole-page test (every warp alike): 16 in-range tokens with slots blk*16 + 0..15.
    const int first = __shfl_sync(FULL, cur.s16, 0);
    const bool whole = __all_sync(FULL, lane >= 16 || (cur.s16 >= 0 && cur.s16 == first + lane &&
                                                       (first & 15) == 0 && (first >> 4) < num_blocks));
    GroupCodes g;
    quant_group<KVD>(raw, lane, j, g);
    if (whole) {
      const uint32_t img_s = smem_u32(my_img + buf * PAGE);
      write_image(img_s, pp, j, g);
      // generic-proxy smem writes -> visible to the bulk copy (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // The issuer first waits until its earlier stores have read their images
      // (the one from this buffer was issued two units ago); past the barrier
      // the team may refill the other buffer.
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync %0, 64;" ::"r"(1 + team) : "memory");
      if (issuer) {
        uint8_t* dst = pool + ((int64_t)(first >> 4) * Hkv + h) * PAGE;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(img_s), "n"(PAGE)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      buf ^= 1;
    } else {
      store_scattered(pool, num_blocks, Hkv, h, cur.slot, j, j == 0, g);
    }
    cur = nxt;
  }
  // the images must stay valid until the bulk copies have read them
  if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  if (span) {  // kvq_profile_next_append: the consumers finish last; CTA end = all teams done
    asm volatile("bar.sync 5, 256;" ::: "memory");
    if (ct == 0) atomicMax(span + 1, global_ns());
  }
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
__device__ __forceinline__ void quant_row(const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                                          int64_t k_stride, int64_t v_stride, const int32_t* __restrict__ slots,
                                          int T, int Hkv, uint8_t* __restrict__ pool, int64_t num_blocks) {
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

template <int KVD>
__global__ void __launch_bounds__(K1R_WARPS * 32) quant_append_rows_kernel(
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int64_t k_stride,
    int64_t v_stride, const int32_t* __restrict__ slots, int T, int Hkv,
    uint8_t* __restrict__ pool, int64_t num_blocks, unsigned long long* span) {
  // A K2 launched behind this kernel with programmatic serialization may start
  // its prologue now; it waits (griddepcontrol.wait) before reading any page.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (span) {  // kvq_profile_next_append: CTA start, and CTA end once every warp is done
    if (threadIdx.x == 0) atomicMin(span, global_ns());
    quant_row<KVD>(k, v, k_stride, v_stride, slots, T, Hkv, pool, num_blocks);
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(span + 1, global_ns());
    return;
  }
  quant_row<KVD>(k, v, k_stride, v_stride, slots, T, Hkv, pool, num_blocks);
}

unsigned read_and_clear_dev_err_append() { return read_and_clear_dev_err_tu(); }

}  // namespace kvq

using namespace kvq_abi;

extern "C" {

// kvq_profile_next_append: one-shot span pointer for this host thread's next K1 launch.
static thread_local unsigned long long* t_next_append_span = nullptr;

int kvq_profile_next_append(uint64_t* span) {
  if (span && !aligned(span, 8)) return fail(KVQ_EINVAL, "profile_next_append: span must be 8-byte aligned");
  t_next_append_span = reinterpret_cast<unsigned long long*>(span);
  return KVQ_OK;
}

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
  if ((int64_t)T * Hkv > INT32_MAX / 2) return fail(KVQ_EINVAL, "quant_append: too many (token, head) rows");
  auto st = static_cast<cudaStream_t>(stream);
  unsigned long long* const span = t_next_append_span;
  t_next_append_span = nullptr;
  // Same (max-shared) L1/smem carveout as K2 so a decode step never pays an
  // SM reconfiguration between the append and the attention kernel.
  static const bool carve = [] {
    const void* fns[] = {(const void*)kvq::quant_append_tile_kernel<KVQ_INT8>,
                         (const void*)kvq::quant_append_tile_kernel<KVQ_FP8_E4M3>,
                         (const void*)kvq::quant_append_rows_kernel<KVQ_INT8>,
                         (const void*)kvq::quant_append_rows_kernel<KVQ_FP8_E4M3>};
    for (const void* f : fns)
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    for (int i = 0; i < 2; ++i)
      cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, kvq::K1T_SMEM);
    return true;
  }();
  (void)carve;
  const auto kp = static_cast<const __nv_bfloat16*>(k);
  const auto vp = static_cast<const __nv_bfloat16*>(v);
  auto* pp = static_cast<uint8_t*>(pool);
  const bool rows16 = aligned(k, 16) && aligned(v, 16) && (k_token_stride % 8) == 0 && (v_token_stride % 8) == 0;
  // Tile kernel: the rows are fetched by TMA tensor loads through two maps over
  // the [T][Hkv * 128] K and V views (box = 16 tokens x one head).  Decode-
  // shaped batches (latency-bound), rows only 8-byte aligned, and views the TMA
  // cannot describe (e.g. a token stride below the row length) take the
  // one-warp-per-row kernel instead.
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  CUtensorMap maps[2];
  bool tile = (int64_t)T * Hkv > kvq::K1_ROWS_MAX && rows16 && encode != nullptr;
  for (int m = 0; m < 2 && tile; ++m) {
    const cuuint64_t dims[2] = {(cuuint64_t)kvq::HD * Hkv, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)(m ? v_token_stride : k_token_stride) * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kvq::HD, 16};
    const cuuint32_t estr[2] = {1, 1};
    tile = encode(&maps[m], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(m ? v : k), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (!tile) {
    const unsigned nblk = (unsigned)((T * Hkv + kvq::K1R_WARPS - 1) / kvq::K1R_WARPS);
    if (kv_dtype == KVQ_INT8)
      kvq::quant_append_rows_kernel<KVQ_INT8><<<nblk, kvq::K1R_WARPS * 32, 0, st>>>(
          kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks, span);
    else
      kvq::quant_append_rows_kernel<KVQ_FP8_E4M3><<<nblk, kvq::K1R_WARPS * 32, 0, st>>>(
          kp, vp, k_token_stride, v_token_stride, slot_mapping, T, Hkv, pp, num_blocks, span);
    return check_launch("quant_append");
  }
  const int64_t nunits = (int64_t)((T + 15) / 16) * Hkv;
  if (nunits > INT32_MAX / 2) return fail(KVQ_EINVAL, "quant_append: too many tokens");
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(nunits, (int64_t)sms * 2);
  if (kv_dtype == KVQ_INT8)
    kvq::quant_append_tile_kernel<KVQ_INT8><<<grid, kvq::K1T_THREADS, kvq::K1T_SMEM, st>>>(
        maps[0], maps[1], slot_mapping, T, Hkv, pp, num_blocks, (int)nunits, span);
  else
    kvq::quant_append_tile_kernel<KVQ_FP8_E4M3><<<grid, kvq::K1T_THREADS, kvq::K1T_SMEM, st>>>(
        maps[0], maps[1], slot_mapping, T, Hkv, pp, num_blocks, (int)nunits, span);
  return check_launch("quant_append");
}

}  // extern "C"
