// kvq_common.cuh -- shared by the libkvq translation units: constants, the
// page layout, PTX helpers (shared-memory addresses, mbarriers,
// TMA bulk copies, warp MMA, code conversions) and the C-ABI error helpers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <type_traits>

#include "kvq.h"

namespace kvq {

constexpr int HD = 128;
constexpr int BS = 16;
constexpr int PAGE = KVQ_PAGE_BYTES;
constexpr int V_OFF = 2048;
constexpr int KS_OFF = 4096;
constexpr int VS_OFF = 4160;
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// Page layout helpers.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int k_code_off(int tok, int d) {
  // Row pair p = tok & 7 holds tokens p and p + 8 (256 B).  Its 16-byte unit
  // (4j + c) ^ ((p & 1) << 2) is one MMA A-fragment quad:
  //   [K[p][16c+4j..+3], K[p+8][16c+4j..+3], K[p][64+16c+4j..+3], K[p+8][64+16c+4j..+3]]
  const int p = tok & 7, hi_row = tok >> 3;
  const int half = d >> 6, dd = d & 63;
  const int c = dd >> 4, j = (dd >> 2) & 3, e = d & 3;
  const int unit = (4 * j + c) ^ ((p & 1) << 2);
  return p * 256 + unit * 16 + (2 * half + hi_row) * 4 + e;
}
__host__ __device__ __forceinline__ int v_code_off(int tok, int d) {
  const int L = 2 * d + (tok & 1);
  const int R = 2 * (tok >> 1) + (L >> 7);
  const int l = L & 127;
  return V_OFF + R * 128 + (((l >> 4) ^ (R & 7)) << 4) + (l & 15);
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
// PTX helpers: shared-memory addresses, mbarriers, bulk async copy, MMA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "KVQ_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra KVQ_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// The same on 32-bit shared-window addresses (no generic -> shared conversion).
__device__ __forceinline__ void mbar_arrive_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "KVQ_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra KVQ_WAITS_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, uint64_t src, uint32_t bytes, uint32_t bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
template <int OFF>
__device__ __forceinline__ uint4 lds128_at(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(a), "n"(OFF));
  return r;
}
template <int OFF>
__device__ __forceinline__ float lds32f_at(uint32_t a) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(r) : "r"(a), "n"(OFF));
  return r;
}
__device__ __forceinline__ float lds32f(const uint8_t* p) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ float2 lds64f(const uint8_t* p) {
  float2 r;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma16832_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                            uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_s8x4(int a, int b, int c, int d) {
  return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) |
         ((uint32_t)d << 24);
}
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Exact 2^k for integer k (clamped to the normal fp32 range).
__device__ __forceinline__ float pow2i(int k) {
  k = max(-126, min(127, k));
  return __int_as_float((127 + k) << 23);
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Codes of 4 consecutive values of one row (contract): y = x * inv
// (RN, never contracted); INT8 rint_even + clamp (NaN -> 0), FP8 satfinite RNE.
// Shared by K1's one-warp-per-row kernel and K2's fused append (bit-identical).
template <int KVD>
__device__ __forceinline__ uint32_t quant_codes4(const float (&x)[4], float inv) {
  float y[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) y[e] = __fmul_rn(x[e], inv);
  if constexpr (KVD == KVQ_FP8_E4M3) {
    uint16_t l, h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(l) : "f"(y[1]), "f"(y[0]));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(y[3]), "f"(y[2]));
    return (uint32_t)l | ((uint32_t)h << 16);
  } else {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = max(-127, min(127, __float2int_rn(y[e])));  // NaN -> 0, saturating
      word |= ((uint32_t)(c & 0xff)) << (8 * e);
    }
    return word;
  }
}

// 8-bit codes -> two f16x2 registers (exact for every INT8 / E4M3 code).
// Input bytes (b0, b1, b2, b3) -> lo = (b0, b1), hi = (b2, b3).  With
// BIASED (INT8 only) the values are code + 1152 and the caller removes the
// bias after the MMA (saves two HSUB2 per word).
template <int KVD, bool BIASED = false>
__device__ __forceinline__ void codes_to_f16x2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  if constexpr (KVD == KVQ_FP8_E4M3) {
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "cvt.rn.f16x2.e4m3x2 %0, l;\n\tcvt.rn.f16x2.e4m3x2 %1, h;\n}"
        : "=r"(lo), "=r"(hi)
        : "r"(w));
  } else {
    // Offset-binary magic: fp16(0x64XX) = 1024 + XX; XX = code ^ 0x80 = code + 128.
    const uint32_t u = w ^ 0x80808080u;
    asm("prmt.b32 %0, %1, %2, 0x7170;" : "=r"(lo) : "r"(u), "r"(0x64646464u));
    asm("prmt.b32 %0, %1, %2, 0x7372;" : "=r"(hi) : "r"(u), "r"(0x64646464u));
    if (!BIASED) {
      const uint32_t magic = 0x64806480u;  // (1152, 1152)
      asm("sub.f16x2 %0, %0, %1;" : "+r"(lo) : "r"(magic));
      asm("sub.f16x2 %0, %0, %1;" : "+r"(hi) : "r"(magic));
    }
  }
}

// Device-side caller-error word (kvq_check_device_errors): kernels that meet
// an argument they cannot honour (an out-of-range block id, slot or length)
// still do something safe (skip / clamp) but OR a bit in here.  One copy per
// translation unit (no relocatable device code); each TU that sets bits
// exports a reader, read_and_clear_dev_err().
static __device__ unsigned int g_dev_err;
__device__ __forceinline__ void flag_dev_err(unsigned bit) { atomicOr(&g_dev_err, bit); }
static inline unsigned read_and_clear_dev_err_tu() {
  unsigned v = 0;
  const unsigned zero = 0;
  if (cudaMemcpyFromSymbol(&v, g_dev_err, sizeof(v)) != cudaSuccess) return 0x80000000u;
  if (v && cudaMemcpyToSymbol(g_dev_err, &zero, sizeof(zero)) != cudaSuccess) return v | 0x80000000u;
  return v;
}
unsigned read_and_clear_dev_err_append();
unsigned read_and_clear_dev_err_decode();

}  // namespace kvq

// C-ABI error reporting: a thread-local message behind kvq_last_error().
namespace kvq_abi {
extern thread_local char g_err[512];
inline int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
inline int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return KVQ_ECUDA;
  }
  return KVQ_OK;
}
inline int check_device() {
  static std::atomic<unsigned long long> verified{0};  // bit d: device d is sm_100 (checked once)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(KVQ_ECUDA, "cudaGetDevice failed");
  if (dev < 64 && ((verified.load(std::memory_order_relaxed) >> dev) & 1ull)) return KVQ_OK;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return fail(KVQ_EUNSUPPORTED, "libkvq is built for sm_100a (B200) only");
  if (dev < 64) verified.fetch_or(1ull << dev, std::memory_order_relaxed);
  return KVQ_OK;
}
inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
}  // namespace kvq_abi
