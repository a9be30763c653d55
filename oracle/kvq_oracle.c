/*
 * kvq_oracle.c -- CPU restatement of the quantized paged-KV decode path.
 * TEST INFRASTRUCTURE ONLY (see kvq_oracle.h for provenance and the
 * "parity unpinned" note).  Build: oracle/Makefile (-O3 -ffp-contract=off
 * -pthread).
 *
 * Semantics follow PAPER.md:471-474 ("quantized from FP16/BF16 to lower
 * precision (typically INT8 ... or FP8) during the generation ... dynamic
 * scaling") and BASELINE.json.north_star ("INT8 or FP8-E4M3 with per-token,
 * per-head scales"; "GQA with split-KV and an online-softmax merge"), under the
 * rounding contract of DESIGN.md §3:
 *
 *   amax  = max_d |x_d|                        (fp32, NaN-ignoring fmaxf)
 *   scale = amax / QMAX                        (IEEE fp32 division, RN)
 *   inv   = amax > 0 ? QMAX / amax : 0         (IEEE fp32 division, RN)
 *   y_d   = x_d * inv                          (fp32 multiply, RN, no FMA)
 *   INT8: code = clamp(rint_even(y), -127, 127), NaN -> 0   (QMAX = 127)
 *   FP8 : code = e4m3 RNE with satfinite (|y| >= 448 -> +-448, NaN -> 0x7F)
 *                                                            (QMAX = 448)
 */
#include "kvq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint8_t kvqo_f32_to_e4m3_satfinite(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint8_t sign = (uint8_t)((u >> 24) & 0x80u);
  if (isnan(x)) return 0x7F; /* cvt.rn.satfinite: NaN -> canonical NaN */
  const float a = fabsf(x);
  if (a >= 448.0f) return sign | 0x7E; /* satfinite (also +-inf) */
  if (a < 0.015625f) {                 /* below 2^-6: subnormal grid m * 2^-9 */
    const float m = rintf(a * 512.0f); /* exact scaling; RNE */
    return sign | (uint8_t)m;          /* m == 8 encodes 2^-6 = 0x08 */
  }
  int e;
  (void)frexpf(a, &e); /* a = f * 2^e, f in [0.5, 1) */
  e -= 1;              /* a = mant * 2^e, mant in [1, 2) */
  const float mant = ldexpf(a, -e);
  float m = rintf((mant - 1.0f) * 8.0f); /* exact; RNE */
  if (m == 8.0f) {
    m = 0.0f;
    e += 1;
  }
  return sign | (uint8_t)(((e + 7) << 3) | (int)m);
}

float kvqo_e4m3_to_f32(uint8_t c) {
  const int s = c >> 7, ex = (c >> 3) & 0xF, m = c & 7;
  float v;
  if (ex == 0xF && m == 7) return NAN;
  if (ex == 0)
    v = ldexpf((float)m, -9);
  else
    v = ldexpf(1.0f + (float)m / 8.0f, ex - 7);
  return s ? -v : v;
}

int8_t kvqo_f32_to_int8_sat(float y) {
  /* == clamp(cvt.rni.s32.f32(y), -127, 127): NaN -> 0, +-inf saturate. */
  if (isnan(y)) return 0;
  const float r = rintf(y);
  if (r >= 127.0f) return 127;
  if (r <= -127.0f) return -127;
  return (int8_t)r;
}

static void quantize_row(const uint16_t* x, int kv_dtype, uint8_t* codes, float* scale_out) {
  const float qmax = kv_dtype == KVQO_FP8_E4M3 ? 448.0f : 127.0f;
  float xf[KVQO_HEAD_DIM];
  float amax = 0.0f;
  for (int d = 0; d < KVQO_HEAD_DIM; ++d) {
    xf[d] = bf16_to_f32(x[d]);
    amax = fmaxf(amax, fabsf(xf[d]));
  }
  const float scale = amax / qmax;
  const float inv = amax > 0.0f ? qmax / amax : 0.0f;
  for (int d = 0; d < KVQO_HEAD_DIM; ++d) {
    const float y = xf[d] * inv;
    codes[d] = kv_dtype == KVQO_FP8_E4M3 ? kvqo_f32_to_e4m3_satfinite(y)
                                         : (uint8_t)kvqo_f32_to_int8_sat(y);
  }
  *scale_out = scale;
}

void kvqo_quantize_rows(const uint16_t* x, int64_t rows, int kv_dtype, uint8_t* codes,
                        float* scales) {
  for (int64_t r = 0; r < rows; ++r)
    quantize_row(x + r * KVQO_HEAD_DIM, kv_dtype, codes + r * KVQO_HEAD_DIM, scales + r);
}

/* Page layout.  K: row pair p = t & 7 (tokens p, p+8; 256 B)
 * of 16-byte units; unit (4j + c) ^ ((p & 1) << 2) holds, as 4-byte words,
 * K[p][16c+4j..], K[p+8][16c+4j..], K[p][64+16c+4j..], K[p+8][64+16c+4j..].
 * V: token pairs interleaved -- pair-row
 * p = t/2 holds byte 2d + (t & 1); the 256-byte pair-row is two 128-byte rows
 * R = 2p + (L >= 128) whose chunks are stored at j ^ (R & 7).  Scales: K at
 * 4096 + 4t, V at 4160 + 4t (fp32). */
int kvqo_code_offset(int kv, int token, int d) {
  if (kv == 0) {
    const int p = token & 7, hi_row = token >> 3;
    const int half = d >> 6, dd = d & 63;
    const int c = dd >> 4, j = (dd >> 2) & 3;
    const int unit = (4 * j + c) ^ ((p & 1) << 2);
    return p * 256 + unit * 16 + (2 * half + hi_row) * 4 + (d & 3);
  }
  const int L = 2 * d + (token & 1);
  const int R = 2 * (token >> 1) + (L >> 7);
  const int l = L & 127;
  return 2048 + R * 128 + (((l >> 4) ^ (R & 7)) << 4) + (l & 15);
}

int kvqo_scale_offset(int kv, int token) { return 4096 + kv * 64 + 4 * token; }

void kvqo_quant_append(const uint16_t* k, const uint16_t* v, const int32_t* slot_mapping, int T,
                       int Hkv, int kv_dtype, uint8_t* pool, int64_t num_blocks) {
  for (int t = 0; t < T; ++t) {
    const int32_t slot = slot_mapping[t];
    if (slot < 0) continue;
    const int64_t blk = slot / KVQO_BLOCK;
    const int off = slot % KVQO_BLOCK;
    if (blk >= num_blocks) abort();
    for (int h = 0; h < Hkv; ++h) {
      uint8_t* page = pool + (blk * Hkv + h) * (int64_t)KVQO_PAGE_BYTES;
      for (int kv = 0; kv < 2; ++kv) {
        const uint16_t* src = (kv ? v : k) + ((int64_t)t * Hkv + h) * KVQO_HEAD_DIM;
        uint8_t codes[KVQO_HEAD_DIM];
        float scale;
        quantize_row(src, kv_dtype, codes, &scale);
        for (int d = 0; d < KVQO_HEAD_DIM; ++d) page[kvqo_code_offset(kv, off, d)] = codes[d];
        memcpy(page + kvqo_scale_offset(kv, off), &scale, 4);
      }
    }
  }
}

void kvqo_unpack_pool(const uint8_t* pool, int64_t num_blocks, int Hkv, uint8_t* codes,
                      float* scales) {
  for (int64_t p = 0; p < num_blocks * Hkv; ++p) {
    const uint8_t* page = pool + p * KVQO_PAGE_BYTES;
    for (int kv = 0; kv < 2; ++kv)
      for (int t = 0; t < KVQO_BLOCK; ++t) {
        uint8_t* row = codes + ((p * 2 + kv) * KVQO_BLOCK + t) * KVQO_HEAD_DIM;
        for (int d = 0; d < KVQO_HEAD_DIM; ++d) row[d] = page[kvqo_code_offset(kv, t, d)];
        memcpy(scales + (p * 2 + kv) * KVQO_BLOCK + t, page + kvqo_scale_offset(kv, t), 4);
      }
  }
}

void kvqo_pack_pool(const uint8_t* codes, const float* scales, int64_t num_blocks, int Hkv,
                    uint8_t* pool) {
  for (int64_t p = 0; p < num_blocks * Hkv; ++p) {
    uint8_t* page = pool + p * KVQO_PAGE_BYTES;
    for (int kv = 0; kv < 2; ++kv)
      for (int t = 0; t < KVQO_BLOCK; ++t) {
        const uint8_t* row = codes + ((p * 2 + kv) * KVQO_BLOCK + t) * KVQO_HEAD_DIM;
        for (int d = 0; d < KVQO_HEAD_DIM; ++d) page[kvqo_code_offset(kv, t, d)] = row[d];
        memcpy(page + kvqo_scale_offset(kv, t), scales + (p * 2 + kv) * KVQO_BLOCK + t, 4);
      }
  }
}

int kvqo_num_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* Dequantized value lookup tables: deq = (float)code * scale in fp32. */
static float code_value(uint8_t c, int kv_dtype) {
  return kv_dtype == KVQO_FP8_E4M3 ? kvqo_e4m3_to_f32(c) : (float)(int8_t)c;
}

typedef struct {
  const uint16_t* q;
  const uint8_t* pool;
  const int32_t* block_table;
  const int32_t* seq_lens;
  int B, Hq, Hkv, max_blocks, g;
  float sm_scale;
  float* out;
  float* lse;
  const float* lut;
  int64_t next; /* work counter (atomic) */
} attn_job;

static int koff[KVQO_BLOCK][KVQO_HEAD_DIM], voff[KVQO_BLOCK][KVQO_HEAD_DIM];
static pthread_once_t off_once = PTHREAD_ONCE_INIT;
static void init_offsets(void) {
  for (int t = 0; t < KVQO_BLOCK; ++t)
    for (int d = 0; d < KVQO_HEAD_DIM; ++d) {
      koff[t][d] = kvqo_code_offset(0, t, d);
      voff[t][d] = kvqo_code_offset(1, t, d);
    }
}

/* One (sequence, kv-head) pair: exact two-pass softmax in fp64 over the fp32
 * dequantized K/V (deq = (float)code * scale). */
static void attn_one(const attn_job* j, int64_t bh) {
  const int g = j->g, Hq = j->Hq, Hkv = j->Hkv;
  const int b = (int)(bh / Hkv), h = (int)(bh % Hkv);
  const int L = j->seq_lens[b];
  double qd[16][KVQO_HEAD_DIM];
  for (int i = 0; i < g; ++i)
    for (int d = 0; d < KVQO_HEAD_DIM; ++d)
      qd[i][d] = bf16_to_f32(j->q[((int64_t)b * Hq + h * g + i) * KVQO_HEAD_DIM + d]);
  double* s = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1) * g);
  double m[16], l[16], acc[16][KVQO_HEAD_DIM];
  for (int i = 0; i < g; ++i) m[i] = -INFINITY;
  for (int t = 0; t < L; ++t) {
    const int32_t blk = j->block_table[(int64_t)b * j->max_blocks + t / KVQO_BLOCK];
    const uint8_t* page = j->pool + ((int64_t)blk * Hkv + h) * KVQO_PAGE_BYTES;
    const int o = t % KVQO_BLOCK;
    float ks;
    memcpy(&ks, page + kvqo_scale_offset(0, o), 4);
    float kd[KVQO_HEAD_DIM];
    for (int d = 0; d < KVQO_HEAD_DIM; ++d) kd[d] = j->lut[page[koff[o][d]]] * ks;
    for (int i = 0; i < g; ++i) {
      double dot = 0.0;
      for (int d = 0; d < KVQO_HEAD_DIM; ++d) dot += qd[i][d] * (double)kd[d];
      const double sv = dot * (double)j->sm_scale;
      s[(int64_t)t * g + i] = sv;
      if (sv > m[i]) m[i] = sv;
    }
  }
  for (int i = 0; i < g; ++i) {
    l[i] = 0.0;
    for (int d = 0; d < KVQO_HEAD_DIM; ++d) acc[i][d] = 0.0;
  }
  for (int t = 0; t < L; ++t) {
    const int32_t blk = j->block_table[(int64_t)b * j->max_blocks + t / KVQO_BLOCK];
    const uint8_t* page = j->pool + ((int64_t)blk * Hkv + h) * KVQO_PAGE_BYTES;
    const int o = t % KVQO_BLOCK;
    float vs;
    memcpy(&vs, page + kvqo_scale_offset(1, o), 4);
    float vd[KVQO_HEAD_DIM];
    for (int d = 0; d < KVQO_HEAD_DIM; ++d) vd[d] = j->lut[page[voff[o][d]]] * vs;
    for (int i = 0; i < g; ++i) {
      const double p = exp(s[(int64_t)t * g + i] - m[i]);
      l[i] += p;
      for (int d = 0; d < KVQO_HEAD_DIM; ++d) acc[i][d] += p * (double)vd[d];
    }
  }
  for (int i = 0; i < g; ++i) {
    float* o = j->out + ((int64_t)b * Hq + h * g + i) * KVQO_HEAD_DIM;
    for (int d = 0; d < KVQO_HEAD_DIM; ++d) o[d] = L > 0 ? (float)(acc[i][d] / l[i]) : 0.0f;
    if (j->lse) j->lse[(int64_t)b * Hq + h * g + i] = L > 0 ? (float)(m[i] + log(l[i])) : -INFINITY;
  }
  free(s);
}

static void* attn_worker(void* arg) {
  attn_job* j = (attn_job*)arg;
  const int64_t n = (int64_t)j->B * j->Hkv;
  for (;;) {
    const int64_t bh = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (bh >= n) break;
    attn_one(j, bh);
  }
  return NULL;
}

void kvqo_decode_attn(const uint16_t* q, const uint8_t* pool, const int32_t* block_table,
                      const int32_t* seq_lens, int B, int Hq, int Hkv, int max_blocks,
                      int kv_dtype, float sm_scale, float* out, float* lse, int nthreads) {
  if (Hkv <= 0 || Hq % Hkv != 0 || Hq / Hkv > 16) abort();
  pthread_once(&off_once, init_offsets);
  float lut[256];
  for (int c = 0; c < 256; ++c) lut[c] = code_value((uint8_t)c, kv_dtype);
  attn_job job = {q, pool, block_table, seq_lens, B, Hq, Hkv, max_blocks, Hq / Hkv,
                  sm_scale, out, lse, lut, 0};
  if (nthreads <= 0) nthreads = kvqo_num_threads();
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, attn_worker, &job);
  attn_worker(&job);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
}
