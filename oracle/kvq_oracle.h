/*
 * kvq_oracle.h -- CPU restatement (TEST INFRASTRUCTURE ONLY) of the quantized
 * paged-KV decode path: quantize-on-append + paged GQA decode attention.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  The product path
 * (paper_2605_29639_b200) never links or calls it.
 *
 * Provenance.  The reference (arxiv/paper_2605_29639, RTP-LLM; servesim) has
 * NO implementation of this path: SPEC.md:8 puts "GPU kernels and attention
 * math ... quantization numerics" out of scope, and PAPER.md:468-477 is ten
 * lines of prose ("On-the-fly Quantization: The Key and Value tensors are
 * quantized from FP16/BF16 to lower precision (typically INT8, INT4 or FP8)
 * during the generation ... dynamic scaling").  This file restates that prose
 * plus BASELINE.json.north_star (per-token, per-head scales; GQA; split-KV;
 * online softmax) under the rounding contract in DESIGN.md §3.
 *
 *   PARITY UNPINNED against the reference: there are no reference golden
 *   vectors for this path.  The restatement is instead pinned by
 *     - contract known-answer tests (tests/golden/kat_*.json),
 *     - two independent FP8 encoders (torch float8_e4m3fn, ml_dtypes),
 *     - a second, numpy restatement (oracle/oracle_np.py),
 *   and the block-lifecycle rules the allocator follows are pinned against
 *   the reference itself (servesim TieredCacheStore traces, tests/golden/).
 *
 * Compile with -ffp-contract=off: the quantizer must perform exactly the fp32
 * operations of the contract (no FMA contraction), so codes are bit-exact with
 * the CUDA kernel.
 */
#ifndef KVQ_ORACLE_H
#define KVQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { KVQO_INT8 = 0, KVQO_FP8_E4M3 = 1 };
enum { KVQO_HEAD_DIM = 128, KVQO_BLOCK = 16, KVQO_PAGE_BYTES = 4224 };

/* Scalar codecs. */
uint8_t kvqo_f32_to_e4m3_satfinite(float x);
float kvqo_e4m3_to_f32(uint8_t c);
int8_t kvqo_f32_to_int8_sat(float y);

/* Quantize `rows` rows of 128 bf16 values (raw uint16 bits).
 * codes[rows*128], scales[rows]. */
void kvqo_quantize_rows(const uint16_t* x, int64_t rows, int kv_dtype, uint8_t* codes,
                        float* scales);

/* Physical page layout: byte offset of logical element
 * (kv, token, d) inside one 4224-byte (block, head) page. kv: 0 = K, 1 = V. */
int kvqo_code_offset(int kv, int token, int d);
int kvqo_scale_offset(int kv, int token);

/* quantize-on-append: scatter T new tokens into pool[num_blocks][Hkv][4224].
 * slot_mapping[t] = block*16 + offset; negative slots are skipped. */
void kvqo_quant_append(const uint16_t* k, const uint16_t* v, const int32_t* slot_mapping, int T,
                       int Hkv, int kv_dtype, uint8_t* pool, int64_t num_blocks);

/* Unpack the whole pool to logical codes [NB][Hkv][2][16][128] and scales
 * [NB][Hkv][2][16] (pack is the inverse). */
void kvqo_unpack_pool(const uint8_t* pool, int64_t num_blocks, int Hkv, uint8_t* codes,
                      float* scales);
void kvqo_pack_pool(const uint8_t* codes, const float* scales, int64_t num_blocks, int Hkv,
                    uint8_t* pool);

/* Paged GQA decode attention over the quantized pool (dequantize in fp32,
 * accumulate in fp64).  q: bf16 [B][Hq][128]; out: fp32 [B][Hq][128];
 * lse (optional, may be NULL): fp32 natural-log LSE of the scaled scores
 * [B][Hq].  seq_lens[b] == 0 gives out = 0.  nthreads <= 0: all cores. */
void kvqo_decode_attn(const uint16_t* q, const uint8_t* pool, const int32_t* block_table,
                      const int32_t* seq_lens, int B, int Hq, int Hkv, int max_blocks,
                      int kv_dtype, float sm_scale, float* out, float* lse, int nthreads);

int kvqo_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
