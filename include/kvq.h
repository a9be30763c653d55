/*
 * kvq.h -- C ABI of the B200 quantized paged-KV decode path
 * (libkvq.so, built from paper_2605_29639_b200/csrc/ for sm_100a).
 *
 * This is the drop-in boundary.  Plain pointers, sizes and a CUDA stream
 * handle passed as `void*` (a cudaStream_t / CUstream); no torch types.  The
 * library never allocates, frees, synchronises or copies host<->device, so
 * every entry point is stream-ordered and CUDA-graph capturable.  The caller
 * owns every buffer, including the workspace.
 *
 * Reference interfaces replaced (arxiv/paper_2605_29639 / servesim; the
 * reference models this path only as scalars):
 *   kvq_quant_append   <- the GPU-tier KV write of an uncached suffix,
 *                         simulator.py:384-396 (store.insert(h, GPU,
 *                         _block_bytes(), ...)), sized by
 *                         CostModel.kv_bytes_per_token, cost.py:41,73-74;
 *                         semantics from PAPER.md:471-475.
 *   kvq_decode_attn    <- CostModel.decode_step_us, cost.py:62-65, called
 *                         from ClusterSim._decode_dur / _on_decode_step,
 *                         simulator.py:499-517.
 *   kvq_copy_blocks    <- the "partial block is exclusive" rule,
 *                         tiered_cache.py:355-363 (copy-on-write of a shared
 *                         partial tail block on fork).
 *   kvq_page_bytes     <- ClusterSim._block_bytes, simulator.py:178-179.
 *   kvq_block_hashes   <- generate_hash_keys, blocks.py:51-69 (prefix-reuse
 *                         identity of quantized pages).
 *
 * Error convention (mirrors the reference's ValueError / RuntimeError split,
 * errors.py:6-33): 0 = ok; KVQ_EINVAL (shape / dtype / alignment);
 * KVQ_EUNSUPPORTED (not sm_100, unknown kv dtype); KVQ_ECUDA (launch error).
 * kvq_last_error() returns a thread-local message for the last failure.
 */
#ifndef KVQ_H
#define KVQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVQ_ABI_VERSION 5 /* 2: peer gather, decode_step (+flags), pipeline submitter, block gather/scatter;
                             3: kvq_check_device_errors, kvq_profile_next_decode;
                             4: kvq_profile_next_append;
                             5: kvq_decode_pages_per_split_rows */
#define KVQ_HEAD_DIM 128  /* d */
#define KVQ_BLOCK_SIZE 16 /* tokens per page */
#define KVQ_PAGE_BYTES 4224 /* one (block, kv head): 2x16x128 codes + 2x16 fp32 scales */

enum kvq_status { KVQ_OK = 0, KVQ_EINVAL = -1, KVQ_EUNSUPPORTED = -2, KVQ_ECUDA = -3 };
enum kvq_kv_dtype { KVQ_INT8 = 0, KVQ_FP8_E4M3 = 1 };
enum kvq_out_dtype { KVQ_OUT_BF16 = 0, KVQ_OUT_F32 = 1 };
enum kvq_out_layout { KVQ_OUT_BHD = 0 /* [B][Hq][d] */, KVQ_OUT_HBD = 1 /* [Hq][B][d] */ };

int kvq_version(void);
const char* kvq_last_error(void);
size_t kvq_page_bytes(void);

/* Caller errors the kernels can only see on the device.  The kernels never
 * fault on them: an out-of-range block id is read as block 0, a length past
 * max_blocks * 16 is clamped, a slot past the pool is skipped -- and a bit is
 * set in a device-side error word:
 *   KVQ_DERR_BLOCK_ID  K2 met block_table[b][i] outside [0, num_blocks) among
 *                      a sequence's visible pages;
 *   KVQ_DERR_SEQ_LEN   K2 met seq_lens[b] > max_blocks * 16 or < 0;
 *   KVQ_DERR_SLOT      K1 (or the fused append) met slot >= 0 with
 *                      slot / 16 >= num_blocks (slot < 0 is "skip", not an error).
 * kvq_check_device_errors synchronizes `stream`, reads and clears the word
 * (all kernels of this process on the current device), and returns KVQ_OK, or
 * KVQ_EINVAL with the bits in kvq_last_error() and in *bits (may be NULL).
 * It synchronizes: a validation / debug call, not for the step path.  The
 * oracle abort()s on the same inputs (oracle/kvq_oracle.c). */
enum kvq_device_error { KVQ_DERR_BLOCK_ID = 1, KVQ_DERR_SEQ_LEN = 2, KVQ_DERR_SLOT = 4 };
int kvq_check_device_errors(void* stream, uint32_t* bits);

/* Profiling (bench.py's roofline): the next K2 launch this host thread issues
 * (kvq_decode_attn*, kvq_decode_step*) records its grid span in device memory:
 * span[0] = min over CTAs of the start %globaltimer, span[1] = max end (ns).
 * The caller sets span[0] = UINT64_MAX, span[1] = 0 beforehand.  One-shot; the
 * pointer is a kernel parameter, so a CUDA-graph capture keeps it (one span
 * per captured launch) and the kernel times itself inside a PDL-chained step.
 * NULL cancels a pending request. */
int kvq_profile_next_decode(uint64_t* span);
/* The same for the next K1 launch (kvq_quant_append, or the K1 half of
 * kvq_decode_step*). */
int kvq_profile_next_append(uint64_t* span);

/* Quantize-on-append (K1).  k, v: bf16 [T][Hkv][128] with token strides
 * k_token_stride / v_token_stride (in elements; head stride is 128, rows
 * 8-byte aligned).  slot_mapping[t] = block * 16 + offset; slot < 0 skips
 * token t.  pool: uint8 [num_blocks][Hkv][KVQ_PAGE_BYTES] (16-byte aligned).
 * Per (token, head, K|V) row: amax -> scale = amax/QMAX -> codes
 * (DESIGN.md §3), written into the page layout of DESIGN.md §2. */
int kvq_quant_append(const void* k, const void* v, int64_t k_token_stride,
                     int64_t v_token_stride, const int32_t* slot_mapping, int32_t T,
                     int32_t Hkv, int32_t kv_dtype, void* pool, int64_t num_blocks,
                     void* stream);

/* Workspace for kvq_decode_attn: per-(sequence, kv head) arrival counters
 * (offset 0, round_up(B * Hkv * 4, 256) bytes) used by the fused split-KV
 * combine, then the split partials (fp32 O + LSE).  The counter region must be
 * zero on entry; the kernel leaves it zero again (graph-replay safe).  When a
 * workspace is reused for a larger B * Hkv than the PREVIOUS call's, re-zero
 * the counter prefix: beyond the previous call's counters lie its partials. */
size_t kvq_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t max_splits);

/* Split-KV geometry: pages per split chosen for a workload of `B` sequences,
 * `Hkv` kv heads and `total_pages` pages summed over sequences (pass
 * B * max_blocks when only the bound is known).  Returns pages_per_split >= 1;
 * max_splits = ceil(max_blocks / pages_per_split). */
int32_t kvq_decode_pages_per_split(int32_t B, int32_t Hkv, int64_t total_pages,
                                   int32_t max_blocks);
/* The same for `rows` query rows per kv head ((Hq / Hkv) * q_len; the call
 * above assumes <= 8).  More than 8 rows run the two-n-tile variant, whose
 * split combine costs more per split: equal-length launches of 1-8 waves then
 * get longer splits (C4 at P = 8: 238 -> 192 us).  ABI 5. */
int32_t kvq_decode_pages_per_split_rows(int32_t B, int32_t Hkv, int32_t rows, int64_t total_pages,
                                        int32_t max_blocks);

/* Paged GQA decode attention (K2 + fused split-KV combine).
 *   q:           bf16 [B][Hq][128], batch stride q_batch_stride (elements)
 *   pool:        uint8 [num_blocks][Hkv][KVQ_PAGE_BYTES]
 *   block_table: int32 [B][max_blocks]; seq_lens: int32 [B] (<= 16*max_blocks)
 *   sm_scale:    softmax scale (typically 1/sqrt(128))
 *   out:         bf16 or fp32, layout per out_layout
 * Hq % Hkv == 0 and Hq / Hkv <= 16.  seq_lens[b] == 0 yields zeros. */
int kvq_decode_attn(const void* q, int64_t q_batch_stride, const void* pool, int64_t num_blocks,
                    const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                    int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype, float sm_scale,
                    int32_t pages_per_split, void* workspace, size_t workspace_bytes, void* out,
                    int32_t out_dtype, int32_t out_layout, void* stream);

/* Host-only.  Chained 64-bit keys of the complete `block_size`-token blocks
 * of `tokens[0..n)` (FNV-1a over little-endian 8-byte words, chained from
 * `prev_key`, or from the standard seed when 0): the prefix-reuse identity of
 * quantized pages, same definition as the reference's block keys
 * (blocks.py:29-69).  Returns the number of keys written, or KVQ_EINVAL. */
int64_t kvq_block_hashes(const int64_t* tokens, int64_t n, int32_t block_size, uint64_t prev_key,
                         uint64_t* out);

/* Multi-query variant (speculative scoring / MTP): q_len query
 * tokens per sequence, q: bf16 [B][q_len][Hq][128] (batch stride
 * q_batch_stride, token stride Hq*128), causal within the q_len new tokens:
 * query i sees seq_lens[b] - (q_len - 1 - i) tokens (seq_lens counts all of
 * them).  out: [B*q_len][Hq][d] (KVQ_OUT_BHD) or [Hq][B*q_len][d].  Needs
 * (Hq / Hkv) * q_len <= 16; size the workspace with
 * kvq_decode_workspace_bytes(B, Hq * q_len, Hkv, max_splits).
 * kvq_decode_attn is the q_len == 1 case.  Replaces the ScoreModel forward
 * seam, spec_decode.py:98-107. */
int kvq_decode_attn_mq(const void* q, int64_t q_batch_stride, int32_t q_len, const void* pool,
                       int64_t num_blocks, const int32_t* block_table, int32_t max_blocks,
                       const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype,
                       float sm_scale, int32_t pages_per_split, void* workspace,
                       size_t workspace_bytes, void* out, int32_t out_dtype, int32_t out_layout,
                       void* stream);

/* Copy whole pages (all kv heads of a block): pairs[2*i] = src block,
 * pairs[2*i+1] = dst block (device int32). */
int kvq_copy_blocks(void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* pairs,
                    int32_t n_pairs, void* stream);
/* PD KV transfer (replaces the payload of _migrate_kv,
 * simulator.py:485-497): gather blocks block_ids[0..n) of the pool (all kv
 * heads) into a packed uint8 [n][Hkv][KVQ_PAGE_BYTES] buffer -- the wire
 * format -- and scatter such a buffer into the receiver's blocks. */
int kvq_gather_blocks(const void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* block_ids,
                      int32_t n, void* out, void* stream);
int kvq_scatter_blocks(void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* block_ids,
                       int32_t n, const void* in, void* stream);

/* ---- KV-head sharding with the output all-gather fused into K2 ----------
 * Replaces the separate all-gather of the sharded decode (the
 * reference models TP only as cost parameters).  Every
 * rank owns one "symmetric" buffer per output slot: a control block
 * (KVQ_PEER_CTL_BYTES) followed by the global bf16 output [Hq][B][128].
 * Each rank maps every peer's buffer (CUDA IPC over NVLink / NVSwitch), and
 * its K2 writes each finished output row straight into all P copies, then
 * bumps a "done" counter in every peer's control block.  The last CTA of the
 * grid waits until all P ranks' rows of this use have landed, so when K2
 * completes on a rank, its global output is complete: no collective launch,
 * and the transfer overlaps the attention tile by tile.  Slot reuse is safe:
 * K2 releases the slot's previous use at start (stream order guarantees that
 * use was consumed), and a writer waits for every rank's release before
 * overwriting.  All protocol state lives in device memory, so the launch is
 * CUDA-graph capturable.  Spins time out after ~10 s and set the error word
 * of the local control block instead of hanging. */
#define KVQ_MAX_PEERS 8
#define KVQ_PEER_CTL_BYTES 256 /* uint32 words: [0] done [1] uses [2] error [3] arrivals [32+i] free[i] */
#define KVQ_IPC_HANDLE_BYTES 64
typedef struct kvq_peer_out {
  int32_t n_peers;          /* P, 2..KVQ_MAX_PEERS */
  int32_t rank;             /* this rank's index in out[] / ctl[] */
  int32_t head_offset;      /* first global q head this rank computes */
  int32_t batch_global;     /* B of the global [Hq][B][128] output */
  const int32_t* seq_map;   /* device int32 [B_local]: local sequence -> global row (NULL = identity) */
  uint32_t writers_per_use; /* sum over ranks of B_r * Hkv_r: done increments per use */
  uint32_t reserved;
  void* out[KVQ_MAX_PEERS]; /* rank i's global output of this slot (mapped into this process) */
  void* ctl[KVQ_MAX_PEERS]; /* rank i's control block of this slot */
} kvq_peer_out;

/* kvq_decode_attn with the gather fused: same arguments, but the output goes
 * to peer->out[0..P) (bf16, [Hq_global][batch_global][128], rows of heads
 * head_offset .. head_offset + Hq) instead of an `out` pointer.  q_len == 1. */
int kvq_decode_attn_peer(const void* q, int64_t q_batch_stride, const void* pool, int64_t num_blocks,
                         const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                         int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype, float sm_scale,
                         int32_t pages_per_split, void* workspace, size_t workspace_bytes,
                         const kvq_peer_out* peer, void* stream);

/* One decode step in one call: kvq_quant_append of the T new rows, then
 * kvq_decode_attn (or, with `peer`, kvq_decode_attn_peer; `out` is then
 * ignored and must be bf16 head-major).  K2 is launched with programmatic
 * stream serialization right behind K1 (PDL): its launch and prologue (q,
 * block-table and barrier setup) overlap K1, and it waits for K1
 * (griddepcontrol.wait) before reading any page.  Valid because K1 writes
 * only pages; q, block_table and seq_lens must be ready when the call is
 * enqueued, as for any stream-ordered call.  With flags & KVQ_STEP_APPEND_TAIL_ONLY
 * the caller promises that, for every sequence K2 attends, the appended rows lie
 * in its last page (a decode step's new token; rows of sequences K2 does not
 * attend, e.g. chunked-prefill chunks, may go anywhere): K2 then streams every
 * other page while K1 runs and waits for K1 only before each last page.
 * Replaces the decode-step pair the reference charges as one constant,
 * simulator.py:499-517. */
#define KVQ_STEP_APPEND_TAIL_ONLY 1
/* flags & KVQ_STEP_FUSED_APPEND: no K1 launch.  The caller promises T == B and
 * that row b of k / v is sequence b's newest token: position seq_lens[b] - 1,
 * slot_mapping[b] its slot in block_table[b] (a plain decode step).  The K2 CTA
 * holding that page quantizes the row (K1's rounding contract, bit-identical),
 * writes it to the pool and attends over it.  q_len == 1, no peer gather. */
#define KVQ_STEP_FUSED_APPEND 2
int kvq_decode_step(const void* k, const void* v, int64_t k_token_stride, int64_t v_token_stride,
                    const int32_t* slot_mapping, int32_t T, const void* q, int64_t q_batch_stride,
                    void* pool, int64_t num_blocks, const int32_t* block_table, int32_t max_blocks,
                    const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype,
                    float sm_scale, int32_t pages_per_split, void* workspace, size_t workspace_bytes,
                    void* out, int32_t out_dtype, int32_t out_layout, const kvq_peer_out* peer,
                    int32_t flags, void* stream);

/* Speculative-decoding verify step: kvq_decode_step with q_len
 * new tokens per sequence -- K1 appends their rows, then the causal
 * multi-query K2 of kvq_decode_attn_mq (q: bf16 [B][q_len][Hq][128]).  The
 * tail-only flag is ignored for q_len > 1 (the new rows may span two pages);
 * no fused gather (peer must be NULL unless q_len == 1). */
int kvq_decode_step_mq(const void* k, const void* v, int64_t k_token_stride, int64_t v_token_stride,
                       const int32_t* slot_mapping, int32_t T, const void* q, int64_t q_batch_stride,
                       int32_t q_len, void* pool, int64_t num_blocks, const int32_t* block_table,
                       int32_t max_blocks, const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv,
                       int32_t kv_dtype, float sm_scale, int32_t pages_per_split, void* workspace,
                       size_t workspace_bytes, void* out, int32_t out_dtype, int32_t out_layout,
                       const kvq_peer_out* peer, int32_t flags, void* stream);

/* Host-side step submission of a double-buffered serving pipeline, in one
 * native call instead of ~10 runtime calls from the host language: upload the
 * step's packed inputs (pinned host -> device) on `h2d_stream`, run the slot's
 * captured device step (a cudaGraphExec_t holding kvq_decode_step and, when
 * sharded, the gather) on `compute_stream`, download the output on
 * `d2h_stream`, with the three events ordering slot reuse (the caller creates
 * them; `reuse` = the slot ran before).  The session runtime behind
 * DecodeSession.submit_staged; replaces the per-step host work of the
 * reference's decode loop, simulator.py:499-517. */
typedef struct kvq_pipe_step {
  void* h2d_stream;
  void* compute_stream;
  void* d2h_stream;
  void* graph_exec;
  void* dev_in;
  const void* host_in;
  size_t in_bytes;
  const void* dev_out;
  void* host_out;
  size_t out_bytes;
  void* ev_in_ready;
  void* ev_done;
  void* ev_out_done;
  int32_t reuse;
  int32_t reserved;
} kvq_pipe_step;
int kvq_pipeline_submit(const kvq_pipe_step* step);

/* Symmetric-buffer plumbing (setup time only, not on the step path):
 * allocate `bytes` of zeroed device memory on the current device and return
 * its IPC handle; map a peer's handle into this process; unmap; free. */
int kvq_sym_alloc(size_t bytes, void** ptr, void* ipc_handle);
int kvq_sym_open(const void* ipc_handle, void** ptr);
int kvq_sym_close(void* ptr);
int kvq_sym_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_H */
