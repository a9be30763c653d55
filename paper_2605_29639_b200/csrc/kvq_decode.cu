// kvq_decode.cu -- K2, paged GQA decode attention over the quantized pool:
// TMA bulk page streaming, INT8 / E4M3 QK^T and PV on the tensor cores,
// online softmax, fused split-KV combine; variants for multi-query scoring
// and for the KV-head output gather fused over peer memory.  Entry points:
// kvq_decode_attn{,_mq,_peer}, kvq_decode_step, split geometry, workspace.
#include "kvq_common.cuh"

#include <algorithm>

#include <mutex>
#include <set>
#include <utility>

namespace kvq {

// ---------------------------------------------------------------------------
// K2: paged decode attention.
// ---------------------------------------------------------------------------
struct DecodeParams {
  const __nv_bfloat16* q;
  int64_t q_stride_b;
  const uint8_t* pool;
  int64_t num_blocks;
  const int32_t* block_table;
  int max_blocks;
  const int32_t* seq_lens;
  int B, Hq, Hkv, g;
  int q_len;            // query tokens per sequence (1 = decode; k+1 = speculative scoring)
  int G;                // query rows per kv head = g * q_len (<= 16)
  float sm_scale_log2;  // sm_scale * log2(e)
  int pages_per_split, max_splits;
  float* part_o;    // [B*Hq][max_splits][128]
  float* part_lse;  // [B*Hq][max_splits]   (log2 units)
  int* counters;    // [B*Hkv]
  void* out;
  int out_f32, out_hbd;
  kvq_peer_out peer;    // n_peers == 0: local output only (no fused gather)
  int tail_only;        // behind K1 (PDL): K1's rows lie only in each sequence's last page
  // MODE 3 (kvq_decode_step with KVQ_STEP_FUSED_APPEND): row b of ak / av is
  // sequence b's newest token (position seq_lens[b] - 1, slot aslots[b]); the
  // CTA holding that page quantizes it (K1's contract) instead of a K1 launch.
  const __nv_bfloat16* ak;
  const __nv_bfloat16* av;
  int64_t ak_stride, av_stride;
  const int32_t* aslots;
  // kvq_profile_next_decode: when set, the grid's span (min CTA start, max CTA
  // end, %globaltimer ns) is recorded here; nullptr for every ordinary launch.
  unsigned long long* span;
};

constexpr int NW = 4;  // warps per CTA; every warp streams its own pages
constexpr int THREADS = 32 * NW;

// Per-variant geometry.  NT = n-tiles of 8 query heads (g <= 8 -> 1, g <= 16 -> 2).
template <bool HI>
struct Geo {
  static constexpr int NT = HI ? 2 : 1;
  static constexpr int S = 3;     // ring slots (pages in flight) per warp
  static constexpr int CTAS = 4;  // resident CTAs per SM (regs + smem)
  // g > 8 keeps the Q^T fragments in shared memory (one copy per CTA, read with
  // one conflict-free LDS.64 per k-step) so the live set fits 128 registers.
  static constexpr size_t QSM = HI ? (size_t)NT * 8 * 32 * 8 : 0;  // [nt][k-step pair][lane] uint4
  static constexpr size_t SMEM = (size_t)NW * S * PAGE + QSM + NW * S * sizeof(uint64_t) + 16;
  static constexpr size_t PATCH = 32 * 8 + 16;  // MODE 3: the appended row's codes + scales
  static_assert((size_t)NW * S * PAGE >= (size_t)NW * 16 * HD * 4 + 2 * NW * 16 * 4,
                "merge scratch must fit in the ring");
};
constexpr int CTAS_PER_SM = 4;  // used by the split heuristic (g <= 8 variant)
// Largest log2 softmax weight p = 2^u relative to a row's reference point m (l is fp32).
constexpr float UMAX = 100.0f;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

// ---------------------------------------------------------------------------
// Fused KV-head gather over peer memory (kvq_peer_out, include/kvq.h).
// Control block words (uint32) of one output slot on one rank:
//   DONE  -- rows-written counter, bumped once per finished (sequence, kv head)
//            by the writing CTA of every rank (system-scope release add);
//   USES  -- completed uses of the slot on this rank (local);
//   ERR   -- set when a spin times out;
//   ARR   -- grid arrival counter of the running K2 (self-resetting);
//   FREE+i -- uses of the slot rank i has released (written by rank i).
// ---------------------------------------------------------------------------
constexpr int CTL_DONE = 0, CTL_USES = 1, CTL_ERR = 2, CTL_ARR = 3, CTL_FREE = 32;
constexpr unsigned long long SPIN_TIMEOUT_NS = 10ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
// Spin until (int)(*w - target) >= 0; on timeout set the error word and give up.
__device__ __noinline__ void spin_until(const uint32_t* w, uint32_t target, uint32_t* err) {
  const unsigned long long t0 = global_ns();
  while ((int)(ld_acquire_sys(w) - target) < 0) {
    if (global_ns() - t0 > SPIN_TIMEOUT_NS) {
      atomicExch(err, 1u);
      return;
    }
    __nanosleep(64);
  }
}
__device__ __forceinline__ uint32_t* peer_ctl(const kvq_peer_out& pe, int r) {
  return reinterpret_cast<uint32_t*>(pe.ctl[r]);
}
// CTA entry (thread 0): this rank has consumed every earlier use of the slot
// (stream order), so release them to every writer.  Idempotent per CTA.
__device__ __forceinline__ void peer_release(const kvq_peer_out& pe) {
  const uint32_t uses = *reinterpret_cast<volatile uint32_t*>(peer_ctl(pe, pe.rank) + CTL_USES);
  for (int r = 0; r < pe.n_peers; ++r) st_release_sys(peer_ctl(pe, r) + CTL_FREE + pe.rank, uses);
}
// Before a CTA's final output stores: every rank must have released the slot's previous use.
__device__ __forceinline__ void peer_acquire(const kvq_peer_out& pe) {
  if (threadIdx.x == 0) {
    uint32_t* mine = peer_ctl(pe, pe.rank);
    const uint32_t uses = *reinterpret_cast<volatile uint32_t*>(mine + CTL_USES);
    for (int r = 0; r < pe.n_peers; ++r) spin_until(mine + CTL_FREE + r, uses, mine + CTL_ERR);
  }
  __syncthreads();
}
// After a CTA's final output stores: publish them (system scope) and count one writer on every rank.
__device__ __forceinline__ void peer_signal(const kvq_peer_out& pe) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < pe.n_peers; ++r) red_add_release_sys(peer_ctl(pe, r) + CTL_DONE, 1u);
}
// CTA exit (thread 0): the last CTA of the grid waits until every rank's rows of
// this use have landed here, then counts the use.  K2 completing == gather done.
__device__ __forceinline__ void peer_arrive(const kvq_peer_out& pe) {
  uint32_t* mine = peer_ctl(pe, pe.rank);
  const uint32_t total = gridDim.x * gridDim.y * gridDim.z;
  uint32_t prev;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(mine + CTL_ARR) : "memory");
  if (prev != total - 1) return;
  mine[CTL_ARR] = 0;
  const uint32_t uses = *reinterpret_cast<volatile uint32_t*>(mine + CTL_USES);
  spin_until(mine + CTL_DONE, (uses + 1) * pe.writers_per_use, mine + CTL_ERR);
  *reinterpret_cast<volatile uint32_t*>(mine + CTL_USES) = uses + 1;
  __threadfence();
}

// Query row j of kv head h (j < G) is query token i = j / g of head h*g + j % g.
// Output rows are query tokens t = b * q_len + i: [T][Hq][d] or head-major [Hq][T][d].
template <bool PEER>
__device__ __forceinline__ void store_out(const DecodeParams& p, int b, int h, int j, int d0,
                                          const float* vals) {
  const int i = j / p.g, head = h * p.g + j % p.g;
  if constexpr (PEER) {  // fused gather: bf16 row into every rank's global [Hq][B][d]
    const int gb = p.peer.seq_map ? __ldg(p.peer.seq_map + b) : b;
    const int64_t grow = (int64_t)(p.peer.head_offset + head) * p.peer.batch_global + gb;
    uint4 w;
    w.x = pack_bf16x2(vals[0], vals[1]);
    w.y = pack_bf16x2(vals[2], vals[3]);
    w.z = pack_bf16x2(vals[4], vals[5]);
    w.w = pack_bf16x2(vals[6], vals[7]);
    for (int r = 0; r < p.peer.n_peers; ++r)
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.peer.out[r]) + grow * HD + d0) = w;
    return;
  }
  const int64_t t = (int64_t)b * p.q_len + i;
  const int64_t row = p.out_hbd ? ((int64_t)head * p.B * p.q_len + t) : (t * p.Hq + head);
  if (p.out_f32) {
    float* o = reinterpret_cast<float*>(p.out) + row * HD + d0;
    *reinterpret_cast<float4*>(o) = make_float4(vals[0], vals[1], vals[2], vals[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(vals[4], vals[5], vals[6], vals[7]);
  } else {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + row * HD + d0;
    uint4 w;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(vals[0], vals[1]);
    __nv_bfloat162 t1 = __floats2bfloat162_rn(vals[2], vals[3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(vals[4], vals[5]);
    __nv_bfloat162 t3 = __floats2bfloat162_rn(vals[6], vals[7]);
    w.x = *reinterpret_cast<uint32_t*>(&t0);
    w.y = *reinterpret_cast<uint32_t*>(&t1);
    w.z = *reinterpret_cast<uint32_t*>(&t2);
    w.w = *reinterpret_cast<uint32_t*>(&t3);
    *reinterpret_cast<uint4*>(o) = w;
  }
}

__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// Per-warp page stream: warp w of the CTA owns pages w, w + NW, w + 2NW, ...
// of the split; page j of the warp lands in slot j % S of the warp's ring.
template <int S>
struct PageStream {
  const int32_t* bt;       // block table row, offset to the split's first page
  uint64_t head_base;      // global address of (block 0, this kv head)
  uint32_t blk_stride;     // Hkv * PAGE (< 2^28)
  int64_t num_blocks;
  int warp, nj;            // nj = pages this warp processes
  uint32_t ring_s;         // this warp's S slots (shared-window address)
  uint32_t full_s;         // this warp's S barriers (shared-window address)
  uint64_t policy;
  int cur, nxt;            // block ids of pages [base, base+32) and [base+32, base+64) (lane-parallel)
  int base;
  int wait_j;              // page whose copy must wait for K1 (griddepcontrol.wait), or -1

  __device__ __forceinline__ int load_ids(int j0, int lane) const {
    const int j = j0 + lane;
    int blk = j < nj ? __ldg(bt + warp + j * NW) : 0;
    if ((unsigned)blk >= (unsigned long long)num_blocks) {  // caller error: read block 0, report
      flag_dev_err(KVQ_DERR_BLOCK_ID);
      blk = 0;
    }
    return blk;
  }
  __device__ __forceinline__ void init(int lane) {
    base = 0;
    cur = load_ids(0, lane);
    nxt = nj > 32 ? load_ids(32, lane) : 0;
  }
  // Issue the bulk copy of page j into slot s (j >= base, all lanes participate).
  // Addresses: 32-bit shared-window offsets (slot s is a compile-time constant
  // in the unrolled page loop) and one wide multiply-add for the page's global
  // address, so the issue path holds few registers and needs no generic ->
  // shared conversions.
  __device__ __forceinline__ void issue(int j, int lane, int s) {
    if (j >= base + 32) {  // advance the id window (warp-uniform)
      base += 32;
      cur = nxt;
      nxt = load_ids(base + 32, lane);
    }
    const uint32_t blk = (uint32_t)__shfl_sync(FULL, cur, j - base);
    if (lane == 0) {
      if (j == wait_j) asm volatile("griddepcontrol.wait;" ::: "memory");
      const uint32_t bar = full_s + 8 * s;
      mbar_arrive_expect_tx_s(bar, PAGE);
      bulk_g2s_s(ring_s + s * PAGE, head_base + (uint64_t)blk * blk_stride, PAGE, bar, policy);
    }
  }
};

// Thread mapping (lane = 4r + c).  Tensor-core tiles put the 16 tokens of a
// page (QK^T) and 16-row slices of d (PV) on M, the query heads of the GQA
// group on N (8 per n-tile):
//   QK^T : S^T[16 tok x 8 heads]  = K[16 x 128]  . Q^T     (8 k-steps)
//   PV   : O^T[16 d x 8 heads]   += V^T[16 x 16 tok] . P'^T (8 m-tiles)
// K rows are token rows of the page; V is stored token-pair interleaved so a
// 32-bit word holds (d, t0), (d, t1), (d+1, t0), (d+1, t1) -- exactly two
// f16x2 A-fragment registers.  P'^T comes from the S^T accumulator through one
// movmatrix transpose per 8x8 block.  d is permuted inside each k-step /
// m-tile so every thread reads 16-byte chunks (bank-conflict-free given the
// page swizzle).
// MODE: 0 = decode, 1 = multi-query (q_len > 1), 2 = decode with the fused peer gather.
template <int KVD, bool HI, int MODE>
__device__ __forceinline__ void decode_cta(const DecodeParams& p, uint8_t* smem) {
  constexpr bool MQ = MODE == 1, PEER = MODE == 2, FUSED = MODE == 3;
  constexpr int NT = Geo<HI>::NT;
  constexpr int S = Geo<HI>::S;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NW * S * PAGE);
  int* flag = reinterpret_cast<int*>(bars + NW * S);
  uint2* qsm = reinterpret_cast<uint2*>(smem + NW * S * PAGE + NW * S * sizeof(uint64_t) + 16);

  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  // MQ: q_len > 1 query tokens per sequence (compile-time off for plain decode).
  const int g = p.g, G = MQ ? p.G : p.g, qlen = MQ ? p.q_len : 1;
  const int L_in = __ldg(p.seq_lens + b);
  const int L = min(L_in, p.max_blocks * BS);
  if ((L_in > L || L_in < 0) && threadIdx.x == 0 && blockIdx.x == 0) flag_dev_err(KVQ_DERR_SEQ_LEN);
  const int npages = (L + BS - 1) / BS;
  const int nsplit = max(1, (npages + p.pages_per_split - 1) / p.pages_per_split);
  if (split >= nsplit) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (L <= 0) {  // empty sequence: zeros, nothing to combine
    if constexpr (PEER) peer_acquire(p.peer);
    const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int idx = threadIdx.x; idx < G * (HD / 8); idx += THREADS)
      store_out<PEER>(p, b, h, idx / (HD / 8), (idx % (HD / 8)) * 8, z);
    if constexpr (PEER) peer_signal(p.peer);
    return;
  }
  const int pg0 = split * p.pages_per_split;
  const int n = min(npages, pg0 + p.pages_per_split) - pg0;

  // Q loads go out first: their latency overlaps the page-stream setup below.
  uint4 raw[NT][4];
  {
    const int r = lane >> 2, c = lane & 3;
    const __nv_bfloat16* qb = p.q + (int64_t)b * p.q_stride_b;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int j = 8 * nt + r;  // query row: token j / g, head h*g + j % g
      const bool valid = j < G;
      const __nv_bfloat16* src = MQ ? qb + ((int64_t)(j / g) * p.Hq + h * g + j % g) * HD
                                    : qb + (int64_t)(h * g + j) * HD;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = (u < 2 ? 16 * c + 8 * u : 64 + 16 * c + 8 * (u - 2));
        raw[nt][u] = valid ? __ldg(reinterpret_cast<const uint4*>(src + d)) : make_uint4(0, 0, 0, 0);
      }
    }
  }

  PageStream<S> ps;
  ps.bt = p.block_table + (int64_t)b * p.max_blocks + pg0;
  ps.head_base = reinterpret_cast<uint64_t>(p.pool) + (uint64_t)h * PAGE;
  ps.blk_stride = (uint32_t)p.Hkv * PAGE;
  ps.num_blocks = p.num_blocks;
  ps.warp = warp;
  ps.nj = n > warp ? (n - warp + NW - 1) / NW : 0;
  ps.ring_s = smem_u32(smem + warp * S * PAGE);
  ps.full_s = smem_u32(bars + warp * S);
  ps.policy = policy_evict_first();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(bars + warp * S + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  ps.init(lane);
  // Launched behind K1 with programmatic serialization (kvq_decode_step): the
  // prologue above (q, block table, barriers) overlapped K1.  Pages may hold
  // K1's rows, so wait for it here -- or, when the caller promises that K1
  // wrote only each sequence's last page (a decode step's new token), only
  // before that one page's copy, so the rest of the sequence streams while K1
  // runs.  A no-op for an ordinary launch.
  ps.wait_j = -1;
  if (!p.tail_only) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    const int last = npages - 1 - pg0;  // split-local index of the sequence's last page
    if (last >= 0 && last < n && last % NW == warp) ps.wait_j = last / NW;
  }
#pragma unroll 1
  for (int j = 0; j < S && j < ps.nj; ++j) ps.issue(j, lane, j);

  // MODE 3: the warp that owns the sequence's last page quantizes the new row
  // (one warp per row, lane l: d [4l, 4l+4), exactly K1's rows kernel), stores
  // it to the pool for later steps, and keeps it in shared memory to patch into
  // its copy of that page when it lands (the bulk copy may read the old bytes).
  int patch_j = -1, ptok = 0;
  uint32_t* patch = reinterpret_cast<uint32_t*>(smem + NW * S * PAGE + NW * S * sizeof(uint64_t) + 16 +
                                                Geo<HI>::QSM);
  if constexpr (FUSED) {
    const int last = npages - 1 - pg0;
    if (last >= 0 && last < n && last % NW == warp) {
      patch_j = last / NW;
      ptok = (L - 1) & (BS - 1);
      const uint2 kw = __ldg(reinterpret_cast<const uint2*>(p.ak + (int64_t)b * p.ak_stride + h * HD + 4 * lane));
      const uint2 vw = __ldg(reinterpret_cast<const uint2*>(p.av + (int64_t)b * p.av_stride + h * HD + 4 * lane));
      const int aslot = __ldg(p.aslots + b);
      const float xk[4] = {__uint_as_float(kw.x << 16), __uint_as_float(kw.x & 0xffff0000u),
                           __uint_as_float(kw.y << 16), __uint_as_float(kw.y & 0xffff0000u)};
      const float xv[4] = {__uint_as_float(vw.x << 16), __uint_as_float(vw.x & 0xffff0000u),
                           __uint_as_float(vw.y << 16), __uint_as_float(vw.y & 0xffff0000u)};
      float ak = fmaxf(fmaxf(fabsf(xk[0]), fabsf(xk[1])), fmaxf(fabsf(xk[2]), fabsf(xk[3])));
      float av = fmaxf(fmaxf(fabsf(xv[0]), fabsf(xv[1])), fmaxf(fabsf(xv[2]), fabsf(xv[3])));
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        ak = fmaxf(ak, __shfl_xor_sync(FULL, ak, o));
        av = fmaxf(av, __shfl_xor_sync(FULL, av, o));
      }
      const float qmax = KVD == KVQ_FP8_E4M3 ? 448.0f : 127.0f;
      const uint32_t ck = quant_codes4<KVD>(xk, ak > 0.0f ? __fdiv_rn(qmax, ak) : 0.0f);
      const uint32_t cv = quant_codes4<KVD>(xv, av > 0.0f ? __fdiv_rn(qmax, av) : 0.0f);
      const float sc = __fdiv_rn(lane ? av : ak, qmax);  // lanes 0 / 1: K / V scale
      patch[2 * lane] = ck;
      patch[2 * lane + 1] = cv;
      if (lane < 2) patch[64 + lane] = __float_as_uint(sc);
      // An invalid slot is skipped, as K1 does: the row reaches neither the pool
      // nor this CTA's copy of the page (so the output equals K1 + K2's).
      if (aslot < 0 || (aslot >> 4) >= p.num_blocks) {
        patch_j = -1;
        if (aslot >= 0 && lane == 0 && h == 0) flag_dev_err(KVQ_DERR_SLOT);
      } else {
        uint8_t* page = const_cast<uint8_t*>(p.pool) + ((int64_t)(aslot >> 4) * p.Hkv + h) * PAGE;
        const int tok = aslot & 15;
        *reinterpret_cast<uint32_t*>(page + k_code_off(tok, 4 * lane)) = ck;
#pragma unroll
        for (int e = 0; e < 4; ++e) page[v_code_off(tok, 4 * lane + e)] = (uint8_t)(cv >> (8 * e));
        if (lane < 2) *reinterpret_cast<float*>(page + (lane ? VS_OFF : KS_OFF) + 4 * tok) = sc;
      }
      __syncwarp();
    }
  }

  const int r = lane >> 2, c = lane & 3;

  // Q^T B-fragments: n-tile nt holds head 8nt + r; k-step i covers
  // d = base(i) + {0,1} (b0) and base(i) + {2,3} (b1),
  // base(i) = (i < 4 ? 16c + 4i : 64 + 16c + 4(i-4)).
  uint32_t qf[NT][8][2];
  float qscale;
  {
    float amax = 0.0f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t w[4] = {raw[nt][u].x, raw[nt][u].y, raw[nt][u].z, raw[nt][u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          amax = fmaxf(amax, fabsf(__uint_as_float(w[e] << 16)));
          amax = fmaxf(amax, fabsf(__uint_as_float(w[e] & 0xffff0000u)));
        }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, o));
    if constexpr (KVD == KVQ_INT8) {
      // INT8 K feeds the s8 tensor cores directly (no dequantisation at all):
      // q = s1 * (q1 + q2 / 256) with int8 q1, q2, two IMMA per k-step,
      // S = s1 * (acc1 + acc2 / 256).  s1 is a power of two (amax / s1 in
      // [64, 127.5), else one binade up; amax over the GQA group), q1 =
      // floor(q / s1 + 1/2) leaves |residual| <= s1 / 2, so q2 = residual *
      // 256 / s1 fits [-128, 128] (128 clamps to 127: <= s1 / 256, only on
      // exact ties).  The two terms hold every bf16 element >= s1 / 2 (its
      // 8-bit mantissa) EXACTLY; only elements below ~amax / 128 round, by
      // <= s1 / 512.  (Round 1 used q2 = residual * 128 / s1, exact only from
      // s1 up: at queries x40, logit std ~70 log2 units, its score error gave
      // 2.9e-3 on an attention-sink row; with s1 = amax / 127 every element
      // rounded.)
      // IMMA k-step j (32 of d): b0 = q[head][16c + 4j .. +3], b1 =
      // q[head][64 + 16c + 4j .. +3], stored as qf[nt][2j] = term 1 (b0, b1),
      // qf[nt][2j + 1] = term 2.
      int qex = 0;
      if (amax > 0.0f) frexpf(amax, &qex);  // amax = m * 2^qex, m in [0.5, 1)
      if (amax * pow2i(7 - qex) > 127.49f) ++qex;
      const float s1 = amax > 0.0f ? pow2i(qex - 7) : 0.0f;
      const float inv1 = amax > 0.0f ? pow2i(7 - qex) : 0.0f;
      qscale = p.sm_scale_log2 * s1 * 0.00390625f;  // S = s1 * (256 acc1 + acc2) / 256
      // g > 8: the fragments go to shared memory once per CTA; warp 0 makes them
      if (!HI || warp == 0)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            // 4 bf16 at d = (half ? 64 : 0) + 16c + 4jj: raw[nt][2*half + jj/2], words 2*(jj&1), +1
            const uint4 rw = raw[nt][2 * half + (jj >> 1)];
            const uint32_t wa = (jj & 1) ? rw.z : rw.x, wb = (jj & 1) ? rw.w : rw.y;
            const float v[4] = {__uint_as_float(wa << 16), __uint_as_float(wa & 0xffff0000u),
                                __uint_as_float(wb << 16), __uint_as_float(wb & 0xffff0000u)};
            int t1[4], t2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              t1[e] = max(-127, min(127, __float2int_rd(__fadd_rn(v[e] * inv1, 0.5f))));
              const float res = fmaf(-(float)t1[e], s1, v[e]);
              t2[e] = max(-128, min(127, __float2int_rn(res * inv1 * 256.0f)));
            }
            qf[nt][2 * jj][half] = pack_s8x4(t1[0], t1[1], t1[2], t1[3]);
            qf[nt][2 * jj + 1][half] = pack_s8x4(t2[0], t2[1], t2[2], t2[3]);
          }
    } else {
      // Exact power-of-two prescale so max|q'| < 2^14 (fp16-safe); undone in qscale.
      int ex = 0;
      if (amax > 0.0f) frexpf(amax, &ex);
      const float pre = pow2i(14 - ex);
      qscale = p.sm_scale_log2 / pre;
      if (!HI || warp == 0)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w[4] = {raw[nt][u].x, raw[nt][u].y, raw[nt][u].z, raw[nt][u].w};
          uint32_t hw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            hw[e] = pack_half2(__uint_as_float(w[e] << 16) * pre,
                               __uint_as_float(w[e] & 0xffff0000u) * pre);
          const int i0 = 2 * u;  // uint4 u holds d = base(i0) .. base(i0) + 7
          qf[nt][i0][0] = hw[0];
          qf[nt][i0][1] = hw[1];
          qf[nt][i0 + 1][0] = hw[2];
          qf[nt][i0 + 1][1] = hw[3];
        }
    }
  }
  if (HI) {  // publish the (identical in every warp) fragments once per CTA
    if (warp == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 8; i += 2)
          reinterpret_cast<uint4*>(qsm)[(nt * 4 + i / 2) * 32 + lane] =
              make_uint4(qf[nt][i][0], qf[nt][i][1], qf[nt][i + 1][0], qf[nt][i + 1][1]);
    }
    __syncthreads();
  }

  // Per-thread smem offsets inside a page, as bases plus immediates.  K unit i
  // of row pair r = {K[r][16c+4i..], K[r+8][16c+4i..], K[r][64+16c+4i..],
  // K[r+8][64+16c+4i..]} sits at r*256 + 16c + 64*(i ^ (r & 1)) (the XOR is the
  // bank swizzle; every lane must read the same unit per k-step, since the MMA
  // shares the Q^T fragment across rows), so units 0, 2 are kb02 + {0, 128}
  // and units 1, 3 are kb13 + {0, 128}.  V: tokens 2c, 2c+1 at vb0 (d [8r, 8r+8))
  // / vb1 (d [64+8r, ..)); tokens 8+2c, 9+2c 1024 bytes further.
  const uint32_t kb02 = r * 256 + 16 * c + 64 * (r & 1);
  const uint32_t kb13 = r * 256 + 16 * c + 64 * ((r & 1) ^ 1);
  const uint32_t vb0 = V_OFF + (2 * c) * 128 + ((r ^ (2 * c)) << 4);
  const uint32_t vb1 = V_OFF + (2 * c + 1) * 128 + ((r ^ (2 * c + 1)) << 4);
  const uint32_t sb = 4 * r;
  const uint32_t ring_s = ps.ring_s;

  // O^T accumulators: o[nt][mt] : c0 = (d = DA, head 2c), c1 = (DA, 2c+1),
  // c2 = (DA+1, 2c), c3 = (DA+1, 2c+1); DA = (mt < 4 ? 8r + 2mt : 64 + 8r + 2(mt-4)).
  float o[NT][8][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[nt][i][0] = o[nt][i][1] = o[nt][i][2] = o[nt][i][3] = 0.0f;
  // Softmax state for rows 8nt + 2c + e (e = 0, 1); l is this thread's partial sum.
  // Rows past the GQA group (j >= G) start at m = +inf: their scores come out
  // as -inf (p = 0) and never trigger a rescale, with no per-score check.
  float m[NT][2], l[NT][2];
  bool hvalid[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      hvalid[nt][e] = 8 * nt + 2 * c + e < G;
      m[nt][e] = hvalid[nt][e] ? -INFINITY : INFINITY;
      l[nt][e] = 0.0f;
    }
  // Causal visibility of query row j (token i = j / g of q_len): L - (q_len - 1 - i);
  // only evaluated on tail pages, so it costs no registers in the steady state.
  const int L_all = L - (qlen - 1);  // tokens visible to every query row
  auto vis = [&](int nt, int e) { return MQ ? L_all + (8 * nt + 2 * c + e) / g : L; };

  // The page loop is unrolled by the ring depth S, so every slot's shared
  // addresses (page, barrier) are immediates and the slot / phase counters
  // vanish (at the g = 16 variant's 128-register cap they had been spilled
  // and the page addresses rematerialised from SR_TID / SR_CgaCtaId).
  // (Not for the multi-query variant: its larger live set spilled in the
  // unrolled form, q_len = 4 0.42 -> 0.49 ms; there the slot stays a loop
  // variable.)
  constexpr int STEP = MQ ? 1 : S;
  uint32_t phase = 0;
  int slot_rt = 0;  // MQ: the slot of page j0
#pragma unroll 1
  for (int j0 = 0; j0 < ps.nj; j0 += STEP) {
#pragma unroll
  for (int sl = 0; sl < STEP; ++sl) {
    const int j = j0 + sl;
    if (j >= ps.nj) break;
    const int slot = MQ ? slot_rt : sl;
    mbar_wait_s(ps.full_s + 8 * slot, phase);
    const uint32_t pgs = ring_s + slot * PAGE;
    if (FUSED && j == patch_j) {  // the new row over the copy's (possibly stale) bytes
      const uint32_t cv = patch[2 * lane + 1];
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(pgs + k_code_off(ptok, 4 * lane)), "r"(patch[2 * lane]) : "memory");
#pragma unroll
      for (int e = 0; e < 4; ++e)
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(pgs + v_code_off(ptok, 4 * lane + e)), "r"((cv >> (8 * e)) & 0xffu)
                     : "memory");
      if (lane < 2)
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(pgs + (lane ? VS_OFF : KS_OFF) + 4 * ptok), "r"(patch[64 + lane])
                     : "memory");
      // generic-proxy writes into a slot the bulk copy will refill later
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    const uint4 k0 = lds128_at<0>(pgs + kb02), k2 = lds128_at<128>(pgs + kb02);
    const uint4 k1 = lds128_at<0>(pgs + kb13), k3 = lds128_at<128>(pgs + kb13);
    uint4 v0, v1, v2, v3;
    if (!HI) {
      v0 = lds128_at<0>(pgs + vb0), v1 = lds128_at<0>(pgs + vb1);
      v2 = lds128_at<1024>(pgs + vb0), v3 = lds128_at<1024>(pgs + vb1);
    }
    const float ks_r = lds32f_at<KS_OFF>(pgs + sb), ks_r8 = lds32f_at<KS_OFF + 32>(pgs + sb);
    const float vs_r0 = lds32f_at<VS_OFF>(pgs + sb), vs_r80 = lds32f_at<VS_OFF + 32>(pgs + sb);

    // ---- S^T = K . Q^T
    //   INT8: s8 tensor cores on the raw codes, two Q terms combined in integer
    //         (128 acc1 + acc2; the 1/128 lives in qscale), 4 k-steps of 32.
    //   FP8 : codes -> f16 (exact), 8 k-steps of 16; g <= 8 uses two chains for ILP.
    constexpr bool TWO_CHAINS = !HI;
    float st[NT][4];
    {
      // kr[i] / kr8[i]: 4 codes of token r / r+8 at k-step i's d range
      const uint32_t kr[8] = {k0.x, k1.x, k2.x, k3.x, k0.z, k1.z, k2.z, k3.z};
      const uint32_t kr8[8] = {k0.y, k1.y, k2.y, k3.y, k0.w, k1.w, k2.w, k3.w};
      uint4 qpair[NT];
      if constexpr (KVD == KVQ_INT8) {
        // g > 8: one n-tile at a time (its 8 accumulators, then its scores),
        // so the live set stays under the 128-register cap; g <= 8: k-steps
        // outer, both n-tiles' chains interleaved.
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          int acc1[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            uint32_t t1b0, t1b1, t2b0, t2b1;
            if constexpr (HI) {
              qpair[nt] = lds128(reinterpret_cast<const uint8_t*>(
                  reinterpret_cast<const uint4*>(qsm) + (nt * 4 + jj) * 32 + lane));
              t1b0 = qpair[nt].x; t1b1 = qpair[nt].y; t2b0 = qpair[nt].z; t2b1 = qpair[nt].w;
            } else {
              t1b0 = qf[nt][2 * jj][0]; t1b1 = qf[nt][2 * jj][1];
              t2b0 = qf[nt][2 * jj + 1][0]; t2b1 = qf[nt][2 * jj + 1][1];
            }
            mma16832_s8(acc1, kr[jj], kr8[jj], kr[4 + jj], kr8[4 + jj], t1b0, t1b1);
            mma16832_s8(acc2, kr[jj], kr8[jj], kr[4 + jj], kr8[4 + jj], t2b0, t2b1);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) st[nt][e] = __int2float_rn(acc1[e] * 256 + acc2[e]);
        }
      } else {
        float sa[NT][4], sb2[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) sa[nt][e] = sb2[nt][e] = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t a0, a2, a1, a3;
          codes_to_f16x2<KVD>(kr[i], a0, a2);
          codes_to_f16x2<KVD>(kr8[i], a1, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint32_t b0, b1;
            if constexpr (HI) {
              if ((i & 1) == 0) qpair[nt] = lds128(reinterpret_cast<const uint8_t*>(
                                    reinterpret_cast<const uint4*>(qsm) + (nt * 4 + i / 2) * 32 + lane));
              b0 = (i & 1) ? qpair[nt].z : qpair[nt].x;
              b1 = (i & 1) ? qpair[nt].w : qpair[nt].y;
            } else {
              b0 = qf[nt][i][0];
              b1 = qf[nt][i][1];
            }
            mma16816((TWO_CHAINS && i >= 4) ? sb2[nt] : sa[nt], a0, a1, a2, a3, b0, b1);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) st[nt][e] = TWO_CHAINS ? sa[nt][e] + sb2[nt][e] : sa[nt][e];
      }
    }
    if (HI) {  // g > 8: load V only after QK^T retired (keeps the live set under 128 regs)
      uint32_t dep;
      asm volatile("mov.b32 %0, 0;" : "=r"(dep) : "f"(st[0][0]), "f"(st[NT - 1][3]));
      v0 = lds128_at<0>(pgs + vb0 + dep), v1 = lds128_at<0>(pgs + vb1 + dep);
      v2 = lds128_at<1024>(pgs + vb0 + dep), v3 = lds128_at<1024>(pgs + vb1 + dep);
    }
    const int tok_base = (pg0 + warp + j * NW) * BS;

    // ---- softmax + PV of one page.  TAIL pages (some token past a query row's
    // visible length) get the masked instantiation; every other page runs the
    // unmasked one.
    auto page_tail = [&](auto tail_c) {
      constexpr bool TAIL = decltype(tail_c)::value;
      float vs_r = vs_r0, vs_r8 = vs_r80;
      if (TAIL) {
        if (tok_base + r >= L) vs_r = 0.0f;
        if (tok_base + r + 8 >= L) vs_r8 = 0.0f;
      }
      const float kq_r = ks_r * qscale, kq_r8 = ks_r8 * qscale;
      // scores relative to the running max, log2 units: u = S^T * scale_k * qscale - m (one FFMA);
      // st[nt]: [0]=(r,2c) [1]=(r,2c+1) [2]=(r+8,2c) [3]=(r+8,2c+1)
      auto visible = [&](int nt, int q4) { return !TAIL || tok_base + (q4 < 2 ? r : r + 8) < vis(nt, q4 & 1); };
      float u[NT][4];
      float umax = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          u[nt][q4] = fmaf(st[nt][q4], q4 < 2 ? kq_r : kq_r8, -m[nt][q4 & 1]);
          if (TAIL && !visible(nt, q4)) u[nt][q4] = -INFINITY;
          umax = fmaxf(umax, u[nt][q4]);
        }
      // ---- lazy rescale.  P' = p * scale_v is f16, so each row's reference
      //      point m is anchored on the largest CONTRIBUTION p * scale_v seen
      //      (log2: max of score + log2(scale_v)), not on the largest score:
      //      a dominant token with V ~ 0 (an attention sink) or a page whose V
      //      scales spread 2^20 then keeps the tokens that make up the output
      //      in f16's normal range.  p itself spans [2^-UMAX.., 2^UMAX] (l is
      //      fp32), which also absorbs the V scales' magnitude.  Fast path: one
      //      per-thread bound 2^umax * max(scale_v) <= 2^12 (P' far from f16
      //      overflow) + a warp vote; the exact per-row maxima (shuffle
      //      reductions) are computed only on the rare pages that move m.
      //      (Round 1 anchored m on the max score and kept a separate per-warp
      //      V normaliser 2^E: P' lost precision wherever the weight and the V
      //      scale of the tokens that matter were far from those two maxima.)
      const bool trig = __any_sync(FULL, umax > UMAX || fast_exp2(umax) * fmaxf(vs_r, vs_r8) > 4096.0f);
      if (trig) {
        // log2 of each token's V scale (-inf for scale 0 / masked tokens)
        const float lw_r = __log2f(vs_r), lw_r8 = __log2f(vs_r8);
        float mx[NT][2], cx[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float s0 = visible(nt, e) ? __fmul_rn(st[nt][e], kq_r) : -INFINITY;
            const float s8 = visible(nt, e + 2) ? __fmul_rn(st[nt][e + 2], kq_r8) : -INFINITY;
            mx[nt][e] = fmaxf(s0, s8);
            cx[nt][e] = fmaxf(s0 + lw_r, s8 + lw_r8);
          }
#pragma unroll
        for (int o2 = 4; o2 <= 16; o2 <<= 1)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              mx[nt][e] = fmaxf(mx[nt][e], __shfl_xor_sync(FULL, mx[nt][e], o2));
              cx[nt][e] = fmaxf(cx[nt][e], __shfl_xor_sync(FULL, cx[nt][e], o2));
            }
        // per-token cap on u so P' <= 2^12 even where fp32 cannot resolve the scores
        const float ucap_r = fminf(UMAX, 12.0f - lw_r), ucap_r8 = fminf(UMAX, 12.0f - lw_r8);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float f[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // m moves (up only) when this page's largest P' would pass 2^12 or its
            // largest p 2^UMAX; never for rows past G (m = +inf).
            const bool nm = cx[nt][e] > m[nt][e] + 12.0f || mx[nt][e] > m[nt][e] + UMAX;
            const float mn = fmaxf(cx[nt][e], mx[nt][e] - UMAX);
            const float cl = nm ? fast_exp2(m[nt][e] - mn) : 1.0f;
            if (nm) m[nt][e] = mn;
            l[nt][e] *= cl;
            f[e] = cl;
          }
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            o[nt][mt][0] *= f[0];
            o[nt][mt][1] *= f[1];
            o[nt][mt][2] *= f[0];
            o[nt][mt][3] *= f[1];
          }
          // Recompute from the ROUNDED product, as m was: the row's max-score
          // token gets u >= 0 (so l >= 1).  The fast path's FFMA is exact
          // instead; the two differ by half an ulp of m, which only matters past
          // |m| ~ 2^27 (log2 units; fp32 cannot resolve such scores) -- there the
          // caps keep p <= 2^UMAX and P' <= 2^12 (no 0/0, no inf).
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            u[nt][q4] = fminf(__fadd_rn(__fmul_rn(st[nt][q4], q4 < 2 ? kq_r : kq_r8), -m[nt][q4 & 1]),
                              q4 < 2 ? ucap_r : ucap_r8);
            if (TAIL && !visible(nt, q4)) u[nt][q4] = -INFINITY;
          }
        }
      }
      // ---- p (fp32, for l) and P' = p * scale_v (fp16) -> P'^T B-fragments
      const float w_r = vs_r, w_r8 = vs_r8;
      uint32_t pb[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float pv[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          pv[q4] = fast_exp2(u[nt][q4]);
          l[nt][q4 & 1] += pv[q4];
        }
        // 8x8 blocks: rows = tokens (r | r+8), cols = heads (2c, 2c+1)
        const uint32_t x0 = pack_half2(pv[0] * w_r, pv[1] * w_r);
        const uint32_t x1 = pack_half2(pv[2] * w_r8, pv[3] * w_r8);
        pb[nt][0] = movmatrix_trans(x0);  // (tokens 2c, 2c+1 ; head r)
        pb[nt][1] = movmatrix_trans(x1);  // (tokens 8+2c, 9+2c ; head r)
      }
      // ---- O^T += V^T . P'^T
      const uint32_t va[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};  // tokens 2c, 2c+1
      const uint32_t vbw[8] = {v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};  // tokens 8+2c, 9+2c
      uint32_t vmask_a = 0xffffffffu, vmask_b = 0xffffffffu;
      if (KVD == KVQ_FP8_E4M3 && TAIL) {  // garbage E4M3 codes may be NaN: zero masked tokens
        vmask_a = (tok_base + 2 * c < L ? 0x0000ffffu : 0u) | (tok_base + 2 * c + 1 < L ? 0xffff0000u : 0u);
        vmask_b = (tok_base + 8 + 2 * c < L ? 0x0000ffffu : 0u) | (tok_base + 9 + 2 * c < L ? 0xffff0000u : 0u);
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a0, a1, a2, a3;
        codes_to_f16x2<KVD>(va[mt], a0, a1);   // (DA, tok 2c|2c+1), (DA+1, ...)
        codes_to_f16x2<KVD>(vbw[mt], a2, a3);  // (DA, tok 8+2c|9+2c), (DA+1, ...)
        if (KVD == KVQ_FP8_E4M3 && TAIL) {
          a0 &= vmask_a;
          a1 &= vmask_a;
          a2 &= vmask_b;
          a3 &= vmask_b;
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma16816(o[nt][mt], a0, a1, a2, a3, pb[nt][0], pb[nt][1]);
      }
    };
    if (tok_base + BS > L_all) page_tail(std::true_type{});
    else page_tail(std::false_type{});

    // ---- refill this slot with page j + S.  Every LDS of the slot has
    // returned (its registers were consumed by the MMAs above) in every lane
    // (__syncwarp), so the async-proxy overwrite cannot race the reads.
    if (j + S < ps.nj) {
      __syncwarp();
      ps.issue(j + S, lane, slot);
    }
  }
    if (MQ) {
      if (++slot_rt == S) slot_rt = 0, phase ^= 1;
    } else {
      phase ^= 1;
    }
  }

  // ===== CTA merge of the NW warps =====
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int o2 = 4; o2 <= 16; o2 <<= 1) l[nt][e] += __shfl_xor_sync(FULL, l[nt][e], o2);
  __syncthreads();  // every ring slot consumed: reuse smem as merge scratch
  float* so = reinterpret_cast<float*>(smem);  // [NW][16 heads][128]
  float* sm = so + NW * 16 * HD;               // [NW][16] m
  float* sl = sm + NW * 16;                    // [NW][16] l
  if (r == 0) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sm[warp * 16 + 8 * nt + 2 * c + e] = hvalid[nt][e] ? m[nt][e] : -INFINITY;
        sl[warp * 16 + 8 * nt + 2 * c + e] = l[nt][e];
      }
  }
  __syncthreads();
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float f[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int hh = 8 * nt + 2 * c + e;
      float M = -INFINITY;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) M = fmaxf(M, sm[w2 * 16 + hh]);
      f[e] = (hvalid[nt][e] && m[nt][e] > -INFINITY) ? fast_exp2(m[nt][e] - M) : 0.0f;
    }
    float* mine = so + (warp * 16 + 8 * nt + 2 * c) * HD;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int da = (mt < 4 ? 8 * r + 2 * mt : 64 + 8 * r + 2 * (mt - 4));
      *reinterpret_cast<float2*>(mine + da) = make_float2(o[nt][mt][0] * f[0], o[nt][mt][2] * f[0]);
      *reinterpret_cast<float2*>(mine + HD + da) = make_float2(o[nt][mt][1] * f[1], o[nt][mt][3] * f[1]);
    }
  }
  __syncthreads();
  if (PEER && nsplit == 1) peer_acquire(p.peer);
  // Each thread finalises 8 contiguous d of one head row.
  const int tid = threadIdx.x;
  const int nrow_items = G * (HD / 8);
  for (int item = tid; item < nrow_items; item += THREADS) {
    const int row = item / (HD / 8), d0 = (item % (HD / 8)) * 8;
    float M = -INFINITY;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) M = fmaxf(M, sm[w2 * 16 + row]);
    float lsum = 0.0f;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) {
      const float mw = sm[w2 * 16 + row];
      if (mw == -INFINITY) continue;  // warp saw no page
      lsum += sl[w2 * 16 + row] * fast_exp2(mw - M);
      const float* src = so + (w2 * 16 + row) * HD + d0;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += src[e];
    }
    // lsum == 0: no token of this split is visible to the row (multi-query: a
    // split holding only the last draft tokens' positions); partial O = 0 with
    // LSE = -inf, so the combine weighs it 0 (not 0 * NaN).
    const float inv = lsum > 0.0f ? 1.0f / lsum : 0.0f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
    const int64_t vrow = ((int64_t)b * p.Hkv + h) * G + row;  // partial row of (b, h, query row)
    if (nsplit == 1) {
      store_out<PEER>(p, b, h, row, d0, acc);
    } else {
      float* dst = p.part_o + (vrow * p.max_splits + split) * HD + d0;
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
      if (d0 == 0) p.part_lse[vrow * p.max_splits + split] = M + __log2f(lsum);
    }
  }
  if (nsplit == 1) {
    if constexpr (PEER) peer_signal(p.peer);
    return;
  }

  // ===== fused split-KV combine: the last CTA of (b, h) merges all splits =====
  // bar.sync orders every thread's partial stores before thread 0's gpu-scope
  // acq_rel atomic (its release is cumulative), which publishes the split; the
  // last arriver's acquire + bar.sync make every split's partials visible.  No
  // per-thread fence.
  __syncthreads();
  if (tid == 0) {
    int* ctr = p.counters + (int64_t)b * p.Hkv + h;
    int prev;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
    const int last = prev == nsplit - 1;
    if (last) asm volatile("st.relaxed.gpu.s32 [%0], 0;" ::"l"(ctr) : "memory");  // reset for replay
    *flag = last;
  }
  __syncthreads();
  if (!*flag) return;
  if constexpr (PEER) peer_acquire(p.peer);
  if (!HI && nsplit >= 8 && G * nsplit + 16 <= NW * S * PAGE / 4) {
    // Many splits (small batches over long contexts), g <= 8.  With 16 rows the
    // per-item pairing below measured slower on C4, whose equal-length splits
    // put a combine at every wave boundary; with a few splits the extra phase
    // does not pay (A/B: tools/ab_decode.py GRAPH=1).
    // Phase A: per row, the max LSE and normalised weights, once, into shared
    // memory (the ring is free: every page was consumed).  Warps take rows,
    // lanes take splits.
    float* wsm = reinterpret_cast<float*>(smem);  // [G][nsplit] weights, then [G] 1 / sum
    for (int row = warp; row < G; row += NW) {
      const float* lse = p.part_lse + (((int64_t)b * p.Hkv + h) * G + row) * p.max_splits;
      float M = -INFINITY;
      for (int sp = lane; sp < nsplit; sp += 32) M = fmaxf(M, __ldcg(lse + sp));
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(FULL, M, o2));
      float ws = 0.0f;
      for (int sp = lane; sp < nsplit; sp += 32) {
        const float w = fast_exp2(__ldcg(lse + sp) - M);
        wsm[row * nsplit + sp] = w;
        ws += w;
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) ws += __shfl_xor_sync(FULL, ws, o2);
      if (lane == 0) wsm[G * nsplit + row] = 1.0f / ws;
    }
    __syncthreads();
    // Phase B: an item (row, 8 contiguous d) is shared by two neighbouring lanes,
    // each summing half of the splits; one shuffle merges them.  G * 32 work
    // units keep every thread's loads independent and in flight.
    const int h1 = (nsplit + 1) >> 1;
    for (int it = tid; it < nrow_items * 2; it += THREADS) {
      const int item = it >> 1, half = it & 1;
      const int row = item / (HD / 8), d0 = (item % (HD / 8)) * 8;
      const int64_t base = (((int64_t)b * p.Hkv + h) * G + row) * p.max_splits;
      const float* w = wsm + row * nsplit;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const int s0 = half ? h1 : 0, s1 = half ? nsplit : h1;
#pragma unroll 4
      for (int sp = s0; sp < s1; ++sp) {
        const float wgt = w[sp];
        const float4 a = __ldcg(reinterpret_cast<const float4*>(p.part_o + (base + sp) * HD + d0));
        const float4 cc = __ldcg(reinterpret_cast<const float4*>(p.part_o + (base + sp) * HD + d0 + 4));
        acc[0] += wgt * a.x;
        acc[1] += wgt * a.y;
        acc[2] += wgt * a.z;
        acc[3] += wgt * a.w;
        acc[4] += wgt * cc.x;
        acc[5] += wgt * cc.y;
        acc[6] += wgt * cc.z;
        acc[7] += wgt * cc.w;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(FULL, acc[e], 1);
      if (!half) {
        const float inv = wsm[G * nsplit + row];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] *= inv;
        store_out<PEER>(p, b, h, row, d0, acc);
      }
    }
    if constexpr (PEER) peer_signal(p.peer);
    return;
  }
  for (int item = tid; item < nrow_items; item += THREADS) {
    const int row = item / (HD / 8), d0 = (item % (HD / 8)) * 8;
    const int64_t base = (((int64_t)b * p.Hkv + h) * G + row) * p.max_splits;
    float M = -INFINITY;
#pragma unroll 4
    for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, __ldcg(p.part_lse + base + sp));
    float wsum = 0.0f, acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
    for (int sp = 0; sp < nsplit; ++sp) {
      const float wgt = fast_exp2(__ldcg(p.part_lse + base + sp) - M);
      wsum += wgt;
      const float4 a = __ldcg(reinterpret_cast<const float4*>(p.part_o + (base + sp) * HD + d0));
      const float4 cc = __ldcg(reinterpret_cast<const float4*>(p.part_o + (base + sp) * HD + d0 + 4));
      acc[0] += wgt * a.x;
      acc[1] += wgt * a.y;
      acc[2] += wgt * a.z;
      acc[3] += wgt * a.w;
      acc[4] += wgt * cc.x;
      acc[5] += wgt * cc.y;
      acc[6] += wgt * cc.z;
      acc[7] += wgt * cc.w;
    }
    const float inv = 1.0f / wsum;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
    store_out<PEER>(p, b, h, row, d0, acc);
  }
  if constexpr (PEER) peer_signal(p.peer);
}

#ifdef KVQ_TIMELINE
// Debug builds only (tools/timeline.py): per-CTA start / end %globaltimer and SM id.
__device__ unsigned long long g_timeline[1 << 17][3];
#endif

template <int KVD, bool HI, int MODE>
__global__ void __launch_bounds__(THREADS, Geo<HI>::CTAS) decode_kernel(const DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
#ifdef KVQ_TIMELINE
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  if (p.span && threadIdx.x == 0) atomicMin(p.span, global_ns());
  if (MODE == 2 && threadIdx.x == 0) peer_release(p.peer);
  decode_cta<KVD, HI, MODE>(p, smem);
  if (MODE == 2 && threadIdx.x == 0) peer_arrive(p.peer);
  if (p.span) {  // CTA-uniform: every path out of decode_cta is
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(p.span + 1, global_ns());
  }
#ifdef KVQ_TIMELINE
  if (threadIdx.x == 0) {
    unsigned long long t1;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    const size_t i = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
    if (i < (1 << 17)) {
      g_timeline[i][0] = t0;
      g_timeline[i][1] = t1;
      g_timeline[i][2] = sm;
    }
  }
#endif
}

unsigned read_and_clear_dev_err_decode() { return read_and_clear_dev_err_tu(); }

}  // namespace kvq

using namespace kvq_abi;

extern "C" {

size_t kvq_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t max_splits) {
  const size_t po = (size_t)B * Hq * max_splits * KVQ_HEAD_DIM * sizeof(float);
  const size_t pl = (size_t)B * Hq * max_splits * sizeof(float);
  const size_t cnt = (size_t)B * Hkv * sizeof(int);
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return up(cnt) + up(po) + up(pl);
}

int32_t kvq_decode_pages_per_split(int32_t B, int32_t Hkv, int64_t total_pages, int32_t max_blocks) {
  return kvq_decode_pages_per_split_rows(B, Hkv, 8, total_pages, max_blocks);
}

int32_t kvq_decode_pages_per_split_rows(int32_t B, int32_t Hkv, int32_t rows, int64_t total_pages,
                                        int32_t max_blocks) {
  // Large launches: uniform splits of <= 128 pages (540 KB of KV per CTA) so the
  // ragged tail is at most one short CTA (512 for equal lengths); as few waves
  // of CTAs_PER_SM x SMs as that allows.  Small launches: a latency cost model.
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  } else {
    cudaGetLastError();
  }
  const int64_t slots = (int64_t)sms * kvq::CTAS_PER_SM;
  const int64_t work = total_pages * (int64_t)Hkv;
  if (max_blocks > 0 && work <= slots * 128) {
    // Small, latency-bound launch (one wave at 128-page splits): pick the split
    // size from a cost model fitted to cold-L2 timings of B = 1..32 shapes
    // (tools/ab_decode.py FLUSH=1 PPS=...; each layer's KV is cold in serving):
    //   t = waves * (6 us + pages_per_cta * t_page) + 0.1 us * (splits - 1)
    //       + 0.01 us * concurrent CTAs,
    //   t_page = max(concurrent CTAs * 4224 B / 6.0 TB/s, 0.18 us),
    // the second term being the fused combine (one CTA merges every split), the
    // third the dispatch / ramp cost of a wider grid (equal-length batches;
    // ragged ones below use the first, L2-warm fit).
    static const int cand[] = {8, 9, 10, 12, 14, 16, 19, 22, 26, 30, 35, 41, 48, 56, 64, 75, 88, 103, 120, 140,
                               164, 192, 224, 262, 306, 358, 419, 490, 573, 670, 784, 917, 1073, 1255};
    // Ragged batches (total below B * max_blocks): sum_b ceil(n_b / pps) is
    // estimated as total / pps + B / 2 per head, and the waves count
    // fractionally -- CTAs of unequal length backfill the slots a wave leaves.
    // (C2's shape split over 8 ranks, one kv head each: 66 -> 55 us.)
    const int64_t per = max_blocks;  // the longest sequence sets the latency
    const int64_t pairs0 = (int64_t)B * Hkv;
    const bool ragged = total_pages * 20 < (int64_t)B * max_blocks * 19;
    double best_t = 1e30;
    int64_t best = per < 8 ? per : 8;
    for (int c : cand) {
      if (c > per) break;
      const int64_t ns = (per + c - 1) / c;
      const int64_t pps_eff = (per + ns - 1) / ns;
      int64_t ctas = pairs0 * ns;
      if (ragged) ctas = std::min(ctas, (int64_t)Hkv * ((total_pages + pps_eff - 1) / pps_eff + (B + 1) / 2));
      const double nw = ragged ? std::max(1.0, (double)ctas / slots) : (double)((ctas + slots - 1) / slots);
      const double conc = (double)std::min(ctas, slots);
      // Ragged batches keep the first (L2-warm) fit, t_page >= 0.22 us and no
      // width term: the cold fit over-favours long CTAs there (B = 8 ragged
      // 26.6 -> 28.7 us), the longest sequence setting the time either way.
      const double t = ragged ? nw * (4.5 + pps_eff * std::max(conc * 4224.0 / 6.9e6, 0.22)) + 0.14 * (ns - 1)
                              : nw * (6.0 + pps_eff * std::max(conc * 4224.0 / 6.0e6, 0.18)) + 0.1 * (ns - 1) +
                                    0.01 * conc;
      if (t < best_t) {
        best_t = t;
        best = pps_eff;
      }
    }
    return (int32_t)std::max<int64_t>(1, std::min<int64_t>(best, per));
  }
  // Equal-length batches have no ragged tail to protect: allow 512-page
  // splits (4x less split prologue / partial traffic / combine work).
  // (Only for big launches -- >= 8 waves at 128-page splits, e.g. C3 / C4: in the
  // few-wave range the 512 cap left ~1 wave of very long CTAs, B = 32 x 8K
  // 110 us vs 92 us at 128 pages.)
  const bool equal = max_blocks > 0 && total_pages * 20 >= (int64_t)B * max_blocks * 19;
  const bool uniform = equal && work >= slots * 128 * 8;
  if (equal && !uniform && rows > 8) {
    // g > 8 (two n-tiles, C4's shapes), 1-8 waves at 128-page splits, equal
    // lengths (C4 at P = 4 / 8: 32-128 long sequences per rank).  Its split
    // combine is serial per (sequence, kv head) in the last CTA and costs
    // ~0.75 us per split (fit to tools/ab_decode.py PPS sweeps), so the
    // 128-page cap costs up to 20 % (C4 at P = 8: 238 us at 111 pages, 192 at
    // 507).  Pick the split from a wave model instead: full waves at the
    // all-slots page time, the remainder wave at its own concurrency's,
    //   t = full * pps * tp(slots) + [rem] pps * tp(rem) + 0.75 us * splits,
    //   tp(c) = max(c * 4224 B / 6.3 TB/s, 0.33 us).
    // Candidates: fixed sizes plus the splits that fill k whole waves exactly
    // (k = 1..8); within 1 % of the best modelled time the wider grid wins
    // (C4 at P = 8: 576 CTAs at 456 pages 189 us vs 544 at 482 pages 194 us).
    static const int fixed[] = {64, 96, 128, 170, 255, 340, 507, 768, 1024, 1536, 2048};
    const int64_t per = max_blocks, pairs = (int64_t)B * Hkv;
    int64_t cand[sizeof(fixed) / sizeof(fixed[0]) + 8];
    int nc = 0;
    for (int c : fixed) cand[nc++] = c;
    for (int k = 1; k <= 8; ++k) {
      const int64_t ns = k * slots / pairs;
      if (ns >= 1) cand[nc++] = (per + ns - 1) / ns;
    }
    auto tp = [](double c) { return std::max(c * 4224.0 / 6.3e6, 0.33); };
    double t_of[sizeof(cand) / sizeof(cand[0])];
    int64_t pps_of[sizeof(cand) / sizeof(cand[0])], ctas_of[sizeof(cand) / sizeof(cand[0])];
    double best_t = 1e30;
    for (int i = 0; i < nc; ++i) {
      const int64_t c = std::min<int64_t>(std::max<int64_t>(cand[i], 1), per);
      const int64_t ns = (per + c - 1) / c, pps_eff = (per + ns - 1) / ns, ctas = pairs * ns;
      const int64_t full = ctas / slots, rem = ctas - full * slots;
      t_of[i] = full * pps_eff * tp((double)slots) + (rem ? pps_eff * tp((double)rem) : 0.0) + 0.75 * ns;
      pps_of[i] = pps_eff;
      ctas_of[i] = ctas;
      best_t = std::min(best_t, t_of[i]);
    }
    int64_t best = std::min<int64_t>(per, 128), best_ctas = -1;
    for (int i = 0; i < nc; ++i)
      if (t_of[i] <= 1.01 * best_t && ctas_of[i] > best_ctas) {
        best_ctas = ctas_of[i];
        best = pps_of[i];
      }
    return (int32_t)std::max<int64_t>(1, best);
  }
  const int64_t cap = uniform ? 512 : 128;
  const int64_t waves = (work + slots * cap - 1) / (slots * cap);
  int64_t pps = (work + slots * (waves > 0 ? waves : 1) - 1) / (slots * (waves > 0 ? waves : 1));
  // Single wave: leave room for each (sequence, head)'s rounded-up last split so
  // the grid really fits one wave (a second, nearly empty wave doubles latency).
  const int64_t pairs = (int64_t)B * Hkv;
  if (waves <= 1 && slots > pairs) pps = (work + (slots - pairs) - 1) / (slots - pairs);
  if (pps < 8) pps = 8;
  if (pps > cap) pps = cap;
  if (max_blocks > 0 && pps > max_blocks) pps = max_blocks;
  return (int32_t)(pps > 0 ? pps : 1);
}

// Function attributes (dynamic smem size, max-shared carveout) are set once
// per (device, kernel variant), not on every launch: two cudaFuncSetAttribute
// calls cost microseconds of host time per call on the eager path.
static cudaError_t set_attributes_once(const void* kernel, int smem_bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kernel})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done.insert({dev, kernel});
  return e;
}

// kvq_profile_next_decode: one-shot span pointer for this host thread's next K2 launch.
static thread_local unsigned long long* t_next_span = nullptr;

static int decode_attn_impl(const void* q, int64_t q_batch_stride, int32_t q_len, const void* pool,
                            int64_t num_blocks, const int32_t* block_table, int32_t max_blocks,
                            const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype,
                            float sm_scale, int32_t pages_per_split, void* workspace,
                            size_t workspace_bytes, void* out, int32_t out_dtype, int32_t out_layout,
                            const kvq_peer_out* peer, void* stream, bool pdl = false, bool tail_only = false,
                            const void* fk = nullptr, const void* fv = nullptr, int64_t fk_stride = 0,
                            int64_t fv_stride = 0, const int32_t* fslots = nullptr) {
  if (B < 0 || Hq <= 0 || Hkv <= 0 || max_blocks <= 0 || num_blocks <= 0 || q_len <= 0)
    return fail(KVQ_EINVAL, "decode_attn: bad sizes");
  if (B == 0) return KVQ_OK;
  if (Hq % Hkv != 0 || (Hq / Hkv) * q_len > 16)
    return fail(KVQ_EINVAL, "decode_attn: need Hq % Hkv == 0 and (Hq / Hkv) * q_len <= 16");
  if (!q || !pool || !block_table || !seq_lens || !out || !workspace)
    return fail(KVQ_EINVAL, "decode_attn: null pointer");
  if (!aligned(q, 16) || (q_batch_stride % 8) || !aligned(pool, 16) || !aligned(out, 16) ||
      !aligned(workspace, 256))
    return fail(KVQ_EINVAL, "decode_attn: q/pool/out must be 16-byte aligned, workspace 256-byte");
  if (kv_dtype != KVQ_INT8 && kv_dtype != KVQ_FP8_E4M3)
    return fail(KVQ_EUNSUPPORTED, "decode_attn: unknown kv dtype");
  if (out_dtype != KVQ_OUT_BF16 && out_dtype != KVQ_OUT_F32)
    return fail(KVQ_EINVAL, "decode_attn: bad out dtype");
  if (out_layout != KVQ_OUT_BHD && out_layout != KVQ_OUT_HBD)
    return fail(KVQ_EINVAL, "decode_attn: bad out layout");
  if (pages_per_split <= 0)
    pages_per_split = kvq_decode_pages_per_split_rows(B, Hkv, (Hq / Hkv) * q_len, (int64_t)B * max_blocks, max_blocks);
  const int max_splits = (max_blocks + pages_per_split - 1) / pages_per_split;
  const int64_t rows = (int64_t)Hq * q_len;  // query rows per sequence
  if (workspace_bytes < kvq_decode_workspace_bytes(B, (int32_t)rows, Hkv, max_splits))
    return fail(KVQ_EINVAL, "decode_attn: workspace too small");
  if (int rc = check_device()) return rc;

  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  kvq::DecodeParams prm;
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.q_stride_b = q_batch_stride;
  prm.pool = static_cast<const uint8_t*>(pool);
  prm.num_blocks = num_blocks;
  prm.block_table = block_table;
  prm.max_blocks = max_blocks;
  prm.seq_lens = seq_lens;
  prm.B = B;
  prm.Hq = Hq;
  prm.Hkv = Hkv;
  prm.g = Hq / Hkv;
  prm.q_len = q_len;
  prm.G = prm.g * q_len;
  prm.sm_scale_log2 = sm_scale * 1.4426950408889634f;
  prm.pages_per_split = pages_per_split;
  prm.max_splits = max_splits;
  prm.counters = reinterpret_cast<int*>(ws);
  prm.part_o = reinterpret_cast<float*>(ws + up((size_t)B * Hkv * sizeof(int)));
  prm.part_lse = reinterpret_cast<float*>(ws + up((size_t)B * Hkv * sizeof(int)) +
                                          up((size_t)B * rows * max_splits * KVQ_HEAD_DIM * sizeof(float)));
  prm.out = out;
  prm.out_f32 = out_dtype == KVQ_OUT_F32;
  prm.out_hbd = out_layout == KVQ_OUT_HBD;
  prm.peer = kvq_peer_out{};
  if (peer) prm.peer = *peer;
  prm.tail_only = pdl && tail_only;
  const bool fused = fk != nullptr;
  prm.ak = static_cast<const __nv_bfloat16*>(fk);
  prm.av = static_cast<const __nv_bfloat16*>(fv);
  prm.ak_stride = fk_stride;
  prm.av_stride = fv_stride;
  prm.aslots = fslots;
  prm.span = t_next_span;
  t_next_span = nullptr;

  const dim3 grid((unsigned)max_splits, (unsigned)Hkv, (unsigned)B);
  auto st = static_cast<cudaStream_t>(stream);
  const bool hi = prm.G > 8;
  const size_t smem_bytes = (hi ? kvq::Geo<true>::SMEM : kvq::Geo<false>::SMEM) + (fused ? kvq::Geo<false>::PATCH : 0);
  auto launch = [&](auto kernel) -> int {
    cudaError_t e = set_attributes_once(reinterpret_cast<const void*>(kernel), (int)smem_bytes);
    if (e != cudaSuccess) return fail(KVQ_ECUDA, cudaGetErrorString(e));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kvq::THREADS);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kernel, prm);
    if (e != cudaSuccess) return fail(KVQ_ECUDA, cudaGetErrorString(e));
    return check_launch("decode_attn");
  };
  const int mode = fused ? 3 : peer ? 2 : (q_len > 1 ? 1 : 0);
  if (mode == 3) {
    if (kv_dtype == KVQ_INT8)
      return hi ? launch(kvq::decode_kernel<KVQ_INT8, true, 3>) : launch(kvq::decode_kernel<KVQ_INT8, false, 3>);
    return hi ? launch(kvq::decode_kernel<KVQ_FP8_E4M3, true, 3>) : launch(kvq::decode_kernel<KVQ_FP8_E4M3, false, 3>);
  }
  if (kv_dtype == KVQ_INT8) {
    if (mode == 2) return hi ? launch(kvq::decode_kernel<KVQ_INT8, true, 2>) : launch(kvq::decode_kernel<KVQ_INT8, false, 2>);
    if (mode == 1) return hi ? launch(kvq::decode_kernel<KVQ_INT8, true, 1>) : launch(kvq::decode_kernel<KVQ_INT8, false, 1>);
    return hi ? launch(kvq::decode_kernel<KVQ_INT8, true, 0>) : launch(kvq::decode_kernel<KVQ_INT8, false, 0>);
  }
  if (mode == 2)
    return hi ? launch(kvq::decode_kernel<KVQ_FP8_E4M3, true, 2>) : launch(kvq::decode_kernel<KVQ_FP8_E4M3, false, 2>);
  if (mode == 1)
    return hi ? launch(kvq::decode_kernel<KVQ_FP8_E4M3, true, 1>) : launch(kvq::decode_kernel<KVQ_FP8_E4M3, false, 1>);
  return hi ? launch(kvq::decode_kernel<KVQ_FP8_E4M3, true, 0>) : launch(kvq::decode_kernel<KVQ_FP8_E4M3, false, 0>);
}

int kvq_decode_step_mq(const void* k, const void* v, int64_t k_token_stride, int64_t v_token_stride,
                       const int32_t* slot_mapping, int32_t T, const void* q, int64_t q_batch_stride,
                       int32_t q_len, void* pool, int64_t num_blocks, const int32_t* block_table,
                       int32_t max_blocks, const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv,
                       int32_t kv_dtype, float sm_scale, int32_t pages_per_split, void* workspace,
                       size_t workspace_bytes, void* out, int32_t out_dtype, int32_t out_layout,
                       const kvq_peer_out* peer, int32_t flags, void* stream) {
  if (flags & ~(KVQ_STEP_APPEND_TAIL_ONLY | KVQ_STEP_FUSED_APPEND)) return fail(KVQ_EINVAL, "decode_step: unknown flags");
  if (q_len <= 0) return fail(KVQ_EINVAL, "decode_step: bad q_len");
  if (flags & KVQ_STEP_FUSED_APPEND) {
    // No K1 launch: K2's CTA holding each sequence's last page quantizes the row.
    if (q_len != 1 || peer || T != B)
      return fail(KVQ_EINVAL, "decode_step: KVQ_STEP_FUSED_APPEND needs q_len == 1, no peer gather and T == B");
    if (kv_dtype != KVQ_INT8 && kv_dtype != KVQ_FP8_E4M3)
      return fail(KVQ_EUNSUPPORTED, "decode_step: unknown kv dtype");
    if (B > 0 && (!k || !v || !slot_mapping))
      return fail(KVQ_EINVAL, "decode_step: null pointer");
    if (!aligned(k, 8) || !aligned(v, 8) || (k_token_stride % 4) || (v_token_stride % 4) ||
        k_token_stride < (int64_t)Hkv * KVQ_HEAD_DIM || v_token_stride < (int64_t)Hkv * KVQ_HEAD_DIM)
      return fail(KVQ_EINVAL, "decode_step: k/v rows must be 8-byte aligned with a token stride >= Hkv * 128");
    return decode_attn_impl(q, q_batch_stride, 1, pool, num_blocks, block_table, max_blocks, seq_lens, B, Hq, Hkv,
                            kv_dtype, sm_scale, pages_per_split, workspace, workspace_bytes, out, out_dtype,
                            out_layout, nullptr, stream, false, false, k, v, k_token_stride, v_token_stride,
                            slot_mapping);
  }
  if (peer && q_len != 1) return fail(KVQ_EINVAL, "decode_step: the fused gather takes one query token per sequence");
  if (peer && (out_dtype != KVQ_OUT_BF16 || out_layout != KVQ_OUT_HBD))
    return fail(KVQ_EINVAL, "decode_step: the fused gather writes bf16 head-major rows");
  if (int rc = kvq_quant_append(k, v, k_token_stride, v_token_stride, slot_mapping, T, Hkv, kv_dtype, pool,
                                num_blocks, stream))
    return rc;
  if (peer) {
    const int P = peer->n_peers;
    if (P < 2 || P > KVQ_MAX_PEERS || peer->rank < 0 || peer->rank >= P || peer->head_offset < 0 ||
        peer->batch_global < B || peer->writers_per_use == 0)
      return fail(KVQ_EINVAL, "decode_step: bad peer descriptor");
    for (int r = 0; r < P; ++r)
      if (!peer->out[r] || !peer->ctl[r] || !aligned(peer->out[r], 16) || !aligned(peer->ctl[r], 128))
        return fail(KVQ_EINVAL, "decode_step: peer out (16 B) / ctl (128 B) pointers missing or misaligned");
    out = peer->out[peer->rank];
  }
  // K2 is launched with programmatic stream serialization right behind K1, so
  // its launch and prologue overlap K1 (K1 never writes q, the table or lens).
  // q_len > 1 new tokens may span two pages: the tail-only wait does not apply.
  const bool tail_only = (flags & KVQ_STEP_APPEND_TAIL_ONLY) != 0 && q_len == 1;
  return decode_attn_impl(q, q_batch_stride, q_len, pool, num_blocks, block_table, max_blocks, seq_lens, B, Hq,
                          Hkv, kv_dtype, sm_scale, pages_per_split, workspace, workspace_bytes, out, out_dtype,
                          out_layout, peer, stream, /*pdl=*/T > 0, tail_only);
}

int kvq_decode_step(const void* k, const void* v, int64_t k_token_stride, int64_t v_token_stride,
                    const int32_t* slot_mapping, int32_t T, const void* q, int64_t q_batch_stride,
                    void* pool, int64_t num_blocks, const int32_t* block_table, int32_t max_blocks,
                    const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype,
                    float sm_scale, int32_t pages_per_split, void* workspace, size_t workspace_bytes,
                    void* out, int32_t out_dtype, int32_t out_layout, const kvq_peer_out* peer,
                    int32_t flags, void* stream) {
  return kvq_decode_step_mq(k, v, k_token_stride, v_token_stride, slot_mapping, T, q, q_batch_stride, 1, pool,
                            num_blocks, block_table, max_blocks, seq_lens, B, Hq, Hkv, kv_dtype, sm_scale,
                            pages_per_split, workspace, workspace_bytes, out, out_dtype, out_layout, peer, flags,
                            stream);
}

int kvq_decode_attn_mq(const void* q, int64_t q_batch_stride, int32_t q_len, const void* pool,
                       int64_t num_blocks, const int32_t* block_table, int32_t max_blocks,
                       const int32_t* seq_lens, int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype,
                       float sm_scale, int32_t pages_per_split, void* workspace,
                       size_t workspace_bytes, void* out, int32_t out_dtype, int32_t out_layout,
                       void* stream) {
  return decode_attn_impl(q, q_batch_stride, q_len, pool, num_blocks, block_table, max_blocks, seq_lens, B,
                          Hq, Hkv, kv_dtype, sm_scale, pages_per_split, workspace, workspace_bytes, out,
                          out_dtype, out_layout, nullptr, stream);
}

int kvq_decode_attn_peer(const void* q, int64_t q_batch_stride, const void* pool, int64_t num_blocks,
                         const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                         int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype, float sm_scale,
                         int32_t pages_per_split, void* workspace, size_t workspace_bytes,
                         const kvq_peer_out* peer, void* stream) {
  if (!peer) return fail(KVQ_EINVAL, "decode_attn_peer: null peer descriptor");
  const int P = peer->n_peers;
  if (P < 2 || P > KVQ_MAX_PEERS || peer->rank < 0 || peer->rank >= P)
    return fail(KVQ_EINVAL, "decode_attn_peer: need 2 <= n_peers <= 8 and 0 <= rank < n_peers");
  if (peer->head_offset < 0 || peer->batch_global < B || peer->writers_per_use == 0)
    return fail(KVQ_EINVAL, "decode_attn_peer: bad head_offset / batch_global / writers_per_use");
  for (int r = 0; r < P; ++r)
    if (!peer->out[r] || !peer->ctl[r] || !aligned(peer->out[r], 16) || !aligned(peer->ctl[r], 128))
      return fail(KVQ_EINVAL, "decode_attn_peer: peer out (16 B) / ctl (128 B) pointers missing or misaligned");
  // `out` is not written in peer mode; the rank's own copy stands in for validation.
  return decode_attn_impl(q, q_batch_stride, 1, pool, num_blocks, block_table, max_blocks, seq_lens, B, Hq,
                          Hkv, kv_dtype, sm_scale, pages_per_split, workspace, workspace_bytes,
                          peer->out[peer->rank], KVQ_OUT_BF16, KVQ_OUT_HBD, peer, stream);
}

int kvq_decode_attn(const void* q, int64_t q_batch_stride, const void* pool, int64_t num_blocks,
                    const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                    int32_t B, int32_t Hq, int32_t Hkv, int32_t kv_dtype, float sm_scale,
                    int32_t pages_per_split, void* workspace, size_t workspace_bytes, void* out,
                    int32_t out_dtype, int32_t out_layout, void* stream) {
  return kvq_decode_attn_mq(q, q_batch_stride, 1, pool, num_blocks, block_table, max_blocks, seq_lens,
                            B, Hq, Hkv, kv_dtype, sm_scale, pages_per_split, workspace, workspace_bytes,
                            out, out_dtype, out_layout, stream);
}

int kvq_profile_next_decode(uint64_t* span) {
  if (span && !aligned(span, 8)) return fail(KVQ_EINVAL, "profile_next_decode: span must be 8-byte aligned");
  t_next_span = reinterpret_cast<unsigned long long*>(span);
  return KVQ_OK;
}

#ifdef KVQ_TIMELINE
int kvq_debug_timeline(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, kvq::g_timeline, bytes) == cudaSuccess ? 0 : -3;
}
#endif

}  // extern "C"
