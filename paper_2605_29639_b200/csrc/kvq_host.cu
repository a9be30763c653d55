// kvq_host.cu -- host-side native parts of libkvq (no device code).
//
//   kvq_version / kvq_last_error / kvq_page_bytes: ABI identity and errors.
//   kvq_pipeline_submit: the serving loop's per-step enqueue (upload, step
//   graph, download) in one call.  kvq_sym_*: IPC-shareable buffers of the
//   fused peer gather.
//   kvq_block_hashes: chained 64-bit block keys for prefix reuse of quantized
//   pages.  Same key definition as the reference's prefix-cache identity
//   (servesim blocks.py:29-69: FNV-1a over 8-byte little-endian words; the
//   first block chained from the golden-ratio seed; one key per complete block,
//   none for a trailing partial block), so keys computed here match the
//   reference's for equal block sizes (pinned by tests/test_prefix.py against
//   the reference's frozen value, test_blocks.py:63-66).
#include <stdint.h>

#include "kvq_common.cuh"

namespace {
constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x00000100000001B3ull;
constexpr uint64_t kChainSeed = 0x9E3779B97F4A7C15ull;

inline uint64_t mix_word(uint64_t h, uint64_t w) {
  for (int i = 0; i < 8; ++i) {
    h = (h ^ (w & 0xFFu)) * kFnvPrime;
    w >>= 8;
  }
  return h;
}
}  // namespace

extern "C" int64_t kvq_block_hashes(const int64_t* tokens, int64_t n, int32_t block_size,
                                    uint64_t prev_key, uint64_t* out) {
  if (block_size < 1 || n < 0 || (n > 0 && !tokens)) return KVQ_EINVAL;
  const int64_t nkeys = n / block_size;
  if (nkeys > 0 && !out) return KVQ_EINVAL;
  uint64_t prev = prev_key ? prev_key : kChainSeed;
  for (int64_t b = 0; b < nkeys; ++b) {
    uint64_t h = mix_word(kFnvOffset, prev);
    for (int32_t i = 0; i < block_size; ++i) h = mix_word(h, (uint64_t)tokens[b * block_size + i]);
    out[b] = h;
    prev = h;
  }
  return nkeys;
}

// ---------------------------------------------------------------------------
// Host runtime: version / error reporting, the serving loop's step submitter,
// symmetric (IPC-shareable) buffers for the fused peer gather.
// ---------------------------------------------------------------------------
namespace kvq_abi {
thread_local char g_err[512] = "";
}
using namespace kvq_abi;

extern "C" {

int kvq_version(void) { return KVQ_ABI_VERSION; }

const char* kvq_last_error(void) { return g_err; }

size_t kvq_page_bytes(void) { return KVQ_PAGE_BYTES; }

int kvq_check_device_errors(void* stream, uint32_t* bits) {
  if (bits) *bits = 0;
  const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(KVQ_ECUDA, cudaGetErrorString(e));
  const unsigned v = kvq::read_and_clear_dev_err_append() | kvq::read_and_clear_dev_err_decode();
  if (v & 0x80000000u) return fail(KVQ_ECUDA, "check_device_errors: cannot read the device error word");
  if (bits) *bits = v;
  if (!v) return KVQ_OK;
  snprintf(g_err, sizeof(g_err), "device-side caller error(s):%s%s%s",
           (v & KVQ_DERR_BLOCK_ID) ? " block id out of range [0, num_blocks) (KVQ_DERR_BLOCK_ID);" : "",
           (v & KVQ_DERR_SEQ_LEN) ? " seq_lens outside [0, max_blocks * 16] (KVQ_DERR_SEQ_LEN);" : "",
           (v & KVQ_DERR_SLOT) ? " slot past the pool (KVQ_DERR_SLOT);" : "");
  return KVQ_EINVAL;
}

int kvq_pipeline_submit(const kvq_pipe_step* s) {
  if (!s || !s->graph_exec || !s->dev_in || !s->host_in || !s->dev_out || !s->host_out || !s->ev_in_ready ||
      !s->ev_done || !s->ev_out_done)
    return fail(KVQ_EINVAL, "pipeline_submit: null handle or buffer");
  auto h2d = static_cast<cudaStream_t>(s->h2d_stream);
  auto cmp = static_cast<cudaStream_t>(s->compute_stream);
  auto d2h = static_cast<cudaStream_t>(s->d2h_stream);
  auto in_ready = static_cast<cudaEvent_t>(s->ev_in_ready);
  auto done = static_cast<cudaEvent_t>(s->ev_done);
  auto out_done = static_cast<cudaEvent_t>(s->ev_out_done);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  if (s->reuse) ok(cudaStreamWaitEvent(h2d, done, 0));      // the slot's previous kernels read dev_in
  ok(cudaMemcpyAsync(s->dev_in, s->host_in, s->in_bytes, cudaMemcpyHostToDevice, h2d));
  ok(cudaEventRecord(in_ready, h2d));
  ok(cudaStreamWaitEvent(cmp, in_ready, 0));
  if (s->reuse) ok(cudaStreamWaitEvent(cmp, out_done, 0));  // the slot's previous download read dev_out
  ok(cudaGraphLaunch(static_cast<cudaGraphExec_t>(s->graph_exec), cmp));
  ok(cudaEventRecord(done, cmp));
  ok(cudaStreamWaitEvent(d2h, done, 0));
  ok(cudaMemcpyAsync(s->host_out, s->dev_out, s->out_bytes, cudaMemcpyDeviceToHost, d2h));
  ok(cudaEventRecord(out_done, d2h));
  if (e != cudaSuccess) return fail(KVQ_ECUDA, cudaGetErrorString(e));
  return KVQ_OK;
}

int kvq_sym_alloc(size_t bytes, void** ptr, void* ipc_handle) {
  if (!ptr || !ipc_handle || bytes == 0) return fail(KVQ_EINVAL, "sym_alloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return fail(KVQ_ECUDA, cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == KVQ_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(ipc_handle, &h, sizeof(h));
  *ptr = p;
  return KVQ_OK;
}

int kvq_sym_open(const void* ipc_handle, void** ptr) {
  if (!ptr || !ipc_handle) return fail(KVQ_EINVAL, "sym_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(KVQ_ECUDA, cudaGetErrorString(e));
  return KVQ_OK;
}

int kvq_sym_close(void* ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? KVQ_OK : fail(KVQ_ECUDA, cudaGetErrorString(e));
}

int kvq_sym_free(void* ptr) {
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? KVQ_OK : fail(KVQ_ECUDA, cudaGetErrorString(e));
}

}  // extern "C"
