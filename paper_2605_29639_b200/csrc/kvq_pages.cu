// kvq_pages.cu -- K3, whole-block page copies: copy-on-write of shared
// tails (kvq_copy_blocks) and the PD-transfer wire format (kvq_gather_blocks /
// kvq_scatter_blocks).
#include "kvq_common.cuh"

namespace kvq {

// ---------------------------------------------------------------------------
// K3: page copies for copy-on-write.
// ---------------------------------------------------------------------------
// Whole-block page copies (all kv heads of a block, Hkv * 4224 bytes):
// dst block dst_ids[i * dst_step] <- src block src_ids[i * src_step]; a null id
// list is the identity (gather into / scatter from a packed buffer).  One CTA
// per block, four 16-byte loads in flight per thread before the stores.
__global__ void __launch_bounds__(256) copy_pages_kernel(const uint8_t* __restrict__ src, int64_t src_blocks,
                                                         const int32_t* __restrict__ src_ids, int src_step,
                                                         uint8_t* __restrict__ dst, int64_t dst_blocks,
                                                         const int32_t* __restrict__ dst_ids, int dst_step,
                                                         int Hkv) {
  const int i = blockIdx.x;
  const int64_t sb = src_ids ? (int64_t)__ldg(src_ids + (int64_t)i * src_step) : i;
  const int64_t db = dst_ids ? (int64_t)__ldg(dst_ids + (int64_t)i * dst_step) : i;
  if (sb < 0 || sb >= src_blocks || db < 0 || db >= dst_blocks) return;
  const int64_t n16 = (int64_t)Hkv * PAGE / 16;
  const uint4* s = reinterpret_cast<const uint4*>(src + sb * (int64_t)Hkv * PAGE);
  uint4* d = reinterpret_cast<uint4*>(dst + db * (int64_t)Hkv * PAGE);
  for (int64_t j0 = threadIdx.x; j0 < n16; j0 += 4 * 256) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u * 256 < n16) r[u] = __ldcs(s + j0 + u * 256);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u * 256 < n16) __stcs(d + j0 + u * 256, r[u]);
  }
}

}  // namespace kvq

using namespace kvq_abi;

extern "C" {

int kvq_copy_blocks(void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* pairs,
                    int32_t n_pairs, void* stream) {
  if (n_pairs < 0 || Hkv <= 0 || num_blocks <= 0) return fail(KVQ_EINVAL, "copy_blocks: bad sizes");
  if (n_pairs == 0) return KVQ_OK;
  if (!pool || !pairs) return fail(KVQ_EINVAL, "copy_blocks: null pointer");
  if (!aligned(pool, 16)) return fail(KVQ_EINVAL, "copy_blocks: pool must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  auto* p = static_cast<uint8_t*>(pool);
  kvq::copy_pages_kernel<<<n_pairs, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, num_blocks, pairs, 2, p,
                                                                                  num_blocks, pairs + 1, 2, Hkv);
  return check_launch("copy_blocks");
}

int kvq_gather_blocks(const void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* block_ids, int32_t n,
                      void* out, void* stream) {
  if (n < 0 || Hkv <= 0 || num_blocks <= 0) return fail(KVQ_EINVAL, "gather_blocks: bad sizes");
  if (n == 0) return KVQ_OK;
  if (!pool || !block_ids || !out) return fail(KVQ_EINVAL, "gather_blocks: null pointer");
  if (!aligned(pool, 16) || !aligned(out, 16)) return fail(KVQ_EINVAL, "gather_blocks: buffers must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  kvq::copy_pages_kernel<<<n, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(pool), num_blocks, block_ids, 1, static_cast<uint8_t*>(out), n, nullptr, 1, Hkv);
  return check_launch("gather_blocks");
}

int kvq_scatter_blocks(void* pool, int64_t num_blocks, int32_t Hkv, const int32_t* block_ids, int32_t n,
                       const void* in, void* stream) {
  if (n < 0 || Hkv <= 0 || num_blocks <= 0) return fail(KVQ_EINVAL, "scatter_blocks: bad sizes");
  if (n == 0) return KVQ_OK;
  if (!pool || !block_ids || !in) return fail(KVQ_EINVAL, "scatter_blocks: null pointer");
  if (!aligned(pool, 16) || !aligned(in, 16)) return fail(KVQ_EINVAL, "scatter_blocks: buffers must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  kvq::copy_pages_kernel<<<n, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(in), n, nullptr, 1, static_cast<uint8_t*>(pool), num_blocks, block_ids, 1, Hkv);
  return check_launch("scatter_blocks");
}

}  // extern "C"
