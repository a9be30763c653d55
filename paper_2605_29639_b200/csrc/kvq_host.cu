// kvq_host.cu -- host-side native helpers of libkvq (no device code).
//
//   kvq_block_hashes: chained 64-bit block keys for prefix reuse of quantized
//   pages.  Same key definition as the reference's prefix-cache identity
//   (servesim blocks.py:29-69: FNV-1a over 8-byte little-endian words; the
//   first block chained from the golden-ratio seed; one key per complete block,
//   none for a trailing partial block), so keys computed here match the
//   reference's for equal block sizes (pinned by tests/test_prefix.py against
//   the reference's frozen value, test_blocks.py:63-66).
#include <stdint.h>

#include "kvq.h"

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
