"""B200-native quantized paged-KV decode path (arxiv/paper_2605_29639, RTP-LLM
§7.2.2 "KV Cache Quantization").

Public API (mirrors the plugin surface named in BASELINE.json.north_star):
block allocator / block table, quantize-on-append, paged decode attention,
KV-head sharding.  Compute runs in hand-written sm_100a kernels behind the C
ABI of ``libkvq.so`` (include/kvq.h).
"""
from .cache import (BlockAllocator, BlockTable, CacheThrashError, KVCacheSpec, PagedKVCache,
                    unpack_pages)
from .ops import check_device_errors, copy_blocks, decode_step, paged_decode_attention, paged_decode_attention_gathered, quantize_append

__all__ = [
    "BlockAllocator", "BlockTable", "CacheThrashError", "KVCacheSpec", "PagedKVCache",
    "unpack_pages", "check_device_errors", "copy_blocks", "decode_step", "paged_decode_attention", "paged_decode_attention_gathered",
    "quantize_append",
]
__version__ = "0.1.0"
