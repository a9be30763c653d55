"""Prefix reuse of quantized pages across requests, with a pinned-host tier
(SURVEY.md §8f-3).

This mirrors the reference's hierarchical cache for the two tiers the data
path touches.  The reference simulator moves only metadata; here the payload
is the quantized pages themselves:

* **GPU tier.** Full pages are keyed by their chained prefix hash
  (``blocks.py:51-69``, computed natively by ``kvq_block_hashes``) and shared
  by reference count.  A finished request's hashed pages stay resident,
  unreferenced, and LRU-evictable (``tiered_cache.py:189-252``).  A new
  request with the same prefix reuses them without re-quantizing
  (``simulator.py:360-396``: matched prefix vs. uncached suffix).
* **Local-CPU tier.** An evicted hashed page is copied device-to-host into
  pinned memory.  A later request that misses on the GPU but hits here
  promotes the page back with one host-to-device copy (the reference's
  ``LOAD_TO_GPU`` step, ``tiered_cache.py:277-317``).  The page moves
  bit-identical at 4224 B per (block, kv head), so an offloaded 8-bit prefix
  costs half the PCIe bytes of bf16.

All device copies are stream-ordered on the current stream: the offload of a
victim page precedes any append into its block, and a promotion precedes the
attention that reads it.
"""
from __future__ import annotations

from collections import OrderedDict
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from ._lib import PAGE_BYTES
from .cache import BlockAllocator, KVCacheSpec, PagedKVCache


class HostTier:
    """LRU store of whole evicted blocks (all kv heads) in pinned host memory."""

    def __init__(self, capacity_blocks: int, num_kv_heads: int, pin: Optional[bool] = None):
        if capacity_blocks <= 0:
            raise ValueError("capacity_blocks must be positive")
        pin = torch.cuda.is_available() if pin is None else pin
        self.store = torch.empty((capacity_blocks, num_kv_heads, PAGE_BYTES), dtype=torch.uint8,
                                 pin_memory=pin)
        self.capacity = capacity_blocks
        self._slot: "OrderedDict[object, int]" = OrderedDict()  # key -> slot, LRU first
        self._free = list(range(capacity_blocks - 1, -1, -1))
        self.offloaded = self.promoted = self.dropped = 0

    def __contains__(self, key) -> bool:
        return key in self._slot

    def put(self, key, pages: torch.Tensor) -> None:
        if key in self._slot:
            self._slot.move_to_end(key)
            return
        if not self._free:  # drop the least recently used host page
            _, slot = self._slot.popitem(last=False)
            self._free.append(slot)
            self.dropped += 1
        slot = self._free.pop()
        self.store[slot].copy_(pages, non_blocking=True)
        self._slot[key] = slot
        self.offloaded += 1

    def take(self, key) -> Optional[torch.Tensor]:
        """The host pages of ``key`` (the slot stays valid until the next put)."""
        slot = self._slot.get(key)
        if slot is None:
            return None
        self._slot.move_to_end(key)
        self.promoted += 1
        return self.store[slot]


class PrefixKVCache:
    """A paged quantized KV cache whose full pages are reused across requests
    by prefix hash, with an optional pinned-host tier for evicted pages.

    ``admit(seq, tokens)`` returns ``(cached_tokens, slots)``.  Only the
    ``tokens[cached_tokens:]`` suffix needs ``quantize_append`` into ``slots``.
    """

    def __init__(self, spec: KVCacheSpec, num_blocks: int, device="cuda", host_blocks: int = 0):
        self.spec = spec
        self.cache = PagedKVCache(spec, num_blocks, device=device)
        self.alloc = BlockAllocator(num_blocks, bytes_per_block=spec.bytes_per_block)
        self.host = HostTier(host_blocks, spec.num_kv_heads,
                             pin=(torch.device(device).type == "cuda")) if host_blocks else None
        self.alloc.pool.on_evict = self._offload
        self.gpu_hit_tokens = self.host_hit_tokens = self.computed_tokens = 0

    # pool callbacks ----------------------------------------------------------
    def _offload(self, key, block: int) -> None:
        if self.host is not None and key[0] == "h":
            self.host.put(key, self.cache.pool[block])

    def _promote(self, key) -> bool:
        if self.host is None or key not in self.host:
            return False
        pages = self.host.take(key)
        blk = self.alloc.pool.insert(key, self.alloc.block_size, self.alloc.clock)
        self.cache.pool[blk].copy_(pages, non_blocking=True)
        self.host_hit_tokens += self.alloc.block_size
        return True

    # request API ---------------------------------------------------------------
    def admit(self, seq_id, tokens: Sequence[int]) -> Tuple[int, List[int]]:
        before = self.host_hit_tokens
        cached = self.alloc.allocate_prefix(seq_id, tokens, promote=self._promote)
        self.gpu_hit_tokens += cached - (self.host_hit_tokens - before)
        slots = self.alloc.append_tokens(seq_id, tokens[cached:])
        self.computed_tokens += len(tokens) - cached
        return cached, slots

    def extend(self, seq_id, tokens: Sequence[int]) -> List[int]:
        """Decode-time append of known tokens (pages that fill become reusable)."""
        self.computed_tokens += len(tokens)
        return self.alloc.append_tokens(seq_id, tokens)

    def free(self, seq_id) -> None:
        self.alloc.free(seq_id)

    def block_table(self, seq_ids, max_blocks=None):
        return self.alloc.block_table(seq_ids, max_blocks)

    def stats(self) -> Dict[str, int]:
        return {"gpu_hit_tokens": self.gpu_hit_tokens, "host_hit_tokens": self.host_hit_tokens,
                "computed_tokens": self.computed_tokens,
                "host_offloaded": self.host.offloaded if self.host else 0,
                "host_dropped": self.host.dropped if self.host else 0}
