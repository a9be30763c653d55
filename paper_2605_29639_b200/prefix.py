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
  pinned memory -- the reference's ``writeback_on_evict`` demotion
  (``tiered_cache.py:254-275``): only when the key is not already on the
  host and only when it fits *without cascading* (a full host tier drops the
  victim; it never evicts a host page to make room).  A later request that
  misses on the GPU but hits here promotes the page back with one
  host-to-device copy (the reference's ``LOAD_TO_GPU`` step,
  ``tiered_cache.py:277-317``); the host copy stays resident, as in the
  reference.  The page moves bit-identical at 4224 B per (block, kv head), so
  an offloaded 8-bit prefix costs half the PCIe bytes of bf16.

All device copies are stream-ordered on the current stream: the offload of a
victim page precedes any append into its block, and a promotion precedes the
attention that reads it.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import torch

from ._lib import PAGE_BYTES
from .cache import BlockAllocator, CacheThrashError, KVCacheSpec, PagedKVCache


class HostTier:
    """Store of whole evicted blocks (all kv heads) in pinned host memory, with
    the reference's LOCAL_CPU demotion rule (``tiered_cache.py:254-275``):
    a demoted key is inserted only if absent and only if a slot is free; a
    full tier drops the new victim instead of evicting (no cascade).  With
    only the GPU tier above it nothing else ever evicts a host page, so a
    slot handed out by :meth:`take` stays valid."""

    def __init__(self, capacity_blocks: int, num_kv_heads: int, pin: Optional[bool] = None):
        if capacity_blocks <= 0:
            raise ValueError("capacity_blocks must be positive")
        pin = torch.cuda.is_available() if pin is None else pin
        self.store = torch.empty((capacity_blocks, num_kv_heads, PAGE_BYTES), dtype=torch.uint8,
                                 pin_memory=pin)
        self.capacity = capacity_blocks
        self._slot: Dict[object, int] = {}   # key -> slot
        self._free = list(range(capacity_blocks - 1, -1, -1))
        self.offloaded = self.promoted = self.dropped = 0

    def __contains__(self, key) -> bool:
        return key in self._slot

    def keys(self) -> List[object]:
        return list(self._slot)

    def put(self, key, pages: torch.Tensor) -> bool:
        """Demote ``key``'s pages; False when it is already here or there is no
        free slot (best effort, as the reference: nothing is evicted)."""
        if key in self._slot:
            return False
        if not self._free:
            self.dropped += 1
            return False
        slot = self._free.pop()
        self.store[slot].copy_(pages, non_blocking=True)
        self._slot[key] = slot
        self.offloaded += 1
        return True

    def take(self, key) -> Optional[torch.Tensor]:
        """The host pages of ``key`` (the copy stays resident)."""
        slot = self._slot.get(key)
        if slot is None:
            return None
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
        # Insert first: it may evict a GPU page, whose offload runs now, so the
        # host slot read below cannot be reused under the copy.
        blk = self.alloc.pool.insert(key, self.alloc.block_size, self.alloc.clock)
        pages = self.host.take(key)
        self.cache.pool[blk].copy_(pages, non_blocking=True)
        self.host_hit_tokens += self.alloc.block_size
        return True

    # request API ---------------------------------------------------------------
    def admit(self, seq_id, tokens: Sequence[int]) -> Tuple[int, List[int]]:
        """Register ``seq_id`` for prompt ``tokens``.  On
        :class:`CacheThrashError` everything the request acquired is released
        before the error propagates (the reference's ``_dispatch_prefill``:
        ``release_and_update(acquired)`` then raise, ``simulator.py:397-400``), so the
        caller can requeue it."""
        before = self.host_hit_tokens
        try:
            cached = self.alloc.allocate_prefix(seq_id, tokens, promote=self._promote)
            slots = self.alloc.append_tokens(seq_id, tokens[cached:])
        except CacheThrashError:
            if seq_id in self.alloc:
                self.alloc.free(seq_id)
            self.host_hit_tokens = before
            raise
        self.gpu_hit_tokens += cached - (self.host_hit_tokens - before)
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
