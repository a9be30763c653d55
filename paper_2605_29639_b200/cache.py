"""Paged quantized KV cache: spec, device pool, block allocator, block table.

Block-lifecycle rules follow the reference's GPU tier exactly
(arxiv/paper_2605_29639 servesim, ``tiered_cache.py``):

* full blocks are reference-counted and shareable
  (``CacheBlockEntry`` invariants, ``tiered_cache.py:105-116``; ``SPEC.md`` "a
  full block (watermark == block_size) may have ref_count > 1");
* a partial block is exclusive -- acquiring it twice raises
  ``ValueError("partial block is exclusive")`` (``tiered_cache.py:358-363``);
* the watermark only grows, up to ``block_size``
  (``set_watermark``, ``tiered_cache.py:344-351``);
* releasing an unreferenced block raises ``ValueError("double release")``
  (``tiered_cache.py:327-342``);
* running out of blocks raises :class:`CacheThrashError` carrying the bytes
  still needed (``errors.py:14-25``), which the caller turns into backpressure
  (``simulator.py:339-345``).

What the reference keeps as metadata only (``CacheBlockEntry`` has no payload)
is here backed by a device pool of 4224-byte pages per (block, kv head):
``pool[num_blocks][Hkv][4224]``.  The page size (16 tokens) is
decoupled from the reference's prefix-hash granularity (64 tokens,
``blocks.py:29``): a 64-token hash block is four pages.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np
import torch

from ._lib import BLOCK_SIZE, HEAD_DIM, KVQ_FP8_E4M3, KVQ_INT8, PAGE_BYTES

KV_DTYPES = {"int8": KVQ_INT8, "fp8_e4m3": KVQ_FP8_E4M3}


class CacheThrashError(RuntimeError):
    """No free block: every block is referenced (mirrors servesim's
    ``CacheThrashError(tier, bytes_needed)``, ``errors.py:14-25``)."""

    def __init__(self, bytes_needed: int):
        super().__init__(f"gpu cache thrash: {bytes_needed} bytes still needed")
        self.tier = "gpu"
        self.bytes_needed = bytes_needed


@dataclass(frozen=True)
class KVCacheSpec:
    """Geometry of one attention layer's quantized KV cache."""

    num_kv_heads: int
    head_dim: int = HEAD_DIM
    block_size: int = BLOCK_SIZE
    kv_dtype: str = "int8"

    def __post_init__(self):
        if self.head_dim != HEAD_DIM:
            raise ValueError(f"head_dim must be {HEAD_DIM}")
        if self.block_size != BLOCK_SIZE:
            raise ValueError(f"block_size must be {BLOCK_SIZE}")
        if self.kv_dtype not in KV_DTYPES:
            raise ValueError(f"kv_dtype must be one of {sorted(KV_DTYPES)}")
        if self.num_kv_heads <= 0:
            raise ValueError("num_kv_heads must be positive")

    @property
    def kv_dtype_id(self) -> int:
        return KV_DTYPES[self.kv_dtype]

    @property
    def bytes_per_block(self) -> int:
        """Bytes of one block across all kv heads (the reference's
        ``_block_bytes``, ``simulator.py:178-179``)."""
        return self.num_kv_heads * PAGE_BYTES

    @property
    def kv_bytes_per_token(self) -> int:
        """Algorithmic bytes per token per layer: codes + fp32 scales (the
        reference's ``CostModel.kv_bytes_per_token``, ``cost.py:41``)."""
        return self.num_kv_heads * (2 * self.head_dim + 2 * 4)


class PagedKVCache:
    """Device pool ``uint8[num_blocks][Hkv][4224]`` for one layer."""

    def __init__(self, spec: KVCacheSpec, num_blocks: int, device="cuda", pool=None):
        if num_blocks <= 0:
            raise ValueError("num_blocks must be positive")
        self.spec = spec
        self.num_blocks = num_blocks
        if pool is None:
            pool = torch.zeros((num_blocks, spec.num_kv_heads, PAGE_BYTES), dtype=torch.uint8,
                               device=device)
        if tuple(pool.shape) != (num_blocks, spec.num_kv_heads, PAGE_BYTES) or pool.dtype != torch.uint8:
            raise ValueError("pool must be uint8 [num_blocks, Hkv, 4224]")
        if not pool.is_contiguous():
            raise ValueError("pool must be contiguous")
        self.pool = pool

    @property
    def device(self):
        return self.pool.device

    def nbytes(self) -> int:
        return self.pool.numel()


# ---------------------------------------------------------------------------
# Logical <-> physical page layout (host-side, for tests and inspection).
# ---------------------------------------------------------------------------
def _layout_index() -> Tuple[np.ndarray, np.ndarray]:
    """code_idx[kv, t, d] and scale_idx[kv, t]: byte offsets inside a page
    (same formulas as csrc/kvq_common.cuh k_code_off / v_code_off)."""
    code = np.zeros((2, BLOCK_SIZE, HEAD_DIM), dtype=np.int64)
    for t in range(BLOCK_SIZE):
        for d in range(HEAD_DIM):
            pr, hi_row, half, dd = t & 7, t >> 3, d >> 6, d & 63
            unit = (4 * ((dd >> 2) & 3) + (dd >> 4)) ^ ((pr & 1) << 2)
            code[0, t, d] = pr * 256 + unit * 16 + (2 * half + hi_row) * 4 + (d & 3)
            L = 2 * d + (t & 1)
            R = 2 * (t >> 1) + (L >> 7)
            l = L & 127
            code[1, t, d] = 2048 + R * 128 + (((l >> 4) ^ (R & 7)) << 4) + (l & 15)
    scale = np.zeros((2, BLOCK_SIZE), dtype=np.int64)
    for kv in range(2):
        for t in range(BLOCK_SIZE):
            scale[kv, t] = 4096 + kv * 64 + 4 * t
    return code, scale


CODE_INDEX, SCALE_INDEX = _layout_index()


def unpack_pages(pages: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """``uint8[..., 4224]`` -> logical codes ``uint8[..., 2, 16, 128]`` and
    scales ``float32[..., 2, 16]``."""
    pages = pages.contiguous()
    idx = torch.as_tensor(CODE_INDEX.reshape(-1), device=pages.device)
    codes = pages.index_select(-1, idx).reshape(*pages.shape[:-1], 2, BLOCK_SIZE, HEAD_DIM)
    sidx = torch.as_tensor(SCALE_INDEX.reshape(-1), device=pages.device)
    sb = pages.index_select(-1, (sidx[:, None] + torch.arange(4, device=pages.device)).reshape(-1))
    scales = sb.reshape(*pages.shape[:-1], 2 * BLOCK_SIZE, 4).contiguous().view(torch.float32)
    return codes, scales.reshape(*pages.shape[:-1], 2, BLOCK_SIZE)


# ---------------------------------------------------------------------------
# Block pool: residency + lifecycle of physical pages (the reference's GPU tier)
# ---------------------------------------------------------------------------
@dataclass
class BlockEntry:
    """One resident page set (the reference's ``CacheBlockEntry``,
    ``tiered_cache.py:105-116``) plus the physical block it occupies."""

    key: object
    block: int
    seq_no: int          # insertion order: the reference's monotonic block_id (LRU tie-break)
    watermark: int
    ref_count: int = 0
    last_access: int = 0


class BlockPool:
    """Residency of ``num_blocks`` physical pages under the reference GPU-tier
    rules: insert (evicting least-recently-used unreferenced entries, ties by
    insertion order, ``tiered_cache.py:189-252``), acquire (partial blocks are
    exclusive, ``:355-363``), release (``:327-342``), grow-only watermark
    (``:344-351``).  Unreferenced entries stay resident (reusable by key) until
    evicted or dropped."""

    def __init__(self, num_blocks: int, block_size: int = BLOCK_SIZE, bytes_per_block: int = 1):
        if num_blocks <= 0:
            raise ValueError("num_blocks must be positive")
        self.num_blocks, self.block_size, self.bytes_per_block = num_blocks, block_size, bytes_per_block
        self._free: List[int] = list(range(num_blocks - 1, -1, -1))  # pop() -> lowest id first
        self._entries: Dict[object, BlockEntry] = {}
        self._heap: List[Tuple[int, int, object]] = []  # lazy (last_access, seq_no, key)
        self._by_block: Dict[int, object] = {}
        self._seq = 0
        self._unref = 0          # resident entries with ref_count == 0 (evictable)
        self.on_evict = None     # callable(key, block) before an evicted block is reused
        self.mutation_count = 0

    # -- introspection
    def __len__(self) -> int:
        return len(self._entries)

    @property
    def num_free(self) -> int:
        return len(self._free)

    @property
    def num_evictable(self) -> int:
        return self._unref

    def entry(self, key) -> Optional[BlockEntry]:
        return self._entries.get(key)

    def key_of(self, block: int):
        return self._by_block.get(block)

    def lookup(self, key) -> Optional[int]:
        e = self._entries.get(key)
        return None if e is None else e.block

    def keys(self):
        return list(self._entries)

    def is_partial(self, e: BlockEntry) -> bool:
        return e.watermark < self.block_size

    # -- mutation
    def insert(self, key, watermark: int, clock: int = 0) -> int:
        if not 0 <= watermark <= self.block_size:
            raise ValueError("watermark out of range")
        if key in self._entries:
            raise ValueError("duplicate insert")
        if not self._free:
            self.evict(1)
        blk = self._free.pop()
        e = BlockEntry(key=key, block=blk, seq_no=self._seq, watermark=watermark, last_access=clock)
        self._seq += 1
        self._entries[key] = e
        self._by_block[blk] = key
        self._unref += 1
        self.mutation_count += 1
        heapq.heappush(self._heap, (clock, e.seq_no, key))
        return blk

    def evict(self, nblocks: int) -> List[object]:
        """Drop unreferenced entries, oldest first; partial progress stands
        when it raises (as the reference's ``evict``)."""
        if nblocks <= 0:
            raise ValueError("bytes_needed must be positive")
        out: List[object] = []
        while len(out) < nblocks:
            while self._heap:
                la, sq, k = self._heap[0]
                e = self._entries.get(k)
                if e is not None and e.ref_count == 0 and e.last_access == la and e.seq_no == sq:
                    break
                heapq.heappop(self._heap)
            if not self._heap:
                raise CacheThrashError((nblocks - len(out)) * self.bytes_per_block)
            _, _, k = heapq.heappop(self._heap)
            if self.on_evict is not None:
                self.on_evict(k, self._entries[k].block)
            self.drop(k)
            out.append(k)
        return out

    def drop(self, key) -> int:
        e = self._entries.pop(key)
        if e.ref_count:
            self._entries[key] = e
            raise ValueError("cannot drop a referenced block")
        self._free.append(e.block)
        del self._by_block[e.block]
        self._unref -= 1
        self.mutation_count += 1
        return e.block

    def acquire(self, key, clock: int = 0) -> BlockEntry:
        e = self._entries.get(key)
        if e is None:
            raise KeyError(f"no entry for {key!r}")
        if self.is_partial(e) and e.ref_count >= 1:
            raise ValueError("partial block is exclusive")
        if e.ref_count == 0:
            self._unref -= 1
        e.ref_count += 1
        self._touch(e, clock)
        return e

    def release(self, keys: Iterable, clock: int = 0) -> None:
        for k in keys:
            e = self._entries.get(k)
            if e is None or e.ref_count <= 0:
                raise ValueError("double release")
            e.ref_count -= 1
            if e.ref_count == 0:
                self._unref += 1
            self._touch(e, clock)

    def set_watermark(self, key, watermark: int) -> None:
        e = self._entries.get(key)
        if e is None:
            raise KeyError(f"no entry for {key!r}")
        if not e.watermark <= watermark <= self.block_size:
            raise ValueError("watermark may only grow, up to block_size")
        e.watermark = watermark

    def rekey(self, old, new) -> None:
        """Give a resident entry a new key (e.g. its content hash once full)."""
        if new in self._entries:
            raise ValueError("duplicate insert")
        e = self._entries.pop(old)
        e.key = new
        self._entries[new] = e
        self._by_block[e.block] = new
        if e.ref_count == 0:
            heapq.heappush(self._heap, (e.last_access, e.seq_no, new))

    def _touch(self, e: BlockEntry, clock: int) -> None:
        e.last_access = clock
        if e.ref_count == 0:
            heapq.heappush(self._heap, (clock, e.seq_no, e.key))


# ---------------------------------------------------------------------------
# Block allocator (sequences on top of the pool; device pages are copied by
# kvq_copy_blocks)
# ---------------------------------------------------------------------------
@dataclass
class _Seq:
    keys: List[object] = field(default_factory=list)
    length: int = 0
    hashing: bool = False                  # token ids known: full pages get prefix keys
    last_hash: int = 0                     # chain key of the last full page (0 = seed)
    tail_tokens: List[int] = field(default_factory=list)
    blocks: List[int] = field(default_factory=list)  # physical block of each key (fixed while referenced)


def block_hashes(tokens: Sequence[int], block_size: int = BLOCK_SIZE, prev_key: int = 0) -> List[int]:
    """Chained 64-bit keys of the complete pages of ``tokens`` (native
    ``kvq_block_hashes``; the reference's block identity, ``blocks.py:51-69``)."""
    from . import _lib
    toks = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
    n = len(toks) // block_size
    out = np.zeros(max(n, 1), dtype=np.uint64)
    got = _lib.load().kvq_block_hashes(toks.ctypes.data if len(toks) else None, len(toks), block_size,
                                       prev_key, out.ctypes.data)
    if got < 0:
        raise ValueError("kvq_block_hashes: bad arguments")
    return [int(x) for x in out[:got]]


class BlockAllocator:
    """Per-sequence block lists over a :class:`BlockPool`.

    ``append_slots`` returns the slot ids (``block * 16 + offset``) the new
    tokens occupy; ``fork`` shares every full block of the parent and copies
    its partial tail (partial blocks are exclusive), returning the
    ``(src, dst)`` page copies the caller must apply on the device before the
    child appends.  Private blocks are returned to the free list as soon as
    their last reference is released.
    """

    def __init__(self, num_blocks: int, block_size: int = BLOCK_SIZE, bytes_per_block: int = 1):
        if block_size != BLOCK_SIZE:
            raise ValueError(f"block_size must be {BLOCK_SIZE}")
        self.pool = BlockPool(num_blocks, block_size, bytes_per_block)
        self.num_blocks, self.block_size = num_blocks, block_size
        self.bytes_per_block = bytes_per_block
        self._seqs: Dict[object, _Seq] = {}
        self._anon = 0
        self.clock = 0

    # -- introspection
    @property
    def num_free(self) -> int:
        return self.pool.num_free

    def _entry_of_block(self, block: int) -> Optional[BlockEntry]:
        k = self.pool.key_of(block)
        return None if k is None else self.pool.entry(k)

    def ref_count(self, block: int) -> int:
        e = self._entry_of_block(block)
        return 0 if e is None else e.ref_count

    def watermark(self, block: int) -> int:
        e = self._entry_of_block(block)
        return 0 if e is None else e.watermark

    def block_ids(self, seq_id) -> List[int]:
        return list(self._seq(seq_id).blocks)

    def seq_len(self, seq_id) -> int:
        return self._seq(seq_id).length

    def seq_ids(self) -> List[object]:
        return list(self._seqs)

    def __contains__(self, seq_id) -> bool:
        return seq_id in self._seqs

    def _seq(self, seq_id) -> _Seq:
        try:
            return self._seqs[seq_id]
        except KeyError:
            raise KeyError(f"unknown sequence {seq_id!r}") from None

    @property
    def num_available(self) -> int:
        """Free blocks plus cached (unreferenced, evictable) prefix pages."""
        return self.pool.num_free + self.pool.num_evictable

    def _new_block(self) -> object:
        key = ("anon", self._anon)
        self._anon += 1
        if not self.num_available:
            raise CacheThrashError(self.bytes_per_block)
        self.pool.insert(key, 0, self.clock)  # evicts the LRU cached page when no block is free
        self.pool.acquire(key, self.clock)
        return key

    def _release(self, key) -> None:
        self.pool.release([key], self.clock)
        if self.pool.entry(key).ref_count == 0 and key[0] == "anon":
            self.pool.drop(key)  # private page: free now; hashed full pages stay cached

    # -- sequence API
    def allocate(self, seq_id) -> None:
        """Register an empty sequence."""
        if seq_id in self._seqs:
            raise ValueError(f"sequence {seq_id!r} already exists")
        self._seqs[seq_id] = _Seq()

    def append_slots(self, seq_id, n: int) -> List[int]:
        """Reserve ``n`` token slots at the end of ``seq_id``.  Atomic: on
        :class:`CacheThrashError` nothing changes.

        Without token ids a prefix-hashed sequence (one admitted through
        :meth:`allocate_prefix` / :meth:`append_tokens`) stops hashing: its
        later pages are private and never keyed, since a key must describe
        the page's tokens (the pages already keyed keep their keys)."""
        s = self._seq(seq_id)
        slots = self._append(s, n)
        self._stop_hashing(s)
        return slots

    @staticmethod
    def _stop_hashing(s: "_Seq") -> None:
        if s.hashing:
            s.hashing = False
            s.tail_tokens = []

    def _append(self, s: "_Seq", n: int) -> List[int]:
        if n < 0:
            raise ValueError("n must be >= 0")
        bs = self.block_size
        tail_room = (bs - s.length % bs) % bs if s.keys else 0
        new_blocks = -(-(n - tail_room) // bs) if n > tail_room else 0
        if new_blocks > self.num_available:
            raise CacheThrashError((new_blocks - self.num_available) * self.bytes_per_block)
        self.clock += 1
        slots: List[int] = []
        pos = s.length
        while len(slots) < n:
            if pos % bs == 0:
                key = self._new_block()
                s.keys.append(key)
                s.blocks.append(self.pool.entry(key).block)
            key = s.keys[pos // bs]
            e = self.pool.entry(key)
            take = min(n - len(slots), bs - pos % bs)
            base = e.block * bs + pos % bs
            slots.extend(range(base, base + take))
            pos += take
            self.pool.set_watermark(key, pos - (pos - 1) // bs * bs)
        s.length = pos
        return slots

    def append_one(self, seq_ids: Sequence) -> np.ndarray:
        """The decode step's slots: one new token for each of ``seq_ids`` (the
        batched form of ``append_slots(s, 1)``, same rules); returns int32
        ``block * 16 + offset`` per sequence.  Atomic: on
        :class:`CacheThrashError` nothing changes.  Like :meth:`append_slots`,
        a prefix-hashed sequence stops hashing (its decoded tokens' ids are not
        known here)."""
        seqs = [self._seq(s) for s in seq_ids]
        bs = self.block_size
        need = sum(1 for s in seqs if s.length % bs == 0)
        if need > self.num_available:
            raise CacheThrashError((need - self.num_available) * self.bytes_per_block)
        self.clock += 1
        out = np.empty(len(seqs), dtype=np.int32)
        entries = self.pool._entries
        for i, s in enumerate(seqs):
            off = s.length % bs
            if off == 0:
                key = self._new_block()
                s.keys.append(key)
                s.blocks.append(entries[key].block)
            e = entries[s.keys[-1]]
            if e.watermark > off + 1:  # the grow-only rule of set_watermark
                raise ValueError("watermark may only grow, up to block_size")
            e.watermark = off + 1
            out[i] = s.blocks[-1] * bs + off
            s.length += 1
            if s.hashing:
                self._stop_hashing(s)
        return out

    def fork(self, parent_id, child_id) -> List[Tuple[int, int]]:
        """New sequence sharing the parent's full blocks; the partial tail is
        copied (``(src, dst)`` page copies returned for the device)."""
        if child_id in self._seqs:
            raise ValueError(f"sequence {child_id!r} already exists")
        p = self._seq(parent_id)
        self.clock += 1
        tail = p.keys[-1] if p.keys else None
        partial_tail = tail is not None and self.pool.is_partial(self.pool.entry(tail))
        if partial_tail and not self.num_available:
            raise CacheThrashError(self.bytes_per_block)
        keys: List[object] = []
        for k in (p.keys[:-1] if partial_tail else p.keys):
            self.pool.acquire(k, self.clock)  # full: shareable
            keys.append(k)
        copies: List[Tuple[int, int]] = []
        if partial_tail:
            dst = self._new_block()
            self.pool.set_watermark(dst, self.pool.entry(tail).watermark)
            keys.append(dst)
            copies.append((self.pool.lookup(tail), self.pool.lookup(dst)))
        self._seqs[child_id] = _Seq(keys=keys, length=p.length, hashing=p.hashing,
                                    last_hash=p.last_hash, tail_tokens=list(p.tail_tokens),
                                    blocks=[self.pool.lookup(k) for k in keys])
        return copies

    # -- prefix reuse (reference prefix identity blocks.py:51-69)
    def allocate_prefix(self, seq_id, tokens: Sequence[int], promote=None) -> int:
        """Register ``seq_id`` for prompt ``tokens`` and share the longest run
        of leading full pages already resident under their chained keys
        (``promote(key) -> bool`` may first bring a page back from a lower
        tier).  Returns the number of prompt tokens covered; append the rest
        with :meth:`append_tokens`."""
        self.allocate(seq_id)
        s = self._seqs[seq_id]
        s.hashing = True
        self.clock += 1
        for h in block_hashes(tokens, self.block_size):
            key = ("h", h)
            if self.pool.entry(key) is None and not (promote is not None and promote(key)):
                break
            s.blocks.append(self.pool.acquire(key, self.clock).block)
            s.keys.append(key)
            s.length += self.block_size
            s.last_hash = h
        return s.length

    def append_tokens(self, seq_id, tokens: Sequence[int]) -> List[int]:
        """:meth:`append_slots` for known token ids: every page the tokens
        complete is re-keyed to its chained prefix key, so later requests
        with the same prefix can share it (it stays cached after free)."""
        s = self._seq(seq_id)
        if not s.hashing:
            if s.length:
                raise ValueError("sequence was filled without token ids")
            s.hashing = True
        first_page = s.length // self.block_size
        slots = self._append(s, len(tokens))
        pending = s.tail_tokens + [int(t) for t in tokens]
        nfull = len(pending) // self.block_size
        if nfull:
            hashes = block_hashes(pending[: nfull * self.block_size], self.block_size, s.last_hash)
            for i, h in enumerate(hashes):
                page = first_page + i
                old, new = s.keys[page], ("h", h)
                if old[0] == "anon" and self.pool.entry(new) is None:
                    self.pool.rekey(old, new)
                    s.keys[page] = new
            s.last_hash = hashes[-1]
        s.tail_tokens = pending[nfull * self.block_size:]
        return slots

    def free(self, seq_id) -> None:
        s = self._seqs.pop(seq_id, None)
        if s is None:
            raise KeyError(f"unknown sequence {seq_id!r}")
        self.clock += 1
        for k in s.keys:
            self._release(k)

    # -- device views
    def block_table(self, seq_ids: Sequence, max_blocks: Optional[int] = None) -> np.ndarray:
        rows = [self._seq(s).blocks for s in seq_ids]
        mb = max_blocks if max_blocks is not None else max([len(r) for r in rows] + [1])
        out = np.zeros((len(rows), mb), dtype=np.int32)
        for i, r in enumerate(rows):
            if len(r) > mb:
                raise ValueError("max_blocks too small")
            out[i, : len(r)] = r
        return out

    def seq_lens(self, seq_ids: Sequence) -> np.ndarray:
        return np.array([self._seq(s).length for s in seq_ids], dtype=np.int32)

    # -- invariants (for tests; cf. test_tiered_cache.py:243-327)
    def check_invariants(self) -> None:
        counts: Dict[object, int] = {}
        for s in self._seqs.values():
            assert len(s.keys) == -(-s.length // self.block_size), "block count vs length"
            assert s.blocks == [self.pool.lookup(k) for k in s.keys], "cached block ids"
            for i, k in enumerate(s.keys):
                counts[k] = counts.get(k, 0) + 1
                full = (i + 1) * self.block_size <= s.length
                wm = self.block_size if full else s.length - i * self.block_size
                assert self.pool.entry(k).watermark == wm, "watermark mismatch"
        blocks = set()
        unref = 0
        for k, e in self.pool._entries.items():
            assert e.ref_count == counts.get(k, 0), f"refcount mismatch on {k!r}"
            if e.ref_count == 0:
                unref += 1
                assert k[0] == "h" and e.watermark == self.block_size, "only full hashed pages stay cached"
            assert e.block not in blocks, "physical block mapped twice"
            blocks.add(e.block)
            if e.watermark < self.block_size:
                assert e.ref_count <= 1, "shared partial block"
        free = set(self.pool._free)
        assert len(free) == len(self.pool._free), "free list duplicates"
        assert not (free & blocks), "free block still mapped"
        assert len(free) + len(blocks) == self.num_blocks, "blocks lost"
        assert unref == self.pool.num_evictable, "evictable counter"


class BlockTable:
    """Device-resident ``int32[max_seqs, max_blocks]`` table plus ``seq_lens``,
    updated incrementally: each row remembers which sequence it holds and how
    many of its block ids are already on the device, so a decode step moves
    only the block ids appended since the last sync (a few per step) and the
    lengths, instead of rebuilding the table.

    The host never waits for the device: the delta (flat index, block id) and
    the lengths are written into a pinned staging slot (a ring of ``depth``),
    copied host-to-device with ``non_blocking`` copies -- on ``copy_stream``
    when given, so the transfer overlaps the kernels still running -- and
    scattered into the table on the current (compute) stream, which orders
    the update after every earlier kernel that reads the table and before
    every later one."""

    def __init__(self, max_seqs: int, max_blocks: int, device="cuda", depth: int = 2):
        self.max_seqs, self.max_blocks = max_seqs, max_blocks
        self.device = torch.device(device)
        self.table = torch.zeros((max_seqs, max_blocks), dtype=torch.int32, device=device)
        self.seq_lens = torch.zeros((max_seqs,), dtype=torch.int32, device=device)
        self._row_seq: List[object] = [None] * max_seqs   # the _Seq a row holds
        self._row_n = np.zeros((max_seqs,), dtype=np.int64)  # its block ids already on the device
        self._host_lens = np.zeros((max_seqs,), dtype=np.int32)
        self._depth = max(1, depth)
        self._ring: List[dict] = []
        self._next = 0
        self._grow(max(64, max_seqs))

    def _grow(self, cap: int) -> None:
        """(Re)allocate the staging ring for ``cap`` updates per sync."""
        cuda = self.device.type == "cuda"
        for r in self._ring:   # the old slots may still feed in-flight copies
            if r["copied"] is not None:
                r["copied"].synchronize()
        self._cap = cap
        self._ring = []
        for _ in range(self._depth):
            host = torch.empty((2 * cap + self.max_seqs,), dtype=torch.int64, pin_memory=cuda)
            dev = torch.empty_like(host, device=self.device)
            self._ring.append(dict(host=host, hnp=host.numpy(), dev=dev, copied=None, used=None))

    def sync(self, alloc: BlockAllocator, seq_ids: Sequence, copy_stream=None) -> int:
        """Push the rows of ``seq_ids`` (row i <- seq_ids[i]); returns the
        number of table entries transferred.  Asynchronous (see the class
        docstring); with ``copy_stream`` the current stream waits for the copy
        before the scatter."""
        n = len(seq_ids)
        if n > self.max_seqs:
            raise ValueError("more sequences than table rows")
        idx: List[int] = []
        vals: List[int] = []
        lens = np.empty((n,), dtype=np.int32)
        mb = self.max_blocks
        for i, sid in enumerate(seq_ids):
            s = alloc._seq(sid)
            if self._row_seq[i] is not s:       # row now holds another sequence: rewrite it
                self._row_seq[i] = s
                self._row_n[i] = 0
            b = s.blocks
            k0 = int(self._row_n[i])
            if len(b) > k0:
                if len(b) > mb:
                    raise ValueError("max_blocks too small")
                idx.extend(range(i * mb + k0, i * mb + len(b)))
                vals.extend(b[k0:])
                self._row_n[i] = len(b)
            lens[i] = s.length
        new_lens = not np.array_equal(lens, self._host_lens[:n])
        if not idx and not new_lens:
            return 0
        if len(idx) > self._cap:
            self._grow(max(len(idx), 2 * self._cap))
        r = self._ring[self._next]
        self._next = (self._next + 1) % self._depth
        if r["copied"] is not None:
            r["copied"].synchronize()           # its previous upload (depth syncs ago) has been read
        m, cap = len(idx), self._cap
        h = r["hnp"]
        h[:m] = idx
        h[cap:cap + m] = vals
        h[2 * cap:2 * cap + n] = lens
        cuda = self.device.type == "cuda"
        cur = torch.cuda.current_stream(self.device) if cuda else None
        cs = copy_stream if (cuda and copy_stream is not None) else cur
        if cuda:
            with torch.cuda.stream(cs):
                if r["used"] is not None:
                    cs.wait_event(r["used"])    # the scatter that read this device slot has run
                r["dev"][:m].copy_(r["host"][:m], non_blocking=True)
                r["dev"][cap:cap + m].copy_(r["host"][cap:cap + m], non_blocking=True)
                r["dev"][2 * cap:2 * cap + n].copy_(r["host"][2 * cap:2 * cap + n], non_blocking=True)
                r["copied"] = torch.cuda.Event()
                r["copied"].record(cs)
            if cs is not cur:
                cur.wait_event(r["copied"])
        else:
            r["dev"][:2 * cap + n].copy_(r["host"][:2 * cap + n])
        d = r["dev"]
        if m:
            self.table.view(-1).index_copy_(0, d[:m], d[cap:cap + m].to(torch.int32))
        if new_lens:
            self.seq_lens[:n].copy_(d[2 * cap:2 * cap + n])
            self._host_lens[:n] = lens
        if cuda:
            r["used"] = torch.cuda.Event()
            r["used"].record(cur)
        return m
