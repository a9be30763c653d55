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
    (same formulas as kvq_kernels.cu k_code_off / v_code_off)."""
    code = np.zeros((2, BLOCK_SIZE, HEAD_DIM), dtype=np.int64)
    for t in range(BLOCK_SIZE):
        for d in range(HEAD_DIM):
            j = d >> 4
            code[0, t, d] = t * 128 + ((j ^ ((t & 1) << 2)) << 4) + (d & 15)
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
# Block allocator (host bookkeeping; device pages are copied by kvq_copy_blocks)
# ---------------------------------------------------------------------------
@dataclass
class _Block:
    ref_count: int = 0
    watermark: int = 0


@dataclass
class _Seq:
    blocks: List[int] = field(default_factory=list)
    length: int = 0


class BlockAllocator:
    """Free list + refcounts + per-sequence block lists.

    ``append_slots`` returns the slot ids (``block * 16 + offset``) the new
    tokens occupy; ``fork`` shares every full block of the parent and copies
    its partial tail (partial blocks are exclusive), returning the
    ``(src, dst)`` page copies the caller must apply on the device before the
    child appends.
    """

    def __init__(self, num_blocks: int, block_size: int = BLOCK_SIZE, bytes_per_block: int = 1):
        if num_blocks <= 0:
            raise ValueError("num_blocks must be positive")
        if block_size != BLOCK_SIZE:
            raise ValueError(f"block_size must be {BLOCK_SIZE}")
        self.num_blocks = num_blocks
        self.block_size = block_size
        self.bytes_per_block = bytes_per_block
        self._blocks = [_Block() for _ in range(num_blocks)]
        # LIFO free list, lowest ids handed out first (deterministic replay).
        self._free: List[int] = list(range(num_blocks - 1, -1, -1))
        self._seqs: Dict[object, _Seq] = {}

    # -- introspection ------------------------------------------------------
    @property
    def num_free(self) -> int:
        return len(self._free)

    def ref_count(self, block: int) -> int:
        return self._blocks[block].ref_count

    def watermark(self, block: int) -> int:
        return self._blocks[block].watermark

    def is_full(self, block: int) -> bool:
        return self._blocks[block].watermark == self.block_size

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

    # -- block primitives (the reference's acquire / release / set_watermark)
    def _new_block(self) -> int:
        if not self._free:
            raise CacheThrashError(self.bytes_per_block)
        blk = self._free.pop()
        self._blocks[blk] = _Block(ref_count=0, watermark=0)
        self._acquire(blk)
        return blk

    def _acquire(self, blk: int) -> None:
        e = self._blocks[blk]
        if e.watermark < self.block_size and e.ref_count >= 1:
            raise ValueError("partial block is exclusive")
        e.ref_count += 1

    def _release(self, blk: int) -> None:
        e = self._blocks[blk]
        if e.ref_count <= 0:
            raise ValueError("double release")
        e.ref_count -= 1
        if e.ref_count == 0:
            e.watermark = 0
            self._free.append(blk)

    def _set_watermark(self, blk: int, watermark: int) -> None:
        e = self._blocks[blk]
        if not e.watermark <= watermark <= self.block_size:
            raise ValueError("watermark may only grow, up to block_size")
        e.watermark = watermark

    # -- sequence API ---------------------------------------------------------
    def allocate(self, seq_id) -> None:
        """Register an empty sequence."""
        if seq_id in self._seqs:
            raise ValueError(f"sequence {seq_id!r} already exists")
        self._seqs[seq_id] = _Seq()

    def append_slots(self, seq_id, n: int) -> List[int]:
        """Reserve ``n`` token slots at the end of ``seq_id``.

        Atomic: on :class:`CacheThrashError` nothing changes."""
        if n < 0:
            raise ValueError("n must be >= 0")
        s = self._seq(seq_id)
        bs = self.block_size
        tail_room = (bs - s.length % bs) % bs if s.blocks else 0
        new_blocks = -(-(n - tail_room) // bs) if n > tail_room else 0
        if new_blocks > len(self._free):
            raise CacheThrashError((new_blocks - len(self._free)) * self.bytes_per_block)
        slots: List[int] = []
        pos = s.length
        for _ in range(n):
            if pos % bs == 0 and pos // bs == len(s.blocks):
                s.blocks.append(self._new_block())
            blk = s.blocks[pos // bs]
            # Appends only ever land in an exclusively-owned (partial) block.
            assert self._blocks[blk].ref_count == 1
            slots.append(blk * bs + pos % bs)
            pos += 1
            self._set_watermark(blk, pos - (pos - 1) // bs * bs)
        s.length = pos
        return slots

    def fork(self, parent_id, child_id) -> List[Tuple[int, int]]:
        """New sequence sharing the parent's full blocks; the partial tail is
        copied (``(src, dst)`` page copies returned for the device)."""
        if child_id in self._seqs:
            raise ValueError(f"sequence {child_id!r} already exists")
        p = self._seq(parent_id)
        copies: List[Tuple[int, int]] = []
        blocks: List[int] = []
        partial_tail = p.blocks and not self.is_full(p.blocks[-1])
        if partial_tail and not self._free:
            raise CacheThrashError(self.bytes_per_block)
        for blk in p.blocks[:-1] if partial_tail else p.blocks:
            self._acquire(blk)  # full: shareable
            blocks.append(blk)
        if partial_tail:
            src = p.blocks[-1]
            dst = self._new_block()
            self._set_watermark(dst, self.watermark(src))
            blocks.append(dst)
            copies.append((src, dst))
        self._seqs[child_id] = _Seq(blocks=blocks, length=p.length)
        return copies

    def free(self, seq_id) -> None:
        s = self._seqs.pop(seq_id, None)
        if s is None:
            raise KeyError(f"unknown sequence {seq_id!r}")
        for blk in s.blocks:
            self._release(blk)

    # -- device views ---------------------------------------------------------
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

    # -- invariants (for tests; cf. test_tiered_cache.py:243-327) ---------------
    def check_invariants(self) -> None:
        counts = [0] * self.num_blocks
        for s in self._seqs.values():
            assert len(s.blocks) == -(-s.length // self.block_size), "block count vs length"
            for i, blk in enumerate(s.blocks):
                counts[blk] += 1
                full = (i + 1) * self.block_size <= s.length
                wm = self.block_size if full else s.length - i * self.block_size
                assert self._blocks[blk].watermark == wm, "watermark mismatch"
        free = set(self._free)
        assert len(free) == len(self._free), "free list duplicates"
        for blk, e in enumerate(self._blocks):
            assert e.ref_count == counts[blk], f"refcount mismatch on block {blk}"
            assert (e.ref_count == 0) == (blk in free), "free list vs refcount"
            if e.watermark < self.block_size:
                assert e.ref_count <= 1, "shared partial block"


class BlockTable:
    """Device-resident ``int32[max_seqs, max_blocks]`` table plus ``seq_lens``,
    updated incrementally (only changed entries cross host->device)."""

    def __init__(self, max_seqs: int, max_blocks: int, device="cuda"):
        self.max_seqs, self.max_blocks = max_seqs, max_blocks
        self.table = torch.zeros((max_seqs, max_blocks), dtype=torch.int32, device=device)
        self.seq_lens = torch.zeros((max_seqs,), dtype=torch.int32, device=device)
        self._host = np.zeros((max_seqs, max_blocks), dtype=np.int32)
        self._host_lens = np.zeros((max_seqs,), dtype=np.int32)

    def sync(self, alloc: BlockAllocator, seq_ids: Sequence) -> int:
        """Push the rows of ``seq_ids`` (row i <- seq_ids[i]); returns the
        number of table entries transferred."""
        tab = alloc.block_table(seq_ids, self.max_blocks)
        lens = alloc.seq_lens(seq_ids)
        n = len(seq_ids)
        diff = np.nonzero(tab != self._host[:n])
        moved = 0
        if diff[0].size:
            upd = np.stack([diff[0], diff[1], tab[diff]], axis=1).astype(np.int64)
            u = torch.from_numpy(upd).to(self.table.device, non_blocking=False)
            self.table[u[:, 0], u[:, 1]] = u[:, 2].to(torch.int32)
            self._host[:n] = tab
            moved = int(diff[0].size)
        if not np.array_equal(lens, self._host_lens[:n]):
            self.seq_lens[:n].copy_(torch.from_numpy(lens))
            self._host_lens[:n] = lens
        return moved
