"""Quantized prefill->decode KV transfer.

The reference moves a request's KV from the prefill worker to the decode
worker in ``ClusterSim._migrate_kv`` (``simulator.py:485-497``).  It prices
the move as one RDMA transfer of ``kv_bytes(seq_len)`` (``simulator.py:461-463``).
The paper ships this over NCCL (``PAPER.md:620``).  Here the wire format is
the page format itself: 4224 bytes per (block, kv head), holding 8-bit codes
plus fp32 scales.  That is 264 B per token per head, against 512 B for bf16
K/V, or 51.6 %.  The receiver does not re-quantize, so the decode worker's
pages are bit-identical to the prefill worker's.

Transport is ``torch.distributed`` point-to-point: NCCL over NVLink between
GPUs.  Pages are gathered into one contiguous staging buffer by one
``kvq_gather_blocks`` launch and scattered on arrival by one
``kvq_scatter_blocks`` launch (native page-copy kernel).  Both are device-side
copies, so the only host<->device traffic is the 16-byte header.  The page
copies are the only pluggable part (``export=`` / ``import_=``): the gloo tests
on CPU pass their own host copies; the product path is CUDA-only.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib
from ._lib import PAGE_BYTES
from .cache import BlockAllocator, PagedKVCache


def wire_bytes_per_token(num_kv_heads: int) -> int:
    """Bytes on the wire per token per layer: codes + fp32 scales."""
    return num_kv_heads * PAGE_BYTES // 16


def _ids(block_ids, device) -> torch.Tensor:
    """Block ids as a device int32 tensor (a device tensor passes through)."""
    if isinstance(block_ids, torch.Tensor) and block_ids.is_cuda and block_ids.dtype == torch.int32:
        return block_ids.contiguous()
    import numpy as np
    return torch.from_numpy(np.asarray(block_ids, dtype=np.int32)).to(device)


def export_pages(cache: PagedKVCache, block_ids: Sequence[int]) -> torch.Tensor:
    """``uint8[n, Hkv, 4224]`` copy of the given blocks' pages (all heads):
    ``kvq_gather_blocks`` on the device."""
    n, hkv = len(block_ids), cache.spec.num_kv_heads
    if not cache.pool.is_cuda:
        raise ValueError("export_pages: the pool must be a CUDA tensor")
    out = torch.empty((n, hkv, PAGE_BYTES), dtype=torch.uint8, device=cache.device)
    if n:
        idx = _ids(block_ids, cache.device)
        st = _lib.load().kvq_gather_blocks(cache.pool.data_ptr(), cache.num_blocks, hkv, idx.data_ptr(), n,
                                           out.data_ptr(), torch.cuda.current_stream(cache.device).cuda_stream)
        _lib.check("kvq_gather_blocks", st)
    return out


def import_pages(cache: PagedKVCache, block_ids: Sequence[int], pages: torch.Tensor) -> None:
    """Scatter a packed page buffer into the given blocks (``kvq_scatter_blocks``)."""
    if pages.shape[1:] != cache.pool.shape[1:] or pages.shape[0] != len(block_ids):
        raise ValueError("page buffer does not match the destination pool")
    if not cache.pool.is_cuda or not pages.is_cuda or not pages.is_contiguous() or pages.dtype != torch.uint8:
        raise ValueError("import_pages: pages must be a contiguous uint8 CUDA tensor")
    n = len(block_ids)
    if n:
        idx = _ids(block_ids, cache.device)
        st = _lib.load().kvq_scatter_blocks(cache.pool.data_ptr(), cache.num_blocks, cache.spec.num_kv_heads,
                                            idx.data_ptr(), n, pages.data_ptr(),
                                            torch.cuda.current_stream(cache.device).cuda_stream)
        _lib.check("kvq_scatter_blocks", st)


def send_sequence(cache: PagedKVCache, alloc: BlockAllocator, seq_id, dst: int,
                  group: Optional[dist.ProcessGroup] = None, export=export_pages) -> int:
    """Send ``seq_id``'s length and pages to rank ``dst``; returns payload bytes."""
    blocks = alloc.block_ids(seq_id)
    header = torch.tensor([alloc.seq_len(seq_id), len(blocks)], dtype=torch.int64, device=cache.device)
    dist.send(header, dst, group=group)
    if blocks:
        pages = export(cache, blocks)
        dist.send(pages, dst, group=group)
        return pages.numel()
    return 0


def recv_sequence(cache: PagedKVCache, alloc: BlockAllocator, seq_id, src: int,
                  group: Optional[dist.ProcessGroup] = None, import_=import_pages) -> List[int]:
    """Receive a sequence from rank ``src`` into freshly allocated blocks of
    this worker's pool (``alloc.allocate`` + ``append_slots``); returns the
    new block ids.  Raises :class:`CacheThrashError` (nothing received into
    the pool) when the blocks do not fit."""
    header = torch.empty(2, dtype=torch.int64, device=cache.device)
    dist.recv(header, src, group=group)
    length, nblocks = (int(x) for x in header.tolist())
    pages = torch.empty((nblocks, cache.spec.num_kv_heads, PAGE_BYTES), dtype=torch.uint8,
                        device=cache.device)
    if nblocks:
        dist.recv(pages, src, group=group)
    alloc.allocate(seq_id)
    try:
        alloc.append_slots(seq_id, length)
    except Exception:
        alloc.free(seq_id)
        raise
    blocks = alloc.block_ids(seq_id)
    if len(blocks) != nblocks:
        raise RuntimeError("sender and receiver disagree on the block count")
    if nblocks:
        import_(cache, blocks, pages)
    return blocks
