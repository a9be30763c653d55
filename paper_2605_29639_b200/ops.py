"""Python entry points of the path (the plugin surface), each a thin call
through the C ABI of libkvq.so.  There is no CPU fallback: a tensor that is not
on a CUDA device, or a missing library, raises.

* :func:`quantize_append`       -> ``kvq_quant_append``  (K1)
* :func:`paged_decode_attention` -> ``kvq_decode_attn``  (K2 + fused combine)
* :func:`paged_decode_attention_gathered` -> ``kvq_decode_attn_peer`` (K2 with
  the KV-head output all-gather fused in, over peer memory)
* :func:`decode_step`            -> ``kvq_decode_step``  (K1 + K2 in one call, PDL-overlapped)
* :func:`copy_blocks`            -> ``kvq_copy_blocks``  (copy-on-write pages)
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from .cache import PagedKVCache

_WS_CACHE: Dict[Tuple[int, int], list] = {}


def _stream_handle(device: torch.device) -> int:
    """Raw cudaStream_t of the current stream (torch's C accessor when present:
    ``torch.cuda.current_stream()`` costs several microseconds per call)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return raw(idx) if raw is not None else torch.cuda.current_stream(device).cuda_stream


def check_device_errors(device=None) -> None:
    """Raise ``ValueError`` if a kernel met an out-of-range block id, sequence
    length or slot since the last check (``kvq_check_device_errors``: the
    kernels skip or clamp such input instead of faulting, and report it here).
    Synchronizes the current stream: a validation call, not for the step path."""
    import ctypes
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    bits = ctypes.c_uint32(0)
    _lib.check("kvq_check_device_errors", _lib.load().kvq_check_device_errors(_stream_handle(dev), ctypes.byref(bits)))


def profile_next_decode(span: Optional[torch.Tensor]) -> None:
    """Make this thread's next K2 launch record its grid span (start / end
    %globaltimer, ns) into ``span`` (a CUDA uint64/int64 tensor of 2, preset
    to (max, 0)); ``None`` cancels (``kvq_profile_next_decode``).  Capturable."""
    if span is not None:
        _require_cuda("profile_next_decode", span)
        if span.dtype not in (torch.int64, torch.uint64) or span.numel() < 2:
            raise ValueError("profile_next_decode: span must hold 2 x 64-bit")
    _lib.check("kvq_profile_next_decode",
               _lib.load().kvq_profile_next_decode(span.data_ptr() if span is not None else None))


def profile_next_append(span: Optional[torch.Tensor]) -> None:
    """The same for this thread's next K1 launch (``kvq_profile_next_append``)."""
    if span is not None:
        _require_cuda("profile_next_append", span)
        if span.dtype not in (torch.int64, torch.uint64) or span.numel() < 2:
            raise ValueError("profile_next_append: span must hold 2 x 64-bit")
    _lib.check("kvq_profile_next_append",
               _lib.load().kvq_profile_next_append(span.data_ptr() if span is not None else None))


def _require_cuda(name: str, *ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise ValueError(f"{name}: tensors must be on a CUDA device (no CPU fallback)")


def _check_append(fn: str, cache: PagedKVCache, k: torch.Tensor, v: torch.Tensor,
                  slot_mapping: torch.Tensor) -> None:
    _require_cuda(fn, k, v, slot_mapping, cache.pool)
    spec = cache.spec
    for name, t in (("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or t.dim() != 3 or t.shape[1:] != (spec.num_kv_heads, 128):
            raise ValueError(f"{fn}: {name} must be bf16 [T, {spec.num_kv_heads}, 128]")
        if t.stride(2) != 1 or t.stride(1) != 128:
            raise ValueError(f"{fn}: {name} heads must be contiguous")
    if k.shape[0] != v.shape[0] or slot_mapping.shape != (k.shape[0],):
        raise ValueError(f"{fn}: T mismatch")
    if slot_mapping.dtype != torch.int32 or not slot_mapping.is_contiguous():
        raise ValueError(f"{fn}: slot_mapping must be contiguous int32")


def quantize_append(cache: PagedKVCache, k: torch.Tensor, v: torch.Tensor,
                    slot_mapping: torch.Tensor) -> None:
    """Quantize new K/V rows and scatter them into their pages.

    k, v: bf16 ``[T, Hkv, 128]`` (token stride may exceed ``Hkv*128``, e.g.
    slices of a fused QKV buffer); slot_mapping: int32 ``[T]`` with
    ``block * 16 + offset`` (negative = skip)."""
    _check_append("quantize_append", cache, k, v, slot_mapping)
    spec = cache.spec
    lib = _lib.load()
    st = lib.kvq_quant_append(k.data_ptr(), v.data_ptr(), k.stride(0), v.stride(0),
                              slot_mapping.data_ptr(), k.shape[0], spec.num_kv_heads,
                              spec.kv_dtype_id, cache.pool.data_ptr(), cache.num_blocks,
                              _stream_handle(k.device))
    _lib.check("kvq_quant_append", st)


def pages_per_split(batch: int, num_kv_heads: int, total_pages: int, max_blocks: int, rows: int = 8) -> int:
    """Split-KV pages per split (``kvq_decode_pages_per_split_rows``); ``rows``
    = query rows per kv head, (Hq / Hkv) * q_len."""
    return int(_lib.load().kvq_decode_pages_per_split_rows(batch, num_kv_heads, rows, total_pages, max_blocks))


def workspace_bytes(batch: int, num_q_heads: int, num_kv_heads: int, max_splits: int) -> int:
    return int(_lib.load().kvq_decode_workspace_bytes(batch, num_q_heads, num_kv_heads, max_splits))


def _workspace(device: torch.device, nbytes: int, counter_bytes: int) -> torch.Tensor:
    """Per-(device, stream) cached workspace.  Its first ``counter_bytes`` (the
    split-combine arrival counters, offset 0) must be zero on entry.  The
    kernel leaves its own counters zero, but writes partials right after them,
    so only the LAST call's counter region is known clean: a call with a
    larger batch x kv-head count than the last one re-zeroes its prefix (a
    large -> small -> large sequence would otherwise find the small call's
    partials in its counters)."""
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           _stream_handle(device))
    ent = _WS_CACHE.get(key)
    if ent is None or ent[0].numel() < nbytes:
        ent = [torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device), counter_bytes]
        _WS_CACHE[key] = ent
    elif counter_bytes > ent[1]:
        ent[0][:counter_bytes].zero_()
    ent[1] = counter_bytes
    return ent[0]


def paged_decode_attention(q: torch.Tensor, cache: PagedKVCache, block_table: torch.Tensor,
                           seq_lens: torch.Tensor, *, sm_scale: Optional[float] = None,
                           pages_per_split: Optional[int] = None,
                           total_pages: Optional[int] = None,
                           out: Optional[torch.Tensor] = None,
                           out_dtype: torch.dtype = torch.bfloat16, head_major: bool = False,
                           workspace: Optional[torch.Tensor] = None,
                           num_splits: Optional[int] = None) -> torch.Tensor:
    """GQA decode attention of one query token per sequence over the paged,
    quantized KV cache -- or, with ``q`` of shape ``[B, q_len, Hq, 128]``, of
    ``q_len`` new tokens per sequence (speculative scoring / MTP), causal
    among them: token i sees ``seq_lens[b] - (q_len - 1 - i)`` tokens, so
    ``seq_lens`` counts all of them (they must already be appended).

    q: bf16 ``[B, Hq, 128]``; block_table: int32 ``[B, max_blocks]``;
    seq_lens: int32 ``[B]``.  Returns ``[B, Hq, 128]`` (or ``[Hq, B, 128]``
    with ``head_major=True``, the layout the KV-head all-gather wants) in
    ``out_dtype`` (bf16 or fp32).  ``total_pages`` (sum of per-sequence
    pages, when the host knows it) sharpens the split-KV geometry;
    ``num_splits`` (SURVEY §8b's name) instead fixes the split count of the
    longest sequence: ``pages_per_split = ceil(max_blocks / num_splits)``.
    ``workspace`` (uint8, ``workspace_bytes(...)`` long, zeroed before first
    use; the kernel leaves it reusable for the same batch x kv-head count)
    defaults to a per-stream cached buffer -- pass your own when capturing
    the call in a CUDA graph, so eager calls of other shapes on the stream
    cannot dirty the graph's split-combine counters."""
    _require_cuda("paged_decode_attention", q, block_table, seq_lens, cache.pool)
    spec = cache.spec
    multi = q.dim() == 4  # [B, q_len, Hq, 128]: speculative scoring / MTP (causal among the new tokens)
    if q.dtype != torch.bfloat16 or q.dim() not in (3, 4) or q.shape[-1] != 128 or q.stride(-1) != 1:
        raise ValueError("paged_decode_attention: q must be bf16 [B, Hq, 128] or [B, q_len, Hq, 128]")
    B, Hq = q.shape[0], q.shape[-2]
    q_len = q.shape[1] if multi else 1
    if q.stride(-2) != 128 or (multi and q.stride(1) != Hq * 128):
        raise ValueError("paged_decode_attention: q heads (and query tokens) must be contiguous")
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B \
            or not block_table.is_contiguous():
        raise ValueError("paged_decode_attention: block_table must be contiguous int32 [B, max_blocks]")
    if seq_lens.dtype != torch.int32 or seq_lens.shape != (B,) or not seq_lens.is_contiguous():
        raise ValueError("paged_decode_attention: seq_lens must be contiguous int32 [B]")
    if out_dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("paged_decode_attention: out_dtype must be bf16 or fp32")
    max_blocks = block_table.shape[1]
    if head_major:
        shape = (Hq, B * q_len, 128)
    else:
        shape = (B, q_len, Hq, 128) if multi else (B, Hq, 128)
    if out is None:
        out = torch.empty(shape, dtype=out_dtype, device=q.device)
    elif tuple(out.shape) != shape or out.dtype != out_dtype or not out.is_contiguous():
        raise ValueError(f"paged_decode_attention: out must be contiguous {out_dtype} {shape}")
    if B == 0:
        return out
    if sm_scale is None:
        sm_scale = 1.0 / math.sqrt(128)
    lib = _lib.load()
    if num_splits is not None:
        if pages_per_split is not None or num_splits < 1:
            raise ValueError("paged_decode_attention: give num_splits >= 1 or pages_per_split, not both")
        pages_per_split = -(-max_blocks // int(num_splits))
    pps = pages_per_split or lib.kvq_decode_pages_per_split_rows(
        B, spec.num_kv_heads, Hq // spec.num_kv_heads * q_len,
        total_pages if total_pages is not None else B * max_blocks, max_blocks)
    max_splits = -(-max_blocks // pps)
    nbytes = lib.kvq_decode_workspace_bytes(B, Hq * q_len, spec.num_kv_heads, max_splits)
    if workspace is None:
        workspace = _workspace(q.device, nbytes, ((B * spec.num_kv_heads * 4 + 255) // 256) * 256)
    elif workspace.numel() * workspace.element_size() < nbytes:
        raise ValueError(f"paged_decode_attention: workspace needs {nbytes} bytes")
    st = lib.kvq_decode_attn_mq(
        q.data_ptr(), q.stride(0), q_len, cache.pool.data_ptr(), cache.num_blocks,
        block_table.data_ptr(), max_blocks, seq_lens.data_ptr(), B, Hq, spec.num_kv_heads,
        spec.kv_dtype_id, float(sm_scale), int(pps), workspace.data_ptr(),
        workspace.numel() * workspace.element_size(), out.data_ptr(),
        _lib.KVQ_OUT_F32 if out_dtype == torch.float32 else _lib.KVQ_OUT_BF16,
        _lib.KVQ_OUT_HBD if head_major else _lib.KVQ_OUT_BHD, _stream_handle(q.device))
    _lib.check("kvq_decode_attn", st)
    return out


def paged_decode_attention_gathered(q: torch.Tensor, cache: PagedKVCache, block_table: torch.Tensor,
                                    seq_lens: torch.Tensor, peer, slot: int = 0, *,
                                    sm_scale: Optional[float] = None,
                                    pages_per_split: Optional[int] = None,
                                    total_pages: Optional[int] = None,
                                    workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """KV-head-sharded decode attention with the output all-gather fused into
    K2 (``kvq_decode_attn_peer``): this rank attends its sequences over its
    heads (``q``: bf16 ``[B_r, Hq_r, 128]``) and every finished row is stored
    into all ranks' copies of the global output.  ``peer`` is a
    :class:`paper_2605_29639_b200.shard.PeerOutput`; returns its ``out(slot)``
    (``[Hq, B, 128]`` bf16), complete on this rank once the launch completes."""
    _require_cuda("paged_decode_attention_gathered", q, block_table, seq_lens, cache.pool)
    spec = cache.spec
    if q.dtype != torch.bfloat16 or q.dim() != 3 or q.shape[-1] != 128 or q.stride(-1) != 1 \
            or q.stride(-2) != 128:
        raise ValueError("paged_decode_attention_gathered: q must be bf16 [B, Hq, 128] with contiguous heads")
    B, Hq = q.shape[0], q.shape[1]
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B \
            or not block_table.is_contiguous():
        raise ValueError("paged_decode_attention_gathered: block_table must be contiguous int32 [B, max_blocks]")
    if seq_lens.dtype != torch.int32 or seq_lens.shape != (B,) or not seq_lens.is_contiguous():
        raise ValueError("paged_decode_attention_gathered: seq_lens must be contiguous int32 [B]")
    if not 0 <= slot < peer.slots:
        raise ValueError("paged_decode_attention_gathered: bad slot")
    if peer.plan.q_range[1] - peer.plan.q_range[0] != Hq:
        raise ValueError("paged_decode_attention_gathered: q heads do not match the shard plan")
    if B == 0:
        return peer.out(slot)
    if sm_scale is None:
        sm_scale = 1.0 / math.sqrt(128)
    lib = _lib.load()
    max_blocks = block_table.shape[1]
    pps = pages_per_split or lib.kvq_decode_pages_per_split_rows(
        B, spec.num_kv_heads, Hq // spec.num_kv_heads,
        total_pages if total_pages is not None else B * max_blocks, max_blocks)
    max_splits = -(-max_blocks // pps)
    nbytes = lib.kvq_decode_workspace_bytes(B, Hq, spec.num_kv_heads, max_splits)
    if workspace is None:
        workspace = _workspace(q.device, nbytes, ((B * spec.num_kv_heads * 4 + 255) // 256) * 256)
    elif workspace.numel() * workspace.element_size() < nbytes:
        raise ValueError(f"paged_decode_attention_gathered: workspace needs {nbytes} bytes")
    import ctypes
    st = lib.kvq_decode_attn_peer(
        q.data_ptr(), q.stride(0), cache.pool.data_ptr(), cache.num_blocks, block_table.data_ptr(),
        max_blocks, seq_lens.data_ptr(), B, Hq, spec.num_kv_heads, spec.kv_dtype_id, float(sm_scale),
        int(pps), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        ctypes.addressof(peer.descs[slot]), _stream_handle(q.device))
    _lib.check("kvq_decode_attn_peer", st)
    return peer.out(slot)


def decode_step(cache: PagedKVCache, k: torch.Tensor, v: torch.Tensor, slot_mapping: torch.Tensor,
                q: torch.Tensor, block_table: torch.Tensor, seq_lens: torch.Tensor, *,
                sm_scale: Optional[float] = None, pages_per_split: Optional[int] = None,
                total_pages: Optional[int] = None, out: Optional[torch.Tensor] = None,
                out_dtype: torch.dtype = torch.bfloat16, head_major: bool = False,
                workspace: Optional[torch.Tensor] = None, peer=None, slot: int = 0,
                append_tail_only: bool = False, fused_append: bool = False) -> torch.Tensor:
    """One decode step in one call (``kvq_decode_step``): :func:`quantize_append`
    of the new rows, then :func:`paged_decode_attention` (or, with ``peer``,
    :func:`paged_decode_attention_gathered`), with K2 launched behind K1 by
    programmatic dependent launch so its launch and prologue overlap K1.
    Same arguments and results as the two calls in sequence.

    ``append_tail_only=True`` promises that, for every attended sequence, the
    appended rows lie in its last page (true of a decode step's new token;
    rows of sequences not in ``q``, e.g. prefill chunks, may go anywhere):
    K2 then streams all other pages while K1 runs.

    ``q`` of shape ``[B, q_len, Hq, 128]`` makes it a speculative-decoding
    verify step (``kvq_decode_step_mq``): the ``q_len`` draft tokens' rows are
    appended and scored causally, as :func:`paged_decode_attention` does for a
    4-D ``q`` (``append_tail_only`` does not apply; no ``peer``).

    ``fused_append=True`` (``KVQ_STEP_FUSED_APPEND``) launches no K1: row b of
    ``k`` / ``v`` must be sequence b's newest token (position
    ``seq_lens[b] - 1``, slot ``slot_mapping[b]``), and the K2 CTA holding that
    page quantizes it itself -- same pool bytes and output as the two calls.
    One query token per sequence, no ``peer``."""
    _check_append("decode_step", cache, k, v, slot_mapping)
    _require_cuda("decode_step", q, block_table, seq_lens)
    spec = cache.spec
    multi = q.dim() == 4
    if q.dtype != torch.bfloat16 or q.dim() not in (3, 4) or q.shape[-1] != 128 or q.stride(-1) != 1 \
            or q.stride(-2) != 128:
        raise ValueError("decode_step: q must be bf16 [B, Hq, 128] or [B, q_len, Hq, 128], contiguous heads")
    B, Hq = q.shape[0], q.shape[-2]
    q_len = q.shape[1] if multi else 1
    if multi and (q.stride(1) != Hq * 128 or peer is not None):
        raise ValueError("decode_step: multi-query q needs contiguous tokens and no peer gather")
    if fused_append and (multi or peer is not None or k.shape[0] != B):
        raise ValueError("decode_step: fused_append needs one new row per sequence (T == B), "
                         "one query token and no peer gather")
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B \
            or not block_table.is_contiguous():
        raise ValueError("decode_step: block_table must be contiguous int32 [B, max_blocks]")
    if seq_lens.dtype != torch.int32 or seq_lens.shape != (B,) or not seq_lens.is_contiguous():
        raise ValueError("decode_step: seq_lens must be contiguous int32 [B]")
    import ctypes
    desc = None
    if peer is not None:
        if not 0 <= slot < peer.slots or peer.plan.q_range[1] - peer.plan.q_range[0] != Hq:
            raise ValueError("decode_step: bad slot, or q heads do not match the shard plan")
        out, out_dtype, head_major = peer.out(slot), torch.bfloat16, True
        desc = ctypes.addressof(peer.descs[slot])
    else:
        shape = (Hq, B * q_len, 128) if head_major else ((B, q_len, Hq, 128) if multi else (B, Hq, 128))
        if out is None:
            out = torch.empty(shape, dtype=out_dtype, device=q.device)
        elif tuple(out.shape) != shape or out.dtype != out_dtype or not out.is_contiguous():
            raise ValueError(f"decode_step: out must be contiguous {out_dtype} {shape}")
        if out_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("decode_step: out_dtype must be bf16 or fp32")
    if sm_scale is None:
        sm_scale = 1.0 / math.sqrt(128)
    lib = _lib.load()
    max_blocks = block_table.shape[1]
    pps = pages_per_split or lib.kvq_decode_pages_per_split_rows(
        B, spec.num_kv_heads, Hq // spec.num_kv_heads * q_len,
        total_pages if total_pages is not None else B * max_blocks, max_blocks)
    max_splits = -(-max_blocks // pps)
    nbytes = lib.kvq_decode_workspace_bytes(B, Hq * q_len, spec.num_kv_heads, max_splits)
    if workspace is None:
        workspace = _workspace(q.device, nbytes, ((B * spec.num_kv_heads * 4 + 255) // 256) * 256)
    elif workspace.numel() * workspace.element_size() < nbytes:
        raise ValueError(f"decode_step: workspace needs {nbytes} bytes")
    st = lib.kvq_decode_step_mq(
        k.data_ptr(), v.data_ptr(), k.stride(0), v.stride(0), slot_mapping.data_ptr(), k.shape[0],
        q.data_ptr(), q.stride(0), q_len, cache.pool.data_ptr(), cache.num_blocks, block_table.data_ptr(),
        max_blocks,
        seq_lens.data_ptr(), B, Hq, spec.num_kv_heads, spec.kv_dtype_id, float(sm_scale), int(pps),
        workspace.data_ptr(), workspace.numel() * workspace.element_size(), out.data_ptr(),
        _lib.KVQ_OUT_F32 if out_dtype == torch.float32 else _lib.KVQ_OUT_BF16,
        _lib.KVQ_OUT_HBD if head_major else _lib.KVQ_OUT_BHD, desc,
        (_lib.KVQ_STEP_APPEND_TAIL_ONLY if append_tail_only else 0)
        | (_lib.KVQ_STEP_FUSED_APPEND if fused_append else 0), _stream_handle(q.device))
    _lib.check("kvq_decode_step", st)
    return out


def copy_blocks(cache: PagedKVCache, pairs: Sequence[Tuple[int, int]]) -> None:
    """Apply ``(src, dst)`` whole-block page copies (fork copy-on-write)."""
    if not pairs:
        return
    _require_cuda("copy_blocks", cache.pool)
    t = torch.as_tensor(np.asarray(pairs, dtype=np.int32).reshape(-1), device=cache.device)
    st = _lib.load().kvq_copy_blocks(cache.pool.data_ptr(), cache.num_blocks,
                                     cache.spec.num_kv_heads, t.data_ptr(), len(pairs),
                                     _stream_handle(cache.device))
    _lib.check("kvq_copy_blocks", st)
