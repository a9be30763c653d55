"""KV-head tensor parallelism for the decode path (one process per GPU).

Rank r of P owns KV heads ``[r*Hkv/P, (r+1)*Hkv/P)`` and the query heads of
their GQA groups ``[r*Hq/P, (r+1)*Hq/P)``; block tables and sequence lengths
are replicated (block ids are identical on every rank, each rank's pool holds
only its heads).  Append and attention need no communication; the only
exchange is one all-gather of the per-rank outputs.  Outputs are produced
head-major (``[Hq/P, B, 128]``), so NCCL's rank-major concatenation is already
``[Hq, B, 128]`` and no transpose kernel runs.

The reference models TP only as scalar cost parameters (SPEC.md:8,
PAPER.md:440-450); this module is the executed counterpart for the attention
op.  With P == 1 there is no collective at all.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def head_partition(num_q_heads: int, num_kv_heads: int, world: int, rank: int
                   ) -> Tuple[Tuple[int, int], Tuple[int, int]]:
    """((kv_lo, kv_hi), (q_lo, q_hi)) owned by ``rank``."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if num_q_heads % num_kv_heads:
        raise ValueError("num_q_heads must be a multiple of num_kv_heads")
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads cannot be split over {world} ranks")
    kv = num_kv_heads // world
    g = num_q_heads // num_kv_heads
    return (rank * kv, (rank + 1) * kv), (rank * kv * g, (rank + 1) * kv * g)


def lpt_assign(lengths: Sequence[int], bins: int) -> List[List[int]]:
    """Longest-processing-time greedy balance of sequences (by context length,
    i.e. KV bytes) over ``bins``: longest first, each to the least-loaded bin,
    ties to the lowest bin -- the reference's file balancer
    (``load_planner.py:145-157``) applied to KV tokens.  Bins come back sorted."""
    loads = [0] * bins
    out: List[List[int]] = [[] for _ in range(bins)]
    for i in sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i)):
        j = min(range(bins), key=lambda j: (loads[j], j))
        loads[j] += int(lengths[i])
        out[j].append(i)
    return [sorted(x) for x in out]


@dataclass
class ShardPlan:
    """2-D (KV head group x batch part) partition for one rank.

    ``h_split = gcd(Hkv, P)`` head groups x ``b_split = P / h_split`` batch
    parts; rank = head_group * b_split + batch_part.  With Hkv % P == 0 this is
    the plain KV-head split (b_split = 1).  C4 (Hkv = 4, P = 8) gets 4 head
    groups x 2 token-balanced batch halves, so no GPU idles and no extra
    exchange is needed beyond the one all-gather."""
    world: int
    rank: int
    h_split: int
    b_split: int
    kv_range: Tuple[int, int]
    q_range: Tuple[int, int]
    seqs: np.ndarray                 # global sequence ids this rank attends (sorted)
    parts: List[List[int]]           # sequences of every batch part
    b_max: int                       # padded per-rank batch for the all-gather

    @property
    def num_q_local(self) -> int:
        return self.q_range[1] - self.q_range[0]

    def gather_index(self, num_q_heads: int, batch: int) -> np.ndarray:
        """Flat row index into the gathered ``[P, Hq_loc, b_max]`` buffer for
        every output row ``(h, b)`` of ``[Hq, B]``."""
        hq_loc = num_q_heads // self.h_split
        idx = np.zeros((num_q_heads, batch), dtype=np.int64)
        for hg in range(self.h_split):
            for bs, seqs in enumerate(self.parts):
                rk = hg * self.b_split + bs
                for pos, b in enumerate(seqs):
                    for hl in range(hq_loc):
                        idx[hg * hq_loc + hl, b] = (rk * hq_loc + hl) * self.b_max + pos
        return idx.reshape(-1)


def plan_shards(num_q_heads: int, num_kv_heads: int, world: int, rank: int,
                seq_lens: Sequence[int]) -> ShardPlan:
    if num_q_heads % num_kv_heads:
        raise ValueError("num_q_heads must be a multiple of num_kv_heads")
    h_split = math.gcd(num_kv_heads, world)
    b_split = world // h_split
    if len(seq_lens) < b_split:
        raise ValueError("fewer sequences than batch parts")
    hg, bs = divmod(rank, b_split)
    kv = num_kv_heads // h_split
    g = num_q_heads // num_kv_heads
    parts = lpt_assign(seq_lens, b_split)
    return ShardPlan(world, rank, h_split, b_split, (hg * kv, (hg + 1) * kv),
                     (hg * kv * g, (hg + 1) * kv * g), np.asarray(parts[bs], dtype=np.int64),
                     parts, max(len(x) for x in parts))


class ShardedDecodeAttention:
    """Decode attention over KV-head shards.

    ``local_attention(q_local) -> out_local[Hq/P, B, 128]`` runs this rank's
    heads (the CUDA path by default; tests on CPU/gloo inject the oracle, the
    product never does).  ``__call__(q_full)`` slices this rank's query heads,
    runs the local op and all-gathers to ``[Hq, B, 128]``.
    """

    def __init__(self, num_q_heads: int, num_kv_heads: int,
                 group: Optional[dist.ProcessGroup] = None,
                 local_attention: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.Hq, self.Hkv = num_q_heads, num_kv_heads
        (self.kv_lo, self.kv_hi), (self.q_lo, self.q_hi) = head_partition(
            num_q_heads, num_kv_heads, self.world, self.rank)
        self.local_attention = local_attention

    def local_kv_slice(self, x: torch.Tensor, dim: int = 1) -> torch.Tensor:
        """This rank's KV heads of a ``[T, Hkv, d]`` tensor (for the append)."""
        return x.narrow(dim, self.kv_lo, self.kv_hi - self.kv_lo)

    def local_q_slice(self, q: torch.Tensor) -> torch.Tensor:
        return q.narrow(1, self.q_lo, self.q_hi - self.q_lo)

    def __call__(self, q: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if self.local_attention is None:
            raise RuntimeError("no local attention op configured")
        q_loc = self.local_q_slice(q).contiguous()
        o_loc = self.local_attention(q_loc)
        if tuple(o_loc.shape) != (self.q_hi - self.q_lo, q.shape[0], q.shape[2]):
            raise ValueError("local attention must return head-major [Hq/P, B, d]")
        if self.world == 1:
            return o_loc
        if out is None:
            out = torch.empty((self.Hq, q.shape[0], q.shape[2]), dtype=o_loc.dtype,
                              device=o_loc.device)
        dist.all_gather_into_tensor(out, o_loc.contiguous(), group=self.group)
        return out


class OutputGather:
    """Assembles ``[Hq, B, d]`` from every rank's head-major ``[Hq_loc, B_r, d]``:
    one all-gather of equal-size padded pieces, then (only when the batch is
    split) one row gather.  Buffers are preallocated, so the call is stream-
    ordered and can run inside a serving loop without allocation."""

    def __init__(self, plan: "ShardPlan", num_q_heads: int, batch: int, dtype, device,
                 group: Optional[dist.ProcessGroup] = None):
        self.plan, self.group = plan, group
        hq_loc = plan.num_q_local
        self.piece = torch.zeros((hq_loc, plan.b_max, 128), dtype=dtype, device=device)
        self.gathered = torch.empty((plan.world * hq_loc, plan.b_max, 128), dtype=dtype, device=device)
        self.simple = plan.b_split == 1   # rank-major concat is already [Hq, B, d]
        self.idx = (None if self.simple else
                    torch.as_tensor(plan.gather_index(num_q_heads, batch), device=device))
        self.out = self.gathered.view(num_q_heads, batch, 128) if self.simple else \
            torch.empty((num_q_heads, batch, 128), dtype=dtype, device=device)

    def __call__(self, out_local: torch.Tensor) -> torch.Tensor:
        if self.simple:
            dist.all_gather_into_tensor(self.gathered, out_local.contiguous(), group=self.group)
            return self.out
        self.piece[:, : out_local.shape[1]].copy_(out_local)
        dist.all_gather_into_tensor(self.gathered, self.piece, group=self.group)
        torch.index_select(self.gathered.view(-1, 128), 0, self.idx, out=self.out.view(-1, 128))
        return self.out


class Sharded2DDecodeAttention:
    """Decode attention over a 2-D (KV head group x batch part) partition.

    ``local_attention(q_local[B_r, Hq_loc, d]) -> [Hq_loc, B_r, d]`` attends this
    rank's sequences over its heads (rows of ``plan.seqs``); :class:`OutputGather`
    assembles ``[Hq, B, d]``."""

    def __init__(self, num_q_heads: int, num_kv_heads: int, seq_lens: Sequence[int],
                 group: Optional[dist.ProcessGroup] = None,
                 local_attention: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.Hq, self.Hkv, self.B = num_q_heads, num_kv_heads, len(seq_lens)
        self.plan = plan_shards(num_q_heads, num_kv_heads, self.world, self.rank, seq_lens)
        self.local_attention = local_attention
        self._gather = None

    def local_q(self, q: torch.Tensor) -> torch.Tensor:
        q0, q1 = self.plan.q_range
        seqs = torch.as_tensor(self.plan.seqs, device=q.device)
        return q.index_select(0, seqs)[:, q0:q1].contiguous()

    def __call__(self, q: torch.Tensor) -> torch.Tensor:
        o_loc = self.local_attention(self.local_q(q))          # [Hq_loc, B_r, d]
        if self.world == 1:
            return o_loc
        if self._gather is None:
            self._gather = OutputGather(self.plan, self.Hq, self.B, o_loc.dtype, o_loc.device, self.group)
        return self._gather(o_loc)


def cuda_local_attention(cache, block_table, seq_lens, **kw) -> Callable[[torch.Tensor], torch.Tensor]:
    """The product local op: libkvq decode attention, head-major output."""
    from .ops import paged_decode_attention

    def run(q_loc: torch.Tensor) -> torch.Tensor:
        return paged_decode_attention(q_loc, cache, block_table, seq_lens, head_major=True, **kw)

    return run


class _RawCuda:
    """``__cuda_array_interface__`` wrapper so torch can view memory that libkvq
    allocated (the symmetric buffers are not torch allocations)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class PeerOutput:
    """Symmetric output buffers for the all-gather fused into K2.

    Every rank allocates ``slots`` x (control block + global bf16 output
    ``[Hq, B, 128]``) with ``kvq_sym_alloc``, the IPC handles are exchanged
    once over ``group`` (any backend; this is setup, not the step path) and
    each rank maps all peers' buffers.  :func:`ops.paged_decode_attention_gathered`
    then runs K2 with ``kvq_peer_out`` so each finished row is stored into
    every rank's copy over NVLink while the attention streams; when the launch
    completes on a rank, :meth:`out` holds all ranks' heads -- there is no
    separate collective.  With the 2-D partition (``plan.b_split > 1``) each
    rank's rows land at their global batch positions through ``seq_map``.

    Slot reuse is protected on the device (K2 releases a slot's previous use
    at entry and writers wait for every rank's release), so callers only keep
    the usual stream order: consume slot s's output before the next K2 that
    uses slot s is enqueued on the same stream (DecodeSession does, through
    its per-slot events)."""

    def __init__(self, plan: ShardPlan, num_q_heads: int, batch: int, num_kv_heads: int,
                 device: torch.device, group: Optional[dist.ProcessGroup] = None, slots: int = 1):
        import ctypes

        from . import _lib
        lib = _lib.load()
        if not 2 <= plan.world <= _lib.MAX_PEERS:
            raise ValueError(f"fused gather needs 2..{_lib.MAX_PEERS} ranks, got {plan.world}")
        self.plan, self.P, self.rank, self.slots = plan, plan.world, plan.rank, slots
        self.Hq, self.B, self.device = num_q_heads, batch, torch.device(device)
        self.out_bytes = num_q_heads * batch * 128 * 2
        self.slot_bytes = _lib.PEER_CTL_BYTES + ((self.out_bytes + 255) // 256) * 256
        with torch.cuda.device(self.device):
            ptr, handle = ctypes.c_void_p(), (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
            _lib.check("kvq_sym_alloc", lib.kvq_sym_alloc(slots * self.slot_bytes, ctypes.byref(ptr), handle))
            self._own = ptr.value
            handles: List[Optional[bytes]] = [None] * self.P
            dist.all_gather_object(handles, bytes(handle), group=group)
            self._bases, self._opened = [], []
            err = None
            for r, h in enumerate(handles):
                if r == self.rank:
                    self._bases.append(self._own)
                    continue
                p = ctypes.c_void_p()
                st = lib.kvq_sym_open(h, ctypes.byref(p))
                if st != _lib.KVQ_OK:
                    err = f"rank {self.rank}: kvq_sym_open of rank {r}: {lib.kvq_last_error().decode()}"
                    break
                self._bases.append(p.value)
                self._opened.append(p.value)
            # Every rank must agree before anyone relies on the mapping: a rank
            # that cannot map its peers makes all ranks raise (and fall back),
            # instead of leaving the others waiting in a barrier.
            errs: List[Optional[str]] = [None] * self.P
            dist.all_gather_object(errs, err, group=group)
            failed = [e for e in errs if e]
            if failed:
                for q in self._opened:
                    lib.kvq_sym_close(q)
                lib.kvq_sym_free(self._own)
                self._own, self._opened = None, []
                raise RuntimeError("fused peer gather unavailable: " + "; ".join(failed))
        self.group = group
        # rows of this rank's sequences in the global output (identity for a pure head split)
        self.seq_map = (None if plan.b_split == 1 else
                        torch.as_tensor(plan.seqs.astype(np.int32), device=self.device))
        self.writers_per_use = batch * num_kv_heads  # every global (sequence, kv head) writes once
        self.descs = []
        for s in range(slots):
            d = _lib.PeerOutDesc()
            d.n_peers, d.rank = self.P, self.rank
            d.head_offset, d.batch_global = plan.q_range[0], batch
            d.seq_map = self.seq_map.data_ptr() if self.seq_map is not None else None
            d.writers_per_use = self.writers_per_use
            for r in range(self.P):
                d.ctl[r] = self._bases[r] + s * self.slot_bytes
                d.out[r] = self._bases[r] + s * self.slot_bytes + _lib.PEER_CTL_BYTES
            self.descs.append(d)
        self._outs = [torch.as_tensor(_RawCuda(self._own + s * self.slot_bytes + _lib.PEER_CTL_BYTES,
                                               (num_q_heads, batch, 128), "<i2"), device=self.device)
                      .view(torch.bfloat16) for s in range(slots)]
        self._ctls = [torch.as_tensor(_RawCuda(self._own + s * self.slot_bytes, (_lib.PEER_CTL_BYTES // 4,),
                                               "<i4"), device=self.device) for s in range(slots)]
        dist.barrier(group=group)  # every rank mapped before anyone writes

    def out(self, slot: int = 0) -> torch.Tensor:
        """This rank's copy of the global output ``[Hq, B, 128]`` (bf16) of ``slot``."""
        return self._outs[slot]

    def control(self, slot: int = 0) -> torch.Tensor:
        """int32 view of the slot's control block (done, uses, error, arrivals, free[P])."""
        return self._ctls[slot]

    def errors(self) -> int:
        """Number of slots whose protocol spin timed out (synchronises)."""
        return int(sum(int(c[2].item() != 0) for c in self._ctls))

    def close(self) -> None:
        """Unmap peers and free this rank's buffer (collective: barrier first,
        so no peer still writes into it)."""
        from . import _lib
        if self._own is None:
            return
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        lib = _lib.load()
        with torch.cuda.device(self.device):
            for p in self._opened:
                lib.kvq_sym_close(p)
            lib.kvq_sym_free(self._own)
        self._own, self._opened, self._outs, self._ctls = None, [], [], []
