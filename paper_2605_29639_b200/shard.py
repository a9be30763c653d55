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

from typing import Callable, Optional, Tuple

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


def cuda_local_attention(cache, block_table, seq_lens, **kw) -> Callable[[torch.Tensor], torch.Tensor]:
    """The product local op: libkvq decode attention, head-major output."""
    from .ops import paged_decode_attention

    def run(q_loc: torch.Tensor) -> torch.Tensor:
        return paged_decode_attention(q_loc, cache, block_table, seq_lens, head_major=True, **kw)

    return run
