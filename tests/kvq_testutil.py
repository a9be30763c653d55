"""Shared synthetic-input builders for the tests (SURVEY.md §8d 'Synthetic
inputs': K/V = N(0,1) x per-(token, head) factor exp(N(0, 0.5)); four fixed K
outlier channels x8; Q = N(0,1); block ids a random permutation)."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle as O

OUTLIER_CHANNELS = (3, 40, 77, 121)


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def make_kv(T: int, Hkv: int, seed: int, outliers: bool = True, kind: str = "k") -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, Hkv, 128), generator=g)
    x = x * torch.exp(0.5 * torch.randn((T, Hkv, 1), generator=g))
    if outliers and kind == "k":
        x[..., list(OUTLIER_CHANNELS)] *= 8.0
    return x.to(torch.bfloat16)


def make_q(B: int, Hq: int, seed: int) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    return torch.randn((B, Hq, 128), generator=g).to(torch.bfloat16)


class Scenario:
    """A paged cache filled with `seq_lens` tokens per sequence at random
    (non-contiguous) blocks, built on the CPU oracle so the GPU side can be
    fed identical bytes."""

    def __init__(self, seq_lens, Hq, Hkv, kv_dtype, seed=0, extra_blocks=3, max_blocks=None):
        self.seq_lens = np.asarray(seq_lens, dtype=np.int32)
        self.B = len(seq_lens)
        self.Hq, self.Hkv, self.kv_dtype = Hq, Hkv, kv_dtype
        nblk = [int(math.ceil(L / 16)) for L in self.seq_lens]
        self.max_blocks = max_blocks or max(nblk + [1])
        self.num_blocks = sum(nblk) + extra_blocks
        rng = np.random.default_rng(seed)
        perm = rng.permutation(self.num_blocks).astype(np.int32)
        self.block_table = np.zeros((self.B, self.max_blocks), dtype=np.int32)
        slots = []
        pos = 0
        for b, L in enumerate(self.seq_lens):
            self.block_table[b, : nblk[b]] = perm[pos : pos + nblk[b]]
            pos += nblk[b]
            for t in range(L):
                slots.append(self.block_table[b, t // 16] * 16 + t % 16)
        self.slots = np.asarray(slots, dtype=np.int32)
        T = len(slots)
        self.k = make_kv(T, Hkv, seed + 11, kind="k")
        self.v = make_kv(T, Hkv, seed + 12, kind="v")
        self.q = make_q(self.B, Hq, seed + 13)
        self.pool = np.zeros((self.num_blocks, Hkv, O.PAGE), dtype=np.uint8)
        if T:
            O.quant_append(bf16_bits(self.k), bf16_bits(self.v), self.slots, kv_dtype, self.pool)

    def oracle_out(self, sm_scale=None):
        return O.decode_attn(bf16_bits(self.q), self.pool, self.block_table, self.seq_lens, self.Hkv,
                             self.kv_dtype, sm_scale)


def int8_two_term_q(q: torch.Tensor, Hkv: int) -> np.ndarray:
    """The INT8 path's query rounding (kvq_decode.cu, decode_cta: 'INT8 K feeds
    the s8 tensor cores directly'): per (sequence, kv head) group a power-of-two
    step s1 with amax / s1 in [64, 127.5), q1 = floor(q / s1 + 1/2), q2 =
    clamp(rint((q - q1 s1) * 256 / s1), -128, 127), q' = s1 (q1 + q2 / 256).
    Lets a test separate that (documented) score rounding from P' numerics."""
    x = q.float().numpy().astype(np.float64)
    B, Hq = x.shape[:2]
    g = Hq // Hkv
    out = np.zeros_like(x)
    for b in range(B):
        for h in range(Hkv):
            grp = x[b, h * g:(h + 1) * g]
            a = np.abs(grp).max()
            if a == 0:
                continue
            ex = np.frexp(a)[1]
            if a * 2.0 ** (7 - ex) > 127.49:
                ex += 1
            s1 = 2.0 ** (ex - 7)
            q1 = np.clip(np.floor(grp / s1 + 0.5), -127, 127)
            q2 = np.clip(np.rint((grp - q1 * s1) / s1 * 256), -128, 127)
            out[b, h * g:(h + 1) * g] = s1 * (q1 + q2 / 256)
    return out


def dense_kv(sc: "Scenario"):
    """Dequantised dense K/V [B, Hkv, Lmax, 128] of a Scenario's pages (fp64)."""
    codes, scales = O.unpack_pool(sc.pool)
    vals = O.code_values_np(codes, sc.kv_dtype).astype(np.float64) * scales[..., None].astype(np.float64)
    Lmax = max(int(sc.seq_lens.max()), 1)
    k = np.zeros((sc.B, sc.Hkv, Lmax, 128))
    v = np.zeros_like(k)
    for b, L in enumerate(sc.seq_lens):
        n = -(-int(L) // 16)
        blk = sc.block_table[b, :n]
        k[b, :, :L] = vals[blk, :, 0].transpose(1, 0, 2, 3).reshape(sc.Hkv, -1, 128)[:, :L]
        v[b, :, :L] = vals[blk, :, 1].transpose(1, 0, 2, 3).reshape(sc.Hkv, -1, 128)[:, :L]
    return k, v
