"""CPU oracle for the quantized paged-KV decode path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline; ``paper_2605_29639_b200`` never does.

Two independent restatements of the same contract:

* ``libkvq_oracle.so`` (``kvq_oracle.c``, plain C, -ffp-contract=off) --
  quantizer, page packing and a multi-threaded paged decode attention
  (fp32 dequantisation, fp64 accumulation);
* the numpy functions below (``*_np``), written separately from the C code.

PARITY UNPINNED against the reference: arxiv/paper_2605_29639 contains no
implementation of this path (the semantics are the prose of
PAPER.md:468-477 plus BASELINE.json.north_star).  The restatements are pinned
to each other, to the contract known-answer vectors in tests/golden/, and (FP8)
to two third-party encoders (torch ``float8_e4m3fn``, ``ml_dtypes``).
"""
from __future__ import annotations

import ctypes
import math
import time
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
LIB_PATH = ORACLE_DIR / "libkvq_oracle.so"
HEAD_DIM, BLOCK, PAGE = 128, 16, 4224
INT8, FP8_E4M3 = 0, 1
QMAX = {INT8: 127.0, FP8_E4M3: 448.0}

_lib = None


def lib() -> ctypes.CDLL:
    """Load (building if needed) the C oracle."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import subprocess
            subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        L.kvqo_f32_to_e4m3_satfinite.restype = ctypes.c_uint8
        L.kvqo_f32_to_e4m3_satfinite.argtypes = [f32]
        L.kvqo_e4m3_to_f32.restype = f32
        L.kvqo_e4m3_to_f32.argtypes = [ctypes.c_uint8]
        L.kvqo_quantize_rows.restype = None
        L.kvqo_quantize_rows.argtypes = [vp, i64, ctypes.c_int, vp, vp]
        L.kvqo_code_offset.restype = ctypes.c_int
        L.kvqo_code_offset.argtypes = [ctypes.c_int] * 3
        L.kvqo_quant_append.restype = None
        L.kvqo_quant_append.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, i64]
        L.kvqo_unpack_pool.restype = None
        L.kvqo_unpack_pool.argtypes = [vp, i64, ctypes.c_int, vp, vp]
        L.kvqo_pack_pool.restype = None
        L.kvqo_pack_pool.argtypes = [vp, vp, i64, ctypes.c_int, vp]
        L.kvqo_decode_attn.restype = None
        L.kvqo_decode_attn.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, f32, vp, vp, ctypes.c_int]
        L.kvqo_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# bf16 helpers (inputs are raw uint16 bit patterns)
# ---------------------------------------------------------------------------
def bf16_bits_to_f32(x: np.ndarray) -> np.ndarray:
    return (x.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (NaN kept quiet)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    out = ((u + r) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    out[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return out


# ---------------------------------------------------------------------------
# C oracle wrappers
# ---------------------------------------------------------------------------
def quantize_rows(x_bits: np.ndarray, kv_dtype: int) -> Tuple[np.ndarray, np.ndarray]:
    x = np.ascontiguousarray(x_bits, dtype=np.uint16).reshape(-1, HEAD_DIM)
    codes = np.zeros(x.shape, dtype=np.uint8)
    scales = np.zeros(x.shape[0], dtype=np.float32)
    lib().kvqo_quantize_rows(_p(x), x.shape[0], kv_dtype, _p(codes), _p(scales))
    return codes, scales


def quant_append(k_bits: np.ndarray, v_bits: np.ndarray, slot_mapping: np.ndarray, kv_dtype: int,
                 pool: np.ndarray) -> None:
    """In-place append into ``pool`` (uint8 [NB, Hkv, 4224])."""
    k = np.ascontiguousarray(k_bits, dtype=np.uint16)
    v = np.ascontiguousarray(v_bits, dtype=np.uint16)
    sm = np.ascontiguousarray(slot_mapping, dtype=np.int32)
    T, Hkv = k.shape[0], k.shape[1]
    lib().kvqo_quant_append(_p(k), _p(v), _p(sm), T, Hkv, kv_dtype, _p(pool), pool.shape[0])


def unpack_pool(pool: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    NB, Hkv = pool.shape[:2]
    codes = np.zeros((NB, Hkv, 2, BLOCK, HEAD_DIM), dtype=np.uint8)
    scales = np.zeros((NB, Hkv, 2, BLOCK), dtype=np.float32)
    lib().kvqo_unpack_pool(_p(np.ascontiguousarray(pool)), NB, Hkv, _p(codes), _p(scales))
    return codes, scales


def pack_pool(codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
    NB, Hkv = codes.shape[:2]
    pool = np.zeros((NB, Hkv, PAGE), dtype=np.uint8)
    lib().kvqo_pack_pool(_p(np.ascontiguousarray(codes)), _p(np.ascontiguousarray(scales, np.float32)),
                         NB, Hkv, _p(pool))
    return pool


def decode_attn(q_bits: np.ndarray, pool: np.ndarray, block_table: np.ndarray,
                seq_lens: np.ndarray, num_kv_heads: int, kv_dtype: int,
                sm_scale: Optional[float] = None, nthreads: int = 0,
                with_lse: bool = False):
    """fp32 [B, Hq, 128] (+ natural-log LSE [B, Hq])."""
    q = np.ascontiguousarray(q_bits, dtype=np.uint16)
    B, Hq = q.shape[:2]
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    out = np.zeros((B, Hq, HEAD_DIM), dtype=np.float32)
    lse = np.zeros((B, Hq), dtype=np.float32)
    if sm_scale is None:
        sm_scale = 1.0 / math.sqrt(HEAD_DIM)
    lib().kvqo_decode_attn(_p(q), _p(np.ascontiguousarray(pool)), _p(bt), _p(sl), B, Hq,
                           num_kv_heads, bt.shape[1], kv_dtype, sm_scale, _p(out), _p(lse),
                           nthreads)
    return (out, lse) if with_lse else out


def num_threads() -> int:
    return int(lib().kvqo_num_threads())


# ---------------------------------------------------------------------------
# numpy restatement (independent of the C code; small inputs)
# ---------------------------------------------------------------------------
def e4m3_encode_np(y: np.ndarray) -> np.ndarray:
    """fp32 -> E4M3 bits, round-to-nearest-even, satfinite, NaN -> 0x7F."""
    y = np.asarray(y, dtype=np.float32)
    sign = ((y.view(np.uint32) >> 24) & 0x80).astype(np.uint8)
    a = np.abs(y).astype(np.float64)  # exact
    out = np.zeros(y.shape, dtype=np.uint8)
    sub = a < 2.0 ** -6
    out[sub] = np.rint(a[sub] * 512.0).astype(np.uint8)
    norm = (~sub) & (a < 448.0)
    if norm.any():
        e = np.floor(np.log2(a[norm])).astype(np.int64)
        mant = a[norm] / np.exp2(e)
        # guard log2 rounding at exact powers of two
        e = np.where(mant >= 2.0, e + 1, np.where(mant < 1.0, e - 1, e))
        mant = a[norm] / np.exp2(e)
        m = np.rint((mant - 1.0) * 8.0).astype(np.int64)
        e = np.where(m == 8, e + 1, e)
        m = np.where(m == 8, 0, m)
        out[norm] = (((e + 7) << 3) | m).astype(np.uint8)
    out[(a >= 448.0) & ~np.isnan(y)] = 0x7E
    out |= sign
    out[np.isnan(y)] = 0x7F
    return out


def e4m3_decode_np(c: np.ndarray) -> np.ndarray:
    c = np.asarray(c, dtype=np.uint8).astype(np.int64)
    s = np.where(c >> 7, -1.0, 1.0)
    ex, m = (c >> 3) & 0xF, c & 7
    v = np.where(ex == 0, m * 2.0 ** -9, (1.0 + m / 8.0) * np.exp2(ex - 7.0))
    v = np.where((ex == 0xF) & (m == 7), np.nan, v)
    return (s * v).astype(np.float32)


def quantize_rows_np(x_bits: np.ndarray, kv_dtype: int) -> Tuple[np.ndarray, np.ndarray]:
    x = bf16_bits_to_f32(np.asarray(x_bits, dtype=np.uint16).reshape(-1, HEAD_DIM))
    qmax = np.float32(QMAX[kv_dtype])
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        amax = np.fmax.reduce(np.abs(x), axis=1, initial=np.float32(0.0)).astype(np.float32)
        scale = (amax / qmax).astype(np.float32)
        inv = np.where(amax > 0, qmax / np.where(amax > 0, amax, 1), 0).astype(np.float32)
        y = (x * inv[:, None]).astype(np.float32)
        if kv_dtype == FP8_E4M3:
            codes = e4m3_encode_np(y)
        else:
            r = np.rint(y)
            c = np.clip(np.nan_to_num(r, nan=0.0, posinf=127, neginf=-127), -127, 127)
            codes = c.astype(np.int8).view(np.uint8)
    return codes, scale


def code_values_np(codes: np.ndarray, kv_dtype: int) -> np.ndarray:
    return e4m3_decode_np(codes) if kv_dtype == FP8_E4M3 else codes.view(np.int8).astype(np.float32)


def decode_attn_np(q: np.ndarray, k_deq: np.ndarray, v_deq: np.ndarray, seq_lens: np.ndarray,
                   sm_scale: Optional[float] = None, splits: int = 1) -> np.ndarray:
    """Reference attention over dequantised dense K/V ``[B, Hkv, Lmax, 128]``
    (fp64), optionally as ``splits`` split-KV partials merged by LSE -- the
    split-invariance oracle."""
    B, Hq = q.shape[:2]
    Hkv = k_deq.shape[1]
    g = Hq // Hkv
    if sm_scale is None:
        sm_scale = 1.0 / math.sqrt(HEAD_DIM)
    out = np.zeros((B, Hq, HEAD_DIM), dtype=np.float64)
    for b in range(B):
        L = int(seq_lens[b])
        if L == 0:
            continue
        bounds = np.linspace(0, L, splits + 1).astype(int)
        for hq in range(Hq):
            h = hq // g
            parts = []
            for s in range(splits):
                lo, hi = bounds[s], bounds[s + 1]
                if hi <= lo:
                    continue
                sc = k_deq[b, h, lo:hi].astype(np.float64) @ q[b, hq].astype(np.float64) * sm_scale
                m = sc.max()
                p = np.exp(sc - m)
                parts.append((m + np.log(p.sum()), (p @ v_deq[b, h, lo:hi].astype(np.float64)) / p.sum()))
            M = max(x[0] for x in parts)
            w = np.array([np.exp(x[0] - M) for x in parts])
            out[b, hq] = sum(wi * x[1] for wi, x in zip(w, parts)) / w.sum()
    return out


def timed_decode_attn(*args, **kw):
    t0 = time.perf_counter()
    r = decode_attn(*args, **kw)
    return r, time.perf_counter() - t0
