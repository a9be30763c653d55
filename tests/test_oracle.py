"""The CPU oracle pinned before it is trusted: contract KATs (hand-derived and
cross-checked with third-party FP8 encoders), agreement of the two independent
restatements (C and numpy), page-layout round trips, attention properties
(split-KV invariance, GQA == repeated-KV MHA, dequantisation error bounds) and
the attention math against PyTorch's scaled_dot_product_attention."""
import json
import math
from pathlib import Path

import ml_dtypes
import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_kat_fixture():
    rows = json.loads((GOLDEN / "kat_quant.json").read_text())
    assert len(rows) >= 36
    for r in rows:
        bits = np.asarray(r["x_bf16"], dtype=np.uint16)[None]
        for impl in (O.quantize_rows, O.quantize_rows_np):
            codes, scale = impl(bits, r["kv_dtype"])
            if "codes_head" in r:
                assert list(codes[0, : len(r["codes_head"])]) == r["codes_head"], (impl, r["name"])
                assert scale[0] == r["scale"], r["name"]
            else:
                assert list(codes[0]) == r["codes"], (impl, r["name"])
                assert int(scale.view(np.uint32)[0]) == r["scale_bits"], r["name"]


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
def test_c_and_numpy_quantizers_agree(kv_dtype):
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((3000, 128)) * np.exp2(rng.integers(-30, 30, (3000, 1)))).astype(np.float32)
    x[0] = 0
    x[1, 3] = np.nan
    x[2, 4] = np.inf
    x[3] = 1e-39
    bits = O.f32_to_bf16_bits(x)
    c1, s1 = O.quantize_rows(bits, kv_dtype)
    c2, s2 = O.quantize_rows_np(bits, kv_dtype)
    assert np.array_equal(c1, c2)
    assert np.array_equal(s1.view(np.uint32), s2.view(np.uint32))


def test_e4m3_encoder_matches_third_party():
    rng = np.random.default_rng(3)
    y = (rng.standard_normal(200000) * np.exp2(rng.integers(-14, 10, 200000))).astype(np.float32)
    y = np.concatenate([y, np.float32([464, 479.99, 480, -500, np.inf, -np.inf, 2 ** -10, 3 * 2 ** -11])])
    mine = O.e4m3_encode_np(y)
    ml = np.clip(y, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    tt = torch.from_numpy(np.clip(y, -448, 448)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(mine, ml) and np.array_equal(mine, tt)
    c = np.array([O.lib().kvqo_f32_to_e4m3_satfinite(float(v)) for v in y[-3000:]], np.uint8)
    assert np.array_equal(c, mine[-3000:])
    # decode is exact and inverse on every non-NaN code
    codes = np.arange(256, dtype=np.uint8)
    vals = O.e4m3_decode_np(codes)
    ok = ~np.isnan(vals)
    assert np.array_equal(O.e4m3_encode_np(vals[ok]), codes[ok])
    assert np.array_equal(vals[ok], np.array([O.lib().kvqo_e4m3_to_f32(int(c)) for c in codes[ok]], np.float32))


def test_page_layout_is_a_bijection():
    offs = {O.lib().kvqo_code_offset(kv, t, d) for kv in range(2) for t in range(16) for d in range(128)}
    assert offs == set(range(4096))
    rng = np.random.default_rng(0)
    codes = rng.integers(0, 256, (5, 3, 2, 16, 128), dtype=np.uint8)
    scales = rng.standard_normal((5, 3, 2, 16)).astype(np.float32)
    pool = O.pack_pool(codes, scales)
    c2, s2 = O.unpack_pool(pool)
    assert np.array_equal(codes, c2) and np.array_equal(scales, s2)
    from paper_2605_29639_b200 import unpack_pages
    c3, s3 = unpack_pages(torch.from_numpy(pool))
    assert np.array_equal(c3.numpy(), codes) and np.array_equal(s3.numpy(), scales)


@settings(max_examples=60, deadline=None)
@given(st.integers(min_value=-60, max_value=60), st.integers(0, 2 ** 31 - 1), st.sampled_from([O.INT8, O.FP8_E4M3]))
def test_dequant_error_bound(e, seed, kv_dtype):
    """|x - code*scale| <= scale/2 (INT8) and <= half an E4M3 ulp of |x|/scale
    times scale (FP8), plus the fp32 rounding of inv/scale (2^-21 |x|)."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((4, 128)) * 2.0 ** e).astype(np.float32)
    bits = O.f32_to_bf16_bits(x)
    xf = O.bf16_bits_to_f32(bits).astype(np.float64)
    codes, scale = O.quantize_rows(bits, kv_dtype)
    deq = O.code_values_np(codes, kv_dtype).astype(np.float64) * scale[:, None]
    s = scale.astype(np.float64)[:, None]
    if kv_dtype == O.INT8:
        assert np.all(np.abs(xf - deq) <= s * 0.5 + np.abs(xf) * 2.0 ** -21 + 1e-45)
    else:
        y = np.abs(xf) / np.where(s > 0, s, 1)
        ulp = np.where(y >= 2 ** -6, 2.0 ** (np.floor(np.log2(np.maximum(y, 2 ** -6))) - 3), 2.0 ** -9)
        assert np.all(np.abs(xf - deq) <= 0.5 * ulp * s + np.abs(xf) * 2.0 ** -21 + 1e-45)


def _dense(pool, table, lens, kv_dtype):
    codes, scales = O.unpack_pool(pool)
    B, Hkv, Lm = len(lens), pool.shape[1], max(int(max(lens)), 1)
    kd = np.zeros((B, Hkv, Lm, 128))
    vd = np.zeros((B, Hkv, Lm, 128))
    for b in range(B):
        for t in range(int(lens[b])):
            blk, o = table[b, t // 16], t % 16
            kd[b, :, t] = (O.code_values_np(codes[blk, :, 0, o], kv_dtype) * scales[blk, :, 0, o][:, None])
            vd[b, :, t] = (O.code_values_np(codes[blk, :, 1, o], kv_dtype) * scales[blk, :, 1, o][:, None])
    return kd, vd


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
def test_attention_oracles_agree_and_split_invariant(kv_dtype):
    from kvq_testutil import Scenario, bf16_bits
    sc = Scenario([40, 17, 0, 33, 130], 16, 4, kv_dtype, seed=2)
    ref, lse = O.decode_attn(bits := bf16_bits(sc.q), sc.pool, sc.block_table, sc.seq_lens, 4, kv_dtype,
                             with_lse=True)
    kd, vd = _dense(sc.pool, sc.block_table, sc.seq_lens, kv_dtype)
    q = O.bf16_bits_to_f32(bits)
    r1 = O.decode_attn_np(q, kd, vd, sc.seq_lens)
    assert np.abs(ref - r1).max() <= 1e-6 * max(1, np.abs(r1).max())
    for splits in (2, 3, 7):
        rs = O.decode_attn_np(q, kd, vd, sc.seq_lens, splits=splits)
        assert np.abs(rs - r1).max() <= 1e-12 * max(1, np.abs(r1).max())
    assert np.all(ref[3] == ref[3]) and np.all(ref[2] == 0) and np.isneginf(lse[2]).all()


def test_gqa_equals_repeated_kv_mha():
    from kvq_testutil import Scenario, bf16_bits
    sc = Scenario([50, 64], 8, 2, O.INT8, seed=9)
    gqa = sc.oracle_out()
    # MHA: replicate each KV head g times in the pool
    g = 4
    pool_mha = np.repeat(sc.pool, g, axis=1)
    mha = O.decode_attn(bf16_bits(sc.q), pool_mha, sc.block_table, sc.seq_lens, 8, O.INT8)
    assert np.array_equal(gqa, mha)


def test_oracle_threads_deterministic():
    from kvq_testutil import Scenario, bf16_bits
    sc = Scenario([300, 100, 257], 32, 8, O.FP8_E4M3, seed=1)
    a = O.decode_attn(bf16_bits(sc.q), sc.pool, sc.block_table, sc.seq_lens, 8, O.FP8_E4M3, nthreads=1)
    b = O.decode_attn(bf16_bits(sc.q), sc.pool, sc.block_table, sc.seq_lens, 8, O.FP8_E4M3, nthreads=8)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
def test_attention_oracle_matches_torch_sdpa(kv_dtype):
    """The attention oracle against an independent implementation: PyTorch's
    scaled_dot_product_attention (fp64, GQA via enable_gqa) over the same
    dequantized K/V (code * scale, read back through the page layout).  This
    pins the oracle's softmax / GQA / masking math to third-party code; the
    quantizer is pinned by the KATs above."""
    from kvq_testutil import Scenario, bf16_bits
    Hq, Hkv = 32, 8
    sc = Scenario([1, 15, 16, 17, 300, 1029], Hq, Hkv, kv_dtype, seed=12)
    ref = O.decode_attn(bits := bf16_bits(sc.q), sc.pool, sc.block_table, sc.seq_lens, Hkv, kv_dtype)
    kd, vd = _dense(sc.pool, sc.block_table, sc.seq_lens, kv_dtype)   # [B, Hkv, T, d]
    q = torch.from_numpy(O.bf16_bits_to_f32(bits)).double()             # [B, Hq, d]
    for b, L in enumerate(sc.seq_lens):
        k = torch.from_numpy(kd[b, :, :L]).double()[None]                # [1, Hkv, L, d]
        v = torch.from_numpy(vd[b, :, :L]).double()[None]
        o = torch.nn.functional.scaled_dot_product_attention(q[b][None, :, None], k, v, enable_gqa=True,
                                                             scale=1.0 / math.sqrt(128))[0, :, 0]
        assert np.abs(ref[b] - o.numpy()).max() <= 2e-6 * max(1.0, float(o.abs().max())), b
