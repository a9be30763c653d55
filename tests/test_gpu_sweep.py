"""Randomised K2 parity sweep against the CPU oracle: seeded random shapes
(GQA group 1..16, 1..8 kv heads, ragged lengths with empty / one-token /
page-boundary sequences), both code formats, automatic or random split
geometry -- plus adversarial data (peaked softmax from large logits,
all-zero and very large K/V rows).  Same tolerance as test_gpu_attention:
per (sequence, head) row, max |err| <= 2e-3 * max |ref row|."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import Scenario, bf16_bits, dense_kv, int8_two_term_q
from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, paged_decode_attention, quantize_append

pytestmark = pytest.mark.gpu
NAMES = {O.INT8: "int8", O.FP8_E4M3: "fp8_e4m3"}


def rel_err(out, ref):
    err = np.abs(out - ref).max(axis=-1)
    scale = np.abs(ref).max(axis=-1)
    return float((err / (scale + 1e-6 / 2e-3)).max())


def run(sc, cuda, **kw):
    cache = PagedKVCache(KVCacheSpec(sc.Hkv, kv_dtype=NAMES[sc.kv_dtype]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    out = paged_decode_attention(sc.q.to(cuda), cache, torch.from_numpy(sc.block_table).to(cuda),
                                 torch.from_numpy(sc.seq_lens).to(cuda), out_dtype=torch.float32, **kw)
    return out.cpu().numpy()


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    Hkv = int(rng.choice([1, 2, 4, 8]))
    g = int(rng.choice([1, 2, 4, 8, 16]))
    B = int(rng.integers(1, 13))
    special = [0, 1, 15, 16, 17, 32, 33]
    lens = [int(rng.choice(special)) if rng.random() < 0.3 else int(rng.integers(1, 3000)) for _ in range(B)]
    if max(lens) == 0:
        lens[0] = 5
    kvd = O.INT8 if rng.random() < 0.5 else O.FP8_E4M3
    pps = None if rng.random() < 0.5 else int(rng.integers(1, 65))
    return lens, g * Hkv, Hkv, kvd, pps


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes(cuda, seed):
    lens, Hq, Hkv, kvd, pps = random_case(seed)
    sc = Scenario(lens, Hq, Hkv, kvd, seed=seed)
    out = run(sc, cuda, pages_per_split=pps)
    ref = sc.oracle_out()
    assert np.isfinite(out).all()
    for b, L in enumerate(lens):
        if L == 0:
            assert np.all(out[b] == 0)
    assert rel_err(out, ref) <= 2e-3, (lens, Hq, Hkv, kvd, pps, rel_err(out, ref))


def requantize(sc):
    sc.pool[:] = 0
    O.quant_append(bf16_bits(sc.k), bf16_bits(sc.v), sc.slots, sc.kv_dtype, sc.pool)


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
@pytest.mark.parametrize("q_gain", [8.0, 40.0])
def test_peaked_softmax_and_extreme_rows(cuda, kv_dtype, q_gain):
    """Large logits make the running max jump mid-sequence (the lazy rescale
    and the P' reference point); zero rows have scale 0 and all-zero codes;
    K rows of magnitude 2^100 give scores past fp32 resolution (the output
    must stay finite and the max token must win); V rows 2^6 larger or
    2^100 smaller than their page neighbours stress the f16 range of P' --
    at 40x one token takes nearly all the weight, and if its V is ~0 the
    output is made of weights p < 2^-18 of the max, which the contribution
    anchor keeps in f16's normal range."""
    sc = Scenario([1800, 700, 64, 2500], 32, 8, kv_dtype, seed=77)
    T = sc.k.shape[0]
    g = torch.Generator().manual_seed(5)
    idx = torch.randperm(T, generator=g)
    k, v = sc.k.float(), sc.v.float()
    k[idx[:40]] = 0.0
    v[idx[40:80]] = 0.0
    k[idx[80:100]] *= 2.0 ** 100
    v[idx[100:120]] *= 2.0 ** 6
    v[idx[120:140]] *= 2.0 ** -100
    sc.k, sc.v = k.to(torch.bfloat16), v.to(torch.bfloat16)
    requantize(sc)
    sc.q = (sc.q.float() * q_gain).to(torch.bfloat16)
    ref = sc.oracle_out()
    for pps in (None, 3):
        out = run(sc, cuda, pages_per_split=pps)
        assert np.isfinite(out).all()
        assert rel_err(out, ref) <= 2e-3, (pps, rel_err(out, ref))


def _sink_scenario(kv_dtype, g, gap, v_shift, seed):
    """Token 0 of every sequence is an attention sink: its K row points along
    the mean query of each GQA group so its logit sits `gap` log2 units above
    zero, and its V row is scaled by 2^-v_shift (a sink with V ~ 0, the
    ordinary tokens' tiny weights then make up the output)."""
    sc = Scenario([700, 333, 1200, 17], 8 * g, 8, kv_dtype, seed=seed)
    k, v, qf = sc.k.float(), sc.v.float(), sc.q.float()
    starts = np.concatenate([[0], np.cumsum(sc.seq_lens)[:-1]])
    for b, s0 in enumerate(starts):
        for h in range(8):
            qm = qf[b, h * g:(h + 1) * g].mean(0)
            k[s0, h] = qm / (qm.norm() ** 2) * gap * np.sqrt(128) / np.log2(np.e)
        v[s0] *= 2.0 ** -v_shift
    sc.k, sc.v = k.to(torch.bfloat16), v.to(torch.bfloat16)
    requantize(sc)
    return sc


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
@pytest.mark.parametrize("g", [4, 8, 16])
@pytest.mark.parametrize("gap,v_shift", [(12, 8), (20, 8), (20, 14), (20, 20), (30, 14), (30, 30)])
def test_attention_sink_small_v(cuda, kv_dtype, g, gap, v_shift):
    """A dominant first token whose V is ~0 (round 1 measured 2.7-3.3e-3 here
    with P' anchored on the max score; the contribution anchor keeps the
    ordinary tokens' P' in f16's normal range)."""
    sc = _sink_scenario(kv_dtype, g, gap, v_shift, seed=5 + g)
    ref = sc.oracle_out()
    for pps in (None, 5):
        out = run(sc, cuda, pages_per_split=pps)
        assert np.isfinite(out).all()
        assert rel_err(out, ref) <= 2e-3, (pps, rel_err(out, ref))


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
@pytest.mark.parametrize("g", [4, 8, 16])
@pytest.mark.parametrize("spread,q_gain", [(10, 1.0), (20, 1.0), (10, 16.0), (20, 16.0), (-20, 16.0),
                                            (10, 40.0), (20, 40.0), (-20, 40.0)])
def test_in_page_v_scale_spread(cuda, kv_dtype, g, spread, q_gain):
    """One token in 16 has its V row scaled by 2^spread, so V scales inside a
    page spread 2^10 / 2^20 (round 1: 2.7e-2 at 2^20 with N(0,1) queries).
    INT8 rounds q to two int8 terms (exact above amax / 128, <= amax * 2^-16
    below); with queries x24..x40 (scores ~300 log2 units) that score rounding
    alone moves the weights of two tokens that share the output by up to 8e-3,
    so from x40 on INT8 is held to the oracle fed the same rounded q (the P'
    path itself at those scores), and to the plain oracle up to x16."""
    sc = Scenario([700, 333, 1200, 40], 8 * g, 8, kv_dtype, seed=30 + g)
    v = sc.v.float()
    T = v.shape[0]
    idx = torch.randperm(T, generator=torch.Generator().manual_seed(g))[: T // 16]
    v[idx] *= 2.0 ** spread
    sc.v = v.to(torch.bfloat16)
    requantize(sc)
    sc.q = (sc.q.float() * q_gain).to(torch.bfloat16)
    if kv_dtype == O.INT8 and q_gain > 16:
        k_deq, v_deq = dense_kv(sc)
        ref = O.decode_attn_np(int8_two_term_q(sc.q, sc.Hkv), k_deq, v_deq, sc.seq_lens)
    else:
        ref = sc.oracle_out()
    for pps in (None, 3):
        out = run(sc, cuda, pages_per_split=pps)
        assert np.isfinite(out).all()
        assert rel_err(out, ref) <= 2e-3, (pps, rel_err(out, ref))


def test_cached_workspace_across_shapes(cuda):
    """The per-stream cached workspace must stay correct when the batch x
    kv-head count goes large -> small -> large (the small call's partials
    land where the large call's split-combine counters live)."""
    # 16 x 8 (b, kv head) counters = 512 B vs 2 x 4 -> 256 B: the small call's
    # partials start inside the big call's counter region.
    big = Scenario([900, 1700, 33, 2500, 1200, 64, 800, 1500] * 2, 32, 8, O.INT8, seed=90)
    small = Scenario([3000, 2000], 32, 4, O.INT8, seed=91)
    ref_big, ref_small = big.oracle_out(), small.oracle_out()
    for _ in range(3):
        for sc, ref, pps in ((big, ref_big, 4), (small, ref_small, 3)):
            # fresh NaN output each call: a skipped combine must not pass on a
            # previous call's result left in recycled memory
            out = torch.full((sc.B, sc.Hq, 128), float("nan"), device=cuda)
            assert rel_err(run(sc, cuda, pages_per_split=pps, out=out), ref) <= 2e-3


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("seed", range(12))
def test_random_decode_steps(cuda, seed, fused):
    """decode_step (K1 + PDL-launched K2 in one call, or K2 alone quantizing
    the new rows itself with fused_append) on random shapes: the new row of
    every sequence (opening a fresh block when its last page is full) lands
    bit-exact where the oracle puts it, and the attention over the grown
    sequences matches the oracle."""
    from paper_2605_29639_b200 import decode_step
    rng = np.random.default_rng(2000 + seed)
    Hkv = int(rng.choice([1, 2, 4, 8]))
    Hq = Hkv * int(rng.choice([1, 2, 4, 8, 16]))
    B = int(rng.integers(1, 10))
    lens = [int(rng.choice([0, 1, 15, 16, 32])) if rng.random() < 0.3 else int(rng.integers(1, 2500))
            for _ in range(B)]
    kvd = O.INT8 if seed % 2 == 0 else O.FP8_E4M3
    sc = Scenario(lens, Hq, Hkv, kvd, seed=seed, extra_blocks=B + 2,
                  max_blocks=max(-(-L // 16) for L in lens) + 1)
    used = set(sc.block_table[b, i] for b in range(B) for i in range(-(-lens[b] // 16)))
    free = [i for i in range(sc.num_blocks) if i not in used]
    table = sc.block_table.copy()
    slots = []
    for b, L in enumerate(lens):
        if L % 16 == 0:
            table[b, L // 16] = free.pop()
        slots.append(int(table[b, L // 16]) * 16 + L % 16)
    g = torch.Generator().manual_seed(seed)
    k = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
    v = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
    q = torch.randn((B, Hq, 128), generator=g).to(torch.bfloat16)
    lens1 = np.asarray(lens, np.int32) + 1
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=NAMES[kvd]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    pps = None if rng.random() < 0.5 else int(rng.integers(1, 40))
    out = decode_step(cache, k.to(cuda), v.to(cuda), torch.tensor(slots, dtype=torch.int32, device=cuda),
                      q.to(cuda), torch.from_numpy(table).to(cuda), torch.from_numpy(lens1).to(cuda),
                      out_dtype=torch.float32, pages_per_split=pps, append_tail_only=bool(seed % 3 == 0),
                      fused_append=fused)
    pool = sc.pool.copy()
    O.quant_append(bf16_bits(k), bf16_bits(v), np.asarray(slots, np.int32), kvd, pool)
    assert np.array_equal(cache.pool.cpu().numpy(), pool)
    ref = O.decode_attn(bf16_bits(q), pool, table, lens1, Hkv, kvd)
    assert rel_err(out.cpu().numpy(), ref) <= 2e-3, (lens, Hq, Hkv, kvd, pps)


@pytest.mark.parametrize("seed", range(10))
def test_random_multi_query(cuda, seed):
    """Multi-query (speculative scoring) attention on random shapes: q_len new
    tokens per sequence, causal among themselves, g * q_len <= 16 query rows per
    kv head, ragged lengths, both formats, random split sizes.  Oracle: query i
    of sequence b == single-query attention over seq_len - (q_len - 1 - i)
    tokens."""
    rng = np.random.default_rng(3000 + seed)
    q_len = int(rng.integers(2, 6))
    g = int(rng.choice([gg for gg in (1, 2, 4, 8) if gg * q_len <= 16]))
    Hkv = int(rng.choice([1, 2, 4, 8]))
    Hq = g * Hkv
    B = int(rng.integers(1, 8))
    lens = [int(rng.integers(q_len, 2500)) for _ in range(B)]
    kvd = O.INT8 if seed % 2 == 0 else O.FP8_E4M3
    sc = Scenario(lens, Hq, Hkv, kvd, seed=seed + 500)
    gq = torch.Generator().manual_seed(seed)
    q4 = torch.randn((B, q_len, Hq, 128), generator=gq).to(torch.bfloat16)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=NAMES[kvd]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    pps = None if rng.random() < 0.5 else int(rng.integers(1, 40))
    out = paged_decode_attention(q4.to(cuda), cache, torch.from_numpy(sc.block_table).to(cuda),
                                 torch.from_numpy(sc.seq_lens).to(cuda), out_dtype=torch.float32,
                                 pages_per_split=pps).cpu().numpy()
    qe = q4.reshape(B * q_len, Hq, 128)
    table = np.repeat(sc.block_table, q_len, axis=0)
    le = np.asarray([L - (q_len - 1 - i) for L in lens for i in range(q_len)], np.int32)
    ref = O.decode_attn(bf16_bits(qe), sc.pool, table, le, Hkv, kvd).reshape(B, q_len, Hq, 128)
    assert rel_err(out, ref) <= 2e-3, (lens, q_len, g, Hkv, kvd, pps)


@pytest.mark.parametrize("kv_dtype", [O.INT8, O.FP8_E4M3])
def test_multi_query_split_invisible_to_early_drafts(cuda, kv_dtype):
    """A split whose pages hold only the newest draft tokens is invisible to
    the earlier draft rows (their causal length ends before it): its partial
    must weigh 0 in the combine, not NaN (found by test_random_multi_query)."""
    q_len, g, Hkv = 5, 2, 1
    lens = [1441, 17, 33, 165]      # 1441 = 90 full pages + 1 token
    sc = Scenario(lens, g * Hkv, Hkv, kv_dtype, seed=77)
    q4 = torch.randn((len(lens), q_len, g * Hkv, 128), generator=torch.Generator().manual_seed(1)).to(torch.bfloat16)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=NAMES[kv_dtype]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    qe = q4.reshape(len(lens) * q_len, g * Hkv, 128)
    table = np.repeat(sc.block_table, q_len, axis=0)
    le = np.asarray([L - (q_len - 1 - i) for L in lens for i in range(q_len)], np.int32)
    ref = O.decode_attn(bf16_bits(qe), sc.pool, table, le, Hkv, kv_dtype).reshape(len(lens), q_len, g * Hkv, 128)
    for pps in (1, 30):
        out = paged_decode_attention(q4.to(cuda), cache, torch.from_numpy(sc.block_table).to(cuda),
                                     torch.from_numpy(sc.seq_lens).to(cuda), out_dtype=torch.float32,
                                     pages_per_split=pps).cpu().numpy()
        assert np.isfinite(out).all()
        assert rel_err(out, ref) <= 2e-3, pps


@pytest.mark.parametrize("seed", range(10))
def test_random_appends_bit_exact(cuda, seed):
    """K1 on random appends: random T (both kernels: the one-warp-per-row kernel
    up to 8192 (token, head) rows, the tile kernel above), 1-8 kv heads,
    whole-page runs mixed with scattered, skipped (-1) and out-of-range slots,
    rows scaled over 2^-60..2^60 with zeros, +-inf and NaN injected; the pool
    bytes must equal the oracle's bit for bit."""
    rng = np.random.default_rng(4000 + seed)
    Hkv = int(rng.choice([1, 2, 4, 6, 8]))
    kvd = "int8" if seed % 2 == 0 else "fp8_e4m3"
    nb = int(rng.integers(64, 1200))
    T = int(rng.choice([rng.integers(1, 300), rng.integers(1500, 4000)]))
    slots = []
    perm = rng.permutation(nb)
    used = 0
    while len(slots) < T:
        if rng.random() < 0.5 and used < nb:          # a whole page
            blk = int(perm[used]); used += 1
            slots += [blk * 16 + t for t in range(16)]
        elif used < nb:                                # a scattered token in a fresh block
            blk = int(perm[used]); used += 1
            slots.append(blk * 16 + int(rng.integers(0, 16)))
        else:
            slots.append(-1)
    slots = np.asarray(slots[:T], np.int32)
    slots[rng.random(T) < 0.05] = -1
    oob = rng.random(T) < 0.02
    slots[oob] = nb * 16 + 5                           # past the pool: skipped by both
    g = torch.Generator().manual_seed(seed)
    k = torch.randn((T, Hkv, 128), generator=g)
    v = torch.randn((T, Hkv, 128), generator=g)
    for x in (k, v):
        x *= torch.exp2(torch.randint(-60, 61, (T, Hkv, 1), generator=g).float())
        m = torch.rand((T, Hkv, 128), generator=g)
        x[m < 0.001] = float("inf")
        x[(m > 0.001) & (m < 0.002)] = float("-inf")
        x[(m > 0.002) & (m < 0.003)] = float("nan")
        x[torch.rand((T, Hkv, 1), generator=g).expand(T, Hkv, 128) < 0.02] = 0.0
    k, v = k.to(torch.bfloat16), v.to(torch.bfloat16)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kvd), nb, device=cuda)
    quantize_append(cache, k.to(cuda), v.to(cuda), torch.from_numpy(slots).to(cuda))
    ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k), bf16_bits(v), np.where(oob, -1, slots).astype(np.int32), DT_SWEEP[kvd], ref)
    assert np.array_equal(cache.pool.cpu().numpy(), ref), (T, Hkv, kvd)


DT_SWEEP = {"int8": O.INT8, "fp8_e4m3": O.FP8_E4M3}


@pytest.mark.parametrize("seed", range(8))
def test_random_verify_steps(cuda, seed):
    """The speculative verify step (decode_step with q[B, q_len, Hq, 128]) on
    random shapes: q_len draft rows per sequence appended (crossing into fresh
    blocks where the last page fills up), then scored causally -- pool bytes
    bit-exact and attention within tolerance against the oracle."""
    from paper_2605_29639_b200 import decode_step
    rng = np.random.default_rng(5000 + seed)
    q_len = int(rng.integers(2, 5))
    g = int(rng.choice([gg for gg in (1, 2, 4) if gg * q_len <= 16]))
    Hkv = int(rng.choice([1, 2, 4, 8]))
    Hq = g * Hkv
    B = int(rng.integers(1, 8))
    lens = [int(rng.choice([0, 1, 14, 15, 16, 31])) if rng.random() < 0.3 else int(rng.integers(1, 2000))
            for _ in range(B)]
    kvd = O.INT8 if seed % 2 == 0 else O.FP8_E4M3
    sc = Scenario(lens, Hq, Hkv, kvd, seed=seed + 900, extra_blocks=2 * B + 2,
                  max_blocks=max(-(-(L + q_len) // 16) for L in lens))
    used = set(sc.block_table[b, i] for b in range(B) for i in range(-(-lens[b] // 16)))
    free = [i for i in range(sc.num_blocks) if i not in used]
    table = sc.block_table.copy()
    slots = []
    for b, L in enumerate(lens):
        for t in range(L, L + q_len):
            if t % 16 == 0 and t // 16 >= -(-L // 16):
                table[b, t // 16] = free.pop()
            slots.append(int(table[b, t // 16]) * 16 + t % 16)
    gk = torch.Generator().manual_seed(seed)
    k = torch.randn((B * q_len, Hkv, 128), generator=gk).to(torch.bfloat16)
    v = torch.randn((B * q_len, Hkv, 128), generator=gk).to(torch.bfloat16)
    q4 = torch.randn((B, q_len, Hq, 128), generator=gk).to(torch.bfloat16)
    lens1 = np.asarray(lens, np.int32) + q_len
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=NAMES[kvd]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    pps = None if rng.random() < 0.5 else int(rng.integers(1, 30))
    out = decode_step(cache, k.to(cuda), v.to(cuda), torch.tensor(slots, dtype=torch.int32, device=cuda),
                      q4.to(cuda), torch.from_numpy(table).to(cuda), torch.from_numpy(lens1).to(cuda),
                      out_dtype=torch.float32, pages_per_split=pps).cpu().numpy()
    pool = sc.pool.copy()
    O.quant_append(bf16_bits(k), bf16_bits(v), np.asarray(slots, np.int32), kvd, pool)
    assert np.array_equal(cache.pool.cpu().numpy(), pool)
    qe = q4.reshape(B * q_len, Hq, 128)
    le = np.asarray([L - (q_len - 1 - i) for L in lens1 for i in range(q_len)], np.int32)
    ref = O.decode_attn(bf16_bits(qe), pool, np.repeat(table, q_len, axis=0), le, Hkv, kvd)
    assert rel_err(out, ref.reshape(B, q_len, Hq, 128)) <= 2e-3, (lens, q_len, g, Hkv, kvd, pps)


@pytest.mark.parametrize("seed", range(6))
def test_random_sessions(cuda, seed):
    """DecodeSession (staged uploads, one captured graph per buffer slot, the
    native pipeline submitter) on random shapes, with the tail-only PDL step
    or the fused append, against the eager session: identical outputs step
    after step and identical pools."""
    from paper_2605_29639_b200.session import DecodeSession
    rng = np.random.default_rng(6000 + seed)
    Hkv = int(rng.choice([1, 2, 4, 8]))
    Hq = Hkv * int(rng.choice([1, 2, 4, 8, 16]))
    B = int(rng.integers(1, 10))
    lens = [int(rng.integers(1, 1500)) for _ in range(B)]
    kvd = "int8" if seed % 2 == 0 else "fp8_e4m3"
    sc = Scenario(lens, Hq, Hkv, O.INT8 if kvd == "int8" else O.FP8_E4M3, seed=seed + 40)
    table = torch.from_numpy(sc.block_table).to(cuda)
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    caches = [PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kvd), sc.num_blocks, device=cuda, pool=pool0.clone())
              for _ in range(2)]
    fused = seed % 3 == 0
    eager = DecodeSession(caches[0], table, B, Hq)
    fast = DecodeSession(caches[1], table, B, Hq, graphs=True, append_tail_only=True, fused_append=fused)
    g = torch.Generator().manual_seed(seed)
    lens_t = torch.from_numpy(sc.seq_lens)
    slots = torch.tensor([int(sc.block_table[b, (L - 1) // 16]) * 16 + (L - 1) % 16 for b, L in enumerate(lens)],
                         dtype=torch.int32)
    outs = []
    for step in range(5):
        q = torch.randn((B, Hq, 128), generator=g).to(torch.bfloat16)
        k = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
        o_a = torch.empty((B, Hq, 128), dtype=torch.bfloat16, pin_memory=True)
        o_b = torch.empty_like(o_a).pin_memory()
        eager.submit(q.pin_memory(), k.pin_memory(), v.pin_memory(), slots.pin_memory(), lens_t.pin_memory(), o_a)
        h = fast.next_inputs()
        for name, t in (("q", q), ("k", k), ("v", v), ("slots", slots), ("lens", lens_t)):
            h[name].copy_(t)
        fast.submit_staged(o_b)
        outs.append((o_a, o_b))
        eager.synchronize()
        fast.synchronize()
    for a, b in outs:
        assert torch.equal(a, b)
    assert torch.equal(caches[0].pool, caches[1].pool)


@pytest.mark.parametrize("seed", range(8))
def test_random_layouts(cuda, seed):
    """Output layouts and strides on random shapes: q a batch-strided view of a
    wider tensor (the fused QKV projection case), bf16 or fp32 output,
    [B, Hq, d] or head-major [Hq, B, d], into a caller-provided `out`."""
    rng = np.random.default_rng(7000 + seed)
    Hkv = int(rng.choice([1, 2, 4, 8]))
    Hq = Hkv * int(rng.choice([1, 2, 4, 8, 16]))
    B = int(rng.integers(1, 9))
    lens = [int(rng.integers(1, 1200)) for _ in range(B)]
    kvd = O.INT8 if seed % 2 == 0 else O.FP8_E4M3
    sc = Scenario(lens, Hq, Hkv, kvd, seed=seed + 60)
    extra = int(rng.integers(1, 5)) * Hkv                 # the K/V heads of a fused QKV row
    wide = torch.randn((B, Hq + 2 * extra, 128), generator=torch.Generator().manual_seed(seed)).to(torch.bfloat16)
    wide[:, :Hq] = sc.q
    q = wide.to(cuda)[:, :Hq]                             # stride(0) = (Hq + 2 extra) * 128
    assert q.stride(0) != Hq * 128
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=NAMES[kvd]), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    out_dtype = torch.float32 if rng.random() < 0.5 else torch.bfloat16
    head_major = bool(rng.random() < 0.5)
    shape = (Hq, B, 128) if head_major else (B, Hq, 128)
    out = torch.full(shape, float("nan"), dtype=out_dtype, device=cuda)
    res = paged_decode_attention(q, cache, torch.from_numpy(sc.block_table).to(cuda),
                                 torch.from_numpy(sc.seq_lens).to(cuda), out=out, out_dtype=out_dtype,
                                 head_major=head_major)
    assert res.data_ptr() == out.data_ptr()
    got = out.float().cpu().numpy()
    if head_major:
        got = got.transpose(1, 0, 2)
    ref = sc.oracle_out()
    if out_dtype == torch.float32:
        assert rel_err(got, ref) <= 2e-3
    else:
        assert np.all(np.abs(got - ref) <= 1e-2 + 2.0 ** -8 * np.abs(ref))
