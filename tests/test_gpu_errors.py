"""Caller errors the kernels can only see on the device (kvq_check_device_errors,
include/kvq.h): an out-of-range block id (K2), a sequence length past the
table (K2), a slot past the pool (K1 both kernels, the fused append).  The
kernels skip or clamp instead of faulting and report a bit; the oracle
abort()s on the same inputs.  Plus: the fused append skips an invalid slot
exactly as K1 does (output == K1 + K2)."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import Scenario
from paper_2605_29639_b200 import (KVCacheSpec, PagedKVCache, check_device_errors, decode_step,
                                   paged_decode_attention, quantize_append)

pytestmark = pytest.mark.gpu


def _clear():
    """Bits left by earlier tests that pass out-of-range input on purpose."""
    try:
        check_device_errors()
    except ValueError:
        pass


def _setup(cuda):
    _clear()
    sc = Scenario([300, 17, 64], 32, 8, O.INT8, seed=3, extra_blocks=4)
    cache = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=torch.from_numpy(sc.pool).to(cuda))
    return sc, cache


def test_clean_calls_report_nothing(cuda):
    sc, cache = _setup(cuda)
    paged_decode_attention(sc.q.to(cuda), cache, torch.from_numpy(sc.block_table).to(cuda),
                           torch.from_numpy(sc.seq_lens).to(cuda))
    check_device_errors()


def test_block_id_out_of_range(cuda):
    sc, cache = _setup(cuda)
    table = sc.block_table.copy()
    table[1, 0] = sc.num_blocks + 5
    paged_decode_attention(sc.q.to(cuda), cache, torch.from_numpy(table).to(cuda),
                           torch.from_numpy(sc.seq_lens).to(cuda))
    with pytest.raises(ValueError, match="KVQ_DERR_BLOCK_ID"):
        check_device_errors()
    check_device_errors()                               # read-and-clear


def test_seq_len_past_the_table(cuda):
    sc, cache = _setup(cuda)
    lens = sc.seq_lens.copy()
    lens[2] = sc.block_table.shape[1] * 16 + 1
    paged_decode_attention(sc.q.to(cuda), cache, torch.from_numpy(sc.block_table).to(cuda),
                           torch.from_numpy(lens).to(cuda))
    with pytest.raises(ValueError, match="KVQ_DERR_SEQ_LEN"):
        check_device_errors()


@pytest.mark.parametrize("T", [3, 4096])   # one-warp-per-row kernel / tile kernel
def test_slot_past_the_pool(cuda, T):
    _clear()
    cache = PagedKVCache(KVCacheSpec(8), 300, device=cuda)
    k = torch.randn((T, 8, 128), device=cuda).to(torch.bfloat16)
    slots = torch.arange(T, dtype=torch.int32, device=cuda)
    slots[T // 2] = 300 * 16 + 3                          # past the pool
    slots[0] = -1                                         # skip: not an error
    quantize_append(cache, k, k, slots)
    with pytest.raises(ValueError, match="KVQ_DERR_SLOT"):
        check_device_errors()
    slots[T // 2] = -7
    quantize_append(cache, k, k, slots)
    check_device_errors()


@pytest.mark.parametrize("Hq", [32, 128])
def test_fused_append_invalid_slots_match_k1(cuda, Hq):
    """Rows with a negative slot are skipped by K1; the fused append must skip
    them too (no pool write, no patch of the CTA's page copy), and an
    out-of-range slot is skipped and reported."""
    _clear()
    lens = [300, 17, 1020, 64]
    sc = Scenario(lens, Hq, 8, O.INT8, seed=8, extra_blocks=6, max_blocks=65)
    table = torch.from_numpy(sc.block_table).to(cuda)
    slots_np = [int(sc.block_table[b, (L - 1) // 16]) * 16 + (L - 1) % 16 for b, L in enumerate(lens)]
    slots_np[1] = -1
    slots_np[3] = -5
    slots = torch.tensor(slots_np, dtype=torch.int32, device=cuda)
    lens_t = torch.tensor(lens, dtype=torch.int32, device=cuda)
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    a = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone())
    b = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone())
    g = torch.Generator(device=cuda).manual_seed(1)
    k = torch.randn((4, 8, 128), device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn((4, 8, 128), device=cuda, generator=g).to(torch.bfloat16)
    q = torch.randn((4, Hq, 128), device=cuda, generator=g).to(torch.bfloat16)
    oa = decode_step(a, k, v, slots, q, table, lens_t, out_dtype=torch.float32, fused_append=True)
    ob = decode_step(b, k, v, slots, q, table, lens_t, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(a.pool, b.pool) and torch.equal(oa, ob)
    check_device_errors()
    slots[2] = sc.num_blocks * 16
    decode_step(a, k, v, slots, q, table, lens_t, out_dtype=torch.float32, fused_append=True)
    with pytest.raises(ValueError, match="KVQ_DERR_SLOT"):
        check_device_errors()
    assert np.isfinite(oa.cpu().numpy()).all()
