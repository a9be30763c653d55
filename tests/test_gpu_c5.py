"""C5 at full size against the oracle: the chunked-prefill + decode mix with
prefix-shared blocks (BASELINE.json configs[4]; bench.py run_c5 builds the
same mix).  252 decode sequences in groups of 8 fork a 1,024-token (64-block)
prefix and own a private suffix ~U{64..3072}; one decode step appends 4 x 2K
prefill-chunk rows plus every sequence's newest token (K1) and attends the 252
sequences (K2 PDL-launched behind K1, tail-only wait).  Every page written by
K1 is bit-identical to the oracle's, and EVERY attended sequence's output is
within 2e-3 of the oracle's, for INT8 and FP8.  The shared prefix pages are
written once and read by 8 sequences each (the reference's shared-full /
exclusive-partial rule, tiered_cache.py:355-363, via BlockAllocator.fork)."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import bf16_bits
from paper_2605_29639_b200 import BlockAllocator, KVCacheSpec, PagedKVCache, decode_step, quantize_append

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("kvd,kvo", [("int8", O.INT8), ("fp8_e4m3", O.FP8_E4M3)])
def test_c5_mix_every_sequence_vs_oracle(cuda, kvd, kvo):
    B, Hq, Hkv, G, prefix, chunk, n_pf = 252, 32, 8, 8, 1024, 2048, 4
    suffix = np.random.default_rng(5).integers(64, 3073, size=B)
    ngroups = -(-B // G)
    spec = KVCacheSpec(Hkv, kv_dtype=kvd)
    nb = ngroups * prefix // 16 + int(np.ceil((suffix + 1) / 16).sum()) + B + n_pf * chunk // 16 + 64
    alloc = BlockAllocator(nb, bytes_per_block=spec.bytes_per_block)
    cache = PagedKVCache(spec, nb, device=cuda)
    ref_pool = np.zeros((nb, Hkv, O.PAGE), np.uint8)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(7 + kvo)

    def rows(n):
        x = torch.randn((2, n, Hkv, 128), device=cuda, generator=gen)
        return (x * torch.exp(0.5 * torch.randn((2, n, Hkv, 1), device=cuda, generator=gen))).to(torch.bfloat16)

    def append(slots, kv):  # K1 on the GPU, the oracle's quantizer into the CPU pool
        quantize_append(cache, kv[0], kv[1], torch.tensor(slots, dtype=torch.int32, device=cuda))
        O.quant_append(bf16_bits(kv[0]), bf16_bits(kv[1]), np.asarray(slots, np.int32), kvo, ref_pool)

    seqs = []
    for gi in range(ngroups):
        pid = ("prefix", gi)
        alloc.allocate(pid)
        append(alloc.append_slots(pid, prefix), rows(prefix))
        for j in range(G):
            b = gi * G + j
            if b >= B:
                break
            assert alloc.fork(pid, b) == []          # block-aligned prefix: shared, nothing copied
            append(alloc.append_slots(b, int(suffix[b])), rows(int(suffix[b])))
            seqs.append(b)
        alloc.free(pid)
    shared = alloc.block_ids(0)[: prefix // 16]
    assert all(alloc.ref_count(blk) == G for blk in shared)
    # one step: 4 prefill chunks (sequences K2 does not attend) + each decode sequence's newest token
    pf_slots = []
    for i in range(n_pf):
        alloc.allocate(("prefill", i))
        pf_slots += alloc.append_slots(("prefill", i), chunk)
    dec_slots = [int(s) for s in alloc.append_one(seqs)]
    alloc.check_invariants()
    step_kv = rows(len(pf_slots) + B)
    slots = pf_slots + dec_slots
    table = alloc.block_table(seqs)
    lens = alloc.seq_lens(seqs)
    q = torch.randn((B, Hq, 128), device=cuda, generator=gen).to(torch.bfloat16)
    out = decode_step(cache, step_kv[0], step_kv[1], torch.tensor(slots, dtype=torch.int32, device=cuda), q,
                      torch.from_numpy(table).to(cuda), torch.from_numpy(lens).to(cuda),
                      out_dtype=torch.float32, append_tail_only=True)
    O.quant_append(bf16_bits(step_kv[0]), bf16_bits(step_kv[1]), np.asarray(slots, np.int32), kvo, ref_pool)
    torch.cuda.synchronize()
    gpu_pool = cache.pool.cpu().numpy()
    assert np.array_equal(gpu_pool, ref_pool), int((gpu_pool != ref_pool).sum())
    ref = O.decode_attn(bf16_bits(q), ref_pool, table, lens, Hkv, kvo)
    o = out.cpu().numpy()
    err = np.abs(o - ref).max(-1) / (np.abs(ref).max(-1) + 5e-4)
    assert np.isfinite(o).all()
    assert err.max() <= 2e-3, float(err.max())
