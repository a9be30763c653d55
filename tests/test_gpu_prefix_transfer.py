"""On the B200: prefix-cached pages promoted back from the pinned-host tier
and pages exported/imported for a PD transfer feed the decode kernel exactly
as freshly quantized pages do."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import bf16_bits, make_kv, make_q
from paper_2605_29639_b200 import (KVCacheSpec, PagedKVCache, copy_blocks, paged_decode_attention,
                                   quantize_append)
from paper_2605_29639_b200.prefix import PrefixKVCache
from paper_2605_29639_b200.transfer import export_pages, import_pages

pytestmark = pytest.mark.gpu


def test_host_tier_round_trip_then_attention(cuda):
    spec = KVCacheSpec(8, kv_dtype="int8")
    pkv = PrefixKVCache(spec, 40, device=cuda, host_blocks=64)
    a = list(range(300, 300 + 400))                       # 25 pages
    _, slots = pkv.admit("A", a)
    k, v = make_kv(400, 8, 41), make_kv(400, 8, 42, kind="v")
    quantize_append(pkv.cache, k.to(cuda), v.to(cuda), torch.tensor(slots, dtype=torch.int32, device=cuda))
    ref_pages = pkv.cache.pool[torch.as_tensor(pkv.alloc.block_ids("A"), device=cuda)].cpu()
    pkv.free("A")
    _, s2 = pkv.admit("X", list(range(9000, 9000 + 480)))   # 30 pages: evicts A's
    pkv.free("X")
    cached, rest = pkv.admit("A2", a + [7])
    assert cached == 400 and pkv.stats()["host_hit_tokens"] > 0
    quantize_append(pkv.cache, make_kv(1, 8, 43).to(cuda), make_kv(1, 8, 44, kind="v").to(cuda),
                    torch.tensor(rest, dtype=torch.int32, device=cuda))
    blocks = pkv.alloc.block_ids("A2")
    got = pkv.cache.pool[torch.as_tensor(blocks[:25], device=cuda)].cpu()
    assert torch.equal(got, ref_pages)
    q = make_q(1, 32, 45)
    table = torch.tensor([blocks], dtype=torch.int32, device=cuda)
    out = paged_decode_attention(q.to(cuda), pkv.cache, table, torch.tensor([401], dtype=torch.int32, device=cuda),
                                 out_dtype=torch.float32).cpu().numpy()
    pool = pkv.cache.pool.cpu().numpy()
    ref = O.decode_attn(bf16_bits(q), pool, np.asarray([blocks], np.int32), np.asarray([401], np.int32), 8, O.INT8)
    err = np.abs(out - ref).max(-1) / np.abs(ref).max(-1)
    assert err.max() <= 2e-3


def test_export_import_pages(cuda):
    spec = KVCacheSpec(4, kv_dtype="fp8_e4m3")
    src = PagedKVCache(spec, 10, device=cuda)
    src.pool.copy_(torch.randint(0, 256, src.pool.shape, dtype=torch.uint8, device=cuda))
    dst = PagedKVCache(spec, 10, device=cuda)
    pages = export_pages(src, [3, 7, 1])
    import_pages(dst, [0, 5, 9], pages)
    for s, d in ((3, 0), (7, 5), (1, 9)):
        assert torch.equal(src.pool[s], dst.pool[d])


@pytest.mark.parametrize("Hkv", [1, 3, 8])
def test_gather_scatter_blocks_native(cuda, Hkv):
    """kvq_gather_blocks / kvq_scatter_blocks (the PD wire format) and the
    copy-on-write kvq_copy_blocks move whole blocks bit for bit, for odd head
    counts and many blocks; out-of-range ids are skipped."""
    nb = 700
    src = PagedKVCache(KVCacheSpec(Hkv), nb, device=cuda)
    src.pool.random_(0, 256)
    rng = np.random.default_rng(Hkv)
    ids = rng.permutation(nb)[:500].tolist()
    pages = export_pages(src, ids)
    assert torch.equal(pages, src.pool[torch.as_tensor(ids, device=cuda)])
    dst = PagedKVCache(KVCacheSpec(Hkv), nb, device=cuda)
    dids = rng.permutation(nb)[:500].tolist()
    import_pages(dst, dids, pages)
    assert torch.equal(dst.pool[torch.as_tensor(dids, device=cuda)], pages)
    untouched = sorted(set(range(nb)) - set(dids))
    assert int(dst.pool[torch.as_tensor(untouched, device=cuda)].count_nonzero()) == 0
    before = dst.pool.clone()
    copy_blocks(dst, [(dids[0], dids[1]), (nb + 5, dids[2])])       # second pair is out of range: skipped
    torch.cuda.synchronize()
    assert torch.equal(dst.pool[dids[1]], before[dids[0]]) and torch.equal(dst.pool[dids[2]], before[dids[2]])
