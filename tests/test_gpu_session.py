"""DecodeSession: pipelined host->device->host decode steps produce exactly the
outputs of direct op calls, step after step (double buffering is race-free),
and CUDA-graph replays of K1/K2 reproduce them too."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import Scenario
from paper_2605_29639_b200 import (KVCacheSpec, PagedKVCache, decode_step, paged_decode_attention,
                                   quantize_append)
from paper_2605_29639_b200.session import DecodeSession

pytestmark = pytest.mark.gpu


def test_session_matches_direct_calls(cuda):
    sc = Scenario([100, 37, 700, 16], 32, 8, O.INT8, seed=21, extra_blocks=20)
    B = sc.B
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    table = torch.from_numpy(sc.block_table).to(cuda)
    lens = sc.seq_lens.copy()
    # extra block capacity: append into a fresh block per step where needed
    cache_a = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone())
    cache_b = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone())
    free = [b for b in range(sc.num_blocks) if b not in set(sc.block_table.reshape(-1).tolist())]
    tab = sc.block_table.copy()
    mb = tab.shape[1]
    tab = np.concatenate([tab, np.zeros((B, 8), np.int32)], 1)
    table = torch.from_numpy(tab).to(cuda)
    sess = DecodeSession(cache_b, table, B, 32)
    g = torch.Generator().manual_seed(5)
    outs_direct, outs_sess, hosts = [], [], []
    for step in range(6):
        slots = []
        for b in range(B):
            pos = lens[b]
            if pos % 16 == 0:
                tab[b, pos // 16] = free.pop()
            slots.append(tab[b, pos // 16] * 16 + pos % 16)
        lens = lens + 1
        table.copy_(torch.from_numpy(tab))
        q = torch.randn((B, 32, 128), generator=g).to(torch.bfloat16)
        k = torch.randn((B, 8, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((B, 8, 128), generator=g).to(torch.bfloat16)
        sl = torch.tensor(slots, dtype=torch.int32)
        ln = torch.from_numpy(lens.astype(np.int32))
        quantize_append(cache_a, k.to(cuda), v.to(cuda), sl.to(cuda))
        outs_direct.append(paged_decode_attention(q.to(cuda), cache_a, table, ln.to(cuda)).cpu())
        host = [t.pin_memory() for t in (q, k, v, sl, ln)]
        o_h = torch.empty((B, 32, 128), dtype=torch.bfloat16, pin_memory=True)
        hosts.append(host)
        sess.submit(*host, o_h)
        outs_sess.append(o_h)
        torch.cuda.synchronize()   # table edits between steps are host-side; keep ordering simple
    sess.synchronize()
    for a, b in zip(outs_direct, outs_sess):
        assert torch.equal(a, b)
    assert torch.equal(cache_a.pool, cache_b.pool)


def test_session_back_to_back_and_graphs(cuda):
    sc = Scenario([300, 1200, 64], 64, 8, O.FP8_E4M3, seed=22)
    cache = PagedKVCache(KVCacheSpec(8, kv_dtype="fp8_e4m3"), sc.num_blocks, device=cuda,
                         pool=torch.from_numpy(sc.pool).to(cuda))
    table = torch.from_numpy(sc.block_table).to(cuda)
    sess = DecodeSession(cache, table, sc.B, 64, head_major=True)
    # slot -1: no append, so every step is identical -> identical outputs
    q = sc.q.pin_memory()
    k = torch.zeros((sc.B, 8, 128), dtype=torch.bfloat16).pin_memory()
    sl = torch.full((sc.B,), -1, dtype=torch.int32).pin_memory()
    ln = torch.from_numpy(sc.seq_lens).pin_memory()
    outs = [torch.empty((64, sc.B, 128), dtype=torch.bfloat16, pin_memory=True) for _ in range(8)]
    for o in outs:
        sess.submit(q, k, k, sl, ln, o)
    sess.synchronize()
    ref = sc.oracle_out().transpose(1, 0, 2)
    for o in outs:
        assert torch.equal(o, outs[0])
    assert np.all(np.abs(outs[0].float().numpy() - ref) <= 1e-2 + 2.0 ** -8 * np.abs(ref))
    g1, g2 = sess.capture()
    buf = sess.device_buffers(0)
    buf["out"].zero_()
    g1.replay()
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(buf["out"].cpu(), outs[0])


@pytest.mark.parametrize("staged", [False, True])
def test_session_graphs_and_staged_match_eager(cuda, staged):
    """graphs=True (one captured graph per buffer slot) and the single-copy
    staged upload give the eager session's bytes, step after step, while the
    steps' inputs change."""
    sc = Scenario([200, 33, 900, 17, 64], 32, 8, O.INT8, seed=23, extra_blocks=4)
    table = torch.from_numpy(sc.block_table).to(cuda)
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    caches = [PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone()) for _ in range(2)]
    eager = DecodeSession(caches[0], table, sc.B, 32)
    fast = DecodeSession(caches[1], table, sc.B, 32, graphs=True)
    g = torch.Generator().manual_seed(9)
    lens = torch.from_numpy(sc.seq_lens)
    # re-append the last token of each sequence with new values each step
    slots = torch.tensor([int(sc.block_table[b, (L - 1) // 16]) * 16 + (L - 1) % 16
                          for b, L in enumerate(sc.seq_lens)], dtype=torch.int32)
    outs = []
    for step in range(7):
        q = torch.randn((sc.B, 32, 128), generator=g).to(torch.bfloat16)
        k = torch.randn((sc.B, 8, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((sc.B, 8, 128), generator=g).to(torch.bfloat16)
        o_a = torch.empty((sc.B, 32, 128), dtype=torch.bfloat16, pin_memory=True)
        o_b = torch.empty_like(o_a).pin_memory()
        eager.submit(q.pin_memory(), k.pin_memory(), v.pin_memory(), slots.pin_memory(), lens.pin_memory(), o_a)
        if staged:
            h = fast.next_inputs()
            for name, t in (("q", q), ("k", k), ("v", v), ("slots", slots), ("lens", lens)):
                h[name].copy_(t)
            fast.submit_staged(o_b)
        else:
            fast.submit(q.pin_memory(), k.pin_memory(), v.pin_memory(), slots.pin_memory(), lens.pin_memory(), o_b)
        outs.append((o_a, o_b))
        eager.synchronize()   # the two sessions share nothing but keep their pools in lock step
        fast.synchronize()
    for a, b in outs:
        assert torch.equal(a, b)
    assert torch.equal(caches[0].pool, caches[1].pool)
    assert len({int(o[0].float().sum()) for o in outs}) > 1, "inputs must change between steps"


@pytest.mark.parametrize("tail_only", [False, True])
@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_decode_step_matches_two_calls(cuda, kv_dtype, tail_only):
    """kvq_decode_step (K2 PDL-launched behind K1) == quantize_append then
    paged_decode_attention: identical pages, identical output, eager and in a
    CUDA graph replayed with new rows; the appended rows are visible to K2."""
    kvo = O.INT8 if kv_dtype == "int8" else O.FP8_E4M3
    sc = Scenario([300, 17, 1020, 60, 1999], 32, 8, kvo, seed=21)  # each last page has room
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    a = PagedKVCache(KVCacheSpec(8, kv_dtype=kv_dtype), sc.num_blocks, device=cuda, pool=pool0.clone())
    b = PagedKVCache(KVCacheSpec(8, kv_dtype=kv_dtype), sc.num_blocks, device=cuda, pool=pool0.clone())
    table = torch.from_numpy(sc.block_table).to(cuda)
    # one new token per sequence at position seq_len (tables have room: extra blocks appended)
    lens = sc.seq_lens.astype(np.int64)
    assert all(lens[i] // 16 < -(-lens[i] // 16) for i in range(sc.B))
    slots = torch.from_numpy((sc.block_table[np.arange(sc.B), lens // 16].astype(np.int64) * 16
                              + lens % 16).astype(np.int32)).to(cuda)
    lens1 = torch.from_numpy((lens + 1).astype(np.int32)).to(cuda)
    g = torch.Generator(device=cuda).manual_seed(5)
    k = torch.randn((sc.B, 8, 128), device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn((sc.B, 8, 128), device=cuda, generator=g).to(torch.bfloat16)
    q = torch.randn((sc.B, 32, 128), device=cuda, generator=g).to(torch.bfloat16)
    out_a = decode_step(a, k, v, slots, q, table, lens1, out_dtype=torch.float32, pages_per_split=8,
                        append_tail_only=tail_only)
    quantize_append(b, k, v, slots)
    out_b = paged_decode_attention(q, b, table, lens1, out_dtype=torch.float32, pages_per_split=8)
    torch.cuda.synchronize()
    assert torch.equal(a.pool, b.pool)
    assert torch.equal(out_a, out_b)
    # graph of the fused step, replayed with fresh rows
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=cuda)
    out_g = torch.empty((sc.B, 32, 128), dtype=torch.float32, device=cuda)
    gr = torch.cuda.CUDAGraph()
    decode_step(a, k, v, slots, q, table, lens1, out=out_g, out_dtype=torch.float32, pages_per_split=8,
                workspace=ws, append_tail_only=tail_only)
    torch.cuda.synchronize()
    with torch.cuda.graph(gr):
        decode_step(a, k, v, slots, q, table, lens1, out=out_g, out_dtype=torch.float32, pages_per_split=8,
                    workspace=ws, append_tail_only=tail_only)
    for _ in range(3):
        k.copy_(torch.randn((sc.B, 8, 128), device=cuda, generator=g).to(torch.bfloat16))
        v.copy_(torch.randn((sc.B, 8, 128), device=cuda, generator=g).to(torch.bfloat16))
        gr.replay()
        quantize_append(b, k, v, slots)
        ref = paged_decode_attention(q, b, table, lens1, out_dtype=torch.float32, pages_per_split=8)
        torch.cuda.synchronize()
        assert torch.equal(a.pool, b.pool)
        assert torch.equal(out_g, ref)


def test_native_pipeline_back_to_back(cuda):
    """submit_staged through the native submitter (kvq_pipeline_submit) with no
    host synchronisation between steps: every step's download equals the
    direct op calls for that step's inputs (slot reuse is event-ordered)."""
    sc = Scenario([300, 40, 1200, 17, 64, 900], 32, 8, O.INT8, seed=31)
    table = torch.from_numpy(sc.block_table).to(cuda)
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    ref_cache = PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone())
    sess = DecodeSession(PagedKVCache(KVCacheSpec(8), sc.num_blocks, device=cuda, pool=pool0.clone()),
                         table, sc.B, 32, graphs=True)
    g = torch.Generator().manual_seed(3)
    lens = torch.from_numpy(sc.seq_lens)
    slots = torch.tensor([int(sc.block_table[b, (L - 1) // 16]) * 16 + (L - 1) % 16
                          for b, L in enumerate(sc.seq_lens)], dtype=torch.int32)
    steps, refs, outs = 12, [], []
    for step in range(steps):
        q = torch.randn((sc.B, 32, 128), generator=g).to(torch.bfloat16)
        k = torch.randn((sc.B, 8, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((sc.B, 8, 128), generator=g).to(torch.bfloat16)
        quantize_append(ref_cache, k.to(cuda), v.to(cuda), slots.to(cuda))
        refs.append(paged_decode_attention(q.to(cuda), ref_cache, table, lens.to(cuda)).cpu())
        h = sess.next_inputs()                  # waits only for this slot's previous upload
        for name, t in (("q", q), ("k", k), ("v", v), ("slots", slots), ("lens", lens)):
            h[name].copy_(t)
        o = torch.empty((sc.B, 32, 128), dtype=torch.bfloat16, pin_memory=True)
        sess.submit_staged(o)
        outs.append(o)
    sess.synchronize()
    assert all("pipe" in b for b in sess.bufs), "native submitter not used"
    for a, b in zip(refs, outs):
        assert torch.equal(a, b)


def test_serving_loop_growing_sequences(cuda):
    """A decode loop as a server runs it: every step BlockAllocator.append_one
    picks each sequence's slot (new pages across block boundaries), the
    incremental BlockTable pushes only the new block ids into the device table
    the captured graphs read, and DecodeSession(graphs=True) runs the step
    from staged host inputs.  Each step's download equals direct op calls on
    a second cache fed the same rows."""
    from paper_2605_29639_b200 import BlockAllocator, BlockTable
    B, Hq, Hkv, steps = 6, 32, 8, 40
    alloc = BlockAllocator(400)
    g = torch.Generator().manual_seed(11)
    lens0 = [5, 16, 31, 100, 1, 250]
    ca = PagedKVCache(KVCacheSpec(Hkv), 400, device=cuda)
    cb = PagedKVCache(KVCacheSpec(Hkv), 400, device=cuda)
    for s, n in enumerate(lens0):                      # prefill
        alloc.allocate(s)
        sl = torch.tensor(alloc.append_slots(s, n), dtype=torch.int32, device=cuda)
        k = torch.randn((n, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
        v = torch.randn((n, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
        quantize_append(ca, k, v, sl)
        quantize_append(cb, k, v, sl)
    seqs = list(range(B))
    table = BlockTable(B, 64, device=cuda)
    table.sync(alloc, seqs)
    sess = DecodeSession(ca, table.table, B, Hq, graphs=True, pages_per_split=4)
    outs, refs = [], []
    for step in range(steps):
        slots = torch.from_numpy(alloc.append_one(seqs))
        table.sync(alloc, seqs)                          # new pages land in the captured table
        lens = torch.from_numpy(alloc.seq_lens(seqs))
        q = torch.randn((B, Hq, 128), generator=g).to(torch.bfloat16)
        k = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
        v = torch.randn((B, Hkv, 128), generator=g).to(torch.bfloat16)
        h = sess.next_inputs()
        for name, t in (("q", q), ("k", k), ("v", v), ("slots", slots), ("lens", lens)):
            h[name].copy_(t)
        o = torch.empty((B, Hq, 128), dtype=torch.bfloat16, pin_memory=True)
        sess.submit_staged(o)
        outs.append(o)
        quantize_append(cb, k.to(cuda), v.to(cuda), slots.to(cuda))
        refs.append(paged_decode_attention(q.to(cuda), cb, table.table, lens.to(cuda), pages_per_split=4).cpu())
        sess.synchronize()                               # the table is edited on the host between steps
    for a, b in zip(outs, refs):
        assert torch.equal(a, b)
    assert torch.equal(ca.pool, cb.pool)
    alloc.check_invariants()


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_decode_step_tail_only_with_prefill_rows(cuda, kv_dtype):
    """The C5 shape of a step: one append carries whole prefill chunks of
    sequences K2 does not attend plus each attended sequence's newest token;
    with append_tail_only the result equals the two calls in sequence."""
    from paper_2605_29639_b200 import BlockAllocator
    Hq, Hkv = 32, 8
    alloc = BlockAllocator(600)
    g = torch.Generator().manual_seed(4)
    a = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), 600, device=cuda)
    dec = list(range(12))
    for s in dec:                                    # attended sequences with history
        alloc.allocate(s)
        sl = torch.tensor(alloc.append_slots(s, 37 * (s + 1)), dtype=torch.int32, device=cuda)
        kv = torch.randn((2, sl.numel(), Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
        quantize_append(a, kv[0], kv[1], sl)
    b = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), 600, device=cuda, pool=a.pool.clone())
    for p in ("p0", "p1"):                           # prefill chunks (not attended this step)
        alloc.allocate(p)
    pre = alloc.append_slots("p0", 2048) + alloc.append_slots("p1", 1000)
    tail = alloc.append_one(dec).tolist()
    slots = torch.tensor(pre + tail, dtype=torch.int32, device=cuda)
    T = slots.numel()
    k = torch.randn((T, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
    v = torch.randn((T, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
    q = torch.randn((len(dec), Hq, 128), generator=g).to(torch.bfloat16).to(cuda)
    table = torch.from_numpy(alloc.block_table(dec)).to(cuda)
    lens = torch.from_numpy(alloc.seq_lens(dec)).to(cuda)
    out_a = decode_step(a, k, v, slots, q, table, lens, out_dtype=torch.float32, pages_per_split=4,
                        append_tail_only=True)
    quantize_append(b, k, v, slots)
    out_b = paged_decode_attention(q, b, table, lens, out_dtype=torch.float32, pages_per_split=4)
    torch.cuda.synchronize()
    assert torch.equal(a.pool, b.pool)
    assert torch.equal(out_a, out_b)


@pytest.mark.parametrize("q_len", [2, 4])
def test_decode_step_speculative_verify(cuda, q_len):
    """decode_step with q [B, q_len, Hq, d] (kvq_decode_step_mq): appending
    the q_len draft tokens' rows and scoring them causally equals
    quantize_append then the multi-query paged_decode_attention."""
    from paper_2605_29639_b200 import BlockAllocator
    Hq, Hkv, B = 32, 8, 5
    alloc = BlockAllocator(300)
    g = torch.Generator().manual_seed(q_len)
    a = PagedKVCache(KVCacheSpec(Hkv), 300, device=cuda)
    for s, n in enumerate([15, 16, 33, 200, 1]):
        alloc.allocate(s)
        sl = torch.tensor(alloc.append_slots(s, n), dtype=torch.int32, device=cuda)
        kv = torch.randn((2, n, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
        quantize_append(a, kv[0], kv[1], sl)
    b = PagedKVCache(KVCacheSpec(Hkv), 300, device=cuda, pool=a.pool.clone())
    slots = []
    for s in range(B):                                  # q_len draft tokens per sequence, batch-major
        slots += alloc.append_slots(s, q_len)
    slots = torch.tensor(slots, dtype=torch.int32, device=cuda)
    k = torch.randn((B * q_len, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
    v = torch.randn((B * q_len, Hkv, 128), generator=g).to(torch.bfloat16).to(cuda)
    q = torch.randn((B, q_len, Hq, 128), generator=g).to(torch.bfloat16).to(cuda)
    table = torch.from_numpy(alloc.block_table(list(range(B)))).to(cuda)
    lens = torch.from_numpy(alloc.seq_lens(list(range(B)))).to(cuda)
    out_a = decode_step(a, k, v, slots, q, table, lens, out_dtype=torch.float32, pages_per_split=4,
                        append_tail_only=True)      # ignored for q_len > 1
    quantize_append(b, k, v, slots)
    out_b = paged_decode_attention(q, b, table, lens, out_dtype=torch.float32, pages_per_split=4)
    torch.cuda.synchronize()
    assert out_a.shape == (B, q_len, Hq, 128)
    assert torch.equal(a.pool, b.pool)
    assert torch.equal(out_a, out_b)


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
@pytest.mark.parametrize("Hq,Hkv", [(32, 8), (64, 4)])
def test_decode_step_fused_append(cuda, kv_dtype, Hq, Hkv):
    """KVQ_STEP_FUSED_APPEND (no K1 launch; the K2 CTA holding each sequence's
    last page quantizes its new row) == K1 then K2: identical pool bytes and
    bit-identical output, eager and replayed from a CUDA graph with new rows,
    for the g <= 8 and g = 16 variants, including sequences whose new token
    opens a fresh block."""
    kvo = O.INT8 if kv_dtype == "int8" else O.FP8_E4M3
    lens = [300, 17, 1020, 64, 1999, 0, 15]
    sc = Scenario(lens, Hq, Hkv, kvo, seed=41, extra_blocks=10, max_blocks=max(-(-L // 16) for L in lens) + 1)
    used = set(sc.block_table[b, i] for b in range(sc.B) for i in range(-(-lens[b] // 16)))
    free = [i for i in range(sc.num_blocks) if i not in used]
    table_np = sc.block_table.copy()
    slots_np = []
    for b, L in enumerate(lens):
        if L % 16 == 0:
            table_np[b, L // 16] = free.pop()
        slots_np.append(int(table_np[b, L // 16]) * 16 + L % 16)
    table = torch.from_numpy(table_np).to(cuda)
    slots = torch.tensor(slots_np, dtype=torch.int32, device=cuda)
    lens1 = torch.tensor([L + 1 for L in lens], dtype=torch.int32, device=cuda)
    pool0 = torch.from_numpy(sc.pool).to(cuda)
    a = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), sc.num_blocks, device=cuda, pool=pool0.clone())
    b_ = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), sc.num_blocks, device=cuda, pool=pool0.clone())
    g = torch.Generator(device=cuda).manual_seed(6)
    B = len(lens)
    k = torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16)
    q = torch.randn((B, Hq, 128), device=cuda, generator=g).to(torch.bfloat16)
    for pps in (None, 5):
        out_a = decode_step(a, k, v, slots, q, table, lens1, out_dtype=torch.float32, pages_per_split=pps,
                            fused_append=True)
        out_b = decode_step(b_, k, v, slots, q, table, lens1, out_dtype=torch.float32, pages_per_split=pps)
        torch.cuda.synchronize()
        assert torch.equal(a.pool, b_.pool)
        assert torch.equal(out_a, out_b)
    from paper_2605_29639_b200 import ops
    nws = ops.workspace_bytes(B, Hq, Hkv, -(-table.shape[1] // 5))
    ws_a = torch.zeros(nws, dtype=torch.uint8, device=cuda)
    ws_b = torch.zeros(nws, dtype=torch.uint8, device=cuda)
    oa = torch.empty((B, Hq, 128), dtype=torch.float32, device=cuda)
    ob = torch.empty((B, Hq, 128), dtype=torch.float32, device=cuda)
    ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga):
        decode_step(a, k, v, slots, q, table, lens1, out=oa, out_dtype=torch.float32, pages_per_split=5,
                    workspace=ws_a, fused_append=True)
    with torch.cuda.graph(gb):
        decode_step(b_, k, v, slots, q, table, lens1, out=ob, out_dtype=torch.float32, pages_per_split=5,
                    workspace=ws_b)
    for _ in range(3):
        k.copy_(torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16))
        v.copy_(torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16))
        ga.replay()
        gb.replay()
        torch.cuda.synchronize()
        assert torch.equal(a.pool, b_.pool)
        assert torch.equal(oa, ob)
    with pytest.raises(ValueError):
        decode_step(a, k[:2], v[:2], slots[:2], q, table, lens1, fused_append=True)
