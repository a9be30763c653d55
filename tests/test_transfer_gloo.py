"""§8f-2: prefill->decode transfer of quantized pages (page format on the
wire, 51.6 % of bf16 bytes), gloo world_size 2 on CPU.  The decode worker's
pages must be bit-identical to the prefill worker's, landing in whatever
blocks its own allocator hands out."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def host_export(cache, block_ids):
    """Test-side page copy for CPU pools (the product path is kvq_gather_blocks)."""
    return cache.pool.index_select(0, torch.as_tensor([int(b) for b in block_ids], dtype=torch.long))


def host_import(cache, block_ids, pages):
    cache.pool.index_copy_(0, torch.as_tensor([int(b) for b in block_ids], dtype=torch.long), pages)


def _worker(rank, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import oracle as O
    from kvq_testutil import bf16_bits, make_kv
    from paper_2605_29639_b200 import BlockAllocator, KVCacheSpec, PagedKVCache
    from paper_2605_29639_b200.transfer import recv_sequence, send_sequence, wire_bytes_per_token
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    Hkv, L = 4, 181
    spec = KVCacheSpec(Hkv, kv_dtype="fp8_e4m3")
    k, v = make_kv(L, Hkv, 3, kind="k"), make_kv(L, Hkv, 4, kind="v")
    if rank == 0:                                   # prefill worker
        alloc = BlockAllocator(32)
        cache = PagedKVCache(spec, 32, device="cpu")
        alloc.allocate("warmup"); alloc.append_slots("warmup", 40)   # shifts block ids
        alloc.allocate("req")
        slots = np.asarray(alloc.append_slots("req", L), dtype=np.int32)
        pool = cache.pool.numpy()
        O.quant_append(bf16_bits(k), bf16_bits(v), slots, O.FP8_E4M3, pool)
        sent = send_sequence(cache, alloc, "req", 1, export=host_export)
        q.put((rank, sent, sent == -(-L // 16) * Hkv * 4224, wire_bytes_per_token(Hkv) * 2 == Hkv * 264 * 2))
    else:                                           # decode worker
        alloc = BlockAllocator(20)
        cache = PagedKVCache(spec, 20, device="cpu")
        alloc.allocate("other"); alloc.append_slots("other", 5)
        blocks = recv_sequence(cache, alloc, "req", 0, import_=host_import)
        # expected: the same rows quantized on the CPU into this worker's block ids
        exp = np.zeros((20, Hkv, 4224), np.uint8)
        tok = np.arange(L)
        slots = np.asarray([blocks[t // 16] * 16 + t % 16 for t in tok], dtype=np.int32)
        O.quant_append(bf16_bits(k), bf16_bits(v), slots, O.FP8_E4M3, exp)
        got = cache.pool.numpy()
        ok = np.array_equal(got[blocks], exp[blocks]) and alloc.seq_len("req") == L
        alloc.check_invariants()
        q.put((rank, len(blocks), bool(ok), True))
    dist.destroy_process_group()


def test_send_recv_sequence_bit_exact():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res[0][2] and res[0][3], res
    assert res[1][1] == 12 and res[1][2], res
