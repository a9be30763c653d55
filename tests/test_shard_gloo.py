"""KV-head sharding on CPU with the gloo backend, world_size 2 and 4: the
sharded output (each rank attends over its own KV heads' pages, then one
all-gather of head-major outputs) equals the unsharded result bit for bit.
The local op here is the CPU oracle -- a test-only stand-in for the CUDA
kernel (the product path has no CPU fallback)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_29639_b200.shard import ShardedDecodeAttention, head_partition


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import oracle as O
    from kvq_testutil import Scenario, bf16_bits
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Hq, Hkv = 32, 8
    sc = Scenario([70, 33, 150], Hq, Hkv, O.INT8, seed=4)   # identical on every rank (seeded)
    shard = ShardedDecodeAttention(Hq, Hkv)
    kv = slice(shard.kv_lo, shard.kv_hi)
    pool_local = np.ascontiguousarray(sc.pool[:, kv])       # this rank's heads only

    def local_attention(q_loc):
        o = O.decode_attn(bf16_bits(q_loc), pool_local, sc.block_table, sc.seq_lens,
                          shard.kv_hi - shard.kv_lo, O.INT8)
        return torch.from_numpy(o).transpose(0, 1).contiguous()   # head-major [Hq/P, B, d]

    shard.local_attention = local_attention
    out = shard(sc.q)                                        # [Hq, B, d]
    ref = torch.from_numpy(sc.oracle_out()).transpose(0, 1)
    result_q.put((rank, bool(torch.equal(out, ref)), tuple(out.shape)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(shape == (32, 3, 128) for _, _, shape in res)


def test_head_partition():
    assert head_partition(32, 8, 4, 1) == ((2, 4), (8, 16))
    assert head_partition(64, 8, 8, 7) == ((7, 8), (56, 64))
    with pytest.raises(ValueError):
        head_partition(64, 4, 8, 0)        # C4 needs the 2-D (head x batch) split
    with pytest.raises(ValueError):
        head_partition(30, 8, 2, 0)


def _worker_2d(rank, world, port, result_q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import oracle as O
    from kvq_testutil import Scenario, bf16_bits
    from paper_2605_29639_b200.shard import Sharded2DDecodeAttention
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Hq, Hkv = 16, 2          # Hkv < world: 2 head groups x (world/2) batch parts
    lens = [300, 20, 170, 64, 1, 90, 129]
    sc = Scenario(lens, Hq, Hkv, O.INT8, seed=8)
    shard = Sharded2DDecodeAttention(Hq, Hkv, lens)
    pl = shard.plan
    kv = slice(*pl.kv_range)
    pool_local = np.ascontiguousarray(sc.pool[:, kv])
    table_local = sc.block_table[pl.seqs]
    lens_local = sc.seq_lens[pl.seqs]

    def local_attention(q_loc):
        o = O.decode_attn(bf16_bits(q_loc), pool_local, table_local, lens_local,
                          pl.kv_range[1] - pl.kv_range[0], O.INT8)
        return torch.from_numpy(o).transpose(0, 1).contiguous()

    shard.local_attention = local_attention
    out = shard(sc.q)
    ref = torch.from_numpy(sc.oracle_out()).transpose(0, 1)
    result_q.put((rank, bool(torch.equal(out, ref)), pl.h_split, pl.b_split, list(map(int, pl.seqs))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_2d_head_batch_partition(world):
    """C4's case (Hkv < P): KV-head groups x LPT token-balanced batch parts."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, *_ in res), res
    assert all(h == 2 and b == world // 2 for _, _, h, b, _ in res)


def test_lpt_balance():
    from paper_2605_29639_b200.shard import lpt_assign, plan_shards
    parts = lpt_assign([131072] * 64, 2)
    assert [len(p) for p in parts] == [32, 32]
    lens = [8000, 500, 7000, 600, 6000, 700, 3000, 2500]
    parts = lpt_assign(lens, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(lens)))
    loads = [sum(lens[i] for i in p) for p in parts]
    lower = max(max(lens), sum(lens) / 3)
    assert max(loads) <= 4 / 3 * lower          # Graham's LPT bound
    pl = plan_shards(64, 4, 8, 5, [131072] * 64)
    assert (pl.h_split, pl.b_split, pl.kv_range, pl.q_range, len(pl.seqs)) == (4, 2, (2, 3), (32, 48), 32)
