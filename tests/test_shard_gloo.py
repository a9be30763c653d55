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
    res = [q.get(timeout=240) for _ in range(world)]
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
