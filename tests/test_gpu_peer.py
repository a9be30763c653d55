"""The all-gather fused into K2 (kvq_decode_attn_peer), end to end on one GPU.

Two (or four) processes play the ranks on cuda:0 and map each other's symmetric
buffers through CUDA IPC -- the same peer pointers, stores, release/acquire
flags and slot protocol that NVLink peers use across GPUs; only the wire
differs.  Each rank attends its shard (KV-head split, or the 2-D split's batch
part with the LPT seq_map) and its K2 writes every finished row into every
rank's global output.  Checked, for several uses of two slots, eager and
CUDA-graph replays and the DecodeSession pipeline: every rank's global output
equals the unsharded kernel's output bit for bit (same split geometry), and no
protocol spin timed out."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, result_q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    from kvq_testutil import Scenario, make_q
    from paper_2605_29639_b200 import (KVCacheSpec, PagedKVCache, paged_decode_attention,
                                       paged_decode_attention_gathered)
    from paper_2605_29639_b200.session import DecodeSession
    from paper_2605_29639_b200.shard import PeerOutput, plan_shards

    checks = {}
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        kvo = O.INT8
        if mode == "head":      # KV-head tensor parallelism (Hkv % P == 0)
            Hq, Hkv, lens = 32, 8, [70, 33, 150, 0, 400, 17]
        elif mode == "batch":   # one KV head, batch halves balanced by LPT (seq_map)
            Hq, Hkv, lens = 8, 1, [70, 33, 150, 0, 400, 17, 260]
        elif mode == "2d":      # 2-D at world 4: 2 KV-head groups x 2 LPT batch parts (the C4-at-8 shape)
            Hq, Hkv, lens = 16, 2, [70, 33, 150, 0, 400, 17, 260, 90]
        elif mode == "c3p8":    # C3 at P = 8: Qwen2.5-72B heads (64 q / 8 kv), FP8, one kv head per rank
            Hq, Hkv, kvo = 64, 8, O.FP8_E4M3
            lens = [int(x) for x in np.random.default_rng(31).integers(1, 900, size=12)]
        else:                   # c4p8 -- C4 at P = 8: Qwen3-235B heads (64 q / 4 kv, g = 16), INT8,
            Hq, Hkv = 64, 4     # 4 kv-head groups x 2 LPT batch parts
            lens = [int(x) for x in np.random.default_rng(41).integers(1, 1500, size=11)]
        sc = Scenario(lens, Hq, Hkv, kvo, seed=9)             # identical bytes on every rank
        kvd = "fp8_e4m3" if kvo == O.FP8_E4M3 else "int8"
        B = sc.B
        pps = 4
        plan = plan_shards(Hq, Hkv, world, rank, sc.seq_lens)
        (k0, k1), (q0, q1) = plan.kv_range, plan.q_range
        checks["plan"] = (plan.h_split, plan.b_split)
        seqs = torch.as_tensor(plan.seqs)
        full_cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kvd), sc.num_blocks, device=dev,
                                  pool=torch.from_numpy(sc.pool).to(dev))
        loc_cache = PagedKVCache(KVCacheSpec(k1 - k0, kv_dtype=kvd), sc.num_blocks, device=dev,
                                 pool=torch.from_numpy(np.ascontiguousarray(sc.pool[:, k0:k1])).to(dev))
        table_full = torch.from_numpy(sc.block_table).to(dev)
        lens_full = torch.from_numpy(sc.seq_lens).to(dev)
        table_loc = table_full.index_select(0, seqs.to(dev)).contiguous()
        lens_loc = lens_full.index_select(0, seqs.to(dev)).contiguous()
        qs = [make_q(B, Hq, 100 + s).to(dev) for s in range(6)]
        refs = [paged_decode_attention(q, full_cache, table_full, lens_full, head_major=True,
                                       pages_per_split=pps) for q in qs]   # unsharded [Hq, B, d]
        torch.cuda.synchronize()

        def local_q(q):
            return q.index_select(0, seqs.to(dev))[:, q0:q1].contiguous()

        peer = PeerOutput(plan, Hq, B, Hkv, dev, slots=2)
        # 1) eager: 6 uses over 2 slots (slot reuse goes through the release/free protocol)
        ok = True
        for s, q in enumerate(qs):
            out = paged_decode_attention_gathered(local_q(q), loc_cache, table_loc, lens_loc, peer,
                                                  slot=s % 2, pages_per_split=pps)
            torch.cuda.synchronize()
            ok &= bool(torch.equal(out, refs[s]))
        checks["eager"] = ok
        # 2) CUDA graph of the fused launch, replayed with new q contents
        q_in = local_q(qs[0]).clone()
        ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
        paged_decode_attention_gathered(q_in, loc_cache, table_loc, lens_loc, peer, slot=0,
                                        pages_per_split=pps, workspace=ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            paged_decode_attention_gathered(q_in, loc_cache, table_loc, lens_loc, peer, slot=0,
                                            pages_per_split=pps, workspace=ws)
        ok = True
        for s in (3, 1, 4):
            q_in.copy_(local_q(qs[s]))
            g.replay()
            torch.cuda.synchronize()
            ok &= bool(torch.equal(peer.out(0), refs[s]))
        checks["graph"] = ok
        # 3) the serving pipeline: DecodeSession(peer=...) with double-buffered slots and graphs;
        #    slots = -1 skips the append so every step attends the same cache
        sess = DecodeSession(loc_cache, table_loc, len(plan.seqs), q1 - q0, head_major=True, peer=peer,
                             pages_per_split=pps, graphs=True)
        Bl, Hkl = len(plan.seqs), k1 - k0
        kv_h = torch.zeros((Bl, Hkl, 128), dtype=torch.bfloat16).pin_memory()
        slots_h = torch.full((Bl,), -1, dtype=torch.int32).pin_memory()
        lens_h = lens_loc.cpu().pin_memory()
        outs = []
        for s in range(6):
            o_h = torch.empty((Hq, B, 128), dtype=torch.bfloat16).pin_memory()
            sess.submit(local_q(qs[s]).cpu().pin_memory(), kv_h, kv_h, slots_h, lens_h, o_h)
            outs.append(o_h)
        sess.synchronize()
        checks["session"] = all(torch.equal(o, r.cpu()) for o, r in zip(outs, refs))
        checks["no_timeouts"] = peer.errors() == 0
        peer.close()
        dist.destroy_process_group()
    except Exception as e:  # report, do not hang the parent
        checks["exception"] = f"{type(e).__name__}: {e}"
    result_q.put((rank, checks))


def _fail_worker(rank, world, port, result_q):
    """Rank 1 cannot map its peer: every rank must raise (no rank left in a barrier)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    from paper_2605_29639_b200 import _lib
    from paper_2605_29639_b200.shard import PeerOutput, plan_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    if rank == 1:
        lib = _lib.load()
        lib.kvq_sym_open = lambda handle, ptr: _lib.KVQ_ECUDA   # simulated IPC failure
    try:
        PeerOutput(plan_shards(32, 8, world, rank, [100] * 4), 32, 4, 8, torch.device("cuda:0"))
        result_q.put((rank, "no error"))
    except RuntimeError as e:
        result_q.put((rank, "raised" if "unavailable" in str(e) else str(e)))
    dist.destroy_process_group()


def test_peer_setup_failure_is_collective(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=300) for _ in range(2))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert res == {0: "raised", 1: "raised"}


PLANS = {"head": (2, 1), "batch": (1, 2), "2d": (2, 2), "c3p8": (8, 1), "c4p8": (4, 2)}


@pytest.mark.parametrize("mode,world", [("head", 2), ("batch", 2), ("2d", 4), ("c3p8", 8), ("c4p8", 8)])
def test_fused_peer_gather_ranks_on_one_gpu(cuda, mode, world):
    """world 8 runs the two production P = 8 plans at reduced batch: C3 (one
    kv head per rank) and C4 (4 kv-head groups x 2 LPT batch parts, g = 16)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=600) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        c = res[r]
        assert "exception" not in c, c
        assert c == {"plan": PLANS[mode], "eager": True, "graph": True, "session": True, "no_timeouts": True}, \
            (r, c)
