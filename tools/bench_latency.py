"""Small-batch decode latency (interactive serving): GPU time of one K2 launch
through the public op, replayed from a CUDA graph (no host launch cost) --
back to back (L2-warm where the KV fits in L2) and after a 256 MB memset that
evicts L2 (cold: the serving case, one layer's KV is not in L2) -- for
B = 1..32 sequences of the Llama-3-8B attention shape (Hq = 32, Hkv = 8,
INT8), plus C1.  One JSON line per shape.

    python tools/bench_latency.py
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

SHAPES = [(1, 2048), (1, 8192), (1, 32768), (1, 131072), (4, 8192), (8, 2048), (32, 2048), (32, 8192)]


def main():
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, ops, paged_decode_attention
    dev = torch.device("cuda:0")
    Hq, Hkv = 32, 8
    for B, ctx in SHAPES:
        L = ctx + 1
        npg = -(-L // 16)
        NB = B * npg
        pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
        pool[..., 4096:] = torch.full((NB, Hkv, 32), 0.02, device=dev).view(torch.uint8).view(NB, Hkv, 128)
        cache = PagedKVCache(KVCacheSpec(Hkv), NB, device=dev, pool=pool)
        table = torch.from_numpy(np.random.default_rng(B).permutation(NB).astype(np.int32).reshape(B, npg)).to(dev)
        lens = torch.full((B,), L, dtype=torch.int32, device=dev)
        q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
        out = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev)
        pps = ops.pages_per_split(B, Hkv, NB, npg)
        ws = torch.zeros(ops.workspace_bytes(B, Hq, Hkv, -(-npg // pps)), dtype=torch.uint8, device=dev)

        def run():
            paged_decode_attention(q, cache, table, lens, out=out, pages_per_split=pps, workspace=ws)

        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                run()
        g.replay()
        torch.cuda.synchronize()
        times = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 20 * 1e3)
        us = sorted(times)[len(times) // 2]
        # cold L2: a 256 MB memset, then one launch between its own event nodes
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            ev[0].record()
            run()
            ev[1].record()
        cold = []
        for _ in range(15):
            flush.zero_()
            g1.replay()
            torch.cuda.synchronize()
            cold.append(ev[0].elapsed_time(ev[1]) * 1e3)
        cus = sorted(cold)[len(cold) // 2]
        del flush
        byt = B * L * Hkv * 264 + B * Hq * 512 + NB * 4
        print(json.dumps({"B": B, "ctx": ctx, "pages_per_split": pps, "splits": -(-npg // pps), "k2_us": us,
                          "gbs": byt / (us * 1e-6) / 1e9, "tokens_per_s": B / (us * 1e-6),
                          "k2_us_cold_l2": cus, "gbs_cold_l2": byt / (cus * 1e-6) / 1e9}), flush=True)
        del pool, cache


if __name__ == "__main__":
    main()
