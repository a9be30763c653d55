"""Library baseline: flashinfer's paged FP8-E4M3 decode attention on the C3
workload (Qwen2.5-72B shape: Hq = 64, Hkv = 8, d = 128, B = 128, ctx 32K,
page 16) or the C2 shape (B = 256, ragged ctx), next to libkvq's K2 (FP8 and
INT8) on the same shape.  flashinfer reads 256 B per
(token, kv head) (codes only, one scale per tensor); libkvq reads 264 B (codes
+ per-token scales).  Both timed as back-to-back launches with CUDA events.

    python tools/bench_flashinfer.py [--config c3|c2] [--steps K] [--tensor-cores]
"""
import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def timed(fn, steps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


WORKLOADS = {
    "c3": ("C3: B=128, ctx 32K, Hq=64, Hkv=8", 128, 64, 8, None),
    "c2": ("C2 shape: B=256, ragged ctx U{512..8192} (seed 3), Hq=32, Hkv=8", 256, 32, 8, (512, 8192)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--tensor-cores", action="store_true")
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    import flashinfer
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, ops, paged_decode_attention
    dev = torch.device("cuda:0")
    name, B, Hq, Hkv, rag = WORKLOADS[args.config]
    if rag is None:
        lens_np = np.full(B, 32769, dtype=np.int64)
    else:
        lens_np = np.random.default_rng(3).integers(rag[0], rag[1] + 1, size=B).astype(np.int64) + 1
    npgs = -(-lens_np // 16)
    NB = int(npgs.sum())
    mb = int(npgs.max())
    perm = torch.from_numpy(np.random.default_rng(7).permutation(NB).astype(np.int32)).to(dev)
    q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
    lines = []
    ctx_sum = int(lens_np.sum())

    # ---- flashinfer: paged KV [NB, 2, 16, Hkv, 128] fp8 (NHD), random block ids
    kv = (torch.randn((NB, 2, 16, Hkv, 128), device=dev) * 40).to(torch.float8_e4m3fn)
    indptr = torch.from_numpy(np.concatenate([[0], np.cumsum(npgs)]).astype(np.int32)).to(dev)
    last = torch.from_numpy((lens_np - (npgs - 1) * 16).astype(np.int32)).to(dev)
    ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=args.tensor_cores)
    w.plan(indptr, perm, last, Hq, Hkv, 128, 16, q_data_type=torch.bfloat16, kv_data_type=torch.float8_e4m3fn,
           sm_scale=1.0 / math.sqrt(128))
    out = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev)
    t_fi = timed(lambda: w.run(q, kv, out=out, k_scale=0.0125, v_scale=0.03125), args.steps)
    fi_bytes = ctx_sum * Hkv * 256 + B * Hq * 512 + NB * 4
    lines.append({"impl": "flashinfer " + flashinfer.__version__ + (" (tensor cores)" if args.tensor_cores else ""),
                  "workload": name + ", FP8-E4M3 KV, page 16", "ms": t_fi,
                  "gbs": fi_bytes / (t_fi * 1e-3) / 1e9, "tokens_per_s": B / (t_fi * 1e-3)})
    del kv, w, ws
    torch.cuda.empty_cache()

    # ---- libkvq K2 on the same shape: FP8 (same codes width) and INT8
    table_np = np.zeros((B, mb), np.int32)
    pos, pn = 0, perm.cpu().numpy()
    for b in range(B):
        table_np[b, : npgs[b]] = pn[pos: pos + npgs[b]]
        pos += npgs[b]
    table = torch.from_numpy(table_np).to(dev)
    lens = torch.from_numpy(lens_np.astype(np.int32)).to(dev)
    pps = ops.pages_per_split(B, Hkv, NB, mb)
    o2 = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev)
    k_bytes = ctx_sum * Hkv * 264 + B * Hq * 512 + NB * 4
    for kvd in ("fp8_e4m3", "int8"):
        pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
        pool[..., :4096] &= 0xF7
        pool[..., 4096:] = torch.full((NB, Hkv, 32), 0.02, device=dev).view(torch.uint8).view(NB, Hkv, 128)
        cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kvd), NB, device=dev, pool=pool)
        t_k = timed(lambda: paged_decode_attention(q, cache, table, lens, out=o2, pages_per_split=pps), args.steps)
        lines.append({"impl": "libkvq K2", "workload": name + f", {kvd} KV (+ per-token scales)", "ms": t_k,
                      "gbs": k_bytes / (t_k * 1e-3) / 1e9, "tokens_per_s": B / (t_k * 1e-3),
                      "speedup_vs_flashinfer": t_fi / t_k})
        del pool, cache
    for l in lines:
        print(json.dumps(l), flush=True)


if __name__ == "__main__":
    main()
