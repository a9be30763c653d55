"""K1 (quantize-on-append) at the C5 step shape: 4 chunked-prefill sequences
x 2048 tokens in whole pages + 252 decode tokens scattered one per page,
Hkv = 8.  Prints per-launch time and algorithmic GB/s; a handful of launches
so ncu can target it (``-k regex:quant_append -s 5 -c 1``).

    python tools/k1_bench.py [int8|fp8_e4m3] [lib.so ...]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    kv = sys.argv[1] if len(sys.argv) > 1 else "int8"
    libs = sys.argv[2:] or [None]
    import os
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, _lib, ops
    Hkv, prefill, chunk, dec = 8, 4, 2048, 252
    nb = prefill * chunk // 16 + dec + 64
    rng = np.random.default_rng(0)
    perm = rng.permutation(nb).astype(np.int64)
    slots = []
    for i in range(prefill):                      # whole pages, random block per page
        for p in range(chunk // 16):
            blk = perm[i * (chunk // 16) + p]
            slots += [blk * 16 + t for t in range(16)]
    base = prefill * chunk // 16
    slots += [perm[base + j] * 16 + int(rng.integers(0, 16)) for j in range(dec)]
    T = len(slots)
    dev = torch.device("cuda:0")
    sl = torch.tensor(slots, dtype=torch.int32, device=dev)
    k = torch.randn((T, Hkv, 128), device=dev).to(torch.bfloat16)
    v = torch.randn((T, Hkv, 128), device=dev).to(torch.bfloat16)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv), nb, device=dev)
    byt = T * Hkv * (2 * 128 * 2 + 2 * 128 + 8) + 4 * T
    for path in libs:
        if path:
            os.environ["KVQ_LIB_PATH"] = path
            _lib._lib = None
        for _ in range(3):
            ops.quantize_append(cache, k, v, sl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50
        e0.record()
        for _ in range(n):
            ops.quantize_append(cache, k, v, sl)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / n
        # cold L2 (the serving case: the rows come from the QKV projection, the
        # pages were last touched a step ago): a 256 MB memset before each launch
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        cold = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.quantize_append(cache, k, v, sl)
            b.record()
            torch.cuda.synchronize()
            cold.append(a.elapsed_time(b))
        tc = sorted(cold)[len(cold) // 2]
        print(f"K1 {kv} {path or 'in-tree'}: T={T} x {Hkv} heads, {t * 1e3:.2f} us/launch back to back "
              f"({byt / t / 1e6:.0f} GB/s), {tc * 1e3:.2f} us cold-L2 median ({byt / tc / 1e6:.0f} GB/s) "
              f"algorithmic ({byt / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
