#!/usr/bin/env python3
"""Where does a decode step's time go?  Times, on one GPU, graph replays of
K1 alone, K2 alone, [K1, K2] in one graph, and the bench's two-graph step.

    python tools/step_breakdown.py [c1|c2|c3|c4] [--iters 200]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, quantize_append  # noqa: E402
from paper_2605_29639_b200.session import DecodeSession  # noqa: E402


def timed(fn, iters):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(0, 0.002) as cs:
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
    c = cs.summary()
    return a.elapsed_time(b) / iters * 1e3, c["sm_mhz"], ",".join(c["reasons"])  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    B, Hq, Hkv = cfg["B"], cfg["Hq"], cfg["Hkv"]
    lens = bench.ctx_lens(cfg)
    L1 = lens + 1
    nblk = np.ceil(L1 / 16).astype(np.int64)
    nb = int(nblk.sum())
    rng = np.random.default_rng(7)
    perm = rng.permutation(nb).astype(np.int32)
    table = np.zeros((B, int(nblk.max())), dtype=np.int32)
    pos = 0
    for b in range(B):
        table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
        pos += nblk[b]
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=cfg["kv"]), nb, device=dev)
    # Random content through K1 (whole pages).
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    allslots = torch.arange(nb * 16, dtype=torch.int32, device=dev)
    for s0 in range(0, nb * 16, 1 << 16):
        sl = allslots[s0: s0 + (1 << 16)]
        kv = torch.randn((2, sl.numel(), Hkv, 128), device=dev, generator=gen).to(torch.bfloat16)
        quantize_append(cache, kv[0], kv[1], sl)
    table_d = torch.from_numpy(table).to(dev)
    sess = DecodeSession(cache, table_d, B, Hq, total_pages=nb, head_major=True)
    buf = sess.device_buffers(0)
    buf["q"].normal_(generator=gen)
    buf["k"].normal_(generator=gen)
    buf["v"].normal_(generator=gen)
    buf["slots"].copy_(torch.from_numpy((table[np.arange(B), lens // 16].astype(np.int64) * 16
                                         + lens % 16).astype(np.int32)))
    buf["lens"].copy_(torch.from_numpy(L1.astype(np.int32)))
    sess._kernels(buf)
    torch.cuda.synchronize()
    g1, g2 = sess.capture()
    g12 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g12):
        sess._kernels(buf)
    # Unrolled graphs (U copies per replay): GPU time without per-replay CPU overhead.
    U = 20
    gu = {}
    for name, fn in (("K1", lambda: quantize_append(cache, buf["k"], buf["v"], buf["slots"])),
                     ("K2", lambda: sess._kernels(buf, k1=False)),
                     ("K1+K2", lambda: sess._kernels(buf))):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(U):
                fn()
        gu[name] = g
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def bench_style():
        g1.replay()
        ev[0].record()
        g2.replay()
        ev[1].record()

    res = {"K1": timed(g1.replay, args.iters), "K2": timed(g2.replay, args.iters),
           "K1+K2 one graph": timed(g12.replay, args.iters),
           "bench two graphs + events": timed(bench_style, args.iters)}
    for name, g in gu.items():
        t = timed(g.replay, max(1, args.iters // U))
        res[f"{name} x{U} unrolled"] = (t[0] / U,) + t[1:]
    # End to end through DecodeSession.submit (pinned host buffers), eager vs graphs.
    q_h = buf["q"].cpu().pin_memory()
    k_h, v_h = buf["k"].cpu().pin_memory(), buf["v"].cpu().pin_memory()
    s_h, l_h = buf["slots"].cpu().pin_memory(), buf["lens"].cpu().pin_memory()
    o_h = torch.empty((Hq, B, 128), dtype=torch.bfloat16, pin_memory=True)
    for graphs in (False, True):
        se = DecodeSession(cache, table_d, B, Hq, total_pages=nb, head_major=True, graphs=graphs)

        def e2e():
            se.submit(q_h, k_h, v_h, s_h, l_h, o_h)
        for _ in range(5):
            e2e()
        se.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(se.h2d)
        n = args.iters
        for _ in range(n):
            e2e()
        e1.record(se.d2h)
        se.synchronize()
        res[f"e2e graphs={graphs}"] = (e0.elapsed_time(e1) / n * 1e3, None, "")
    print(args.config, f"pps={sess.pps}", " | ".join(f"{k} {v[0]:.2f} us @{v[1]} {v[2]}" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
