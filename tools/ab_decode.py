"""A/B timing of kvq_decode_attn across libkvq builds (any ABI version that
exports kvq_decode_attn / kvq_decode_pages_per_split / workspace_bytes).

    python tools/ab_decode.py CONFIG lib1.so [lib2.so ...]

CONFIG is one of c2, c3, c4 (bench.py shapes).  Pages are random codes with
fixed positive scales (timing only); block ids are a random permutation.
Each lib is timed in alternation (5 rounds x 20 launches, CUDA events), so
box-level drift affects every build alike.  GRAPH=1 replays the 20 launches
from one CUDA graph (GPU time without host launch cost); PPS=n forces the
split size.
"""
import ctypes
import os
import sys

import numpy as np
import torch

SHAPES = {"r8": (8, 32, 8, "ragged", 0), "r32": (32, 32, 8, "ragged", 0), "r64": (64, 32, 8, "ragged", 0), "r64f_p8": (64, 8, 1, "ragged", 1), "c2_p8": (256, 4, 1, "ragged", 0), "c2_p4": (256, 8, 2, "ragged", 0), "c2_p2": (256, 16, 4, "ragged", 0), "c3_p8": (128, 8, 1, 32768, 1), "c4_p8": (32, 16, 1, 131072, 0), "g16_b32_8k": (32, 64, 4, 8192, 0), "g16_b4_32k": (4, 64, 4, 32768, 0), "c3_p2": (128, 32, 4, 32768, 1), "c3_p4": (128, 16, 2, 32768, 1), "g16_b16_32k": (16, 64, 4, 32768, 0), "g16_b8_8k": (8, 64, 4, 8192, 0), "c4_p4": (64, 32, 2, 131072, 0), "b1_8k": (1, 32, 8, 8192, 0), "c2h": (128, 32, 8, "ragged", 0), "c2d": (512, 32, 8, "ragged", 0), "b32_8k": (32, 32, 8, 8192, 0), "b1_128k": (1, 32, 8, 131072, 0), "b64_8k": (64, 32, 8, 8192, 0), "b1_32k": (1, 32, 8, 32768, 0), "b4_8k": (4, 32, 8, 8192, 0), "b32_2k": (32, 32, 8, 2048, 0), "tiny": (1, 32, 8, 15, 0), "b1_2k": (1, 32, 8, 2048, 0), "b8_512": (8, 32, 8, 512, 0), "c2f": (256, 32, 8, "ragged", 1), "c3i": (128, 64, 8, 32768, 0), "c2e": (256, 32, 8, 4352, 0), "c1": (8, 32, 8, 2048, 0), "c2": (256, 32, 8, "ragged", 0), "c3": (128, 64, 8, 32768, 1), "c4": (64, 64, 4, 131072, 0)}


def main():
    cfg, libs = sys.argv[1], sys.argv[2:]
    B, Hq, Hkv, ctx, kvd = SHAPES[cfg]
    lens = (np.random.default_rng(3).integers(512, 8193, size=B) if ctx == "ragged"
            else np.full(B, ctx)).astype(np.int64) + 1
    nblk = -(-lens // 16)
    NB, mb = int(nblk.sum()), int(nblk.max())
    dev = torch.device("cuda:0")
    pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
    if kvd == 1:
        pool[..., :4096] &= 0xF7  # no NaN E4M3 codes
    sc = torch.full((NB, Hkv, 32), 0.02, dtype=torch.float32, device=dev)
    pool[..., 4096:] = sc.view(torch.uint8).view(NB, Hkv, 128)
    perm = (np.random.default_rng(7).permutation(NB) if os.environ.get("PERM", "1") != "0"
            else np.arange(NB)).astype(np.int32)  # PERM=0: contiguous block ids
    table = np.zeros((B, mb), np.int32)
    pos = 0
    for b in range(B):
        table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
        pos += nblk[b]
    table = torch.from_numpy(table).to(dev)
    seq = torch.from_numpy(lens.astype(np.int32)).to(dev)
    q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
    out = torch.empty((Hq, B, 128), dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    runs = []
    for path in libs:
        L = ctypes.CDLL(path)
        L.kvq_decode_pages_per_split.restype = ctypes.c_int32
        L.kvq_decode_pages_per_split.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32]
        if hasattr(L, "kvq_decode_pages_per_split_rows"):
            L.kvq_decode_pages_per_split_rows.restype = ctypes.c_int32
            L.kvq_decode_pages_per_split_rows.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_int64, ctypes.c_int32]
        L.kvq_decode_workspace_bytes.restype = ctypes.c_size_t
        L.kvq_decode_workspace_bytes.argtypes = [ctypes.c_int32] * 4
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.kvq_decode_attn.argtypes = [vp, i64, vp, i64, vp, i32, vp, i32, i32, i32, i32, ctypes.c_float, i32,
                                      vp, ctypes.c_size_t, vp, i32, i32, vp]
        pps = int(os.environ.get("PPS", 0)) or (L.kvq_decode_pages_per_split_rows(B, Hkv, Hq // Hkv, NB, mb) if hasattr(L, "kvq_decode_pages_per_split_rows") else L.kvq_decode_pages_per_split(B, Hkv, NB, mb))
        wsb = L.kvq_decode_workspace_bytes(B, Hq, Hkv, -(-mb // pps) * int(os.environ.get("WSX", 1)))
        ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)

        def launch(L=L, pps=pps, ws=ws, wsb=wsb):
            st = L.kvq_decode_attn(q.data_ptr(), q.stride(0), pool.data_ptr(), NB, table.data_ptr(), mb,
                                   seq.data_ptr(), B, Hq, Hkv, kvd, 0.0884, pps, ws.data_ptr(), wsb,
                                   out.data_ptr(), 0, 1, torch.cuda.current_stream().cuda_stream)
            assert st == 0, st
        launch()
        runs.append((path, launch, []))
    torch.cuda.synchronize()
    if os.environ.get("FLUSH"):  # cold L2: one launch between its own event nodes, a 256 MB memset before each
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(5):
            for path, launch, times in runs:
                ev = (torch.cuda.Event(enable_timing=True, external=True),
                      torch.cuda.Event(enable_timing=True, external=True))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    ev[0].record()
                    launch()
                    ev[1].record()
                for _ in range(6):
                    flush.zero_()
                    g.replay()
                    torch.cuda.synchronize()
                    times.append(ev[0].elapsed_time(ev[1]) / 20)  # printed x20 below, like the other modes
        byt = int(lens.sum()) * Hkv * 264 + B * Hq * 512 + int(nblk.sum()) * 4
        for path, _, times in runs:
            t = min(times)
            med = sorted(times)[len(times) // 2]
            print(f"{cfg} pps={pps} {path}: cold-L2 min {t * 20e3:.1f} us  median {med * 20e3:.1f} us  "
                  f"{byt / (med * 20) / 1e6:.0f} GB/s")
        return
    if os.environ.get("GRAPH"):  # time 20 launches captured in one CUDA graph: GPU time, no host cost
        graphed = []
        for path, launch, times in runs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    launch()
            graphed.append((path, (lambda g=g: g.replay()), times))
        runs = graphed
    for _ in range(5):
        for path, launch, times in runs:
            reps = 1 if os.environ.get("GRAPH") else 20
            for _ in range(3):
                launch()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                launch()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 20)  # 20 launches either way
    byt = int(lens.sum()) * Hkv * 264 + B * Hq * 512 + int(nblk.sum()) * 4
    for path, _, times in runs:
        t = min(times)
        print(f"{cfg} pps={pps} {path}: min {t * 1e3:.1f} us  median {sorted(times)[2] * 1e3:.1f} us  "
              f"{byt / t / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
