"""Per-CTA timeline of one K2 launch (debug build with -DKVQ_TIMELINE, which
records each CTA's %globaltimer start / end and SM id).  Prints the launch
span, how long the grid takes to fill the GPU, how long the last wave drains,
and the active-CTA profile, for one of tools/ab_decode.py's shapes.

    nvcc ... -DKVQ_TIMELINE -o tools/ab/libkvq_tl.so paper_2605_29639_b200/csrc/*.cu
    python tools/timeline.py c2 tools/ab/libkvq_tl.so
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ab_decode import SHAPES  # noqa: E402


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    B, Hq, Hkv, ctx, kvd = SHAPES[cfg]
    lens = (np.random.default_rng(3).integers(512, 8193, size=B) if ctx == "ragged"
            else np.full(B, ctx)).astype(np.int64) + 1
    nblk = -(-lens // 16)
    NB, mb = int(nblk.sum()), int(nblk.max())
    dev = torch.device("cuda:0")
    pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
    if kvd == 1:
        pool[..., :4096] &= 0xF7
    pool[..., 4096:] = torch.full((NB, Hkv, 32), 0.02, device=dev).view(torch.uint8).view(NB, Hkv, 128)
    perm = np.random.default_rng(7).permutation(NB).astype(np.int32)
    table = np.zeros((B, mb), np.int32)
    pos = 0
    for b in range(B):
        table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
        pos += nblk[b]
    table = torch.from_numpy(table).to(dev)
    seq = torch.from_numpy(lens.astype(np.int32)).to(dev)
    q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
    out = torch.empty((Hq, B, 128), dtype=torch.bfloat16, device=dev)
    L = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.kvq_decode_pages_per_split.restype = i32
    L.kvq_decode_pages_per_split.argtypes = [i32, i32, i64, i32]
    L.kvq_decode_workspace_bytes.restype = ctypes.c_size_t
    L.kvq_decode_workspace_bytes.argtypes = [i32] * 4
    L.kvq_decode_attn.argtypes = [vp, i64, vp, i64, vp, i32, vp, i32, i32, i32, i32, ctypes.c_float, i32,
                                  vp, ctypes.c_size_t, vp, i32, i32, vp]
    L.kvq_debug_timeline.argtypes = [vp, ctypes.c_size_t]
    import os
    pps = int(os.environ.get("PPS", 0)) or L.kvq_decode_pages_per_split(B, Hkv, NB, mb)
    ns_max = -(-mb // pps)
    ws = torch.zeros(L.kvq_decode_workspace_bytes(B, Hq, Hkv, ns_max), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream

    def launch():
        rc = L.kvq_decode_attn(q.data_ptr(), Hq * 128, pool.data_ptr(), NB, table.data_ptr(), mb, seq.data_ptr(),
                               B, Hq, Hkv, kvd, 1.0 / 128 ** 0.5, pps, ws.data_ptr(), ws.numel(),
                               out.data_ptr(), 0, 1, stream)
        assert rc == 0, rc

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    launch()
    torch.cuda.synchronize()
    n = ns_max * Hkv * B
    buf = np.zeros((1 << 17, 3), np.uint64)
    assert L.kvq_debug_timeline(buf.ctypes.data, buf.nbytes) == 0
    tl = buf[:n].astype(np.int64)
    # keep the CTAs that had work (split < nsplit of their sequence)
    idx = np.arange(n)
    split, rest = idx % ns_max, idx // ns_max
    b = rest // Hkv
    nsplit = np.maximum(1, -(-nblk[b] // pps))
    work = split < nsplit
    pages = np.minimum(nblk[b], (split + 1) * pps) - split * pps
    t0 = tl[work, 0]
    t1 = tl[work, 1]
    base = t0.min()
    s, e = (t0 - base) / 1e3, (t1 - base) / 1e3
    span = e.max()
    grid = np.arange(0, span + 1, 1.0)
    active = np.array([((s <= t) & (e > t)).sum() for t in grid])
    slots = int(active.max())
    fill = grid[np.argmax(active >= 0.95 * slots)]
    drain_start = grid[len(active) - 1 - np.argmax(active[::-1] >= 0.95 * slots)]
    dur = e - s
    pw = pages[work]
    print(f"{cfg}: pps={pps} CTAs with work={work.sum()} (grid {n}); span {span:.1f} us; "
          f"max concurrent {slots}; 95% filled after {fill:.1f} us; drops below 95% at {drain_start:.1f} us "
          f"(tail {span - drain_start:.1f} us)")
    full = pw == pw.max()
    print(f"  CTA duration: full-size ({pw.max()} pages) median {np.median(dur[full]):.2f} us, "
          f"p10 {np.percentile(dur[full], 10):.2f}, p90 {np.percentile(dur[full], 90):.2f}; "
          f"per page {np.median(dur[full]) / pw.max():.3f} us")
    first = s.argsort()[:200]
    print(f"  first 200 CTAs start within {s[first].max():.2f} us; their median duration {np.median(dur[first]):.2f} us")
    last = e.argsort()[-50:]
    print(f"  last 50 CTAs: start {np.median(s[last]):.1f} us median, pages median {np.median(pw[last]):.0f}, "
          f"duration median {np.median(dur[last]):.2f} us")
    step = max(1, len(grid) // 24)
    print("  active CTAs every %d us:" % step, " ".join(str(int(a)) for a in active[::step]))
    sm = tl[work, 2]
    print(f"  SMs used {len(np.unique(sm))}")


if __name__ == "__main__":
    main()
