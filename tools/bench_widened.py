"""Measurements of the widened rows, one JSON line each.

    python tools/bench_widened.py [--steps K]

* f-4 multi-query decode (speculative scoring / MTP): the C2 workload
  (Llama-3-8B shape, B = 256, ctx U{512..8192}, INT8) with q_len = 1, 2, 4
  query tokens per sequence, causal among them.  K2 time (CUDA events,
  warm), algorithmic bytes (KV + q/out x q_len), fraction of the measured
  HBM peak.  The point: scoring k+1 draft tokens costs about one decode
  step, because the pages are streamed once for all q_len rows.
* f-2 PD transfer, device side: the page export (gather of a sequence's
  blocks into one contiguous buffer) and import (scatter into the receiver's
  blocks) for a 32K-token sequence of the C3 shape (8 KV heads), and the
  wire bytes against bf16.  The NCCL send/recv between GPUs needs two GPUs
  and is not timed here.
* f-3 host tier: offload (device -> pinned host) and promotion (host ->
  device) of whole quantized blocks, GB/s.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def timed(fn, steps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def peak():
    p = REPO / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def multi_query(steps):
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, ops, paged_decode_attention
    dev = torch.device("cuda:0")
    B, Hq, Hkv = 256, 32, 8
    lens = np.random.default_rng(3).integers(512, 8193, size=B).astype(np.int64) + 4
    nblk = -(-lens // 16)
    NB, mb = int(nblk.sum()), int(nblk.max())
    pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
    pool[..., 4096:] = torch.full((NB, Hkv, 32), 0.02, device=dev).view(torch.uint8).view(NB, Hkv, 128)
    cache = PagedKVCache(KVCacheSpec(Hkv), NB, device=dev, pool=pool)
    perm = np.random.default_rng(7).permutation(NB).astype(np.int32)
    table = np.zeros((B, mb), np.int32)
    pos = 0
    for b in range(B):
        table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
        pos += nblk[b]
    table = torch.from_numpy(table).to(dev)
    seq = torch.from_numpy(lens.astype(np.int32)).to(dev)
    pps = ops.pages_per_split(B, Hkv, NB, mb)
    out, base = [], None
    for q_len in (1, 2, 4):
        q = torch.randn((B, q_len, Hq, 128), device=dev).to(torch.bfloat16)
        qq = q[:, 0] if q_len == 1 else q
        o = torch.empty((B, q_len, Hq, 128) if q_len > 1 else (B, Hq, 128), dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: paged_decode_attention(qq, cache, table, seq, out=o, pages_per_split=pps), steps)
        byt = int(lens.sum()) * Hkv * 264 + B * q_len * Hq * 512 + int(nblk.sum()) * 4
        base = base or ms
        out.append({"row": "8f-4 multi-query decode (speculative scoring)", "config": "C2 shape, INT8",
                    "q_len": q_len, "query_rows_per_kv_head": 4 * q_len, "k2_ms": ms,
                    "scored_tokens_per_s": B * q_len / (ms * 1e-3), "achieved_gbs": byt / (ms * 1e-3) / 1e9,
                    "frac": byt / (ms * 1e-3) / 1e9 / peak(), "time_vs_q_len_1": ms / base})
    return out


def transfer(steps):
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache
    from paper_2605_29639_b200.transfer import export_pages, import_pages, wire_bytes_per_token
    dev = torch.device("cuda:0")
    Hkv, tokens = 8, 32768
    nblk = tokens // 16
    NB = 4 * nblk
    src = PagedKVCache(KVCacheSpec(Hkv), NB, device=dev)
    src.pool.random_(0, 256)
    dst = PagedKVCache(KVCacheSpec(Hkv), NB, device=dev)
    rng = np.random.default_rng(0)
    sblocks = rng.permutation(NB)[:nblk].tolist()
    dblocks = rng.permutation(NB)[:nblk].tolist()
    pages = export_pages(src, sblocks)
    # device-side time: block ids already on the device (as a transfer engine holds them)
    sd = torch.as_tensor(sblocks, dtype=torch.int32, device=dev)
    dd = torch.as_tensor(dblocks, dtype=torch.int32, device=dev)
    t_exp = timed(lambda: export_pages(src, sd), steps)
    t_imp = timed(lambda: import_pages(dst, dd, pages), steps)
    # API time with host lists of block ids (host work included)
    t_exp_api = timed(lambda: export_pages(src, sblocks), steps)
    t_imp_api = timed(lambda: import_pages(dst, dblocks, pages), steps)
    import_pages(dst, dblocks, pages)
    torch.cuda.synchronize()
    ok = bool(torch.equal(dst.pool[torch.as_tensor(dblocks, device=dev)], src.pool[torch.as_tensor(sblocks, device=dev)]))
    wire = pages.numel()
    return [{"row": "8f-2 PD transfer (device side)", "config": "C3 shape (8 KV heads), one 32K-token sequence",
             "wire_bytes": wire, "bf16_bytes": tokens * Hkv * 2 * 128 * 2, "wire_vs_bf16": wire / (tokens * Hkv * 512),
             "wire_bytes_per_token": wire_bytes_per_token(Hkv), "export_ms": t_exp, "import_ms": t_imp,
             "export_gbs": 2 * wire / (t_exp * 1e-3) / 1e9, "import_gbs": 2 * wire / (t_imp * 1e-3) / 1e9,
             "export_ms_host_ids": t_exp_api, "import_ms_host_ids": t_imp_api,
             "bit_identical": ok, "note": "GB/s counts read + write (device-resident ids); *_host_ids include "
                                          "building and uploading the id list; the NCCL hop needs 2 GPUs (not timed)"}]


def host_tier(steps):
    dev = torch.device("cuda:0")
    Hkv, nblk = 8, 2048                      # 32K tokens of one layer, 69 MB
    dev_pages = torch.randint(0, 256, (nblk, Hkv, 4224), dtype=torch.uint8, device=dev)
    host = torch.empty((nblk, Hkv, 4224), dtype=torch.uint8, pin_memory=True)
    back = torch.empty_like(dev_pages)
    t_off = timed(lambda: host.copy_(dev_pages, non_blocking=True), steps)
    t_pro = timed(lambda: back.copy_(host, non_blocking=True), steps)
    torch.cuda.synchronize()
    nbytes = dev_pages.numel()
    return [{"row": "8f-3 pinned-host tier", "config": "2048 blocks x 8 KV heads (32K tokens, one layer)",
             "bytes": nbytes, "offload_ms": t_off, "promote_ms": t_pro,
             "offload_gbs": nbytes / (t_off * 1e-3) / 1e9, "promote_gbs": nbytes / (t_pro * 1e-3) / 1e9,
             "bit_identical": bool(torch.equal(back, dev_pages)),
             "bf16_equivalent_bytes": nblk * 16 * Hkv * 512}]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    for fn in (multi_query, transfer, host_tier):
        for line in fn(args.steps):
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
