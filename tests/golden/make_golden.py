#!/usr/bin/env python3
"""Regenerate the committed golden fixtures in tests/golden/.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

* kat_quant.json     -- contract known-answer rows for the quantizer (DESIGN.md
                        §3).  Expected codes are written out by hand from the
                        rounding rules and cross-checked here against two
                        third-party encoders (ml_dtypes, torch float8_e4m3fn)
                        and numpy's rint; random rows carry expected codes
                        computed by numpy + ml_dtypes (independent of the C
                        oracle).
* ref_block_trace.json -- block-lifecycle traces produced by the REFERENCE
                        itself (servesim.tiered_cache.TieredCacheStore, GPU
                        tier, imported from /root/reference): outcome and the
                        full GPU-tier state after every op.  tests replay them
                        on paper_2605_29639_b200.cache.BlockPool.
The reference is only needed to regenerate; the fixtures travel with the repo.
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import ml_dtypes
import numpy as np
import torch

HERE = Path(__file__).resolve().parent


def bf16(x):
    a = np.asarray(x, dtype=np.float32)
    b = torch.from_numpy(a).to(torch.bfloat16)
    assert torch.equal(b.float(), torch.from_numpy(a)), f"not exactly representable in bf16: {x}"
    return b.view(torch.int16).numpy().view(np.uint16)


def row_with(vals, fill, amax_val):
    r = np.full(128, fill, np.float32)
    r[0] = amax_val
    r[1: 1 + len(vals)] = vals
    return r


def kat():
    cases = []
    # INT8, amax = 127 -> scale 1.0, inv 1.0, code = rint_even(x)
    vals = [0.5, 1.5, 2.5, -0.5, -2.5, 126.5, -126.5, -127.0, 3.5, -3.5, 0.25, 100.0]
    want = [0, 2, 2, 0, -2, 126, -126, -127, 4, -4, 0, 100]
    cases.append(dict(name="int8_ties_amax127", kv_dtype=0, x=row_with(vals, 0.0, 127.0),
                      codes_head=[127] + want, scale=1.0))
    # INT8 zero row -> scale 0, codes 0
    cases.append(dict(name="int8_zero_row", kv_dtype=0, x=np.zeros(128, np.float32),
                      codes_head=[0] * 13, scale=0.0))
    # FP8, amax = 448 -> inv 1.0, code = e4m3_rne_satfinite(x)
    vals = [1.0625, 1.1875, 2 ** -10, 3 * 2 ** -11, -448.0, 0.0, -0.0, 240.0, 17.0, 19.0, -2 ** -9, 0.3125]
    want = [0x38, 0x3A, 0x00, 0x01, 0xFE, 0x00, 0x80, 0x77, 0x58, 0x5A, 0x81, 0x2A]
    cases.append(dict(name="fp8_ties_subnormals_amax448", kv_dtype=1, x=row_with(vals, 0.0, 448.0),
                      codes_head=[0x7E] + want, scale=1.0))
    cases.append(dict(name="fp8_zero_row", kv_dtype=1, x=np.zeros(128, np.float32),
                      codes_head=[0] * 13, scale=0.0))
    out = []
    for c in cases:
        x = c["x"]
        bits = bf16(x)
        # cross-check the hand-written expectations with third-party encoders
        if c["kv_dtype"] == 1 and c["scale"] == 1.0:
            ml = np.clip(x, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
            tt = torch.from_numpy(np.clip(x, -448, 448)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
            assert list(ml[:13]) == c["codes_head"], (c["name"], list(ml[:13]))
            assert np.array_equal(ml, tt)
        if c["kv_dtype"] == 0 and c["scale"] == 1.0:
            assert [int(v) for v in np.rint(x[:13])] == c["codes_head"]
        out.append(dict(name=c["name"], kv_dtype=c["kv_dtype"], x_bf16=[int(v) for v in bits],
                        codes_head=[int(v) & 0xFF for v in c["codes_head"]], scale=c["scale"]))
    # random rows: expected from numpy (int8) / ml_dtypes (fp8), fp32 ops
    rng = np.random.default_rng(2024)
    for kv in (0, 1):
        qmax = np.float32(127.0 if kv == 0 else 448.0)
        xs = (rng.standard_normal((16, 128)) * np.exp2(rng.integers(-20, 20, (16, 1)))).astype(np.float32)
        bits = np.stack([torch.from_numpy(r).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
                         for r in xs])
        xf = (bits.astype(np.uint32) << 16).view(np.float32)
        amax = np.abs(xf).max(1)
        scale = (amax / qmax).astype(np.float32)
        inv = (qmax / amax).astype(np.float32)
        y = (xf * inv[:, None]).astype(np.float32)
        if kv == 0:
            codes = np.clip(np.rint(y), -127, 127).astype(np.int8).view(np.uint8)
        else:
            codes = np.clip(y, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
        for i in range(16):
            out.append(dict(name=f"random_{'int8' if kv == 0 else 'fp8'}_{i}", kv_dtype=kv,
                            x_bf16=[int(v) for v in bits[i]], codes=[int(v) for v in codes[i]],
                            scale_bits=int(scale[i:i + 1].view(np.uint32)[0])))
    (HERE / "kat_quant.json").write_text(json.dumps(out, indent=0))
    print(f"kat_quant.json: {len(out)} rows")


def ref_trace(seed: int, n_ops: int, cap_blocks: int):
    from servesim.errors import CacheThrashError
    from servesim.tiered_cache import CacheTier, TierConfig, TieredCacheStore
    size = 4224
    cfg = TierConfig(capacities={CacheTier.GPU: cap_blocks * size, CacheTier.LOCAL_CPU: None,
                                 CacheTier.REMOTE_CPU: None, CacheTier.DIST_STORE: None},
                     block_size=16)
    st = TieredCacheStore(cfg)
    rng = random.Random(seed)
    keys = list(range(1, 3 * cap_blocks))
    ops = []
    clock = 0
    for _ in range(n_ops):
        clock += rng.randrange(0, 3)
        op = rng.choice(["insert", "insert", "acquire", "acquire", "release", "watermark", "evict"])
        k = rng.choice(keys)
        rec = {"op": op, "key": k, "clock": clock}
        try:
            if op == "insert":
                wm = rng.choice([0, 3, 15, 16, 16, 16])
                rec["watermark"] = wm
                st.insert(k, CacheTier.GPU, size, wm, clock)
            elif op == "acquire":
                st.acquire(k, CacheTier.GPU, clock)
            elif op == "release":
                st.release_and_update([k], clock)
            elif op == "watermark":
                wm = rng.choice([1, 8, 16, 17, 2])
                rec["watermark"] = wm
                st.set_watermark(k, CacheTier.GPU, wm)
            elif op == "evict":
                nb = rng.choice([1, 2])
                rec["nblocks"] = nb
                rec["evicted"] = st.evict(CacheTier.GPU, nb * size)
            rec["outcome"] = "ok"
        except CacheThrashError as e:
            rec["outcome"] = f"thrash:{e.bytes_needed // size}"
        except ValueError as e:
            rec["outcome"] = f"ValueError:{e}"
        except KeyError:
            rec["outcome"] = "KeyError"
        state = {}
        for h, e in st.resident_hashes(CacheTier.GPU).items():
            if e.tier == CacheTier.GPU:
                state[str(h)] = [e.ref_count, e.watermark]
        rec["state"] = state
        ops.append(rec)
    return {"seed": seed, "cap_blocks": cap_blocks, "ops": ops}


def ref_host_trace(seed: int, n_ops: int, gpu_blocks: int, cpu_blocks: int):
    """The reference's GPU + LOCAL_CPU tiers with writeback_on_evict: GPU
    evictions demote to the host only when absent there and only when they fit
    without cascading (tiered_cache.py:254-275); fetch_to_gpu promotes a host
    hit back and keeps the host copy (tiered_cache.py:277-317).  Full blocks
    only (the prefix-hashed pages the host tier holds)."""
    from servesim.errors import CacheThrashError
    from servesim.tiered_cache import CacheTier, TierConfig, TieredCacheStore
    size = 4224
    cfg = TierConfig(capacities={CacheTier.GPU: gpu_blocks * size, CacheTier.LOCAL_CPU: cpu_blocks * size,
                                 CacheTier.REMOTE_CPU: None, CacheTier.DIST_STORE: None},
                     block_size=16, writeback_on_evict=True)
    st = TieredCacheStore(cfg)
    rng = random.Random(seed)
    keys = list(range(1, 3 * (gpu_blocks + cpu_blocks)))
    ops = []
    clock = 0
    for _ in range(n_ops):
        clock += rng.randrange(0, 3)
        op = rng.choice(["insert", "insert", "fetch", "fetch", "fetch", "release", "release", "evict"])
        k = rng.choice(keys)
        on_cpu = sorted(h for h in st._entries if CacheTier.LOCAL_CPU in st._entries[h])
        held = sorted(h for h, by in st._entries.items() if CacheTier.GPU in by and by[CacheTier.GPU].ref_count)
        if op == "fetch" and on_cpu and rng.random() < 0.5:
            k = rng.choice(on_cpu)          # exercise promotion
        if op == "release" and held and rng.random() < 0.8:
            k = rng.choice(held)
        rec = {"op": op, "key": k, "clock": clock}
        try:
            if op == "insert":
                st.insert(k, CacheTier.GPU, size, 16, clock)
            elif op == "fetch":
                plan = st.fetch_to_gpu(k, clock)
                rec["hit"] = None if plan.hit_tier is None else plan.hit_tier.name
            elif op == "release":
                st.release_and_update([k], clock)
            elif op == "evict":
                rec["evicted"] = st.evict(CacheTier.GPU, size)
            rec["outcome"] = "ok"
        except CacheThrashError as e:
            rec["outcome"] = f"thrash:{e.bytes_needed // size}"
        except ValueError as e:
            rec["outcome"] = f"ValueError:{e}"
        except KeyError:
            rec["outcome"] = "KeyError"
        rec["gpu"] = {str(h): e.ref_count for h, e in st.resident_hashes(CacheTier.GPU).items()
                      if e.tier == CacheTier.GPU}
        rec["cpu"] = sorted(h for h in st._entries if CacheTier.LOCAL_CPU in st._entries[h])
        ops.append(rec)
    return {"seed": seed, "gpu_blocks": gpu_blocks, "cpu_blocks": cpu_blocks, "ops": ops}


def main():
    kat()
    try:
        import servesim  # noqa: F401
    except ImportError:
        sys.path.insert(0, "/root/reference/pkg/src")
    traces = [ref_trace(s, 400, cap) for s, cap in ((1, 6), (2, 10), (3, 4), (4, 24))]
    (HERE / "ref_block_trace.json").write_text(json.dumps(traces))
    print("ref_block_trace.json:", sum(len(t["ops"]) for t in traces), "ops")
    host = [ref_host_trace(s, 400, g, c) for s, g, c in ((11, 4, 3), (12, 6, 1), (13, 8, 10), (14, 3, 6))]
    (HERE / "ref_host_trace.json").write_text(json.dumps(host))
    print("ref_host_trace.json:", sum(len(t["ops"]) for t in host), "ops")


if __name__ == "__main__":
    main()
