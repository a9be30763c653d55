#!/usr/bin/env python3
"""Benchmark of the quantized paged-KV decode step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--impl ours|reference] [--no-cpu-baseline]

A *step* is one decode step of one attention layer for the whole batch:
quantize-on-append of the B new K/V rows (K1) followed by paged GQA decode
attention over the quantized cache (K2 + fused split-KV combine), plus, when
sharded over N GPUs by KV head, the NCCL all-gather of the per-head outputs.
The step is stationary: each step re-appends the token at position ctx_b and
attends over ctx_b + 1 tokens, so every timed step moves the same bytes.

Default workload (BASELINE.json ``configs[1]``, the config the metric is
quoted on at 1 GPU): Llama-3-8B shape (Hq=32, Hkv=8, d=128), B=256, ragged
ctx ~ U{512..8192}, INT8 KV, block 16.  The KV pool (2.36 GB) is far larger
than L2 (126 MB), so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0 (see the contract in DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

CONFIGS = {
    "c1": dict(workload="C1: Llama-3-8B shape decode attn (Hq=32, Hkv=8, d=128), B=8, ctx 2048, "
                        "INT8 per-token-head KV, block 16", B=8, ctx=("fixed", 2048), Hq=32, Hkv=8,
               kv="int8"),
    "c2": dict(workload="C2: Llama-3-8B shape (Hq=32, Hkv=8, d=128), B=256, ragged ctx ~U{512..8192} "
                        "(seed 3), INT8 per-token-head KV, block 16", B=256, ctx=("uniform", 512, 8192),
               Hq=32, Hkv=8, kv="int8"),
    "c3": dict(workload="C3: Qwen2.5-72B shape (Hq=64, Hkv=8, d=128), B=128, ctx 32768, FP8-E4M3 KV, "
                        "block 16", B=128, ctx=("fixed", 32768), Hq=64, Hkv=8, kv="fp8_e4m3"),
    "c4": dict(workload="C4: Qwen3-235B-A22B shape (Hq=64, Hkv=4, d=128), B=64, ctx 131072, INT8 KV, "
                        "block 16, split-KV", B=64, ctx=("fixed", 131072), Hq=64, Hkv=4, kv="int8"),
    "c5": dict(workload="C5: Llama-3-8B shape (Hq=32, Hkv=8, d=128); per step 4 chunked-prefill appends "
                        "of 2048 tokens + 252 decode sequences in prefix groups of 8 sharing a 1024-token "
                        "(64-block) prefix, private suffix ~U{64..3072}; block 16", B=252, Hq=32, Hkv=8,
               kv="int8", prefill_seqs=4, chunk=2048, group=8, prefix=1024, suffix=(64, 3072)),
}
METRIC = "quantized paged decode-attn tokens/s and HBM GB/s (% of ~8 TB/s) at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0


def ctx_lens(cfg) -> np.ndarray:
    kind = cfg["ctx"][0]
    if kind == "fixed":
        return np.full(cfg["B"], cfg["ctx"][1], dtype=np.int64)
    lo, hi = cfg["ctx"][1], cfg["ctx"][2]
    return np.random.default_rng(3).integers(lo, hi + 1, size=cfg["B"]).astype(np.int64)


def algorithmic_bytes(lens, Hq_loc, Hkv_loc, B):
    """codes + fp32 scales + q in + O out + block-table reads
    (attention), and the append of B rows (K1)."""
    L = lens + 1  # attended length in the stationary step
    attn = int(L.sum()) * Hkv_loc * (2 * 128 + 8) + B * Hq_loc * 128 * 2 * 2 + int(np.ceil(L / 16).sum()) * 4
    append = B * Hkv_loc * (2 * 128 * 2 + 2 * 128 + 2 * 4) + 4 * B
    return attn, append


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncu_traffic(config: str, kv: str):
    """dram__bytes_read + write per K2 launch from profiles/ncu_traffic.json,
    only if that capture measured THIS build (same source hash) and the same
    KV dtype (the kernel's first template argument: 0 INT8, 1 FP8); else None."""
    from paper_2605_29639_b200._build import source_hash
    tp = REPO / "profiles" / "ncu_traffic.json"
    try:
        rec = json.loads(tp.read_text()).get(config, {})
    except (OSError, ValueError):
        return None, None
    if rec.get("src_hash") != source_hash():
        return None, rec.get("src_hash")
    if ("decode_kernel<1" if kv == "fp8_e4m3" else "decode_kernel<0") not in rec.get("kernel", ""):
        return None, rec.get("src_hash")
    return rec.get("dram_bytes_per_launch"), rec.get("src_hash")


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """NVML sampling of SM clocks + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU side: the oracle (reference arm / cpu_baseline) on a bounded sample
# ---------------------------------------------------------------------------
class CpuSample:
    """The oracle (oracle/libkvq_oracle.so) running the same step on the host:
    append of the sample's new rows + paged decode attention, all host threads."""

    def __init__(self, cfg, lens, Hq, Hkv, nseq):
        import oracle as O
        self.O = O
        self.kv = O.INT8 if cfg["kv"] == "int8" else O.FP8_E4M3
        self.lens = lens[:nseq].astype(np.int32)
        self.B, self.Hq, self.Hkv = nseq, Hq, Hkv
        rng = np.random.default_rng(1)
        L1 = self.lens + 1
        nblk = np.ceil(L1 / 16).astype(np.int64)
        self.max_blocks = int(nblk.max())
        nb = int(nblk.sum())
        # Pool of random codes with realistic positive scales (timing only).
        self.pool = rng.integers(0, 256, size=(nb, Hkv, O.PAGE), dtype=np.uint8)
        if self.kv == O.FP8_E4M3:
            self.pool[..., :4096] &= 0xF7  # avoid NaN codes (0x7F / 0xFF)
        sc = (np.abs(rng.standard_normal((nb, Hkv, 32))) * 0.02 + 1e-3).astype(np.float32)
        self.pool[..., 4096:] = sc.view(np.uint8).reshape(nb, Hkv, 128)
        perm = rng.permutation(nb).astype(np.int32)
        self.table = np.zeros((nseq, self.max_blocks), dtype=np.int32)
        pos = 0
        for b in range(nseq):
            self.table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
            pos += nblk[b]
        self.slots = (self.table[np.arange(nseq), self.lens // 16] * 16 + self.lens % 16).astype(np.int32)
        self.q = O.f32_to_bf16_bits(rng.standard_normal((nseq, Hq, 128)).astype(np.float32))
        self.k = O.f32_to_bf16_bits(rng.standard_normal((nseq, Hkv, 128)).astype(np.float32))
        self.v = O.f32_to_bf16_bits(rng.standard_normal((nseq, Hkv, 128)).astype(np.float32))
        self.threads = O.num_threads()

    def step(self):
        self.O.quant_append(self.k, self.v, self.slots, self.kv, self.pool)
        self.O.decode_attn(self.q, self.pool, self.table, self.lens + 1, self.Hkv, self.kv,
                           nthreads=self.threads)

    def describe(self):
        return (f"{self.B} of the workload's sequences (sum ctx {int(self.lens.sum() + self.B)}, "
                f"{self.Hkv} KV heads, {self.Hq} q heads): append + paged decode attention per step, "
                f"{self.threads} host threads, oracle/libkvq_oracle.so")


def cpu_sample_for(cfg, lens, Hq, Hkv, target_step_s):
    """Grow the sample until one step takes ~target_step_s."""
    n = 4
    while True:
        s = CpuSample(cfg, lens, Hq, Hkv, min(n, len(lens)))
        s.step()
        t0 = time.perf_counter()
        s.step()
        dt = time.perf_counter() - t0
        if dt >= target_step_s or n >= len(lens):
            return s, dt
        n = min(len(lens), max(n + 1, int(n * target_step_s / max(dt, 1e-4))))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lens = ctx_lens(cfg)
    sample, _ = cpu_sample_for(cfg, lens, cfg["Hq"], cfg["Hkv"], target_step_s=0.15)
    for _ in range(args.warmup):
        sample.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sample.step()
    dt = (time.perf_counter() - t0) / args.steps
    value = sample.B / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg["kv"].replace("fp8_e4m3", "e4m3"), "data": "synthetic",
        "config": {"workload": cfg["workload"], "sample": sample.describe()},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": sample.threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample.describe()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm: the reference (servesim) has no implementation of this path "
                "(SPEC.md:8); its CPU implementation here is the oracle port of the contract",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # KVQ_BENCH_ONE_GPU=1 (debug only): run every rank on cuda:0 over gloo, to
    # exercise the sharded code path on a single-GPU box.  Timings are then
    # meaningless; the driver never sets it.
    one_gpu = os.environ.get("KVQ_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, quantize_append
    from paper_2605_29639_b200.session import DecodeSession
    from paper_2605_29639_b200.shard import OutputGather, PeerOutput, plan_shards

    B, Hq, Hkv = cfg["B"], cfg["Hq"], cfg["Hkv"]
    lens_all = ctx_lens(cfg)
    # KV-head split when Hkv % N == 0, else KV-head groups x LPT batch parts (C4 at N = 8)
    plan = plan_shards(Hq, Hkv, world, rank, lens_all + 1)
    (kv0, kv1), (q0, q1) = plan.kv_range, plan.q_range
    Hkv_loc, Hq_loc = kv1 - kv0, q1 - q0
    seqs = plan.seqs
    lens = lens_all[seqs]
    B_loc = len(seqs)
    L1 = lens + 1
    nblk = np.ceil(L1 / 16).astype(np.int64)
    max_blocks = int(nblk.max())
    num_blocks = int(nblk.sum())
    rng = np.random.default_rng(7 + rank)
    perm = rng.permutation(num_blocks).astype(np.int32)
    table = np.zeros((B_loc, max_blocks), dtype=np.int32)
    pos = 0
    for b in range(B_loc):
        table[b, : nblk[b]] = perm[pos: pos + nblk[b]]
        pos += nblk[b]
    spec = KVCacheSpec(Hkv_loc, kv_dtype=cfg["kv"])
    cache = PagedKVCache(spec, num_blocks, device=dev)
    table_d = torch.from_numpy(table).to(dev)

    # Fill this rank's pool (its KV heads, its sequences) through K1, in chunks.
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    tok_b = np.repeat(np.arange(B_loc), lens)
    tok_t = np.concatenate([np.arange(L) for L in lens]) if B_loc else np.zeros(0, np.int64)
    all_slots = (table[tok_b, tok_t // 16].astype(np.int64) * 16 + tok_t % 16).astype(np.int32)
    chunk = 1 << 15
    for s0 in range(0, len(all_slots), chunk):
        sl = torch.from_numpy(all_slots[s0: s0 + chunk]).to(dev)
        n = sl.numel()
        kv = torch.randn((2, n, Hkv_loc, 128), device=dev, generator=gen)
        kv = (kv * torch.exp(0.5 * torch.randn((2, n, Hkv_loc, 1), device=dev, generator=gen))).to(torch.bfloat16)
        quantize_append(cache, kv[0], kv[1], sl)
    del kv
    seq_lens_d = torch.from_numpy(L1.astype(np.int32)).to(dev)
    slots_step = torch.from_numpy((table[np.arange(B_loc), lens // 16].astype(np.int64) * 16 + lens % 16)
                                  .astype(np.int32)).to(dev)
    q = torch.randn((B_loc, Hq_loc, 128), device=dev, generator=gen).to(torch.bfloat16)
    k_new = torch.randn((B_loc, Hkv_loc, 128), device=dev, generator=gen).to(torch.bfloat16)
    v_new = torch.randn((B_loc, Hkv_loc, 128), device=dev, generator=gen).to(torch.bfloat16)
    total_pages = int(nblk.sum())

    def make_gather():
        return OutputGather(plan, Hq, B, torch.bfloat16, dev)

    # N > 1: the all-gather is fused into K2 (peer-memory stores + flags) unless
    # --gather nccl asks for the separate NCCL collective (the baseline).
    peer = None
    gather_mode = "none" if world == 1 else args.gather
    if gather_mode == "peer":
        try:
            peer = PeerOutput(plan, Hq, B, Hkv, dev, slots=2)
        except Exception as e:  # setup-time capability check (e.g. no CUDA IPC): fall back to NCCL
            print(f"[bench] fused peer gather unavailable ({e}); NCCL all-gather", file=sys.stderr)
            gather_mode = f"nccl (peer setup failed: {type(e).__name__})"
    use_nccl = world > 1 and peer is None
    # The stationary step re-appends each sequence's newest token (its last page).
    # --append fused: no K1 launch, the K2 CTA holding each sequence's last page
    # quantizes the new row (KVQ_STEP_FUSED_APPEND); not combined with the peer gather.
    fused = args.append == "fused" and peer is None
    l2_fits = cache.nbytes() * world <= 4 * 126e6
    sess = DecodeSession(cache, table_d, B_loc, Hq_loc, total_pages=total_pages, head_major=True,
                         gather_factory=make_gather if use_nccl else None, peer=peer,
                         pages_per_split=args.pages_per_split, append_tail_only=True, fused_append=fused)
    buf = sess.device_buffers(0)
    for name, t in (("q", q), ("k", k_new), ("v", v_new), ("slots", slots_step), ("lens", seq_lens_d)):
        buf[name].copy_(t)
    gather_dev = make_gather() if use_nccl else None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region: one CUDA graph of all K steps ---------
    # Each step is [K1, event, K2, event (, all-gather)]; the graph holds the W
    # warm-up steps or the K timed steps unrolled, so there is no per-step host
    # launch in the timed region.  The K2 events are graph event-record nodes.
    sess._kernels(buf)  # warm the kernels (and lazy module loading) before capture
    if use_nccl:
        gather_dev(buf["out"])  # communicator set up before any capture
    torch.cuda.synchronize()
    gather_in_graph = use_nccl and not one_gpu

    # K2's own duration inside the timed PDL steps: every timed K2 records its
    # grid span (first CTA start .. last CTA end, %globaltimer) into its own
    # slot (kvq_profile_next_decode; the pointer is a captured kernel
    # parameter), so the roofline's kernel time comes from the very launches
    # the step time is measured on.
    from paper_2605_29639_b200.ops import profile_next_decode
    spans = torch.zeros((max(args.steps, 1), 2), dtype=torch.int64, device=dev)

    def reset_spans():
        spans[:, 0] = torch.iinfo(torch.int64).max
        spans[:, 1] = 0

    # A pool that fits in L2 (C1) would be timed L2-resident: instead every step
    # is preceded by a 256 MB memset that evicts L2 and bracketed by its own
    # events (the flush is outside the brackets); ms_step is their mean.
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if l2_fits else None
    step_evs = []

    def capture_steps(n, timed):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(n):
                if flush_buf is not None:
                    flush_buf.zero_()
                ev = None
                if flush_buf is not None and timed:
                    ev = (torch.cuda.Event(enable_timing=True, external=True),
                          torch.cuda.Event(enable_timing=True, external=True))
                    ev[0].record()
                if timed:
                    profile_next_decode(spans[i])
                sess.step(buf)  # kvq_decode_step: K2 PDL-launched behind K1 (or the fused K2 alone)
                if ev is not None:
                    ev[1].record()
                    step_evs.append(ev)
                if gather_in_graph:
                    gather_dev(buf["out"])
        return g, []

    graphs = None
    if not use_nccl or gather_in_graph:
        try:
            graphs = capture_steps(args.warmup, False)[0], capture_steps(args.steps, True)
        except Exception as e:  # e.g. a NCCL build that cannot be captured: eager gather
            print(f"[bench] step capture with the all-gather failed ({e}); eager gather", file=sys.stderr)
            torch.cuda.synchronize()
    if graphs is not None:
        g_warm, (g_timed, evs) = graphs

        def run_warm():
            g_warm.replay()

        def run_timed():
            g_timed.replay()
    else:  # gloo debug mode (or no NCCL capture): per-step graphs of K1 and K2, eager gather
        g_append, g_attn = sess.capture()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]

        def one(ev=None):
            g_append.replay()
            if ev is not None:
                ev[0].record()
            g_attn.replay()
            if ev is not None:
                ev[1].record()
            if gather_dev is not None:
                gather_dev(buf["out"])

        def run_warm():
            for _ in range(args.warmup):
                one()

        def run_timed():
            for i in range(args.steps):
                one(evs[i])

    run_warm()
    reset_spans()
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        t_start.record()
        run_timed()
        t_end.record()
        torch.cuda.synchronize()
    ms_total = max_over_ranks(t_start.elapsed_time(t_end))
    ms_step = ms_total / args.steps
    if step_evs:  # L2-flushed steps: the mean bracketed step, not the graph span (which holds the flushes)
        ms_step = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in step_evs))
    if evs:  # eager fallback: K2 bracketed by events
        k2_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        k2_src = "CUDA events around K2 (eager fallback path, no PDL)"
    else:
        sp = spans.cpu().numpy()
        ok = sp[:, 0] < np.iinfo(np.int64).max
        k2_ms = float((sp[ok, 1] - sp[ok, 0]).mean()) / 1e6 if ok.any() else float("nan")
        k2_src = ("grid span of every timed K2 inside the PDL step graph (first CTA start to last CTA "
                  "end, %globaltimer; kvq_profile_next_decode)")
    n_k2 = len(evs) if evs else int(args.steps)
    k2_ms = max_over_ranks(k2_ms)

    # ---- end-to-end through the public API with pinned host buffers ----------
    # DecodeSession with graphs: each step = one H2D copy of the pinned staging
    # blob (q | k | v | slots | lens), the captured K1/K2 (/gather) graph, one
    # D2H copy of O.  The stationary inputs are written into both slots'
    # staging blobs once; every step still uploads them.
    es = DecodeSession(cache, table_d, B_loc, Hq_loc, total_pages=total_pages, head_major=True,
                       gather_factory=make_gather if use_nccl else None, peer=peer,
                       pages_per_split=args.pages_per_split, graphs=not (one_gpu and use_nccl),
                       append_tail_only=True, fused_append=fused)
    host_inputs = {"q": q, "k": k_new, "v": v_new, "slots": slots_step, "lens": seq_lens_d}
    for b in es.bufs:
        for name, t in host_inputs.items():
            b["host"][name].copy_(t.cpu())
    o_h = torch.empty((Hq, B, 128), dtype=torch.bfloat16, pin_memory=True)

    def e2e_step():
        es.submit_staged(o_h)

    for _ in range(args.warmup):
        e2e_step()
    es.synchronize()
    barrier()
    if flush_buf is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(es.h2d)
        for _ in range(args.steps):
            e2e_step()
        e1.record(es.d2h)
        es.synchronize()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    else:  # L2 flushed before every step: serialized per-step latency, upload to download
        tot = 0.0
        for _ in range(args.steps):
            flush_buf.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(es.h2d)
            e2e_step()
            e1.record(es.d2h)
            es.synchronize()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        e2e_ms = max_over_ranks(tot / args.steps)
    h2d = es.in_bytes
    d2h = o_h.numel() * o_h.element_size()

    # ---- CPU baseline (rank 0, N = 1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample, dt1 = cpu_sample_for(cfg, lens, Hq, Hkv, target_step_s=1.0)
        reps, t0 = 0, time.perf_counter()
        while True:
            sample.step()
            reps += 1
            if time.perf_counter() - t0 >= args.cpu_seconds and reps >= 3:
                break
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": sample.B / dt, "unit": "tokens/s", "cores": sample.threads, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": sample.describe() + f"; {reps} reps, {dt * 1e3:.1f} ms/step"}

    peer_errors = peer.errors() if peer is not None else 0
    if peer is not None:
        peer.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    if peer_errors:
        raise SystemExit(f"fused peer gather: {peer_errors} slot(s) timed out")
    attn_bytes, append_bytes = algorithmic_bytes(lens, Hq_loc, Hkv_loc, B_loc)
    peak, peak_kind = measured_peak()
    achieved = attn_bytes / (k2_ms * 1e-3) / 1e9
    from paper_2605_29639_b200._build import source_hash
    traffic, traffic_hash = (ncu_traffic(args.config, cfg["kv"]) if world == 1 else (None, None))
    value = B / (ms_step * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": cfg["kv"].replace("fp8_e4m3", "e4m3"), "data": "synthetic",
        "config": {"workload": cfg["workload"], "name": args.config, "global_batch": B,
                   "sum_ctx": int((lens_all + 1).sum()),
                   "gather": {"none": "none (1 GPU)",
                              "peer": "fused into K2: peer-memory row stores + done/free flags (no collective launch)",
                              "nccl": "NCCL all_gather_into_tensor after K2"}.get(gather_mode, gather_mode),
                   "parallelism": (f"kv-head tp{world}" if plan.b_split == 1 else
                                   f"{plan.h_split} kv-head groups x {plan.b_split} LPT batch parts")
                   if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (pool %.2f GB vs 126 MB L2); no flush" % (cache.nbytes() * world / 1e9)
                   if not l2_fits else "pool fits in L2: a 256 MB memset evicts L2 before every step (outside the "
                                       "step's event brackets); value and e2e are per-step means of flushed steps",
                   "append": "fused into K2 (KVQ_STEP_FUSED_APPEND: no K1 launch)" if fused
                   else "K1 + K2 (PDL, tail-only wait)",
                   "step": "K1 append of B rows + K2 paged decode attention (+ the gather if N>1); "
                           "stationary ctx; the K timed steps are one CUDA graph (kvq_decode_step per step: K2 "
                           "launched behind K1 with programmatic dependent launch, waiting for K1 only before "
                           "each sequence's last page; unrolled); K2 time = each timed K2's own grid span "
                           "inside that graph",
                   "e2e": "DecodeSession(graphs=True).submit_staged: one H2D of the pinned q/k/v/slots/lens "
                          "staging blob, graph of K1, K2 (, all-gather), D2H of O; double-buffered copy "
                          "streams overlap adjacent steps",
                   "compute": "TMA bulk page copies; QK^T: INT8 codes on s8 tensor cores (mma m16n8k32, two-term int8 Q) / E4M3 codes -> f16 (mma m16n8k16); PV: codes -> f16, mma m16n8k16 f32 accumulate"},
        "hbm_gbs_algorithmic_step": (attn_bytes + append_bytes) / (ms_step * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": "kvq::decode_kernel",
                     "algorithmic_bytes_per_launch": attn_bytes, "avg_launch_ms": k2_ms,
                     "launches_sampled": n_k2, "kernel_time": k2_src,
                     "traffic_source": ("ncu --set full of this build (profiles/ncu_traffic.json, src_hash "
                                        f"{traffic_hash})") if traffic is not None else
                     f"none for this build (profiles/ncu_traffic.json has src_hash {traffic_hash})",
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                     else "fallback 6.65 TB/s (B200_PROFILING.md)"},
        "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": (1 if fused else 2) * args.steps,
        "clocks": sampler.summary(),
        "build": {"src_hash": source_hash()},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# Serving loop: a whole model step (all layers) driven by the allocator
# ---------------------------------------------------------------------------
def run_serving(args, cfg):
    """--serving: the decode loop of a model with --layers attention layers,
    as a server runs it (simulator.py:504-517).  Per model step the host calls
    BlockAllocator.append_one (each sequence's new slot; sequences grow),
    BlockTable.sync (new block ids + lengths, pinned staging, copy stream) and
    uploads the slots, then launches kvq_decode_step (K1 + PDL K2) for every
    layer's pool.  The host never waits for the device (--table-sync legacy
    instead synchronizes the compute stream before each sync, the round-1
    behaviour of the pageable copies).  Reports the model step's device time
    against the same layers replayed from a CUDA graph with no host work, and
    the host time per step."""
    import torch
    from paper_2605_29639_b200 import BlockAllocator, BlockTable, KVCacheSpec, PagedKVCache, quantize_append
    from paper_2605_29639_b200 import ops

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B, Hq, Hkv, layers = cfg["B"], cfg["Hq"], cfg["Hkv"], args.layers
    lens = ctx_lens(cfg)
    steps_total = args.warmup + args.steps + 2
    nb = int(np.ceil((lens + steps_total) / 16).sum()) + B + 16
    spec = KVCacheSpec(Hkv, kv_dtype=cfg["kv"])
    alloc = BlockAllocator(nb, bytes_per_block=spec.bytes_per_block)
    alloc.pool._free = [int(x) for x in np.random.default_rng(7).permutation(nb)]  # random block ids, as the stationary bench
    seqs = list(range(B))
    slots0 = []
    for b in seqs:
        alloc.allocate(b)
        slots0 += alloc.append_slots(b, int(lens[b]))
    caches = [PagedKVCache(spec, nb, device=dev) for _ in range(layers)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    sl_all = torch.tensor(slots0, dtype=torch.int32, device=dev)
    for s0 in range(0, sl_all.numel(), 1 << 15):
        sl = sl_all[s0: s0 + (1 << 15)]
        kv = torch.randn((2, sl.numel(), Hkv, 128), device=dev, generator=gen)
        kv = (kv * torch.exp(0.5 * torch.randn((2, sl.numel(), Hkv, 1), device=dev, generator=gen))).to(torch.bfloat16)
        quantize_append(caches[0], kv[0], kv[1], sl)
    del kv
    for c in caches[1:]:
        c.pool.copy_(caches[0].pool)
    max_blocks = int(np.ceil((lens.max() + steps_total) / 16)) + 1
    table = BlockTable(B, max_blocks, device=dev)
    table.sync(alloc, seqs)
    q = torch.randn((B, Hq, 128), device=dev, generator=gen).to(torch.bfloat16)
    k_new = torch.randn((B, Hkv, 128), device=dev, generator=gen).to(torch.bfloat16)
    v_new = torch.randn((B, Hkv, 128), device=dev, generator=gen).to(torch.bfloat16)
    out = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev)
    total_pages = int(np.ceil((lens + 1) / 16).sum())
    pps = ops.pages_per_split(B, Hkv, total_pages, max_blocks, rows=Hq // Hkv)
    ws = torch.zeros(ops.workspace_bytes(B, Hq, Hkv, -(-max_blocks // pps)), dtype=torch.uint8, device=dev)
    compute = torch.cuda.current_stream(dev)
    copy_stream = torch.cuda.Stream(dev)
    slot_host = [torch.empty((B,), dtype=torch.int32, pin_memory=True) for _ in range(2)]
    slot_dev = [torch.empty((B,), dtype=torch.int32, device=dev) for _ in range(2)]
    slot_ev = [None, None]
    legacy = args.table_sync == "legacy"

    def layer_steps(slots_d):
        for c in caches:
            ops.decode_step(c, k_new, v_new, slots_d, q, table.table, table.seq_lens, out=out,
                            pages_per_split=pps, workspace=ws, append_tail_only=True)

    host_s, wait_s = [], []
    step_graphs = [None, None]

    def launch_layers(i):
        if args.serving_graphs:   # one CUDA graph of all layers' launches per slot buffer
            if step_graphs[i] is None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=torch.cuda.Stream(dev)):
                    layer_steps(slot_dev[i])
                step_graphs[i] = g
            step_graphs[i].replay()
        else:
            layer_steps(slot_dev[i])

    def model_step(t):
        i = t % 2
        w0 = time.perf_counter()
        if legacy:
            compute.synchronize()
        if slot_ev[i] is not None:
            slot_ev[i].synchronize()  # bounded run-ahead: this slot buffer's step (t - 2) is done
        h0 = time.perf_counter()
        new = alloc.append_one(seqs)
        slot_host[i].numpy()[:] = new
        with torch.cuda.stream(copy_stream):
            slot_dev[i].copy_(slot_host[i], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        table.sync(alloc, seqs, copy_stream=copy_stream)
        compute.wait_event(ev)
        host_s.append(time.perf_counter() - h0)
        wait_s.append(h0 - w0)
        launch_layers(i)
        slot_ev[i] = torch.cuda.Event()
        slot_ev[i].record(compute)

    for t in range(args.warmup):
        model_step(t)
    torch.cuda.synchronize()
    host_s.clear()
    wait_s.clear()
    sampler = ClockSampler(0)
    with sampler:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        for t in range(args.steps):
            model_step(args.warmup + t)
        e1.record()
        launch_s = time.perf_counter() - w0
        torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / args.steps
    # the same layers with no host work: one step's launches in a CUDA graph
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer_steps(slot_dev[0])
    g.replay()
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record()
    for _ in range(args.steps):
        g.replay()
    d1.record()
    torch.cuda.synchronize()
    ms_graph = d0.elapsed_time(d1) / args.steps
    alloc.check_invariants()
    attn_bytes, append_bytes = algorithmic_bytes(lens + args.warmup + args.steps // 2, Hq, Hkv, B)
    line = {
        "mode": "serving", "metric": METRIC, "value": B / (ms_step * 1e-3), "unit": "decoded tokens/s (model)",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "layers": layers,
        "ms_per_model_step": ms_step, "ms_per_layer": ms_step / layers,
        "graph_ms_per_model_step": ms_graph, "overhead_vs_graph": ms_step / ms_graph - 1,
        "host_ms_per_step": 1e3 * statistics.mean(host_s),
        "host_wait_ms_per_step": 1e3 * statistics.mean(wait_s),
        "host_loop_ms_per_step": 1e3 * launch_s / args.steps,
        "host_ahead": 1e3 * (launch_s - sum(wait_s)) / args.steps < ms_step,
        "launch": "one CUDA graph of the layers' launches per step" if args.serving_graphs
        else "ops.decode_step per layer (eager)",
        "table_sync": "legacy (compute stream synchronized before each step's host work)" if legacy
        else "async (pinned staging, copy stream, no host wait)",
        "hbm_gbs_per_layer": (attn_bytes + append_bytes) / (ms_step / layers * 1e-3) / 1e9,
        "dtype": cfg["kv"].replace("fp8_e4m3", "e4m3"), "data": "synthetic",
        "config": {"workload": cfg["workload"] + f"; {layers} layers, one pool each (%.1f GB)"
                   % (layers * caches[0].nbytes() / 1e9), "pages_per_split": pps,
                   "step": "host: append_one + BlockTable.sync + slot upload; device: kvq_decode_step "
                           "(K1 + PDL K2) per layer; sequences grow by one token per step; "
                           "host_ms = append_one + sync + upload, host_wait_ms = waiting for the slot "
                           "buffer of step t - 2 (bounded run-ahead)"},
        "gpu_launches": 2 * layers * args.steps, "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# C5: chunked-prefill append + decode mix with prefix-shared blocks
# ---------------------------------------------------------------------------
def run_c5(args, cfg):
    """One step = K1 over 4 x 2048 prefill tokens + 252 decode tokens, then K2
    over the 252 decode sequences, whose block tables share each group's
    64-block prefix (BlockAllocator.fork).  Reports decode tokens/s, prefill
    append GB/s, logical vs DRAM bytes and the quantisation error against
    fp32 attention over the unquantised K/V (first prefix group)."""
    import torch
    from paper_2605_29639_b200 import (BlockAllocator, KVCacheSpec, PagedKVCache,
                                       paged_decode_attention, quantize_append)

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B, Hq, Hkv, G = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["group"]
    rng = np.random.default_rng(5)
    suffix = rng.integers(cfg["suffix"][0], cfg["suffix"][1] + 1, size=B)
    ngroups = -(-B // G)
    spec = KVCacheSpec(Hkv, kv_dtype=cfg["kv"])
    need = ngroups * cfg["prefix"] // 16 + int(np.ceil((suffix + 1) / 16).sum()) + B \
        + cfg["prefill_seqs"] * cfg["chunk"] // 16 + 64
    alloc = BlockAllocator(need, bytes_per_block=spec.bytes_per_block)
    cache = PagedKVCache(spec, need, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)

    def kv_rows(n):
        x = torch.randn((2, n, Hkv, 128), device=dev, generator=gen)
        return (x * torch.exp(0.5 * torch.randn((2, n, Hkv, 1), device=dev, generator=gen))).to(torch.bfloat16)

    keep = {}  # bf16 K/V of group 0 for the error report: seq -> (k, v)
    seqs = []
    for gi in range(ngroups):
        pid = ("prefix", gi)
        alloc.allocate(pid)
        sl = alloc.append_slots(pid, cfg["prefix"])
        kv = kv_rows(cfg["prefix"])
        quantize_append(cache, kv[0], kv[1], torch.tensor(sl, dtype=torch.int32, device=dev))
        for j in range(G):
            b = gi * G + j
            if b >= B:
                break
            alloc.fork(pid, b)  # prefix is block aligned: shares all 64 blocks, copies nothing
            sl2 = alloc.append_slots(b, int(suffix[b]))
            kv2 = kv_rows(int(suffix[b]))
            quantize_append(cache, kv2[0], kv2[1], torch.tensor(sl2, dtype=torch.int32, device=dev))
            if gi == 0:
                keep[b] = (torch.cat([kv[0], kv2[0]]), torch.cat([kv[1], kv2[1]]))
            seqs.append(b)
        alloc.free(pid)  # children keep the prefix blocks referenced
    # decode token slot (stationary: position ctx_b re-written every step)
    dec_slots = []
    for b in seqs:
        dec_slots.append(alloc.append_slots(b, 1)[0])
    ctx = alloc.seq_lens(seqs)                      # includes the decode token
    table = torch.from_numpy(alloc.block_table(seqs)).to(dev)
    lens_d = torch.from_numpy(ctx).to(dev)
    # prefill chunks: 4 sequences, stationary 2048-token chunk each
    pf_slots = []
    for i in range(cfg["prefill_seqs"]):
        alloc.allocate(("prefill", i))
        pf_slots += alloc.append_slots(("prefill", i), cfg["chunk"])
    alloc.check_invariants()
    T = len(pf_slots) + B
    kv_step = kv_rows(T)
    slots_step = torch.tensor(pf_slots + dec_slots, dtype=torch.int32, device=dev)
    q = torch.randn((B, Hq, 128), device=dev, generator=gen).to(torch.bfloat16)
    total_pages = int(np.ceil(ctx / 16).sum())
    from paper_2605_29639_b200 import ops
    pps = ops.pages_per_split(B, Hkv, total_pages, table.shape[1], rows=Hq // Hkv)
    ws = torch.zeros(ops.workspace_bytes(B, Hq, Hkv, -(-table.shape[1] // pps)), dtype=torch.uint8, device=dev)
    out = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev)
    dec_k = kv_step[0][len(pf_slots):]
    dec_v = kv_step[1][len(pf_slots):]

    def k1():
        quantize_append(cache, kv_step[0], kv_step[1], slots_step)

    def k2():
        paged_decode_attention(q, cache, table, lens_d, out=out, pages_per_split=pps, workspace=ws)

    def step():  # kvq_decode_step: K1 over all appended rows, K2 PDL-launched behind it; the
        # prefill chunks belong to sequences K2 does not attend and each decode row is its
        # sequence's newest token, so K2 streams all but the last pages while K1 runs
        ops.decode_step(cache, kv_step[0], kv_step[1], slots_step, q, table, lens_d, out=out,
                        pages_per_split=pps, workspace=ws, append_tail_only=True)

    from paper_2605_29639_b200.ops import profile_next_append, profile_next_decode
    spans = torch.zeros((max(args.steps, 1), 2), dtype=torch.int64, device=dev)
    k1_step_spans = torch.zeros_like(spans)   # K1 inside the timed step graph
    k1_spans = torch.zeros_like(spans)        # K1 alone, one launch per graph replay
    k1(); k2(); step(); torch.cuda.synchronize()
    g_k1, g_warm, g_timed = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    k1_span_slot = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.graph(g_k1):
        profile_next_append(k1_span_slot)
        k1()
    with torch.cuda.graph(g_warm):
        for _ in range(args.warmup):
            step()
    with torch.cuda.graph(g_timed):   # K steps unrolled; each K2 records its own grid span
        for i in range(args.steps):
            profile_next_decode(spans[i])
            profile_next_append(k1_step_spans[i])
            step()
    g_warm.replay()
    for sp_ in (spans, k1_step_spans):
        sp_[:, 0] = torch.iinfo(torch.int64).max
        sp_[:, 1] = 0
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    with sampler:
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        g_timed.replay()
        t1.record()
        torch.cuda.synchronize()
    ms_step = t0.elapsed_time(t1) / args.steps
    sp = spans.cpu().numpy()
    k2_ms = float((sp[:, 1] - sp[:, 0]).mean()) / 1e6   # K2 inside the PDL step (overlaps K1's tail)
    k1_step_ms = float((k1_step_spans[:, 1] - k1_step_spans[:, 0]).float().mean()) / 1e6
    # K1 alone (its own graph, replayed back to back, bracketed by events; and
    # its grid span, copied out of the graph's span slot after every replay):
    # the prefill-append rate
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for i in range(args.steps):
        k1_span_slot[0] = torch.iinfo(torch.int64).max
        k1_span_slot[1] = 0
        ev[i][0].record(); g_k1.replay(); ev[i][1].record()
        k1_spans[i].copy_(k1_span_slot)
    torch.cuda.synchronize()
    k1_event_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    k1_ms = float((k1_spans[:, 1] - k1_spans[:, 0]).float().mean()) / 1e6

    # quantisation error vs fp32 attention over the unquantised K/V (group 0),
    # with the stationary decode token included
    k2()
    torch.cuda.synchronize()
    errs = []
    for i, b in enumerate(list(keep)):
        kk = torch.cat([keep[b][0], dec_k[b:b + 1]]).float()   # [L, Hkv, d]
        vv = torch.cat([keep[b][1], dec_v[b:b + 1]]).float()
        qq = q[b].float().view(Hkv, Hq // Hkv, 128)
        s_ = torch.einsum("hgd,lhd->hgl", qq, kk) / math.sqrt(128)
        ref = torch.einsum("hgl,lhd->hgd", torch.softmax(s_, -1), vv).reshape(Hq, 128)
        o = out[b].float()
        errs.append(((o - ref).abs().max().item(), ((o - ref).abs().max() / ref.abs().max()).item()))
    attn_logical = int(ctx.sum()) * Hkv * 264 + B * Hq * 512 + total_pages * 4
    attn_unique_kv = (ngroups * cfg["prefix"] + int((ctx - cfg["prefix"]).sum())) * Hkv * 264
    attn_unique = attn_unique_kv + B * Hq * 512 + total_pages * 4
    append_bytes = T * Hkv * (2 * 128 * 2 + 2 * 128 + 8) + 4 * T
    peak, peak_kind = measured_peak()
    # HBM roofline on the bytes that must come from DRAM: each shared prefix
    # page once (the 8 sequences of a group re-read it from L2)
    achieved = attn_unique / (k2_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": B / (ms_step * 1e-3), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg["kv"].replace("fp8_e4m3", "e4m3"),
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "name": "c5", "decode_seqs": B, "sum_ctx": int(ctx.sum()),
                   "prefill_tokens_per_step": len(pf_slots), "prefix_groups": ngroups,
                   "l2": "pool %.2f GB; shared prefixes are re-read by 8 sequences (L2 hits expected)"
                         % (cache.nbytes() / 1e9)},
        "k1_ms": k1_ms, "k1_event_ms": k1_event_ms, "k1_in_step_ms": k1_step_ms, "k2_ms": k2_ms,
        "append_bytes": append_bytes,
        "append_gbs": append_bytes / (k1_ms * 1e-3) / 1e9,
        "append_frac": append_bytes / (k1_ms * 1e-3) / 1e9 / peak,
        "k1_time": "k1_ms: grid span of K1 alone (first CTA start to last CTA end, %globaltimer; "
                   "kvq_profile_next_append), its graph replayed back to back; k1_event_ms: CUDA events "
                   "around each replay (adds the graph launch); k1_in_step_ms: K1's span inside the timed "
                   "PDL step graph (K2 streams beside it)",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic("c5", cfg["kv"])[0], "kernel": "kvq::decode_kernel",
                     "algorithmic_bytes_per_launch": attn_unique, "unique_kv_bytes": attn_unique_kv,
                     "logical_bytes_per_launch": attn_logical,
                     "logical_gbs": attn_logical / (k2_ms * 1e-3) / 1e9,
                     "avg_launch_ms": k2_ms, "peak_source": peak_kind,
                     "kernel_time": "grid span of every timed K2 inside the PDL step graph",
                     "note": "achieved = unique bytes (each shared prefix page once, + q/O + table) / K2 time; "
                             "logical_gbs counts every sequence's reads of its prefix"},
        "quant_error_vs_fp32_unquantized": {"max_abs": max(e[0] for e in errs),
                                            "max_rel_to_row_max": max(e[1] for e in errs),
                                            "sequences": len(errs)},
        "gpu_launches": 2 * args.steps, "clocks": sampler.summary(),
        "build": {"src_hash": __import__("paper_2605_29639_b200._build", fromlist=["x"]).source_hash()},
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--pages-per-split", type=int, default=None,
                    help="override the split-KV geometry (default: kvq_decode_pages_per_split)")
    ap.add_argument("--append", default="pdl", choices=["pdl", "fused"],
                    help="C1-C4: append the step's new rows with K1 + PDL-launched K2 (pdl) or inside K2 "
                         "(fused: no K1 launch; 1 GPU / NCCL gather only)")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N > 1: fuse the KV-head output all-gather into K2 over peer memory (default) "
                         "or run NCCL all_gather_into_tensor after K2")
    ap.add_argument("--serving", action="store_true",
                    help="drive --layers layers per model step from the allocator + BlockTable (run_serving)")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--serving-graphs", action="store_true",
                    help="--serving: replay one CUDA graph of all layers' launches per model step")
    ap.add_argument("--table-sync", default="async", choices=["async", "legacy"])
    ap.add_argument("--kv", default=None, choices=["int8", "fp8_e4m3"],
                    help="override the config's KV dtype (the C5 INT8 vs FP8 sweep)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = dict(CONFIGS[args.config])
    if args.kv:
        cfg["kv"] = args.kv
        cfg["workload"] = cfg["workload"].replace("INT8", args.kv.upper()) + f" [{args.kv} KV]"
    if args.serving:
        run_serving(args, cfg)
    elif args.config == "c5":
        if args.impl == "reference":
            raise SystemExit("--impl reference is defined on the headline config (c2)")
        run_c5(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
