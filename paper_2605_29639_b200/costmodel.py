"""Calibrated decode cost model.

The reference prices a decode step with one constant:
``CostModel.decode_step_us(n) = decode_us_per_token * (1 + coeff * (n - 1))``
(``pkg/src/servesim/cost.py:62-65``).  The default is 10 ms whatever the
context length, head count, KV dtype or page layout.  This module replaces
that constant with the bytes-based time the B200 kernels actually achieve:

    t_layer(n, ctx) = launch_us + n * ctx * kv_bytes_per_token / bw
    decode_step_us(n) = base_us + layers * t_layer(n, mean_ctx)

Here ``kv_bytes_per_token`` is the quantized footprint of one layer: codes
plus fp32 scales, i.e. ``KVCacheSpec.kv_bytes_per_token``. ``launch_us`` and
``bw`` are fitted to ``bench.py`` measurements.

Two more reference seams are priced from the same kernels:

* ``spec_iteration_us`` (``cost.py:67-71``, charged at ``simulator.py:499-502``
  when speculative decoding is on): the scoring forward is the multi-query
  K2 (``kvq_decode_attn_mq``, q_len = k + 1 tokens per sequence).  It streams
  the KV once per pass of <= 16 query rows per kv head and costs a measured
  factor over a decode step (1.02x at 8 rows, 1.24x at 16 on
  the C2 shape), instead of the constant ``spec_score_us`` = 10 ms.
* ``prefill_us`` (``cost.py:51-60``, ``simulator.py:404-406``): the reference's
  affine prefill model stays (its GEMM/attention work is not this path), plus
  the quantize-on-append (K1) of every computed token in every layer at the
  measured K1 rate (``bench.py --config c5`` ``append_gbs``).

``make_servesim_cost_model`` builds a subclass of the reference's
``CostModel``, so a servesim config can use it unchanged
(``SimConfig.cost``, ``config.py:188-220``; consumed at
``simulator.py:499-502``).  servesim is imported only when that function is
called, so the package never depends on the reference at run time.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, List, Sequence, Tuple


@dataclass(frozen=True)
class DecodeFit:
    launch_us: float          # per-layer fixed cost (launches, prologue, tail)
    bytes_per_us: float       # effective KV streaming rate
    points: int

    def layer_us(self, kv_bytes: float) -> float:
        return self.launch_us + kv_bytes / self.bytes_per_us


def fit_decode(points: Sequence[Tuple[float, float]]) -> DecodeFit:
    """Least-squares fit of ``t_us = launch_us + bytes / bw`` to
    ``(algorithmic_bytes, t_us)`` points.  With a single point the launch term
    is taken as 0."""
    pts = [(float(b), float(t)) for b, t in points]
    if not pts:
        raise ValueError("need at least one measurement")
    if len(pts) == 1:
        b, t = pts[0]
        return DecodeFit(0.0, b / t, 1)
    n = len(pts)
    mb = sum(b for b, _ in pts) / n
    mt = sum(t for _, t in pts) / n
    sbb = sum((b - mb) ** 2 for b, _ in pts)
    sbt = sum((b - mb) * (t - mt) for b, t in pts)
    if sbb <= 0 or sbt <= 0:
        raise ValueError("degenerate measurements")
    slope = sbt / sbb                     # us per byte
    launch = max(0.0, mt - slope * mb)
    return DecodeFit(launch, 1.0 / slope, n)


def points_from_bench(lines: Iterable[dict]) -> List[Tuple[float, float]]:
    """(algorithmic bytes, K2 microseconds) from ``bench.py`` JSON lines."""
    out = []
    for d in lines:
        r = d.get("roofline") or {}
        if "algorithmic_bytes_per_launch" in r and r.get("avg_launch_ms"):
            out.append((float(r["algorithmic_bytes_per_launch"]), float(r["avg_launch_ms"]) * 1e3))
    return out


def decode_step_us(fit: DecodeFit, concurrent: int, mean_ctx: int, kv_bytes_per_token: int,
                   layers: int, base_us: float = 0.0) -> float:
    n = max(1, concurrent)
    return base_us + layers * fit.layer_us(n * mean_ctx * kv_bytes_per_token)


# Multi-query K2 time over a decode step's, by query rows per kv head in one
# pass (tools/bench_widened.py on the C2 shape: q_len 1 / 2 / 4
# at g = 4 -> 4 / 8 / 16 rows: 0.346 / 0.353 / 0.429 ms).
MQ_FACTOR = ((4, 1.0), (8, 1.02), (16, 1.24))
MAX_ROWS = 16   # kernel limit: (Hq / Hkv) * q_len <= 16 query rows per launch


def scoring_passes(heads_per_kv: int, q_len: int) -> List[int]:
    """Query rows per kv head of each multi-query launch that scores q_len
    tokens (the draft tokens are split across launches of <= 16 rows)."""
    if heads_per_kv > MAX_ROWS:
        raise ValueError("more than 16 query heads per kv head")
    per = MAX_ROWS // max(1, heads_per_kv)
    out, left = [], q_len
    while left > 0:
        t = min(per, left)
        out.append(t * heads_per_kv)
        left -= t
    return out


def mq_factor(rows: int) -> float:
    for limit, f in MQ_FACTOR:
        if rows <= limit:
            return f
    raise ValueError("more than 16 query rows per kv head in one launch")


def append_bytes_per_token(num_kv_heads: int) -> int:
    """K1's algorithmic bytes per appended token per layer: bf16 K and V read,
    codes + fp32 scales written, the slot read."""
    return num_kv_heads * (2 * 128 * 2 + 2 * 128 + 2 * 4) + 4


def make_servesim_cost_model(fit: DecodeFit, *, layers: int, mean_ctx_tokens: int,
                             kv_bytes_per_token: int, base_us: float = 0.0, heads_per_kv: int = 4,
                             num_kv_heads: int = 8, spec_q_len: int = 0, append_launch_us: float = 0.0,
                             append_bytes_per_us: float = 0.0, **cost_kwargs):
    """A ``servesim.cost.CostModel`` whose ``decode_step_us`` is the measured
    B200 decode-attention time.  ``kv_bytes_per_token`` is per layer (for
    example 2,112 for Llama-3-8B with INT8 codes and fp32 scales);
    ``CostModel.kv_bytes()`` reports the whole model (× layers), as servesim
    expects.

    ``spec_q_len`` (the speculative k + 1; 0 leaves ``spec_iteration_us`` to
    the reference) prices the scoring forward as multi-query K2 passes;
    ``append_bytes_per_us`` > 0 (the measured K1 rate) adds the quantize-on-
    append of every prefilled token to ``prefill_us``."""
    from servesim.cost import CostModel, as_fraction, us_round_half_up

    @dataclass(frozen=True)
    class MeasuredCostModel(CostModel):
        layers: int = 32
        mean_ctx_tokens: int = 4352
        kv_bytes_per_token_layer: int = 2112
        launch_us: float = 0.0
        hbm_bytes_per_us: float = 6.5e6
        base_us: float = 0.0
        heads_per_kv: int = 4
        num_kv_heads: int = 8
        spec_q_len: int = 0
        append_launch_us: float = 0.0
        append_bytes_per_us: float = 0.0

        def _layer_stream(self, n: int) -> Fraction:
            return Fraction(n * self.mean_ctx_tokens * self.kv_bytes_per_token_layer) / as_fraction(
                self.hbm_bytes_per_us)

        def decode_step_us(self, concurrent: int = 1) -> int:
            n = max(1, concurrent)
            per_layer = as_fraction(self.launch_us) + self._layer_stream(n)
            return max(1, us_round_half_up(as_fraction(self.base_us) + self.layers * per_layer))

        def spec_iteration_us(self, concurrent: int = 1) -> int:
            if self.spec_q_len <= 0:
                return super().spec_iteration_us(concurrent)
            n = max(1, concurrent)
            per_layer = sum(as_fraction(self.launch_us) + self._layer_stream(n) * as_fraction(mq_factor(rows))
                            for rows in scoring_passes(self.heads_per_kv, self.spec_q_len))
            return max(1, us_round_half_up(Fraction(self.spec_draft_us) + as_fraction(self.base_us) +
                                           self.layers * per_layer))

        def prefill_us(self, seq_tokens: int, batch_tokens: int = 0) -> int:
            base = super().prefill_us(seq_tokens, batch_tokens)
            if self.append_bytes_per_us <= 0 or seq_tokens <= 0:
                return base
            k1 = as_fraction(self.append_launch_us) + Fraction(
                seq_tokens * append_bytes_per_token(self.num_kv_heads)) / as_fraction(self.append_bytes_per_us)
            return base + us_round_half_up(self.layers * k1)

    return MeasuredCostModel(layers=layers, mean_ctx_tokens=mean_ctx_tokens,
                             kv_bytes_per_token_layer=kv_bytes_per_token,
                             kv_bytes_per_token=kv_bytes_per_token * layers,
                             launch_us=fit.launch_us, hbm_bytes_per_us=fit.bytes_per_us,
                             base_us=base_us, heads_per_kv=heads_per_kv, num_kv_heads=num_kv_heads,
                             spec_q_len=spec_q_len, append_launch_us=append_launch_us,
                             append_bytes_per_us=append_bytes_per_us, **cost_kwargs)
