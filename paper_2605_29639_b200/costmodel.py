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


def make_servesim_cost_model(fit: DecodeFit, *, layers: int, mean_ctx_tokens: int,
                             kv_bytes_per_token: int, base_us: float = 0.0, **cost_kwargs):
    """A ``servesim.cost.CostModel`` whose ``decode_step_us`` is the measured
    B200 decode-attention time.  ``kv_bytes_per_token`` is per layer (for
    example 2,112 for Llama-3-8B with INT8 codes and fp32 scales);
    ``CostModel.kv_bytes()`` reports the whole model (× layers), as servesim
    expects."""
    from servesim.cost import CostModel, as_fraction, us_round_half_up

    @dataclass(frozen=True)
    class MeasuredCostModel(CostModel):
        layers: int = 32
        mean_ctx_tokens: int = 4352
        kv_bytes_per_token_layer: int = 2112
        launch_us: float = 0.0
        hbm_bytes_per_us: float = 6.5e6
        base_us: float = 0.0

        def decode_step_us(self, concurrent: int = 1) -> int:
            n = max(1, concurrent)
            per_layer = as_fraction(self.launch_us) + Fraction(
                n * self.mean_ctx_tokens * self.kv_bytes_per_token_layer) / as_fraction(self.hbm_bytes_per_us)
            return max(1, us_round_half_up(as_fraction(self.base_us) + self.layers * per_layer))

    return MeasuredCostModel(layers=layers, mean_ctx_tokens=mean_ctx_tokens,
                             kv_bytes_per_token_layer=kv_bytes_per_token,
                             kv_bytes_per_token=kv_bytes_per_token * layers,
                             launch_us=fit.launch_us, hbm_bytes_per_us=fit.bytes_per_us,
                             base_us=base_us, **cost_kwargs)
