"""§8f-1: the calibrated decode cost model, fitted to bench measurements and
plugged into the reference simulator's own CostModel seam (cost.py:62-65,
simulator.py:499-502).  The servesim part runs only where the reference is
importable (this container); the fit itself is pure host code."""
import sys
from pathlib import Path

import pytest

from paper_2605_29639_b200.costmodel import (DecodeFit, decode_step_us, fit_decode,
                                             make_servesim_cost_model, points_from_bench)


def test_fit_recovers_line():
    pts = [(b, 7.0 + b / 6.5e6) for b in (3.5e7, 1.38e9, 2.38e9, 8.86e9)]
    f = fit_decode(pts)
    assert abs(f.launch_us - 7.0) < 1e-6 and abs(f.bytes_per_us - 6.5e6) / 6.5e6 < 1e-9
    assert fit_decode([(1e9, 200.0)]).bytes_per_us == 5e6


def test_points_from_bench_lines():
    line = {"roofline": {"algorithmic_bytes_per_launch": 2380465480, "avg_launch_ms": 0.3628}}
    assert points_from_bench([line, {"roofline": {}}]) == [(2380465480.0, 362.8)]


def test_decode_step_scales_with_context_and_batch():
    f = DecodeFit(launch_us=5.0, bytes_per_us=6.5e6, points=3)
    t1 = decode_step_us(f, 1, 4352, 2112, layers=32)
    t256 = decode_step_us(f, 256, 4352, 2112, layers=32)
    assert t1 == pytest.approx(32 * (5 + 4352 * 2112 / 6.5e6))
    assert t256 > 100 * t1 / 2


def _servesim():
    try:
        import servesim  # noqa: F401
        return True
    except ImportError:
        p = Path("/root/reference/pkg/src")
        if p.exists():
            sys.path.insert(0, str(p))
            return True
    return False


@pytest.mark.skipif(not _servesim(), reason="reference simulator not available")
def test_plugs_into_servesim_simulation():
    from servesim.config import SimConfig
    from servesim.cost import CostModel
    from servesim.simulator import run
    from servesim.workload import synth_trace

    f = DecodeFit(launch_us=6.0, bytes_per_us=6.5e6, points=4)
    cm = make_servesim_cost_model(f, layers=32, mean_ctx_tokens=4352, kv_bytes_per_token=2112)
    assert isinstance(cm, CostModel)
    assert cm.kv_bytes(10) == 10 * 2112 * 32
    assert cm.decode_step_us(1) == round(32 * (6.0 + 4352 * 2112 / 6.5e6))
    trace = synth_trace("qa", 20, seed=1)
    base = run(trace, SimConfig(), seed=1)
    meas = run(trace, SimConfig(cost=cm), seed=1)
    # the calibrated B200 step (~1.5 ms for 32 layers at 4K ctx) is far below the 10 ms constant
    assert meas.to_dict()["decode_span_mean_us"] < base.to_dict()["decode_span_mean_us"]
    assert meas.to_dict()["tokens_per_sec"] > base.to_dict()["tokens_per_sec"]


def test_scoring_passes_and_factors():
    from paper_2605_29639_b200.costmodel import append_bytes_per_token, mq_factor, scoring_passes
    assert scoring_passes(4, 1) == [4] and scoring_passes(4, 4) == [16]
    assert scoring_passes(4, 9) == [16, 16, 4]          # k = 8 draft tokens at g = 4: three passes
    assert scoring_passes(16, 2) == [16, 16]
    assert (mq_factor(4), mq_factor(8), mq_factor(16)) == (1.0, 1.02, 1.24)
    assert append_bytes_per_token(8) == 8 * 776 + 4


@pytest.mark.skipif(not _servesim(), reason="reference simulator not available")
def test_spec_scoring_and_prefill_append_in_servesim():
    """With speculative decoding on, the simulator charges spec_iteration_us
    (simulator.py:499-502): priced here as multi-query K2 passes instead of
    the constant spec_score_us; prefill_us gains the K1 append of every
    computed token in every layer."""
    from servesim.config import SimConfig, SpecSettings
    from servesim.cost import CostModel
    from servesim.simulator import run
    from servesim.workload import synth_trace

    f = DecodeFit(launch_us=6.0, bytes_per_us=6.5e6, points=4)
    kw = dict(layers=32, mean_ctx_tokens=4352, kv_bytes_per_token=2112, heads_per_kv=4, num_kv_heads=8)
    cm = make_servesim_cost_model(f, spec_q_len=4, append_bytes_per_us=2.8e6, append_launch_us=3.0, **kw)
    plain = make_servesim_cost_model(f, **kw)
    dec = cm.decode_step_us(8)
    assert cm.spec_iteration_us(8) == round(cm.spec_draft_us + 32 * (6.0 + 8 * 4352 * 2112 / 6.5e6 * 1.24))
    assert dec < cm.spec_iteration_us(8) < CostModel().spec_iteration_us(8)
    assert plain.spec_iteration_us(8) == CostModel().spec_iteration_us(8)   # spec_q_len 0: the reference's
    assert cm.prefill_us(2048) == CostModel().prefill_us(2048) + round(32 * (3.0 + 2048 * 6212 / 2.8e6))
    assert plain.prefill_us(2048) == CostModel().prefill_us(2048)
    trace = synth_trace("qa", 20, seed=1)
    spec = SpecSettings(enabled=True, k=3)
    base = run(trace, SimConfig(speculative=spec), seed=1).to_dict()
    meas = run(trace, SimConfig(cost=cm, speculative=spec), seed=1).to_dict()
    assert meas["decode_span_mean_us"] < base["decode_span_mean_us"]
    assert meas["tokens_per_sec"] > base["tokens_per_sec"]
