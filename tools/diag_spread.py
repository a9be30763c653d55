"""K2 outputs of the in-page V-scale spread cases (tests/test_gpu_sweep.py
test_in_page_v_scale_spread) at three split sizes, saved with the oracle to
gpurun_out/diag_spread.npz for offline comparison with a kernel model."""
import sys
import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from test_gpu_sweep import run, requantize  # noqa: E402
from kvq_testutil import Scenario  # noqa: E402

cuda = torch.device("cuda:0")
res = {}
CASES = [(1, 16, 20, 1.0), (0, 16, 20, 1.0), (0, 16, 10, 40.0), (0, 8, -20, 40.0), (0, 4, 20, 1.0)]
if len(sys.argv) > 1:  # e.g. "0,16,10,16 0,16,0,40"
    CASES = [tuple(float(x) if i == 3 else int(x) for i, x in enumerate(a.split(","))) for a in sys.argv[1:]]
for kvd, g, spread, gain in CASES:
    sc = Scenario([700, 333, 1200, 40], 8 * g, 8, kvd, seed=30 + g)
    v = sc.v.float()
    T = v.shape[0]
    idx = torch.randperm(T, generator=torch.Generator().manual_seed(g))[: T // 16]
    v[idx] *= 2.0 ** spread
    sc.v = v.to(torch.bfloat16)
    requantize(sc)
    sc.q = (sc.q.float() * gain).to(torch.bfloat16)
    ref = sc.oracle_out()
    key = f"{kvd}_{g}_{spread}_{gain}"
    for pps in (None, 3, 1000):
        out = run(sc, cuda, pages_per_split=pps)
        err = np.abs(out - ref).max(-1) / (np.abs(ref).max(-1) + 5e-4)
        b, h = np.unravel_index(err.argmax(), err.shape)
        print(key, pps, f"max {err.max():.2e} at b={b} h={h} refmax={np.abs(ref[b, h]).max():.3e}", flush=True)
        res[f"{key}_{pps}"] = out
    res[f"{key}_ref"] = ref
np.savez("gpurun_out/diag_spread.npz", **res)
