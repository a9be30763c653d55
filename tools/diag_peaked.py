"""Per-row error of the adversarial peaked-softmax case (tests/test_gpu_sweep.py)
for both formats, gains 8 / 40 and three split sizes; saves outputs + oracle
to gpurun_out/diag_peaked.npz for offline comparison with a kernel model."""
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
for kvd in (O.INT8, O.FP8_E4M3):
    for gain in (8.0, 40.0):
        sc = Scenario([1800, 700, 64, 2500], 32, 8, kvd, seed=77)
        T = sc.k.shape[0]
        idx = torch.randperm(T, generator=torch.Generator().manual_seed(5))
        k, v = sc.k.float(), sc.v.float()
        k[idx[:40]] = 0.0
        v[idx[40:80]] = 0.0
        k[idx[80:100]] *= 2.0 ** 100
        v[idx[100:120]] *= 2.0 ** 6
        v[idx[120:140]] *= 2.0 ** -100
        sc.k, sc.v = k.to(torch.bfloat16), v.to(torch.bfloat16)
        requantize(sc)
        sc.q = (sc.q.float() * gain).to(torch.bfloat16)
        ref = sc.oracle_out()
        for pps in (None, 3, 1000):
            out = run(sc, cuda, pages_per_split=pps)
            err = np.abs(out - ref).max(-1) / (np.abs(ref).max(-1) + 5e-4)
            b, h = np.unravel_index(err.argmax(), err.shape)
            print(kvd, gain, pps, f"max {err.max():.2e} at b={b} h={h} refmax={np.abs(ref[b, h]).max():.3e}",
                  flush=True)
            res[f"{kvd}_{gain}_{pps}"] = out
        res[f"{kvd}_{gain}_ref"] = ref
np.savez("gpurun_out/diag_peaked.npz", **res)
