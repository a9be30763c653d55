"""Extended seeds of the randomised GPU sweeps in tests/test_gpu_sweep.py
(the test suite runs 6-24 seeds each; this runs hundreds to thousands).

    python tools/stress_sweeps.py
"""
import sys, time, torch
from pathlib import Path
REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO / "tests")); sys.path.insert(0, str(REPO))
import test_gpu_sweep as t
dev = torch.device("cuda:0")
t0 = time.time()
fails = []
def run(name, fn, seeds, *extra):
    n = 0
    for s in seeds:
        try:
            fn(dev, s, *extra) if not extra else fn(dev, s, *extra)
            n += 1
        except Exception as e:
            fails.append((name, s, extra, repr(e)[:300]))
    print(name, extra, "ok", n, "of", len(list(seeds)), "t=%.0fs" % (time.time() - t0), flush=True)
run("random_appends", t.test_random_appends_bit_exact, range(1000, 3000))
run("random_shapes", t.test_random_shapes, range(1000, 1800))
run("random_decode_steps", t.test_random_decode_steps, range(1000, 1400), False)
run("random_decode_steps_fused", t.test_random_decode_steps, range(1000, 1300), True)
run("random_multi_query", t.test_random_multi_query, range(1000, 1400))
run("random_verify_steps", t.test_random_verify_steps, range(1000, 1300))
print("FAILS", len(fails))
for f in fails: print(f)
