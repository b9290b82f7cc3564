"""Randomised long-line check of the sort's blur tiers (direct fold and FFT at
the long lengths 1024..6144, both axes, odd channel counts, every value
distribution of fuzz_api) against the oracle's SciPy fold.
usage: python tools/fuzz_blur_long.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2312_13299_b200 import blur as gblur  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)


def values(shape):
    kind = int(g.integers(0, 5))
    if kind == 0:
        return g.normal(0, 1, shape)
    if kind == 1:
        return g.uniform(0, 1, shape)
    if kind == 2:
        return g.normal(0, 1, shape) * 10.0 ** g.uniform(-20, 20, (1, 1, shape[-1]))
    if kind == 3:
        v = g.normal(0, 1, shape)
        return v - v.mean(axis=(0, 1), keepdims=True)  # zero-mean: outputs near zero
    return g.integers(-3, 4, shape).astype(np.float64)


bad = 0
for c in range(cases):
    long_n = int(g.integers(1000, 4097))
    short_n = int(g.integers(2, 9))
    H, W = (long_n, short_n) if g.random() < 0.5 else (short_n, long_n)
    C = int(g.integers(1, 6))
    r = float(g.uniform(1.0, 0.5 * long_n))
    tier = int(g.integers(0, 2))
    x = values((H, W, C)).astype(np.float32)
    try:
        got, fb = gblur.blur_target_tiers(x, r, tier)
        ok = np.array_equal(got, O.blur_target(x, r))
    except Exception as e:  # noqa: BLE001
        ok, fb = False, repr(e)[:200]
    if not ok:
        bad += 1
        print(f"MISMATCH {c}: {H}x{W}x{C} r={r:.3f} tier={tier} fb={fb}")
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
