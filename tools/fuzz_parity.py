"""Randomised PARITY-vs-oracle sweep over small shapes and SortConfig values
(side 2..48, D 1..24, decay, threshold, min block, start radius, value
distributions).  Prints every mismatch; exit status 1 if any.
usage: python tools/fuzz_parity.py [cases] [seed] [side_min] [side_max]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
SMIN = int(sys.argv[3]) if len(sys.argv) > 3 else 2    # side range (defaults: 2 .. 48)
SMAX = int(sys.argv[4]) if len(sys.argv) > 4 else 48
bad = 0
for c in range(cases):
    side = int(g.integers(SMIN, SMAX + 1))
    D = int(g.integers(1, 25))
    dist = g.integers(0, 4)
    n = side * side
    if dist == 0:
        f = g.normal(0, 1, (n, D))
    elif dist == 1:
        f = g.uniform(0, 1, (n, D))
    elif dist == 2:
        f = g.integers(-2, 3, (n, D)).astype(np.float64)
    else:
        f = g.normal(0, 1, (n, D)) * 10.0 ** g.uniform(-20, 20, (1, D))
    kw = dict(rng_seed=int(g.integers(0, 1000)))
    okw = dict(rng_seed=kw["rng_seed"])
    if g.random() < 0.5:
        kw["radius_decay"] = okw["radius_decay"] = float(g.uniform(0.5, 0.98))
    if g.random() < 0.5:
        kw["improvement_threshold"] = okw["improvement_threshold"] = float(10 ** g.uniform(-6, -1))
    if g.random() < 0.4:
        kw["min_block_size"] = okw["min_block_size"] = int(g.integers(2, 40))
    if g.random() < 0.3:
        hmax = int(math.ceil(max(side / 2.0 - 1.0, 2.0))) + 1
        r = float(g.uniform(0.5, hmax))
        kw["initial_radius"] = r
        okw["initial_radius_override"] = r
    try:
        perm, rep = plas.sort_grid_report(f, plas.SortConfig(**kw))
        want, wrep = O.sort_grid_report(f, **okw)
        ok = (np.array_equal(perm, want) and rep.reorders == wrep["reorders"]
              and [v for _, t in rep.radius_trace for v in t] == [v for _, t in wrep["radius_trace"] for v in t])
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", repr(e)[:200])
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: side={side} D={D} dist={dist} kw={kw}")
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
