"""Replay fuzz_parity.py's case generator to case C and diagnose the first divergence."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from oracle import oracle as O  # noqa: E402

target_case = int(sys.argv[1]); seed = int(sys.argv[2])
g = np.random.default_rng(seed)
for c in range(target_case + 1):
    side = int(g.integers(2, 49)); D = int(g.integers(1, 25)); dist = g.integers(0, 4); n = side * side
    if dist == 0: f = g.normal(0, 1, (n, D))
    elif dist == 1: f = g.uniform(0, 1, (n, D))
    elif dist == 2: f = g.integers(-2, 3, (n, D)).astype(np.float64)
    else: f = g.normal(0, 1, (n, D)) * 10.0 ** g.uniform(-20, 20, (1, D))
    kw = dict(rng_seed=int(g.integers(0, 1000))); okw = dict(rng_seed=kw["rng_seed"])
    if g.random() < 0.5: kw["radius_decay"] = okw["radius_decay"] = float(g.uniform(0.5, 0.98))
    if g.random() < 0.5: kw["improvement_threshold"] = okw["improvement_threshold"] = float(10 ** g.uniform(-6, -1))
    if g.random() < 0.4: kw["min_block_size"] = okw["min_block_size"] = int(g.integers(2, 40))
    if g.random() < 0.3:
        hmax = int(math.ceil(max(side / 2.0 - 1.0, 2.0))) + 1
        r = float(g.uniform(0.5, hmax)); kw["initial_radius"] = r; okw["initial_radius_override"] = r
print("case", target_case, side, D, dist, kw)
print("channel scales", np.abs(f).max(axis=0))
perm, rep = plas.sort_grid_report(f, plas.SortConfig(**kw))
want, wrep = O.sort_grid_report(f, **okw)
print("perm equal", np.array_equal(perm, want), "reorders", rep.reorders, wrep["reorders"])
a = [(r, list(t)) for r, t in rep.radius_trace]; b = [(r, list(t)) for r, t in wrep["radius_trace"]]
for li, ((ra, ta), (rb, tb)) in enumerate(zip(a, b)):
    if ra != rb or ta != tb:
        print("first divergent level", li, "radius", ra, rb)
        for pi, (x, y) in enumerate(zip(ta, tb)):
            if x != y:
                print("  pass", pi, x, y, (x - y) / y if y else None); break
        print("  lens", len(ta), len(tb))
        break
# blur of the initial grid at the first radius
f32 = f.astype(np.float32)
ip = O.initial_perm(n, kw["rng_seed"]) if hasattr(O, "initial_perm") else None
r0 = a[0][0]
grid = f32.reshape(side, side, D)
gt = plas.blur_target(grid, r0); ot = O.blur_target(grid, r0)
print("blur equal on the raw grid", np.array_equal(gt, ot), np.argwhere(gt != ot)[:5])
print("initial/final vad", rep.initial_vad, wrep["initial_vad"], rep.final_vad, wrep["final_vad"])
