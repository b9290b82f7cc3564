"""Replay fuzz_parity.py cases and dump inputs + GPU results (for a comparison
with the real reference in a container that has it)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def cases(seed, upto, smin=2, smax=48):
    g = np.random.default_rng(seed)
    for c in range(upto + 1):
        side = int(g.integers(smin, smax + 1)); D = int(g.integers(1, 25)); dist = g.integers(0, 4); n = side * side
        if dist == 0: f = g.normal(0, 1, (n, D))
        elif dist == 1: f = g.uniform(0, 1, (n, D))
        elif dist == 2: f = g.integers(-2, 3, (n, D)).astype(np.float64)
        else: f = g.normal(0, 1, (n, D)) * 10.0 ** g.uniform(-20, 20, (1, D))
        kw = dict(rng_seed=int(g.integers(0, 1000)))
        if g.random() < 0.5: kw["radius_decay"] = float(g.uniform(0.5, 0.98))
        if g.random() < 0.5: kw["improvement_threshold"] = float(10 ** g.uniform(-6, -1))
        if g.random() < 0.4: kw["min_block_size"] = int(g.integers(2, 40))
        if g.random() < 0.3:
            hmax = int(math.ceil(max(side / 2.0 - 1.0, 2.0))) + 1
            kw["initial_radius"] = float(g.uniform(0.5, hmax))
        yield c, f, kw


if __name__ == "__main__":
    import paper_2312_13299_b200 as plas
    seed = int(sys.argv[1]); want = [int(x) for x in sys.argv[2].split(",")]; out = sys.argv[3]
    arrs = {}
    for c, f, kw in cases(seed, max(want)):
        if c not in want:
            continue
        perm, rep = plas.sort_grid_report(f, plas.SortConfig(**kw))
        arrs[f"f{c}"] = f
        arrs[f"perm{c}"] = perm
        arrs[f"trace{c}"] = np.array([v for _, t in rep.radius_trace for v in t])
        arrs[f"vad{c}"] = np.array([rep.initial_vad, rep.final_vad])
        arrs[f"reorders{c}"] = np.array([rep.reorders])
    np.savez(out, **arrs)
    print("dumped", sorted(arrs))
