"""Warm-start re-sorts for a training loop (not in the reference).

After a densification / pruning step the attribute set changes a little; the
previous permutation is then a good start.  This measures, on the C2 workload
(1024^2 x 14, DEVICE mode): a cold sort, a simulated densification (a fraction
`--churn` of the rows replaced by fresh draws of the same generator, the rest
kept), then the re-sort cold (reference schedule) and warm (initial_perm =
the previous permutation, start radius r0 / k for several k).  Reports device
sort time, passes and the neighbour-L2 smoothness of each result.

usage: python tools/warm_start.py [--churn 0.05] [--out profiles/r02_warm_start.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import synthetic  # noqa: E402


def run(feat, cfg, initial_perm=None):
    torch.cuda.synchronize()
    perm, rep = plas.sort_on_device(feat, cfg, initial_perm=initial_perm)
    torch.cuda.synchronize()
    side = int(round(feat.shape[0] ** 0.5))
    grid = feat[perm].reshape(side, side, -1).cpu().numpy()
    return perm, {"gpu_ms": round(rep["gpu_ms"], 2), "passes": int(rep["reorders"]),
                  "levels": len(rep["radius_trace"]), "nbr_l2": synthetic.neighbour_l2(grid)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--churn", type=float, default=0.05)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    side = 1024
    f0 = synthetic.c2(0, side)
    fresh = synthetic.c2(1, side)  # the same generator, another seed: "new" Gaussians
    rng = np.random.default_rng(11)
    n = side * side
    swap = rng.choice(n, int(a.churn * n), replace=False)
    f1 = f0.copy()
    f1[swap] = fresh[swap]
    d0 = torch.from_numpy(f0).cuda()
    d1 = torch.from_numpy(f1).cuda()
    base = dict(rng_seed=0, rng_mode="device")
    run(d0, plas.SortConfig(**base))  # warm-up (graph instantiation)
    perm0, cold0 = run(d0, plas.SortConfig(**base))
    r0 = plas.initial_radius(side)
    rows = {"first sort (cold)": cold0}
    _, rows["re-sort cold"] = run(d1, plas.SortConfig(**base))
    prev = perm0.cpu().numpy()
    _, rows["no re-sort (previous perm)"] = (None, {"gpu_ms": 0.0, "passes": 0, "levels": 0, "nbr_l2": synthetic.neighbour_l2(
        f1[prev].reshape(side, side, -1))})
    for k in (2, 4, 8, 16, 32):
        cfg = plas.SortConfig(initial_radius=r0 / k, **base)
        run(d1, cfg, initial_perm=prev)  # warm-up of this schedule's graph
        _, rows[f"re-sort warm, r0/{k}"] = run(d1, cfg, initial_perm=prev)
    res = {"what": "C2 1024^2 x 14, DEVICE mode, one B200: re-sort after replacing "
                   f"{a.churn:.0%} of the rows (synthetic.c2 seed 1 rows) -- cold vs warm start "
                   "(initial_perm = previous permutation, smaller start radius)",
           "churn": a.churn, "r0": r0, "rows": rows}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
