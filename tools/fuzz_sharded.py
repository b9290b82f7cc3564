"""Randomised check of the multi-GPU protocol on one device (sharded.EmulatedGroup:
world ranks as host threads with copy-based collectives, no kernel waits on
another): every rank's permutation, pass count and trace must equal the 1-GPU
sort, in PARITY and DEVICE mode, over random shapes / configs.
usage: python tools/fuzz_sharded.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import sharded  # noqa: E402
from tools.fuzz_dump import cases as gen  # noqa: E402

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = np.random.default_rng(seed + 1000)
bad = 0
done = 0
for c, f, kw in gen(seed, 10 * ncases):
    if done >= ncases:
        break
    if f.shape[0] < 64:  # at least 8 x 8: a band per rank
        continue
    done += 1
    kw["rng_mode"] = "device" if g.random() < 0.5 else "parity"
    world = int(g.integers(2, 5))
    cfg = plas.SortConfig(**kw)
    t = torch.from_numpy(f).cuda()
    try:
        # sharded PARITY sorts decide on the exact fixed-point statistic (the
        # NumPy-order one needs every cell on one GPU): compare with the 1-GPU
        # sort on the same statistic
        if kw["rng_mode"] == "parity":
            os.environ["PLAS_NP_STATS"] = "0"
        p1, r1 = plas.sort_on_device(t, cfg)
        os.environ.pop("PLAS_NP_STATS", None)
        p1 = p1.cpu().numpy()
        tr1 = [v for _, tt in r1["radius_trace"] for v in tt]
        ok = True
        for pr, rep in sharded.sort_emulated(t, cfg, world):
            ok &= np.array_equal(pr, p1) and rep["reorders"] == r1["reorders"] and \
                [v for _, tt in rep["radius_trace"] for v in tt] == tr1
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", repr(e)[:200])
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: n={f.shape[0]} D={f.shape[1]} world={world} kw={kw}")
print(f"{done} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
