"""Randomised DEVICE-mode checks (no reference value exists for the device
draws): valid permutation, run-to-run determinism, and the CUDA-graph run equal
to the host-stepped run of the same kernels, over random shapes / configs /
value ranges.  usage: python tools/fuzz_device.py [cases] [seed] [side_min] [side_max]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import _lib  # noqa: E402
from paper_2312_13299_b200.plas import SortPlan  # noqa: E402
from tools.fuzz_dump import cases as gen  # noqa: E402

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
smin = int(sys.argv[3]) if len(sys.argv) > 3 else 2
smax = int(sys.argv[4]) if len(sys.argv) > 4 else 48
bad = 0
for c, f, kw in gen(seed, ncases - 1, smin, smax):
    kw["rng_mode"] = "device"
    n, D = f.shape
    cfg = plas.SortConfig(**kw)
    t = torch.from_numpy(f).cuda()
    outs = []
    try:
        for prof in (None, None, _lib.SortProfile()):
            perm = torch.empty(n, dtype=torch.int64, device="cuda")
            rep = SortPlan(n, D, cfg).run(t, perm, None, prof)
            outs.append((perm.cpu().numpy(), rep["reorders"], [v for _, tr in rep["radius_trace"] for v in tr]))
        p0 = outs[0][0]
        ok = np.array_equal(np.sort(p0), np.arange(n)) and all(
            np.array_equal(p0, o[0]) and outs[0][1] == o[1] and outs[0][2] == o[2] for o in outs[1:])
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", repr(e)[:200])
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: n={n} D={D} kw={kw}")
print(f"{ncases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
