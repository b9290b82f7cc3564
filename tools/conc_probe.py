"""Concurrent sorts from host threads (diagnostics for test_concurrent_sorts_from_threads).

python tools/conc_probe.py MODE REPEATS   MODE: device | parity | mixed
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2312_13299_b200 as plas  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "mixed"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = np.random.default_rng(21)
shapes = [(48, 3), (64, 4), (48, 3), (32, 6), (64, 4), (40, 2)]
feats = [g.uniform(size=(s * s, d)).astype(np.float32) for s, d in shapes]
rm = {"device": lambda i: "device", "parity": lambda i: "parity", "mixed": lambda i: "device" if i % 2 else "parity"}[mode]
cfgs = [plas.SortConfig(rng_seed=i, rng_mode=rm(i)) for i in range(len(shapes))]
alone = [plas.sort_grid(f, c) for f, c in zip(feats, cfgs)]
out = [None] * len(shapes)
errs = []


def run(i):
    try:
        with torch.cuda.stream(torch.cuda.Stream()):
            for _ in range(reps):
                out[i] = plas.sort_grid(feats[i], cfgs[i])
                if not np.array_equal(out[i], alone[i]):
                    errs.append(f"thread {i}: result differs")
    except Exception as exc:
        errs.append(f"thread {i}: {exc}")


threads = [threading.Thread(target=run, args=(i,)) for i in range(len(shapes))]
for t in threads:
    t.start()
for t in threads:
    t.join()
print(mode, "OK" if not errs else "FAIL " + " | ".join(errs[:3]))
