"""Timing breakdown of smoothness_loss on the sorted-grid-sized planes (diagnostics)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import synthetic  # noqa: E402
from paper_2312_13299_b200.smoothness import smoothness_plane_device  # noqa: E402

side = 1024
f = synthetic.c2(0)
planes = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in synthetic.smoothness_planes(f, side).items()}
stack = plas.GridStack(plas.GridLayout(side), planes)
params = plas.SmoothnessParams()
for _ in range(3):
    plas.smoothness_loss(stack, params, return_device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    plas.smoothness_loss(stack, params, return_device=True)
torch.cuda.synchronize()
print("smoothness_loss wall ms", (time.perf_counter() - t0) * 100)
rot = planes["rotation"]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    smoothness_plane_device(rot, 0.91, params)
e1.record()
e1.synchronize()
print("rotation plane device ms", e0.elapsed_time(e1) / 10)
t0 = time.perf_counter()
for _ in range(10):
    smoothness_plane_device(rot, 0.91, params)
torch.cuda.synchronize()
print("rotation plane wall ms", (time.perf_counter() - t0) * 100)
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    plas.smoothness_loss(stack, params, return_device=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
