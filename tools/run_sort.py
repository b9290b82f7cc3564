"""Run sorts for profiling (ncu / compute-sanitizer) and print per-kernel CUDA-event times.

python tools/run_sort.py MODE CONFIG COUNT
MODE: device (one CUDA graph), stepped (device draws, host-stepped launches), parity
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import _lib, synthetic  # noqa: E402
from paper_2312_13299_b200.plas import SortPlan  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "device"
cfgname = sys.argv[2] if len(sys.argv) > 2 else "C2"
count = int(sys.argv[3]) if len(sys.argv) > 3 else 1
f = torch.from_numpy(synthetic.make(cfgname, 0)).cuda()
n, D = f.shape
cfg = plas.SortConfig(rng_mode="parity" if mode == "parity" else "device")
prof = None
for _ in range(count):
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    prof = _lib.SortProfile() if mode == "stepped" else None
    rep = SortPlan(n, D, cfg).run(f, perm, None, prof)
torch.cuda.synchronize()
print("passes", rep["reorders"], "levels", len(rep["radius_trace"]), "gpu_ms", round(rep["gpu_ms"], 2),
      "moved", rep["cells_moved"], "exact", rep["exact_warps"])
if prof is not None:
    for name in ("pass", "blur0", "blur1", "border", "distance", "control", "select"):
        ms, cnt = getattr(prof, f"ms_{name}"), getattr(prof, f"n_{name}")
        print(f"  {name:9s} {ms:9.3f} ms  {cnt:6d} launches  {1e3 * ms / max(cnt, 1):8.2f} us avg")
