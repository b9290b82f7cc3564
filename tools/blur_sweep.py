"""Time the sort's level-blur tiers (plas_blur_target_tiers) on an HxWxC grid
across radii: python tools/blur_sweep.py 1024x1024x14 [tiers=0,1] [radii...]"""
import math, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2312_13299_b200 import _lib
from paper_2312_13299_b200.blur import gaussian_weights

shape = tuple(int(x) for x in sys.argv[1].split("x"))
tiers = [int(t) for t in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
radii = [float(r) for r in sys.argv[3:]] or [2, 4, 8, 16, 24, 32, 48, 63, 64, 96, 128, 200, 300, 500]
H, W, C = shape
L = _lib.lib()
g = torch.randn(H, W, C, device="cuda", dtype=torch.float32)
out = torch.empty_like(g)
fb = np.zeros(2, dtype=np.int64)
for r in radii:
    h = int(math.ceil(r))
    w = gaussian_weights(r / 2.0, h)
    ws = _lib.workspace(L.plas_blur_tiers_workspace_bytes(H, W, C, h), "tiers")
    row = [f"r={r:6.1f} h={h:4d}"]
    for t in tiers:
        if t == 2 and h > 16:
            continue
        def call():
            _lib.check(L.plas_blur_target_tiers(_lib.ptr(g), _lib.ptr(out), H, W, C, _lib.ptr(w), h, t,
                                                _lib.ptr(fb), _lib.ptr(ws), ws.numel(), _lib.stream_handle()), "tiers")
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            call()
        e1.record()
        torch.cuda.synchronize()
        row.append(f"tier{t} {e0.elapsed_time(e1) / n * 1000:8.1f} us fb={fb[0]}+{fb[1]}")
    print("  ".join(row), flush=True)
