"""Summarise PLAS_LEVEL_TRACE=1 stderr of a stepped sort: K3 launch time per regime
(tile regime = levels whose beta puts the block in shared memory)."""
import re, sys
tile_beta = int(sys.argv[2]) if len(sys.argv) > 2 else 16
agg = {}
for line in open(sys.argv[1]):
    m = re.search(r"beta\s+(\d+).*passes\s+(\d+) pass\s+([\d.]+) us", line)
    if not m:
        continue
    beta, n, us = int(m.group(1)), int(m.group(2)), float(m.group(3))
    key = "tile" if beta <= tile_beta else ("gather<=64" if beta <= 64 else "gather>64")
    a = agg.setdefault(key, [0, 0.0])
    a[0] += n
    a[1] += n * us
for k, (n, t) in sorted(agg.items()):
    print(f"{k:12s} passes {n:5d}  avg {t / max(n, 1):7.2f} us  total {t / 1e3:7.2f} ms")
