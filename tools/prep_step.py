"""One feature-prep step (bench.py run_prep) for profiling: python tools/prep_step.py [reps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2312_13299_b200 import splats as ps

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n, side = 1_100_000, 1024
g = np.random.default_rng(0)
cl = {"positions": g.normal(0, 3, (n, 3)), "sh_dc": g.normal(0, 0.5, (n, 3)), "sh_rest": g.normal(0, 0.1, (n, 45)),
      "opacity_logit": g.normal(0, 2, n), "scale_log": g.normal(-4, 1, (n, 3)), "rotation": g.normal(0, 1, (n, 4))}
fields = tuple(cl)
dev = {f: torch.from_numpy(np.ascontiguousarray(v)).cuda() for f, v in cl.items()}
keep = side * side
perm = torch.from_numpy(np.random.default_rng(1).permutation(keep)).cuda()
attr_of = dict(zip(ps.ATTRIBUTES, fields))
for _ in range(reps):
    surv = ps.prune_indices(dev["opacity_logit"], keep)
    pr = {f: ps.gather_rows(dev[f], surv) for f in fields}
    feats, _, _ = ps.normalize_features({a: pr[f] for a, f in attr_of.items()})
    applied = {f: ps.gather_rows(pr[f], perm) for f in fields}
torch.cuda.synchronize()
print("ok", feats.shape)
