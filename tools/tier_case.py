import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2312_13299_b200 import blur as gblur
from oracle import oracle as O
shape = tuple(int(x) for x in sys.argv[1].split("x")); r = float(sys.argv[2])
g = np.random.default_rng(17).normal(0, 1, shape).astype(np.float32)
t = time.time()
got, fb = gblur.blur_target_tiers(g, r, 1)
print(shape, r, "fb", fb, "ok" if np.array_equal(got, O.blur_target(g, r)) else "MISMATCH", round(time.time() - t, 2), flush=True)
