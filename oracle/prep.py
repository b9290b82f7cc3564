"""CPU restatement of the reference's caller-side feature preparation --
TEST INFRASTRUCTURE (tests/ and bench.py's reference arm only).

Follows sogs 0.1.0 splats.py:
  * prune_survivors   <- prune_to_grid, splats.py:139-152
  * normalize_columns <- normalize_for_sorting, splats.py:184-216 with
                         SplatCloud.activated, splats.py:86-93
The product computes these on the GPU (paper_2312_13299_b200/csrc/prep.cuh).
"""

import numpy as np

ORDER = ("position", "sh_dc", "sh_rest", "opacity", "scale", "rotation")
DEFAULT_WEIGHTS = {"position": 1.0, "sh_dc": 1.0, "sh_rest": 0.0, "opacity": 0.0, "scale": 1.0,
                   "rotation": 0.0}


def prune_survivors(opacity_logit, keep):
    """Indices kept by prune_to_grid: rank every Gaussian by (logit, index)
    ascending -- the order of a stable argsort (splats.py:149) -- drop the
    n - keep lowest, return the rest in index order (splats.py:150)."""
    x = np.asarray(opacity_logit, dtype=np.float64).reshape(-1)
    n = x.shape[0]
    if keep > n:
        raise ValueError("layout does not fit the cloud")
    idx = np.arange(n)
    ranked = np.lexsort((idx, x))  # primary key: logit, then index
    return np.sort(ranked[n - keep:])


def activate(name, raw):
    """SplatCloud.activated (splats.py:86-93): sigmoid for opacity, exp for scale."""
    raw = np.asarray(raw, dtype=np.float64)
    if name == "opacity":
        return 1.0 / (1.0 + np.exp(-raw))
    if name == "scale":
        return np.exp(raw)
    return raw


def normalize_columns(attrs, weights=None):
    """normalize_for_sorting: per activated channel, lo/hi over the cloud;
    column = ((v - lo) / span) * w with span = hi - lo (1 where hi <= lo, and
    those columns are then 0); weight-0 and empty attributes contribute no
    column; all-dropped -> one zero column.  Returns (features, mins, maxs)."""
    w_all = dict(DEFAULT_WEIGHTS, **(weights or {}))
    mins, maxs, cols = {}, {}, []
    n = None
    for name in ORDER:
        v = activate(name, attrs[name])
        v = v.reshape(v.shape[0], -1)
        n = v.shape[0]
        lo = np.array([v[:, c].min() for c in range(v.shape[1])], dtype=np.float64)
        hi = np.array([v[:, c].max() for c in range(v.shape[1])], dtype=np.float64)
        mins[name], maxs[name] = lo, hi
        w = w_all[name]
        if w == 0.0 or v.shape[1] == 0:
            continue
        out = np.empty_like(v)
        for c in range(v.shape[1]):
            if hi[c] > lo[c]:
                out[:, c] = ((v[:, c] - lo[c]) / (hi[c] - lo[c])) * w
            else:
                out[:, c] = 0.0
        cols.append(out)
    feats = np.concatenate(cols, axis=1) if cols else np.zeros((n, 1))
    return feats, mins, maxs


# ---- quantization
PLANE_LAYOUT = {"position": (3, 1), "sh_dc": (3, 1), "opacity": (1, 1), "scale": (3, 1), "rotation": (1, 4),
                "sh_rest": (3, 15)}  # bundle.py:25-32


def quantize_attribute_planes(name, values, levels, clip=None):
    """bundle.compress's per-attribute step (bundle.py:158-176): positions are
    contracted (quantization.py:8-11); the range per channel is the clip pair or,
    data-driven, (min, max) with max replaced by min + 1 on a constant channel
    (bundle.py:104-109); index = floor(unit (levels - 1) + 0.5) of the clamped
    affine position (quantization.py:28-41); channels sliced into images of
    PLANE_LAYOUT[name][0] samples.  Returns (planes int64 (images, n, per_image), lo, hi)."""
    v = np.asarray(values, dtype=np.float64)
    v = v.reshape(v.shape[0], -1)
    if name == "position":
        v = np.sign(v) * np.log1p(np.abs(v))
    n, C = v.shape
    if clip is None:
        lo = np.array([v[:, c].min() for c in range(C)])
        hi = np.array([v[:, c].max() for c in range(C)])
        hi = np.where(hi > lo, hi, lo + 1.0)
    else:
        lo, hi = np.full(C, float(clip[0])), np.full(C, float(clip[1]))
    idx = np.empty((n, C), dtype=np.int64)
    for c in range(C):
        x = np.minimum(np.maximum(v[:, c], lo[c]), hi[c])
        idx[:, c] = np.floor((x - lo[c]) / (hi[c] - lo[c]) * (levels - 1) + 0.5).astype(np.int64)
    per_image = PLANE_LAYOUT[name][0]
    planes = np.stack([idx[:, i * per_image:(i + 1) * per_image] for i in range(C // per_image)])
    return planes, lo, hi
