"""Data model at the sort boundary and the caller-side feature preparation on the GPU.

Mirrors the reference's ``sogs.splats`` (splats.py): ``SplatCloud``,
``GridLayout``, ``build_grid_layout``, ``GridStack``, ``NormalizationSpec``,
``prune_to_grid`` and ``normalize_for_sorting``, plus the
device-resident forms the GPU pipeline uses (``prune_indices``,
``normalize_features``, ``gather_rows``).  The selection, the activated-value
min/max and the affine map run in CUDA kernels (csrc/prep.cuh) behind
``plas_prune_to_grid`` / ``plas_normalize_for_sorting`` / ``plas_gather_rows``.
"""

import math
from dataclasses import dataclass, field

import numpy as np

ATTRIBUTES = ("position", "sh_dc", "sh_rest", "opacity", "scale", "rotation")

# channel counts of the fixed-size attributes; sh_rest has 0 or 45 (splats.py:12-15)
CHANNELS = {"position": 3, "sh_dc": 3, "opacity": 1, "scale": 3, "rotation": 4}
SH_REST_SIZES = (0, 45)

# activation as the renderer sees the attribute (splats.py:86-93): 1 sigmoid, 2 exp
ACTIVATION = {"position": 0, "sh_dc": 0, "sh_rest": 0, "opacity": 1, "scale": 2, "rotation": 0}

# Default per-attribute sorting weights (splats.py:17-24); SortConfig default.
DEFAULT_SORT_WEIGHTS = {
    "position": 1.0,
    "sh_dc": 1.0,
    "sh_rest": 0.0,
    "opacity": 0.0,
    "scale": 1.0,
    "rotation": 0.0,
}


@dataclass(frozen=True)
class GridLayout:
    side: int

    def __post_init__(self):
        if self.side < 1:
            raise ValueError("grid side must be positive")

    @property
    def cells(self):
        return self.side * self.side


@dataclass(frozen=True)
class GridStack:
    """Per-attribute 2D planes sharing one permutation; one cell per Gaussian."""

    layout: GridLayout
    planes: dict = field(default_factory=dict)

    def __post_init__(self):
        side = self.layout.side
        for name, plane in self.planes.items():
            if name not in ATTRIBUTES:
                raise ValueError(f"unknown attribute {name!r}")
            if tuple(plane.shape[:2]) != (side, side):
                raise ValueError(f"plane {name!r} is {tuple(plane.shape[:2])}, expected {(side, side)}")


def sigmoid(x):
    """splats.py:27-28 (host, fp64)."""
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


@dataclass(frozen=True)
class SplatCloud:
    """splats.py:31-104: un-activated Gaussian parameters, validated and held as fp64."""

    positions: np.ndarray
    sh_dc: np.ndarray
    sh_rest: np.ndarray
    opacity_logit: np.ndarray
    scale_log: np.ndarray
    rotation: np.ndarray

    def __post_init__(self):
        pos = np.atleast_2d(np.asarray(self.positions, dtype=np.float64))
        n = pos.shape[0]
        if n < 1:
            raise ValueError("a SplatCloud needs at least one Gaussian")
        arrays = {
            "positions": (pos, (n, 3)),
            "sh_dc": (np.asarray(self.sh_dc, dtype=np.float64), (n, 3)),
            "sh_rest": (np.asarray(self.sh_rest, dtype=np.float64).reshape(n, -1), None),
            "opacity_logit": (np.asarray(self.opacity_logit, dtype=np.float64).reshape(-1), (n,)),
            "scale_log": (np.asarray(self.scale_log, dtype=np.float64), (n, 3)),
            "rotation": (np.asarray(self.rotation, dtype=np.float64), (n, 4)),
        }
        for name, (arr, shape) in arrays.items():
            if shape is not None and arr.shape != shape:
                raise ValueError(f"{name}: expected shape {shape}, got {arr.shape}")
            if not np.all(np.isfinite(arr)):
                raise ValueError(f"{name} contains NaN/Inf")
            object.__setattr__(self, name, arr)
        if self.sh_rest.shape[1] not in SH_REST_SIZES:
            raise ValueError(f"sh_rest must have 0 or 45 columns, got {self.sh_rest.shape[1]}")

    @property
    def n(self):
        return self.positions.shape[0]

    @property
    def sh_degree(self):
        return 3 if self.sh_rest.shape[1] == 45 else 0

    def attribute(self, name):
        """Un-activated values of one attribute as an (n, C) array."""
        if name == "position":
            return self.positions
        if name == "opacity":
            return self.opacity_logit.reshape(-1, 1)
        if name == "scale":
            return self.scale_log
        return getattr(self, name)

    def activated(self, name):
        """Attribute values as the renderer sees them (host fp64)."""
        raw = self.attribute(name)
        if name == "opacity":
            return sigmoid(raw)
        if name == "scale":
            return np.exp(raw)
        return raw

    def select(self, index):
        """New cloud with the rows picked by ``index`` (in that order), gathered on the GPU."""
        idx = np.asarray(index, dtype=np.int64)
        cols = {}
        for field_name in ("positions", "sh_dc", "sh_rest", "opacity_logit", "scale_log", "rotation"):
            cols[field_name] = gather_rows_host(getattr(self, field_name), idx)
        return SplatCloud(**cols)


def build_grid_layout(n):
    """splats.py:132-136: largest square grid that n points fill completely."""
    if n < 1:
        raise ValueError("need at least one point to build a grid layout")
    return GridLayout(side=math.isqrt(n))


@dataclass(frozen=True)
class NormalizationSpec:
    """splats.py:155-181: per-attribute [0,1] affine map (activated mins / maxs) and weights."""

    mins: dict
    maxs: dict
    weights: dict

    def constant_channels(self, name):
        return self.maxs[name] <= self.mins[name]

    def denormalize(self, name, columns):
        w = self.weights[name]
        lo, hi = self.mins[name], self.maxs[name]
        const = self.constant_channels(name)
        span = np.where(const, 1.0, hi - lo)
        out = np.asarray(columns, dtype=np.float64) / w * span + lo
        out[:, const] = lo[const]
        return out


# ---------------------------------------------------------------- device forms
def prune_indices(opacity_logit, keep):
    """Indices (CUDA int64, increasing) of the `keep` Gaussians a stable ascending
    argsort of the logits puts last (splats.py:148-151), by plas_prune_to_grid."""
    import torch
    from . import _lib
    L = _lib.lib()
    x = _lib.to_device(opacity_logit, torch.float64).reshape(-1)
    n = x.numel()
    keep = int(keep)
    if keep > n:
        raise ValueError("layout does not fit the cloud")
    out = torch.empty(keep, dtype=torch.int64, device=x.device)
    ws = _lib.workspace(L.plas_prune_workspace_bytes(n), "prep")
    _lib.check(L.plas_prune_to_grid(_lib.ptr(x), n, keep, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_handle()), "prune_to_grid")
    return out


def normalize_features(attrs, weights=None):
    """normalize_for_sorting (splats.py:184-216) on device tensors.

    attrs: {name: (n, C) fp64 tensor of UN-activated values} for the names in
    ATTRIBUTES (sh_rest may have 0 columns).  Returns (features (n, D) CUDA
    fp64, mins {name: CUDA fp64 (C,)}, maxs {...}); D = 1 with zeros when every
    weight is 0, as the reference."""
    import torch
    from . import _lib
    weights = dict(DEFAULT_SORT_WEIGHTS, **(weights or {}))
    for name, w in weights.items():
        if name not in ATTRIBUTES:
            raise ValueError(f"unknown attribute {name!r}")
        if w < 0:
            raise ValueError("sorting weights must be >= 0")
    L = _lib.lib()
    tens, descs, ch, cols, n = {}, [], [], 0, None
    for name in ATTRIBUTES:
        t = _lib.to_device(attrs[name], torch.float64)
        t = t.reshape(t.shape[0], -1)
        n = t.shape[0] if n is None else n
        if t.shape[0] != n:
            raise ValueError("attributes disagree on the number of Gaussians")
        tens[name] = t
        c = t.shape[1]
        w = float(weights[name])
        descs.append(_lib.Attr(values=t.data_ptr() if c else None, row_stride=max(c, 1), channels=c,
                               activation=ACTIVATION[name], weight=w))
        ch.append(c)
        if w != 0.0 and c > 0:
            cols += c
    total = sum(ch)
    mins = torch.empty(max(total, 1), dtype=torch.float64, device="cuda")
    maxs = torch.empty_like(mins)
    feat = torch.zeros((n, max(cols, 1)), dtype=torch.float64, device="cuda")
    arr = (_lib.Attr * len(descs))(*descs)
    ws = _lib.workspace(L.plas_normalize_workspace_bytes(n, total), "prep")
    _lib.check(L.plas_normalize_for_sorting(arr, len(descs), n, _lib.ptr(feat) if cols else None, cols,
                                            _lib.ptr(mins), _lib.ptr(maxs), _lib.ptr(ws), ws.numel(),
                                            _lib.stream_handle()), "normalize_for_sorting")
    mn, mx, off = {}, {}, 0
    for name, c in zip(ATTRIBUTES, ch):
        mn[name], mx[name] = mins[off:off + c], maxs[off:off + c]
        off += c
    return feat, mn, mx


def gather_rows(t, index):
    """t[index] for a CUDA tensor (rows = first dim) by plas_gather_rows."""
    import torch
    from . import _lib
    L = _lib.lib()
    t = t.contiguous()
    idx = _lib.to_device(index, torch.int64).reshape(-1)
    out = torch.empty((idx.numel(),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    row_bytes = t.element_size() * (t[0].numel() if t.shape[0] else 0)
    _lib.check(L.plas_gather_rows(_lib.ptr(t), row_bytes, _lib.ptr(idx), idx.numel(), _lib.ptr(out),
                                  _lib.stream_handle()), "gather_rows")
    return out


def gather_rows_host(a, index):
    """numpy a[index] computed on the GPU (rows of a 1-D or 2-D fp64 array)."""
    import torch
    from . import _lib
    a = np.ascontiguousarray(a)
    if a.shape[0] == 0 or a.size == 0:
        return a[index]
    t = _lib.to_device(a, torch.float64 if a.dtype == np.float64 else torch.from_numpy(a[:0]).dtype)
    return gather_rows(t, np.asarray(index, dtype=np.int64)).cpu().numpy()


# ---------------------------------------------------------------- reference API
def prune_to_grid(cloud, layout):
    """splats.py:139-152: drop the lowest-opacity Gaussians so exactly side**2
    remain (stable ties by index, survivors in index order); selection on the GPU."""
    keep = layout.cells
    if keep > cloud.n:
        raise ValueError("layout does not fit the cloud")
    if keep == cloud.n:
        return cloud
    survivors = prune_indices(cloud.opacity_logit, keep).cpu().numpy()
    return cloud.select(survivors)


def normalize_for_sorting(cloud, weights=None):
    """splats.py:184-216: (features (n, D) fp64 ndarray, NormalizationSpec), on the GPU."""
    weights_full = dict(DEFAULT_SORT_WEIGHTS, **(weights or {}))
    attrs = {name: cloud.attribute(name) for name in ATTRIBUTES}
    feat, mn, mx = normalize_features(attrs, weights)
    mins = {k: v.cpu().numpy() for k, v in mn.items()}
    maxs = {k: v.cpu().numpy() for k, v in mx.items()}
    return feat.cpu().numpy(), NormalizationSpec(mins=mins, maxs=maxs, weights=weights_full)
