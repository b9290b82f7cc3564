"""Separable Gaussian blur with border renormalization (drop-in for sogs.blur, blur.py:1-30).

All three functions run the plas_blur kernels (exact SciPy correlate1d
arithmetic, zero padding).  float32 grids keep the reference's float32
rounding after each axis; any other dtype is computed in float64.
"""

import numpy as np

from . import _lib
from .schedule import gaussian_weights


def _grid3(grid):
    import torch
    _lib.lib()
    if isinstance(grid, torch.Tensor):
        g = grid
        dt = torch.float32 if g.dtype == torch.float32 else torch.float64
        g = g.to(device="cuda", dtype=dt).contiguous()
        shape = tuple(g.shape)
    else:
        a = np.asarray(grid)
        dt = np.float32 if a.dtype == np.float32 else np.float64
        a = np.ascontiguousarray(a, dtype=dt)
        shape = a.shape
        g = torch.from_numpy(a).cuda()
    if len(shape) < 2:
        raise ValueError("grid must be (H, W) or (H, W, C)")
    H, W = shape[0], shape[1]
    C = int(np.prod(shape[2:])) if len(shape) > 2 else 1
    return g, H, W, C, shape


def _run(grid, sigma, radius, op):
    import torch
    L = _lib.lib()
    g, H, W, C, shape = _grid3(grid)
    w = gaussian_weights(sigma, radius)
    dtype = _lib.PLAS_F32 if g.dtype == torch.float32 else _lib.PLAS_F64
    out = torch.empty_like(g)
    ws = _lib.workspace(L.plas_aux_workspace_bytes(H, W, C), "aux")
    _lib.check(L.plas_blur(_lib.ptr(g), _lib.ptr(out), dtype, H, W, C, _lib.ptr(w), radius, op,
                           _lib.ptr(ws), ws.numel(), _lib.stream_handle()), "blur")
    if isinstance(grid, torch.Tensor):
        return out.reshape(shape)
    return out.cpu().numpy().reshape(shape)


def separable_blur(grid, sigma, radius):
    """Zero-padded separable Gaussian filter over the first two axes (blur.py:7-10)."""
    return _run(grid, sigma, radius, _lib.PLAS_BLUR_SEPARABLE)


def border_weight(shape, sigma, radius):
    """Per-cell sum of in-bounds kernel weights (blur.py:13-15), float64 (H, W)."""
    import torch
    L = _lib.lib()
    H, W = int(shape[0]), int(shape[1])
    w = gaussian_weights(sigma, radius)
    out = torch.empty((H, W), dtype=torch.float64, device="cuda")
    ws = _lib.workspace(L.plas_aux_workspace_bytes(H, W, 1), "aux")
    _lib.check(L.plas_blur(None, _lib.ptr(out), _lib.PLAS_F64, H, W, 1, _lib.ptr(w), radius,
                           _lib.PLAS_BLUR_BORDER_WEIGHT, _lib.ptr(ws), ws.numel(),
                           _lib.stream_handle()), "border_weight")
    return out.cpu().numpy()


def renormalized_blur(grid, sigma, radius):
    """Gaussian blur whose kernel is renormalized at the border (blur.py:18-30)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    if radius < 1:
        raise ValueError("radius must be >= 1")
    return _run(grid, sigma, radius, _lib.PLAS_BLUR_RENORMALIZED)


def blur_target_tiers(grid, radius, tier):
    """blur_target (plas.py:64-68) of a float32 (H, W, C) grid through the sort's
    level-blur tiers (tier 0: direct fast fold, 1: FFT), each certified against the
    SciPy fold with exact recomputation of uncertain outputs.  Returns
    (target, (fallbacks axis 0, fallbacks axis 1)).  Test / diagnostics entry."""
    import math

    import torch
    L = _lib.lib()
    a = np.ascontiguousarray(np.asarray(grid, dtype=np.float32))
    shape = a.shape
    H, W = shape[0], shape[1]
    C = int(np.prod(shape[2:])) if len(shape) > 2 else 1
    h = int(math.ceil(radius))
    w = gaussian_weights(radius / 2.0, h)
    g = torch.from_numpy(a).cuda()
    out = torch.empty_like(g)
    ws = _lib.workspace(L.plas_blur_tiers_workspace_bytes(H, W, C, h), "tiers")
    fb = np.zeros(2, dtype=np.int64)
    _lib.check(L.plas_blur_target_tiers(_lib.ptr(g), _lib.ptr(out), H, W, C, _lib.ptr(w), h, int(tier),
                                        _lib.ptr(fb), _lib.ptr(ws), ws.numel(), _lib.stream_handle()),
               "blur_target_tiers")
    return out.cpu().numpy().reshape(shape), (int(fb[0]), int(fb[1]))
