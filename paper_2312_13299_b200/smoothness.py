"""Smoothness regularizer fwd/bwd on the GPU (drop-in for smoothness.py:1-97).

``smoothness_loss`` runs plas_smoothness_plane per weighted plane in float64
(the reference's tests compare at rtol 1e-12).  ``huber``/``huber_grad`` are
the reference's elementwise helpers (smoothness.py:41-54), kept as host
NumPy utilities: they are API conveniences, not the hot path.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .schedule import gaussian_weights

DEFAULT_SMOOTHNESS_WEIGHTS = {
    "position": 0.0,
    "sh_dc": 0.0,
    "sh_rest": 0.0,
    "opacity": 0.09,
    "scale": 0.0,
    "rotation": 0.91,
}


@dataclass(frozen=True)
class SmoothnessParams:
    """smoothness.py:19-38."""

    kernel_size: int = 5
    sigma: float = 3.0
    overall_multiplier: float = 1.0
    huber_delta: float = 1.0
    weights: dict = field(default_factory=lambda: dict(DEFAULT_SMOOTHNESS_WEIGHTS))
    detach_target: bool = False

    def __post_init__(self):
        if self.kernel_size < 1 or self.kernel_size % 2 == 0:
            raise ValueError("kernel_size must be odd and >= 1")
        if self.sigma <= 0:
            raise ValueError("sigma must be positive")
        if self.huber_delta <= 0:
            raise ValueError("huber_delta must be positive")
        if any(w < 0 for w in self.weights.values()):
            raise ValueError("weights must be >= 0")


def huber(x, delta):
    """0.5*x**2 inside |x| <= delta, linear with matching slope outside."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    return np.where(a <= delta, 0.5 * x * x, delta * (a - 0.5 * delta))


def huber_grad(x, delta):
    if delta <= 0:
        raise ValueError("delta must be positive")
    return np.clip(np.asarray(x, dtype=np.float64), -delta, delta)


def smoothness_plane_device(plane, coeff, params):
    """One plane on the device: (mean Huber, grad tensor).  plane: CUDA f64 (H, W, C)."""
    import torch
    L = _lib.lib()
    shp = tuple(plane.shape)
    H, W = shp[0], shp[1]
    C = int(np.prod(shp[2:])) if len(shp) > 2 else 1
    radius = params.kernel_size // 2
    w = gaussian_weights(params.sigma, radius) if radius > 0 else np.ones(1)
    grad = torch.empty_like(plane)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = _lib.workspace(L.plas_aux_workspace_bytes(H, W, C), "aux")
    _lib.check(L.plas_smoothness_plane(_lib.ptr(plane), _lib.ptr(grad), H, W, C, float(coeff),
                                       float(params.huber_delta), int(bool(params.detach_target)),
                                       _lib.ptr(w), radius, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                       _lib.stream_handle()), "smoothness")
    return out, grad


def smoothness_loss(stack, params=None, return_device=False):
    """Weighted Huber penalty between each plane and its blurred version.

    Returns (loss, gradients) as the reference does (smoothness.py:57-97);
    with ``return_device=True`` the gradients stay CUDA tensors.
    """
    import torch
    params = params or SmoothnessParams()
    loss = 0.0
    gradients = {}
    means = []  # (coeff, device mean): one host sync at the end
    for name, plane in stack.planes.items():
        weight = params.weights.get(name, 0.0)
        coeff = params.overall_multiplier * weight
        is_t = isinstance(plane, torch.Tensor)
        shape = tuple(plane.shape)
        size = int(np.prod(shape))
        if coeff == 0.0 or size == 0:
            gradients[name] = (torch.zeros(shape, dtype=torch.float64, device="cuda") if return_device
                               else np.zeros(shape))
            continue
        dev = _lib.to_device(plane if is_t else np.asarray(plane, dtype=np.float64), torch.float64)
        mean, grad = smoothness_plane_device(dev, coeff, params)
        means.append((coeff, mean))
        gradients[name] = grad if return_device else grad.cpu().numpy()
    if means:
        vals = torch.cat([m for _, m in means]).cpu().tolist()
        for (coeff, _), v in zip(means, vals):
            loss += coeff * float(v)  # smoothness.py:88, plane order
    return loss, gradients


# ---------------------------------------------------------------- trainer integration
def _plane_function():
    import torch

    class SmoothnessPlane(torch.autograd.Function):
        """coeff * mean(Huber(plane - blur(plane))) of one plane with its exact
        gradient from the fused kernel (forward computes both; backward scales)."""

        @staticmethod
        def forward(ctx, plane, coeff, params):
            x = plane.detach().to(dtype=torch.float64).contiguous()
            mean, grad = smoothness_plane_device(x, coeff, params)
            ctx.save_for_backward(grad)
            ctx.out_dtype = plane.dtype
            return (mean * coeff).reshape(())

        @staticmethod
        def backward(ctx, g):
            (grad,) = ctx.saved_tensors
            return (grad * g).to(ctx.out_dtype), None, None

    return SmoothnessPlane


_SmoothnessPlane = None


def smoothness_loss_autograd(planes, params=None):
    """smoothness_loss (smoothness.py:57-97) as a differentiable torch scalar for a
    training loop: planes = {attribute: (side, side[, C]) CUDA tensor} (any float
    dtype, requires_grad as the trainer likes); the sum over weighted planes in
    dict order, as the reference accumulates it.  loss.backward() delivers the
    same gradients smoothness_loss returns."""
    import torch
    global _SmoothnessPlane
    if _SmoothnessPlane is None:
        _SmoothnessPlane = _plane_function()
    params = params or SmoothnessParams()
    total = None
    for name, plane in planes.items():
        coeff = params.overall_multiplier * params.weights.get(name, 0.0)
        if coeff == 0.0 or plane.numel() == 0:
            continue
        term = _SmoothnessPlane.apply(plane, coeff, params)
        total = term if total is None else total + term
    if total is None:
        total = torch.zeros((), dtype=torch.float64, device="cuda")
    return total
