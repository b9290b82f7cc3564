"""Host-side schedule: radii, block sizes and Gaussian weights (data-independent).

* radii by repeated fp64 multiplication from the start radius (plas.py:246,
  251, 274) -- never r0 * decay**k, which differs in the last ulp and would
  change sigma = r/2;
* beta = min(max(min_block, int(r) + 1), side)       (plas.py:60-61);
* half-width h = ceil(r), sigma = r/2                 (plas.py:64-68);
* weights exactly as scipy.ndimage._filters._gaussian_kernel1d(sigma, 0, h)
  computes them with NumPy (exp, then division by the NumPy sum), so the
  device blur sees bit-identical coefficients to SciPy's correlate1d.
"""

import math

import numpy as np


def initial_radius(side):
    """plas.py:54-57."""
    return max(side / 2.0 - 1.0, 2.0)


def block_size(side, radius, min_block_size=16):
    """plas.py:60-61."""
    return min(max(min_block_size, int(radius) + 1), side)


def radii(side, radius_decay, start=None):
    r = initial_radius(side) if start is None else float(start)
    out = []
    while r >= 1.0:
        out.append(r)
        r *= radius_decay
    return out


def gaussian_weights(sigma, half_width):
    """Centre-first half kernel w[0..h] of scipy's _gaussian_kernel1d(sigma, 0, h)."""
    sigma2 = sigma * sigma
    x = np.arange(-half_width, half_width + 1)
    phi = np.exp(-0.5 / sigma2 * x ** 2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[half_width:], dtype=np.float64)


class Schedule:
    """Per-level (radius, beta, h, weights) table uploaded once per sort."""

    def __init__(self, side, radius_decay, min_block_size=16, start=None):
        self.side = side
        self.radii = radii(side, radius_decay, start)
        self.betas = [block_size(side, r, min_block_size) for r in self.radii]
        self.half_widths = [int(math.ceil(r)) for r in self.radii]
        ws = [gaussian_weights(r / 2.0, h) for r, h in zip(self.radii, self.half_widths)]
        self.weight_offsets = np.zeros(max(len(ws), 1), dtype=np.int64)
        if ws:
            self.weight_offsets[1:len(ws)] = np.cumsum([len(w) for w in ws])[:-1]
        self.weights = np.concatenate(ws) if ws else np.zeros(1)
        self.radii_arr = np.asarray(self.radii if self.radii else [0.0], dtype=np.float64)

    @property
    def num_levels(self):
        return len(self.radii)
