"""Seeded synthetic stand-ins for the BASELINE.json configs C0-C4.

The reference ships no generator for 3DGS-like attributes (its fixtures are
``pkg/tests/conftest.py:9-47``); BASELINE.json names the distributions and
SURVEY.md section 8(d) fixes the draw order used here.  Everything is drawn from
``numpy.random.default_rng(data_seed)`` in the order listed and each channel
is standardised as (x - mean) / std in float64, so the GPU side and the CPU
reference consume bit-identical arrays on any host with the same NumPy.
"""

import numpy as np

CONFIGS = {
    "C0": {"side": 64, "dim": 3},
    "C1": {"side": 256, "dim": 6},
    "C2": {"side": 1024, "dim": 14},
    "C3": {"side": 2048, "dim": 59},
    "C4": {"side": 4096, "dim": 14},
}


def _standardise(x):
    x = np.asarray(x, dtype=np.float64)
    mean = x.mean(axis=0)
    std = x.std(axis=0)
    std = np.where(std > 0, std, 1.0)
    return (x - mean) / std


def _mixture_xyz(rng, n, k):
    means = rng.uniform(-5.0, 5.0, (k, 3))
    stds = rng.uniform(0.1, 1.0, (k, 3))
    comp = rng.integers(0, k, n)
    xyz = means[comp] + rng.normal(0.0, 1.0, (n, 3)) * stds[comp]
    return xyz, comp


def c0(data_seed=0, side=64):
    """uniform[0,1) RGB vectors (BASELINE.json configs[0])."""
    rng = np.random.default_rng(data_seed)
    return rng.random((side * side, 3))


def c1(data_seed=0, side=256):
    """16-component GMM xyz + component-correlated rgb, standardised (configs[1])."""
    rng = np.random.default_rng(data_seed)
    n = side * side
    xyz, comp = _mixture_xyz(rng, n, 16)
    colour = rng.uniform(0.0, 1.0, (16, 3))
    rgb = np.clip(colour[comp] + rng.normal(0.0, 0.05, (n, 3)), 0.0, 1.0)
    return _standardise(np.concatenate([xyz, rgb], axis=1))


def c2(data_seed=0, side=1024):
    """14-channel 3DGS-like attributes, standardised (configs[2]; also configs[4] at side 4096)."""
    rng = np.random.default_rng(data_seed)
    n = side * side
    xyz, _ = _mixture_xyz(rng, n, 64)
    dc = rng.normal(0.0, 0.5, (n, 3))
    log_scale = rng.normal(-4.0, 1.0, (n, 3))
    quat = rng.normal(0.0, 1.0, (n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    opacity = rng.normal(0.0, 2.0, (n, 1))
    return _standardise(np.concatenate([xyz, dc, log_scale, quat, opacity], axis=1))


def c3(data_seed=0, side=2048):
    """configs[2] channels + 45 SH-rest N(0, 0.1) channels weighted 0.2 after standardising."""
    base = c2(data_seed, side)
    rng = np.random.default_rng(data_seed + 1)
    sh = _standardise(rng.normal(0.0, 0.1, (side * side, 45))) * 0.2
    return np.concatenate([base, sh], axis=1)


def c4(data_seed=0, side=4096):
    return c2(data_seed, side)


GENERATORS = {"C0": c0, "C1": c1, "C2": c2, "C3": c3, "C4": c4}


def make(config, data_seed=0, side=None):
    gen = GENERATORS[config]
    return gen(data_seed) if side is None else gen(data_seed, side)


def smoothness_planes(features, side):
    """Split a sorted configs[2] grid into the reference's attribute planes."""
    g = np.asarray(features, dtype=np.float64).reshape(side, side, -1)
    return {
        "position": g[..., 0:3],
        "sh_dc": g[..., 3:6],
        "scale": g[..., 6:9],
        "rotation": g[..., 9:13],
        "opacity": g[..., 13:14],
    }


def neighbour_l2(grid):
    """fp64 mean L2 distance over all 4-neighbour pairs."""
    g = np.asarray(grid, dtype=np.float64)
    dv = np.sqrt(((g[1:] - g[:-1]) ** 2).sum(axis=-1))
    dh = np.sqrt(((g[:, 1:] - g[:, :-1]) ** 2).sum(axis=-1))
    return float((dv.sum() + dh.sum()) / (dv.size + dh.size))
