"""ctypes wrapper of the C oracle (oracle/plas_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
``--impl reference`` arm) import this module.  The product package never does.

The host-side schedule and kernel weights are restated here independently of
the product (``paper_2312_13299_b200/schedule.py``) so that a test can check
the two against each other and against SciPy:
  * radii by repeated fp64 multiplication (plas.py:246, 274),
  * Gaussian weights as scipy.ndimage._filters._gaussian_kernel1d computes them
    (sigma = r/2, half-width ceil(r), NumPy exp, normalised by NumPy sum).
"""

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
LIB_PATH = os.path.join(BUILD, "libplas_oracle.so")
SRC = os.path.join(HERE, "plas_oracle.c")

_lib = None


def build(force=False):
    os.makedirs(BUILD, exist_ok=True)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o",
                               LIB_PATH, SRC, "-lm"])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, f64, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        L.oracle_seed_key.argtypes = [u64, P]
        L.oracle_rng_size.restype = i32
        L.oracle_rng_init.argtypes = [P, u64]
        L.oracle_rng_integers.argtypes = [P, i64]
        L.oracle_rng_integers.restype = i64
        L.oracle_rng_permutation.argtypes = [P, i64, P]
        for name in ("oracle_separable_blur_f32", "oracle_separable_blur_f64",
                     "oracle_blur_target_f32", "oracle_blur_target_f64"):
            getattr(L, name).argtypes = [P, i32, i32, i32, P, i32, P]
        L.oracle_border_weight.argtypes = [i32, i32, P, i32, P]
        L.oracle_assign_groups.argtypes = [P, P, P, i32, i32, P, i64, i32]
        L.oracle_reassign_block.argtypes = [P, P, P, i32, i32, P, i64, P, i64]
        L.oracle_grid_distance_f32.argtypes = [P, P, i64, i32, i32]
        L.oracle_grid_distance_f32.restype = f64
        L.oracle_vad_f32.argtypes = [P, i32, i32, i32, i32]
        L.oracle_vad_f32.restype = f64
        L.oracle_sort.argtypes = [P, i64, i32, i64, f64, i32, i32, P, P, P, P, P, i64, f64, P, P,
                                  P, i64, P, P]
        L.oracle_sort.restype = i64
        L.oracle_smoothness_plane.argtypes = [P, i32, i32, i32, f64, f64, i32, P, i32, P]
        L.oracle_smoothness_plane.restype = f64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- schedule
def initial_radius(side):
    return max(side / 2.0 - 1.0, 2.0)  # plas.py:54-57


def radii(side, decay, r0=None):
    r = initial_radius(side) if r0 is None else float(r0)
    out = []
    while r >= 1.0:  # plas.py:251, 274
        out.append(r)
        r *= decay
    return out


def gaussian_weights(sigma, h):
    """scipy.ndimage._filters._gaussian_kernel1d(sigma, 0, h), returned as w[0..h] (centre first)."""
    sigma2 = sigma * sigma
    x = np.arange(-h, h + 1)
    phi = np.exp(-0.5 / sigma2 * x ** 2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[h:], dtype=np.float64)


# ---------------------------------------------------------------- RNG
class Rng:
    """NumPy Generator(Philox(seed)) restated in C (plas.py:240)."""

    def __init__(self, seed):
        self.buf = ctypes.create_string_buffer(lib().oracle_rng_size())
        lib().oracle_rng_init(self.buf, seed)

    def integers(self, high):
        return int(lib().oracle_rng_integers(self.buf, high))

    def permutation(self, n):
        out = np.empty(n, dtype=np.int64)
        lib().oracle_rng_permutation(self.buf, n, _p(out))
        return out


def seed_key(seed):
    k = np.zeros(2, dtype=np.uint64)
    lib().oracle_seed_key(seed, _p(k))
    return [int(k[0]), int(k[1])]


# ---------------------------------------------------------------- blur
def blur_target(grid, radius):
    """plas.py:64-68: dtype-preserving (f32 -> f32 parity arithmetic, f64 -> f64)."""
    grid = np.asarray(grid)
    h = int(math.ceil(radius))
    w = gaussian_weights(radius / 2.0, h)
    return renormalized_blur(grid, radius / 2.0, h, w)


def renormalized_blur(grid, sigma, h, w=None):
    if w is None:
        w = gaussian_weights(sigma, h)
    shp = grid.shape
    g3 = grid.reshape(shp[0], shp[1], -1)
    H, W, C = g3.shape
    if grid.dtype == np.float32:
        g3 = np.ascontiguousarray(g3)
        out = np.empty_like(g3)
        lib().oracle_blur_target_f32(_p(g3), H, W, C, _p(w), h, _p(out))
    else:
        g3 = np.ascontiguousarray(g3, dtype=np.float64)
        out = np.empty_like(g3)
        lib().oracle_blur_target_f64(_p(g3), H, W, C, _p(w), h, _p(out))
    return out.reshape(shp)


def separable_blur(grid, sigma, h):
    w = gaussian_weights(sigma, h)
    shp = grid.shape
    g3 = np.ascontiguousarray(np.asarray(grid, dtype=np.float64).reshape(shp[0], shp[1], -1))
    out = np.empty_like(g3)
    lib().oracle_separable_blur_f64(_p(g3), g3.shape[0], g3.shape[1], g3.shape[2], _p(w), h, _p(out))
    return out.reshape(shp)


def border_weight(shape, sigma, h):
    w = gaussian_weights(sigma, h)
    den = np.empty(shape[:2], dtype=np.float64)
    lib().oracle_border_weight(shape[0], shape[1], _p(w), h, _p(den))
    return den


# ---------------------------------------------------------------- assign
def reassign_block(feat, point_idx, target, positions, grouping):
    """plas.py:173-193, in place on float32 feat / int64 point_idx."""
    assert feat.dtype == np.float32 and feat.flags.c_contiguous
    assert point_idx.dtype == np.int64 and target.dtype == np.float32
    positions = np.ascontiguousarray(positions, dtype=np.int64)
    grouping = np.ascontiguousarray(grouping, dtype=np.int64)
    D = feat.shape[1]
    lib().oracle_reassign_block(_p(feat), _p(point_idx), _p(np.ascontiguousarray(target)), D, D,
                                _p(positions), len(positions), _p(grouping), len(grouping))


def grid_distance(a, b):
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    D = a.shape[-1]
    return float(lib().oracle_grid_distance_f32(_p(a), _p(b), a.size // D, D, D))


def vad(grid):
    g = np.ascontiguousarray(grid, dtype=np.float32)
    if g.ndim == 2:
        g = g[..., None]
    return float(lib().oracle_vad_f32(_p(g), g.shape[0], g.shape[1], g.shape[2], g.shape[2]))


# ---------------------------------------------------------------- sort
def sort_grid_report(features, rng_seed=0, improvement_threshold=1e-4, radius_decay=0.95,
                     min_block_size=16, initial_radius_override=None, init_perm=None,
                     max_passes=0, max_seconds=0.0):
    """plas.py:226-286.  Returns (perm, report dict) with the reference's fields."""
    f = np.ascontiguousarray(features, dtype=np.float64)
    n, D = f.shape
    side = math.isqrt(n)
    rs = radii(side, radius_decay, initial_radius_override)
    hs = np.array([int(math.ceil(r)) for r in rs], dtype=np.int32)
    ws = [gaussian_weights(r / 2.0, int(h)) for r, h in zip(rs, hs)]
    woff = np.zeros(max(len(ws), 1), dtype=np.int64)
    if ws:
        woff[1:] = np.cumsum([len(w) for w in ws])[:-1]
    wcat = np.concatenate(ws) if ws else np.zeros(1)
    L = len(rs)
    perm = np.empty(n, dtype=np.int64)
    counts = np.zeros(max(L, 1), dtype=np.int64)
    cap = 1 << 16
    while True:
        trace = np.empty(cap, dtype=np.float64)
        vads = np.zeros(2, dtype=np.float64)
        lv = np.zeros(1, dtype=np.int64)
        ip = None if init_perm is None else np.ascontiguousarray(init_perm, dtype=np.int64)
        passes = lib().oracle_sort(_p(f), n, D, rng_seed, improvement_threshold, min_block_size, L,
                                   _p(np.asarray(rs, dtype=np.float64)), _p(hs), _p(wcat), _p(woff),
                                   None if ip is None else _p(ip), max_passes, float(max_seconds), _p(perm), _p(counts),
                                   _p(trace), cap, _p(vads), _p(lv))
        if passes >= 0:
            break
        cap *= 4
    traces = []
    pos = 0
    for li in range(int(lv[0])):
        c = int(counts[li])
        traces.append((rs[li], tuple(float(v) for v in trace[pos:pos + c])))
        pos += c
    report = {"initial_vad": float(vads[0]), "final_vad": float(vads[1]), "reorders": int(passes),
              "radius_trace": tuple(traces)}
    return perm, report


def smoothness_plane(plane, coeff, delta, detach, sigma, kernel_size):
    plane = np.ascontiguousarray(plane, dtype=np.float64)
    H, W = plane.shape[:2]
    C = plane.size // (H * W)
    h = kernel_size // 2
    w = gaussian_weights(sigma, h) if h > 0 else np.ones(1)
    grad = np.empty_like(plane)
    loss = lib().oracle_smoothness_plane(_p(plane), H, W, C, coeff, delta, int(bool(detach)), _p(w),
                                         h, _p(grad))
    return float(loss), grad
