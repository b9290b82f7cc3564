"""PLAS sorter: drop-in for the reference's ``sogs.plas`` (plas.py:1-301).

Same names, argument meaning and error behaviour as the reference; the work
runs in libplas_b200.so (hand-written sm_100a kernels):

  sort_grid / sort_grid_report  -> plas_sort            (plas.py:226-301)
  blur_target                   -> plas_blur            (plas.py:64-68)
  grid_distance                 -> plas_grid_distance   (plas.py:71-84)
  reassign_block                -> plas_assign_groups   (plas.py:173-193)

``partition_blocks``, ``initial_radius``, ``block_size`` and ``PERMUTATIONS``
are the reference's host-side integer geometry/tables (plas.py:31-34, 54-61,
87-110) and stay on the host.

Two RNG modes (``SortConfig.rng_mode``):
  "parity" (default): NumPy-exact Generator(Philox(seed)) draws, so the
      permutation is bit-identical to the reference CPU implementation;
  "device": Philox4x64-10 draws and grouping generated on the GPU; the whole
      sort is one CUDA graph with no host round trip (the timed headline mode).
"""

import ctypes
import itertools
import functools
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .blur import renormalized_blur
from .metrics import SortReport
from .schedule import Schedule, block_size, gaussian_weights, initial_radius  # noqa: F401
from .splats import DEFAULT_SORT_WEIGHTS

PERMUTATIONS = {
    k: np.array(list(itertools.permutations(range(k))), dtype=np.int64) for k in (1, 2, 3, 4)
}

RNG_MODES = {"parity": _lib.PLAS_RNG_PARITY, "device": _lib.PLAS_RNG_DEVICE}


@dataclass(frozen=True)
class SortConfig:
    """plas.py:37-51, plus two B200 extensions with reference-compatible defaults.

    initial_radius: start radius override (None = reference rule, plas.py:54-57);
        BASELINE.json configs[0] quotes "start radius 32".
    rng_mode: "parity" (bit-identical to the reference) or "device".
    """

    improvement_threshold: float = 1e-4
    radius_decay: float = 0.95
    min_block_size: int = 16
    rng_seed: int = 0
    weights: dict = field(default_factory=lambda: dict(DEFAULT_SORT_WEIGHTS))
    initial_radius: float = None
    rng_mode: str = "parity"

    def __post_init__(self):
        if not (0.0 < self.radius_decay < 1.0):
            raise ValueError("radius_decay must be in (0, 1)")
        if self.improvement_threshold <= 0.0:
            raise ValueError("improvement_threshold must be positive")
        if self.min_block_size < 2:
            raise ValueError("min_block_size must be >= 2")
        if self.rng_mode not in RNG_MODES:
            raise ValueError(f"rng_mode must be one of {sorted(RNG_MODES)}")
        if self.initial_radius is not None and not self.initial_radius > 0:
            raise ValueError("initial_radius must be positive")


def blur_target(grid, radius):
    """Low-pass-filtered copy of the grid: sigma = radius/2, half-width ceil(radius)."""
    if radius <= 0:
        raise ValueError("blur radius must be positive")
    return renormalized_blur(grid, radius / 2.0, int(math.ceil(radius)))


def grid_distance(grid, target, weights=None):
    """Mean Euclidean distance between grid and target cells (plas.py:71-84),
    summed in NumPy's pairwise order on the GPU: the same float as the reference."""
    import torch
    grid = np.asarray(grid, dtype=np.float64) if not isinstance(grid, torch.Tensor) else grid
    target = np.asarray(target, dtype=np.float64) if not isinstance(target, torch.Tensor) else target
    if tuple(grid.shape) != tuple(target.shape):
        raise ValueError("grid and target shapes must match")
    D = grid.shape[-1]
    n = int(np.prod(grid.shape[:-1])) if len(grid.shape) > 1 else 1
    L = _lib.lib()
    a = _lib.to_device(grid, torch.float64).reshape(-1)
    b = _lib.to_device(target, torch.float64).reshape(-1)
    w = None if weights is None else _lib.to_device(np.asarray(weights, dtype=np.float64), torch.float64)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = _lib.workspace(L.plas_grid_distance_workspace_bytes(n), "gdist")
    _lib.check(L.plas_grid_distance(_lib.ptr(a), _lib.ptr(b), _lib.ptr(w), n, D, _lib.ptr(out),
                                    _lib.ptr(ws), ws.numel(), _lib.stream_handle()), "grid_distance")
    return float(out.item())


def _segments(side, beta, delta):
    bounds = [0]
    x = delta if delta > 0 else beta
    while x < side:
        bounds.append(x)
        x += beta
    bounds.append(side)
    return list(zip(bounds[:-1], bounds[1:]))


def partition_blocks(side, radius, dy, dx, min_block_size=16):
    """Shifted block tiling (plas.py:97-110); every cell lands in exactly one block."""
    beta = block_size(side, radius, min_block_size)
    if not (0 <= dy < beta and 0 <= dx < beta):
        raise ValueError("offsets must satisfy 0 <= delta < block size")
    return [(y0, y1, x0, x1) for y0, y1 in _segments(side, beta, dy)
            for x0, x1 in _segments(side, beta, dx)]


def _row_stride(dim):
    return (dim + 3) // 4 * 4


def reassign_block(feat, point_idx, target, positions, grouping):
    """Re-assign one block's cells in place (plas.py:173-193) on the GPU.

    ``feat`` (float32, (n, D)) and ``point_idx`` (int64, (n,)) are updated in
    place exactly as the reference's numba kernel updates them.  A float32
    ``target`` (what the reference's sort passes, plas.py:252-254) takes the
    fused K3 group kernel; any other target dtype makes the reference's numba
    code difference and square in float64, which ``plas_assign_groups_f64t``
    reproduces (the target is widened to float64 first, as numba promotes it).
    """
    import torch
    tgt = np.asarray(target)
    f64t = tgt.dtype != np.float32
    m = len(positions)
    grouping = np.asarray(grouping, dtype=np.int64)
    local = grouping[grouping < m]
    ordered = np.asarray(positions, dtype=np.int64)[local]
    g4 = (m // 4) * 4
    rest = m - g4
    if not g4 and rest < 2:
        return
    L = _lib.lib()
    feat_np = np.asarray(feat)
    n, D = feat_np.shape
    S = _row_stride(D)
    fpad = np.zeros((n, S), dtype=np.float32)
    fpad[:, :D] = feat_np
    tpad = np.zeros((n, S), dtype=np.float64 if f64t else np.float32)
    tpad[:, :D] = tgt
    f_dev = torch.from_numpy(fpad).cuda()
    t_dev = torch.from_numpy(tpad).cuda()
    i_dev = torch.from_numpy(np.ascontiguousarray(point_idx, dtype=np.int64)).cuda()
    st = _lib.stream_handle()
    fn = L.plas_assign_groups_f64t if f64t else L.plas_assign_groups
    if f64t and D > 64:
        raise ValueError("reassign_block: a float64 target supports at most 64 channels")
    if g4:
        groups = torch.from_numpy(np.ascontiguousarray(ordered[:g4].reshape(-1, 4))).cuda()
        _lib.check(fn(_lib.ptr(f_dev), _lib.ptr(i_dev), _lib.ptr(t_dev), D, S,
                      _lib.ptr(groups), g4 // 4, 4, st), "assign_groups")
    if rest >= 2:
        groups = torch.from_numpy(np.ascontiguousarray(ordered[g4:].reshape(1, rest))).cuda()
        _lib.check(fn(_lib.ptr(f_dev), _lib.ptr(i_dev), _lib.ptr(t_dev), D, S,
                      _lib.ptr(groups), 1, rest, st), "assign_groups")
    feat[...] = f_dev.cpu().numpy()[:, :D]
    point_idx[...] = i_dev.cpu().numpy()


# ----------------------------------------------------------------------------
# sort
# ----------------------------------------------------------------------------
def _validate(features):
    """plas.py:227-237 (finiteness is checked on the device -> ValueError)."""
    import torch
    if isinstance(features, torch.Tensor):
        t = features
        if t.dim() != 2:
            raise ValueError("features must be a (side**2, D) matrix")
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        n = t.shape[0]
    else:
        arr = np.asarray(features)
        if arr.dtype != np.float32:
            arr = np.asarray(features, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("features must be a (side**2, D) matrix")
        t = arr
        n = arr.shape[0]
    side = math.isqrt(n)
    if side * side != n:
        raise ValueError("feature count must be a perfect square")
    if side < 2:
        raise ValueError("grid side must be at least 2")
    if t.shape[1] < 1:
        raise ValueError("features must have at least one channel")
    return t, n, side


@functools.lru_cache(maxsize=64)
def max_start_half_width(side):
    """Largest level half-width ceil(r) a sort of this side supports: the
    reference rule's ceil(max(side/2 - 1, 2)) plus one (csrc blur_pad)."""
    return int(math.ceil(max(side / 2.0 - 1.0, 2.0))) + 1


def _schedule(side, radius_decay, min_block_size, start):
    """Schedules are pure functions of these four values (read-only after
    construction), so repeated sorts of one shape reuse the host tables."""
    return Schedule(side, radius_decay, min_block_size, start)


class SortPlan:
    """Host-side state of one sort shape: schedule, workspace and the C-ABI call."""

    def __init__(self, n, dim, config):
        self.n = n
        self.dim = dim
        self.side = math.isqrt(n)
        self.config = config
        self.mode = RNG_MODES[config.rng_mode]
        if config.initial_radius is not None:
            # the sort's zero-padded blur buffers cover half-widths up to the
            # reference rule's ceil(side/2 - 1) plus one (BASELINE configs[0]
            # starts at 32 on a 64-cell side); larger start radii are rejected
            # here (the C ABI returns PLAS_ERR_INVALID for them)
            hmax = max_start_half_width(self.side)
            if math.ceil(config.initial_radius) > hmax:
                raise ValueError(f"initial_radius {config.initial_radius} exceeds the largest start radius "
                                 f"for a {self.side}-cell side (ceil(r) <= {hmax})")
        self.schedule = _schedule(self.side, config.radius_decay, config.min_block_size,
                                 config.initial_radius)
        self.trace_capacity = max(64 * max(self.schedule.num_levels, 1), 4096)

    def run(self, features_dev, perm_out, initial_perm=None, profile=None, shard=None):
        """features_dev: CUDA f32/f64 (n, dim); perm_out: CUDA int64 (n,). Returns report fields.

        profile: optional _lib.SortProfile filled with per-kernel CUDA-event times
        (host-stepped execution of the same kernels).
        shard: optional sharded.ShardSpec (rank, world, exchange) for a multi-GPU sort;
        every rank calls run() with identical arguments."""
        import torch
        L = _lib.lib()
        sch = self.schedule
        world = shard.world if shard is not None else 1
        xb = None
        if world > 1:
            dev = features_dev.device
            xb = {"send": torch.zeros(2 * self.n, dtype=torch.int32, device=dev),
                  "recv": torch.zeros(2 * self.n * world, dtype=torch.int32, device=dev),
                  "part": torch.zeros(_lib.XPART, dtype=torch.float64, device=dev),
                  "part_all": torch.zeros(_lib.XPART * world, dtype=torch.float64, device=dev)}

            def _cb(_ctx, op, a, b, sizes):
                ex = shard.exchange
                try:
                    if op == _lib.PLAS_XCHG_PASS:
                        return int(ex(xb["send"], xb["recv"], xb["part"], xb["part_all"]))
                    if op == _lib.PLAS_XCHG_ALLGATHER:
                        ex.allgather(xb["ws"], int(b), int(a))
                        return 0
                    if op == _lib.PLAS_XCHG_ALLTOALL:
                        sz = [int(sizes[i]) for i in range(2 * world)]
                        ex.alltoall(xb["ws"], int(a), int(b), sz[:world], sz[world:])
                        return 0
                    raise ValueError(f"unknown exchange op {op}")
                except Exception as exc:  # never raise through the C ABI
                    xb["error"] = exc
                    return -1
            xb["cb"] = _lib.EXCHANGE_FN(_cb)
        while True:
            wsb = L.plas_sort_workspace_bytes_sharded(self.n, self.dim, sch.num_levels, len(sch.weights),
                                                      self.trace_capacity, self.mode, world)
            ws = _lib.workspace(wsb, "sort")  # per thread and stream (_lib.workspace)
            if xb is not None:
                xb["ws"] = ws
            args = _lib.SortArgs()
            args.features = _lib.ptr(features_dev)
            args.features_dtype = _lib.PLAS_F32 if features_dev.dtype == torch.float32 else _lib.PLAS_F64
            args.dim = self.dim
            args.n = self.n
            args.improvement_threshold = self.config.improvement_threshold
            args.radius_decay = self.config.radius_decay
            args.initial_radius = float("nan") if self.config.initial_radius is None else float(
                self.config.initial_radius)
            args.min_block_size = self.config.min_block_size
            args.seed = int(self.config.rng_seed)
            args.rng_mode = self.mode
            args.num_levels = sch.num_levels
            args.radii = _lib.ptr(sch.radii_arr)
            args.weights = _lib.ptr(sch.weights)
            args.weight_offsets = _lib.ptr(sch.weight_offsets)
            args.initial_perm = None if initial_perm is None else _lib.ptr(initial_perm)
            args.trace_capacity = self.trace_capacity
            args.stream = _lib.stream_handle()
            args.profile = None if profile is None else ctypes.cast(ctypes.pointer(profile), ctypes.c_void_p)
            if world > 1:
                args.rank, args.world = shard.rank, world
                args.exchange = xb["cb"]
                args.xchg_send, args.xchg_recv = _lib.ptr(xb["send"]), _lib.ptr(xb["recv"])
                args.xchg_part, args.xchg_part_all = _lib.ptr(xb["part"]), _lib.ptr(xb["part_all"])
            counts = np.zeros(max(sch.num_levels, 1), dtype=np.int64)
            trace = np.zeros(self.trace_capacity, dtype=np.float64)
            res = _lib.SortResult()
            res.perm = _lib.ptr(perm_out)
            res.level_counts = _lib.ptr(counts)
            res.trace = _lib.ptr(trace)
            code = L.plas_sort(args, res, _lib.ptr(ws), ws.numel())
            if code == _lib.PLAS_ERR_CAPACITY:
                self.trace_capacity *= 4
                continue
            if xb is not None and "error" in xb:
                raise RuntimeError(f"exchange failed on rank {shard.rank}") from xb["error"]
            _lib.check(code, "plas_sort")
            break
        traces = []
        pos = 0
        for li in range(res.levels_done):
            c = int(counts[li])
            traces.append((sch.radii[li], tuple(float(v) for v in trace[pos:pos + c])))
            pos += c
        return {
            "initial_vad": float(res.initial_vad),
            "final_vad": float(res.final_vad),
            "reorders": int(res.reorders),
            "radius_trace": tuple(traces),
            "gpu_ms": float(res.gpu_ms),
            "cells_moved": int(res.cells_moved),
            "exact_warps": int(res.exact_warps),
            "banded_levels": int(res.banded_levels),
        }


def sort_on_device(features, config=None, initial_perm=None, profile=None):
    """Device-resident sort: CUDA tensor in, (CUDA int64 perm, report dict) out."""
    import torch
    config = config or SortConfig()
    t, n, side = _validate(features)
    _lib.lib()
    if not isinstance(t, torch.Tensor):
        t = torch.from_numpy(np.ascontiguousarray(t))
    t = t.to("cuda").contiguous()
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    ip = None
    if initial_perm is not None:
        ip = _lib.to_device(np.asarray(initial_perm, dtype=np.int64), torch.int64)
    rep = SortPlan(n, t.shape[1], config).run(t, perm, ip, profile)
    return perm, rep


def _sort(features, config, threads, initial_perm=None):
    import torch
    t, n, side = _validate(features)
    _lib.lib()  # fails loudly without the extension / a CUDA device
    started = time.perf_counter()
    if isinstance(t, torch.Tensor):
        # pinned host tensors are copied asynchronously on the current stream
        dev = t.to("cuda", non_blocking=t.device.type == "cpu" and t.is_pinned()).contiguous()
    else:
        dev = torch.from_numpy(np.ascontiguousarray(t)).to("cuda")
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    ip = None
    if initial_perm is not None:
        ip = _lib.to_device(np.asarray(initial_perm, dtype=np.int64), torch.int64)
    rep = SortPlan(n, dev.shape[1], config).run(dev, perm, ip)
    perm_host = perm.cpu().numpy()
    report = SortReport(
        initial_vad=rep["initial_vad"],
        final_vad=rep["final_vad"],
        reorders=rep["reorders"],
        wall_time_s=time.perf_counter() - started,
        radius_trace=rep["radius_trace"],
    )
    return perm_host, report


def sort_grid(features, config=None, threads=1):
    """Sort features into a locality-preserving square grid (plas.py:289-296).

    Returns ``perm`` such that ``features[perm]`` reshaped row-major is the
    sorted grid.  ``threads`` is accepted for API compatibility; results never
    depend on it (the reference guarantees the same, tests/test_plas.py:310-315).
    """
    perm, _ = _sort(features, config or SortConfig(), threads)
    return perm


def sort_grid_report(features, config=None, threads=1):
    """Like sort_grid, but also returns a SortReport (plas.py:299-301)."""
    return _sort(features, config or SortConfig(), threads)
