#!/usr/bin/env python
"""bench.py -- PLAS sort hot path on BASELINE.json configs[2] (1024^2 x 14 fp32).

One "step" = one full PLAS sort to convergence of a 1024x1024 grid of 14
standardised 3DGS-like attributes (seeded synthetic stand-in).
  value : grid-elems/s = N * passes / device time, inputs resident in HBM,
          timed with CUDA events around each sort (L2 flushed before each step);
  e2e   : the same metric through the public API sort_grid() with the features
          in pinned host memory (H2D of the fp64 features + D2H of the int64
          permutation inside the timed region);
  roofline: the dominant kernel's algorithmic bytes / its CUDA-event duration,
          from an event-instrumented host-stepped replay of the same sort;
  cpu_baseline: the reference's own CPU sort (baseline/_ref/sogs, numba+SciPy,
          all host threads): its blur / pass / distance functions timed on the
          same workload (~10 s of CPU) and composed over the full schedule
          (cpu_reference_sample); the C oracle port if baseline/_ref is absent.
N > 1 (torchrun): every rank sorts its own independent grid (data seed = rank),
no data-path collective; value = sum of rank units / max rank time ("weak").
"""

import argparse
import json
import math
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "plas_sort_grid_elems_per_s"
UNIT = "grid-elems/s"
WORKLOADS = {
    "C0": dict(cfg=dict(radius_decay=0.5, improvement_threshold=1e-5)),
    "C1": dict(cfg={}),
    "C2": dict(cfg={}),
    "C3": dict(cfg={}),
    "C4": dict(cfg={}),
}


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    p.add_argument("--side", type=int, default=None, help="override grid side (testing)")
    p.add_argument("--mode", default="device", choices=["device", "parity"])
    p.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU work per sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-profile", action="store_true")
    p.add_argument("--no-smoothness", action="store_true")
    p.add_argument("--no-prep", action="store_true", help="skip the feature-prep (SURVEY 8(f) #1) line")
    p.add_argument("--sharded", action="store_true",
                   help="N > 1: shard ONE grid over the ranks (strong scaling; sharded.py) instead of "
                        "one independent grid per rank")
    return p.parse_args(argv)


# ---------------------------------------------------------------------------- ranks
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, backend):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist if world > 1 else None


def combine(units, seconds, dist, device):
    """Whole-job aggregate: sum of units over ranks, max of time over ranks."""
    if dist is None:
        return float(units), float(seconds)
    import torch
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(u.item()), float(t.item())


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        if shutil.which("nvidia-smi") is None:
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.fh = open(self.path, "w")
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "200"],
                                     stdout=self.fh, stderr=subprocess.DEVNULL)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU reference
REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _reference_module():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "sogs")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_bench"))
    sys.dont_write_bytecode = True
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import sogs.plas as rp
    except Exception:
        return None
    return rp


def reference_level_passes(config):
    """The reference's own per-level pass counts at sort seed 0 (tests/golden), if recorded."""
    path = os.path.join(REPO, "tests", "golden", f"{config.lower()}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        rows = d if isinstance(d, list) else [d]
        row = next(r for r in rows if r["cfg"].get("rng_seed", 0) == 0 and r.get("initial_radius") is None)
        return [c - 1 for c in row["counts"]]  # trace entries per level = passes + 1
    except Exception:
        return None


def _fit_line(xs, ys):
    if len(xs) < 2 or max(xs) == min(xs):
        return 0.0, float(np.mean(ys))
    b, a = np.polyfit(np.asarray(xs, float), np.asarray(ys, float), 1)
    return float(b), float(a)


def cpu_reference_sample(features, cfg_kw, budget_s, level_passes, counts_source, threads=None):
    """The reference CPU sort's throughput on this host, from a bounded sample.

    A full reference sort of C2 takes ~9-10 min on the host, so it is not run
    whole.  Instead the reference's own functions (baseline/_ref sogs: blur_target,
    _reassign_pass with its thread pool, grid_distance) are timed on the same
    workload at a few radii (blur cost is linear in the half-width ceil(r)) and a
    few block sizes, and composed over the full radius schedule with the per-level
    pass counts `level_passes`:
        T = sum_l [ blur(h_l) + gd + P_l * (reassign(beta_l) + gd) ].
    A prefix of the sort would be biased: its first level alone has the largest
    blur (h = 511).  Small configs (estimated < budget) run the whole sort.
    Falls back to the C oracle port (oracle/) when baseline/_ref is absent.
    """
    n, D = features.shape
    side = math.isqrt(n)
    threads = threads or os.cpu_count()
    rp = _reference_module()
    if rp is None:
        from oracle import oracle
        t0 = time.perf_counter()
        _, rep = oracle.sort_grid_report(features, max_seconds=budget_s, **cfg_kw)
        el = time.perf_counter() - t0
        return {"value": n * rep["reorders"] / el, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"prefix: first {rep['reorders']} passes of the sort, {el:.1f} s; C oracle port "
                          "(baseline/_ref absent)"}
    rp.sort_grid(np.random.default_rng(0).random((64, 3)), rp.SortConfig(), threads=threads)  # numba JIT
    cfg = rp.SortConfig(**cfg_kw)
    radii_l, r = [], rp.initial_radius(side)
    while r >= 1.0:
        radii_l.append(r)
        r *= cfg.radius_decay
    if n <= 65536:  # C0 / C1: the whole sort fits the budget
        t0 = time.perf_counter()
        _, rep = rp.sort_grid_report(features, cfg, threads=threads)
        el = time.perf_counter() - t0
        return {"value": n * rep.reorders / el, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"full reference sort (baseline/_ref sogs, threads={threads}): "
                          f"{rep.reorders} passes in {el:.2f} s"}
    t_start = time.perf_counter()
    rng = np.random.Generator(np.random.Philox(0))
    perm0 = rng.permutation(n)
    feat = np.ascontiguousarray(np.asarray(features, dtype=np.float64)[perm0], dtype=np.float32)
    cell_grid = np.arange(n, dtype=np.int64).reshape(side, side)
    from concurrent.futures import ThreadPoolExecutor
    ex = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    # blur: three radii from the lower part of the schedule (cost ~ a + b h)
    hs = sorted({int(math.ceil(radii_l[i])) for i in (len(radii_l) - 1, len(radii_l) // 3, len(radii_l) // 5)})
    blur_t, target = [], None
    for h in hs:
        t0 = time.perf_counter()
        target = np.ascontiguousarray(rp.blur_target(feat.reshape(side, side, -1), float(h)).reshape(n, -1),
                                      dtype=np.float32)
        blur_t.append(time.perf_counter() - t0)
    bb, ba = _fit_line(hs, blur_t)
    gds = []
    for _ in range(3):
        t0 = time.perf_counter()
        rp.grid_distance(feat, target)
        gds.append(time.perf_counter() - t0)
    gd = min(gds)
    # passes: three block sizes, two passes each
    betas = sorted({rp.block_size(side, radii_l[i], cfg.min_block_size)
                    for i in (0, len(radii_l) // 4, len(radii_l) - 1)})
    pass_t = []
    for beta in betas:
        ts = []
        for _ in range(2):
            dy, dx = int(rng.integers(0, beta)), int(rng.integers(0, beta))
            mp = rng.permutation(beta * beta)
            t0 = time.perf_counter()
            rp._reassign_pass(feat, perm0, target, cell_grid, beta, dy, dx, mp, ex, threads)
            ts.append(time.perf_counter() - t0)
        pass_t.append(min(ts))
    if ex is not None:
        ex.shutdown()
    sampled = time.perf_counter() - t_start
    if level_passes is None or len(level_passes) != len(radii_l):
        level_passes = [9] * len(radii_l)  # C2 reference mean (1089 passes / 122 levels)
        counts_source = "assumed 9 per level"
    total = 0.0
    for r_l, p_l in zip(radii_l, level_passes):
        h = int(math.ceil(r_l))
        beta = rp.block_size(side, r_l, cfg.min_block_size)
        t_pass = float(np.interp(beta, betas, pass_t)) + gd
        total += max(ba + bb * h, 0.0) + gd + p_l * t_pass
    passes = int(sum(level_passes))
    return {"value": n * passes / total, "unit": UNIT, "cores": threads, "kind": "reference",
            "estimated_sort_s": round(total, 1),
            "sample": f"reference functions (baseline/_ref sogs 0.1.0: blur_target at h={hs}, "
                      f"_reassign_pass(threads={threads}) at beta={betas}, grid_distance) timed on this host on "
                      f"the {side}^2x{D} workload ({sampled:.1f} s of CPU work), composed over the "
                      f"{len(radii_l)}-level schedule with {passes} passes "
                      f"(per-level pass counts: {counts_source}): "
                      f"estimated full reference sort {total:.1f} s"}


# ---------------------------------------------------------------------------- ours
def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


NCU_LISTS = {"C2": "r02_launches_c2.json", "C3": "r02_launches_c3.json", "C4": "r02_launches_c4.json"}  # per workload (round 2 build)


def ncu_traffic(config, prefixes=("pass_kernel", "pass_kernel_pipe", "tile_pass_kernel")):
    """DRAM bytes (read + write) per K3 launch from the committed ncu launch list of
    this workload (profiles/, tools/launch_summary.py), launch-weighted over the
    gather and tile variants; None if that workload has no list."""
    if config not in NCU_LISTS:
        return None
    path = os.path.join(REPO, "profiles", NCU_LISTS[config])
    try:
        with open(path) as f:
            ks = json.load(f)["kernels"]
        sel = [v for k, v in ks.items() if k.split("<")[0] in prefixes]
        launches = sum(v["launches"] for v in sel)
        return int(sum(v["dram_bytes_per_launch"] * v["launches"] for v in sel) / launches) if launches else None
    except Exception:
        return None


# fp64 peak of this pool's B200 for the blur's compute roof: tools/fp64_micro.cu
# measured DADD / DMUL / DFMA at 18.4 Gop/s x 1e3 each (64 per clock per SM at
# 1.965 GHz), i.e. 36.8 TFLOP/s counting an FMA as two (profiles/r02_fp64_peak.txt)
FP64_PEAK_TFLOPS = 36.8


def _fft_len_for(side, h):
    """plas_b200.cu fft_choose_code: the shortest 2^k (5..13), 3 2^k (9..11) or
    5 2^k (9..10) with side + h <= L and side <= the length's output capacity."""
    best = None
    for k in range(5, 14):
        L = 1 << k
        if side + h <= L and side <= L // 2:
            best = L if best is None else min(best, L)
    for m, ks, cap in ((3, range(9, 12), 2), (5, range(9, 11), 4)):
        for k in ks:
            L = m << k
            if side + h <= L and side <= cap << k:
                best = L if best is None else min(best, L)
    return best


def blur_flops(side, D, radii):
    """fp64 flops of the sort's level blurs under the library's tier rules
    (plas_b200.cu: FFT from h >= 48 / 64 (40 for rows wider than 16 floats)
    while side + h fits the longest length; the one-kernel tile tier for h <= 4
    on rows of <= 16 floats; the direct fold otherwise).  Direct / tile: 3h + 1
    per output and axis (a DADD and a DFMA per tap pair, the centre product);
    FFT: two complex transforms of 5 L log2 L per line pair and axis."""
    S = (D + 3) // 4 * 4
    h0 = math.ceil(max(side / 2.0 - 1.0, 2.0))
    L_top = _fft_len_for(side, h0)
    min_h = 40 if S > 16 else (48 if (L_top or 0) <= 2048 else 64)
    pairs = side * ((D + 1) // 2)
    total = 0.0
    for r in radii:
        h = math.ceil(r)
        if L_top and h >= min_h and side + h <= L_top:
            L = _fft_len_for(side, h) or L_top
            total += 2 * pairs * 2 * 5 * L * math.log2(L)
        else:
            total += 2 * side * side * D * (3 * h + 1)
    return total


def run_smoothness(feats, perm_np, side, device, peak, steps=5):
    """Smoothness-loss fwd+bwd (smoothness.py:57-97) on the sorted grid, default
    SmoothnessParams (opacity 0.09, rotation 0.91: C_w = 5 channels), fp64 as the
    reference; planes resident in HBM, CUDA events.  Algorithmic bytes: each
    weighted plane element read once and its gradient written once (16 B fp64)."""
    import torch
    import paper_2312_13299_b200 as plas
    from paper_2312_13299_b200 import synthetic
    planes_np = synthetic.smoothness_planes(feats[perm_np], side)
    planes = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in planes_np.items()}
    stack = plas.GridStack(plas.GridLayout(side), planes)
    params = plas.SmoothnessParams()
    for _ in range(3):
        plas.smoothness_loss(stack, params, return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss, _ = plas.smoothness_loss(stack, params, return_device=True)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    cw = sum(v.shape[-1] for k, v in planes_np.items() if params.weights.get(k, 0.0) > 0)
    alg = side * side * cw * 16
    out = {"what": "smoothness_loss fwd+bwd, default SmoothnessParams, fp64, sorted C2 grid",
           "ms": round(ms, 3), "loss": loss, "weighted_channels": cw,
           "algorithmic_bytes": alg, "achieved_GBps": round(alg / ms / 1e6, 1),
           "hbm_frac": round(alg / ms / 1e6 / peak, 4)}
    rp = _reference_module()
    if rp is not None:
        import sogs.smoothness as rs
        from sogs.splats import GridLayout as RL, GridStack as RS
        rstack = RS(RL(side), planes_np)
        rs.smoothness_loss(rstack, rs.SmoothnessParams())
        t0 = time.perf_counter()
        rl, _ = rs.smoothness_loss(rstack, rs.SmoothnessParams())
        out["reference_cpu_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
        out["reference_loss"] = rl
        out["loss_rel_diff"] = abs(loss - rl) / max(abs(rl), 1e-300)
    return out


def run_prep(device, peak, steps=5, n=1_100_000, side=1024, seed=0):
    """SURVEY 8(f) #1 on the GPU: prune_to_grid -> select (every attribute row
    gathered) -> normalize_for_sorting -> the post-sort permutation apply of every
    attribute (bundle.py:134-160), on a seeded degree-3 cloud of n Gaussians
    pruned to side^2; device-resident, CUDA events.  Algorithmic bytes per
    kept Gaussian: select and apply each read + write all 59 fp64 channels
    (2 x 944 B), normalize reads the 9 weighted raw channels and writes 9
    features (144 B), the logit is read once (8 B).  Next to the reference's
    own prune_to_grid + normalize_for_sorting + values[perm] on the host."""
    import torch
    from paper_2312_13299_b200 import quantization as pq
    from paper_2312_13299_b200 import splats as ps
    g = np.random.default_rng(seed)
    cl = {"positions": g.normal(0, 3, (n, 3)), "sh_dc": g.normal(0, 0.5, (n, 3)),
          "sh_rest": g.normal(0, 0.1, (n, 45)), "opacity_logit": g.normal(0, 2, n),
          "scale_log": g.normal(-4, 1, (n, 3)), "rotation": g.normal(0, 1, (n, 4))}
    fields = ("positions", "sh_dc", "sh_rest", "opacity_logit", "scale_log", "rotation")
    attr_of = dict(zip(ps.ATTRIBUTES, fields))
    dev = {f: torch.from_numpy(np.ascontiguousarray(cl[f])).to(device) for f in fields}
    keep = side * side
    perm = torch.from_numpy(np.random.default_rng(seed + 1).permutation(keep)).to(device)

    qspec = pq.default_quant_spec()

    def step():
        surv = ps.prune_indices(dev["opacity_logit"], keep)
        pr = {f: ps.gather_rows(dev[f], surv) for f in fields}
        feats, _, _ = ps.normalize_features({a: pr[f] for a, f in attr_of.items()})
        applied = {f: ps.gather_rows(pr[f], perm) for f in fields}
        planes = {a: pq.quantize_planes(a, applied[f], qspec[a], host_ranges=False)[0] for a, f in attr_of.items()}
        return surv, feats, planes

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        surv, feats, _ = step()
    e1.record()
    e1.synchronize()
    ms_eager = e0.elapsed_time(e1) / steps
    # the same step captured once in a CUDA graph: device time without the
    # Python / ctypes launch overhead of its ~40 small launches
    graph = torch.cuda.CUDAGraph()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph, stream=stream):
            gsurv, gfeats, _ = step()
    torch.cuda.current_stream().wait_stream(stream)
    graph.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        graph.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if not (torch.equal(gsurv, surv) and torch.equal(gfeats, feats)):
        raise RuntimeError("graph replay of the prep step differs from the eager step")
    alg = keep * (2 * 944 + 144 + 472 + 59 * 2) + n * 8  # + quantize: read 59 fp64, write <= 2 B pixels
    out = {"what": f"bundle.compress up to the PNG encode: prune_to_grid + select + normalize_for_sorting + "
                   f"permutation apply + contract/quantize/plane packing, {n} Gaussians (degree-3, 59 channels) "
                   f"-> {side}x{side}, fp64, device-resident (the sort itself is the main line)",
           "ms": round(ms, 3), "ms_eager": round(ms_eager, 3), "algorithmic_bytes": alg, "achieved_GBps": round(alg / ms / 1e6, 1),
           "hbm_frac": round(alg / ms / 1e6 / peak, 4)}
    rp = _reference_module()
    if rp is not None:
        from sogs import splats as rsp
        cloud = rsp.SplatCloud(**cl)
        layout = rsp.GridLayout(side)
        pnp = perm.cpu().numpy()
        from sogs import bundle as rbd
        from sogs import quantization as rq
        rspec = rq.default_quant_spec()
        t0 = time.perf_counter()
        pruned = rsp.prune_to_grid(cloud, layout)
        rfeat, _ = rsp.normalize_for_sorting(pruned)
        ref_planes = {}
        for a in rsp.ATTRIBUTES:  # bundle.py:158-176 without the PNG encode
            vals = pruned.attribute(a)[pnp]
            if a == "position":
                vals = rq.contract(vals)
            idx, _, _ = rbd._quantize_attribute(vals, rspec[a])
            per_image = rbd.PLANE_GROUPS[a][0]
            ref_planes[a] = [idx[:, i * per_image:(i + 1) * per_image] for i in range(vals.shape[1] // per_image)]
        out["reference_cpu_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
        _, _, gplanes = step()
        out["planes_identical"] = bool(all(
            np.array_equal(gplanes[a].cpu().numpy().astype(np.int64), np.stack(ref_planes[a])) for a in ref_planes))
        order = np.argsort(cloud.opacity_logit, kind="stable")
        out["survivors_identical"] = bool(np.array_equal(surv.cpu().numpy(), np.sort(order[n - keep:])))
        f = feats.cpu().numpy()
        out["features_max_ulp"] = int(np.abs(f.view(np.int64) - rfeat.view(np.int64)).max())
    return out


def run_ours(args):
    import torch
    import paper_2312_13299_b200 as plas
    from paper_2312_13299_b200 import _lib, synthetic
    from paper_2312_13299_b200.plas import SortPlan, sort_on_device

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist(world, "nccl")
    device = torch.device("cuda", local)
    sharded_run = args.sharded and world > 1
    # independent grids: data seed = rank; sharded: every rank holds the same grid
    feats = synthetic.make(args.config, data_seed=0 if sharded_run else rank, side=args.side)
    n, D = feats.shape
    side = math.isqrt(n)
    cfg = plas.SortConfig(rng_seed=0, rng_mode=args.mode, **WORKLOADS[args.config]["cfg"])
    dev = torch.from_numpy(feats).to(device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    if sharded_run:
        from paper_2312_13299_b200 import sharded
        exchange = sharded.DistExchange()

        def sort_on_device(x, c):  # noqa: F811 -- this rank's share of one sharded sort
            return sharded.sort_on_device_sharded(x, c, rank, world, exchange)

    for _ in range(args.warmup):
        sort_on_device(dev, cfg)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize()
    step_ms, passes, levels = [], [], []
    rep = None
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        perm, rep = sort_on_device(dev, cfg)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        passes.append(rep["reorders"])
        levels.append(len(rep["radius_trace"]))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    if sharded_run:  # one grid for the whole job: count its units once
        units, secs = combine(n * sum(passes) / world, sum(step_ms) / 1e3, dist, device)
    else:
        units, secs = combine(n * sum(passes), sum(step_ms) / 1e3, dist, device)
    value = units / secs
    ms_per_step = secs * 1e3 / args.steps

    perm_np = perm.cpu().numpy()
    grid = feats[perm_np].reshape(side, side, D)
    quality = {"nbr_l2": synthetic.neighbour_l2(grid), "final_vad": rep["final_vad"],
               "initial_vad": rep["initial_vad"], "passes": passes[-1], "levels": levels[-1],
               "sort_time_s": statistics.median(step_ms) / 1e3}

    # ---- e2e through the public API, pinned host features, perm back to host
    e2e = None
    if not args.no_e2e and not sharded_run:
        host = torch.from_numpy(feats).pin_memory()
        plas.sort_grid(host, cfg)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e_ms, e_units = [], 0
        for k in range(args.steps):
            flush.fill_(k & 0xff)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p_host, r = plas.sort_grid_report(host, cfg)
            e_ms.append((time.perf_counter() - t0) * 1e3)
            e_units += n * r.reorders
        eu, es = combine(e_units, sum(e_ms) / 1e3, dist, device)
        e2e = {"value": eu / es, "unit": UNIT, "h2d_bytes_per_step": int(feats.nbytes),
               "d2h_bytes_per_step": int(n * 8), "ms_per_step": es * 1e3 / args.steps}

    # ---- per-kernel CUDA-event times (host-stepped replay of one sort)
    roofline = None
    kernel_ms = None
    if not args.no_profile and not sharded_run:
        prof = _lib.SortProfile()
        perm_p = torch.empty(n, dtype=torch.int64, device=device)
        SortPlan(n, D, cfg).run(dev, perm_p, None, prof)
        kernel_ms = {}
        for name in ("pass", "blur0", "blur1", "border", "distance", "control", "select"):
            ms, cnt = getattr(prof, f"ms_{name}"), getattr(prof, f"n_{name}")
            kernel_ms[name] = {"total_ms": round(ms, 3), "launches": int(cnt),
                               "avg_us": round(1e3 * ms / cnt, 2) if cnt else None}
        peak, peak_kind = measured_peak()
        S = (D + 3) // 4 * 4
        # every pass reads each cell's fp32 feature row and target row (8D bytes)
        alg_pass = n * 8 * D
        avg_pass_s = prof.ms_pass / prof.n_pass / 1e3
        blur_total = prof.ms_blur0 + prof.ms_blur1
        dominant = "pass_kernel" if prof.ms_pass >= blur_total else "blur"
        achieved = alg_pass / avg_pass_s / 1e9
        roofline = {"bound": "hbm", "kernel": "K3 pass kernels (pass_kernel_pipe gather + tile_pass_kernel: fused assign+swap)",
                    "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                    "algorithmic_bytes_per_launch": alg_pass, "avg_launch_us": round(avg_pass_s * 1e6, 2),
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                    "dominant_by_time": dominant,
                    "time_share_pass": round(prof.ms_pass / max(1e-9, prof.ms_pass + blur_total + prof.ms_border
                                                                  + prof.ms_distance + prof.ms_control), 3)}
        # the blur at large radius is fp64-compute-bound; its HBM fraction is reported for context
        alg_blur = n * 8 * D
        b_avg = (prof.ms_blur0 + prof.ms_blur1) / max(1, prof.n_blur0 + prof.n_blur1) / 1e3
        roofline["blur_hbm_frac"] = round(alg_blur / b_avg / 1e9 / peak, 4) if b_avg else None
        # ... and against its compute roof: analytic fp64 flops of every level's
        # blur over the blur kernels' CUDA-event time
        flops = blur_flops(side, D, [r for r, _ in rep["radius_trace"]])
        tf = flops / (blur_total / 1e3) / 1e12 if blur_total else None
        roofline["blur_fp64"] = {"flops_per_sort": flops, "achieved_tflops": round(tf, 2) if tf else None,
                                 "peak_tflops": FP64_PEAK_TFLOPS, "frac": round(tf / FP64_PEAK_TFLOPS, 4) if tf else None,
                                 "peak_source": "tools/fp64_micro.cu on this pool's B200 (DFMA 64/clk/SM), "
                                                "profiles/r02_fp64_peak.txt"}

    smooth = None
    if args.config == "C2" and not args.no_smoothness:
        smooth = run_smoothness(feats, perm_np, side, device, measured_peak()[0])
    prep = None
    if args.config == "C2" and not args.no_prep and rank == 0:
        prep = run_prep(device, measured_peak()[0])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(feats, WORKLOADS[args.config]["cfg"], args.cpu_budget,
                                   [len(t) - 1 for _, t in rep["radius_trace"]], "this GPU run's")

    # kernels launched per sort by our library (plas_b200.cu): 6 init + 5 final;
    # DEVICE (one graph) per level: set-up, border weight, blur (FFT: 2 + 2
    # fallback kernels for h >= 48 (side <= 1024) or 64; tile: 1 for h <= PLAS_TILE_BLUR_HMAX (default 0: off);
    # direct: 2 + 2), level
    # statistics, and the pass loop in iterations of PLAS_PASS_UNROLL (default 6)
    # passes (K3 + statistics each; the slots after the level's last pass
    # launch and return at once).
    # PARITY (host-stepped) per level: begin, 2 border, blur (FFT adds the
    # spectrum kernel), level statistics, level end; per pass: set-pass, class
    # select, K3, statistics.
    # plas_b200.cu fft_min_h: 40 for rows wider than 16 floats, else 48 when the
    # longest FFT length is <= 2048 (side 1024 -> 1536), 64 above
    fft_min_h = 40 if D > 16 else (48 if side <= 1024 else 64)

    def blur_launches(h, device):
        if h >= fft_min_h:
            return 4 if device else 5
        hmax = int(os.environ.get("PLAS_TILE_BLUR_HMAX", "0"))  # plas_b200.cu tile_blur_hmax(): off by default
        return 1 if h <= hmax and D <= 16 else 4
    per_level = []
    unroll = max(1, min(8, int(os.environ.get("PLAS_PASS_UNROLL", "6"))))  # plas_b200.cu pass_unroll()
    for r, tr in rep["radius_trace"]:
        h, p = math.ceil(r), len(tr) - 1
        if args.mode == "device":
            per_level.append(2 + blur_launches(h, True) + 1 + 2 * unroll * (-(-p // unroll)))
        else:
            per_level.append(3 + blur_launches(h, False) + 2 + 4 * p)
    launches = args.steps * (11 + sum(per_level))  # every timed step runs the same (deterministic) sort
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong" if sharded_run else "weak", "vs_baseline": None,
        "dtype": "f32 data, f64 accumulate", "data": "synthetic",
        "config": {"workload": f"{args.config} {side}x{side}x{D} PLAS sort to convergence "
                               f"(BASELINE.json configs[{args.config[1]}])",
                   "side": side, "dim": D, "rng_mode": args.mode, "seed": 0,
                   "sort_config": WORKLOADS[args.config]["cfg"] or "SortConfig defaults",
                   "l2": "256 MiB buffer written before every timed step (outside the events)",
                   "parallelism": (f"one grid sharded over {world} ranks (per-rank group ranges, NCCL "
                                   "all-gather of moved cells + fp64 partials per pass)") if sharded_run
                   else f"{world} independent grid(s), one per rank"},
        "quality": quality, "e2e": e2e, "roofline": roofline, "kernel_ms": kernel_ms, "smoothness": smooth, "prep": prep,
        "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return  # the reference arm runs on rank 0 only
    from paper_2312_13299_b200 import synthetic
    feats = synthetic.make(args.config, data_seed=0, side=args.side)
    n, D = feats.shape
    side = math.isqrt(n)
    budget = max(3.0, min(args.cpu_budget, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    samples = []
    for k in range(args.warmup + args.steps):
        r = cpu_reference_sample(feats, WORKLOADS[args.config]["cfg"], budget,
                                 reference_level_passes(args.config), "the reference's own seed-0 run")
        if k >= args.warmup:
            vals.append(r["value"])
            samples.append(r)
    v = statistics.mean(vals)
    last = samples[-1]
    line = {
        "metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(s.get("estimated_sort_s", n * sum(
            reference_level_passes(args.config) or [0]) / max(s["value"], 1)) for s in samples), 1),
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 data, f64 accumulate", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{args.config} {side}x{side}x{D} PLAS sort to convergence on the host CPU "
                               "(reference functions timed on a bounded sample per step, composed over "
                               "the full schedule; see cpu_baseline.sample)",
                   "side": side, "dim": D},
        "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
