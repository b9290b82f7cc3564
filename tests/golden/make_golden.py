"""Generate the golden fixtures by running the UNMODIFIED reference here.

The reference (`/root/reference/pkg/src/sogs`) is pure Python + numba + SciPy
and can only be imported in the build container; the GPU box has no
`/root/reference`.  This script imports it read-only (numba's on-disk cache is
redirected to /tmp so nothing is written into the reference tree) and stores
small fixtures under tests/golden/ that the CPU oracle tests and the GPU parity
tests compare against.

Usage:  python tests/golden/make_golden.py PART [PART ...]
PART in: versions rng blur assign metrics bench smooth sort_small c0 c1 c2 paired_null_c0 paired_null_c1
"""

import hashlib
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import sogs  # noqa: E402  (the reference)
from sogs import plas as ref_plas  # noqa: E402
from sogs import blur as ref_blur  # noqa: E402
from sogs import metrics as ref_metrics  # noqa: E402
from sogs import smoothness as ref_smooth  # noqa: E402
from sogs.splats import GridLayout, GridStack  # noqa: E402

from paper_2312_13299_b200 import synthetic  # noqa: E402


def out(name):
    return os.path.join(HERE, name)


def perm_sha(perm):
    return hashlib.sha256(np.asarray(perm, dtype="<i8").tobytes()).hexdigest()


def report_dict(report):
    radii, counts, values = [], [], []
    for r, trace in report.radius_trace:
        radii.append(float(r))
        counts.append(len(trace))
        values.extend(float(v) for v in trace)
    return {
        "initial_vad": float(report.initial_vad),
        "final_vad": float(report.final_vad),
        "reorders": int(report.reorders),
        "radii": radii,
        "counts": counts,
        "values": values,
    }


def part_versions():
    import numba
    import scipy
    info = {
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "numba": numba.__version__,
        "python": sys.version.split()[0],
        "reference": "sogs " + sogs.__version__ + " (/root/reference/pkg)",
    }
    with open(out("versions.json"), "w") as f:
        json.dump(info, f, indent=1)


def part_rng():
    """Pins NumPy's Generator(Philox) stream as the reference draws it (plas.py:240-262)."""
    cases = []
    for seed in (0, 1, 5, 12345, 2 ** 40 + 7):
        key = np.random.SeedSequence(seed).generate_state(2, np.uint64)
        rng = np.random.Generator(np.random.Philox(seed))
        seq = []
        seq.append(["perm", 37, rng.permutation(37).tolist()])
        for beta in (16, 17, 33, 100, 512):
            seq.append(["int", beta, int(rng.integers(0, beta))])
            seq.append(["int", beta, int(rng.integers(0, beta))])
            seq.append(["perm", beta * beta if beta < 100 else beta, rng.permutation(
                beta * beta if beta < 100 else beta).tolist()])
        seq.append(["perm", 1, rng.permutation(1).tolist()])
        seq.append(["perm", 2, rng.permutation(2).tolist()])
        big = rng.permutation(70000)
        seq.append(["perm_sha", 70000, perm_sha(big)])
        seq.append(["int", 3, int(rng.integers(0, 3))])
        cases.append({"seed": seed, "key": [int(k) for k in key], "draws": seq})
    with open(out("rng.json"), "w") as f:
        json.dump(cases, f)


def blur_input(seed, side, dim):
    return np.random.default_rng(seed).normal(0.0, 1.0, (side, side, dim)).astype(np.float32)


def part_blur():
    """Bit patterns of blur_target (f32, plas.py:64-68) and renormalized_blur (f64, blur.py:18-30)."""
    arrays = {}
    meta = []
    i = 0
    for side, dim in ((37, 3), (64, 14), (33, 6), (16, 1)):
        # inputs are regenerated from blur_input(seed) by the tests; big outputs stored as sha256
        grid = blur_input(1000 + side, side, dim)
        for radius in (1.0, 1.9, 2.5, 7.3, 15.5, max(side / 2.0 - 1.0, 2.0), 40.0):
            tgt = ref_plas.blur_target(grid, radius)
            assert tgt.dtype == np.float32
            entry = {"i": i, "side": side, "dim": dim, "radius": radius, "dtype": "f32",
                     "seed": 1000 + side, "sha": hashlib.sha256(tgt.tobytes()).hexdigest()}
            if side * side * dim <= 37 * 37 * 3:
                arrays[f"out{i}"] = tgt
            meta.append(entry)
            i += 1
    rng = np.random.default_rng(11)
    for shape, sigma, radius in (((8, 9, 2), 0.5, 1), ((8, 9, 2), 1.0, 2), ((8, 9, 2), 2.5, 5),
                                 ((7, 7), 1.0, 2), ((12, 5, 4), 3.0, 2), ((30, 30, 3), 7.0, 14)):
        grid = rng.uniform(0.0, 1.0, shape)
        arrays[f"in{i}"] = grid
        arrays[f"out{i}"] = ref_blur.renormalized_blur(grid, sigma, radius)
        arrays[f"sep{i}"] = ref_blur.separable_blur(grid, sigma, radius)
        arrays[f"den{i}"] = ref_blur.border_weight(grid.shape, sigma, radius)
        meta.append({"i": i, "shape": list(shape), "sigma": sigma, "radius": radius, "dtype": "f64"})
        i += 1
    np.savez_compressed(out("blur.npz"), **arrays)
    with open(out("blur.json"), "w") as f:
        json.dump(meta, f)


def part_assign():
    """reassign_block (plas.py:173-193) on random blocks, incl. leftovers and ties."""
    rng = np.random.default_rng(21)
    arrays = {}
    cases = 0
    for _ in range(200):
        m = int(rng.integers(2, 40))
        n = m + int(rng.integers(0, 10))
        D = int(rng.integers(1, 20))
        feat = rng.uniform(0, 1, (n, D)).astype(np.float32)
        if rng.random() < 0.2:  # exact ties
            feat = np.round(feat * 2).astype(np.float32) / 2
        target = rng.uniform(0, 1, (n, D)).astype(np.float32)
        if rng.random() < 0.2:
            target = np.round(target * 2).astype(np.float32) / 2
        positions = rng.permutation(n)[:m].astype(np.int64)
        grouping = rng.permutation(m + int(rng.integers(0, 5))).astype(np.int64)
        f = feat.copy()
        idx = np.arange(n, dtype=np.int64)
        ref_plas.reassign_block(f, idx, target, positions, grouping)
        arrays[f"feat{cases}"] = feat
        arrays[f"target{cases}"] = target
        arrays[f"positions{cases}"] = positions
        arrays[f"grouping{cases}"] = grouping
        arrays[f"idx_out{cases}"] = idx
        arrays[f"feat_out{cases}"] = f
        cases += 1
    arrays["count"] = np.array(cases)
    np.savez_compressed(out("assign.npz"), **arrays)


def part_metrics():
    rng = np.random.default_rng(31)
    arrays = {}
    for i, shape in enumerate([(2, 2), (3, 5), (6, 4, 3), (24, 24, 14), (17, 33, 1)]):
        g = rng.uniform(0, 255, shape)
        arrays[f"vad_in{i}"] = g
        arrays[f"vad_out{i}"] = np.array(ref_metrics.vad(g))
    for i, shape in enumerate([(16, 3), (4, 4, 3), (300, 14)]):
        a = rng.normal(0, 1, shape)
        b = rng.normal(0, 1, shape)
        w = rng.uniform(0.5, 2.0, shape[-1])
        arrays[f"gd_a{i}"] = a
        arrays[f"gd_b{i}"] = b
        arrays[f"gd_w{i}"] = w
        arrays[f"gd_out{i}"] = np.array(ref_plas.grid_distance(a, b))
        arrays[f"gd_outw{i}"] = np.array(ref_plas.grid_distance(a, b, weights=w))
    np.savez_compressed(out("metrics.npz"), **arrays)


def part_bench():
    """metrics.bench_sort rows (minus the wall time), its CSV, and attribute_psnr cases."""
    rows = ref_metrics.bench_sort([2, 8, 16], channels=3, seeds=(0, 1))
    rows += ref_metrics.bench_sort([12], channels=5, seeds=(7,))
    keep = [{k: v for k, v in r.items() if k != "time_s"} for r in rows]
    fixed = [dict(r, time_s=0.125) for r in rows]
    rng = np.random.default_rng(5)
    psnr = []
    for shape, peak in [((16, 16), 255.0), ((7, 9, 3), 1.0), ((33,), 2.5)]:
        a = rng.uniform(0, peak, shape)
        b = np.clip(a + rng.normal(0, 0.01 * peak, shape), 0, peak)
        psnr.append({"a": a.ravel().tolist(), "b": b.ravel().tolist(), "shape": list(shape), "peak": peak,
                     "psnr": ref_metrics.attribute_psnr(a, b, peak)})
    with open(out("bench.json"), "w") as f:
        json.dump({"rows": keep, "csv_rows": fixed, "csv": ref_metrics.bench_rows_to_csv(fixed),
                   "fields": list(ref_metrics.BENCH_CSV_FIELDS), "psnr": psnr}, f)


def part_smooth():
    """smoothness_loss (smoothness.py:57-97) on small stacks."""
    rng = np.random.default_rng(41)
    arrays = {}
    meta = []
    channels = {"opacity": 1, "rotation": 4, "sh_dc": 3, "scale": 3, "position": 3}
    i = 0
    for side, names, kw in ((6, ("opacity", "rotation"), {}),
                            (8, ("opacity", "rotation"), {"huber_delta": 0.25, "overall_multiplier": 1.7}),
                            (5, ("opacity", "rotation"), {"detach_target": True, "huber_delta": 0.8}),
                            (33, tuple(channels), {"weights": {k: 0.3 for k in channels}}),
                            (16, ("rotation",), {"kernel_size": 7, "sigma": 1.5}),
                            (9, ("opacity",), {"kernel_size": 1}),
                            (20, ("rotation", "opacity"), {"kernel_size": 13, "sigma": 3.0}),
                            (12, ("opacity", "sh_dc"), {"kernel_size": 41, "sigma": 10.0})):
        planes = {n: rng.normal(0, 1.5, (side, side, channels[n])) for n in names}
        params = ref_smooth.SmoothnessParams(**kw)
        loss, grads = ref_smooth.smoothness_loss(GridStack(layout=GridLayout(side), planes=planes), params)
        for n in names:
            arrays[f"{i}_in_{n}"] = planes[n]
            arrays[f"{i}_grad_{n}"] = grads[n]
        meta.append({"i": i, "side": side, "names": list(names), "params": kw, "loss": loss})
        i += 1
    np.savez_compressed(out("smooth.npz"), **arrays)
    with open(out("smooth.json"), "w") as f:
        json.dump(meta, f)


def sort_case(features, cfg_kw, initial_radius=None):
    cfg = ref_plas.SortConfig(**cfg_kw)
    saved = ref_plas.initial_radius
    if initial_radius is not None:
        ref_plas.initial_radius = lambda side: float(initial_radius)
    try:
        t0 = time.perf_counter()
        perm, report = ref_plas.sort_grid_report(features, cfg, threads=1)
        elapsed = time.perf_counter() - t0
    finally:
        ref_plas.initial_radius = saved
    side = int(round(len(perm) ** 0.5))
    grid = np.asarray(features, dtype=np.float64)[perm].reshape(side, side, -1)
    d = report_dict(report)
    d["nbr_l2"] = synthetic.neighbour_l2(grid)
    d["sha"] = perm_sha(perm)
    d["time_s"] = elapsed
    d["cfg"] = cfg_kw
    d["initial_radius"] = initial_radius
    return perm, d


def part_sort_small():
    """The reference test suite's sort inputs (tests/test_plas.py:230-315 shapes) + edge cases."""
    cases = []
    arrays = {}

    def add(name, features, cfg_kw, initial_radius=None):
        perm, d = sort_case(features, cfg_kw, initial_radius)
        d["name"] = name
        arrays[f"features_{name}"] = np.asarray(features, dtype=np.float64)
        arrays[f"perm_{name}"] = np.asarray(perm, dtype=np.int64)
        cases.append(d)

    rng = np.random.default_rng(0)
    add("bij64", rng.uniform(0, 1, (64, 3)), {"rng_seed": 1})
    rng = np.random.default_rng(2)
    f = rng.uniform(0, 1, (256, 3))
    add("det256_s5", f, {"rng_seed": 5})
    add("det256_s6", f, {"rng_seed": 6})
    rng = np.random.default_rng(3)
    add("vad32", rng.uniform(0, 1, (32 * 32, 3)), {"rng_seed": 0})
    add("const16", np.zeros((16, 2)), {"rng_seed": 0})
    for seed in range(4):
        add(f"mono2x2_s{seed}", np.array([[0.0], [1.0], [2.0], [3.0]]) / 3.0, {"rng_seed": seed})
    rng = np.random.default_rng(4)
    add("trace24", rng.uniform(0, 1, (24 * 24, 3)), {"rng_seed": 0})
    rng = np.random.default_rng(5)
    add("thr40", rng.uniform(0, 1, (40 * 40, 3)), {"rng_seed": 3})
    rng = np.random.default_rng(6)
    add("d1_side9", rng.uniform(0, 1, (81, 1)), {"rng_seed": 2})
    add("d8_side23", rng.normal(0, 1, (23 * 23, 8)), {"rng_seed": 7, "min_block_size": 4})
    add("d20_side17", rng.normal(0, 1, (17 * 17, 20)), {"rng_seed": 8, "radius_decay": 0.7})
    add("side3", rng.uniform(0, 1, (9, 2)), {"rng_seed": 9})
    add("side2", rng.uniform(0, 1, (4, 5)), {"rng_seed": 10})
    add("ties", np.round(rng.uniform(0, 1, (48 * 48, 2)) * 3) / 3, {"rng_seed": 11})
    add("d70_side12", rng.normal(0, 1, (144, 70)), {"rng_seed": 12})
    np.savez_compressed(out("sort_small.npz"), **arrays)
    with open(out("sort_small.json"), "w") as f:
        json.dump(cases, f)


def part_c0():
    """BASELINE configs[0]: 64x64x3 uniform, decay 0.5, threshold 1e-5; seeds 0-9 (+ r0=32 override)."""
    features = synthetic.c0(0)
    cases = []
    perms = {}
    for seed in range(10):
        perm, d = sort_case(features, {"rng_seed": seed, "radius_decay": 0.5, "improvement_threshold": 1e-5})
        perms[f"s{seed}"] = perm.astype(np.uint16)
        cases.append(d)
    for seed in range(4):
        perm, d = sort_case(features, {"rng_seed": seed, "radius_decay": 0.5, "improvement_threshold": 1e-5},
                            initial_radius=32.0)
        perms[f"r32_s{seed}"] = perm.astype(np.uint16)
        cases.append(d)
    np.savez_compressed(out("c0.npz"), **perms)
    with open(out("c0.json"), "w") as f:
        json.dump(cases, f)


def part_c1():
    """BASELINE configs[1]: 256x256x6 GMM, default SortConfig; seeds 0-3."""
    features = synthetic.c1(0)
    cases = []
    perms = {}
    for seed in range(int(os.environ.get("C1_SEEDS", "4"))):
        perm, d = sort_case(features, {"rng_seed": seed})
        perms[f"s{seed}"] = perm.astype(np.uint16)
        cases.append(d)
        print("c1", seed, d["reorders"], d["time_s"], flush=True)
    np.savez_compressed(out("c1.npz"), **perms)
    with open(out("c1.json"), "w") as f:
        json.dump(cases, f)


def part_c2():
    """BASELINE configs[2]: 1024x1024x14; seed 0. Stores the perm sha256 + head (4 MiB perm not committed)."""
    features = synthetic.c2(0)
    perm, d = sort_case(features, {"rng_seed": 0})
    d["head"] = perm[:256].tolist()
    d["tail"] = perm[-256:].tolist()
    with open(out("c2.json"), "w") as f:
        json.dump(d, f)
    print("c2", d["reorders"], d["time_s"], d["nbr_l2"], flush=True)


class _SplitStreamGenerator:
    """Generator stand-in for the null arm of the paired protocol: the first
    permutation(n) (draw #1, plas.py:241) comes from Generator(Philox(seed)),
    every later draw (plas.py:260-262) from the independent Generator(Philox(seed + offset))."""

    def __init__(self, seed, offset):
        self._init = np.random.Generator(np.random.Philox(seed))
        self._pass = np.random.Generator(np.random.Philox(seed + offset))
        self._first = True

    def permutation(self, n):
        if self._first:
            self._first = False
            return self._init.permutation(n)
        return self._pass.permutation(n)

    def integers(self, *a, **k):
        return self._pass.integers(*a, **k)


class _NumpyShim:
    def __init__(self, seed, offset):
        import types
        self.random = types.SimpleNamespace(
            Generator=lambda bitgen: _SplitStreamGenerator(seed, offset), Philox=lambda s: None)

    def __getattr__(self, name):
        return getattr(np, name)


def _null_run(args):
    """One reference sort (the unmodified sogs code path) with draw #1 from `seed`
    and every pass draw from an independent stream `seed + offset`."""
    features, cfg_kw, seed, offset = args
    ref_plas.np = _NumpyShim(seed, offset)
    try:
        perm, _ = ref_plas.sort_grid_report(features, ref_plas.SortConfig(rng_seed=seed, **cfg_kw), threads=1)
    finally:
        ref_plas.np = np
    side = int(round(len(perm) ** 0.5))
    return synthetic.neighbour_l2(np.asarray(features, dtype=np.float64)[perm].reshape(side, side, -1))


def _own_run(args):
    features, cfg_kw, seed = args
    _, d = sort_case(features, dict(cfg_kw, rng_seed=seed))
    return d["nbr_l2"]


def _paired_null(name, features, cfg_kw, seeds, offsets=(1000, 2000)):
    """Reference runs per seed for the paired DEVICE-mode protocol:
    `ref` = the reference's own stream; `null` = reference-law runs that share only
    the initial permutation (the noise floor an equal-in-law stream must match)."""
    from multiprocessing import Pool
    sort_case(np.random.default_rng(0).random((64, 3)), {})  # numba JIT before the workers fork
    with Pool(os.cpu_count()) as pool:
        own = pool.map(_own_run, [(features, cfg_kw, s) for s in seeds])
        nulls = pool.map(_null_run, [(features, cfg_kw, s, o) for s in seeds for o in offsets])
    rows = []
    for i, s in enumerate(seeds):
        rows.append({"seed": s, "nbr_l2": own[i], "null_offsets": list(offsets),
                     "null_nbr_l2": nulls[i * len(offsets):(i + 1) * len(offsets)]})
    with open(out(name), "w") as f:
        json.dump({"cfg": cfg_kw, "rows": rows}, f)


def part_paired_null_c0():
    _paired_null("paired_null_c0.json", synthetic.c0(0), {"radius_decay": 0.5, "improvement_threshold": 1e-5},
                 list(range(int(os.environ.get("PAIRED_C0", "80")))))


def part_paired_null_c1():
    _paired_null("paired_null_c1.json", synthetic.c1(0), {}, list(range(int(os.environ.get("PAIRED_C1", "32")))))


def _prep_cloud(seed, n, sh_rest, ties=False):
    g = np.random.default_rng(seed)
    logit = g.normal(0.0, 2.0, n)
    if ties:  # heavy ties, and both signed zeros
        logit = np.round(logit, 1)
        logit[g.integers(0, n, n // 20)] = 0.0
        logit[g.integers(0, n, n // 20)] = -0.0
    return dict(positions=g.normal(0, 3, (n, 3)), sh_dc=g.normal(0, 0.5, (n, 3)),
                sh_rest=g.normal(0, 0.1, (n, sh_rest)), opacity_logit=logit,
                scale_log=g.normal(-4, 1, (n, 3)), rotation=g.normal(0, 1, (n, 4)))


def part_prep():
    """prune_to_grid + normalize_for_sorting (splats.py:139-216) on seeded clouds,
    run by the reference; inputs and outputs to prep.npz."""
    from sogs import splats as ref_splats
    arrays = {}
    cases = [("a", 0, 1500, 45, True, None), ("b", 1, 300, 0, False, {"opacity": 0.5, "rotation": 2.0}),
             ("c", 2, 530, 45, True, {"sh_rest": 0.25, "position": 0.0}),
             ("d", 3, 64, 0, False, {k: 0.0 for k in ("position", "sh_dc", "scale")})]
    for name, seed, n, shr, ties, weights in cases:
        cl = _prep_cloud(seed, n, shr, ties)
        if name == "c":  # one constant channel
            cl["sh_dc"][:, 1] = 0.25
        cloud = ref_splats.SplatCloud(**cl)
        layout = ref_splats.build_grid_layout(n)
        pruned = ref_splats.prune_to_grid(cloud, layout)
        order = np.argsort(cloud.opacity_logit, kind="stable")
        survivors = np.sort(order[cloud.n - layout.cells:])
        assert np.array_equal(pruned.positions, cloud.positions[survivors])
        feats, spec = ref_splats.normalize_for_sorting(pruned, weights)
        for k, v in cl.items():
            arrays[f"{name}_in_{k}"] = v
        arrays[f"{name}_keep"] = np.int64(layout.cells)
        arrays[f"{name}_survivors"] = survivors.astype(np.int64)
        arrays[f"{name}_features"] = feats
        for k in ref_splats.ATTRIBUTES:
            arrays[f"{name}_min_{k}"] = spec.mins[k]
            arrays[f"{name}_max_{k}"] = spec.maxs[k]
        arrays[f"{name}_weights"] = np.array([spec.weights[k] for k in ref_splats.ATTRIBUTES])
    np.savez_compressed(out("prep.npz"), **arrays)


def part_quant():
    """bundle.compress's per-attribute quantization (bundle.py:102-115, 158-176,
    quantization.py:8-41) by the reference on a seeded grid-ordered cloud:
    values -> pixel planes (uint16) and manifest lo / hi, to quant.npz."""
    from sogs import bundle as ref_bundle
    from sogs import quantization as ref_q
    arrays = {}
    side = 24
    n = side * side
    cl = _prep_cloud(7, n, 45, ties=False)
    cl["positions"][:5] = [[0.0, -0.0, 1e-300], [5e3, -5e3, 0.5], [1.0, 1.0, 1.0], [-1.0, 2.0, -3.0], [0, 0, 0]]
    cl["scale_log"][:, 2] = -3.0  # a constant data-driven channel
    cl["sh_dc"][:3] = [[-9.0, 9.0, 1.0], [4.0, -2.0, 0.0], [3.999999, -1.999999, 0.5]]  # clipping
    cloud = ref_splats_cloud(cl)
    spec = ref_q.default_quant_spec()
    for name in ref_bundle.ATTRIBUTES:
        values = cloud.attribute(name)
        if values.shape[1] == 0:
            continue
        if name == "position":
            values = ref_q.contract(values)
        indices, lo, hi = ref_bundle._quantize_attribute(values, spec[name])
        per_image, count = ref_bundle.PLANE_GROUPS[name]
        needed = values.shape[1] // per_image
        planes = np.stack([indices[:, i * per_image:(i + 1) * per_image] for i in range(needed)])
        arrays[f"{name}_in"] = cloud.attribute(name)
        arrays[f"{name}_planes"] = planes.astype(np.uint16)
        arrays[f"{name}_lo"] = np.array(lo)
        arrays[f"{name}_hi"] = np.array(hi)
    np.savez_compressed(out("quant.npz"), **arrays)


def ref_splats_cloud(cl):
    from sogs import splats as ref_splats
    return ref_splats.SplatCloud(**cl)


PARTS = {k[5:]: v for k, v in globals().items() if k.startswith("part_")}

if __name__ == "__main__":
    for name in sys.argv[1:]:
        t0 = time.time()
        PARTS[name]()
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)
