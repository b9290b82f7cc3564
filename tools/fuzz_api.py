"""Randomised sweep of the non-sort entry points against their checkers:
blur_target (API, f32 and f64) and the sort's blur tiers vs the C oracle's
SciPy fold; grid_distance and vad vs NumPy's own expressions of the reference
(plas.py:71-84, metrics.py:25-40); reassign_block, quantize_planes,
prune_indices, normalize_for_sorting and smoothness_loss vs the oracle.  Shapes,
radii (past the grid too), and value ranges (1e-20 .. 1e20 scales, zeros,
constants, signed zeros) are drawn at random.  Prints every mismatch; exit 1
if any.   usage: python tools/fuzz_api.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_13299_b200 as plas  # noqa: E402
from paper_2312_13299_b200 import blur as gblur  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)


def values(shape):
    kind = int(g.integers(0, 6))
    if kind == 0:
        return g.normal(0, 1, shape)
    if kind == 1:
        return g.uniform(0, 1, shape)
    if kind == 2:
        return g.normal(0, 1, shape) * 10.0 ** g.uniform(-20, 20, (1,) * (len(shape) - 1) + (shape[-1],))
    if kind == 3:
        return np.full(shape, float(g.normal()))
    if kind == 4:
        v = g.normal(0, 1, shape)
        v[g.random(shape) < 0.5] = 0.0
        v[g.random(shape) < 0.1] = -0.0
        return v
    return g.integers(-3, 4, shape).astype(np.float64)


def np_grid_distance(a, b):  # plas.py:71-84, NumPy's own evaluation
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.sqrt(((a - b) ** 2).sum(axis=1)).mean())


def np_vad(grid):  # metrics.py:25-40
    gr = np.asarray(grid, dtype=np.float64)
    if gr.ndim == 2:
        gr = gr[..., None]
    d = np.concatenate([np.abs(np.diff(gr, axis=0)).ravel(), np.abs(np.diff(gr, axis=1)).ravel()])
    return float(d.var())


bad = 0
for c in range(cases):
    what = int(g.integers(0, 9))
    try:
        if what == 0:  # API blur, dtype preserving
            H, W, C = int(g.integers(1, 60)), int(g.integers(1, 60)), int(g.integers(1, 6))
            r = float(g.uniform(0.3, 1.5 * max(H, W)))
            dt = np.float32 if g.random() < 0.6 else np.float64
            x = values((H, W, C)).astype(dt)
            got, want = plas.blur_target(x, r), O.blur_target(x, r)
            ok = got.dtype == want.dtype and np.array_equal(got, want)
            tag = f"blur {H}x{W}x{C} {dt.__name__} r={r:.3f}"
        elif what == 1:  # the sort's tiers (direct / FFT) on a square grid
            side, C = int(g.integers(8, 200)), int(g.integers(1, 8))
            r = float(g.uniform(1.0, max(side / 2.0 - 1.0, 2.0)))
            tier = int(g.integers(0, 2))
            x = values((side, side, C)).astype(np.float32)
            got, _ = gblur.blur_target_tiers(x, r, tier)
            ok = np.array_equal(got, O.blur_target(x, r))
            tag = f"tiers {side}^2x{C} r={r:.3f} tier={tier}"
        elif what == 2:
            n, D = int(g.integers(1, 3000)), int(g.integers(1, 40))
            a, b = values((n, D)), values((n, D))
            got, want = plas.grid_distance(a, b), np_grid_distance(a, b)
            ok = got == want or (np.isnan(got) and np.isnan(want))
            tag = f"grid_distance n={n} D={D} {got!r} {want!r}"
        elif what == 3:
            H, W, C = int(g.integers(2, 80)), int(g.integers(2, 80)), int(g.integers(1, 6))
            x = values((H, W, C)).astype(np.float32 if g.random() < 0.6 else np.float64)
            got, want = plas.vad(x), np_vad(x)
            ok = got == want or (np.isnan(got) and np.isnan(want))
            tag = f"vad {H}x{W}x{C} {x.dtype} {got!r} {want!r}"
        elif what == 5:  # quantize / contract / plane packing vs the oracle
            import torch
            from paper_2312_13299_b200 import quantization as q
            from oracle import prep as oprep
            name = ["position", "sh_dc", "sh_rest", "rotation", "scale", "opacity"][int(g.integers(0, 6))]
            C = {"position": 3, "sh_dc": 3, "sh_rest": 45, "rotation": 4, "scale": 3, "opacity": 1}[name]
            n = int(g.integers(1, 3000))
            v = values((n, C))
            spec = q.default_quant_spec()[name]
            SPEC = {"position": (2 ** 14, None), "sh_dc": (2 ** 8, (-2.0, 4.0)), "sh_rest": (2 ** 5, (-1.0, 1.0)),
                    "opacity": (2 ** 6, (-6.0, 12.0)), "scale": (2 ** 6, None), "rotation": (2 ** 6, (-1.0, 2.0))}
            # (tests/test_quant.py SPEC: the oracle's levels / clip of default_quant_spec)
            levels, clip = SPEC[name]
            planes, lo, hi = oprep.quantize_attribute_planes(name, v, levels, clip)
            images, glo, ghi = q.quantize_planes(name, torch.from_numpy(v).cuda(), spec)
            ok = (np.array_equal(images.cpu().numpy().astype(np.int64), planes)
                  and np.array_equal(np.array(glo), lo) and np.array_equal(np.array(ghi), hi))
            tag = f"quantize {name} n={n}"
        elif what == 6:  # prune survivors vs the oracle
            from paper_2312_13299_b200.splats import prune_indices
            from oracle import prep as oprep
            n = int(g.integers(1, 5000))
            x = values((n, 1))[:, 0]
            keep = int(g.integers(1, n + 1))
            ok = np.array_equal(prune_indices(x, keep).cpu().numpy(), oprep.prune_survivors(x, keep))
            tag = f"prune n={n} keep={keep}"
        elif what == 7:  # normalize_for_sorting vs the oracle (activations: <= 4 ulp)
            from paper_2312_13299_b200.splats import normalize_features
            from oracle import prep as oprep
            n = int(g.integers(1, 3000))
            chans = {"position": 3, "sh_dc": 3, "sh_rest": 45 if g.random() < 0.3 else 0, "opacity": 1,
                     "scale": 3, "rotation": 4}
            attrs = {}
            for a, C in chans.items():
                v = values((n, C)) if C else np.zeros((n, 0))
                if a in ("opacity", "scale"):
                    v = np.clip(v, -50.0, 50.0)  # finite activations
                attrs[a] = v
            wts = {a: float(g.choice([0.0, 0.5, 1.0, 2.0])) for a in chans}
            feats, mins, maxs = normalize_features(attrs, wts)
            ofe, omi, oma = oprep.normalize_columns(attrs, wts)
            feats = feats.cpu().numpy()

            def ulp(a, b):
                a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
                b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
                return int(np.abs(a - b).max(initial=0))
            ok = feats.shape == ofe.shape
            why = ""
            for a in chans:
                tol = 4 if a in ("opacity", "scale") else 0
                um, uM = ulp(mins[a].cpu().numpy(), omi[a]), ulp(maxs[a].cpu().numpy(), oma[a])
                if um > tol or uM > tol:
                    ok = False
                    why += f" {a}: min/max ulp {um}/{uM}"
            if ok:
                col = 0
                for a in ("position", "sh_dc", "sh_rest", "opacity", "scale", "rotation"):
                    C = chans[a]
                    if wts[a] == 0.0 or C == 0:
                        continue
                    got, exp = feats[:, col:col + C], ofe[:, col:col + C]
                    if a in ("opacity", "scale"):
                        # a last-bit difference of the activation (NumPy's SIMD exp is not
                        # correctly rounded) is amplified by the affine map to ~ulp(max|v|) / span
                        act = oprep.activate(a, attrs[a]).reshape(n, -1)
                        span = np.maximum(oma[a] - omi[a], 1e-300)
                        amp = 8 * np.spacing(np.abs(act).max(axis=0)) / span * wts[a]
                        good = bool(np.all(np.abs(got - exp) <= amp + 1e-15 * wts[a]))
                    else:
                        good = bool(np.array_equal(got, exp))
                    if not good:
                        ok = False
                        why += f" {a}: features"
                    col += C
            tag = f"normalize n={n} weights={wts}{why}"
        elif what == 8:  # smoothness_loss vs the oracle (loss and gradients exact)
            side = int(g.integers(2, 40))
            names = [nm for nm in ("position", "sh_dc", "scale", "rotation", "opacity") if g.random() < 0.6] or ["opacity"]
            chans = {"position": 3, "sh_dc": 3, "scale": 3, "rotation": 4, "opacity": 1}
            planes = {nm: values((side, side, chans[nm])) for nm in names}
            ks = int(g.choice([1, 3, 5, 7, 9, 11, 13, 21, 41]))
            params = plas.SmoothnessParams(kernel_size=ks, sigma=float(g.uniform(0.3, 8.0)),
                                           overall_multiplier=float(g.uniform(0.1, 3.0)),
                                           huber_delta=float(10 ** g.uniform(-3, 2)),
                                           weights={nm: float(g.choice([0.0, 0.3, 1.0])) for nm in names},
                                           detach_target=bool(g.random() < 0.3))
            loss, grads = plas.smoothness_loss(plas.GridStack(plas.GridLayout(side), planes), params)
            total, ok = 0.0, True
            for nm in names:
                coeff = params.overall_multiplier * params.weights.get(nm, 0.0)
                if coeff == 0.0:
                    ok &= bool(np.all(grads[nm] == 0.0))
                    continue
                l1, g1 = O.smoothness_plane(planes[nm], coeff, params.huber_delta, params.detach_target,
                                            params.sigma, params.kernel_size)
                total += l1
                ok &= bool(np.array_equal(grads[nm], g1))
            ok &= loss == total
            tag = f"smoothness side={side} k={ks} planes={names} {loss!r} {total!r}"
        else:
            m, D = int(g.integers(1, 40)), int(g.integers(1, 20))
            n = m + int(g.integers(0, 10))
            feat = values((n, D)).astype(np.float32)
            target = values((n, D)).astype(np.float32)
            idx = np.arange(n, dtype=np.int64)
            positions = g.permutation(n)[:m]
            grouping = g.permutation(m + int(g.integers(0, 5)))
            f1, i1 = feat.copy(), idx.copy()
            f2, i2 = feat.copy(), idx.copy()
            plas.reassign_block(f1, i1, target, positions, grouping)
            O.reassign_block(f2, i2, target, positions, grouping)
            ok = np.array_equal(f1, f2) and np.array_equal(i1, i2)
            tag = f"reassign m={m} n={n} D={D}"
    except Exception as e:  # noqa: BLE001
        ok = False
        tag = f"case kind {what}: {e!r}"[:300]
    if not ok:
        bad += 1
        print("MISMATCH", c, tag)
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
