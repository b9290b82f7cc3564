"""Caller-side feature preparation: prune_to_grid and
normalize_for_sorting (splats.py:139-216) and the row gather (bundle.py:160).

CPU: the oracle restatement (oracle/prep.py) against the reference-generated
fixtures (tests/golden/prep.npz, make_golden.py part_prep).
GPU: the CUDA path against the same fixtures -- survivors bit-exact
(index work); features bit-exact for the channels without activation and
within 4 ulp for sigmoid / exp channels (the GPU's exp and NumPy's exp are
both faithful but not correctly rounded, so they may differ in the last bit).
"""
import os

import numpy as np
import pytest

from oracle import prep as oprep

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "prep.npz"))
CASES = sorted({k.split("_")[0] for k in G.files})
ATTRS = ("position", "sh_dc", "sh_rest", "opacity", "scale", "rotation")
FIELDS = ("positions", "sh_dc", "sh_rest", "opacity_logit", "scale_log", "rotation")
ATTR_OF = dict(zip(ATTRS, FIELDS))


def case_inputs(c):
    return {f: G[f"{c}_in_{f}"] for f in FIELDS}


def weights_of(c):
    return dict(zip(ATTRS, G[f"{c}_weights"].tolist()))


def pruned_attrs(c):
    cl = case_inputs(c)
    s = G[f"{c}_survivors"]
    out = {}
    for a, f in ATTR_OF.items():
        v = cl[f][s]
        out[a] = v.reshape(v.shape[0], -1)
    return out


@pytest.mark.parametrize("c", CASES)
def test_oracle_prune_matches_reference(c):
    got = oprep.prune_survivors(G[f"{c}_in_opacity_logit"], int(G[f"{c}_keep"]))
    assert np.array_equal(got, G[f"{c}_survivors"])


@pytest.mark.parametrize("c", CASES)
def test_oracle_normalize_matches_reference(c):
    feats, mins, maxs = oprep.normalize_columns(pruned_attrs(c), weights_of(c))
    assert np.array_equal(feats, G[f"{c}_features"])
    for a in ATTRS:
        assert np.array_equal(mins[a], G[f"{c}_min_{a}"]) and np.array_equal(maxs[a], G[f"{c}_max_{a}"])


def test_oracle_prune_edge_cases():
    x = np.array([0.5, -0.0, 0.0, 0.5, -1.0, 2.0, 0.5])
    assert oprep.prune_survivors(x, 4).tolist() == [0, 3, 5, 6]  # ties by index, -0 == +0
    assert oprep.prune_survivors(x, 7).tolist() == list(range(7))
    assert oprep.prune_survivors(x, 1).tolist() == [5]


def ulp_diff(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(a - b)


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES)
def test_gpu_prune_matches_reference(c):
    from paper_2312_13299_b200.splats import prune_indices
    got = prune_indices(G[f"{c}_in_opacity_logit"], int(G[f"{c}_keep"])).cpu().numpy()
    assert np.array_equal(got, G[f"{c}_survivors"])


@pytest.mark.gpu
def test_gpu_prune_edge_cases_and_sizes():
    from paper_2312_13299_b200.splats import prune_indices
    x = np.array([0.5, -0.0, 0.0, 0.5, -1.0, 2.0, 0.5])
    for keep in range(1, 8):
        assert np.array_equal(prune_indices(x, keep).cpu().numpy(), oprep.prune_survivors(x, keep))
    g = np.random.default_rng(5)
    for n in (1, 2, 4095, 4096, 4097, 100_003):
        for kind in ("normal", "ties", "const", "extreme"):
            if kind == "normal":
                x = g.normal(size=n)
            elif kind == "ties":
                x = g.integers(-3, 4, n).astype(np.float64) * 0.5
                x[g.integers(0, n, max(n // 10, 1))] = -0.0
            elif kind == "const":
                x = np.full(n, 1.5)
            else:
                x = g.choice([-1e308, -5e-324, 0.0, 5e-324, 1e308, 1.0], n)
            for keep in {1, max(n // 3, 1), n - 1 if n > 1 else 1, n}:
                got = prune_indices(x, keep).cpu().numpy()
                assert np.array_equal(got, oprep.prune_survivors(x, keep)), (n, kind, keep)
    with pytest.raises(ValueError):
        prune_indices(np.zeros(3), 4)


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES)
def test_gpu_normalize_matches_reference(c):
    from paper_2312_13299_b200.splats import normalize_features
    feats, mins, maxs = normalize_features(pruned_attrs(c), weights_of(c))
    feats = feats.cpu().numpy()
    ref = G[f"{c}_features"]
    assert feats.shape == ref.shape
    w = weights_of(c)
    col = 0
    for a in ATTRS:
        ch = pruned_attrs(c)[a].shape[1]
        lo, hi = mins[a].cpu().numpy(), maxs[a].cpu().numpy()
        tol = 0 if a not in ("opacity", "scale") else 4
        assert ulp_diff(lo, G[f"{c}_min_{a}"]).max(initial=0) <= tol, a
        assert ulp_diff(hi, G[f"{c}_max_{a}"]).max(initial=0) <= tol, a
        if w[a] == 0.0 or ch == 0:
            continue
        got, exp = feats[:, col:col + ch], ref[:, col:col + ch]
        if tol == 0:
            assert np.array_equal(got, exp), a
        else:  # the affine map amplifies a last-bit exp difference by at most span / value
            np.testing.assert_allclose(got, exp, rtol=1e-12, atol=1e-14 * max(w[a], 1.0), err_msg=a)
        col += ch


@pytest.mark.gpu
def test_gpu_reference_api_round_trip():
    import paper_2312_13299_b200 as plas
    cl = case_inputs("a")
    cloud = plas.SplatCloud(**cl)
    layout = plas.build_grid_layout(cloud.n)
    pruned = plas.prune_to_grid(cloud, layout)
    s = G["a_survivors"]
    for f in FIELDS:
        assert np.array_equal(getattr(pruned, f), np.asarray(cl[f], dtype=np.float64)[s]), f
    feats, spec = plas.normalize_for_sorting(pruned)
    np.testing.assert_allclose(feats, G["a_features"], rtol=1e-12, atol=1e-14)
    assert spec.weights == dict(zip(ATTRS, G["a_weights"].tolist()))


@pytest.mark.gpu
def test_gpu_gather_rows_bit_exact():
    import torch
    from paper_2312_13299_b200.splats import gather_rows
    g = np.random.default_rng(3)
    perm = torch.from_numpy(g.permutation(1000)).cuda()
    for shape, dt in (((1000, 45), torch.float64), ((1000, 3), torch.float64), ((1000,), torch.float64),
                      ((1000, 14), torch.float32), ((1000, 3), torch.uint8), ((1000, 4), torch.int16)):
        t = (torch.randn(shape, dtype=torch.float64) * 100).to(dt).cuda()
        assert torch.equal(gather_rows(t, perm), t[perm]), (shape, dt)
