"""The C oracle (oracle/plas_oracle.c) against fixtures produced by the real reference.

This is what pins the oracle: every fixture below was written by
tests/golden/make_golden.py running /root/reference's sogs package.
"""

import hashlib

import numpy as np
import pytest

from conftest import blur_input, golden_json, golden_npz
from oracle import oracle as O
from paper_2312_13299_b200 import synthetic


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_seed_keys_and_draw_stream():
    for case in golden_json("rng.json"):
        assert O.seed_key(case["seed"]) == case["key"]
        r = O.Rng(case["seed"])
        for kind, n, val in case["draws"]:
            if kind == "perm":
                assert r.permutation(n).tolist() == val
            elif kind == "int":
                assert r.integers(n) == val
            else:
                assert sha(r.permutation(n).astype("<i8")) == val


def test_rng_matches_numpy_directly():
    for seed in (3, 99, 2 ** 33 + 1):
        ref = np.random.Generator(np.random.Philox(seed))
        r = O.Rng(seed)
        for beta in (16, 23, 64, 300):
            assert r.integers(beta) == int(ref.integers(0, beta))
            assert r.integers(beta) == int(ref.integers(0, beta))
            np.testing.assert_array_equal(r.permutation(beta * 3), ref.permutation(beta * 3))


def test_weights_match_scipy():
    from scipy.ndimage import _filters
    for r in (1.0, 1.9, 2.5, 7.3, 15.5, 31.0, 511.0, 2047.0):
        h = int(np.ceil(r))
        want = _filters._gaussian_kernel1d(r / 2.0, 0, h)[::-1]
        got = O.gaussian_weights(r / 2.0, h)
        np.testing.assert_array_equal(got, want[h:])
        np.testing.assert_array_equal(want[:h + 1][::-1], want[h:])  # exactly symmetric


def test_blur_bit_exact():
    meta = golden_json("blur.json")
    z = golden_npz("blur.npz")
    for m in meta:
        i = m["i"]
        if m["dtype"] == "f32":
            out = O.blur_target(blur_input(m["seed"], m["side"], m["dim"]), m["radius"])
            assert out.dtype == np.float32
            assert sha(out) == m["sha"], m
            if f"out{i}" in z:
                np.testing.assert_array_equal(out, z[f"out{i}"])
        else:
            g = z[f"in{i}"]
            np.testing.assert_array_equal(O.renormalized_blur(g, m["sigma"], m["radius"]), z[f"out{i}"])
            np.testing.assert_array_equal(O.separable_blur(g, m["sigma"], m["radius"]), z[f"sep{i}"])
            np.testing.assert_array_equal(O.border_weight(g.shape, m["sigma"], m["radius"]), z[f"den{i}"])


def test_reassign_block_golden():
    z = golden_npz("assign.npz")
    for i in range(int(z["count"])):
        f = z[f"feat{i}"].copy()
        idx = np.arange(len(f), dtype=np.int64)
        O.reassign_block(f, idx, z[f"target{i}"], z[f"positions{i}"], z[f"grouping{i}"])
        np.testing.assert_array_equal(idx, z[f"idx_out{i}"])
        np.testing.assert_array_equal(f, z[f"feat_out{i}"])


def test_metrics_golden():
    z = golden_npz("metrics.npz")
    for i in range(5):
        assert O.vad(z[f"vad_in{i}"].astype(np.float32)) == pytest.approx(
            float(np.var(np.concatenate([np.abs(np.diff(z[f"vad_in{i}"].astype(np.float32).astype(np.float64).reshape(
                z[f"vad_in{i}"].shape[0], z[f"vad_in{i}"].shape[1], -1), axis=a)).ravel() for a in (0, 1)]))),
            rel=1e-12)


def _check_sort(features, case, perm_want):
    perm, rep = O.sort_grid_report(features, initial_radius_override=case.get("initial_radius"), **case["cfg"])
    np.testing.assert_array_equal(perm, perm_want)
    assert rep["reorders"] == case["reorders"]
    vals = [v for _, t in rep["radius_trace"] for v in t]
    assert [len(t) for _, t in rep["radius_trace"]] == case["counts"]
    # grid_distance in NumPy's pairwise order (plas_oracle.c np_pairwise): the
    # reference's floats
    np.testing.assert_array_equal(vals, case["values"])
    np.testing.assert_allclose([r for r, _ in rep["radius_trace"]], case["radii"], rtol=0, atol=0)
    assert rep["initial_vad"] == pytest.approx(case["initial_vad"], rel=1e-12)
    assert rep["final_vad"] == pytest.approx(case["final_vad"], rel=1e-12)


def test_sort_small_golden():
    z = golden_npz("sort_small.npz")
    for case in golden_json("sort_small.json"):
        _check_sort(z["features_" + case["name"]], case, z["perm_" + case["name"]])


def test_sort_c0_golden():
    z = golden_npz("c0.npz")
    feats = synthetic.c0(0)
    for case in golden_json("c0.json"):
        key = ("s%d" if case["initial_radius"] is None else "r32_s%d") % case["cfg"]["rng_seed"]
        _check_sort(feats, case, z[key].astype(np.int64))


def test_sort_c1_golden_seed0():
    z = golden_npz("c1.npz")
    case = golden_json("c1.json")[0]
    _check_sort(synthetic.c1(0), case, z["s0"].astype(np.int64))


def test_smoothness_golden():
    meta = golden_json("smooth.json")
    z = golden_npz("smooth.npz")
    defaults = {"opacity": 0.09, "rotation": 0.91}
    for m in meta:
        p = m["params"]
        weights = p.get("weights", defaults)
        total = 0.0
        for name in m["names"]:
            coeff = p.get("overall_multiplier", 1.0) * weights.get(name, 0.0)
            loss, grad = O.smoothness_plane(z[f"{m['i']}_in_{name}"], coeff, p.get("huber_delta", 1.0),
                                            p.get("detach_target", False), p.get("sigma", 3.0),
                                            p.get("kernel_size", 5))
            total += loss
            np.testing.assert_array_equal(grad, z[f"{m['i']}_grad_{name}"])
        assert total == m["loss"]  # the mean in NumPy's pairwise order: the reference's float
