"""Quantization after the sort: contract + range + quantize +
plane packing (bundle.py:102-115, 158-176; quantization.py:8-41).

CPU: the oracle restatement against reference-generated fixtures
(tests/golden/quant.npz, make_golden.py part_quant).  GPU: quantize_planes
against the same fixtures, bit-exact (pixel values and manifest ranges).
"""
import os

import numpy as np
import pytest

from oracle import prep as oprep

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "quant.npz"))
NAMES = sorted({k.rsplit("_", 1)[0] for k in G.files if k.endswith("_planes")})
SPEC = {"position": (2 ** 14, None), "sh_dc": (2 ** 8, (-2.0, 4.0)), "sh_rest": (2 ** 5, (-1.0, 1.0)),
        "opacity": (2 ** 6, (-6.0, 12.0)), "scale": (2 ** 6, None), "rotation": (2 ** 6, (-1.0, 2.0))}


@pytest.mark.parametrize("name", NAMES)
def test_oracle_quantize_matches_reference(name):
    levels, clip = SPEC[name]
    planes, lo, hi = oprep.quantize_attribute_planes(name, G[f"{name}_in"], levels, clip)
    assert np.array_equal(planes, G[f"{name}_planes"].astype(np.int64))
    assert np.array_equal(lo, G[f"{name}_lo"]) and np.array_equal(hi, G[f"{name}_hi"])


def test_host_mirror_functions():
    from paper_2312_13299_b200 import quantization as q
    x = np.array([-3.0, -0.0, 0.0, 2.5, 1e6])
    assert np.array_equal(q.expand(q.contract(x)), np.sign(x) * np.expm1(np.log1p(np.abs(x))))
    assert q.quantize([-1.0, 0.5, 2.0], 0.0, 1.0, 3).tolist() == [0, 1, 2]
    assert np.allclose(q.dequantize([0, 1, 2], 0.0, 1.0, 3), [0.0, 0.5, 1.0])
    with pytest.raises(ValueError):
        q.quantize([0.0], 1.0, 1.0, 4)
    with pytest.raises(ValueError):
        q.AttributeQuant(1)
    assert q.default_quant_spec()["position"].bit_depth == 16


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_quantize_planes_bit_exact(name):
    from paper_2312_13299_b200 import quantization as q
    spec = q.default_quant_spec()[name]
    images, lo, hi = q.quantize_planes(name, G[f"{name}_in"], spec)
    assert np.array_equal(images.cpu().numpy().astype(np.int64), G[f"{name}_planes"].astype(np.int64))
    assert np.array_equal(np.array(lo), G[f"{name}_lo"]) and np.array_equal(np.array(hi), G[f"{name}_hi"])


@pytest.mark.gpu
def test_gpu_quantize_random_against_oracle():
    import torch
    from paper_2312_13299_b200 import quantization as q
    g = np.random.default_rng(11)
    for name, C in (("position", 3), ("sh_rest", 45), ("rotation", 4), ("scale", 3), ("opacity", 1)):
        v = g.normal(0, 4, (5000, C))
        v[g.integers(0, 5000, 50)] = 0.0
        levels, clip = SPEC[name]
        planes, lo, hi = oprep.quantize_attribute_planes(name, v, levels, clip)
        images, glo, ghi = q.quantize_planes(name, torch.from_numpy(v).cuda(), q.default_quant_spec()[name])
        assert np.array_equal(images.cpu().numpy().astype(np.int64), planes), name
        assert np.array_equal(np.array(glo), lo) and np.array_equal(np.array(ghi), hi), name
