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


@pytest.mark.gpu
def test_gpu_position_contraction_correctly_rounded():
    """contract(x) = sign(x) ln(1 + |x|) (quantization.py:8-11) with a correctly
    rounded logarithm (prep.cuh log1p_cr): every contracted value equals the
    60-digit decimal logarithm rounded to double, so the data-driven ranges
    match the reference's wherever its libm log1p rounds correctly (NumPy's did
    not for 52 of 50,000 random arguments)."""
    from decimal import Decimal, getcontext
    import torch
    from paper_2312_13299_b200 import quantization as q
    getcontext().prec = 60
    g = np.random.default_rng(17)
    vals = np.concatenate([g.normal(0, 1, 600), g.normal(0, 1, 300) * 1e10, g.uniform(0, 1e-8, 100),
                           g.uniform(0, 40, 600), [0.0, -0.0, 1e-300, 5e-324, 1.0, 1e300]])
    v = torch.from_numpy(np.repeat(vals[:, None], 3, axis=1)).cuda()
    spec = q.default_quant_spec()["position"]
    for i, x in enumerate(vals):
        _, lo, _ = q.quantize_planes("position", v[i:i + 1], spec)
        a = abs(float(x))
        # (below 1e-20, ln(1 + a) = a - a^2/2 + ... rounds to a)
        cr = (float((Decimal(a) + 1).ln()) if a >= 1e-20 else a) if a > 0 else 0.0
        want = (1.0 if x > 0 else -1.0) * cr if x != 0 else 0.0
        assert lo[0] == want, (x, lo[0], want)
