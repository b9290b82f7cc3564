"""CPU-only checks: the C-ABI library loads and exports include/plas_b200.h,
the host schedule matches the reference rules and SciPy, the host RNG is
NumPy-exact, and the Python boundary raises ValueError where the reference does."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import REPO
from oracle import oracle as O
from paper_2312_13299_b200 import _lib, schedule
import paper_2312_13299_b200 as plas

HEADER = os.path.join(REPO, "include", "plas_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(plas_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.load_library()  # no CUDA call
    names = header_functions()
    assert names, "no declarations parsed"
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"
    assert L.plas_abi_version() == 5
    assert L.plas_sizeof_sort_args() == ctypes.sizeof(_lib.SortArgs)
    assert L.plas_sizeof_sort_result() == ctypes.sizeof(_lib.SortResult)


def test_host_rng_is_numpy_exact():
    L = _lib.load_library()
    for seed in (0, 1, 7, 12345, 2 ** 40 + 7):
        key = np.zeros(2, dtype=np.uint64)
        L.plas_seed_key(seed, _lib.ptr(key))
        assert [int(k) for k in key] == [int(k) for k in np.random.SeedSequence(seed).generate_state(2, np.uint64)]
        for n in (1, 2, 37, 4096, 70001):
            out = np.empty(n, dtype=np.int64)
            assert L.plas_host_permutation(seed, n, _lib.ptr(out)) == 0
            np.testing.assert_array_equal(out, np.random.Generator(np.random.Philox(seed)).permutation(n))


def test_schedule_matches_reference_rules_and_scipy():
    from scipy.ndimage import _filters
    assert schedule.initial_radius(512) == 255.0 and schedule.initial_radius(4) == 2.0
    assert schedule.block_size(512, 40.7) == 41 and schedule.block_size(8, 100.0) == 8
    for side, decay in ((64, 0.5), (256, 0.95), (1024, 0.95), (4096, 0.95)):
        s = schedule.Schedule(side, decay)
        assert s.radii == O.radii(side, decay)
        r = schedule.initial_radius(side)
        for got in s.radii:  # repeated multiplication, not pow
            assert got == r
            r *= decay
        L = _lib.load_library()
        assert L.plas_num_levels(side * side, decay, float("nan")) == len(s.radii)
        for rr, h in list(zip(s.radii, s.half_widths))[:: max(1, len(s.radii) // 7)]:
            w = _filters._gaussian_kernel1d(rr / 2.0, 0, h)
            np.testing.assert_array_equal(schedule.gaussian_weights(rr / 2.0, h), w[h:])
    assert len(schedule.Schedule(1024, 0.95).radii) == 122
    assert len(schedule.Schedule(64, 0.5, start=32.0).radii) == 6


def test_partition_blocks_reference_examples():
    assert plas.partition_blocks(16, 10.0, 0, 0) == [(0, 16, 0, 16)]
    assert sorted(plas.partition_blocks(16, 10.0, 8, 8)) == [(0, 8, 0, 8), (0, 8, 8, 16), (8, 16, 0, 8), (8, 16, 8, 16)]
    rng = np.random.default_rng(1)
    for _ in range(25):
        side = int(rng.integers(2, 40))
        radius = float(rng.uniform(1, 30))
        beta = plas.block_size(side, radius)
        dy, dx = int(rng.integers(0, beta)), int(rng.integers(0, beta))
        cover = np.zeros((side, side), dtype=int)
        for y0, y1, x0, x1 in plas.partition_blocks(side, radius, dy, dx):
            cover[y0:y1, x0:x1] += 1
        assert np.all(cover == 1)
    with pytest.raises(ValueError):
        plas.partition_blocks(16, 10.0, 16, 0)


def test_validation_errors_without_gpu():
    with pytest.raises(ValueError):
        plas.SortConfig(radius_decay=1.0)
    with pytest.raises(ValueError):
        plas.SortConfig(improvement_threshold=0.0)
    with pytest.raises(ValueError):
        plas.SortConfig(min_block_size=1)
    with pytest.raises(ValueError):
        plas.SortConfig(rng_mode="cpu")
    with pytest.raises(ValueError):
        plas.sort_grid(np.zeros((10, 2)))
    with pytest.raises(ValueError):
        plas.sort_grid(np.zeros((1, 2)))
    with pytest.raises(ValueError):
        plas.blur_target(np.zeros((4, 4)), 0.0)
    with pytest.raises(ValueError):
        plas.SmoothnessParams(kernel_size=4)
    with pytest.raises(ValueError):
        plas.SmoothnessParams(weights={"opacity": -1.0})
    assert plas.huber(3.0, 1.0) == pytest.approx(2.5)
    assert plas.huber(0.5, 1.0) == pytest.approx(0.125)
    np.testing.assert_allclose(plas.huber_grad(np.linspace(-3, 3, 41), 1.0), np.clip(np.linspace(-3, 3, 41), -1, 1))
    assert tuple(plas.PERMUTATIONS[4][0]) == (0, 1, 2, 3) and plas.PERMUTATIONS[4].shape == (24, 4)


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        plas.sort_grid(np.random.default_rng(0).random((16, 3)))


def test_device_mode_feistel_is_a_bijection():
    # host restatement of common.cuh Feistel (DEVICE-mode grouping law)
    def mix32(x):
        x ^= x >> 16
        x = (x * 0x7feb352d) & 0xffffffff
        x ^= x >> 15
        x = (x * 0x846ca68b) & 0xffffffff
        x ^= x >> 16
        return x

    def feistel(key, m):
        bits = max(2, math.ceil(math.log2(m)) if m > 1 else 2)
        lb, rb = bits >> 1, bits - (bits >> 1)
        keys = []
        for _ in range(6):
            key = (key * 6364136223846793005 + 1442695040888963407) & (2 ** 64 - 1)
            keys.append(key >> 32)

        def once(x):
            a, b = lb, rb
            L, R = x >> b, x & ((1 << b) - 1)
            for r in range(6):
                f = mix32(R ^ keys[r]) & ((1 << a) - 1)
                L, R = R, L ^ f
                a, b = b, a
            return (L << b) | R

        def apply(i):
            x = once(i)
            while x >= m:
                x = once(x)
            return x
        return apply

    for m in (2, 3, 5, 16, 17, 255, 256, 1000, 4096):
        f = feistel(0x1234567 + m, m)
        assert sorted(f(i) for i in range(m)) == list(range(m))


def test_integration_ctypes_stub_matches_library():
    """The ctypes stub INTEGRATION.md shows a maintainer declares the same
    plas_sort_args / plas_sort_result layout as the library (sizeof checks; no
    CUDA call)."""
    import ctypes
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "INTEGRATION.md")).read()
    i = src.index("## 2. Binding the C ABI directly")
    j = src.index("```python", i) + len("```python")
    code = src[j: src.index("```", j)].split("def sort_grid")[0]
    code = code.replace('ctypes.CDLL("paper_2312_13299_b200/libplas_b200.so")',
                        f'ctypes.CDLL("{os.path.join(root, "paper_2312_13299_b200", "libplas_b200.so")}")')
    ns = {}
    exec(code, ns)
    L = ns["L"]
    L.plas_sizeof_sort_result.restype = ctypes.c_size_t
    assert ctypes.sizeof(ns["SortArgs"]) == L.plas_sizeof_sort_args()
    assert ctypes.sizeof(ns["SortResult"]) == L.plas_sizeof_sort_result()
