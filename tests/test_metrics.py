"""metrics.py drop-in: bench_sort / bench_rows_to_csv / attribute_psnr.

Fixtures: tests/golden/bench.json, made by running the reference's
metrics.bench_sort / bench_rows_to_csv / attribute_psnr
(tests/golden/make_golden.py bench).  CPU tests pin the oracle (a sort of
each bench grid by the C restatement, VAD by the reference's NumPy formula)
and the host-side CSV / argument checks; GPU tests run bench_sort through the
CUDA path.
"""

import math

import numpy as np
import pytest

from conftest import golden_json
from oracle import oracle as O
from paper_2312_13299_b200 import metrics


def _vad64(grid):
    """metrics.py:25-40, restated for the oracle check."""
    g = np.asarray(grid, dtype=np.float64)
    d = np.concatenate([np.abs(np.diff(g, axis=0)).reshape(-1), np.abs(np.diff(g, axis=1)).reshape(-1)])
    return float(d.var())


def _bench_data(side, channels, seed):
    return np.random.default_rng(seed).uniform(0.0, 255.0, (side * side, channels))


def test_bench_csv_matches_reference():
    g = golden_json("bench.json")
    assert list(metrics.BENCH_CSV_FIELDS) == g["fields"]
    assert metrics.bench_rows_to_csv(g["csv_rows"]) == g["csv"]
    assert metrics.bench_rows_to_csv([]) == ",".join(g["fields"]) + "\n"


def test_bench_and_psnr_argument_errors():
    with pytest.raises(ValueError, match="bench sides must be >= 2"):
        metrics.bench_sort([1])
    with pytest.raises(ValueError, match="peak must be positive"):
        metrics.attribute_psnr(np.zeros(3), np.zeros(3), 0.0)
    with pytest.raises(ValueError, match="plane shapes must match"):
        metrics.attribute_psnr(np.zeros(3), np.zeros(4), 1.0)


def test_oracle_reproduces_bench_rows():
    """The oracle sort + the reference's VAD formula give the reference's rows."""
    for row in golden_json("bench.json")["rows"]:
        side, ch, seed = row["side"], row["channels"], row["seed"]
        data = _bench_data(side, ch, seed)
        perm, rep = O.sort_grid_report(data / 255.0, rng_seed=seed)
        assert rep["reorders"] == row["reorders"]
        assert round(_vad64(data.reshape(side, side, ch)), 4) == row["vad_initial"]
        assert round(_vad64(data[np.asarray(perm)].reshape(side, side, ch)), 4) == row["vad_final"]


@pytest.mark.gpu
def test_bench_sort_matches_reference_rows():
    g = golden_json("bench.json")
    rows = metrics.bench_sort([2, 8, 16], channels=3, seeds=(0, 1))
    rows += metrics.bench_sort([12], channels=5, seeds=(7,))
    assert len(rows) == len(g["rows"])
    for got, want in zip(rows, g["rows"]):
        assert got["time_s"] >= 0.0
        assert {k: v for k, v in got.items() if k != "time_s"} == want
    assert metrics.bench_rows_to_csv(rows).splitlines()[0] == ",".join(g["fields"])


@pytest.mark.gpu
def test_attribute_psnr_matches_reference():
    for case in golden_json("bench.json")["psnr"]:
        a = np.array(case["a"]).reshape(case["shape"])
        b = np.array(case["b"]).reshape(case["shape"])
        assert metrics.attribute_psnr(a, b, case["peak"]) == pytest.approx(case["psnr"], rel=1e-12)
    a = np.random.default_rng(0).uniform(0, 1, (5, 5))
    assert metrics.attribute_psnr(a, a.copy(), 1.0) == math.inf
