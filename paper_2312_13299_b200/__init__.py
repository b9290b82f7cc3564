"""B200-native PLAS sort hot path (arXiv 2312.13299, "Self-Organizing Gaussian Grids").

Drop-in for the reference package's sort path (``sogs.plas``, ``sogs.blur``,
``sogs.smoothness``, ``sogs.metrics.vad/SortReport``); the compute runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/plas_b200.h.
Importing the package does not touch the GPU; the first GPU call loads
libplas_b200.so and fails loudly if it is missing.
"""

from .metrics import BENCH_CSV_FIELDS, SortReport, attribute_psnr, bench_rows_to_csv, bench_sort, vad
from .plas import (PERMUTATIONS, SortConfig, block_size, blur_target, grid_distance,
                   initial_radius, partition_blocks, reassign_block, sort_grid,
                   sort_grid_report, sort_on_device)
from .smoothness import (DEFAULT_SMOOTHNESS_WEIGHTS, SmoothnessParams, huber, huber_grad, smoothness_loss,
                         smoothness_loss_autograd)
from .splats import (DEFAULT_SORT_WEIGHTS, GridLayout, GridStack, NormalizationSpec, SplatCloud,
                     build_grid_layout, normalize_for_sorting, prune_to_grid)

__version__ = "0.1.0"

__all__ = [
    "PERMUTATIONS", "SortConfig", "SortReport", "SmoothnessParams", "GridLayout", "GridStack",
    "DEFAULT_SORT_WEIGHTS", "DEFAULT_SMOOTHNESS_WEIGHTS", "NormalizationSpec", "SplatCloud",
    "block_size", "blur_target", "build_grid_layout", "normalize_for_sorting", "prune_to_grid",
    "grid_distance", "huber", "huber_grad", "initial_radius", "partition_blocks", "reassign_block",
    "smoothness_loss", "smoothness_loss_autograd", "sort_grid", "sort_grid_report", "sort_on_device", "vad",
    "BENCH_CSV_FIELDS", "attribute_psnr", "bench_rows_to_csv", "bench_sort",
]
