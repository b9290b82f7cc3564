"""The two data-model types the sort/smoothness boundary accepts (splats.py:17-24, 119-130, 219-232).

The rest of the reference's data model (SplatCloud, pruning, normalisation)
is caller-side preparation outside the hot path.
"""

from dataclasses import dataclass, field

ATTRIBUTES = ("position", "sh_dc", "sh_rest", "opacity", "scale", "rotation")

# Default per-attribute sorting weights (splats.py:17-24); SortConfig default.
DEFAULT_SORT_WEIGHTS = {
    "position": 1.0,
    "sh_dc": 1.0,
    "sh_rest": 0.0,
    "opacity": 0.0,
    "scale": 1.0,
    "rotation": 0.0,
}


@dataclass(frozen=True)
class GridLayout:
    side: int

    def __post_init__(self):
        if self.side < 1:
            raise ValueError("grid side must be positive")

    @property
    def cells(self):
        return self.side * self.side


@dataclass(frozen=True)
class GridStack:
    """Per-attribute 2D planes sharing one permutation; one cell per Gaussian."""

    layout: GridLayout
    planes: dict = field(default_factory=dict)

    def __post_init__(self):
        side = self.layout.side
        for name, plane in self.planes.items():
            if name not in ATTRIBUTES:
                raise ValueError(f"unknown attribute {name!r}")
            if tuple(plane.shape[:2]) != (side, side):
                raise ValueError(f"plane {name!r} is {tuple(plane.shape[:2])}, expected {(side, side)}")
