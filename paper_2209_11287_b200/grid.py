"""Epsilon-cell grid index built on the GPU (mirror of tilejoin.grid, grid.py:1-133).

`build_index` runs the device builder (tj_build_grid: cell keys, stable radix
sort, cell table, candidate runs) and exports it into the reference's host
shape: `cells` {cell coordinate tuple -> ascending int64 ids},
`ordered_cells` (lexicographic) and `point_order`.  `candidates_for_cell` and
`neighbor_cells` answer from the exported candidate runs, so they show exactly
what the refine kernels iterate over.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .datasets import as_dataset
from .errors import ValidationError
from .join import DEFAULT_K_IDX_CAP, JoinConfig, default_k_idx, DeviceJoin

CellCoord = tuple

__all__ = [
    "DEFAULT_K_IDX_CAP", "GridIndex", "build_index", "candidates_for_cell", "cell_of",
    "default_k_idx", "neighbor_cells",
]


@dataclass(frozen=True)
class GridIndex:
    """Sparse map from occupied cell coordinates to member ids (grid.py:31-50).

    Extra fields expose the device tables: cell_start (CSR of point_order per
    cell), cell_runs/runs (candidate position ranges per cell), cell_cands.
    """

    epsilon: float
    k_idx: int
    cells: dict
    ordered_cells: list
    point_order: np.ndarray
    cell_start: np.ndarray = field(repr=False, default=None)
    cell_runs: np.ndarray = field(repr=False, default=None)
    runs: np.ndarray = field(repr=False, default=None)
    cell_cands: np.ndarray = field(repr=False, default=None)
    cell_pos: dict = field(repr=False, default=None)

    @property
    def n_cells(self) -> int:
        return len(self.ordered_cells)

    def cell_costs(self) -> np.ndarray:
        """|cell| * |cand(cell)| in lexicographic cell order (join.py:170-173)."""
        return np.diff(self.cell_start) * self.cell_cands


def cell_of(point, epsilon: float, k_idx: int) -> CellCoord:
    """Cell coordinate of one point: floor(p_j / epsilon) over the first k_idx dims."""
    p = np.asarray(point, dtype=np.float64).reshape(-1)
    return tuple(int(v) for v in np.floor(p[:k_idx] / epsilon).astype(np.int64))


def build_index(dataset, epsilon: float, k_idx: int | None = None, device: int | None = None) -> GridIndex:
    """Build the grid on the GPU and export it in the reference's host form."""
    ds = as_dataset(dataset)
    if not np.isfinite(epsilon) or epsilon <= 0:
        raise ValidationError(f"epsilon must be positive and finite, got {epsilon}")
    if k_idx is None:
        k_idx = default_k_idx(ds.d)
    job = DeviceJoin(ds, JoinConfig(epsilon=float(epsilon), k_idx=k_idx), device=device)
    info = job.build()
    order, cstart, ccoords, cands, cruns, runs = job.ctx.export(info, k_idx)
    order = order.astype(np.int64)
    ordered = [tuple(int(v) for v in row) for row in ccoords]
    cells = {c: order[cstart[i]: cstart[i + 1]] for i, c in enumerate(ordered)}
    return GridIndex(
        epsilon=float(epsilon), k_idx=int(k_idx), cells=cells, ordered_cells=ordered,
        point_order=order, cell_start=cstart, cell_runs=cruns, runs=runs, cell_cands=cands,
        cell_pos={c: i for i, c in enumerate(ordered)},
    )


def _cell_index(index: GridIndex, cell) -> int:
    cell = tuple(cell)
    if len(cell) != index.k_idx:
        raise ValidationError(f"cell has {len(cell)} coordinates, index has k_idx={index.k_idx}")
    pos = index.cell_pos.get(cell)
    if pos is None:
        raise ValidationError(f"cell {cell} is empty")
    return pos


def candidates_for_cell(index: GridIndex, cell) -> np.ndarray:
    """Ids a query in `cell` is refined against: the device candidate runs, concatenated."""
    c = _cell_index(index, cell)
    runs = index.runs[index.cell_runs[c]: index.cell_runs[c + 1]]
    return np.concatenate([index.point_order[b:e] for b, e in runs])


def neighbor_cells(index: GridIndex, cell) -> list:
    """Occupied cells within Chebyshev distance 1 of `cell`, lexicographic (grid.py:104-118)."""
    cell = tuple(cell)
    if len(cell) != index.k_idx:
        raise ValidationError(f"cell has {len(cell)} coordinates, index has k_idx={index.k_idx}")
    if cell in index.cell_pos:  # answer from the device runs
        c = index.cell_pos[cell]
        out = []
        for b, e in index.runs[index.cell_runs[c]: index.cell_runs[c + 1]]:
            first = int(np.searchsorted(index.cell_start, b, side="right")) - 1
            last = int(np.searchsorted(index.cell_start, e, side="left"))
            out.extend(index.ordered_cells[first:last])
        return out
    # empty query cell: probe the 3^k neighbourhood of the host map
    import itertools

    out = []
    for off in itertools.product((-1, 0, 1), repeat=index.k_idx):
        nb = tuple(a + o for a, o in zip(cell, off))
        if nb in index.cell_pos:
            out.append(nb)
    return out
