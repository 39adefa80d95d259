"""Column stencil and candidate layout, evaluated on the host in float64.

The GPU connectivity generator consumes the per-source candidate layout as a
short table of (target column, probability) blocks; this module produces that
table with the same float64 expressions as the reference so that the
Bernoulli thresholds are bit-identical:

    kernel_probability   corticarc/connectivity.py:159-171
    compute_stencil      corticarc/connectivity.py:201-228
    _candidate_layout    corticarc/connectivity.py:357-380  (block form here)
    grid_totals          corticarc/connectivity.py:293-309
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["Stencil", "kernel_probability", "compute_stencil",
           "layout_blocks", "grid_totals", "expected_fanout"]


def kernel_probability(kernel, r) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    if np.any(r <= 0):
        raise ValueError("kernel_probability requires r > 0")
    if kernel.kind == "gaussian":
        return kernel.amplitude_A * np.exp(-(r * r) / (2.0 * kernel.scale ** 2))
    return kernel.amplitude_A * np.exp(-r / kernel.scale)


@dataclass(frozen=True)
class Stencil:
    radius: int
    offsets: np.ndarray        # (k, 2) (di, dj), centre excluded, (dj, di) row-major
    probabilities: np.ndarray  # (k,), 0 where below cutoff

    def active(self):
        keep = self.probabilities > 0
        return self.offsets[keep], self.probabilities[keep]


def compute_stencil(kernel, grid) -> Stencil:
    r_cut = kernel.cutoff_distance()
    radius = int(math.ceil(r_cut / grid.spacing_alpha)) if r_cut > 0 else 0
    if radius == 0:
        return Stencil(0, np.empty((0, 2), dtype=np.int64), np.empty(0))
    side = np.arange(-radius, radius + 1)
    dj, di = np.meshgrid(side, side, indexing="ij")     # dj outer, di inner
    di, dj = di.ravel(), dj.ravel()
    keep = ~((di == 0) & (dj == 0))
    di, dj = di[keep], dj[keep]
    # one vectorised np.exp call over the whole box, as the reference does,
    # so the SIMD code path (and its ulps) are the same
    p = kernel_probability(kernel, grid.spacing_alpha * np.hypot(di, dj))
    p = np.where(p > kernel.cutoff_p, p, 0.0)
    return Stencil(radius, np.column_stack([di, dj]), p)


def layout_blocks(grid, kernel, stencil: Stencil | None = None):
    """Candidate blocks of an excitatory source, per source column.

    Returns (blk_col, blk_p, blk_count): for source column c the excitatory
    layout is blk_col[c, :blk_count[c]] with probabilities blk_p[c, ...];
    block 0 is always the source's own column with local_p (the autapse slot
    is zeroed per source by the generator).  Inhibitory sources use block 0
    only (connectivity.py:370-379).
    """
    st = stencil if stencil is not None else compute_stencil(kernel, grid)
    offs, probs = st.active()
    ncol = grid.n_columns
    kmax = 1 + len(offs)
    blk_col = np.full((ncol, kmax), -1, dtype=np.int32)
    blk_p = np.zeros((ncol, kmax), dtype=np.float64)
    blk_count = np.zeros(ncol, dtype=np.int32)
    for col in range(ncol):
        ix, iy = grid.column_coords(col)
        blk_col[col, 0] = col
        blk_p[col, 0] = kernel.local_p
        k = 1
        for (di, dj), p in zip(offs, probs):
            tx, ty = ix + int(di), iy + int(dj)
            if 0 <= tx < grid.nx and 0 <= ty < grid.ny:
                blk_col[col, k] = grid.column_index(tx, ty)
                blk_p[col, k] = p
                k += 1
        blk_count[col] = k
    return blk_col, blk_p, blk_count


def grid_totals(kernel, grid):
    """(local, remote) expected synapse totals with border clipping."""
    n = grid.neurons_per_column
    offs, probs = compute_stencil(kernel, grid).active()
    pairs = (np.maximum(grid.nx - np.abs(offs[:, 0]), 0)
             * np.maximum(grid.ny - np.abs(offs[:, 1]), 0))
    remote = float(np.sum(pairs * probs)) * grid.n_excitatory_per_column * n
    local = grid.n_columns * n * kernel.local_p * (n - 1)
    return local, remote


def expected_fanout(kernel, grid) -> float:
    """Population-averaged synapses per neuron of an interior column."""
    n = grid.neurons_per_column
    _, probs = compute_stencil(kernel, grid).active()
    frac = grid.n_excitatory_per_column / n
    return kernel.local_p * (n - 1) + frac * n * float(probs.sum())
