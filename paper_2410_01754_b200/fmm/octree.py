"""Octree view exported from the device plan (reference fmm/octree.py:52-93).

The arrays here are the device's own: the canonical permutation and CSR
leaf offsets from the GPU sort, and the neighbour / M2L partner lists as the
kernels enumerate them (lfmm_export_lists).  They exist so the bit-exact
tree tests can compare them with the reference's ``build_octree``.
"""

from dataclasses import dataclass, field

import numpy as np

NEIGHBOR_OFFSETS = np.array([(x, y, z) for x in (-1, 0, 1) for y in (-1, 0, 1) for z in (-1, 0, 1)], np.int64)
_cube3 = np.array([(x, y, z) for x in range(-3, 4) for y in range(-3, 4) for z in range(-3, 4)], np.int64)
M2L_OFFSETS = _cube3[np.abs(_cube3).max(axis=1) >= 2]
OCTANTS = np.array([(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)], np.int64)


def box_grid(n):
    i = np.arange(n ** 3, dtype=np.int64)
    return np.stack([i // (n * n), (i // n) % n, i % n], axis=1)


def flat_index(grid, n):
    return (grid[..., 0] * n + grid[..., 1]) * n + grid[..., 2]


@dataclass
class LevelGrid:
    n: int
    size: float
    grid: np.ndarray
    m2l: list = field(default_factory=list)
    child_index: np.ndarray = None

    @property
    def num_boxes(self):
        return self.n ** 3

    def centers(self):
        return (self.grid + 0.5) * self.size


@dataclass
class Octree:
    box_length: float
    depth: int
    perm: np.ndarray
    inv_perm: np.ndarray
    positions: np.ndarray
    leaf_of_particle: np.ndarray
    leaf_start: np.ndarray
    nb_box: np.ndarray
    nb_shift: np.ndarray
    levels: list = field(default_factory=list)

    @property
    def num_particles(self):
        return self.positions.shape[0]

    @property
    def num_leaves(self):
        return self.levels[self.depth].num_boxes

    def leaf_centers(self):
        return self.levels[self.depth].centers()


def _group_m2l(src, row):
    """(row, targets, sources) triples in row order, like _build_m2l_lists."""
    nbox = src.shape[0]
    tgt = np.repeat(np.arange(nbox, dtype=np.int64), src.shape[1])
    r = row.reshape(-1)
    s = src.reshape(-1)
    order = np.lexsort((tgt, r))
    r, tgt, s = r[order], tgt[order], s[order]
    out = []
    bounds = np.flatnonzero(np.diff(r)) + 1
    for seg_t, seg_s, seg_r in zip(np.split(tgt, bounds), np.split(s, bounds), np.split(r, bounds)):
        if seg_t.size:
            out.append((int(seg_r[0]), seg_t, seg_s))
    return out


def octree_view(plan, box_length, depth):
    perm, inv, leaf, start, pos = plan.export_tree()
    nb, sh, _, _ = plan.export_lists(0)
    levels = []
    for l in range(depth + 1):
        n = 2 ** l
        lg = LevelGrid(n=n, size=box_length / n, grid=box_grid(n))
        if l >= 1:
            _, _, src, row = plan.export_lists(l)
            lg.m2l = _group_m2l(src, row)
        levels.append(lg)
    for l in range(depth):
        child = (2 * levels[l].grid)[:, None, :] + OCTANTS[None, :, :]
        levels[l].child_index = flat_index(child, levels[l + 1].n)
    return Octree(box_length=float(box_length), depth=depth, perm=perm, inv_perm=inv, positions=pos,
                  leaf_of_particle=leaf, leaf_start=start, nb_box=nb, nb_shift=sh, levels=levels)
