"""Bit-exact octree parity: the device sort and the kernels' own list
enumeration against the reference (golden) and the oracle
(pkg/tests/test_octree.py restated)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2410_01754_b200 import PeriodicSolver, SolverConfig  # noqa: E402
from oracle import lfmm_oracle as orc  # noqa: E402


def tree_of(pos, box, depth):
    return PeriodicSolver(pos, box, SolverConfig(p=4, depth=depth, lattice_mode="off")).tree


@pytest.mark.parametrize("name", ["tree_d1.npz", "tree_d3.npz"])
def test_tree_bit_exact_vs_reference(golden, name):
    g = golden(name)
    t = tree_of(g["positions"], float(g["box"]), int(g["depth"]))
    for key in ("perm", "inv_perm", "leaf_start", "leaf_of_particle", "nb_box", "nb_shift"):
        assert np.array_equal(getattr(t, key), g[key]), key
    assert t.positions.tobytes() == g["positions_sorted"].tobytes()
    for l in range(1, int(g["depth"]) + 1):
        rows = [r for r, _, _ in t.levels[l].m2l]
        assert np.array_equal(rows, g[f"m2l{l}_rows"])
        assert np.array_equal([tg.size for _, tg, _ in t.levels[l].m2l], g[f"m2l{l}_counts"])
        assert np.array_equal(np.concatenate([tg for _, tg, _ in t.levels[l].m2l]), g[f"m2l{l}_targets"])
        assert np.array_equal(np.concatenate([s for _, _, s in t.levels[l].m2l]), g[f"m2l{l}_sources"])
    for l in range(int(g["depth"])):
        assert np.array_equal(t.levels[l].child_index, g[f"child{l}"])


@pytest.mark.parametrize("depth", [0, 2, 4, 5])
def test_tree_bit_exact_vs_oracle(depth):
    rng = np.random.default_rng(depth)
    box = 5.0
    pos = rng.uniform(-box, 2 * box, size=(20000, 3))  # unwrapped: exercises the np.mod wrap
    pos[10] = pos[11]  # exact duplicate
    pos[20, 0] = pos[21, 0]  # tie in x
    pos[30] = [box, 0.0, -0.0]  # exact multiples
    t = tree_of(pos, box, depth)
    o = orc.build_tree(orc.wrap(pos, box), box, depth)
    for key in ("perm", "inv_perm", "leaf_start", "leaf_of_particle", "nb_box", "nb_shift"):
        assert np.array_equal(getattr(t, key), o[key]), key
    assert t.positions.tobytes() == o["positions"].tobytes()
    for l in range(1, depth + 1):
        ref = orc.m2l_pairs(l)
        got = t.levels[l].m2l
        assert len(got) == len(ref)
        for (r1, t1, s1), (r2, t2, s2) in zip(got, ref):
            assert r1 == r2 and np.array_equal(t1, t2) and np.array_equal(s1, s2)


def test_every_box_has_189_partners():
    t = tree_of(np.random.default_rng(0).uniform(0, 1, (100, 3)), 1.0, 3)
    for l in range(1, 4):
        counts = np.zeros(8 ** l, int)
        for _, tg, _ in t.levels[l].m2l:
            np.add.at(counts, tg, 1)
        assert np.all(counts == 189)


def test_positions_round_trip():
    pos = np.random.default_rng(2).uniform(0, 1.0, (50, 3))
    t = tree_of(pos, 1.0, 1)
    assert np.array_equal(t.positions, pos[t.perm])
    assert np.array_equal(t.positions[t.inv_perm], pos)
