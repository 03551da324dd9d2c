"""Host-side logic: config validation, weight algebra, site tables, the
water-box generator, list regrouping and the bench's work accounting."""

import numpy as np
import pytest

from oracle import lfmm_oracle as orc
from paper_2410_01754_b200 import SolverConfig, expand_weights, weight_gradient_matrix
from paper_2410_01754_b200.fmm.octree import M2L_OFFSETS, NEIGHBOR_OFFSETS, _group_m2l
from paper_2410_01754_b200.system import lambda_table, site_tables
from paper_2410_01754_b200.waterbox import generate_water_box


def test_config_validation_messages():
    # solver.py:60-75 messages
    cases = [(dict(p=0), "expansion order p=0 outside"), (dict(depth=7), "tree depth 7 outside"),
             (dict(lattice_mode="weird"), "unknown lattice_mode"), (dict(lattice_mode="shells", shell_cap=1),
                                                                   "shells mode needs shell_cap >= 2"),
             (dict(periodic_near=False, depth=1), "periodic_near=False requires"),
             (dict(intra_site_images="none"), "unknown intra_site_images"), (dict(precision="half"),
                                                                             "unknown precision")]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=msg):
            SolverConfig(**kw).validated()
    SolverConfig().validated()


def test_weights_match_reference_values():
    assert np.allclose(expand_weights([0.345]).values, [0.655, 0.345], atol=1e-15)
    assert np.allclose(expand_weights([0.345, 0.721]).values, [0.182745, 0.096255, 0.472255, 0.248745],
                       atol=1e-15)
    g = weight_gradient_matrix([0.345, 0.721])
    assert np.allclose(g.sum(1), 0.0)
    assert np.allclose(g, orc.weight_grads([0.345, 0.721]))


def test_offset_tables():
    assert NEIGHBOR_OFFSETS.shape == (27, 3) and tuple(NEIGHBOR_OFFSETS[13]) == (0, 0, 0)
    assert M2L_OFFSETS.shape == (316, 3)
    assert np.array_equal(M2L_OFFSETS, orc.M2L_OFF)


@pytest.mark.parametrize("level", [1, 2, 3])
def test_group_m2l_reconstructs_reference_grouping(level):
    ref = orc.m2l_pairs(level)
    nbox = 8 ** level
    src = np.zeros((nbox, 189), np.int64)
    row = np.zeros((nbox, 189), np.int64)
    fill = np.zeros(nbox, int)
    for r, t, s in ref:
        for tt, ss in zip(t, s):
            src[tt, fill[tt]] = ss
            row[tt, fill[tt]] = r
            fill[tt] += 1
    assert np.all(fill == 189)
    got = _group_m2l(src, row)
    assert len(got) == len(ref)
    for (r1, t1, s1), (r2, t2, s2) in zip(got, ref):
        assert r1 == r2 and np.array_equal(t1, t2) and np.array_equal(s1, s2)


def test_water_box_invariants():
    system, lam, info = generate_water_box(3000, 4, forms_per_site=2, seed=0)
    n = system.num_particles
    assert abs(n - 3000) < 200
    assert np.all(system.positions >= 0) and np.all(system.positions < system.box_length)
    assert abs(system.charges.sum()) < 1e-9  # waters neutral, form 0 of every site neutral
    assert abs(info["box_length"] - (1000 / 33.43) ** (1 / 3)) < 1e-12
    for s, v in zip(system.sites, lam.values):
        assert s.num_particles == 10 and s.num_forms == 2
        assert abs(s.form_charges[1].sum() - s.form_charges[0].sum() - 1.0) < 1e-12
        assert 0.05 <= v[0] <= 0.95 and abs(v[0] - 0.5) >= 0.05
        d = np.linalg.norm(system.positions[s.particle_indices][:, None] - system.positions[s.particle_indices][None],
                           axis=-1)
        assert np.all(d[~np.eye(10, dtype=bool)] >= 0.1 - 1e-12)
    # deterministic in the seed
    s2, _, _ = generate_water_box(3000, 4, forms_per_site=2, seed=0)
    assert s2.positions.tobytes() == system.positions.tobytes()


def test_site_and_lambda_tables():
    system, lam, _ = generate_water_box(1500, 3, forms_per_site=4, seed=2)
    ao, ai, nf, fo, fq = site_tables(system)
    assert list(ao) == [0, 10, 20, 30] and list(nf) == [4, 4, 4] and fo[-1] == 120
    tab, nl = lambda_table(system, lam.values)
    assert tab.shape == (3, 4) and list(nl) == [2, 2, 2]
    with pytest.raises(ValueError, match="weights, site has 4 forms"):
        lambda_table(system, [[0.5]] * 3)


def test_bench_pair_count_and_work():
    import bench

    pos = np.random.default_rng(0).uniform(0, 2.0, (300, 3))
    t = orc.build_tree(pos, 2.0, 2)
    want = 0
    start = t["leaf_start"]
    for b in range(64):
        for k in range(27):
            nb = t["nb_box"][b, k]
            want += (start[b + 1] - start[b]) * (start[nb + 1] - start[nb])
    assert bench.pair_count(start, 2) == want - 300
    w = bench.algorithmic_work(10, 5, 1_000_000, 8.2e8, 512)
    assert w["t_m2l"] == 189 * sum(8 ** l for l in range(1, 6)) == 7077672
