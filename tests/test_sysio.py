"""System files (paper_2410_01754_b200/sysio.py) against the reference's own
save_system/load_system output (tests/golden/make_golden_sysio.py): same
arrays on load, byte-identical JSON on save, bit-exact round trips (JSON and
npz), the reference's validation messages."""

import os

import numpy as np
import pytest

from paper_2410_01754_b200 import sysio
from paper_2410_01754_b200.system import LambdaState, ParticleSystem, TitratableSite
from paper_2410_01754_b200.waterbox import generate_water_box

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def test_load_matches_reference_load():
    system, lam = sysio.load_system(os.path.join(GOLDEN, "system_small.json"))
    g = np.load(os.path.join(GOLDEN, "system_small_loaded.npz"))
    assert system.box_length == float(g["box"])
    assert _same(system.positions, g["positions"]) and _same(system.charges, g["charges"])
    for s in range(2):
        assert _same(system.sites[s].particle_indices, g[f"site{s}_idx"])
        assert _same(system.sites[s].form_charges, g[f"site{s}_forms"])
    assert _same(np.concatenate(lam.values), g["lambdas"])
    assert _same(np.concatenate(lam.velocities), g["velocities"])
    assert _same(np.asarray(lam.masses), g["masses"])


def test_save_is_byte_identical_to_reference(tmp_path):
    src = os.path.join(GOLDEN, "system_small.json")
    system, lam = sysio.load_system(src)
    out = tmp_path / "s.json"
    sysio.save_system(system, lam, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_npz_round_trip_is_bit_exact(tmp_path):
    system, lam, _ = generate_water_box(3000, 4, seed=2)
    lam = LambdaState(values=[np.asarray(v, float) for v in lam.values],
                      velocities=[np.zeros(len(v)) for v in lam.values], masses=[5.0] * 4)
    p = tmp_path / "s.npz"
    sysio.save_npz(system, lam, p)
    s2, l2 = sysio.load_npz(p)
    assert _same(s2.positions, system.positions) and _same(s2.charges, system.charges)
    for a, b in zip(s2.sites, system.sites):
        assert _same(a.particle_indices, b.particle_indices) and _same(a.form_charges, b.form_charges)
    assert all(_same(a, b) for a, b in zip(l2.values, lam.values))
    # and JSON
    pj = tmp_path / "s.json"
    sysio.save_system(system, lam, pj)
    s3, l3 = sysio.load_system(pj)
    assert _same(s3.positions, system.positions) and _same(s3.charges, system.charges)


def test_validation_messages():
    site = TitratableSite(np.array([0, 1]), np.zeros((3, 2)))
    sysm = ParticleSystem(1.0, np.array([[0.1, 0.2, 0.3], [0.5, 0.5, 1.0]]), np.zeros(2), [site])
    v = sysio.validate_system(sysm)
    assert "positions not wrapped into [0, box_length)" in v
    assert "site 0: form count 3 not a power of two >= 2" in v
    assert sysio.validate_system(ParticleSystem(-1.0, np.zeros((1, 3)), np.zeros(1))) == \
        ["box_length must be positive, got -1.0"]
    assert np.array_equal(sysio.wrap_positions(np.array([[-1e-17, 1.0, 2.5]]), 1.0), [[0.0, 0.0, 0.5]])


def test_load_errors(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text('{"box_length_nm": 2.0, "particles": [{"pos": [0.1, 0.2, 0.3]}]}')
    with pytest.raises(ValueError, match=r"missing field 'q' in particles\[0\]"):
        sysio.load_system(p)
    p.write_text("{")
    with pytest.raises(ValueError, match="parse error"):
        sysio.load_system(p)
