"""Seeded synthetic water boxes with titratable sites.

The reference ships no water-box generator (its generate_random_system is
a jittered grid of random charges and is O(N) per site atom,
generators.py:26-62).  This one is vectorised and feeds the *same* arrays
to the oracle and to the GPU path:

* TIP3P-like rigid waters: O -0.834 e, H +0.417 e, r(OH) 0.09572 nm,
  HOH 104.52 deg, density 33.43 molecules/nm^3 (~100.3 atoms/nm^3);
  molecule centres on a jittered cubic lattice (+-0.1 pitch), uniform random
  orientations.
* Sites: centres with pairwise minimum-image distance >= 1.0 nm; waters
  with an atom within 0.35 nm of a centre are removed; 10 site atoms in a
  0.5 nm-diameter ball with >= 0.1 nm separation (generators.py:44-62 rule).
* Forms follow generators._site_form_charges (generators.py:65-83): base
  U(-0.3, 0.3), each lambda bit adds a net +1 e over <= 4 carriers; the
  base is shifted so form 0 of every site is neutral.
* lambda ~ U(0.05, 0.95) avoiding |lambda - 0.5| < 0.05.
"""

import numpy as np

from .system import LambdaState, ParticleSystem, TitratableSite

WATER_DENSITY = 33.43  # molecules / nm^3
Q_O, Q_H = -0.834, 0.417
R_OH = 0.09572
ANGLE_HOH = np.deg2rad(104.52)
SITE_BALL_RADIUS = 0.25
SITE_MIN_SEP = 0.1
SITE_CLEAR = 0.35
SITE_CENTER_SEP = 1.0


def _random_rotations(rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1),
    ], axis=1)


def _min_image(d, box):
    return d - box * np.round(d / box)


def _site_forms(rng, ns, nf):
    base = rng.uniform(-0.3, 0.3, ns)
    base -= base.mean()  # form 0 neutral
    nl = max(1, (nf - 1).bit_length())
    deltas = []
    for _ in range(nl):
        carriers = rng.choice(ns, size=min(4, ns), replace=False)
        d = np.zeros(ns)
        w = rng.uniform(0.5, 1.0, carriers.size)
        d[carriers] = w / w.sum()
        deltas.append(d)
    forms = np.empty((nf, ns))
    for rho in range(nf):
        q = base.copy()
        for i in range(nl):
            if (rho >> i) & 1:
                q = q + deltas[i]
        forms[rho] = q
    return forms


def generate_water_box(num_atoms, num_sites=0, forms_per_site=2, site_atoms=10, seed=0):
    """Return (ParticleSystem, LambdaState, info) for a ~num_atoms water box."""
    rng = np.random.default_rng(seed)
    n_mol = max(1, int(round(num_atoms / 3.0)))
    box = (n_mol / WATER_DENSITY) ** (1.0 / 3.0)
    # molecule centres on a jittered lattice
    nside = int(np.ceil(n_mol ** (1.0 / 3.0)))
    pitch = box / nside
    g = (np.arange(nside) + 0.5) * pitch
    grid = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    keep = rng.permutation(grid.shape[0])[:n_mol]
    centers = grid[keep] + rng.uniform(-0.1 * pitch, 0.1 * pitch, (n_mol, 3))
    # rigid water geometry in the molecular frame, O at the origin
    half = 0.5 * ANGLE_HOH
    h1 = R_OH * np.array([np.sin(half), 0.0, np.cos(half)])
    h2 = R_OH * np.array([-np.sin(half), 0.0, np.cos(half)])
    com_shift = (h1 + h2) * (1.008 / 18.015)
    local = np.stack([-com_shift, h1 - com_shift, h2 - com_shift])  # (3,3)
    rot = _random_rotations(rng, n_mol)
    atoms = centers[:, None, :] + np.einsum("nij,aj->nai", rot, local)  # (n_mol, 3, 3)

    # titratable sites
    site_centers = []
    tries = 0
    while len(site_centers) < num_sites:
        tries += 1
        if tries > 100000:
            raise RuntimeError("could not place site centres; box too small for the site count")
        c = rng.uniform(0.0, box, 3)
        if site_centers:
            d = _min_image(np.asarray(site_centers) - c, box)
            if np.min((d * d).sum(1)) < SITE_CENTER_SEP ** 2:
                continue
        site_centers.append(c)
    site_centers = np.asarray(site_centers).reshape(-1, 3)
    alive = np.ones(n_mol, bool)
    if num_sites:
        ox = atoms[:, 0, :]
        for c in site_centers:
            d = _min_image(ox - c, box)
            near = np.flatnonzero((d * d).sum(1) < (SITE_CLEAR + 0.2) ** 2)
            if near.size == 0:
                continue
            da = _min_image(atoms[near] - c, box)
            hit = ((da * da).sum(-1) < SITE_CLEAR ** 2).any(1)
            alive[near[hit]] = False
    water = atoms[alive].reshape(-1, 3)
    qw = np.tile([Q_O, Q_H, Q_H], int(alive.sum()))

    site_pos, sites, site_q = [], [], []
    ptr = water.shape[0]
    for c in site_centers:
        pts = []
        while len(pts) < site_atoms:
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            cand = c + u * SITE_BALL_RADIUS * rng.uniform() ** (1.0 / 3.0)
            if pts and np.min(np.linalg.norm(np.asarray(pts) - cand, axis=1)) < SITE_MIN_SEP:
                continue
            pts.append(cand)
        pts = np.asarray(pts)
        forms = _site_forms(rng, site_atoms, forms_per_site)
        sites.append(TitratableSite(np.arange(ptr, ptr + site_atoms), forms))
        site_pos.append(pts)
        site_q.append(forms[0])
        ptr += site_atoms
    pos = np.vstack([water] + site_pos) if site_pos else water
    pos = np.mod(pos, box)
    pos[pos >= box] = 0.0
    q = np.concatenate([qw] + site_q) if site_q else qw
    system = ParticleSystem(box, pos, q, sites)
    lams = []
    for s in sites:
        v = rng.uniform(0.05, 0.95, s.num_lambda)
        bad = np.abs(v - 0.5) < 0.05
        while bad.any():
            v[bad] = rng.uniform(0.05, 0.95, int(bad.sum()))
            bad = np.abs(v - 0.5) < 0.05
        lams.append(v)
    lam = LambdaState(values=lams, velocities=[np.zeros_like(v) for v in lams], masses=[5.0] * len(sites))
    info = dict(n_mol=n_mol, n_water=int(alive.sum()), box_length=box, n_atoms=pos.shape[0])
    return system, lam, info
