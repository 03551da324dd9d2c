"""Particle / site / lambda data model (reference system.py:30-100).

Plain containers; the solver consumes them through the site tables it
uploads to the device (lfmm_sites_set).  ``scale_charges`` here is the host
convenience form of the device kernel used by the hot path.
"""

from dataclasses import dataclass, field

import numpy as np

from .weights import MAX_BRANCHES

MAX_FORMS = 2 ** MAX_BRANCHES


@dataclass
class TitratableSite:
    particle_indices: np.ndarray
    form_charges: np.ndarray

    def __post_init__(self):
        self.particle_indices = np.asarray(self.particle_indices, dtype=np.int64)
        self.form_charges = np.atleast_2d(np.asarray(self.form_charges, dtype=np.float64))

    @property
    def num_particles(self):
        return self.particle_indices.shape[0]

    @property
    def num_forms(self):
        return self.form_charges.shape[0]

    @property
    def num_lambda(self):
        return max(1, (self.num_forms - 1).bit_length())


@dataclass
class ParticleSystem:
    box_length: float
    positions: np.ndarray
    charges: np.ndarray
    sites: list = field(default_factory=list)

    def __post_init__(self):
        self.box_length = float(self.box_length)
        self.positions = np.atleast_2d(np.asarray(self.positions, dtype=np.float64))
        self.charges = np.asarray(self.charges, dtype=np.float64)

    @property
    def num_particles(self):
        return self.positions.shape[0]


@dataclass
class LambdaState:
    values: list
    velocities: list
    masses: list

    def __post_init__(self):
        self.values = [np.asarray(v, dtype=np.float64).copy() for v in self.values]
        self.velocities = [np.asarray(v, dtype=np.float64).copy() for v in self.velocities]
        self.masses = [float(m) for m in self.masses]

    def copy(self):
        return LambdaState(values=[v.copy() for v in self.values], velocities=[v.copy() for v in self.velocities],
                           masses=list(self.masses))

    def fingerprint(self):
        return tuple(tuple(float(x) for x in v) for v in self.values)


def scale_charges(system, tilde_weights):
    """q~: site entries replaced by the weight-blended form charges."""
    if len(tilde_weights) != len(system.sites):
        raise ValueError(f"{len(tilde_weights)} weight vectors for {len(system.sites)} sites")
    q = np.array(system.charges, dtype=np.float64, copy=True)
    for site, tw in zip(system.sites, tilde_weights):
        w = np.asarray(getattr(tw, "values", tw), dtype=np.float64)
        if w.shape != (site.num_forms,):
            raise ValueError(f"weight vector length {w.shape} != form count {site.num_forms}")
        q[site.particle_indices] = w @ site.form_charges
    return q


def site_tables(system):
    """CSR site tables for lfmm_sites_set / lfmm_assemble."""
    sites = system.sites
    ns = [s.num_particles for s in sites]
    nf = [s.num_forms for s in sites]
    atom_off = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    form_off = np.concatenate([[0], np.cumsum([a * b for a, b in zip(ns, nf)])]).astype(np.int64)
    atom_idx = (np.concatenate([s.particle_indices for s in sites]).astype(np.int64)
                if sites else np.zeros(0, np.int64))
    form_q = (np.concatenate([s.form_charges.reshape(-1) for s in sites])
              if sites else np.zeros(0))
    return atom_off, atom_idx, np.asarray(nf, np.int32), form_off, form_q


def lambda_table(system, lam_values):
    """(S,4) padded lambdas and (S,) counts; validates against the forms."""
    s = len(system.sites)
    if len(lam_values) != s:
        raise ValueError(f"{len(lam_values)} lambda vectors for {s} sites")
    lam = np.zeros((s, 4))
    nl = np.zeros(s, np.int32)
    for i, (site, v) in enumerate(zip(system.sites, lam_values)):
        arr = np.asarray(getattr(v, "values", v), dtype=np.float64).reshape(-1)
        if not 1 <= arr.shape[0] <= MAX_BRANCHES:
            raise ValueError(f"need between 1 and {MAX_BRANCHES} lambda values, got shape {arr.shape}")
        if (1 << arr.shape[0]) != site.num_forms:
            raise ValueError(
                f"{arr.shape[0]} lambdas give {1 << arr.shape[0]} weights, site has {site.num_forms} forms"
            )
        lam[i, : arr.shape[0]] = arr
        nl[i] = arr.shape[0]
    return lam, nl
