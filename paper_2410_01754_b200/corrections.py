"""Hamiltonian-interpolation corrections and lambda forces (reference corrections.py).

Drop-in for ``hi_energy_and_forces`` / ``build_corrections`` /
``assemble_lambda_forces`` (corrections.py:157-274).  The per-site Gram
kernels, correction scalars, S_rho pairings and lambda forces are computed
by the fused device kernel ``k_hi_site`` (csrc/lfmm_hi.cuh) from the
potentials the solve left in device memory; this module validates
arguments, uploads the site tables once per (system, solver) pair and wraps
the results in the reference's dataclasses.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .fmm.solver import PeriodicSolver
from .system import lambda_table, site_tables
from .weights import expand_weights


@dataclass(frozen=True)
class CorrectionCharges:
    blend: np.ndarray
    half_offset: np.ndarray
    deviation: np.ndarray


def correction_charges(form_charges, weights):
    qf = np.atleast_2d(np.asarray(form_charges, dtype=np.float64))
    w = np.asarray(getattr(weights, "values", weights), dtype=np.float64)
    qt = w @ qf
    return CorrectionCharges(blend=qt, half_offset=qt[None, :] - 0.5 * qf, deviation=qt[None, :] - qf)


def minimum_image(disp, box_length):
    return disp - box_length * np.round(disp / box_length)


@dataclass
class SiteCorrections:
    weights: object
    charges: CorrectionCharges
    c_p2p: np.ndarray
    c_lattice: np.ndarray
    c_dipole: np.ndarray
    blend_energy: float

    def c_total(self):
        return self.c_p2p + self.c_lattice + self.c_dipole

    def energy_offset(self):
        return self.blend_energy - float(self.weights.values @ self.c_total())


@dataclass
class CorrectionSet:
    sites: list
    fingerprint: tuple
    device_offset: float = None  # fixed-order device sum of the site offsets

    def energy_offset(self):
        if self.device_offset is not None:
            return self.device_offset
        return math.fsum(s.energy_offset() for s in self.sites)


@dataclass
class InterpolationResult:
    energy: float
    forces: list
    mode: str
    solve: object
    corrections: object
    # (N, 3) -grad_r of `energy` when requested (not in the reference, whose
    # only spatial forces are spatial_forces(q~), solver.py:407-427): in HI
    # mode spatial_forces(q~) plus -grad Delta E_site on the site atoms
    spatial_forces: np.ndarray = None


def _fingerprint(lam_values):
    return tuple(tuple(float(x) for x in np.asarray(getattr(v, "values", v)).reshape(-1)) for v in lam_values)


def _bind_sites(solver, system):
    """Upload the site tables once per (system layout) to the solver's plan."""
    plan = solver.plan
    key = (id(system), len(system.sites),
           tuple(int(s.particle_indices.ctypes.data) for s in system.sites[:4]))
    tables = site_tables(system)
    sig = (key, tuple(hash(t.tobytes()) for t in tables))
    if plan.sites_key != sig:
        plan.set_sites(*tables, key=sig)
    return tables


def _site_positions(system):
    if not system.sites:
        return np.zeros((0, 3))
    idx = np.concatenate([s.particle_indices for s in system.sites])
    return np.ascontiguousarray(np.asarray(system.positions, dtype=np.float64)[idx])


def _split_forces(system, lam, nl, forces):
    return [np.array(forces[i, : nl[i]]) for i in range(len(system.sites))]


def _correction_set(system, lam_values, out, plan):
    sites = []
    fo = plan.form_slot_offsets
    for i, (site, v) in enumerate(zip(system.sites, lam_values)):
        w = expand_weights(np.asarray(getattr(v, "values", v)).reshape(-1))
        sl = slice(int(fo[i]), int(fo[i + 1]))
        sites.append(SiteCorrections(
            weights=w,
            charges=correction_charges(site.form_charges, w),
            c_p2p=out["c_p2p"][sl].copy(),
            c_lattice=out["c_lattice"][sl].copy(),
            c_dipole=out["c_dipole"][sl].copy(),
            blend_energy=float(out["blend"][i]),
        ))
    return CorrectionSet(sites=sites, fingerprint=_fingerprint(lam_values), device_offset=float(out["offset"]))


def build_corrections(system, lam_values, solver):
    """Correction scalars of every site (corrections.py:157-193), on the GPU."""
    lam, nl = lambda_table(system, lam_values)
    _bind_sites(solver, system)
    out = solver.plan.hi(lam, nl, _native.MODE_HI, site_positions=_site_positions(system), potentials=None,
                         want_forces=False)
    return _correction_set(system, lam_values, out, solver.plan)


def assemble_lambda_forces(system, lam_values, corrections, potentials):
    """F = -dH/dlambda per site (corrections.py:221-238), on the GPU."""
    fp = _fingerprint(lam_values)
    if corrections is not None and corrections.fingerprint != fp:
        raise ValueError("corrections were built for different lambda values")
    lam, nl = lambda_table(system, lam_values)
    tables = site_tables(system)
    ctot = None
    if corrections is not None:
        ctot = np.concatenate([s.c_total() for s in corrections.sites]) if corrections.sites else np.zeros(0)
    pot = np.asarray(potentials, dtype=np.float64).reshape(-1)
    out = _native.assemble(*tables, lam, nl, ctot, pot)
    return _split_forces(system, lam, nl, out)


def hi_energy_and_forces(system, lam_state, config=None, solver=None, mode="hi", *, spatial_forces=False):
    """One charge-scaled solve plus the fused HI correction (corrections.py:252-274).

    Charge scaling, the solve and the correction/assembly all run on the
    device; the potentials never leave device memory between them.
    ``spatial_forces=True`` (an extension; the reference signature is
    unchanged) also returns -grad_r of the returned energy from the same
    pass: spatial_forces(q~) (solver.py:407-427) on every atom plus, in HI
    mode, -grad Delta E_site on the site atoms (csrc/lfmm_hi.cuh).
    """
    if mode not in ("hi", "qi"):
        raise ValueError(f"unknown mode {mode!r}")
    lam_values = getattr(lam_state, "values", lam_state)
    if solver is None:
        solver = PeriodicSolver(system.positions, system.box_length, config)
    lam, nl = lambda_table(system, lam_values)
    _bind_sites(solver, system)
    plan = solver.plan
    qt = plan.scale_charges(np.asarray(system.charges, dtype=np.float64), lam, nl) if system.sites else \
        np.asarray(system.charges, dtype=np.float64)
    if spatial_forces:
        res, frc = solver.solve_with_forces(qt)
    else:
        res, frc = solver.solve(qt), None
    m = _native.MODE_QI if mode == "qi" else _native.MODE_HI
    out = plan.hi(lam, nl, m, site_positions=_site_positions(system), potentials=None, want_forces=True)
    forces = _split_forces(system, lam, nl, out["forces"])
    if mode == "qi":
        return InterpolationResult(energy=float(res.energy), forces=forces, mode=mode, solve=res, corrections=None,
                                   spatial_forces=frc)
    if frc is not None and system.sites:
        idx = np.concatenate([s.particle_indices for s in system.sites])
        frc[idx] += plan.hi_site_forces()
    corr = _correction_set(system, lam_values, out, plan)
    energy = float(res.energy) + corr.energy_offset()
    return InterpolationResult(energy=energy, forces=forces, mode=mode, solve=res, corrections=corr,
                               spatial_forces=frc)
