"""Drop-in ``PeriodicSolver`` backed by the B200 kernels (reference fmm/solver.py).

Same constructor, attributes, result dataclass and error messages as the
reference (solver.py:36-96, :327-427).  Every number is computed on the GPU
through the C-ABI (include/lfmm.h); this module only converts arguments and
wraps results.  ``precision="double"`` runs the fp64 kernels,
``precision="single"`` the fp32 kernels (true fp32 arithmetic, fp64
energies/reductions), where the reference only rounds fp64 stages.
"""

from dataclasses import dataclass

import numpy as np

from .. import _native
from .octree import octree_view


@dataclass
class SolverConfig:
    p: int = 8
    depth: int = 2
    lattice_mode: str = "converged"
    shell_cap: int = 8
    dipole: bool = True
    periodic_near: bool = True
    precision: str = "double"
    intra_site_images: str = "full"

    def validated(self):
        # messages follow solver.py:60-75 word for word
        if not 1 <= self.p <= 40:
            raise ValueError(f"expansion order p={self.p} outside [1, 40]")
        if not 0 <= self.depth <= 6:
            raise ValueError(f"tree depth {self.depth} outside [0, 6]")
        if self.lattice_mode not in ("converged", "shells", "off"):
            raise ValueError(f"unknown lattice_mode {self.lattice_mode!r}")
        if self.lattice_mode == "shells" and self.shell_cap < 2:
            raise ValueError("shells mode needs shell_cap >= 2")
        if self.precision not in ("double", "single"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.intra_site_images not in ("full", "minimum"):
            raise ValueError(f"unknown intra_site_images {self.intra_site_images!r}")
        if not self.periodic_near and (self.depth != 0 or self.lattice_mode != "off"):
            raise ValueError("periodic_near=False requires depth=0 and lattice_mode='off'")
        return self

    def flags(self):
        return config_flags(self)


def config_flags(cfg):
    """C-ABI flag bits of a solver configuration.  Duck-typed: the
    reference's own SolverConfig objects (solver.py:36-75) are accepted as
    they are, so callers that build configs from lambdafmm (its bench, CLI
    and tests) work unchanged."""
    f = 0
    if cfg.dipole:
        f |= _native.F_DIPOLE
    if cfg.periodic_near:
        f |= _native.F_PERIODIC_NEAR
    if cfg.precision == "single":
        f |= _native.F_FP32
    if cfg.intra_site_images == "minimum":
        f |= _native.F_INTRA_MINIMUM
    return f


@dataclass
class SolveResult:
    potentials: np.ndarray
    near_potentials: np.ndarray
    far_potentials: np.ndarray
    dipole_potentials: np.ndarray
    energy: np.ndarray
    near_energy: np.ndarray
    far_energy: np.ndarray
    dipole_energy: np.ndarray
    root_multipole: np.ndarray
    dipole_vector: np.ndarray
    total_charge: np.ndarray


class PeriodicSolver:
    """Periodic FMM bound to one set of positions and one configuration."""

    def __init__(self, positions, box_length, config=None):
        self.config = (config or SolverConfig()).validated()
        self.box_length = float(box_length)
        cfg = self.config
        pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        self._plan = _native.Plan(pos, self.box_length, cfg.p, cfg.depth, _native.LFMM_LATTICE[cfg.lattice_mode],
                                  cfg.shell_cap, config_flags(cfg))
        self._n = pos.shape[0]
        self._positions = pos
        self._plan64 = None  # fp64 plan of spatial_forces under precision="single"
        self.lattice_matrix = None
        if cfg.lattice_mode != "off":
            lm = self._plan.lattice_matrix()
            lm.flags.writeable = False
            self.lattice_matrix = lm
        self._tree = None

    @property
    def num_particles(self):
        return self._n

    @property
    def tree(self):
        """Octree-compatible view exported from the device (octree.py:71-93)."""
        if self._tree is None:
            self._tree = octree_view(self._plan, self.box_length, self.config.depth)
        return self._tree

    @property
    def plan(self):
        return self._plan

    def _charges(self, charges):
        q = np.asarray(charges, dtype=np.float64)
        single = q.ndim == 1
        q2 = q[:, None] if single else q
        if q2.shape[0] != self.num_particles:
            raise ValueError(f"charges for {q2.shape[0]} particles, solver holds {self.num_particles}")
        return np.ascontiguousarray(q2), single

    def _result(self, out, single):
        def col(a):
            return a[:, 0] if single else a

        def scal(a):
            a = np.asarray(a, dtype=np.float64)
            return a[0] if single else a

        en = out["energies"]
        return SolveResult(
            potentials=col(out["potentials"]),
            near_potentials=col(out["near"]),
            far_potentials=col(out["far"]),
            dipole_potentials=col(out["dip"]),
            energy=scal(en[0]),
            near_energy=scal(en[1]),
            far_energy=scal(en[2]),
            dipole_energy=scal(en[3]),
            root_multipole=out["root"][:, 0] if single else out["root"],
            dipole_vector=out["dipole"][:, 0] if single else out["dipole"],
            total_charge=scal(out["qtot"]),
        )

    def solve(self, charges):
        q2, single = self._charges(charges)
        return self._result(self._plan.solve(q2), single)

    def solve_with_forces(self, charges):
        """One pass for potentials, energies and spatial forces (single column)."""
        q2, single = self._charges(np.asarray(charges, dtype=np.float64).reshape(-1))
        out = self._plan.solve(q2, forces=True)
        return self._result(out, True), out["forces"]

    def spatial_forces(self, charges):
        """Forces -q grad V on every particle, (N, 3) (solver.py:407-427).

        The reference evaluates spatial forces in full fp64 whatever the
        precision knob (its single-precision rounder only touches solve,
        solver.py:357-371, :407-427), so with precision="single" this runs
        on a lazily created fp64 plan over the same positions.  The fused
        fp32 step path (solve_with_forces, lfmm_step) keeps the plan's
        precision."""
        if self.config.precision == "single":
            if self._plan64 is None:
                cfg = self.config
                self._plan64 = _native.Plan(self._positions, self.box_length, cfg.p, cfg.depth,
                                            _native.LFMM_LATTICE[cfg.lattice_mode], cfg.shell_cap,
                                            config_flags(cfg) & ~_native.F_FP32)
            q2, _ = self._charges(np.asarray(charges, dtype=np.float64).reshape(-1))
            return self._plan64.solve(q2, forces=True)["forces"]
        _, f = self.solve_with_forces(charges)
        return f
