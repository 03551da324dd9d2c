"""Reference lambda-dynamics trajectories (pkg/src/lambdafmm/dynamics.py), the
parity target of paper_2410_01754_b200.dynamics.

* ``dyn_spring.npz``: run_trajectory (dynamics.py:214-285) over an analytic
  coupled-spring force field (no solver), thermostatted, two sites with one
  and two lambda slots, sample_every=7.
* ``dyn_frozen.npz``: run_trajectory over FrozenLambdaForceField
  (dynamics.py:88-171) of a small periodic system (the arrays are stored), HI
  mode, full images, p=8, depth=1.

Run where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dynamics.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lambdafmm import dynamics as rd  # noqa: E402
from lambdafmm.fmm.solver import SolverConfig  # noqa: E402
from lambdafmm.system import LambdaState, ParticleSystem, TitratableSite  # noqa: E402
from lambdafmm.units import COULOMB_KJ_PER_MOL  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


class CoupledSprings:
    """F_k = -k (lambda_k - c_k) - g * sum of the other slots (internal units)."""

    def lambda_forces(self, lam_values):
        flat = np.concatenate([np.asarray(v, float) for v in lam_values])
        k, g = 80.0 / COULOMB_KJ_PER_MOL, 15.0 / COULOMB_KJ_PER_MOL
        centre = np.linspace(0.35, 0.65, flat.size)
        f = -k * (flat - centre) - g * (flat.sum() - flat)
        e = 0.5 * k * float(((flat - centre) ** 2).sum())
        out, o = [], 0
        for v in lam_values:
            out.append(f[o:o + len(v)])
            o += len(v)
        return e, out


def traj_arrays(t):
    return dict(times=t.times, lambdas=t.lambdas, velocities=t.velocities, forces=t.forces, energies=t.energies)


def spring():
    lam = LambdaState(values=[np.array([0.3]), np.array([0.6, 0.2])], velocities=[np.array([0.1]), np.zeros(2)],
                      masses=[5.0, 3.0])
    t = rd.run_trajectory(CoupledSprings(), lam, 400, dt=0.002, temperature=300.0, friction=5.0,
                          bias=rd.BiasPotential(4.0), rng=np.random.default_rng(9), sample_every=7)
    np.savez_compressed(os.path.join(OUT, "dyn_spring.npz"), final_values=np.concatenate(lam.values),
                        final_velocities=np.concatenate(lam.velocities), **traj_arrays(t))


def frozen():
    rng = np.random.default_rng(6)
    box, n_bg, ns = 4.0, 40, 4
    pos = [rng.uniform(0, box, (n_bg, 3))]
    q = rng.uniform(-0.5, 0.5, n_bg)
    q -= q.mean()
    sites = []
    for s, nf in enumerate((2, 4)):
        c = rng.uniform(0, box, 3)
        pos.append((c + rng.uniform(-0.25, 0.25, (ns, 3))) % box)
        sites.append(TitratableSite(np.arange(n_bg + s * ns, n_bg + (s + 1) * ns), rng.uniform(-0.5, 0.5, (nf, ns))))
    positions = np.vstack(pos)
    charges = np.concatenate([q, np.zeros(2 * ns)])
    system = ParticleSystem(box, positions, charges, sites)
    lam = LambdaState(values=[np.array([0.4]), np.array([0.7, 0.25])], velocities=[np.zeros(1), np.zeros(2)],
                      masses=[5.0, 5.0])
    field = rd.FrozenLambdaForceField(system, config=SolverConfig(p=8, depth=1))
    t = rd.run_trajectory(field, lam, 150, dt=0.002, temperature=300.0, friction=5.0,
                          rng=np.random.default_rng(21), sample_every=3)
    np.savez_compressed(os.path.join(OUT, "dyn_frozen.npz"), box=box, positions=positions, charges=charges,
                        site0_idx=sites[0].particle_indices, site0_forms=sites[0].form_charges,
                        site1_idx=sites[1].particle_indices, site1_forms=sites[1].form_charges,
                        **traj_arrays(t))


if __name__ == "__main__":
    spring()
    frozen()
    print("wrote dyn_spring.npz dyn_frozen.npz")
