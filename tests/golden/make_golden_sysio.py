"""System-file fixtures written by the REFERENCE (system.py:215-301).

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_sysio.py

system_small.json: the reference's save_system of a small water box with two
sites (4 and 2 forms); system_small_loaded.npz: the arrays the reference's
load_system returns for it (the parity target of paper_2410_01754_b200.sysio).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from lambdafmm import system as rs  # noqa: E402

from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    system, lam, _ = generate_water_box(1500, 2, forms_per_site=4, seed=5)
    sites = [rs.TitratableSite(particle_indices=s.particle_indices, form_charges=s.form_charges) for s in system.sites]
    ref_sys = rs.ParticleSystem(box_length=system.box_length, positions=system.positions, charges=system.charges,
                                sites=sites)
    ref_lam = rs.LambdaState(values=[np.asarray(v, float) for v in lam.values],
                             velocities=[np.full(len(v), 0.01) for v in lam.values], masses=[5.0, 7.5])
    path = os.path.join(OUT, "system_small.json")
    rs.save_system(ref_sys, ref_lam, path)
    s2, l2 = rs.load_system(path)
    np.savez_compressed(os.path.join(OUT, "system_small_loaded.npz"), box=s2.box_length, positions=s2.positions,
                        charges=s2.charges, site0_idx=s2.sites[0].particle_indices,
                        site0_forms=s2.sites[0].form_charges, site1_idx=s2.sites[1].particle_indices,
                        site1_forms=s2.sites[1].form_charges, lambdas=np.concatenate(l2.values),
                        velocities=np.concatenate(l2.velocities), masses=np.asarray(l2.masses))
    print("wrote system_small.json", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
