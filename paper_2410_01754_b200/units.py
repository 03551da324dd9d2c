"""Physical constants (the reference's units.py:16,19); internal energies are e^2/nm."""

COULOMB_KJ_PER_MOL = 138.935458  # kJ mol^-1 nm e^-2
BOLTZMANN_KJ_PER_MOL_K = 0.00831446261815324  # kJ mol^-1 K^-1 (N_A k_B, units.py:19)
