/*
 * lfmm.h — C-ABI of the B200-native periodic FMM + HI (MAHI) electrostatics
 * step (arXiv 2410.01754 hot path).  Plain C types only: pointers, sizes,
 * int status codes.  No torch / CUDA types appear in any signature
 * (streams are passed as void*).
 *
 * The reference has no FFI: its operator API is the Python surface of
 * `lambdafmm`.  Each entry point below names the
 * reference function it stands behind (file:line relative to
 * /root/reference/pkg/src/lambdafmm).  The Python shim
 * `paper_2410_01754_b200` binds these with ctypes and re-exposes the
 * reference names (`PeriodicSolver`, `hi_energy_and_forces`, ...).
 *
 * Status codes: 0 ok; 1 invalid argument (shim raises ValueError);
 * 2 CUDA failure (RuntimeError); 3 non-finite result (NumericalFailure).
 * lfmm_last_error() returns the message of the last failure on the
 * calling thread.
 *
 * Layouts follow numpy C order of the reference arrays:
 *   positions (N,3) f64; charges (N,K) f64 with element [i*K+k];
 *   potentials (N,K); energies (K,); root multipole ((p+1)^2, K) complex
 *   stored as interleaved (re,im) doubles; dipole (3,K); forces (N,3).
 */
#ifndef LFMM_H
#define LFMM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lfmm_plan lfmm_plan;

enum { LFMM_OK = 0, LFMM_EINVAL = 1, LFMM_ECUDA = 2, LFMM_ENONFINITE = 3 };
enum { LFMM_LATTICE_OFF = 0, LFMM_LATTICE_CONVERGED = 1, LFMM_LATTICE_SHELLS = 2 };
enum {
  LFMM_F_DIPOLE = 1,         /* SolverConfig.dipole            solver.py:58  */
  LFMM_F_PERIODIC_NEAR = 2,  /* SolverConfig.periodic_near     solver.py:59  */
  LFMM_F_FP32 = 4,           /* SolverConfig.precision=single  solver.py:60  */
  LFMM_F_INTRA_MINIMUM = 8   /* SolverConfig.intra_site_images solver.py:61  */
};
enum { LFMM_MODE_HI = 0, LFMM_MODE_QI = 1 };

/* Library version string, e.g. "lfmm-b200 0.1.0 sm_100a". */
const char* lfmm_version(void);

/* Copy the last error message of this thread into buf (NUL-terminated). */
int lfmm_last_error(char* buf, int64_t len);

/* PeriodicSolver.__init__  fmm/solver.py:330-343 (+ octree.build_octree
 * fmm/octree.py:114-163, lattice.converged_operator fmm/lattice.py:124-155,
 * shell_sum_operator :109-121).  Validates the knobs exactly like
 * SolverConfig.validated (solver.py:60-75), wraps positions like
 * system.wrap_positions (system.py:103-108), builds the tree and every
 * translation operator on the device.  positions: host (N,3) f64. */
int lfmm_plan_create(const double* positions, int64_t n, double box_length,
                     int p, int depth, int lattice_mode, int shell_cap,
                     int flags, lfmm_plan** out);
int lfmm_plan_destroy(lfmm_plan* plan);

/* Use a caller-owned CUDA stream (cudaStream_t passed as void*); NULL
 * restores the plan's private stream. */
int lfmm_plan_set_stream(lfmm_plan* plan, void* stream);

/* Re-bind new positions (same N): the per-MD-step tree rebuild.  Equivalent
 * to constructing a fresh PeriodicSolver (solver.py:330-336) but reuses the
 * operators.  positions_on_device != 0: `positions` is a device pointer. */
int lfmm_plan_set_positions(lfmm_plan* plan, const double* positions,
                            int positions_on_device);

/* Basic sizes: out[0]=N, out[1]=p, out[2]=depth, out[3]=(p+1)^2,
 * out[4]=leaves, out[5]=flags. */
int lfmm_plan_info(const lfmm_plan* plan, int64_t* out6);

/* Octree export for bit-exact checks against octree.Octree (octree.py:71-93):
 * perm, inv_perm (N) i64; leaf_of_particle (N) i64; leaf_start (8^d+1) i64;
 * positions (N,3) f64 canonical order.  Any pointer may be NULL. */
int lfmm_export_tree(const lfmm_plan* plan, int64_t* perm, int64_t* inv_perm,
                     int64_t* leaf_of_particle, int64_t* leaf_start,
                     double* positions_sorted);

/* Interaction lists exactly as the device kernels enumerate them.
 * nb_box (8^d,27) i64, nb_shift (8^d,27,3) i64   (octree.py:136-139);
 * for level l>=1: m2l_src (8^l,189) i64 and m2l_row (8^l,189) i64, the
 * source box and M2L_OFFSETS row of every (target, slot)   (octree.py:96-111).
 * Any pointer may be NULL. */
int lfmm_export_lists(const lfmm_plan* plan, int level, int64_t* nb_box,
                      int64_t* nb_shift, int64_t* m2l_src, int64_t* m2l_row);

/* PeriodicSolver.lattice_matrix (solver.py:342-343, LatticeOperator.scaled
 * lattice.py:95-100): ((p+1)^2)^2 complex, interleaved, scaled to the box.
 * Returns EINVAL when lattice_mode is off. */
int lfmm_lattice_matrix(const lfmm_plan* plan, double* out_complex);

/* PeriodicSolver.solve (solver.py:349-405) and, when forces != NULL,
 * PeriodicSolver.spatial_forces (solver.py:407-427) from the same pass.
 * charges: (N,K) f64; host pointer unless io_on_device.  Every output may be
 * NULL (not computed/copied).  forces requires K == 1.
 * energies: (4,K) rows = total, near, far, dipole.
 * total_charge: (K,).  Outputs are host pointers unless io_on_device. */
int lfmm_solve(lfmm_plan* plan, const double* charges, int64_t k,
               int io_on_device, double* potentials, double* near_pot,
               double* far_pot, double* dip_pot, double* energies,
               double* root_multipole, double* dipole_vector,
               double* total_charge, double* forces);

/* Titratable-site tables (system.TitratableSite, system.py:30-51).
 * atom_offsets (S+1) i64 CSR into atom_index; atom_index: input-order
 * particle indices; n_forms (S) i32 (power of two, <=16); form_offsets (S+1)
 * i64 CSR into form_charges, site s holds n_forms[s] x n_atoms[s] f64 rows. */
int lfmm_sites_set(lfmm_plan* plan, int64_t n_sites, const int64_t* atom_offsets,
                   const int64_t* atom_index, const int32_t* n_forms,
                   const int64_t* form_offsets, const double* form_charges);

/* HI correction + lambda-force assembly (corrections.py:157-238, 252-274).
 * lambdas: (S,4) f64 padded, n_lambda (S) i32 with 2^n_lambda == n_forms.
 * site_positions: (A,3) f64 caller-supplied site-atom coordinates
 * (corrections.py:173 reads system.positions, not the solver's copy) or NULL
 * to gather them from the plan's raw input positions.
 * potentials: (N,) input-order f64 host array, or NULL to use the
 * potentials of the plan's last solve (device resident, K==1).
 * Outputs (host unless io_on_device; NULL = skip):
 *   c_p2p, c_lattice, c_dipole: per form, CSR like form_offsets/ n_atoms
 *     -> (sum n_forms) f64;  blend_energy (S) f64;  lambda_forces (S,4);
 *   energy_offset (1): sum over sites of e(q~) - w.C (CorrectionSet).
 * mode LFMM_MODE_QI skips the self-term removal (corrections.py:268-270). */
int lfmm_hi(lfmm_plan* plan, const double* lambdas, const int32_t* n_lambda,
            int mode, const double* site_positions, const double* potentials,
            int io_on_device, double* c_p2p, double* c_lattice,
            double* c_dipole, double* blend_energy, double* lambda_forces,
            double* energy_offset);

/* HI spatial forces of the site atoms (no reference counterpart: the
 * reference's only spatial forces are spatial_forces(q~), solver.py:407-427;
 * SURVEY.md §0.2 and §8c).  out (A,3) f64 in site-table atom order:
 * -grad_r Delta E_site, Delta E_site = e(q~) - sum_rho w_rho C_rho
 * (corrections.py:141-143, :179-183) from the last HI-mode lfmm_hi /
 * lfmm_step call.  The HI-consistent force on a site atom is
 * spatial_forces(q~) + this term; lfmm_step in HI mode returns the sum. */
int lfmm_hi_site_forces(lfmm_plan* plan, int io_on_device, double* out);

/* assemble_lambda_forces (corrections.py:221-238) without a plan:
 * S_rho = Q_rho . V[site] (s_values :196-198) and
 * F_k = -sum_rho dw_rho/dlambda_k (S_rho - C_rho)  (k_terms :201-218).
 * Site tables as in lfmm_sites_set; c_total (sum n_forms) f64 per form, or
 * NULL for the plain charge-route (QI) forces; potentials (n_particles,)
 * input order.  All pointers are host pointers.  out: (S,4) f64. */
/* Per-site form Gram B_s = Q_s (K_s + G_s) Q_s^T (HI_MAXF x HI_MAXF = 16 x 16
 * per site, row-major, host output): the correction table of
 * FrozenLambdaForceField (dynamics.py:137-145; K = near_kernel, G =
 * lattice_kernel, corrections.py:46-77), from the same k_hi_site pass as
 * lfmm_hi. */
int lfmm_site_gram(lfmm_plan* plan, const double* lambdas, const int32_t* n_lambda,
                   const double* site_positions, double* gram);

/* Device-resident BAOAB step pieces for the titration coordinates
 * (dynamics.py:214-285 run_trajectory).  All arrays are DEVICE pointers in the
 * (S,4) padded layout of lfmm_step; launched on the plan's stream.
 * stage 0: B A O A with f_total; stage 1: f_total = coulomb f_engine + bias +
 * wall at the current lambdas, then B; stage 2: f_total only.  Normals from a
 * Philox stream indexed by (seed, step, slot). */
int lfmm_lambda_baoab(lfmm_plan* plan, int64_t n_sites, double* lambdas, double* velocities,
                      const int32_t* n_lambda, const double* masses, const double* f_engine,
                      double* f_total, int stage, double dt, double coulomb, double bias_height,
                      double c1, double noise, uint64_t seed, uint64_t step);
/* Trajectory sample `sample` of the live slots (compacted by slot_offsets)
 * into device arrays (n_samples x n_slots) plus the energy in kJ/mol. */
int lfmm_lambda_record(lfmm_plan* plan, int64_t n_sites, const int32_t* slot_offsets,
                       const int32_t* n_lambda, const double* lambdas, const double* velocities,
                       const double* f_total, const double* energy, double coulomb, int64_t n_slots,
                       double* out_lambdas, double* out_velocities, double* out_forces,
                       double* out_energies, int64_t sample);

int lfmm_assemble(int64_t n_sites, const int64_t* atom_offsets, const int64_t* atom_index,
                  const int32_t* n_forms, const int64_t* form_offsets, const double* form_charges,
                  const double* lambdas, const int32_t* n_lambda, const double* c_total,
                  const double* potentials, int64_t n_particles, double* out);

/* scale_charges (system.py:179-197) on the device: charges (N,) with the
 * blended site charges written for the given lambdas. */
int lfmm_scale_charges(lfmm_plan* plan, const double* charges,
                       const double* lambdas, const int32_t* n_lambda,
                       int io_on_device, double* out_charges);

/* One full electrostatics step, the bench unit:
 * [tree rebuild from `positions` if not NULL] -> scale_charges -> solve with
 * potentials + spatial forces -> HI corrections -> lambda forces.
 * plain != 0 runs the fixed-protonation baseline instead (same positions,
 * `charges` used as is, no lambda machinery).
 * Outputs: energy (1) = E_solve + offset; forces (N,3) = -grad E of the
 * returned energy (spatial_forces(q~) plus, in HI mode, -grad Delta E_site on
 * the site atoms, see lfmm_hi_site_forces); lambda_forces (S,4);
 * potentials (N) optional. */
int lfmm_step(lfmm_plan* plan, const double* positions, const double* charges,
              const double* lambdas, const int32_t* n_lambda, int mode,
              int plain, int io_on_device, double* energy, double* forces,
              double* lambda_forces, double* potentials);

/* Per-stage device timing (CUDA events on the plan's stream).  enable != 0
 * starts recording; lfmm_stage_times copies accumulated milliseconds and
 * launch counts for the stages named by lfmm_stage_name(i). */
int lfmm_profile_enable(lfmm_plan* plan, int enable);
int lfmm_stage_count(void);
const char* lfmm_stage_name(int i);
int lfmm_stage_times(lfmm_plan* plan, double* ms, int64_t* launches, int n);

/* Number of kernel launches the library issued since plan creation. */
int64_t lfmm_launch_count(const lfmm_plan* plan);

/* ---- Octree slab decomposition (driven by
 * paper_2410_01754_b200/distributed.py, one rank per GPU).  Each rank owns
 * the leaves with x index in [x0, x1) of the global grid and holds its owned
 * atoms plus a one-leaf halo; levels < lg (boxes spanning ranks) are
 * computed redundantly from the gathered level lg.  No reference counterpart:
 * the reference is single-process. */

/* Re-size the plan's particle arrays for n particles (the local count
 * changes from step to step). */
int lfmm_plan_set_count(lfmm_plan* plan, int64_t n);

/* Owned leaf x-range and shared-level count; restricts P2P/L2P/energies/
 * dipole sums to owned leaves and the tensor-core M2L jobs to owned targets. */
int lfmm_dist_configure(lfmm_plan* plan, int x0, int x1, int lg);

/* phase 1: [tree from positions] + charges [+ lambda scaling] + P2P + P2M +
 * M2M of levels >= lg + exact box charges.  phase 2: levels < lg, lattice,
 * M2L, L2L, L2P, finalize, owned site-atom potentials.  Device pointers.
 * Between the phases the caller all-gathers the owned multipoles of levels
 * >= lg and replaces scal[0..3] by the global dipole and charge sums. */
int lfmm_dist_phase(lfmm_plan* plan, int phase, const double* positions, const double* charges,
                    const double* lambdas, const int32_t* n_lambda, int grad);

/* Device pointers of the exchanged buffers: ptrs[0] multipoles (all levels,
 * ncp per box), [1] scal (D_x, D_y, D_z, Q fp64), [2] energies (total, near,
 * far, dipole), [3] forces (N x 3 local input order), [4] site-atom
 * potentials, [5] lambda forces (S x 4), [6] HI energy offset, [7] the plan's
 * cudaStream_t, [8] per-level max |M/c| of the fp16 tensor-core M2L (uint32
 * float bits, DMAX + 2 entries; after phase 1 it holds this rank's slab of the
 * levels >= lg, which the caller max-reduces across ranks before phase 2).
 * ptrs holds 9 entries; level_off (8 entries): first box of each level. */
int lfmm_dist_buffers(lfmm_plan* plan, void** ptrs, int64_t* level_off, int64_t* ncp);

/* HI corrections + lambda forces for every site from the gathered site-atom
 * potentials (ptrs[4]); site_positions (A x 3, device) caller-supplied.  In
 * HI mode also adds -grad Delta E_site to the local force rows (ptrs[3]) of
 * the site atoms this rank holds (lfmm_hi_site_forces). */
int lfmm_dist_hi(lfmm_plan* plan, const double* site_positions, int mode);

#ifdef __cplusplus
}
#endif
#endif /* LFMM_H */
