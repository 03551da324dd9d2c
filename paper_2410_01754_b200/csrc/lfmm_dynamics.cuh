// lfmm_dynamics.cuh — device-resident BAOAB integrator of the titration
// coordinates (reference: lambdafmm/dynamics.py:214-285, run_trajectory).
//
// The lambdas, their velocities and forces live on the device in the (S, 4)
// padded layout of lfmm_step (slot j < n_lambda[s] of site s is live), so an
// MD loop of lfmm_step (on_device) + these kernels never leaves the GPU.
// Each step of the reference is
//   B: v += (0.5 dt / m) F      A: x += (0.5 dt) v
//   O: v = c1 v + (noise / sqrt(m)) xi     A: x += (0.5 dt) v
//   F = COULOMB F_engine + F_bias + F_wall (at the new x)      B: v += (0.5 dt / m) F
// with the same association order as the numpy expressions.  The normals xi
// come from a counter-based Philox stream (seed, step, slot): reproducible and
// independent of launch geometry, but not numpy's default_rng sequence.
#pragma once

#include <curand_kernel.h>

namespace lfmm {

constexpr double LAM_WALL_LOW = -0.1, LAM_WALL_HIGH = 1.1, LAM_WALL_STRENGTH = 50000.0;  // dynamics.py:31-33

__device__ inline double lam_bias_force(double x, double h) {  // BiasPotential.force, dynamics.py:54-56
  return -32.0 * h * x * (1.0 - x) * (1.0 - 2.0 * x);
}
__device__ inline double lam_wall_force(double x) {  // wall_force, dynamics.py:66-70
  const double over = fmax(x - LAM_WALL_HIGH, 0.0), under = fmax(LAM_WALL_LOW - x, 0.0);
  return 4.0 * LAM_WALL_STRENGTH * (under * under * under - over * over * over);
}

// stage 0: B A O A with the stored total force; stage 1: total force from the
// engine's lambda forces at the current x, then B; stage 2: total force only
// (the initial evaluation)
__global__ void k_lambda_baoab(int n_sites, double* __restrict__ lam, double* __restrict__ vel,
                               const int* __restrict__ nl, const double* __restrict__ mass,
                               const double* __restrict__ f_eng, double* __restrict__ f_tot, int stage, double dt,
                               double coulomb, double bias_h, double c1, double noise, unsigned long long seed,
                               unsigned long long step) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * n_sites) return;
  const int s = i >> 2, j = i & 3;
  if (j >= nl[s]) return;
  const double m = mass[s];
  if (stage == 0) {
    double v = vel[i], x = lam[i];
    v += (0.5 * dt / m) * f_tot[i];
    x += (0.5 * dt) * v;
    curandStatePhilox4_32_10_t st;
    curand_init(seed, (unsigned long long)i, 4ULL * step, &st);
    const double xi = curand_normal_double(&st);
    v = c1 * v + (noise / sqrt(m)) * xi;
    x += (0.5 * dt) * v;
    vel[i] = v;
    lam[i] = x;
    return;
  }
  const double x = lam[i];
  const double f = f_eng[i] * coulomb + lam_bias_force(x, bias_h) + lam_wall_force(x);
  f_tot[i] = f;
  if (stage == 1) vel[i] += (0.5 * dt / m) * f;
}

// trajectory sample `k`: lambdas, velocities, total forces of the live slots
// (compacted in site order) and the engine energy in kJ/mol
__global__ void k_lambda_record(int n_sites, const int* __restrict__ slot_off, const int* __restrict__ nl,
                                const double* __restrict__ lam, const double* __restrict__ vel,
                                const double* __restrict__ f_tot, const double* __restrict__ energy, double coulomb,
                                int n_slots, double* __restrict__ out_x, double* __restrict__ out_v,
                                double* __restrict__ out_f, double* __restrict__ out_e, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) out_e[k] = energy[0] * coulomb;
  if (i >= 4 * n_sites) return;
  const int s = i >> 2, j = i & 3;
  if (j >= nl[s]) return;
  const size_t o = (size_t)k * n_slots + slot_off[s] + j;
  out_x[o] = lam[i];
  out_v[o] = vel[i];
  out_f[o] = f_tot[i];
}

}  // namespace lfmm
