// lfmm_api.cu — the C-ABI (include/lfmm.h) over the B200 kernels.
//
// One plan = one PeriodicSolver (fmm/solver.py:327-427): it owns every device
// buffer (tree, expansions, operators, outputs) and runs on one CUDA stream.
// All work is issued asynchronously on that stream; host<->device copies
// happen only at the API edges (host pointers) or not at all (device
// pointers, io_on_device != 0).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "lfmm_common.cuh"
#include "lfmm_dynamics.cuh"
#include "lfmm_expansions.cuh"
#include "lfmm_hi.cuh"
#include "lfmm_m2l_halo.cuh"
#include "lfmm_p2p.cuh"
#include "lfmm_setup.cuh"
#include "lfmm_translate_tc.cuh"
#include "lfmm_tree.cuh"

using namespace lfmm;

namespace {

thread_local std::string g_last_error;

enum Stage {
  ST_TREE = 0,
  ST_STAGE,
  ST_P2P,
  ST_P2M,
  ST_M2M,
  ST_ROOT,
  ST_DOWN,
  ST_L2L,
  ST_L2P,
  ST_FINAL,
  ST_HI,
  ST_SCALE,
  ST_SETUP,
  ST_PACK,
  ST_COUNT
};
const char* kStageNames[ST_COUNT] = {"tree",  "stage_q", "p2p",      "p2m", "m2m",   "lattice",
                                     "m2l", "l2l", "l2p",   "finalize", "hi",  "scale", "setup", "m2l_pack"};

// ------------------------------------------------------------ kernels ----
// Fixed-order reduction of NQ double-double block partials by one block.
template <int NQ>
__device__ void reduce_parts_dev(const dd* __restrict__ part, int nb, double* __restrict__ out) {
  dd v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = dd{0, 0};
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = min(nb, (int)threadIdx.x * per), b1 = min(nb, b0 + per);
  for (int b = b0; b < b1; ++b)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      dd x;
      x.hi = __ldcg(&part[(size_t)b * NQ + q].hi);
      x.lo = __ldcg(&part[(size_t)b * NQ + q].lo);
      v[q] = dd_add(v[q], x);
    }
  __shared__ dd res[NQ];
  block_reduce_dd<NQ>(v, res);
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) out[q] = res[q].hi + res[q].lo;
}

// true in exactly one block: the last to finish its partial (counter reset)
__device__ bool last_block(int* cnt) {
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(cnt, 1);
    is_last = (old == (int)gridDim.x - 1);
    if (is_last) *cnt = 0;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last != 0;
}

template <class T>
__global__ void k_stage_q(const double* __restrict__ q, int K, int c, const int* __restrict__ perm,
                          const double* __restrict__ pos_sorted, int64_t n, double box,
                          vec4_t<T>* __restrict__ xq, double* __restrict__ qs, dd* __restrict__ part,
                          int* __restrict__ cnt, double* __restrict__ scal, const int* __restrict__ leaf_sorted,
                          int depth, int x0, int x1, const int* __restrict__ leaf_start, float4* __restrict__ pb) {
  dd v[4] = {dd{0, 0}, dd{0, 0}, dd{0, 0}, dd{0, 0}};
  // grid-stride (a few blocks per SM: the last-block counter sees few atomics)
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = perm[k];
    const double qv = q[(size_t)i * K + c];
    xq[k].w = (T)qv;
    qs[k] = qv;
    const int leaf = leaf_sorted[k];
    if (pb) {  // charge half of the source pair (lfmm_tree.cuh k_leaf_rank)
      const int s0 = leaf_start[leaf], r = (int)k - s0;
      reinterpret_cast<float*>(pb + ((s0 + leaf + 1) >> 1) + (r >> 1))[2 + (r & 1)] = (float)qv;
    }
    const int lx = leaf >> (2 * depth);
    if (lx < x0 || lx >= x1) continue;  // halo atom: not this rank's dipole / charge
    const double h = 0.5 * box;
    v[0] = dd_add(v[0], dd_from((pos_sorted[3 * k] - h) * qv));
    v[1] = dd_add(v[1], dd_from((pos_sorted[3 * k + 1] - h) * qv));
    v[2] = dd_add(v[2], dd_from((pos_sorted[3 * k + 2] - h) * qv));
    v[3] = dd_add(v[3], dd_from(qv));
  }
  block_reduce_dd<4>(v, part + (size_t)blockIdx.x * 4);
  if (last_block(cnt)) reduce_parts_dev<4>(part, gridDim.x, scal);
}

template <class T>
__global__ void k_transpose_ops(const T* __restrict__ in, T* __restrict__ out, int ncp, int nmat) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nmat * ncp * ncp) return;
  const int64_t m = i / ((int64_t)ncp * ncp);
  const int r = (int)((i / ncp) % ncp), k = (int)(i % ncp);
  out[(m * ncp + k) * ncp + r] = in[i];
}

template <class T, int CPW, int NS>
inline size_t tr_smem_bytes(int ncp) {
  return sizeof(T) * (NS * (size_t)TR_KC * ncp + NS * (size_t)(8 * CPW) * TR_KC);
}

// one k_translate launch: CPW = 8 columns per warp (64 per CTA) once there
// are enough target columns to fill the GPU (2-stage ring), else 2 (16 per
// CTA) with the whole K extent in flight (latency-bound small levels)
template <class T>
inline void tr_launch(const TrArgs& ta, int ncols_total, int noct, cudaStream_t st) {
  if (ncols_total >= 4096) {
    const unsigned tiles = (unsigned)((ncols_total + 63) / 64);
    k_translate<T, 8, 2><<<dim3(tiles, noct), TR_THREADS, tr_smem_bytes<T, 8, 2>(ta.ncp), st>>>(ta);
  } else {
    const unsigned tiles = (unsigned)((ncols_total + 15) / 16);
    k_translate<T, 2, 4><<<dim3(tiles, noct), TR_THREADS, tr_smem_bytes<T, 2, 4>(ta.ncp), st>>>(ta);
  }
}
// fp32 M2M / L2L on the tensor cores: 64 columns per CTA on the big
// levels, 16 on the small ones (more CTAs in flight)
inline void tt_launch(const TrArgs& ta, int ncols_total, const void* img, cudaStream_t st) {
  const auto* im = static_cast<const unsigned char*>(img);
  if (ncols_total >= 4096)
    k_translate_tc<64, 2><<<dim3((ncols_total + 63) / 64, 8), TT_THREADS, tt_smem_bytes<64, 2>(), st>>>(ta, im);
  else
    k_translate_tc<16, 2><<<dim3((ncols_total + 15) / 16, 8), TT_THREADS, tt_smem_bytes<16, 2>(), st>>>(ta, im);
}
// The 81-97 KB CTAs of k_translate_tc run beside the near-field CTAs only if
// the SMs were configured for the whole shared-memory carveout by the kernels
// running when the near field lands on them (a resident persistent CTA keeps
// the SM from being reconfigured): P2M, charge staging, near field.
// parent levels <= TT_CHAIN_TOP (<= 64 parents) in one k_translate_tc_chain
// launch: 8 octants x 4 tiles of 16 columns
constexpr int TT_CHAIN_TOP = 2;
inline void tt_chain_launch(const TtChain& ch, const void* img, cudaStream_t st) {
  LFMM_CUDA(cudaMemsetAsync(ch.bar, 0, sizeof(unsigned), st));
  k_translate_tc_chain<16, 2><<<8 * 4, TT_THREADS, tt_smem_bytes<16, 2>(), st>>>(
      ch, static_cast<const unsigned char*>(img));
}
inline void tt_set_attrs() {
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tt_smem_bytes<64, 2>()));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tt_smem_bytes<16, 2>()));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc<64, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc<16, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc_chain<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tt_smem_bytes<16, 2>()));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate_tc_chain<16, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_p2m_c<float, 10>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_stage_q<float>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_p2p2<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  LFMM_CUDA(cudaFuncSetAttribute(k_p2p2<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}
template <class T>
inline void tr_set_attrs(int ncp) {
  LFMM_CUDA(cudaFuncSetAttribute(k_translate<T, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tr_smem_bytes<T, 8, 2>(ncp)));
  LFMM_CUDA(cudaFuncSetAttribute(k_translate<T, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tr_smem_bytes<T, 2, 4>(ncp)));
}

// Exact box charges (the l = 0 multipole) at every level.  The fp32 P2M/M2M
// sums of the ~30 repeated water charges per leaf round coherently: summed
// over 32k leaves they leave a fake net charge of ~5e-3 e that the M2L turns
// into a constant far-potential offset of ~4e-4 of max|V| (tools/
// diag_precision.py).  Each box's charge is summed here in fp64 (leaf atoms in
// canonical order, then 8 children per parent, fixed order) and rounded once
// into coefficient 0; only the l = 0 column is replaced, the higher moments
// keep the P2M/M2M values.  Multi-block leaf pass; the last block to finish
// sums the parent levels.
template <class T>
__global__ void k_box_charges(const double* __restrict__ qs, const int* __restrict__ leaf_start, int depth,
                              int64_t leaf_off, int ncp, T* __restrict__ mult, double* __restrict__ boxq,
                              int* __restrict__ cnt, int wmin) {
  // phase 1: thread per leaf, grouped 8 per level-(d-1) parent in octant
  // order; lane 8g of each group then adds its 8 leaves in octant order
  if (depth >= 1) {
    const int pl = depth - 1, pn = 1 << pl, cn = 2 * pn;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int pb = t >> 3, o = t & 7;
    const bool valid = pb < (1 << (3 * pl));
    double c = 0.0;
    if (valid) {
      const int x = pb >> (2 * pl), y = (pb >> pl) & (pn - 1), z = pb & (pn - 1);
      const int leaf = (((2 * x + ((o >> 2) & 1)) * cn) + 2 * y + ((o >> 1) & 1)) * cn + 2 * z + (o & 1);
      for (int i = leaf_start[leaf]; i < leaf_start[leaf + 1]; ++i) c += qs[i];
      boxq[leaf_off + leaf] = c;
      mult[(size_t)(leaf_off + leaf) * ncp] = (T)c;
    }
    double pc = 0.0;
    const int base = (threadIdx.x & 31) & ~7;
#pragma unroll
    for (int k = 0; k < 8; ++k) pc += __shfl_sync(0xffffffffu, c, base + k);
    if (valid && o == 0) {
      const int64_t poff = leaf_off - (1LL << (3 * pl));
      boxq[poff + pb] = pc;
      if (depth - 1 >= wmin) mult[(size_t)(poff + pb) * ncp] = (T)pc;
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    double c = 0.0;
    for (int i = leaf_start[0]; i < leaf_start[1]; ++i) c += qs[i];
    boxq[0] = c;
    mult[0] = (T)c;
  }
  if (depth < 2 || !last_block(cnt)) return;
  // phase 2 (last block): levels d-2 .. 0, 8 children each in octant order
  int64_t child_off = leaf_off - (1LL << (3 * (depth - 1)));
  for (int l = depth - 2; l >= 0; --l) {
    const int n = 1 << l, nb = 1 << (3 * l);
    const int64_t off = child_off - nb;  // level_off[l] (levels are stored consecutively)
    for (int pb = threadIdx.x; pb < nb; pb += blockDim.x) {
      const int x = pb >> (2 * l), y = (pb >> l) & (n - 1), z = pb & (n - 1);
      double c = 0.0;
      for (int o = 0; o < 8; ++o) {
        const int cx = 2 * x + ((o >> 2) & 1), cy = 2 * y + ((o >> 1) & 1), cz = 2 * z + (o & 1);
        c += __ldcg(&boxq[child_off + ((((int64_t)cx << (l + 1)) | (cy)) << (l + 1) | cz)]);
      }
      boxq[off + pb] = c;
      if (l >= wmin) mult[(size_t)(off + pb) * ncp] = (T)c;
    }
    __syncthreads();
    __threadfence_block();
    child_off = off;
  }
}

template <int NQ>
__global__ void k_reduce_parts(const dd* __restrict__ part, int nb, double* __restrict__ out) {
  dd v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = dd{0, 0};
  // contiguous chunks per thread keep the order fixed
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = min(nb, (int)threadIdx.x * per), b1 = min(nb, b0 + per);
  for (int b = b0; b < b1; ++b)
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = dd_add(v[q], part[(size_t)b * NQ + q]);
  __shared__ dd res[NQ];
  block_reduce_dd<NQ>(v, res);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) out[q] = res[q].hi + res[q].lo;
}

template <class T, bool GRAD>
__global__ void k_finalize(int64_t n, int K, int c, const int* __restrict__ perm,
                           const double* __restrict__ pos_sorted, const double* __restrict__ qs,
                           const T* __restrict__ vnear, const T* __restrict__ vfar,
                           const T* __restrict__ gnear, const T* __restrict__ gfar,
                           const double* __restrict__ scal /* Dx,Dy,Dz,Q */, int dipole, double box,
                           double* __restrict__ out_pot, double* __restrict__ out_near,
                           double* __restrict__ out_far, double* __restrict__ out_dip,
                           double* __restrict__ out_forces, dd* __restrict__ part, int* __restrict__ cnt,
                           double* __restrict__ epart, double* __restrict__ energies, double* __restrict__ dvec,
                           double* __restrict__ qtot, const int* __restrict__ leaf_sorted, int depth, int x0,
                           int x1) {
  dd v[2] = {dd{0, 0}, dd{0, 0}};
#pragma unroll 2
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = perm[k];
    const double q = qs[k];
    const double vn = (double)vnear[k], vf = (double)vfar[k];
    const double gam = 2.0 * 3.14159265358979323846 / (3.0 * box * box * box);
    const double h = 0.5 * box;
    double vd = 0.0;
    if (dipole && (out_pot || out_dip))  // the step path outputs forces only: no position reads
      vd = 2.0 * DIPOLE_ETA * gam *
           ((pos_sorted[3 * k] - h) * scal[0] + (pos_sorted[3 * k + 1] - h) * scal[1] +
            (pos_sorted[3 * k + 2] - h) * scal[2]);
    const size_t o = (size_t)i * K + c;
    if (out_pot) out_pot[o] = vn + vf + vd;
    if (out_near) out_near[o] = vn;
    if (out_far) out_far[o] = vf;
    if (out_dip) out_dip[o] = vd;
    if (GRAD && out_forces) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double f = -q * ((double)gnear[3 * k + a] + (double)gfar[3 * k + a]);
        if (dipole) f += -2.0 * DIPOLE_ETA * gam * q * scal[a];
        out_forces[3 * (size_t)i + a] = f;
      }
    }
    const int lx = leaf_sorted[k] >> (2 * depth);
    if (lx < x0 || lx >= x1) continue;  // halo atom: energy counted by its owner
    v[0] = dd_add(v[0], dd_from(q * vn));
    v[1] = dd_add(v[1], dd_from(q * vf));
  }
  block_reduce_dd<2>(v, part + (size_t)blockIdx.x * 2);
  if (last_block(cnt)) {
    reduce_parts_dev<2>(part, gridDim.x, epart);
    __syncthreads();
    if (threadIdx.x == 0) {
      const double gam = 2.0 * 3.14159265358979323846 / (3.0 * box * box * box);
      const double en = 0.5 * epart[0], ef = 0.5 * epart[1];
      const double ed =
          dipole ? DIPOLE_ETA * gam * (scal[0] * scal[0] + scal[1] * scal[1] + scal[2] * scal[2]) : 0.0;
      energies[0 * K + c] = en + ef + ed;
      energies[1 * K + c] = en;
      energies[2 * K + c] = ef;
      energies[3 * K + c] = ed;
      dvec[0 * K + c] = scal[0];
      dvec[1 * K + c] = scal[1];
      dvec[2 * K + c] = scal[2];
      qtot[c] = scal[3];
    }
  }
}

// Total potential at the site atoms straight from the canonical-order
// pieces (the step path skips the input-order potential arrays):
// V = V_near + V_far + 2 eta gamma (r - L/2).D   (solver.py:373-379)
template <class T>
__device__ __forceinline__ double site_pot_at(int i, const int* __restrict__ inv_perm, const T* __restrict__ vnear,
                                              const T* __restrict__ vfar, const double* __restrict__ pos_sorted,
                                              const double* __restrict__ scal, int dipole, double box,
                                              const int* __restrict__ leaf_sorted, int depth, int x0, int x1) {
  if (i < 0) return 0.0;  // site atom held by another rank (distributed.py)
  const int k = inv_perm[i];
  const int lx = leaf_sorted[k] >> (2 * depth);
  if (lx < x0 || lx >= x1) return 0.0;  // halo atom: its owner supplies the potential
  double v = (double)vnear[k] + (double)vfar[k];
  if (dipole) {
    const double gam = 2.0 * 3.14159265358979323846 / (3.0 * box * box * box), h = 0.5 * box;
    v += 2.0 * DIPOLE_ETA * gam *
         ((pos_sorted[3 * k] - h) * scal[0] + (pos_sorted[3 * k + 1] - h) * scal[1] +
          (pos_sorted[3 * k + 2] - h) * scal[2]);
  }
  return v;
}

template <class T>
__global__ void k_site_pot(const int* __restrict__ atom_idx, int n, const int* __restrict__ inv_perm,
                           const T* __restrict__ vnear, const T* __restrict__ vfar,
                           const double* __restrict__ pos_sorted, const double* __restrict__ scal, int dipole,
                           double box, double* __restrict__ out, const int* __restrict__ leaf_sorted, int depth,
                           int x0, int x1) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  out[a] = site_pot_at<T>(atom_idx[a], inv_perm, vnear, vfar, pos_sorted, scal, dipole, box, leaf_sorted, depth, x0,
                          x1);
}

// The single-GPU step's tail in one launch, warp per site: the site-atom
// potentials (k_site_pot), the lambda forces (hi_lambda_site, the sums of
// k_hi_site in its order), the HI spatial forces added into the force rows
// (k_add_site_forces) and the step energy (k_step_energy).  Every value is
// the one the four separate kernels produce.
template <class T>
struct TailArgs {
  const int* inv_perm;
  const T* vnear;
  const T* vfar;
  const double* pos_sorted;
  const double* scal;
  int dipole;
  const int* leaf_sorted;
  int depth, x0, x1;
  double* pot_site;          // A
  double* forces;            // N x 3, input order
  const double* site_force;  // A x 3, or null (QI mode)
  const double* energies;
  const double* off;
  int add_off;
  double* energy_out;
};

template <class T>
__global__ void k_step_tail(HiArgs g, TailArgs<T> t) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *t.energy_out = t.energies[0] + (t.add_off ? t.off[0] : 0.0);
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= g.n_sites) return;
  const int a0 = g.atom_off[s], a1 = g.atom_off[s + 1];
  for (int a = a0 + lane; a < a1; a += 32) {
    const int i = g.atom_idx[a];
    t.pot_site[a] = site_pot_at<T>(i, t.inv_perm, t.vnear, t.vfar, t.pos_sorted, t.scal, t.dipole, g.box,
                                   t.leaf_sorted, t.depth, t.x0, t.x1);
    if (t.site_force && i >= 0)
      for (int k = 0; k < 3; ++k) t.forces[3 * (size_t)i + k] += t.site_force[3 * a + k];
  }
  __syncwarp();
  hi_lambda_site(g, s, lane);
}

// warp per site: S_rho and lambda forces from given potentials and C_rho
__global__ void k_assemble(int S, const int* __restrict__ atom_off, const int* __restrict__ atom_idx,
                           const int* __restrict__ nforms, const int* __restrict__ form_off,
                           const int* __restrict__ fslot_off, const double* __restrict__ form_q,
                           const double* __restrict__ lambdas, const int* __restrict__ nlam,
                           const double* __restrict__ c_total, const double* __restrict__ pot,
                           double* __restrict__ out) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  const int a0 = atom_off[s], ns = atom_off[s + 1] - a0, nf = nforms[s], nl = nlam[s];
  const double* Q = form_q + form_off[s];
  const double* lam = lambdas + 4 * s;
  double f[4] = {0, 0, 0, 0};
  for (int r = 0; r < nf; ++r) {
    double sv = 0.0;
    for (int i = lane; i < ns; i += 32) sv += Q[r * ns + i] * pot[atom_idx[a0 + i]];
    for (int off = 16; off > 0; off >>= 1) sv += __shfl_down_sync(0xffffffffu, sv, off);
    if (c_total) sv -= c_total[fslot_off[s] + r];
    for (int k = 0; k < nl; ++k) f[k] += hi_wgrad(lam, nl, k, r) * sv;
  }
  if (lane == 0)
    for (int k = 0; k < 4; ++k) out[4 * s + k] = k < nl ? -f[k] : 0.0;
}

__global__ void k_step_energy(const double* __restrict__ energies, const double* __restrict__ off, int add,
                              double* __restrict__ out) {
  *out = energies[0] + (add ? off[0] : 0.0);
}

__global__ void k_i32_to_i64(const int* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// ------------------------------------------------------ host helpers ----
// bumped by every device (re)allocation: a captured step graph holds raw
// buffer addresses and is re-captured when this moves
std::atomic<uint64_t> g_alloc_gen{0};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  friend void swap(DevBuf& a, DevBuf& b) noexcept {
    std::swap(a.p, b.p);
    std::swap(a.bytes, b.bytes);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return;
    LFMM_CUDA(cudaMalloc(&p, b));
    bytes = b;
    g_alloc_gen.fetch_add(1);
  }
  void release() {
    if (p) {
      cudaFree(p);
      g_alloc_gen.fetch_add(1);
    }
    p = nullptr;
    bytes = 0;
  }
  template <class U>
  U* as() const {
    return reinterpret_cast<U*>(p);
  }
};

std::once_flag g_const_once;
std::vector<std::array<int, 3>> g_m2l_offsets;  // 316 rows (octree.py:31)

void init_constants() {
  // 1/((l+m)(l-m)) and 1/(2m)
  std::vector<double> inv_lm((PMAX + 2) * (PMAX + 2), 0.0);
  std::vector<float> inv_lm_f((PMAX + 2) * (PMAX + 2), 0.0f);
  std::vector<double> inv2m(PMAX + 2, 0.0);
  std::vector<float> inv2m_f(PMAX + 2, 0.0f);
  for (int l = 0; l <= PMAX + 1; ++l)
    for (int m = 0; m < l; ++m) {
      inv_lm[l * (PMAX + 2) + m] = 1.0 / double((l + m) * (l - m));
      inv_lm_f[l * (PMAX + 2) + m] = (float)inv_lm[l * (PMAX + 2) + m];
    }
  for (int m = 1; m <= PMAX + 1; ++m) {
    inv2m[m] = 1.0 / (2.0 * m);
    inv2m_f[m] = (float)inv2m[m];
  }
  LFMM_CUDA(cudaMemcpyToSymbol(c_inv_lm_d, inv_lm.data(), inv_lm.size() * sizeof(double)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_inv_lm_f, inv_lm_f.data(), inv_lm_f.size() * sizeof(float)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_inv_2m_d, inv2m.data(), inv2m.size() * sizeof(double)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_inv_2m_f, inv2m_f.data(), inv2m_f.size() * sizeof(float)));
  // M2L offsets in lexicographic order over [-3,3]^3 with Chebyshev norm >= 2,
  // and per parity the valid rows (-2-par <= o <= 3-par per axis)
  g_m2l_offsets.clear();
  for (int x = -3; x <= 3; ++x)
    for (int y = -3; y <= 3; ++y)
      for (int z = -3; z <= 3; ++z)
        if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) >= 2) g_m2l_offsets.push_back({x, y, z});
  std::vector<char4> off(8 * NM2L);
  std::vector<short> rows(8 * NM2L);
  for (int par = 0; par < 8; ++par) {
    const int pb[3] = {(par >> 2) & 1, (par >> 1) & 1, par & 1};
    int s = 0;
    for (int r = 0; r < (int)g_m2l_offsets.size(); ++r) {
      bool ok = true;
      for (int a = 0; a < 3; ++a) ok = ok && (-2 - pb[a] <= g_m2l_offsets[r][a]) && (g_m2l_offsets[r][a] <= 3 - pb[a]);
      if (!ok) continue;
      if (s >= NM2L) throw Error{LFMM_ECUDA, "M2L list overflow"};
      off[par * NM2L + s] = make_char4((char)g_m2l_offsets[r][0], (char)g_m2l_offsets[r][1],
                                       (char)g_m2l_offsets[r][2], 0);
      rows[par * NM2L + s] = (short)r;
      ++s;
    }
    if (s != NM2L) throw Error{LFMM_ECUDA, "M2L list size mismatch"};
  }
  LFMM_CUDA(cudaMemcpyToSymbol(c_m2l_off, off.data(), off.size() * sizeof(char4)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_m2l_row, rows.data(), rows.size() * sizeof(short)));
  // halo M2L: per (target class tc, source class sc) the offsets o with
  // tc + o = 2d + sc, as {operator row, d}
  std::vector<int> hn(64, 0);
  std::vector<short> hrow(64 * 27, 0);
  std::vector<char4> hd(64 * 27, make_char4(0, 0, 0, 0));
  for (int tc = 0; tc < 8; ++tc)
    for (int s = 0; s < NM2L; ++s) {
      const char4 o = off[tc * NM2L + s];
      const int tcb[3] = {(tc >> 2) & 1, (tc >> 1) & 1, tc & 1};
      const int oo[3] = {o.x, o.y, o.z};
      int sc = 0, d[3];
      for (int a = 0; a < 3; ++a) {
        const int v = tcb[a] + oo[a];
        const int par = ((v % 2) + 2) % 2;
        d[a] = (v - par) / 2;
        sc = (sc << 1) | par;
      }
      const int tab = tc * 8 + sc;
      if (hn[tab] >= 27) throw Error{LFMM_ECUDA, "halo term table overflow"};
      hrow[tab * 27 + hn[tab]] = rows[tc * NM2L + s];
      hd[tab * 27 + hn[tab]] = make_char4((char)d[0], (char)d[1], (char)d[2], 0);
      hn[tab]++;
    }
  LFMM_CUDA(cudaMemcpyToSymbol(c_hterm_n, hn.data(), hn.size() * sizeof(int)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_hterm_row, hrow.data(), hrow.size() * sizeof(short)));
  LFMM_CUDA(cudaMemcpyToSymbol(c_hterm_d, hd.data(), hd.size() * sizeof(char4)));
}

// process-level cache of unit-box lattice operators, like lru_cache on
// converged_operator / shell_sum_operator (lattice.py:108, :123)
std::mutex g_lat_mu;
std::map<std::tuple<int, int, int>, std::vector<double2>> g_lat_cache;

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// The dynamic shared-memory limit is a per-function, process-wide attribute;
// plans with different halo tiles (e.g. ranks of a slab decomposition driven
// from threads of one process) must not lower it under each other: set it
// once to the device's opt-in maximum.
// Returns the A-ring depth (k_m2l_halo<AS>) whose shared memory fits:
// 14 stages, or 10 when the halo windows of a depth-6 level need the room.
int halo_smem_attr(int rw_cap) {
  static std::once_flag once;
  static int max_optin = 0;
  std::call_once(once, [] {
    int dev = 0;
    LFMM_CUDA(cudaGetDevice(&dev));
    LFMM_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{}, fb{};
    LFMM_CUDA(cudaFuncGetAttributes(&fa, k_m2l_halo<HM_ASTAGES>));
    LFMM_CUDA(cudaFuncGetAttributes(&fb, k_m2l_halo<HM_ASTAGES_SMALL>));
    // static shared memory counts against the same limit
    max_optin -= (int)std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
    LFMM_CUDA(cudaFuncSetAttribute(k_m2l_halo<HM_ASTAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    LFMM_CUDA(
        cudaFuncSetAttribute(k_m2l_halo<HM_ASTAGES_SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
  });
  if (hm_smem_bytes(rw_cap, HM_ASTAGES) <= (size_t)max_optin) return HM_ASTAGES;
  LFMM_REQUIRE(hm_smem_bytes(rw_cap, HM_ASTAGES_SMALL) <= (size_t)max_optin,
               "halo M2L tile needs more shared memory than the device offers");
  return HM_ASTAGES_SMALL;
}

// persistent launch: at most `ctas` CTAs (one per SM) walk the njobs jobs of
// ha.jobs through the zeroed ha.counter
void launch_m2l_halo(HaloArgs ha, int njobs, int ctas, int astages, cudaStream_t st) {
  ha.njobs = njobs;
  LFMM_CUDA(cudaMemsetAsync(ha.counter, 0, sizeof(int), st));
  const unsigned grid = (unsigned)std::max(1, std::min(njobs, ctas));
  if (astages == HM_ASTAGES)
    k_m2l_halo<HM_ASTAGES><<<grid, HM_THREADS, hm_smem_bytes(ha.rw_cap, HM_ASTAGES), st>>>(ha);
  else
    k_m2l_halo<HM_ASTAGES_SMALL><<<grid, HM_THREADS, hm_smem_bytes(ha.rw_cap, HM_ASTAGES_SMALL), st>>>(ha);
}

}  // namespace

// ----------------------------------------------------------------- plan ----
struct lfmm_plan {
  int64_t N = 0;
  double L = 0.0;
  int p = 0, depth = 0, lattice_mode = 0, shell_cap = 0, flags = 0;
  bool fp32 = false;
  int nc = 0, ncp = 0, nleaf = 0;
  double size = 0.0;  // leaf edge
  int64_t level_off[DMAX + 2] = {0};
  int64_t nbox_total = 0;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  // host-I/O overlap for lfmm_step: charges upload and forces download run on
  // io_stream beside the tree build / HI work of `stream`
  cudaStream_t io_stream = nullptr;
  cudaEvent_t ev_q = nullptr, ev_f = nullptr;
  static constexpr int kPosChunks = 4;          // host positions upload in chunks (build_tree)
  cudaEvent_t ev_pos[kPosChunks + 1] = {};     // [0]: main stream ready, [1..]: chunk c landed
  // P2P runs on near_stream (lower priority) beside the far-field chain on
  // `stream`: the latency-bound translation / tree / HI kernels of the chain
  // leave SMs the near field fills.  Serialised when profiling.
  cudaStream_t near_stream = nullptr;
  cudaEvent_t ev_near_in = nullptr, ev_near_out = nullptr;
  bool near_pending = false;
  // HI corrections (site geometry only) run on hi_stream beside the solve
  cudaStream_t hi_stream = nullptr;
  cudaEvent_t ev_hi_in = nullptr, ev_hi_out = nullptr;
  int64_t launches = 0;
  bool profiling = false;
  struct Ev {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> free_events;
  double stage_ms[ST_COUNT] = {0};
  int64_t stage_launch[ST_COUNT] = {0};

  // tree
  DevBuf scan_status;  // k_scan_lookback block states
  DevBuf pos_in, key32, leaf_of, slot_of, counts, cursor, leaf_start, bucket, perm, inv_perm, pos_sorted, leaf_sorted, xq;
  // fp32 near-field source pairs (k_p2p2): [pair_cap] float4 x/y halves, then [pair_cap] z/q halves
  DevBuf pairs;
  int64_t pair_cap = 0;
  DevBuf gram;  // lfmm_site_gram output
  float4* pair_a() { return fp32 ? reinterpret_cast<float4*>(pairs.p) : nullptr; }
  float4* pair_b() { return fp32 ? reinterpret_cast<float4*>(pairs.p) + pair_cap : nullptr; }
  // expansions / operators
  bool use_halo = false;  // fp32 M2L on tcgen05 as shifted-window fp16x3 GEMMs (lfmm_m2l_halo.cuh)
  bool p2p_scalar = false;  // fp32 P2P on the scalar kernel (LFMM_P2P=scalar, A/B checks)
  bool step_mode = false;   // lfmm_step: skip the input-order potential arrays
  // Slab decomposition (distributed.py): this rank owns leaves with x index in
  // [own_x0, own_x1); levels < dist_lg have boxes spanning ranks and are
  // computed redundantly from the gathered level dist_lg.  dist_phase: 0 whole
  // solve, 1 up to the owned multipoles, 2 the rest.
  int own_x0 = 0, own_x1 = 1 << 30, dist_lg = 0, dist_phase = 0;
  DevBuf up_part, up_cnt, counters;
  DevBuf ops16, hm_inv_r, hm_inv_c, hm_jobs, hm_level_max, mult16, ops_m2l_t;
  DevBuf hm_counter;  // job counters of the persistent M2L launches (main, far stream)
  DevBuf p2p_ctl;     // preemptible near field: leaf counter, stop flags of launches 1, 2, 3
  cudaEvent_t ev_m2l_done = nullptr;
  int p2p_c1 = 3, p2p_c2 = 3;  // CTAs per SM of near-field launches 1 and 2 (room for the far-field chains)
  bool p2p_preempt = true;
  // lfmm_step with device-resident inputs as one CUDA graph: captured on the
  // second call with the same arguments, replayed while the arguments, the
  // stream and every device allocation stay the same (LFMM_GRAPH=0: off)
  bool graphs = true;
  uint64_t epoch = 0;  // bumped by every call that changes sizes or tables a captured step bakes in
  struct StepGraph {
    std::array<const void*, 10> ptrs{};
    int mode = -1, plain = -1;
    cudaStream_t stream = nullptr;
    uint64_t gen = 0, epoch = 0;
    bool warm = false;
    cudaGraphExec_t exec = nullptr;
    int64_t nlaunch = 0;
  } step_graph;
  bool near_after_hi = false;  // lfmm_step without a tree rebuild (set per call)
  int nsm = 148;
  int64_t m16_off[DMAX + 2] = {0};
  int hm_njobs = 0, hm_rw_cap = 0, hm_astages = HM_ASTAGES;
  static constexpr int hm_stagger = 8;       // terms issuer 1 lags issuer 0 (capped at AS - 6 in the kernel)
  static constexpr int hm_groups_big = 2;    // M2L jobs (partial slots) per tile at levels >= 4
  static constexpr int hm_groups_small = 8;  // ... at levels < 4 (one source class per job)
  bool m2l_f64_simt = false;  // fp64 M2L on k_gemm_gather instead of k_m2l_f64 (LFMM_M2L64=gather)
  DevBuf mult, loc, partial, ops_m2l, ops_m2m, ops_l2l, ops_lat, lat64t;
  std::vector<double2> lat_unit;  // unit-box complex lattice operator (nc x nc)
  // solve work
  DevBuf boxq, site_pot;
  DevBuf ops_m2m_t, ops_l2l_t, ops_lat_t, tr_cnt;  // k_translate operators ([k][row]) and tile counters
  bool use_tr = false;                  // M2M / L2L on k_translate (ncp == 128)
  bool use_tt = false;                  // ... fp32 on k_translate_tc (tensor cores)
  bool tt_simt = false;                 // LFMM_TRANSLATE=simt: fp32 on k_translate
  DevBuf tt_m2m, tt_l2l;                // k_translate_tc operator images
  DevBuf tt_bar;                        // k_translate_tc_chain grid-barrier counter
  DevBuf q_in, qs, vnear, vfar, gnear, gfar, part, scal, epart, roots;
  DevBuf out_pot, out_near, out_far, out_dip, out_forces, energies, dvec, qtot;
  int64_t last_k = 0;
  bool last_valid = false;
  // sites
  int64_t n_sites = 0, n_site_atoms = 0, n_form_slots = 0;
  int ns_max = 0;
  std::vector<int> h_atom_off, h_atom_idx, h_nforms, h_fslot_off;
  DevBuf atom_off, atom_idx, nforms, form_off, fslot_off, form_q, site_pos, lambdas, nlam, rscr, uscr;
  DevBuf c_p2p, c_lat, c_dip, blend, lam_forces, offsets, offset_total, pot_tmp, q_tmp;
  DevBuf site_force;  // A x 3: -grad Delta E_site of the last HI-mode correction pass
  bool site_force_valid = false;

  size_t tsz() const { return fp32 ? sizeof(float) : sizeof(double); }
  // leaf b's pairs start at (leaf_start[b] + b + 1) / 2 (lfmm_p2p.cuh)
  void ensure_pairs(int64_t nn) {
    if (!fp32) return;
    pair_cap = (nn + nleaf + 2) / 2 + 1;
    pairs.ensure(2 * sizeof(float4) * pair_cap);
  }

  // --- launch bookkeeping ---
  cudaEvent_t get_event() {
    if (!free_events.empty()) {
      cudaEvent_t e = free_events.back();
      free_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    LFMM_CUDA(cudaEventCreate(&e));
    return e;
  }
  // tracing (profiling build, tools/step_trace.py): events on the launching
  // stream around every launch without serialising the streams
  bool tracing = false;
  cudaEvent_t trace_base = nullptr;
  std::vector<Ev> trace;
  cudaStream_t rec_stream = nullptr;  // stream of the launch in flight (launch_on)
  template <class F>
  void launch(int stage, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t rs = rec_stream ? rec_stream : stream;
    if (profiling || tracing) {
      a = get_event();
      b = get_event();
      LFMM_CUDA(cudaEventRecord(a, rs));
    }
    f();
    LFMM_CUDA(cudaGetLastError());
    ++launches;
    stage_launch[stage]++;
    if (profiling) {
      LFMM_CUDA(cudaEventRecord(b, rs));
      pending.push_back({stage, a, b});
    } else if (tracing) {
      LFMM_CUDA(cudaEventRecord(b, rs));
      trace.push_back({stage, a, b});
    }
  }
  template <class F>
  void launch_on(int stage, cudaStream_t st, F&& f) {
    cudaStream_t prev = rec_stream;
    rec_stream = st;
    launch(stage, f);
    rec_stream = prev;
  }
  void harvest() {
    if (pending.empty()) return;
    LFMM_CUDA(cudaStreamSynchronize(stream));
    for (auto& e : pending) {
      float ms = 0.f;
      LFMM_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
      stage_ms[e.stage] += ms;
      free_events.push_back(e.a);
      free_events.push_back(e.b);
    }
    pending.clear();
  }
  ~lfmm_plan() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& e : pending) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    for (auto e : free_events) cudaEventDestroy(e);
    DevBuf* hbufs[] = {&ops16, &hm_inv_r, &hm_inv_c, &hm_jobs, &hm_counter, &p2p_ctl, &hm_level_max, &mult16, &boxq, &site_pot, &ops_m2m_t, &ops_l2l_t, &ops_lat_t, &tr_cnt, &ops_m2l_t, &tt_m2m, &tt_l2l, &scan_status, &tt_bar};
    for (auto* b : hbufs) b->release();
    DevBuf* bufs[] = {&pos_in, &key32, &leaf_of, &slot_of, &counts, &cursor, &leaf_start, &bucket, &perm,
                      &inv_perm, &pos_sorted, &leaf_sorted, &xq, &mult, &loc, &partial, &up_part, &up_cnt, &counters, &ops_m2l, &ops_m2m,
                      &ops_l2l, &ops_lat, &lat64t, &q_in, &qs, &vnear, &vfar, &gnear, &gfar, &part,
                      &scal, &epart, &roots, &out_pot, &out_near, &out_far, &out_dip, &out_forces, &energies,
                      &dvec, &qtot, &atom_off, &atom_idx, &nforms, &form_off, &fslot_off, &form_q,
                      &site_pos, &lambdas, &nlam, &rscr, &uscr, &c_p2p, &c_lat, &c_dip, &blend,
                      &lam_forces, &offsets, &offset_total, &pot_tmp, &q_tmp, &site_force};
    for (auto* b : bufs) b->release();
    if (own_stream) cudaStreamDestroy(own_stream);
    if (io_stream) cudaStreamDestroy(io_stream);
    if (near_stream) cudaStreamDestroy(near_stream);
    if (hi_stream) cudaStreamDestroy(hi_stream);
    if (ev_hi_in) cudaEventDestroy(ev_hi_in);
    if (ev_hi_out) cudaEventDestroy(ev_hi_out);
    if (ev_near_in) cudaEventDestroy(ev_near_in);
    if (ev_near_out) cudaEventDestroy(ev_near_out);
    if (ev_q) cudaEventDestroy(ev_q);
    for (auto e : ev_pos)
      if (e) cudaEventDestroy(e);
    if (ev_m2l_done) cudaEventDestroy(ev_m2l_done);
    if (step_graph.exec) cudaGraphExecDestroy(step_graph.exec);
    if (ev_f) cudaEventDestroy(ev_f);
  }

  // ------------------------------------------------ operator setup ----
  template <class T>
  void realify(int kind, int nmat, const double2* data, int64_t stride, double out_pow, int out_add,
               double in_pow, T* out) {
    const int64_t total = (int64_t)ncp * ncp * nmat;
    launch(ST_SETUP, [&] {
      k_realify<T><<<nblk(total, 256), 256, 0, stream>>>(kind, p, nmat, data, stride, out_pow, out_add, in_pow,
                                                         out, ncp);
    });
  }

  std::vector<double2> build_lattice_unit() {
    const int nco = ncoef(p), P2 = 2 * p, nc2 = ncoef(P2);
    auto key = std::make_tuple(p, lattice_mode, lattice_mode == LFMM_LATTICE_SHELLS ? shell_cap : 0);
    {
      std::lock_guard<std::mutex> lk(g_lat_mu);
      auto it = g_lat_cache.find(key);
      if (it != g_lat_cache.end()) return it->second;
    }
    // image vectors
    auto shell = [](int smin, int smax) {
      std::vector<double> v;
      for (int x = -smax; x <= smax; ++x)
        for (int y = -smax; y <= smax; ++y)
          for (int z = -smax; z <= smax; ++z) {
            const int nrm = std::max(std::abs(x), std::max(std::abs(y), std::abs(z)));
            if (nrm >= smin && nrm <= smax) {
              v.push_back(x);
              v.push_back(y);
              v.push_back(z);
            }
          }
      return v;
    };
    DevBuf vecs, vals, ivsum, rvsum, t_ring, s_hat, bmat, tmp, total, fin;
    ivsum.ensure(sizeof(double2) * nc2);
    LFMM_CUDA(cudaMemsetAsync(ivsum.p, 0, ivsum.bytes, stream));
    auto sum_harmonics = [&](const std::vector<double>& v, int order, int irregular, DevBuf& acc) {
      const int nv = (int)v.size() / 3, ncoefs = ncoef(order);
      const int chunk = 1024;
      vecs.ensure(sizeof(double) * 3 * chunk);
      vals.ensure(sizeof(double2) * (size_t)ncoefs * chunk);
      for (int lo = 0; lo < nv; lo += chunk) {
        const int cnt = std::min(chunk, nv - lo);
        LFMM_CUDA(cudaMemcpyAsync(vecs.p, v.data() + 3 * lo, sizeof(double) * 3 * cnt, cudaMemcpyHostToDevice,
                                  stream));
        launch(ST_SETUP, [&] {
          k_harmonics_full<<<nblk(cnt, 64), 64, 0, stream>>>(vecs.as<double>(), cnt, order, irregular,
                                                              vals.as<double2>());
        });
        launch(ST_SETUP, [&] {
          k_sum_vectors<<<nblk(ncoefs, 128), 128, 0, stream>>>(vals.as<double2>(), cnt, ncoefs,
                                                                acc.as<double2>());
        });
        LFMM_CUDA(cudaStreamSynchronize(stream));  // host vector chunk reuse
      }
    };
    const int64_t nn = (int64_t)nco * nco;
    total.ensure(sizeof(double2) * nn);
    fin.ensure(sizeof(double2) * nn);
    if (lattice_mode == LFMM_LATTICE_SHELLS) {
      auto v = shell(2, shell_cap);
      if (!v.empty()) sum_harmonics(v, P2, 1, ivsum);
      launch(ST_SETUP, [&] {
        k_dense_from_vector<<<nblk(nn, 256), 256, 0, stream>>>(OP_M2L, ivsum.as<double2>(), p, 1.0,
                                                               total.as<double2>());
      });
      launch(ST_SETUP, [&] {
        k_lattice_finish<<<nblk(nn, 256), 256, 0, stream>>>(total.as<double2>(), fin.as<double2>(), p, 0);
      });
    } else {
      // converged_operator: factor-3 telescoping, 24 steps (lattice.py:124-155)
      auto ring = shell(2, 4);
      sum_harmonics(ring, P2, 1, ivsum);
      auto w27 = shell(0, 1);
      rvsum.ensure(sizeof(double2) * nco);
      LFMM_CUDA(cudaMemsetAsync(rvsum.p, 0, rvsum.bytes, stream));
      sum_harmonics(w27, p, 0, rvsum);
      t_ring.ensure(sizeof(double2) * nn);
      s_hat.ensure(sizeof(double2) * nn);
      bmat.ensure(sizeof(double2) * nn);
      tmp.ensure(sizeof(double2) * nn);
      launch(ST_SETUP, [&] {
        k_dense_from_vector<<<nblk(nn, 256), 256, 0, stream>>>(OP_M2L, ivsum.as<double2>(), p, 1.0,
                                                               t_ring.as<double2>());
      });
      launch(ST_SETUP, [&] {
        k_dense_from_vector<<<nblk(nn, 256), 256, 0, stream>>>(OP_M2M, rvsum.as<double2>(), p, 1.0 / 3.0,
                                                               s_hat.as<double2>());
      });
      launch(ST_SETUP, [&] { k_identity<<<nblk(nn, 256), 256, 0, stream>>>(bmat.as<double2>(), nco); });
      LFMM_CUDA(cudaMemsetAsync(total.p, 0, total.bytes, stream));
      dim3 zb(16, 16), zg((nco + 15) / 16, (nco + 15) / 16);
      const int steps = 24;
      for (int k = 0; k < steps; ++k) {
        launch(ST_SETUP, [&] {
          k_zgemm<<<zg, zb, 0, stream>>>(t_ring.as<double2>(), bmat.as<double2>(), tmp.as<double2>(), nco);
        });
        launch(ST_SETUP, [&] {
          k_lattice_accum<<<nblk(nn, 256), 256, 0, stream>>>(total.as<double2>(), tmp.as<double2>(), p, k);
        });
        if (k + 1 < steps) {
          launch(ST_SETUP, [&] {
            k_zgemm<<<zg, zb, 0, stream>>>(s_hat.as<double2>(), bmat.as<double2>(), tmp.as<double2>(), nco);
          });
          swap(bmat, tmp);
        }
      }
      launch(ST_SETUP, [&] {
        k_lattice_finish<<<nblk(nn, 256), 256, 0, stream>>>(total.as<double2>(), fin.as<double2>(), p, 4);
      });
    }
    std::vector<double2> host(nn);
    LFMM_CUDA(cudaMemcpyAsync(host.data(), fin.p, sizeof(double2) * nn, cudaMemcpyDeviceToHost, stream));
    LFMM_CUDA(cudaStreamSynchronize(stream));
    DevBuf* tmpbufs[] = {&vecs, &vals, &ivsum, &rvsum, &t_ring, &s_hat, &bmat, &tmp, &total, &fin};
    for (auto* b : tmpbufs) b->release();
    std::lock_guard<std::mutex> lk(g_lat_mu);
    g_lat_cache[key] = host;
    return host;
  }

  template <class T>
  void build_operators() {
    const size_t opb = (size_t)ncp * ncp * sizeof(T);
    ops_m2l.ensure(opb * NOFF);
    ops_m2m.ensure(opb * 8);
    ops_l2l.ensure(opb * 8);
    DevBuf vecs, vals;
    // M2L: irregular(o, 2p) of the 316 unit offsets
    {
      std::vector<double> v;
      for (auto& o : g_m2l_offsets) {
        v.push_back(o[0]);
        v.push_back(o[1]);
        v.push_back(o[2]);
      }
      const int nc2 = ncoef(2 * p);
      vecs.ensure(sizeof(double) * v.size());
      vals.ensure(sizeof(double2) * (size_t)nc2 * NOFF);
      LFMM_CUDA(cudaMemcpyAsync(vecs.p, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, stream));
      launch(ST_SETUP, [&] {
        k_harmonics_full<<<nblk(NOFF, 64), 64, 0, stream>>>(vecs.as<double>(), NOFF, 2 * p, 1,
                                                             vals.as<double2>());
      });
      realify<T>(OP_M2L, NOFF, vals.as<double2>(), nc2, 1.0, 0, 1.0, ops_m2l.as<T>());
      if (sizeof(T) == 8 && ncp == 128) {  // [k][row] copy for k_m2l_f64
        ops_m2l_t.ensure(opb * NOFF);
        launch(ST_SETUP, [&] {
          k_transpose_ops<T><<<nblk((int64_t)NOFF * ncp * ncp, 256), 256, 0, stream>>>(ops_m2l.as<T>(),
                                                                                  ops_m2l_t.as<T>(), ncp, NOFF);
        });
        static std::once_flag f64_once;
        std::call_once(f64_once, [] {
          LFMM_CUDA(cudaFuncSetAttribute(k_m2l_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F64_SMEM));
        });
      }
      LFMM_CUDA(cudaStreamSynchronize(stream));
    }
    // M2M (parent edge 1, child 1/2): A(d) = gather R(-d), d = (0.5-oct)/2;
    // normalised by child^j; L2L: C = gather R(d)^T, d = (oct-0.5)/2,
    // normalised by child^(j+1)
    for (int which = 0; which < 2; ++which) {
      std::vector<double> v;
      for (int oct = 0; oct < 8; ++oct) {
        const int ob[3] = {(oct >> 2) & 1, (oct >> 1) & 1, oct & 1};
        for (int a = 0; a < 3; ++a) {
          const double d = which == 0 ? (0.5 - ob[a]) * 0.5 : (ob[a] - 0.5) * 0.5;
          v.push_back(which == 0 ? -d : d);
        }
      }
      const int ncr = ncoef(p);
      vecs.ensure(sizeof(double) * v.size());
      vals.ensure(sizeof(double2) * (size_t)ncr * 8);
      LFMM_CUDA(cudaMemcpyAsync(vecs.p, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, stream));
      launch(ST_SETUP, [&] {
        k_harmonics_full<<<1, 64, 0, stream>>>(vecs.as<double>(), 8, p, 0, vals.as<double2>());
      });
      if (which == 0)
        realify<T>(OP_M2M, 8, vals.as<double2>(), ncr, 1.0, 0, 0.5, ops_m2m.as<T>());
      else
        realify<T>(OP_L2L, 8, vals.as<double2>(), ncr, 0.5, 1, 1.0, ops_l2l.as<T>());
      LFMM_CUDA(cudaStreamSynchronize(stream));
    }
    use_tr = (ncp == 128) && depth >= 1;
    if (use_tr) {
      ops_m2m_t.ensure(opb * 8);
      ops_l2l_t.ensure(opb * 8);
      const int64_t tot = (int64_t)8 * ncp * ncp;
      launch(ST_SETUP, [&] {
        k_transpose_ops<T><<<nblk(tot, 256), 256, 0, stream>>>(ops_m2m.as<T>(), ops_m2m_t.as<T>(), ncp, 8);
      });
      launch(ST_SETUP, [&] {
        k_transpose_ops<T><<<nblk(tot, 256), 256, 0, stream>>>(ops_l2l.as<T>(), ops_l2l_t.as<T>(), ncp, 8);
      });
      const int64_t tiles = std::max<int64_t>(1, ((1LL << (3 * (depth - 1))) + 15) / 16);
      tr_cnt.ensure(sizeof(int) * tiles);
      LFMM_CUDA(cudaMemsetAsync(tr_cnt.p, 0, tr_cnt.bytes, stream));
      tr_set_attrs<T>(ncp);
      use_tt = sizeof(T) == 4 && !tt_simt;
      if (use_tt) {
        tt_m2m.ensure((size_t)8 * TT_OPBYTES);
        tt_l2l.ensure((size_t)8 * TT_OPBYTES);
        launch(ST_SETUP, [&] {
          k_tt_ops<<<nblk(8 * 128 * 128, 256), 256, 0, stream>>>(ops_m2m.as<float>(), tt_m2m.as<unsigned char>());
        });
        launch(ST_SETUP, [&] {
          k_tt_ops<<<nblk(8 * 128 * 128, 256), 256, 0, stream>>>(ops_l2l.as<float>(), tt_l2l.as<unsigned char>());
        });
        tt_bar.ensure(sizeof(unsigned) * 4);
        tt_set_attrs();
      }
    }
    if (lattice_mode != LFMM_LATTICE_OFF) {
      lat_unit = build_lattice_unit();
      const int64_t nn = (int64_t)nc * nc;
      vals.ensure(sizeof(double2) * nn);
      LFMM_CUDA(cudaMemcpyAsync(vals.p, lat_unit.data(), sizeof(double2) * nn, cudaMemcpyHostToDevice, stream));
      ops_lat.ensure(opb);
      realify<T>(OP_DENSE, 1, vals.as<double2>(), nn, 1.0, 0, 1.0, ops_lat.as<T>());
      if (use_tr) {
        ops_lat_t.ensure(opb);
        launch(ST_SETUP, [&] {
          k_transpose_ops<T><<<nblk((int64_t)ncp * ncp, 256), 256, 0, stream>>>(ops_lat.as<T>(), ops_lat_t.as<T>(), ncp, 1);
        });
      }
      // fp64 transposed copy for the HI lattice kernel
      DevBuf l64;
      l64.ensure(sizeof(double) * ncp * ncp);
      realify<double>(OP_DENSE, 1, vals.as<double2>(), nn, 1.0, 0, 1.0, l64.as<double>());
      std::vector<double> h(ncp * (size_t)ncp), ht(ncp * (size_t)ncp);
      LFMM_CUDA(cudaMemcpyAsync(h.data(), l64.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, stream));
      LFMM_CUDA(cudaStreamSynchronize(stream));
      for (int a = 0; a < ncp; ++a)
        for (int b = 0; b < ncp; ++b) ht[(size_t)b * ncp + a] = h[(size_t)a * ncp + b];
      lat64t.ensure(sizeof(double) * ht.size());
      LFMM_CUDA(cudaMemcpyAsync(lat64t.p, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice, stream));
      LFMM_CUDA(cudaStreamSynchronize(stream));
      l64.release();
    }
    if (use_halo) build_halo_operators();
    if (fp32) {
      LFMM_CUDA(cudaFuncSetAttribute(k_p2p2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2P2_SMEM));
      LFMM_CUDA(cudaFuncSetAttribute(k_p2p2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2P2_SMEM));

    }
    LFMM_CUDA(cudaStreamSynchronize(stream));
    vecs.release();
    vals.release();
  }

  // Halo M2L operators: power-of-two row/column equilibration of the 316
  // fp32 operators (so fp16 hi/lo pairs keep 22 bits, tools/m2l_fp16_study.py),
  // then the pre-arranged fp16 chunks.  The scales depend on p only.
  void build_halo_operators() {
    const size_t nel = (size_t)NOFF * 128 * 128;
    std::vector<float> h(nel);
    LFMM_CUDA(cudaMemcpyAsync(h.data(), ops_m2l.p, nel * sizeof(float), cudaMemcpyDeviceToHost, stream));
    LFMM_CUDA(cudaStreamSynchronize(stream));
    std::vector<double> amax(128 * 128, 0.0);
    for (size_t o = 0; o < (size_t)NOFF; ++o)
      for (int i = 0; i < 128 * 128; ++i) amax[i] = std::max(amax[i], (double)std::fabs(h[o * 16384 + i]));
    std::vector<double> r(128, 1.0), c(128, 1.0);
    for (int iter = 0; iter < 30; ++iter) {
      for (int a = 0; a < 128; ++a) {
        double m = 0.0;
        for (int b = 0; b < 128; ++b) m = std::max(m, r[a] * amax[a * 128 + b] * c[b]);
        if (m > 0) r[a] /= std::sqrt(m);
      }
      for (int b = 0; b < 128; ++b) {
        double m = 0.0;
        for (int a = 0; a < 128; ++a) m = std::max(m, r[a] * amax[a * 128 + b] * c[b]);
        if (m > 0) c[b] /= std::sqrt(m);
      }
    }
    std::vector<float> rs(128), cs(128), ir(128), ic(128);
    for (int a = 0; a < 128; ++a) {
      const double pr = std::exp2(std::round(std::log2(r[a]))), pc = std::exp2(std::round(std::log2(c[a])));
      rs[a] = (float)pr;
      cs[a] = (float)pc;
      ir[a] = (float)(1.0 / pr);
      ic[a] = (float)(1.0 / pc);
    }
    DevBuf drs, dcs;
    drs.ensure(sizeof(float) * 128);
    dcs.ensure(sizeof(float) * 128);
    hm_inv_r.ensure(sizeof(float) * 128);
    hm_inv_c.ensure(sizeof(float) * 128);
    LFMM_CUDA(cudaMemcpyAsync(drs.p, rs.data(), 512, cudaMemcpyHostToDevice, stream));
    LFMM_CUDA(cudaMemcpyAsync(dcs.p, cs.data(), 512, cudaMemcpyHostToDevice, stream));
    LFMM_CUDA(cudaMemcpyAsync(hm_inv_r.p, ir.data(), 512, cudaMemcpyHostToDevice, stream));
    LFMM_CUDA(cudaMemcpyAsync(hm_inv_c.p, ic.data(), 512, cudaMemcpyHostToDevice, stream));
    ops16.ensure((size_t)NOFF * HM_NKC * HM_ATILE);
    launch(ST_SETUP, [&] {
      k_h16_arrange<<<nblk((int64_t)nel, 256), 256, 0, stream>>>(ops_m2l.as<float>(), drs.as<float>(), dcs.as<float>(),
                                                                 ops16.as<unsigned char>(), NOFF);
    });
    LFMM_CUDA(cudaStreamSynchronize(stream));
    hm_level_max.ensure(sizeof(unsigned int) * (DMAX + 2));
    hm_astages = halo_smem_attr(hm_rw_cap);
  }

  // Halo M2L jobs: (level, target class, 256-row tile of the padded linear
  // class grid, group of source classes); level d first so the small levels
  // fill the tail of the single launch.  Groups: 4 per tile (pairs of source
  // classes with |D| 26+19 / 25+23) at levels >= 4, one source class per job
  // below.  Each group writes its own partial slot.
  void plan_halo_jobs() {
    std::vector<int4> jobs;
    int64_t off = 0;
    hm_rw_cap = 0;
    for (int l = depth; l >= 1; --l) nsplit[l] = (l >= 4) ? hm_groups_big : hm_groups_small;
    for (int l = 1; l <= depth; ++l) {
      part_off[l] = off;
      off += (int64_t)nsplit[l] << (3 * l);
    }
    for (int l = depth; l >= 1; --l) {
      const int h = 1 << (l - 1), Z = h + 2, S = Z * Z + Z + 1, last = h * S;
      const int G = nsplit[l];
      // target classes' x rows owned by this rank (all of them unless a slab
      // decomposition restricts levels >= dist_lg): class position i with
      // 2i + tcx inside the rank's box range at level l
      for (int tc = 0; tc < 8; ++tc) {
        int ia = 0, ib = h;
        if (dist_lg > 0 && l >= dist_lg) {
          const int xl0 = own_x0 >> (depth - l), xl1 = own_x1 >> (depth - l), tcx = (tc >> 2) & 1;
          ia = (xl0 - tcx + 1) >> 1;
          ib = (xl1 - tcx + 1) >> 1;
          if (ia >= ib) continue;
        }
        const int r0 = S + ia * Z * Z, r1 = std::min(last, S + (ib - 1) * Z * Z + h * Z + h);
        // tiles of equal size (a multiple of 16 rows, <= HM_NMAX): a short
        // last tile would cost a full tile's MMA issue for a few rows
        const int rows = r1 + 1 - r0, ntile = (rows + HM_NMAX - 1) / HM_NMAX;
        const int nt16 = ((rows + ntile - 1) / ntile + 15) / 16 * 16;
        for (int t0 = r0; t0 <= r1; t0 += nt16) {
          const int N = std::min(nt16, ((r1 + 1 - t0) + 15) / 16 * 16);
          hm_rw_cap = std::max(hm_rw_cap, hm_rw(N, Z));
          for (int grp = 0; grp < G; ++grp) jobs.push_back(make_int4(l | (tc << 4) | (grp << 8) | (G << 12), t0, N, 0));
        }
      }
    }
    // big jobs first: the small levels' short jobs fill the tail of the
    // persistent launch
    std::stable_sort(jobs.begin(), jobs.end(), [](const int4& a, const int4& b) { return a.z > b.z; });
    int64_t moff = 0;
    for (int l = 1; l <= depth; ++l) {
      m16_off[l] = moff;
      moff += (int64_t)256 * hm_plane_rows(l) * 16;
    }
    mult16.ensure(std::max<int64_t>(moff, 16));
    hm_njobs = (int)jobs.size();
    hm_counter.ensure(sizeof(int) * 2);
    p2p_ctl.ensure(sizeof(int) * 4);
    if (!ev_m2l_done) LFMM_CUDA(cudaEventCreateWithFlags(&ev_m2l_done, cudaEventDisableTiming));
    hm_jobs.ensure(sizeof(int4) * std::max<size_t>(jobs.size(), 1));
    if (!jobs.empty())
      LFMM_CUDA(cudaMemcpyAsync(hm_jobs.p, jobs.data(), sizeof(int4) * jobs.size(), cudaMemcpyHostToDevice, stream));
    LFMM_CUDA(cudaStreamSynchronize(stream));
    partial.ensure(tsz() * ncp * std::max<int64_t>(off, 1));
  }

  // M2L work split: partial slots per level so that every level gets enough
  // CTAs (small levels would otherwise run 189 terms in a single CTA)
  int nsplit[DMAX + 2] = {0};
  int64_t part_off[DMAX + 2] = {0};
  int job_start[DMAX + 3] = {0};
  void plan_m2l_split() {
    const int target_jobs = 4 * 148 * 2;
    int64_t off = 0;
    int jobs = 0;
    for (int l = 1; l <= depth; ++l) {
      const int tiles = 8 * tiles_per_parity(l);
      int ns = (target_jobs + tiles - 1) / tiles;
      ns = std::max(1, std::min(MAX_SPLIT, ns));
      nsplit[l] = ns;
      part_off[l] = off;
      off += (int64_t)ns << (3 * l);
      job_start[l] = jobs;
      jobs += tiles * ns;
    }
    job_start[depth + 1] = jobs;
    partial.ensure(tsz() * ncp * std::max<int64_t>(off, 1));
    if (use_halo) plan_halo_jobs();
    // M2M child split: 8 partial slots of the largest parent level
    const int64_t top = depth >= 1 ? (1LL << (3 * (depth - 1))) : 1;
    up_part.ensure(tsz() * ncp * 8 * top);
    const int64_t ncnt = (int64_t)tiles_all(std::max(depth - 1, 0)) * ((ncp + GB_M - 1) / GB_M) + 8;
    up_cnt.ensure(sizeof(int) * ncnt);
    LFMM_CUDA(cudaMemsetAsync(up_cnt.p, 0, up_cnt.bytes, stream));
  }
  GemmArgs gemm_base() const {
    GemmArgs ga{};
    ga.ncp = ncp;
    ga.depth = depth;
    ga.mult = mult.p;
    ga.loc = loc.p;
    ga.partial = partial.p;
    ga.ops_m2l = ops_m2l.p;
    ga.ops_m2m = ops_m2m.p;
    ga.ops_l2l = ops_l2l.p;
    ga.ops_lat = ops_lat.p;
    ga.up_split = 8;
    ga.up_part = up_part.p;
    ga.up_cnt = up_cnt.as<int>();
    for (int l = 0; l <= depth; ++l) {
      ga.level_off[l] = level_off[l];
      ga.part_off[l] = part_off[l];
      ga.nsplit[l] = nsplit[l];
    }
    for (int l = 0; l <= depth + 1; ++l) ga.job_start[l] = job_start[l];
    return ga;
  }

  // ----------------------------------------------------------- tree ----
  template <class T>
  void build_tree(const double* positions, bool on_device) {
    // host positions of a large system: uploaded in kPosChunks pieces on the
    // io stream, each piece wrapped and counted as soon as it lands (the
    // counting pass hides behind the rest of the upload)
    const bool chunked = !on_device && N >= (1 << 18) && !profiling;
    if (!on_device && !chunked)
      LFMM_CUDA(cudaMemcpyAsync(pos_in.p, positions, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, stream));
    LFMM_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int) * nleaf, stream));
    if (chunked) {
      if (!io_stream) LFMM_CUDA(cudaStreamCreateWithFlags(&io_stream, cudaStreamNonBlocking));
      for (auto& e : ev_pos)
        if (!e) LFMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      LFMM_CUDA(cudaEventRecord(ev_pos[0], stream));  // pos_in no longer read by earlier work
      LFMM_CUDA(cudaStreamWaitEvent(io_stream, ev_pos[0], 0));
      for (int c = 0; c < kPosChunks; ++c) {
        const int64_t i0 = N * c / kPosChunks, i1 = N * (c + 1) / kPosChunks;
        LFMM_CUDA(cudaMemcpyAsync(pos_in.as<double>() + 3 * i0, positions + 3 * i0, sizeof(double) * 3 * (i1 - i0),
                                  cudaMemcpyHostToDevice, io_stream));
        LFMM_CUDA(cudaEventRecord(ev_pos[c + 1], io_stream));
        LFMM_CUDA(cudaStreamWaitEvent(stream, ev_pos[c + 1], 0));
        launch(ST_TREE, [&] {
          k_wrap_cell<<<nblk(i1 - i0, 256), 256, 0, stream>>>(pos_in.as<double>() + 3 * i0, i1 - i0, L, size, depth,
                                                               leaf_of.as<int>() + i0, counts.as<int>(),
                                                               slot_of.as<int>() + i0, nullptr, key32.as<float>() + i0);
        });
      }
    } else if (N > 0) {
      launch(ST_TREE, [&] {
        k_wrap_cell<<<nblk(N, 256), 256, 0, stream>>>(on_device ? positions : pos_in.as<double>(), N, L, size, depth,
                                                       leaf_of.as<int>(), counts.as<int>(),
                                                       slot_of.as<int>(), on_device ? pos_in.as<double>() : nullptr,
                                                       key32.as<float>());
      });
    }
    if (nleaf >= SCAN_TILE) {
      const int sb = (int)((nleaf + SCAN_TILE - 1) / SCAN_TILE);
      scan_status.ensure(sizeof(unsigned long long) * sb);
      LFMM_CUDA(cudaMemsetAsync(scan_status.p, 0, sizeof(unsigned long long) * sb, stream));
      launch(ST_TREE, [&] {
        k_scan_lookback<<<sb, SCAN_THREADS, 0, stream>>>(counts.as<int>(), nleaf, leaf_start.as<int>(),
                                                         scan_status.as<unsigned long long>());
      });
    } else {
      launch(ST_TREE, [&] { k_scan_single<<<1, 1024, 0, stream>>>(counts.as<int>(), nleaf, leaf_start.as<int>()); });
    }
    if (N > 0) {
      launch(ST_TREE, [&] {
        k_scatter_leaf<<<nblk(N, 256), 256, 0, stream>>>(leaf_of.as<int>(), N, leaf_start.as<int>(),
                                                          slot_of.as<int>(), bucket.as<int>());
      });
      launch(ST_TREE, [&] {
        k_leaf_rank<T><<<nblk((int64_t)nleaf * 32, RANK_WARPS * 32), RANK_WARPS * 32, 0, stream>>>(
            pos_in.as<double>(), L, key32.as<float>(), leaf_start.as<int>(), bucket.as<int>(), nleaf, perm.as<int>(), inv_perm.as<int>(),
            depth, size, pos_sorted.as<double>(), xq.as<vec4_t<T>>(), leaf_sorted.as<int>(), pair_a(), pair_b());
      });
    }
    last_valid = false;
  }

  // ---------------------------------------------------------- solve ----
  // k_p2p2: ctas == 0 one warp per leaf; else persistent with that many CTAs
  // over the shared leaf counter p2p_ctl[0], stopped by *stop
  void p2p2_launch(bool grad, int periodic, int ctas, const int* stop, cudaStream_t st) {
    const unsigned grid = ctas > 0 ? (unsigned)ctas : nblk(own_leaves(), P2P2_WARPS);
    int* ctl = ctas > 0 ? p2p_ctl.as<int>() : nullptr;
    if (grad)
      k_p2p2<true><<<grid, P2P2_WARPS * 32, P2P2_SMEM, st>>>(reinterpret_cast<const float4*>(xq.p), pair_a(), pair_b(),
                                                            leaf_start.as<int>(), depth, (float)size, periodic,
                                                            vnear.as<float>(), gnear.as<float>(), own_x0, own_x1, ctl,
                                                            stop);
    else
      k_p2p2<false><<<grid, P2P2_WARPS * 32, P2P2_SMEM, st>>>(reinterpret_cast<const float4*>(xq.p), pair_a(), pair_b(),
                                                             leaf_start.as<int>(), depth, (float)size, periodic,
                                                             vnear.as<float>(), gnear.as<float>(), own_x0, own_x1, ctl,
                                                             stop);
  }
  // leaves of this rank's slab (all of them without a decomposition); the
  // leaf kernels start their grid at leaf plane own_x0
  int64_t own_leaves() const {
    return (int64_t)(std::min(own_x1, 1 << depth) - own_x0) << (2 * depth);
  }
  // parent columns of level pl this rank computes: its x-slab when a slab
  // decomposition owns the level (pl >= dist_lg), else the whole level
  void owned_parents(int pl, int& p0, int& pend) const {
    p0 = 0;
    pend = 1 << (3 * pl);
    if (dist_lg > 0 && pl >= dist_lg) {
      p0 = (own_x0 >> (depth - pl)) << (2 * pl);
      pend = (own_x1 >> (depth - pl)) << (2 * pl);
    }
  }
  template <class T>
  void solve_column(int K, int c, bool grad) {
    const int64_t nb = std::min<int64_t>(nblk(N, 256), 148 * 4);
    const T tsize = (T)size;
    T* M = mult.as<T>();
    T* Lc = loc.as<T>();
    const unsigned rowb = (unsigned)((ncp + GB_M - 1) / GB_M);
    GemmArgs ga = gemm_base();
    auto m2m_level = [&](int l) {
      if (use_tr) {
        TrArgs ta{};
        ta.mode = 0;
        ta.level = l;
        ta.ncp = ncp;
        ta.ops_t = ops_m2m_t.p;
        ta.src = M + level_off[l + 1] * ncp;
        ta.dst = M + level_off[l] * ncp;
        ta.slots = up_part.p;
        ta.cnt = tr_cnt.as<int>();
        owned_parents(l, ta.p0, ta.pend);
        launch(ST_M2M, [&] {
          if (use_tt)
            tt_launch(ta, ta.pend - ta.p0, tt_m2m.p, stream);
          else
            tr_launch<T>(ta, ta.pend - ta.p0, 8, stream);
        });
        return;
      }
      ga.mode = GEMM_UP;
      ga.level = l;
      dim3 grid(tiles_all(l) * ga.up_split, rowb);
      launch(ST_M2M, [&] { k_gemm_gather<T><<<grid, G_THREADS, 0, stream>>>(ga); });
    };
    const int periodic = (flags & LFMM_F_PERIODIC_NEAR) ? 1 : 0;
    const unsigned lb = nblk(own_leaves(), P2P_WARPS);
    const bool side = !profiling;
    if (side && !near_stream) {
      int lo = 0, hi = 0;
      LFMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      LFMM_CUDA(cudaStreamCreateWithPriority(&near_stream, cudaStreamNonBlocking, lo));
      LFMM_CUDA(cudaEventCreateWithFlags(&ev_near_in, cudaEventDisableTiming));
      LFMM_CUDA(cudaEventCreateWithFlags(&ev_near_out, cudaEventDisableTiming));
    }
    auto issue_p2p = [&]() {
    cudaStream_t pst = stream;
    if (side) {
      LFMM_CUDA(cudaEventRecord(ev_near_in, stream));
      LFMM_CUDA(cudaStreamWaitEvent(near_stream, ev_near_in, 0));
      pst = near_stream;
    }
    launch_on(ST_P2P, pst, [&] {
      cudaStream_t stream = pst;
      if (sizeof(T) == 4 && !p2p_scalar) {
        p2p2_launch(grad, periodic, 0, nullptr, stream);
        return;
      }
      if (grad)
        k_p2p<T, true><<<lb, P2P_WARPS * 32, 0, stream>>>(xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, tsize,
                                                           periodic, vnear.as<T>(), gnear.as<T>(), own_x0, own_x1);
      else
        k_p2p<T, false><<<lb, P2P_WARPS * 32, 0, stream>>>(xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, tsize,
                                                            periodic, vnear.as<T>(), gnear.as<T>(), own_x0, own_x1);
    });
    if (side) {
      LFMM_CUDA(cudaEventRecord(ev_near_out, near_stream));
      near_pending = true;
    }
    };
    // Preemptible near field (fp32, tensor-core M2L, single rank): launch 1
    // (p2p_c1 CTAs per SM) runs beside the P2M / M2M / lattice chain and is
    // stopped before the M2L takes every SM; launch 2 (p2p_c2 per SM) runs
    // beside the L2L chain and L2P; launch 3 (full occupancy, main stream)
    // finishes the leaves left.  Each leaf is computed by one warp with the
    // same arithmetic whichever launch takes it.
    const bool preempt = side && p2p_preempt && sizeof(T) == 4 && !p2p_scalar && use_halo && dist_phase == 0;
    int* ctl = p2p_ctl.as<int>();
    if (dist_phase == 2) {
      // levels spanning several ranks, from the gathered level dist_lg
      for (int l = std::min(dist_lg, depth) - 1; l >= 0; --l) m2m_level(l);
    } else {
    launch(ST_STAGE, [&] {
      k_stage_q<T><<<(unsigned)nb, 256, 0, stream>>>(q_in.as<double>(), K, c, perm.as<int>(), pos_sorted.as<double>(),
                                                     N, L, xq.as<vec4_t<T>>(), qs.as<double>(), part.as<dd>(),
                                                     counters.as<int>(), scal.as<double>(), leaf_sorted.as<int>(),
                                                     depth, own_x0, own_x1, leaf_start.as<int>(),
                                                     p2p_scalar ? nullptr : pair_b());
    });
    if (preempt) {
      LFMM_CUDA(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), stream));
      LFMM_CUDA(cudaEventRecord(ev_near_in, stream));
      LFMM_CUDA(cudaStreamWaitEvent(near_stream, ev_near_in, 0));
      // HI side work issued together with the solve (no tree build to hide
      // behind): let it finish before the near field holds the SMs, or its
      // large-smem kernels wait behind the M2L
      if (near_after_hi) LFMM_CUDA(cudaStreamWaitEvent(near_stream, ev_hi_out, 0));
      launch_on(ST_P2P, near_stream, [&] { p2p2_launch(grad, periodic, nsm * p2p_c1, ctl + 1, near_stream); });
    } else {
      issue_p2p();
    }
    launch(ST_P2M, [&] {
      if (p == 10) {
        k_p2m_c<T, 10><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
            xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, (T)(1.0 / size), ncp, M + level_off[depth] * ncp,
            own_x0);
        return;
      }
      k_p2m<T><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
          xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, p, (T)(1.0 / size), ncp, M + level_off[depth] * ncp,
          own_x0);
    });
    {
    {
      // single rank on the tensor cores: the small parent levels in one launch
      const bool chain = use_tt && dist_phase == 0 && dist_lg == 0 && sizeof(T) == 4;
      const int lo = dist_phase == 1 ? dist_lg : 0;
      for (int l = depth - 1; l >= lo; --l) {
        if (chain && l <= TT_CHAIN_TOP) {
          TtChain ch{};
          for (int k = l; k >= 0; --k) {
            TrArgs& ta = ch.lev[ch.nlev++];
            ta.mode = 0;
            ta.level = k;
            ta.ncp = ncp;
            ta.src = M + level_off[k + 1] * ncp;
            ta.dst = M + level_off[k] * ncp;
            ta.slots = up_part.p;
            ta.cnt = tr_cnt.as<int>();
            owned_parents(k, ta.p0, ta.pend);
          }
          ch.bar = tt_bar.as<unsigned>();
          launch(ST_M2M, [&] { tt_chain_launch(ch, tt_m2m.p, stream); });
          break;
        }
        m2m_level(l);
      }
    }
    launch(ST_M2M, [&] {
      k_box_charges<T><<<nblk(nleaf, 256), 256, 0, stream>>>(qs.as<double>(), leaf_start.as<int>(), depth,
                                                             level_off[depth], ncp, M, boxq.as<double>(),
                                                             counters.as<int>() + 2, 0);
    });
    }
    if (dist_phase == 1) {
      // owned multipoles ready for the exchange; the fp16 M2L's per-level
      // scale needs max |M| over the whole level, so each rank reduces its
      // own slab of the levels >= dist_lg here and the caller max-reduces
      // them across ranks (lfmm_dist_buffers [8])
      if (use_halo && sizeof(T) == 4 && dist_lg >= 1) {
        HaloArgs ha{};
        ha.inv_c = hm_inv_c.as<float>();
        for (int l = 0; l <= depth; ++l) ha.level_off[l] = level_off[l];
        const int l0 = std::max(dist_lg, 1);
        ha.lvl0 = l0;
        ha.own_x0 = own_x0;
        ha.own_x1 = own_x1;
        ha.own_depth = depth;
        LFMM_CUDA(cudaMemsetAsync(hm_level_max.p, 0, hm_level_max.bytes, stream));
        const int64_t nown = (int64_t)(own_x1 - own_x0) << (2 * depth);
        launch(ST_PACK, [&] {
          k_level_absmax<<<dim3((unsigned)std::max<int64_t>(1, (nown + 63) / 64), depth - l0 + 1), 256, 0, stream>>>(
              reinterpret_cast<const float*>(mult.p), ha, hm_level_max.as<unsigned int>());
        });
      }
      return;
    }
    }  // up
    if (lattice_mode != LFMM_LATTICE_OFF && use_tr) {
      TrArgs ta{};
      ta.mode = 2;
      ta.ncols = 1;
      ta.ncp = ncp;
      ta.ops_t = ops_lat_t.p;
      ta.src = M;
      ta.dst = Lc;
      launch(ST_ROOT, [&] { tr_launch<T>(ta, 1, 1, stream); });
    } else if (lattice_mode != LFMM_LATTICE_OFF) {
      ga.mode = GEMM_ROOT;
      ga.level = 0;
      dim3 grid(1, rowb);
      launch(ST_ROOT, [&] { k_gemm_gather<T><<<grid, G_THREADS, 0, stream>>>(ga); });
    } else {
      LFMM_CUDA(cudaMemsetAsync(Lc, 0, sizeof(T) * ncp, stream));
    }
    if (depth >= 1) {
      // M2L of every level in one launch (terms split over CTAs), then the
      // L2L sweep adds the partial slots level by level
      if (use_halo && sizeof(T) == 4) {
        HaloArgs ha{};
        ha.mult = reinterpret_cast<const float*>(mult.p);
        ha.partial = reinterpret_cast<float*>(partial.p);
        ha.ops16 = ops16.as<unsigned char>();
        ha.jobs = hm_jobs.as<int4>();
        ha.level_max = hm_level_max.as<unsigned int>();
        ha.inv_r = hm_inv_r.as<float>();
        ha.inv_c = hm_inv_c.as<float>();
        ha.rw_cap = hm_rw_cap;
        ha.stagger = hm_stagger;
        ha.lvl0 = 1;
        ha.mult16 = mult16.as<unsigned char>();
        for (int l = 0; l <= depth; ++l) {
          ha.level_off[l] = level_off[l];
          ha.part_off[l] = part_off[l];
          ha.m16_off[l] = m16_off[l];
        }
        if (dist_phase == 2 && dist_lg >= 1) {
          // levels >= dist_lg: max-reduced across ranks by the caller after
          // phase 1; the shared levels below are complete on every rank
          LFMM_CUDA(cudaMemsetAsync(hm_level_max.p, 0, sizeof(unsigned int) * dist_lg, stream));
          if (dist_lg >= 2)
            launch(ST_PACK, [&] {
              k_level_absmax<<<dim3((unsigned)std::max<int64_t>(1, ((1LL << (3 * (dist_lg - 1))) + 63) / 64),
                                    dist_lg - 1), 256, 0, stream>>>(ha.mult, ha, hm_level_max.as<unsigned int>());
            });
        } else {
          LFMM_CUDA(cudaMemsetAsync(hm_level_max.p, 0, hm_level_max.bytes, stream));
          launch(ST_PACK, [&] {
            k_level_absmax<<<dim3((unsigned)std::max<int64_t>(1, ((1LL << (3 * depth)) + 63) / 64), depth), 256, 0,
                             stream>>>(ha.mult, ha, hm_level_max.as<unsigned int>());
          });
        }
        launch(ST_PACK, [&] {
          // owned levels of a slab decomposition: padded class x-rows
          // [xl0/2, (xl1+1)/2 + 2) hold every source window of the owned
          // targets (class positions [ia, ib) of plan_halo_jobs, +-1 plane)
          int prows = 0;
          for (int l = 1; l <= depth; ++l) {
            const int Z = (1 << (l - 1)) + 2;
            ha.pk_r0[l] = 0;
            ha.pk_r1[l] = hm_plane_rows(l);
            if (dist_lg > 0 && l >= dist_lg) {
              const int xl0 = own_x0 >> (depth - l), xl1 = own_x1 >> (depth - l);
              ha.pk_r0[l] = (xl0 >> 1) * Z * Z;
              ha.pk_r1[l] = std::min(hm_plane_rows(l), (((xl1 + 1) >> 1) + 2) * Z * Z);
            }
            prows = std::max(prows, ha.pk_r1[l] - ha.pk_r0[l]);
          }
          k_pack_mult16<<<dim3((unsigned)((8 * prows + 255) / 256), depth, 8), 256, 0, stream>>>(ha);
        });
        if (preempt) LFMM_CUDA(cudaMemsetAsync(ctl + 1, 1, sizeof(int), stream));  // near field 1 yields the SMs
        launch(ST_DOWN, [&] {
          ha.counter = hm_counter.as<int>();
          launch_m2l_halo(ha, hm_njobs, nsm, hm_astages, stream);
        });
        if (preempt) {
          LFMM_CUDA(cudaEventRecord(ev_m2l_done, stream));
          LFMM_CUDA(cudaStreamWaitEvent(near_stream, ev_m2l_done, 0));
          launch_on(ST_P2P, near_stream, [&] { p2p2_launch(grad, periodic, nsm * p2p_c2, ctl + 2, near_stream); });
          LFMM_CUDA(cudaEventRecord(ev_near_out, near_stream));
          near_pending = true;
        }
      } else {
        ga.mode = GEMM_M2L;
        ga.level = 0;
        if (sizeof(T) == 8 && ncp == 128 && !m2l_f64_simt) {
          ga.ops_m2l_t = ops_m2l_t.p;
          launch(ST_DOWN, [&] { k_m2l_f64<<<ga.job_start[depth + 1], G_THREADS, F64_SMEM, stream>>>(ga); });
        } else {
          dim3 grid(ga.job_start[depth + 1], rowb);
          launch(ST_DOWN, [&] { k_gemm_gather<T><<<grid, G_THREADS, 0, stream>>>(ga); });
        }
      }
      const bool chain_dn = use_tt && dist_phase == 0 && dist_lg == 0 && sizeof(T) == 4;
      int l_first = 1;
      if (chain_dn) {  // child levels 1 .. TT_CHAIN_TOP + 1 in one launch
        TtChain ch{};
        for (int l = 1; l <= std::min(depth, TT_CHAIN_TOP + 1); ++l) {
          TrArgs& ta = ch.lev[ch.nlev++];
          ta.mode = 1;
          ta.level = l;
          ta.ncp = ncp;
          ta.src = Lc + level_off[l - 1] * ncp;
          ta.dst = Lc + level_off[l] * ncp;
          ta.partial = static_cast<const char*>(partial.p) + tsz() * (size_t)part_off[l] * ncp;
          ta.nsplit = nsplit[l];
          owned_parents(l - 1, ta.p0, ta.pend);
          l_first = l + 1;
        }
        ch.bar = tt_bar.as<unsigned>();
        launch(ST_L2L, [&] { tt_chain_launch(ch, tt_l2l.p, stream); });
      }
      for (int l = l_first; l <= depth; ++l) {
        if (use_tr) {
          TrArgs ta{};
          ta.mode = 1;
          ta.level = l;
          ta.ncp = ncp;
          ta.ops_t = ops_l2l_t.p;
          ta.src = Lc + level_off[l - 1] * ncp;
          ta.dst = Lc + level_off[l] * ncp;
          ta.partial = static_cast<const char*>(partial.p) + tsz() * (size_t)part_off[l] * ncp;
          ta.nsplit = nsplit[l];
          owned_parents(l - 1, ta.p0, ta.pend);
          launch(ST_L2L, [&] {
            if (use_tt)
              tt_launch(ta, ta.pend - ta.p0, tt_l2l.p, stream);
            else
              tr_launch<T>(ta, ta.pend - ta.p0, 8, stream);
          });
          continue;
        }
        ga.mode = GEMM_L2L;
        ga.level = l;
        dim3 g2(8 * tiles_per_parity(l), rowb);
        launch(ST_L2L, [&] { k_gemm_gather<T><<<g2, G_THREADS, 0, stream>>>(ga); });
      }
    }
    {
      const int per_warp = ncoef(p) + 3 * p * p;
      int warps = EXP_WARPS;
      while (warps > 1 && (size_t)warps * per_warp * sizeof(T) > 48 * 1024) warps >>= 1;
      const size_t smem = (size_t)warps * per_warp * sizeof(T);
      launch(ST_L2P, [&] {
        if (p == 10 && sizeof(T) == 4) {
          if (grad)
            k_l2p_f2<true, 10><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
                reinterpret_cast<const float4*>(xq.p), leaf_start.as<int>(), depth, (float)size, ncp,
                reinterpret_cast<const float*>(Lc + level_off[depth] * ncp), vfar.as<float>(), gfar.as<float>(), own_x0, own_x1);
          else
            k_l2p_f2<false, 10><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
                reinterpret_cast<const float4*>(xq.p), leaf_start.as<int>(), depth, (float)size, ncp,
                reinterpret_cast<const float*>(Lc + level_off[depth] * ncp), vfar.as<float>(), gfar.as<float>(), own_x0, own_x1);
          return;
        }
        if (p == 10) {
          if (grad)
            k_l2p_c<T, true, 10><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
                xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, tsize, ncp, Lc + level_off[depth] * ncp,
                vfar.as<T>(), gfar.as<T>(), own_x0, own_x1);
          else
            k_l2p_c<T, false, 10><<<nblk(own_leaves(), EXP_WARPS), EXP_WARPS * 32, 0, stream>>>(
                xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, tsize, ncp, Lc + level_off[depth] * ncp,
                vfar.as<T>(), gfar.as<T>(), own_x0, own_x1);
          return;
        }
        if (grad)
          k_l2p<T, true><<<nblk(own_leaves(), warps), warps * 32, smem, stream>>>(
              xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, p, tsize, ncp, Lc + level_off[depth] * ncp,
              vfar.as<T>(), gfar.as<T>(), own_x0, own_x1);
        else
          k_l2p<T, false><<<nblk(own_leaves(), warps), warps * 32, smem, stream>>>(
              xq.as<vec4_t<T>>(), leaf_start.as<int>(), depth, p, tsize, ncp, Lc + level_off[depth] * ncp,
              vfar.as<T>(), gfar.as<T>(), own_x0, own_x1);
      });
    }
    const int dip = (flags & LFMM_F_DIPOLE) ? 1 : 0;
    if (preempt) {  // the remaining leaves at full occupancy
      LFMM_CUDA(cudaMemsetAsync(ctl + 2, 1, sizeof(int), stream));
      launch(ST_P2P, [&] { p2p2_launch(grad, periodic, nsm * 6, ctl + 3, stream); });
    }
    if (near_pending) {  // near field done
      LFMM_CUDA(cudaStreamWaitEvent(stream, ev_near_out, 0));
      near_pending = false;
    }
    launch(ST_FINAL, [&] {
      if (grad)
        k_finalize<T, true><<<(unsigned)nb, 256, 0, stream>>>(
            N, K, c, perm.as<int>(), pos_sorted.as<double>(), qs.as<double>(), vnear.as<T>(), vfar.as<T>(),
            gnear.as<T>(), gfar.as<T>(), scal.as<double>(), dip, L, step_mode ? nullptr : out_pot.as<double>(),
            step_mode ? nullptr : out_near.as<double>(), step_mode ? nullptr : out_far.as<double>(),
            step_mode ? nullptr : out_dip.as<double>(), out_forces.as<double>(), part.as<dd>(), counters.as<int>() + 1,
            epart.as<double>(), energies.as<double>(), dvec.as<double>(), qtot.as<double>(),
            leaf_sorted.as<int>(), depth, own_x0, own_x1);
      else
        k_finalize<T, false><<<(unsigned)nb, 256, 0, stream>>>(
            N, K, c, perm.as<int>(), pos_sorted.as<double>(), qs.as<double>(), vnear.as<T>(), vfar.as<T>(),
            gnear.as<T>(), gfar.as<T>(), scal.as<double>(), dip, L, out_pot.as<double>(), out_near.as<double>(),
            out_far.as<double>(), out_dip.as<double>(), nullptr, part.as<dd>(), counters.as<int>() + 1,
            epart.as<double>(), energies.as<double>(), dvec.as<double>(), qtot.as<double>(),
            leaf_sorted.as<int>(), depth, own_x0, own_x1);
    });
  }

  void ensure_solve_buffers(int64_t K, bool grad) {
    const size_t t = tsz();
    q_in.ensure(sizeof(double) * N * K + 8);
    qs.ensure(sizeof(double) * N + 8);
    vnear.ensure(t * N + 16);
    vfar.ensure(t * N + 16);
    if (grad) {
      gnear.ensure(t * 3 * N + 16);
      gfar.ensure(t * 3 * N + 16);
      out_forces.ensure(sizeof(double) * 3 * N + 8);
    }
    part.ensure(sizeof(dd) * 4 * (nblk(N, 256) + 1));
    out_pot.ensure(sizeof(double) * N * K + 8);
    out_near.ensure(sizeof(double) * N * K + 8);
    out_far.ensure(sizeof(double) * N * K + 8);
    out_dip.ensure(sizeof(double) * N * K + 8);
    energies.ensure(sizeof(double) * 4 * K);
    dvec.ensure(sizeof(double) * 3 * K);
    qtot.ensure(sizeof(double) * K);
  }

  void run_solve(int64_t K, bool grad) {
    roots.ensure(tsz() * ncp * K);
    for (int64_t c = 0; c < K; ++c) {
      if (fp32)
        solve_column<float>((int)K, (int)c, grad);
      else
        solve_column<double>((int)K, (int)c, grad);
      // keep this column's root multipole (level 0 of the upward pass)
      LFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(roots.p) + tsz() * ncp * c, mult.p, tsz() * ncp,
                                cudaMemcpyDeviceToDevice, stream));
    }
    last_k = K;
    last_valid = true;
  }

  void root_multipole_host(int64_t K, int64_t c, double* out /* nc x K complex interleaved */) {
    // leaf-level normalisation: M_l = M^_l * L^l at the root (edge L)
    std::vector<double> hv(ncp);
    const char* src = static_cast<const char*>(roots.p) + tsz() * ncp * c;
    if (fp32) {
      std::vector<float> hf(ncp);
      LFMM_CUDA(cudaMemcpyAsync(hf.data(), src, sizeof(float) * ncp, cudaMemcpyDeviceToHost, stream));
      LFMM_CUDA(cudaStreamSynchronize(stream));
      for (int i = 0; i < ncp; ++i) hv[i] = hf[i];
    } else {
      LFMM_CUDA(cudaMemcpyAsync(hv.data(), src, sizeof(double) * ncp, cudaMemcpyDeviceToHost, stream));
      LFMM_CUDA(cudaStreamSynchronize(stream));
    }
    for (int l = 0; l <= p; ++l) {
      const double sc = std::pow(L, l);
      for (int m = -l; m <= l; ++m) {
        double re, im;
        const int mm = std::abs(m);
        if (mm == 0) {
          re = hv[pk_index(p, l, 0, 0)];
          im = 0.0;
        } else {
          re = hv[pk_index(p, l, mm, 0)];
          im = hv[pk_index(p, l, mm, 1)];
          if (m < 0) {
            const double s = (mm & 1) ? -1.0 : 1.0;
            re *= s;
            im *= -s;
          }
        }
        const size_t o = ((size_t)cidx(l, m) * K + c) * 2;
        out[o] = re * sc;
        out[o + 1] = im * sc;
      }
    }
  }
};

namespace {

int fail(const Error& e) {
  g_last_error = e.msg;
  return e.code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LFMM_OK;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error{LFMM_ECUDA, e.what()});
  }
}

void copy_out(lfmm_plan* pl, double* dst, const DevBuf& src, size_t bytes, int on_device) {
  if (!dst) return;
  LFMM_CUDA(cudaMemcpyAsync(dst, src.p, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            pl->stream));
}

// NumericalFailure (status 3, the reference CLI's _require_finite /
// NumericalFailure, cli.py:24-25, :107-112): the host copies of the energies
// and lambda forces are scanned after the call's final synchronisation
// (device-resident outputs are left to the caller: no extra host sync).
void require_finite(const double* v, int64_t n, const char* what) {
  if (!v) return;
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) throw Error{LFMM_ENONFINITE, std::string("non-finite values in ") + what};
}

void hi_args(lfmm_plan* pl, HiArgs& g) {
  g.n_sites = (int)pl->n_sites;
  g.atom_off = pl->atom_off.as<int>();
  g.atom_idx = pl->atom_idx.as<int>();
  g.nforms = pl->nforms.as<int>();
  g.form_off = pl->form_off.as<int>();
  g.fslot_off = pl->fslot_off.as<int>();
  g.form_q = pl->form_q.as<double>();
  g.lambdas = pl->lambdas.as<double>();
  g.nlam = pl->nlam.as<int>();
  g.site_pos = pl->site_pos.as<double>();
  g.box = pl->L;
  g.p = pl->p;
  g.ncp = pl->ncp;
  g.lat_t = pl->lattice_mode != LFMM_LATTICE_OFF ? pl->lat64t.as<double>() : nullptr;
  g.rscratch = pl->rscr.as<double>();
  g.uscratch = pl->uscr.as<double>();
  g.images_full = (pl->flags & LFMM_F_INTRA_MINIMUM) ? 0 : 1;
  g.dipole = (pl->flags & LFMM_F_DIPOLE) ? 1 : 0;
}

void upload_lambdas(lfmm_plan* pl, const double* lambdas, const int32_t* n_lambda, int on_device) {
  const size_t S = (size_t)pl->n_sites;
  if (S == 0) return;
  LFMM_REQUIRE(lambdas && n_lambda, "lambdas and n_lambda are required");
  if (!on_device) {
    for (size_t s = 0; s < S; ++s) {
      const int nl = n_lambda[s];
      LFMM_REQUIRE(nl >= 1 && nl <= 4, "need between 1 and 4 lambda values per site");
      LFMM_REQUIRE((1 << nl) == pl->h_nforms[s], std::to_string(nl) + " lambdas give " + std::to_string(1 << nl) +
                                                      " weights, site has " + std::to_string(pl->h_nforms[s]) +
                                                      " forms");
    }
  }
  const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  LFMM_CUDA(cudaMemcpyAsync(pl->lambdas.p, lambdas, sizeof(double) * 4 * S, kind, pl->stream));
  LFMM_CUDA(cudaMemcpyAsync(pl->nlam.p, n_lambda, sizeof(int32_t) * S, kind, pl->stream));
}

void run_hi(lfmm_plan* pl, int mode, const double* pot_dev, const double* pot_site = nullptr, double* gram = nullptr) {
  if (pl->n_sites == 0) {
    LFMM_CUDA(cudaMemsetAsync(pl->offset_total.p, 0, sizeof(double), pl->stream));
    return;
  }
  HiArgs g{};
  hi_args(pl, g);
  g.pot = pot_dev;
  g.pot_site = pot_site;
  g.mode = mode;
  g.c_p2p = pl->c_p2p.as<double>();
  g.c_lat = pl->c_lat.as<double>();
  g.c_dip = pl->c_dip.as<double>();
  g.blend = pl->blend.as<double>();
  g.forces = pl->lam_forces.as<double>();
  g.offset = pl->offsets.as<double>();
  g.gram = gram;
  g.site_force = mode == LFMM_MODE_HI ? pl->site_force.as<double>() : nullptr;
  pl->site_force_valid = mode == LFMM_MODE_HI;
  if (mode == LFMM_MODE_HI && g.images_full && g.lat_t) {
    // lattice pair kernel inputs for all site atoms at once: R_t, U_t = T1 R_t
    const int na = (int)pl->n_site_atoms;
    pl->launch(ST_HI, [&] {
      const int apb = std::max(1, 128 / (g.p + 1));
      k_hi_rvec<<<(unsigned)((na + apb - 1) / apb), apb * (g.p + 1), sizeof(double) * apb * g.ncp, pl->stream>>>(
          g.site_pos, na, g.box, g.p, g.ncp, g.rscratch);
    });
    if (g.ncp == 128) {
      TrArgs ta{};
      ta.mode = 2;
      ta.ncols = na;
      ta.ncp = g.ncp;
      ta.ops_t = g.lat_t;
      ta.src = g.rscratch;
      ta.dst = g.uscratch;
      static std::once_flag attr_once;  // process-wide function attribute
      std::call_once(attr_once, [&] {
        tr_set_attrs<double>(g.ncp);
        LFMM_CUDA(cudaFuncSetAttribute(k_cols_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F64_SMEM));
      });
      if (pl->m2l_f64_simt)  // LFMM_M2L64=gather: the SIMT translate kernel here too
        pl->launch(ST_HI, [&] { tr_launch<double>(ta, na, 1, pl->stream); });
      else
        pl->launch(ST_HI, [&] {
          k_cols_f64<<<(unsigned)((na + GB_N - 1) / GB_N), G_THREADS, F64_SMEM, pl->stream>>>(
              g.lat_t, g.rscratch, g.uscratch, na);
        });
    } else {
      pl->launch(ST_HI, [&] {
        k_hi_umat<<<nblk((int64_t)na * g.ncp, 128), 128, 0, pl->stream>>>(g.lat_t, g.rscratch, na, ncoef(g.p), g.ncp,
                                                                          g.uscratch);
      });
    }
  }
  const int ns = pl->ns_max;
  const bool lat_smem = mode == LFMM_MODE_HI && g.images_full && g.lat_t;
  const size_t smem = sizeof(double) * ((size_t)ns + 3 * (size_t)ns * ns + 3 * (size_t)ns +
                                        (lat_smem ? 2 * (size_t)ns * (g.ncp + 1) : 0));
  if (smem > 48 * 1024) {  // raise only (process-wide attribute, see halo_smem_attr)
    static std::mutex mu;
    static size_t cur = 48 * 1024;
    std::lock_guard<std::mutex> lk(mu);
    if (smem > cur) {
      LFMM_CUDA(cudaFuncSetAttribute(k_hi_site, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cur = smem;
    }
  }
  pl->launch(ST_HI, [&] { k_hi_site<<<(unsigned)pl->n_sites, HI_THREADS, smem, pl->stream>>>(g); });
  pl->launch(ST_HI, [&] {
    k_sum_offsets<<<1, 256, 0, pl->stream>>>(pl->offsets.as<double>(), (int)pl->n_sites,
                                             pl->offset_total.as<double>());
  });
}

void add_site_forces(lfmm_plan* pl) {
  if (pl->n_site_atoms == 0) return;
  pl->launch(ST_HI, [&] {
    k_add_site_forces<<<nblk(3 * pl->n_site_atoms, 128), 128, 0, pl->stream>>>(
        pl->out_forces.as<double>(), pl->atom_idx.as<int>(), (int)pl->n_site_atoms, pl->site_force.as<double>());
  });
}

void gather_site_positions(lfmm_plan* pl, const double* site_positions, int on_device) {
  if (pl->n_site_atoms == 0) return;
  if (site_positions) {
    LFMM_CUDA(cudaMemcpyAsync(pl->site_pos.p, site_positions, sizeof(double) * 3 * pl->n_site_atoms,
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, pl->stream));
  } else {
    pl->launch(ST_HI, [&] {
      k_gather_site_pos<<<nblk(pl->n_site_atoms, 128), 128, 0, pl->stream>>>(
          pl->pos_in.as<double>(), pl->atom_idx.as<int>(), (int)pl->n_site_atoms, pl->site_pos.as<double>());
    });
  }
}

void blend_sites(lfmm_plan* pl, double* out_dev) {
  if (pl->n_sites == 0) return;
  HiArgs g{};
  hi_args(pl, g);
  pl->launch(ST_SCALE, [&] { k_blend_sites<<<(unsigned)pl->n_sites, 32, 0, pl->stream>>>(g, out_dev); });
}
void run_scale(lfmm_plan* pl, const double* q_dev, double* out_dev) {
  pl->launch(ST_SCALE, [&] { k_scale_charges<<<nblk(pl->N, 256), 256, 0, pl->stream>>>(q_dev, pl->N, out_dev); });
  blend_sites(pl, out_dev);
}

}  // namespace

// ============================================================ C-ABI ====
extern "C" {

const char* lfmm_version(void) { return "lfmm-b200 0.1.0 sm_100a"; }

#ifdef LFMM_HM_PROF
// profiling build only (tools/step_trace.py): trace the launches of the next
// calls on every stream; lfmm_debug_trace_read returns (stage, start ms, end
// ms) per launch relative to the first traced launch
int lfmm_debug_trace(lfmm_plan* plan, int enable) {
  return guarded([&] {
    plan->tracing = enable != 0;
    for (auto& e : plan->trace) {
      plan->free_events.push_back(e.a);
      plan->free_events.push_back(e.b);
    }
    plan->trace.clear();
  });
}
int64_t lfmm_debug_trace_read(lfmm_plan* plan, double* out, int64_t n) {
  int64_t k = 0;
  LFMM_CUDA(cudaDeviceSynchronize());
  if (plan->trace.empty()) return 0;
  cudaEvent_t base = plan->trace.front().a;
  float t0 = 0.f;
  for (auto& e : plan->trace) {  // earliest start (streams may reorder)
    float ms = 0.f;
    cudaEventElapsedTime(&ms, base, e.a);
    t0 = std::min(t0, ms);
  }
  for (auto& e : plan->trace) {
    if (k >= n) break;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, base, e.a);
    cudaEventElapsedTime(&b, base, e.b);
    out[3 * k] = e.stage;
    out[3 * k + 1] = a - t0;
    out[3 * k + 2] = b - t0;
    ++k;
  }
  return k;
}
// profiling build only: copy the per-CTA M2L timing records (tools/hm_prof.py)
int lfmm_debug_hm_prof(unsigned long long* out, int64_t n) {
  return guarded([&] {
    LFMM_CUDA(cudaDeviceSynchronize());
    LFMM_CUDA(cudaMemcpyFromSymbol(out, g_hm_prof, sizeof(unsigned long long) * 8 * std::min<int64_t>(n, 8192)));
  });
}
#endif

int lfmm_last_error(char* buf, int64_t len) {
  if (!buf || len <= 0) return LFMM_EINVAL;
  std::strncpy(buf, g_last_error.c_str(), (size_t)len - 1);
  buf[len - 1] = '\0';
  return LFMM_OK;
}

int lfmm_plan_create(const double* positions, int64_t n, double box_length, int p, int depth, int lattice_mode,
                     int shell_cap, int flags, lfmm_plan** out) {
  if (!out) return fail(Error{LFMM_EINVAL, "out is NULL"});
  *out = nullptr;
  std::unique_ptr<lfmm_plan> pl(new lfmm_plan());
  int rc = guarded([&] {
    // SolverConfig.validated (solver.py:60-75)
    LFMM_REQUIRE(p >= 1 && p <= PMAX, "expansion order p=" + std::to_string(p) + " outside [1, 40]");
    LFMM_REQUIRE(depth >= 0 && depth <= DMAX, "tree depth " + std::to_string(depth) + " outside [0, 6]");
    LFMM_REQUIRE(lattice_mode >= 0 && lattice_mode <= 2, "unknown lattice_mode");
    LFMM_REQUIRE(lattice_mode != LFMM_LATTICE_SHELLS || shell_cap >= 2, "shells mode needs shell_cap >= 2");
    LFMM_REQUIRE((flags & LFMM_F_PERIODIC_NEAR) || (depth == 0 && lattice_mode == LFMM_LATTICE_OFF),
                 "periodic_near=False requires depth=0 and lattice_mode='off'");
    LFMM_REQUIRE(box_length > 0 && std::isfinite(box_length), "box_length must be positive");
    LFMM_REQUIRE(n >= 0 && n < (1LL << 31), "particle count out of range");
    LFMM_REQUIRE(n == 0 || positions, "positions is NULL");
    for (int64_t i = 0; i < 3 * n; ++i)
      LFMM_REQUIRE(std::isfinite(positions[i]), "positions contain non-finite values");
    int dev = 0;
    LFMM_CUDA(cudaGetDevice(&dev));
    LFMM_CUDA(cudaDeviceGetAttribute(&pl->nsm, cudaDevAttrMultiProcessorCount, dev));
    std::call_once(g_const_once, init_constants);
    pl->N = n;
    pl->L = box_length;
    pl->p = p;
    pl->depth = depth;
    pl->lattice_mode = lattice_mode;
    pl->shell_cap = shell_cap;
    pl->flags = flags;
    pl->fp32 = (flags & LFMM_F_FP32) != 0;
    pl->nc = ncoef(p);
    pl->ncp = ncpad(p);
    {
      // A/B switches, each exercised by tests/test_gpu_variants.py:
      //   LFMM_M2L=simt    fp32 M2L on the SIMT gather kernel (no tensor cores)
      //   LFMM_P2P=scalar  fp32 P2P on the scalar kernel k_p2p
      //   LFMM_P2P=plain   fp32 near field in one launch on the side stream
      //                    (not the preemptible three-launch schedule)
      //   LFMM_M2L64=gather fp64 M2L on the SIMT gather kernel (no DMMA)
      //   LFMM_TRANSLATE=simt fp32 M2M / L2L on the SIMT kernel k_translate
      auto env_is = [](const char* name, const char* val) {
        const char* e = std::getenv(name);
        return e && std::string(e) == val;
      };
      pl->use_halo = pl->fp32 && depth >= 1 && pl->nc > 64 && pl->nc <= 128 && !env_is("LFMM_M2L", "simt");
      if (pl->use_halo) pl->ncp = 128;
      pl->p2p_scalar = env_is("LFMM_P2P", "scalar");
      pl->p2p_preempt = !env_is("LFMM_P2P", "plain");
      pl->graphs = !env_is("LFMM_GRAPH", "0");
      pl->m2l_f64_simt = env_is("LFMM_M2L64", "gather");
      pl->tt_simt = env_is("LFMM_TRANSLATE", "simt");
    }
    pl->nleaf = 1 << (3 * depth);
    pl->size = box_length / double(1 << depth);
    LFMM_CUDA(cudaStreamCreateWithFlags(&pl->own_stream, cudaStreamNonBlocking));
    pl->stream = pl->own_stream;
    int64_t off = 0;
    for (int l = 0; l <= depth; ++l) {
      pl->level_off[l] = off;
      off += 1LL << (3 * l);
    }
    pl->nbox_total = off;
    const size_t t = pl->tsz();
    const int64_t nn = std::max<int64_t>(n, 1);
    pl->pos_in.ensure(sizeof(double) * 3 * nn);
    pl->key32.ensure(sizeof(float) * nn);
    pl->leaf_of.ensure(sizeof(int) * nn);
    pl->slot_of.ensure(sizeof(int) * nn);
    pl->counts.ensure(sizeof(int) * pl->nleaf);
    pl->cursor.ensure(sizeof(int) * (pl->nleaf + pl->nleaf / 1024 + 2));
    pl->leaf_start.ensure(sizeof(int) * (pl->nleaf + 1));
    pl->bucket.ensure(sizeof(int) * nn);
    pl->perm.ensure(sizeof(int) * nn);
    pl->inv_perm.ensure(sizeof(int) * nn);
    pl->pos_sorted.ensure(sizeof(double) * 3 * nn);
    pl->leaf_sorted.ensure(sizeof(int) * nn);
    pl->xq.ensure(4 * t * nn);
    pl->ensure_pairs(nn);
    pl->mult.ensure(t * pl->ncp * off);
    pl->boxq.ensure(sizeof(double) * off);
    pl->loc.ensure(t * pl->ncp * off);
    LFMM_CUDA(cudaMemsetAsync(pl->mult.p, 0, pl->mult.bytes, pl->stream));
    LFMM_CUDA(cudaMemsetAsync(pl->loc.p, 0, pl->loc.bytes, pl->stream));
    pl->plan_m2l_split();
    pl->scal.ensure(sizeof(double) * 8);
    pl->counters.ensure(sizeof(int) * 16);
    LFMM_CUDA(cudaMemsetAsync(pl->counters.p, 0, pl->counters.bytes, pl->stream));
    pl->epart.ensure(sizeof(double) * 4);
    pl->offset_total.ensure(sizeof(double));
    if (pl->fp32)
      pl->build_operators<float>();
    else
      pl->build_operators<double>();
    if (pl->fp32)
      pl->build_tree<float>(positions, false);
    else
      pl->build_tree<double>(positions, false);
    LFMM_CUDA(cudaStreamSynchronize(pl->stream));
  });
  if (rc != LFMM_OK) return rc;
  *out = pl.release();
  return LFMM_OK;
}

int lfmm_plan_destroy(lfmm_plan* plan) {
  delete plan;
  return LFMM_OK;
}

int lfmm_plan_set_stream(lfmm_plan* plan, void* stream) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_CUDA(cudaStreamSynchronize(plan->stream));
    plan->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : plan->own_stream;
  });
}

int lfmm_plan_set_positions(lfmm_plan* plan, const double* positions, int on_device) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(plan->N == 0 || positions, "positions is NULL");
    if (plan->fp32)
      plan->build_tree<float>(positions, on_device != 0);
    else
      plan->build_tree<double>(positions, on_device != 0);
  });
}

int lfmm_plan_info(const lfmm_plan* plan, int64_t* out6) {
  if (!plan || !out6) return fail(Error{LFMM_EINVAL, "NULL argument"});
  out6[0] = plan->N;
  out6[1] = plan->p;
  out6[2] = plan->depth;
  out6[3] = plan->nc;
  out6[4] = plan->nleaf;
  out6[5] = plan->flags;
  return LFMM_OK;
}

int lfmm_export_tree(const lfmm_plan* cplan, int64_t* perm, int64_t* inv_perm, int64_t* leaf_of_particle,
                     int64_t* leaf_start, double* positions_sorted) {
  if (!cplan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  lfmm_plan* plan = const_cast<lfmm_plan*>(cplan);
  return guarded([&] {
    DevBuf tmp;
    const int64_t n = plan->N;
    tmp.ensure(sizeof(int64_t) * (std::max<int64_t>(n, plan->nleaf + 1) + 1));
    auto conv = [&](const DevBuf& src, int64_t cnt, int64_t* dst) {
      if (!dst || cnt == 0) return;
      k_i32_to_i64<<<nblk(cnt, 256), 256, 0, plan->stream>>>(src.as<int>(), cnt, tmp.as<int64_t>());
      LFMM_CUDA(cudaGetLastError());
      LFMM_CUDA(cudaMemcpyAsync(dst, tmp.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, plan->stream));
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
    };
    conv(plan->perm, n, perm);
    conv(plan->inv_perm, n, inv_perm);
    conv(plan->leaf_sorted, n, leaf_of_particle);
    conv(plan->leaf_start, plan->nleaf + 1, leaf_start);
    if (positions_sorted && n > 0) {
      LFMM_CUDA(cudaMemcpyAsync(positions_sorted, plan->pos_sorted.p, sizeof(double) * 3 * n,
                                cudaMemcpyDeviceToHost, plan->stream));
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
    }
    tmp.release();
  });
}

int lfmm_export_lists(const lfmm_plan* cplan, int level, int64_t* nb_box, int64_t* nb_shift, int64_t* m2l_src,
                      int64_t* m2l_row) {
  if (!cplan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  lfmm_plan* plan = const_cast<lfmm_plan*>(cplan);
  return guarded([&] {
    LFMM_REQUIRE(level >= 0 && level <= plan->depth, "level out of range");
    DevBuf a, b;
    if (nb_box || nb_shift) {
      const int64_t cnt = (int64_t)plan->nleaf * 27;
      a.ensure(sizeof(int64_t) * cnt);
      b.ensure(sizeof(int64_t) * cnt * 3);
      k_export_nb<<<nblk(cnt, 256), 256, 0, plan->stream>>>(plan->depth, a.as<int64_t>(), b.as<int64_t>());
      LFMM_CUDA(cudaGetLastError());
      if (nb_box)
        LFMM_CUDA(cudaMemcpyAsync(nb_box, a.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, plan->stream));
      if (nb_shift)
        LFMM_CUDA(cudaMemcpyAsync(nb_shift, b.p, sizeof(int64_t) * cnt * 3, cudaMemcpyDeviceToHost, plan->stream));
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
    }
    if ((m2l_src || m2l_row) && level >= 1) {
      const int64_t cnt = (1LL << (3 * level)) * NM2L;
      a.ensure(sizeof(int64_t) * cnt);
      b.ensure(sizeof(int64_t) * cnt);
      k_export_m2l<<<nblk(cnt, 256), 256, 0, plan->stream>>>(level, a.as<int64_t>(), b.as<int64_t>());
      LFMM_CUDA(cudaGetLastError());
      if (m2l_src)
        LFMM_CUDA(cudaMemcpyAsync(m2l_src, a.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, plan->stream));
      if (m2l_row)
        LFMM_CUDA(cudaMemcpyAsync(m2l_row, b.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, plan->stream));
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
    }
    a.release();
    b.release();
  });
}

int lfmm_lattice_matrix(const lfmm_plan* plan, double* out) {
  if (!plan || !out) return fail(Error{LFMM_EINVAL, "NULL argument"});
  if (plan->lattice_mode == LFMM_LATTICE_OFF) return fail(Error{LFMM_EINVAL, "lattice is off"});
  const int nc = plan->nc;
  // T_L = diag(L^-(n+1)) T_1 diag(L^-j)   (lattice.py:95-100)
  for (int r = 0; r < nc; ++r) {
    const int lr = (int)std::sqrt((double)r);
    const double sr = std::pow(plan->L, -(lr + 1.0));
    for (int c = 0; c < nc; ++c) {
      const int lc = (int)std::sqrt((double)c);
      const double sc = std::pow(plan->L, -(double)lc);
      const double2 v = plan->lat_unit[(size_t)r * nc + c];
      out[2 * ((size_t)r * nc + c)] = sr * v.x * sc;
      out[2 * ((size_t)r * nc + c) + 1] = sr * v.y * sc;
    }
  }
  return LFMM_OK;
}

int lfmm_solve(lfmm_plan* plan, const double* charges, int64_t k, int io_on_device, double* potentials,
               double* near_pot, double* far_pot, double* dip_pot, double* energies, double* root_multipole,
               double* dipole_vector, double* total_charge, double* forces) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(k >= 1, "need at least one charge column");
    LFMM_REQUIRE(!forces || k == 1, "forces need a single charge column");
    LFMM_REQUIRE(plan->N == 0 || charges, "charges is NULL");
    const int64_t N = plan->N;
    const bool grad = forces != nullptr;
    plan->ensure_solve_buffers(k, grad);
    if (N > 0)
      LFMM_CUDA(cudaMemcpyAsync(plan->q_in.p, charges, sizeof(double) * N * k,
                                io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, plan->stream));
    plan->run_solve(k, grad);
    const size_t nk = sizeof(double) * N * k;
    copy_out(plan, potentials, plan->out_pot, nk, io_on_device);
    copy_out(plan, near_pot, plan->out_near, nk, io_on_device);
    copy_out(plan, far_pot, plan->out_far, nk, io_on_device);
    copy_out(plan, dip_pot, plan->out_dip, nk, io_on_device);
    copy_out(plan, energies, plan->energies, sizeof(double) * 4 * k, io_on_device);
    copy_out(plan, dipole_vector, plan->dvec, sizeof(double) * 3 * k, io_on_device);
    copy_out(plan, total_charge, plan->qtot, sizeof(double) * k, io_on_device);
    if (grad) copy_out(plan, forces, plan->out_forces, sizeof(double) * 3 * N, io_on_device);
    if (root_multipole) {
      LFMM_REQUIRE(!io_on_device, "root_multipole is returned to host memory only");
      for (int64_t c = 0; c < k; ++c) plan->root_multipole_host(k, c, root_multipole);
    }
    if (!io_on_device) {
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
      require_finite(energies, 4 * k, "the solve energies");
    }
  });
}

int lfmm_sites_set(lfmm_plan* plan, int64_t n_sites, const int64_t* atom_offsets, const int64_t* atom_index,
                   const int32_t* n_forms, const int64_t* form_offsets, const double* form_charges) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(n_sites >= 0, "n_sites < 0");
    const int64_t S = n_sites;
    std::vector<int> aoff(S + 1), aidx, nf(S), foff(S + 1), fsl(S + 1);
    int ns_max = 0;
    for (int64_t s = 0; s <= S; ++s) {
      aoff[s] = (int)atom_offsets[s];
      foff[s] = (int)form_offsets[s];
    }
    const int64_t A = atom_offsets[S];
    aidx.resize(A);
    for (int64_t a = 0; a < A; ++a) {
      // -1 marks a site atom held by another rank of a slab decomposition
      LFMM_REQUIRE(atom_index[a] >= (plan->dist_lg > 0 ? -1 : 0) && atom_index[a] < plan->N,
                   "site particle index out of range");
      aidx[a] = (int)atom_index[a];
    }
    {
      // sites never share particles (system.validate_system, system.py:135-143);
      // the HI spatial forces rely on it (one writer per force row)
      std::vector<int> owner((size_t)std::max<int64_t>(plan->N, 1), -1);
      for (int64_t s = 0; s < S; ++s)
        for (int a = aoff[s]; a < aoff[s + 1]; ++a) {
          const int i = aidx[a];
          if (i < 0) continue;
          LFMM_REQUIRE(owner[i] != (int)s, "site " + std::to_string(s) + ": duplicate particle indices");
          LFMM_REQUIRE(owner[i] < 0, "site " + std::to_string(s) + ": site overlap on particle indices [" +
                                         std::to_string(i) + "]");
          owner[i] = (int)s;
        }
    }
    fsl[0] = 0;
    for (int64_t s = 0; s < S; ++s) {
      const int ns = aoff[s + 1] - aoff[s];
      LFMM_REQUIRE(ns >= 1, "site " + std::to_string(s) + ": empty particle list");
      nf[s] = n_forms[s];
      LFMM_REQUIRE(nf[s] >= 1 && nf[s] <= HI_MAXF, "site " + std::to_string(s) + ": bad form count");
      LFMM_REQUIRE(foff[s + 1] - foff[s] == nf[s] * ns, "site " + std::to_string(s) + ": form table size");
      fsl[s + 1] = fsl[s] + nf[s];
      ns_max = std::max(ns_max, ns);
    }
    plan->n_sites = S;
    plan->n_site_atoms = A;
    plan->n_form_slots = fsl[S];
    plan->ns_max = ns_max;
    plan->h_atom_off = aoff;
    plan->h_atom_idx = aidx;
    plan->h_nforms = nf;
    plan->h_fslot_off = fsl;
    auto up = [&](DevBuf& d, const void* h, size_t bytes) {
      d.ensure(std::max<size_t>(bytes, 8));
      if (bytes) LFMM_CUDA(cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, plan->stream));
    };
    up(plan->atom_off, aoff.data(), sizeof(int) * (S + 1));
    up(plan->atom_idx, aidx.data(), sizeof(int) * A);
    up(plan->nforms, nf.data(), sizeof(int) * S);
    up(plan->form_off, foff.data(), sizeof(int) * (S + 1));
    up(plan->fslot_off, fsl.data(), sizeof(int) * (S + 1));
    up(plan->form_q, form_charges, sizeof(double) * foff[S]);
    plan->site_pos.ensure(sizeof(double) * 3 * std::max<int64_t>(A, 1));
    plan->lambdas.ensure(sizeof(double) * 4 * std::max<int64_t>(S, 1));
    plan->nlam.ensure(sizeof(int) * std::max<int64_t>(S, 1));
    plan->rscr.ensure(sizeof(double) * plan->ncp * std::max<int64_t>(A, 1));
    plan->uscr.ensure(sizeof(double) * plan->ncp * std::max<int64_t>(A, 1));
    const size_t fs = sizeof(double) * std::max<int64_t>(fsl[S], 1);
    plan->c_p2p.ensure(fs);
    plan->c_lat.ensure(fs);
    plan->c_dip.ensure(fs);
    plan->blend.ensure(sizeof(double) * std::max<int64_t>(S, 1));
    plan->lam_forces.ensure(sizeof(double) * 4 * std::max<int64_t>(S, 1));
    plan->offsets.ensure(sizeof(double) * std::max<int64_t>(S, 1));
    plan->site_force.ensure(sizeof(double) * 3 * std::max<int64_t>(A, 1));
    plan->site_force_valid = false;
    ++plan->epoch;
    LFMM_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int lfmm_hi(lfmm_plan* plan, const double* lambdas, const int32_t* n_lambda, int mode, const double* site_positions,
            const double* potentials, int io_on_device, double* c_p2p, double* c_lattice, double* c_dipole,
            double* blend_energy, double* lambda_forces, double* energy_offset) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(mode == LFMM_MODE_HI || mode == LFMM_MODE_QI, "unknown mode");
    upload_lambdas(plan, lambdas, n_lambda, io_on_device);
    gather_site_positions(plan, site_positions, io_on_device);
    const double* pot = nullptr;
    if (potentials) {
      plan->pot_tmp.ensure(sizeof(double) * std::max<int64_t>(plan->N, 1));
      LFMM_CUDA(cudaMemcpyAsync(plan->pot_tmp.p, potentials, sizeof(double) * plan->N,
                                io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, plan->stream));
      pot = plan->pot_tmp.as<double>();
    } else if (lambda_forces) {
      LFMM_REQUIRE(plan->last_valid && plan->last_k == 1, "no single-column solve to take potentials from");
      pot = plan->out_pot.as<double>();
    }
    run_hi(plan, mode, pot);
    const size_t S = (size_t)plan->n_sites, F = (size_t)plan->n_form_slots;
    copy_out(plan, c_p2p, plan->c_p2p, sizeof(double) * F, io_on_device);
    copy_out(plan, c_lattice, plan->c_lat, sizeof(double) * F, io_on_device);
    copy_out(plan, c_dipole, plan->c_dip, sizeof(double) * F, io_on_device);
    copy_out(plan, blend_energy, plan->blend, sizeof(double) * S, io_on_device);
    copy_out(plan, lambda_forces, plan->lam_forces, sizeof(double) * 4 * S, io_on_device);
    copy_out(plan, energy_offset, plan->offset_total, sizeof(double), io_on_device);
    if (!io_on_device) {
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
      require_finite(lambda_forces, 4 * plan->n_sites, "the lambda forces");
      require_finite(energy_offset, 1, "the HI energy offset");
    }
  });
}

int lfmm_hi_site_forces(lfmm_plan* plan, int io_on_device, double* out) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(out != nullptr || plan->n_site_atoms == 0, "out is NULL");
    LFMM_REQUIRE(plan->site_force_valid, "no HI-mode correction pass to take site forces from");
    copy_out(plan, out, plan->site_force, sizeof(double) * 3 * plan->n_site_atoms, io_on_device);
    if (!io_on_device) LFMM_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int lfmm_lambda_baoab(lfmm_plan* plan, int64_t n_sites, double* lambdas, double* velocities, const int32_t* n_lambda,
                      const double* masses, const double* f_engine, double* f_total, int stage, double dt,
                      double coulomb, double bias_height, double c1, double noise, uint64_t seed, uint64_t step) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(stage >= 0 && stage <= 2, "stage must be 0, 1 or 2");
    LFMM_REQUIRE(n_sites >= 0 && n_sites < (1 << 28), "n_sites out of range");
    if (n_sites == 0) return;
    plan->launch(ST_HI, [&] {
      k_lambda_baoab<<<nblk(4 * n_sites, 128), 128, 0, plan->stream>>>(
          (int)n_sites, lambdas, velocities, n_lambda, masses, f_engine, f_total, stage, dt, coulomb, bias_height, c1,
          noise, (unsigned long long)seed, (unsigned long long)step);
    });
  });
}

int lfmm_lambda_record(lfmm_plan* plan, int64_t n_sites, const int32_t* slot_offsets, const int32_t* n_lambda,
                       const double* lambdas, const double* velocities, const double* f_total, const double* energy,
                       double coulomb, int64_t n_slots, double* out_lambdas, double* out_velocities,
                       double* out_forces, double* out_energies, int64_t sample) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(n_sites >= 0 && sample >= 0, "bad sample");
    plan->launch(ST_HI, [&] {
      k_lambda_record<<<nblk(std::max<int64_t>(4 * n_sites, 1), 128), 128, 0, plan->stream>>>(
          (int)n_sites, slot_offsets, n_lambda, lambdas, velocities, f_total, energy, coulomb, (int)n_slots,
          out_lambdas, out_velocities, out_forces, out_energies, (int)sample);
    });
  });
}

int lfmm_site_gram(lfmm_plan* plan, const double* lambdas, const int32_t* n_lambda, const double* site_positions,
                   double* gram) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(gram != nullptr, "gram is NULL");
    upload_lambdas(plan, lambdas, n_lambda, 0);
    gather_site_positions(plan, site_positions, 0);
    const size_t n = (size_t)plan->n_sites * HI_MAXF * HI_MAXF;
    plan->gram.ensure(sizeof(double) * std::max<size_t>(n, 1));
    LFMM_CUDA(cudaMemsetAsync(plan->gram.p, 0, sizeof(double) * std::max<size_t>(n, 1), plan->stream));
    run_hi(plan, LFMM_MODE_HI, nullptr, nullptr, plan->gram.as<double>());
    if (n) LFMM_CUDA(cudaMemcpyAsync(gram, plan->gram.p, sizeof(double) * n, cudaMemcpyDeviceToHost, plan->stream));
    LFMM_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int lfmm_assemble(int64_t n_sites, const int64_t* atom_offsets, const int64_t* atom_index, const int32_t* n_forms,
                  const int64_t* form_offsets, const double* form_charges, const double* lambdas,
                  const int32_t* n_lambda, const double* c_total, const double* potentials, int64_t n_particles,
                  double* out) {
  return guarded([&] {
    const int64_t S = n_sites;
    LFMM_REQUIRE(S >= 0, "n_sites < 0");
    if (S == 0) return;
    std::vector<int> aoff(S + 1), foff(S + 1), fsl(S + 1, 0), nf(S), nl(S);
    for (int64_t s = 0; s <= S; ++s) {
      aoff[s] = (int)atom_offsets[s];
      foff[s] = (int)form_offsets[s];
    }
    const int64_t A = atom_offsets[S];
    std::vector<int> aidx(A);
    for (int64_t a = 0; a < A; ++a) {
      LFMM_REQUIRE(atom_index[a] >= 0 && atom_index[a] < n_particles, "site particle index out of range");
      aidx[a] = (int)atom_index[a];
    }
    for (int64_t s = 0; s < S; ++s) {
      nf[s] = n_forms[s];
      nl[s] = n_lambda[s];
      LFMM_REQUIRE(nl[s] >= 1 && nl[s] <= 4 && (1 << nl[s]) == nf[s],
                   std::to_string(nl[s]) + " lambdas give " + std::to_string(1 << nl[s]) + " weights, site has " +
                       std::to_string(nf[s]) + " forms");
      fsl[s + 1] = fsl[s] + nf[s];
    }
    DevBuf d_ao, d_ai, d_nf, d_fo, d_fs, d_fq, d_lam, d_nl, d_ct, d_pot, d_out;
    cudaStream_t st;
    LFMM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto up = [&](DevBuf& d, const void* h, size_t bytes) {
      d.ensure(std::max<size_t>(bytes, 8));
      if (bytes) LFMM_CUDA(cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, st));
    };
    up(d_ao, aoff.data(), sizeof(int) * (S + 1));
    up(d_ai, aidx.data(), sizeof(int) * A);
    up(d_nf, nf.data(), sizeof(int) * S);
    up(d_fo, foff.data(), sizeof(int) * (S + 1));
    up(d_fs, fsl.data(), sizeof(int) * (S + 1));
    up(d_fq, form_charges, sizeof(double) * foff[S]);
    up(d_lam, lambdas, sizeof(double) * 4 * S);
    up(d_nl, nl.data(), sizeof(int) * S);
    if (c_total) up(d_ct, c_total, sizeof(double) * fsl[S]);
    up(d_pot, potentials, sizeof(double) * n_particles);
    d_out.ensure(sizeof(double) * 4 * S);
    k_assemble<<<nblk(S, 4), 128, 0, st>>>((int)S, d_ao.as<int>(), d_ai.as<int>(), d_nf.as<int>(), d_fo.as<int>(),
                                           d_fs.as<int>(), d_fq.as<double>(), d_lam.as<double>(), d_nl.as<int>(),
                                           c_total ? d_ct.as<double>() : nullptr, d_pot.as<double>(),
                                           d_out.as<double>());
    LFMM_CUDA(cudaGetLastError());
    LFMM_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(double) * 4 * S, cudaMemcpyDeviceToHost, st));
    LFMM_CUDA(cudaStreamSynchronize(st));
    DevBuf* bufs[] = {&d_ao, &d_ai, &d_nf, &d_fo, &d_fs, &d_fq, &d_lam, &d_nl, &d_ct, &d_pot, &d_out};
    for (auto* b : bufs) b->release();
    cudaStreamDestroy(st);
  });
}

int lfmm_scale_charges(lfmm_plan* plan, const double* charges, const double* lambdas, const int32_t* n_lambda,
                       int io_on_device, double* out_charges) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    const int64_t N = plan->N;
    upload_lambdas(plan, lambdas, n_lambda, io_on_device);
    plan->q_tmp.ensure(sizeof(double) * std::max<int64_t>(N, 1));
    plan->pot_tmp.ensure(sizeof(double) * std::max<int64_t>(N, 1));
    LFMM_CUDA(cudaMemcpyAsync(plan->pot_tmp.p, charges, sizeof(double) * N,
                              io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, plan->stream));
    run_scale(plan, plan->pot_tmp.as<double>(), plan->q_tmp.as<double>());
    copy_out(plan, out_charges, plan->q_tmp, sizeof(double) * N, io_on_device);
    if (!io_on_device) LFMM_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

}  // extern "C"

namespace {
void step_body(lfmm_plan* plan, const double* positions, const double* charges, const double* lambdas,
               const int32_t* n_lambda, int mode, int plain, int io_on_device, double* energy, double* forces,
               double* lambda_forces, double* potentials) {
  {
    const int64_t N = plan->N;
    LFMM_REQUIRE(mode == LFMM_MODE_HI || mode == LFMM_MODE_QI, "unknown mode");
    // device-resident inputs: the lambdas and the HI side work are issued
    // before the tree build, so the HI kernels (site geometry and lambdas
    // only) overlap the latency-bound tree kernels, and the charges (copy +
    // site blend) follow the tree; host inputs keep the positions upload
    // first (the charges upload hides the tree build)
    const bool early = io_on_device && positions && !plain && plan->n_sites > 0 && !plan->profiling &&
                       potentials == nullptr;
    auto tree = [&] {
      if (plan->fp32)
        plan->build_tree<float>(positions, io_on_device != 0);
      else
        plan->build_tree<double>(positions, io_on_device != 0);
    };
    if (positions && !early) tree();
    plan->ensure_solve_buffers(1, true);
    const auto kind = io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const bool overlap = !io_on_device;
    if (overlap) {
      if (!plan->io_stream) LFMM_CUDA(cudaStreamCreateWithFlags(&plan->io_stream, cudaStreamNonBlocking));
      if (!plan->ev_q) LFMM_CUDA(cudaEventCreateWithFlags(&plan->ev_q, cudaEventDisableTiming));
      if (!plan->ev_f) LFMM_CUDA(cudaEventCreateWithFlags(&plan->ev_f, cudaEventDisableTiming));
    }
    const bool blend_q = !(plain || plan->n_sites == 0);
    // scale_charges (system.py:179-197) = the charges copied into q_in, then
    // the site atoms' entries blended over their forms (k_blend_sites)
    auto charges_in = [&] {
      if (overlap) {
        // the charges upload overlaps the tree build
        LFMM_CUDA(cudaMemcpyAsync(plan->q_in.p, charges, sizeof(double) * N, kind, plan->io_stream));
        LFMM_CUDA(cudaEventRecord(plan->ev_q, plan->io_stream));
        LFMM_CUDA(cudaStreamWaitEvent(plan->stream, plan->ev_q, 0));
      } else {
        LFMM_CUDA(cudaMemcpyAsync(plan->q_in.p, charges, sizeof(double) * N, kind, plan->stream));
      }
      if (blend_q) blend_sites(plan, plan->q_in.as<double>());
    };
    if (blend_q) upload_lambdas(plan, lambdas, n_lambda, io_on_device);
    if (!early) charges_in();
    // HI corrections depend on the site geometry and lambdas only: they run
    // beside the solve (unless profiling, which wants serial stage times)
    const bool hi_side = !plain && plan->n_sites > 0 && !plan->profiling && potentials == nullptr;
    if (hi_side) {
      if (!plan->hi_stream) {
        int lo = 0, hi = 0;
        LFMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        LFMM_CUDA(cudaStreamCreateWithPriority(&plan->hi_stream, cudaStreamNonBlocking, lo));
        LFMM_CUDA(cudaEventCreateWithFlags(&plan->ev_hi_in, cudaEventDisableTiming));
        LFMM_CUDA(cudaEventCreateWithFlags(&plan->ev_hi_out, cudaEventDisableTiming));
      }
      LFMM_CUDA(cudaEventRecord(plan->ev_hi_in, plan->stream));
      LFMM_CUDA(cudaStreamWaitEvent(plan->hi_stream, plan->ev_hi_in, 0));
      cudaStream_t main = plan->stream;
      plan->stream = plan->hi_stream;
      try {
        if (early) {  // site atoms straight from the caller's positions (pos_in is filled by the tree build)
          if (plan->n_site_atoms > 0)
            plan->launch(ST_HI, [&] {
              k_gather_site_pos<<<nblk(plan->n_site_atoms, 128), 128, 0, plan->stream>>>(
                  positions, plan->atom_idx.as<int>(), (int)plan->n_site_atoms, plan->site_pos.as<double>());
            });
        } else {
          gather_site_positions(plan, nullptr, 0);
        }
        run_hi(plan, mode, nullptr, nullptr);  // C_rho, blend energies, offsets
      } catch (...) {
        plan->stream = main;
        throw;
      }
      plan->stream = main;
      LFMM_CUDA(cudaEventRecord(plan->ev_hi_out, plan->hi_stream));
    }
    if (early) {  // device inputs: the HI side stream is already running; charges after the tree
      tree();
      charges_in();
    }
    plan->step_mode = potentials == nullptr;
    plan->near_after_hi = hi_side && !early;
    plan->run_solve(1, true);
    plan->near_after_hi = false;
    const bool step_mode = plan->step_mode;
    plan->step_mode = false;
    // HI spatial forces: -grad Delta E_site on the site atoms (k_hi_site,
    // issued on the HI side stream before the solve)
    const bool site_forces = !plain && plan->n_sites > 0 && mode == LFMM_MODE_HI;
    const bool add_off = !plain && plan->n_sites > 0 && mode == LFMM_MODE_HI;
    // step mode with the HI side stream: one tail kernel does site
    // potentials, lambda forces, site forces and the energy
    const bool fused_tail = !plain && plan->n_sites > 0 && step_mode && hi_side;
    if (fused_tail) {
      LFMM_CUDA(cudaStreamWaitEvent(plan->stream, plan->ev_hi_out, 0));
      plan->site_pot.ensure(sizeof(double) * std::max<int64_t>(plan->n_site_atoms, 1));
      HiArgs g{};
      hi_args(plan, g);
      g.pot_site = plan->site_pot.as<double>();
      g.mode = mode;
      g.c_p2p = plan->c_p2p.as<double>();
      g.c_lat = plan->c_lat.as<double>();
      g.c_dip = plan->c_dip.as<double>();
      g.forces = plan->lam_forces.as<double>();
      auto fill = [&](auto& t, auto* vn, auto* vf) {
        t.inv_perm = plan->inv_perm.as<int>();
        t.vnear = vn;
        t.vfar = vf;
        t.pos_sorted = plan->pos_sorted.as<double>();
        t.scal = plan->scal.as<double>();
        t.dipole = (plan->flags & LFMM_F_DIPOLE) ? 1 : 0;
        t.leaf_sorted = plan->leaf_sorted.as<int>();
        t.depth = plan->depth;
        t.x0 = plan->own_x0;
        t.x1 = plan->own_x1;
        t.pot_site = plan->site_pot.as<double>();
        t.forces = plan->out_forces.as<double>();
        t.site_force = site_forces ? plan->site_force.as<double>() : nullptr;
        t.energies = plan->energies.as<double>();
        t.off = plan->offset_total.as<double>();
        t.add_off = add_off ? 1 : 0;
        t.energy_out = plan->scal.as<double>() + 6;
      };
      plan->launch(ST_FINAL, [&] {
        if (plan->fp32) {
          TailArgs<float> t{};
          fill(t, plan->vnear.as<float>(), plan->vfar.as<float>());
          k_step_tail<float><<<nblk(plan->n_sites, 4), 128, 0, plan->stream>>>(g, t);
        } else {
          TailArgs<double> t{};
          fill(t, plan->vnear.as<double>(), plan->vfar.as<double>());
          k_step_tail<double><<<nblk(plan->n_sites, 4), 128, 0, plan->stream>>>(g, t);
        }
      });
    }
    if (overlap && forces) {
      // the forces download overlaps the HI corrections
      LFMM_CUDA(cudaEventRecord(plan->ev_f, plan->stream));
      LFMM_CUDA(cudaStreamWaitEvent(plan->io_stream, plan->ev_f, 0));
      LFMM_CUDA(cudaMemcpyAsync(forces, plan->out_forces.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost,
                                plan->io_stream));
    }
    if (!plain && plan->n_sites > 0 && !fused_tail) {
      gather_site_positions(plan, nullptr, 0);
      if (step_mode) {
        plan->site_pot.ensure(sizeof(double) * std::max<int64_t>(plan->n_site_atoms, 1));
        const int na = (int)plan->n_site_atoms;
        const int dip = (plan->flags & LFMM_F_DIPOLE) ? 1 : 0;
        plan->launch(ST_HI, [&] {
          if (plan->fp32)
            k_site_pot<float><<<nblk(na, 128), 128, 0, plan->stream>>>(
                plan->atom_idx.as<int>(), na, plan->inv_perm.as<int>(), plan->vnear.as<float>(), plan->vfar.as<float>(),
                plan->pos_sorted.as<double>(), plan->scal.as<double>(), dip, plan->L, plan->site_pot.as<double>(),
                plan->leaf_sorted.as<int>(), plan->depth, plan->own_x0, plan->own_x1);
          else
            k_site_pot<double><<<nblk(na, 128), 128, 0, plan->stream>>>(
                plan->atom_idx.as<int>(), na, plan->inv_perm.as<int>(), plan->vnear.as<double>(),
                plan->vfar.as<double>(), plan->pos_sorted.as<double>(), plan->scal.as<double>(), dip, plan->L,
                plan->site_pot.as<double>(), plan->leaf_sorted.as<int>(), plan->depth, plan->own_x0, plan->own_x1);
        });
        run_hi(plan, mode, nullptr, plan->site_pot.as<double>());
      } else {
        run_hi(plan, mode, plan->out_pot.as<double>());
      }
      if (site_forces) add_site_forces(plan);
    }
    // energy = E_solve + sum of site offsets (hi_energy_and_forces :273)
    if (!fused_tail)
      plan->launch(ST_FINAL, [&] {
        k_step_energy<<<1, 1, 0, plan->stream>>>(plan->energies.as<double>(), plan->offset_total.as<double>(),
                                                 add_off ? 1 : 0, plan->scal.as<double>() + 6);
      });
    if (energy)
      LFMM_CUDA(cudaMemcpyAsync(energy, plan->scal.as<double>() + 6, sizeof(double),
                                io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, plan->stream));
    if (!overlap) copy_out(plan, forces, plan->out_forces, sizeof(double) * 3 * N, io_on_device);
    if (!plain) copy_out(plan, lambda_forces, plan->lam_forces, sizeof(double) * 4 * plan->n_sites, io_on_device);
    copy_out(plan, potentials, plan->out_pot, sizeof(double) * N, io_on_device);
    if (!io_on_device) {
      LFMM_CUDA(cudaStreamSynchronize(plan->stream));
      LFMM_CUDA(cudaStreamSynchronize(plan->io_stream));
      require_finite(energy, 1, "the step energy");
      if (!plain) require_finite(lambda_forces, 4 * plan->n_sites, "the lambda forces");
    }
  }
}

// Device-resident step through the plan's step graph (see lfmm_plan::graphs).
// Returns false when the call has to run uncaptured.
bool step_graph_launch(lfmm_plan* plan, const double* positions, const double* charges, const double* lambdas,
                       const int32_t* n_lambda, int mode, int plain, double* energy, double* forces,
                       double* lambda_forces, double* potentials) {
  auto& g = plan->step_graph;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  LFMM_CUDA(cudaStreamIsCapturing(plan->stream, &cs));
  if (cs != cudaStreamCaptureStatusNone) return false;  // the caller is capturing its own graph: record into it
  const std::array<const void*, 10> ptrs{positions, charges, lambdas, n_lambda, energy, forces, lambda_forces,
                                         potentials, nullptr, nullptr};
  const bool same = g.ptrs == ptrs && g.mode == mode && g.plain == plain && g.stream == plan->stream &&
                    g.epoch == plan->epoch;
  if (g.exec && same && g.gen == g_alloc_gen.load()) {
    LFMM_CUDA(cudaGraphLaunch(g.exec, plan->stream));
    plan->launches += g.nlaunch;
    return true;
  }
  if (g.exec) {
    LFMM_CUDA(cudaGraphExecDestroy(g.exec));
    g.exec = nullptr;
  }
  if (!same || !g.warm) {  // first call with these arguments: run it (allocates), capture on the next
    g.ptrs = ptrs;
    g.mode = mode;
    g.plain = plain;
    g.stream = plan->stream;
    g.epoch = plan->epoch;
    g.warm = true;
    return false;
  }
  const uint64_t gen0 = g_alloc_gen.load();
  const int64_t l0 = plan->launches;
  LFMM_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
  cudaGraph_t graph = nullptr;
  try {
    step_body(plan, positions, charges, lambdas, n_lambda, mode, plain, 1, energy, forces, lambda_forces,
              potentials);
  } catch (...) {
    cudaStreamEndCapture(plan->stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    plan->launches = l0;
    plan->graphs = false;  // something in the step cannot be captured: stay uncaptured
    return false;
  }
  const cudaError_t ec = cudaStreamEndCapture(plan->stream, &graph);
  if (ec != cudaSuccess || !graph || g_alloc_gen.load() != gen0) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    plan->launches = l0;
    plan->graphs = false;
    return false;
  }
  const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    cudaGetLastError();
    g.exec = nullptr;
    plan->launches = l0;
    plan->graphs = false;
    return false;
  }
  g.nlaunch = plan->launches - l0;
  g.gen = gen0;
  plan->launches = l0;
  LFMM_CUDA(cudaGraphLaunch(g.exec, plan->stream));
  plan->launches += g.nlaunch;
  return true;
}
}  // namespace

extern "C" {

int lfmm_step(lfmm_plan* plan, const double* positions, const double* charges, const double* lambdas,
              const int32_t* n_lambda, int mode, int plain, int io_on_device, double* energy, double* forces,
              double* lambda_forces, double* potentials) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(mode == LFMM_MODE_HI || mode == LFMM_MODE_QI, "unknown mode");
    if (io_on_device && plan->graphs && !plan->profiling && !plan->tracing &&
        step_graph_launch(plan, positions, charges, lambdas, n_lambda, mode, plain, energy, forces,
                          lambda_forces, potentials))
      return;
    step_body(plan, positions, charges, lambdas, n_lambda, mode, plain, io_on_device, energy, forces,
              lambda_forces, potentials);
  });
}

// ---- slab decomposition (paper_2410_01754_b200/distributed.py) ----
int lfmm_plan_set_count(lfmm_plan* plan, int64_t n) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(n >= 0 && n < (1LL << 31), "particle count out of range");
    ++plan->epoch;
    const int64_t nn = std::max<int64_t>(n, 1);
    const size_t t = plan->tsz();
    plan->pos_in.ensure(sizeof(double) * 3 * nn);
    plan->key32.ensure(sizeof(float) * nn);
    plan->leaf_of.ensure(sizeof(int) * nn);
    plan->slot_of.ensure(sizeof(int) * nn);
    plan->bucket.ensure(sizeof(int) * nn);
    plan->perm.ensure(sizeof(int) * nn);
    plan->inv_perm.ensure(sizeof(int) * nn);
    plan->pos_sorted.ensure(sizeof(double) * 3 * nn);
    plan->leaf_sorted.ensure(sizeof(int) * nn);
    plan->xq.ensure(4 * t * nn);
    plan->ensure_pairs(nn);
    plan->N = n;
    plan->last_valid = false;
  });
}

int lfmm_dist_configure(lfmm_plan* plan, int x0, int x1, int lg) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    const int n = 1 << plan->depth;
    LFMM_REQUIRE(0 <= x0 && x0 < x1 && x1 <= n, "owned leaf x-range outside the grid");
    LFMM_REQUIRE(lg >= 0 && lg <= plan->depth, "bad shared-level count");
    ++plan->epoch;
    plan->own_x0 = x0;
    plan->own_x1 = x1;
    plan->dist_lg = lg;
    if (plan->use_halo) {
      plan->plan_halo_jobs();
      plan->hm_astages = halo_smem_attr(plan->hm_rw_cap);
    }
  });
}

// phase 1: tree + charges (+ lambda scaling) + P2P (owned leaves) + P2M +
// M2M of the levels >= lg + box charges.  phase 2 (after the caller gathered
// the owned multipoles and the dipole/charge sums into the buffers exported
// by lfmm_dist_buffers): shared levels, lattice, M2L, L2L, L2P, finalize,
// owned site-atom potentials.  All pointers are device pointers.
int lfmm_dist_phase(lfmm_plan* plan, int phase, const double* positions, const double* charges,
                    const double* lambdas, const int32_t* n_lambda, int grad) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(phase == 1 || phase == 2, "phase must be 1 or 2");
    const int64_t N = plan->N;
    if (phase == 1) {
      if (positions) {
        if (plan->fp32)
          plan->build_tree<float>(positions, true);
        else
          plan->build_tree<double>(positions, true);
      }
      plan->ensure_solve_buffers(1, grad != 0);
      plan->q_tmp.ensure(sizeof(double) * std::max<int64_t>(N, 1));
      if (lambdas && plan->n_sites > 0) {
        upload_lambdas(plan, lambdas, n_lambda, 1);
        LFMM_CUDA(cudaMemcpyAsync(plan->q_tmp.p, charges, sizeof(double) * N, cudaMemcpyDeviceToDevice, plan->stream));
        run_scale(plan, plan->q_tmp.as<double>(), plan->q_in.as<double>());
      } else if (N > 0) {
        LFMM_CUDA(cudaMemcpyAsync(plan->q_in.p, charges, sizeof(double) * N, cudaMemcpyDeviceToDevice, plan->stream));
      }
    }
    plan->dist_phase = phase;
    plan->step_mode = true;
    try {
      if (plan->fp32)
        plan->solve_column<float>(1, 0, grad != 0);
      else
        plan->solve_column<double>(1, 0, grad != 0);
    } catch (...) {
      plan->dist_phase = 0;
      plan->step_mode = false;
      throw;
    }
    plan->dist_phase = 0;
    plan->step_mode = false;
    if (phase == 2 && plan->n_sites > 0) {
      plan->site_pot.ensure(sizeof(double) * std::max<int64_t>(plan->n_site_atoms, 1));
      const int na = (int)plan->n_site_atoms;
      const int dip = (plan->flags & LFMM_F_DIPOLE) ? 1 : 0;
      plan->launch(ST_HI, [&] {
        if (plan->fp32)
          k_site_pot<float><<<nblk(na, 128), 128, 0, plan->stream>>>(
              plan->atom_idx.as<int>(), na, plan->inv_perm.as<int>(), plan->vnear.as<float>(), plan->vfar.as<float>(),
              plan->pos_sorted.as<double>(), plan->scal.as<double>(), dip, plan->L, plan->site_pot.as<double>(),
              plan->leaf_sorted.as<int>(), plan->depth, plan->own_x0, plan->own_x1);
        else
          k_site_pot<double><<<nblk(na, 128), 128, 0, plan->stream>>>(
              plan->atom_idx.as<int>(), na, plan->inv_perm.as<int>(), plan->vnear.as<double>(),
              plan->vfar.as<double>(), plan->pos_sorted.as<double>(), plan->scal.as<double>(), dip, plan->L,
              plan->site_pot.as<double>(), plan->leaf_sorted.as<int>(), plan->depth, plan->own_x0, plan->own_x1);
      });
    }
  });
}

// device pointers of the buffers the slab decomposition exchanges:
// [0] multipoles (all levels, ncp per box, T), [1] scal (D_x, D_y, D_z, Q as
// fp64), [2] energies (total, near, far, dipole), [3] forces (N x 3, local
// input order), [4] site-atom potentials, [5] lambda forces (S x 4),
// [6] HI energy offset (1), [7] stream, [8] per-level max |M^/c| of the fp16
// M2L (uint32 float bits, DMAX + 2 entries; NULL unless the fp32 tensor-core
// M2L runs); level_off[l] = first box of level l
int lfmm_dist_buffers(lfmm_plan* plan, void** ptrs, int64_t* level_off, int64_t* ncp) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    if (ncp) *ncp = plan->ncp;
    ptrs[0] = plan->mult.p;
    ptrs[1] = plan->scal.p;
    ptrs[2] = plan->energies.p;
    ptrs[3] = plan->out_forces.p;
    ptrs[4] = plan->site_pot.p;
    ptrs[5] = plan->lam_forces.p;
    ptrs[6] = plan->offset_total.p;
    ptrs[7] = reinterpret_cast<void*>(plan->stream);
    ptrs[8] = plan->hm_level_max.p;
    for (int l = 0; l <= DMAX + 1; ++l) level_off[l] = l <= plan->depth + 1 ? plan->level_off[l] : 0;
  });
}

// HI for every site of the (global) site table from the gathered site-atom
// potentials; site positions are caller-supplied (device)
int lfmm_dist_hi(lfmm_plan* plan, const double* site_positions, int mode) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    LFMM_REQUIRE(mode == LFMM_MODE_HI || mode == LFMM_MODE_QI, "unknown mode");
    if (plan->n_sites == 0) return;
    gather_site_positions(plan, site_positions, 1);
    run_hi(plan, mode, nullptr, plan->site_pot.as<double>());
    // HI spatial forces into the local force rows (remote site atoms carry
    // index -1 and are skipped)
    if (mode == LFMM_MODE_HI) add_site_forces(plan);
  });
}

int lfmm_profile_enable(lfmm_plan* plan, int enable) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    plan->harvest();
    plan->profiling = enable != 0;
    for (int i = 0; i < ST_COUNT; ++i) {
      plan->stage_ms[i] = 0.0;
      plan->stage_launch[i] = 0;
    }
  });
}

int lfmm_stage_count(void) { return ST_COUNT; }

const char* lfmm_stage_name(int i) { return (i >= 0 && i < ST_COUNT) ? kStageNames[i] : ""; }

int lfmm_stage_times(lfmm_plan* plan, double* ms, int64_t* launches, int n) {
  if (!plan) return fail(Error{LFMM_EINVAL, "plan is NULL"});
  return guarded([&] {
    plan->harvest();
    for (int i = 0; i < n && i < ST_COUNT; ++i) {
      if (ms) ms[i] = plan->stage_ms[i];
      if (launches) launches[i] = plan->stage_launch[i];
    }
  });
}

int64_t lfmm_launch_count(const lfmm_plan* plan) { return plan ? plan->launches : -1; }

}  // extern "C"
