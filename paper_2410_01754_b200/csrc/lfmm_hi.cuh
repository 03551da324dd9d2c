// lfmm_hi.cuh — Hamiltonian-interpolation (MAHI) correction, one CTA per
// titratable site, fp64 throughout (the per-site work is tiny; the
// potentials it consumes come from the fp32 or fp64 solve).
//
// Per site with lambda weights w (weights.expand_weights, weights.py:54-60),
// forms Q (nf x ns) and blended charges q~ = w Q (system.scale_charges,
// system.py:179-197):
//   K_st  27-image pair kernel, self-image sum on the diagonal, or the
//         minimum-image kernel          (corrections.near_kernel :46-70)
//   G_st  = Re(R(r_s - L/2) T_L R(r_t - L/2)^T)   (lattice_kernel :73-77),
//         evaluated as the lattice operator applied to the unit-charge
//         multipole of atom t and contracted with R of atom s
//   C_rho = Q_rho K h_rho + Q_rho G h_rho + c_dip,  h_rho = q~ - Q_rho/2
//   c_dip = -eta*gamma*|(q~ - Q_rho).(r - L/2)|^2   (c_dipole :112-124)
//   e(q~) = 1/2 q~ (K+G) q~                          (build_corrections :179-183)
//   S_rho = Q_rho . V[site]                          (s_values :196-198)
//   F_k   = -sum_rho dw_rho/dlambda_k (S_rho - C_rho) (assemble :221-238)
// QI mode: F_k = -sum_rho dw_rho/dlambda_k S_rho, no offset.
//
// HI spatial forces on site atoms.  The reference has spatial forces only as
// spatial_forces(q~) (solver.py:407-427); the HI energy adds
//   Delta E_site = e(q~) - sum_rho w_rho C_rho
//                = sum_st W_st (K + G)_st + eta gamma sum_rho w_rho |D_rho|^2,
//   W_st = 1/2 (sum_rho w_rho Q_rho,s Q_rho,t - q~_s q~_t),
//   D_rho = sum_s (q~_s - Q_rho,s)(r_s - L/2)   (c_dipole :112-124),
// which depends on the site's own atom positions only, so
// the HI-consistent force on site atom i is spatial_forces(q~)_i - grad_i
// Delta E_site with
//   grad_i sum W K = 2 sum_{t != i} W_it sum_n -(d_n / |d_n|^3),
//                    d_n = r_i - r_t + n L      (27 images or minimum image)
//   grad_i sum W G = (2 / L^2) Re< grad_x R(x_i), sum_t W_it U_t >,
//                    x = (r - L/2) / L, U_t = T1 R(x_t), gradient ladder
//                    harmonics.py:119-130 (dx R_l^m = (R_{l-1}^{m-1} -
//                    R_{l-1}^{m+1})/2, dy = i (R_{l-1}^{m-1} + R_{l-1}^{m+1})/2,
//                    dz = R_{l-1}^m)
//   grad_i eta gamma sum w |D|^2 = 2 eta gamma sum_rho w_rho (q~_i - Q_rho,i) D_rho.
#pragma once
#include "lfmm_common.cuh"

namespace lfmm {

constexpr int HI_THREADS = 128;
constexpr int HI_MAXF = 16;  // weights.MAX_BRANCHES = 4 -> 16 forms

struct HiArgs {
  int n_sites;
  const int* atom_off;     // S+1
  const int* atom_idx;     // A, input-order particle index
  const int* nforms;       // S
  const int* form_off;     // S+1, offsets into form_q (nf*ns per site)
  const int* fslot_off;    // S+1, offsets of per-form outputs (sum nf)
  const double* form_q;
  const double* lambdas;   // S x 4
  const int* nlam;         // S
  const double* site_pos;  // A x 3 (caller-supplied site positions)
  const double* pot;       // input-order potentials (N), may be null (corrections only)
  const double* pot_site;  // or: potentials at the site atoms (A), from k_site_pot
  double box;
  int p, ncp;
  const double* lat_t;     // packed lattice operator, transposed [in][out], fp64, or null
  double* rscratch;        // A x ncp
  double* uscratch;        // A x ncp
  int images_full;         // intra_site_images == "full"
  int dipole;
  int mode;                // 0 hi, 1 qi
  // outputs
  double* c_p2p;
  double* c_lat;
  double* c_dip;
  double* blend;       // S
  double* forces;      // S x 4
  double* offset;      // S
  double* gram;        // optional: S x HI_MAXF x HI_MAXF, Q (K + G) Q^T (dynamics.py FrozenLambdaForceField)
  double* site_force;  // optional: A x 3, -grad Delta E_site per site atom (HI mode)
};

// R_l^m of a packed conj-symmetric vector, any m (X_l^-m = (-1)^m conj X_l^m,
// harmonics.py:3-8), zero outside |m| <= l
__device__ inline double2 pk_get(const double* a, int p, int l, int m) {
  if (l < 0 || m > l || -m > l) return make_double2(0.0, 0.0);
  if (m == 0) return make_double2(a[l], 0.0);
  const int mm = m < 0 ? -m : m;
  const int c = pk_index(p, l, mm, 0);
  double re = a[c], im = a[c + 1];
  if (m < 0) {
    const double sg = (mm & 1) ? -1.0 : 1.0;
    re *= sg;
    im *= -sg;
  }
  return make_double2(re, im);
}

__device__ inline double hi_weight(const double* lam, int nl, int rho) {
  double w = 1.0;
  for (int k = 0; k < nl; ++k) w *= ((rho >> k) & 1) ? lam[k] : (1.0 - lam[k]);
  return w;
}
__device__ inline double hi_wgrad(const double* lam, int nl, int k, int rho) {
  double g = 1.0;
  for (int i = 0; i < nl; ++i) {
    if (i == k)
      g *= ((rho >> i) & 1) ? 1.0 : -1.0;
    else
      g *= ((rho >> i) & 1) ? lam[i] : (1.0 - lam[i]);
  }
  return g;
}

// Packed weighted dot Re sum_full a b for conj-symmetric packed vectors.
__device__ inline double packed_pair(const double* a, const double* b, int p, int lane_lo, int stride) {
  const int nc = ncoef(p);
  double s = 0.0;
  for (int c = lane_lo; c < nc; c += stride) {
    if (c <= p) {
      s += a[c] * b[c];
    } else {
      const int r = c - (p + 1);
      // entries after the m=0 block come in (re, im) pairs
      s += (r & 1) ? -2.0 * a[c] * b[c] : 2.0 * a[c] * b[c];
    }
  }
  return s;
}

// -grad Delta E_site of every atom of one site (see the header); called by the
// whole CTA of k_hi_site once K, G, R_t/U_t (shared memory) and D_rho are in
// place.  Warp per atom, fixed-order lane sums: reruns are bit-identical.
__device__ __noinline__ void hi_site_force(const HiArgs& g, int s, int a0, int ns, int nf, const double* Q,
                                           const double* qt, const double* w, const double* pos, double* Wm,
                                           const double* Dv, bool lattice, double gamma) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double L = g.box;
  const int p = g.p, ncp = g.ncp, nc = ncoef(p);
  for (int e = tid; e < ns * ns; e += blockDim.x) {
    const int i = e / ns, j = e % ns;
    double acc = 0.0;
    for (int r = 0; r < nf; ++r) acc += w[r] * Q[r * ns + i] * Q[r * ns + j];
    Wm[e] = 0.5 * (acc - qt[i] * qt[j]);
  }
  __syncthreads();
  const int rs = ncp + 1;
  const double* Rs = Wm + ns * ns;
  const double* Us = Rs + (size_t)ns * rs;
  const bool dip = g.images_full && g.dipole;
  for (int i = wid; i < ns; i += blockDim.x / 32) {
    double gx = 0.0, gy = 0.0, gz = 0.0;
    // near kernel: full images, lane n < 27 takes image n of every partner
    // (no integer division per term); minimum image, lanes over partners
    if (g.images_full) {
      const double ox = (lane / 9 - 1) * L, oy = ((lane / 3) % 3 - 1) * L, oz = (lane % 3 - 1) * L;
      if (lane < 27)
        for (int t = 0; t < ns; ++t) {
          if (t == i) continue;
          const double dx = pos[3 * i] - pos[3 * t] + ox, dy = pos[3 * i + 1] - pos[3 * t + 1] + oy,
                       dz = pos[3 * i + 2] - pos[3 * t + 2] + oz;
          const double ir = rsqrt(dx * dx + dy * dy + dz * dz);
          const double c = -2.0 * Wm[i * ns + t] * ir * ir * ir;
          gx = fma(c, dx, gx);
          gy = fma(c, dy, gy);
          gz = fma(c, dz, gz);
        }
    } else {
      for (int t = lane; t < ns; t += 32) {
        if (t == i) continue;
        double dx = pos[3 * i] - pos[3 * t], dy = pos[3 * i + 1] - pos[3 * t + 1], dz = pos[3 * i + 2] - pos[3 * t + 2];
        dx -= L * rint(dx / L);
        dy -= L * rint(dy / L);
        dz -= L * rint(dz / L);
        const double ir = rsqrt(dx * dx + dy * dy + dz * dz);
        const double c = -2.0 * Wm[i * ns + t] * ir * ir * ir;
        gx = fma(c, dx, gx);
        gy = fma(c, dy, gy);
        gz = fma(c, dz, gz);
      }
    }
    // lattice kernel: V = sum_t W_it U_t, contracted with grad_x R(x_i)
    if (lattice) {
      const double* Ri = Rs + (size_t)i * rs;
      double hx = 0.0, hy = 0.0, hz = 0.0;
      for (int c = lane; c < nc; c += 32) {
        double v = 0.0;
        for (int t = 0; t < ns; ++t) v = fma(Wm[i * ns + t], Us[(size_t)t * rs + c], v);
        int l, m, part;
        pk_decode_fast(p, c, l, m, part);
        if (l == 0) continue;
        const double2 A = pk_get(Ri, p, l - 1, m - 1), B = pk_get(Ri, p, l - 1, m + 1), C = pk_get(Ri, p, l - 1, m);
        double dxv, dyv, dzv;
        if (part == 0) {
          dxv = 0.5 * (A.x - B.x);
          dyv = -0.5 * (A.y + B.y);
          dzv = C.x;
        } else {
          dxv = 0.5 * (A.y - B.y);
          dyv = 0.5 * (A.x + B.x);
          dzv = C.y;
        }
        // packed pairing Re sum_full a b: m = 0 once, m > 0 twice, imaginary parts negated
        const double wgt = (m == 0) ? v : (part == 0 ? 2.0 * v : -2.0 * v);
        hx = fma(dxv, wgt, hx);
        hy = fma(dyv, wgt, hy);
        hz = fma(dzv, wgt, hz);
      }
      const double sc = 2.0 / (L * L);
      gx = fma(sc, hx, gx);
      gy = fma(sc, hy, gy);
      gz = fma(sc, hz, gz);
    }
    for (int off = 16; off > 0; off >>= 1) {
      gx += __shfl_down_sync(0xffffffffu, gx, off);
      gy += __shfl_down_sync(0xffffffffu, gy, off);
      gz += __shfl_down_sync(0xffffffffu, gz, off);
    }
    if (lane == 0) {
      if (dip) {
        for (int r = 0; r < nf; ++r) {
          const double c = 2.0 * DIPOLE_ETA * gamma * w[r] * (qt[i] - Q[r * ns + i]);
          gx = fma(c, Dv[3 * r], gx);
          gy = fma(c, Dv[3 * r + 1], gy);
          gz = fma(c, Dv[3 * r + 2], gz);
        }
      }
      double* f = g.site_force + 3 * (size_t)(a0 + i);
      f[0] = -gx;
      f[1] = -gy;
      f[2] = -gz;
    }
  }
}

__global__ void __launch_bounds__(HI_THREADS) k_hi_site(HiArgs g) {
  const int s = blockIdx.x;
  if (s >= g.n_sites) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int a0 = g.atom_off[s], ns = g.atom_off[s + 1] - a0;
  const int nf = g.nforms[s], nl = g.nlam[s];
  const double* Q = g.form_q + g.form_off[s];
  const double L = g.box;
  const int p = g.p, ncp = g.ncp, nc = ncoef(p);

  extern __shared__ double sm[];
  double* qt = sm;               // ns
  double* KG = qt + ns;          // ns*ns (K)
  double* GG = KG + ns * ns;     // ns*ns (G)
  double* pos = GG + ns * ns;    // ns*3
  double* Wm = pos + 3 * ns;     // ns*ns: W_st of the site-force gradient
  __shared__ double lam[4], w[HI_MAXF], Cv[HI_MAXF], Sv[HI_MAXF], Dv[3 * HI_MAXF];

  if (tid < 4) lam[tid] = g.lambdas[4 * s + tid];
  for (int i = tid; i < 3 * ns; i += blockDim.x) pos[i] = g.site_pos[3 * a0 + i];
  __syncthreads();
  if (tid < nf) w[tid] = hi_weight(lam, nl, tid);
  __syncthreads();
  for (int t = tid; t < ns; t += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < nf; ++r) acc += w[r] * Q[r * ns + t];
    qt[t] = acc;
  }
  const bool qi = g.mode == 1;
  const bool lattice = !qi && g.images_full && g.lat_t != nullptr;
  if (!qi) {
    // ---- near kernel K ----
    for (int e = tid; e < ns * ns; e += blockDim.x) {
      const int i = e / ns, j = e % ns;
      const double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
                   dz = pos[3 * i + 2] - pos[3 * j + 2];
      double k = 0.0;
      if (g.images_full) {
#pragma unroll
        for (int n = 0; n < 27; ++n) {
          const int nx = n / 9 - 1, ny = (n / 3) % 3 - 1, nz = n % 3 - 1;
          const double ex = dx + nx * L, ey = dy + ny * L, ez = dz + nz * L;
          const double t = rsqrt(ex * ex + ey * ey + ez * ez);
          k += (i == j && n == 13) ? 0.0 : t;
        }
      } else if (i != j) {
        const double ex = dx - L * rint(dx / L), ey = dy - L * rint(dy / L), ez = dz - L * rint(dz / L);
        k = 1.0 / sqrt(ex * ex + ey * ey + ez * ez);
      }
      KG[e] = k;
    }
    // ---- lattice kernel G: R_t and U_t = T1 R_t come precomputed for all
    // site atoms (k_hi_rvec + one batched GEMM, k_translate mode 2); staged
    // in shared memory, G_st = (1/L) <R_s, U_t>_packed, thread per pair ----
    if (lattice) {
      // rows padded to ncp + 1 doubles: the lanes of a warp read different
      // atoms' rows at the same coefficient, which then fall in different banks
      const int rs = ncp + 1;
      double* Rs = Wm + ns * ns;              // ns x rs
      double* Us = Rs + (size_t)ns * rs;      // ns x rs
      const double* R = g.rscratch + (size_t)a0 * ncp;
      const double* U = g.uscratch + (size_t)a0 * ncp;
      const int nv = ns * ncp;
      for (int e0 = tid; e0 < nv; e0 += 4 * HI_THREADS) {  // four loads of each in flight
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * HI_THREADS < nv) {
            a[u] = R[e0 + u * HI_THREADS];
            b[u] = U[e0 + u * HI_THREADS];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * HI_THREADS < nv) {
            const int e = e0 + u * HI_THREADS, row = e / ncp, col = e - row * ncp;
            Rs[row * rs + col] = a[u];
            Us[row * rs + col] = b[u];
          }
      }
      __syncthreads();
      const double invL = 1.0 / L;
      for (int e = tid; e < ns * ns; e += blockDim.x) {
        const int i = e / ns, j = e % ns;
        const double* a = Rs + (size_t)i * rs;
        const double* b = Us + (size_t)j * rs;
        double v = 0.0;
        for (int c = 0; c <= p; ++c) v = fma(a[c], b[c], v);  // m = 0 block
        // m > 0 pairs: two interleaved chains, combined in a fixed order
        double w0 = 0.0, w1 = 0.0;
        int c = p + 1;
        for (; c + 3 < nc; c += 4) {
          w0 = fma(a[c], b[c], fma(-a[c + 1], b[c + 1], w0));
          w1 = fma(a[c + 2], b[c + 2], fma(-a[c + 3], b[c + 3], w1));
        }
        for (; c < nc; c += 2) w0 = fma(a[c], b[c], fma(-a[c + 1], b[c + 1], w0));
        GG[e] = (v + 2.0 * (w0 + w1)) * invL;
      }
    }
  }
  __syncthreads();

  // ---- optional form Gram B = Q (K + G) Q^T (dynamics.py:137-145) ----
  if (g.gram && !qi) {
    for (int e = tid; e < nf * nf; e += blockDim.x) {
      const int r = e / nf, r2 = e % nf;
      const double* Qa = Q + r * ns;
      const double* Qb = Q + r2 * ns;
      double acc = 0.0;
      for (int j = 0; j < ns; ++j) {
        double t = 0.0;  // (Q_r (K + G))_j
        for (int i = 0; i < ns; ++i) t += Qa[i] * (KG[i * ns + j] + (lattice ? GG[i * ns + j] : 0.0));
        acc += t * Qb[j];
      }
      g.gram[((size_t)s * HI_MAXF + r) * HI_MAXF + r2] = acc;
    }
  }

  // ---- per-form scalars (warp per form) ----
  const double gamma = 2.0 * 3.14159265358979323846 / (3.0 * L * L * L);
  for (int r = wid; r < nf; r += blockDim.x / 32) {
    const double* Qr = Q + r * ns;
    double cp = 0.0, cl = 0.0, sv = 0.0, ddx = 0.0, ddy = 0.0, ddz = 0.0;
    for (int i = lane; i < ns; i += 32) {
      if (!qi) {
        double kh = 0.0, gh = 0.0;
        for (int j = 0; j < ns; ++j) {
          const double h = qt[j] - 0.5 * Qr[j];
          kh += KG[i * ns + j] * h;
          if (lattice) gh += GG[i * ns + j] * h;
        }
        cp += Qr[i] * kh;
        cl += Qr[i] * gh;
        const double dev = qt[i] - Qr[i];
        ddx += dev * (pos[3 * i] - 0.5 * L);
        ddy += dev * (pos[3 * i + 1] - 0.5 * L);
        ddz += dev * (pos[3 * i + 2] - 0.5 * L);
      }
      if (g.pot_site)
        sv += Qr[i] * g.pot_site[a0 + i];
      else if (g.pot)
        sv += Qr[i] * g.pot[g.atom_idx[a0 + i]];
    }
    for (int off = 16; off > 0; off >>= 1) {
      cp += __shfl_down_sync(0xffffffffu, cp, off);
      cl += __shfl_down_sync(0xffffffffu, cl, off);
      sv += __shfl_down_sync(0xffffffffu, sv, off);
      ddx += __shfl_down_sync(0xffffffffu, ddx, off);
      ddy += __shfl_down_sync(0xffffffffu, ddy, off);
      ddz += __shfl_down_sync(0xffffffffu, ddz, off);
    }
    if (lane == 0) {
      const double cd = (!qi && g.images_full && g.dipole) ? -DIPOLE_ETA * gamma * (ddx * ddx + ddy * ddy + ddz * ddz) : 0.0;
      const int slot = g.fslot_off[s] + r;
      if (g.c_p2p) g.c_p2p[slot] = cp;
      if (g.c_lat) g.c_lat[slot] = cl;
      if (g.c_dip) g.c_dip[slot] = cd;
      Cv[r] = cp + cl + cd;
      Sv[r] = sv;
      Dv[3 * r] = ddx;
      Dv[3 * r + 1] = ddy;
      Dv[3 * r + 2] = ddz;
    }
  }
  __syncthreads();
  if (g.site_force && !qi) hi_site_force(g, s, a0, ns, nf, Q, qt, w, pos, Wm, Dv, lattice, gamma);
  // ---- blend energy, offset, lambda forces (warp 0) ----
  if (wid == 0) {
    double eb = 0.0;
    if (!qi) {
      for (int e = lane; e < ns * ns; e += 32) {
        const int i = e / ns, j = e % ns;
        eb += qt[i] * (KG[e] + (lattice ? GG[e] : 0.0)) * qt[j];
      }
      for (int off = 16; off > 0; off >>= 1) eb += __shfl_down_sync(0xffffffffu, eb, off);
      eb *= 0.5;
    }
    if (lane == 0) {
      double wc = 0.0;
      for (int r = 0; r < nf; ++r) wc += w[r] * (qi ? 0.0 : Cv[r]);
      if (g.blend) g.blend[s] = eb;
      if (g.offset) g.offset[s] = qi ? 0.0 : eb - wc;
      if (g.forces) {
        for (int k = 0; k < 4; ++k) {
          double f = 0.0;
          if (k < nl && (g.pot || g.pot_site))
            for (int r = 0; r < nf; ++r) f += hi_wgrad(lam, nl, k, r) * (Sv[r] - (qi ? 0.0 : Cv[r]));
          g.forces[4 * s + k] = k < nl ? -f : 0.0;
        }
      }
    }
  }
}

// R(r_t - L/2) / L-normalised regular harmonics of every site atom (packed,
// fp64), the right-hand sides of the batched U = T1 R GEMM
__global__ void k_hi_rvec(const double* __restrict__ site_pos, int n_atoms, double box, int p, int ncp,
                          double* __restrict__ rscratch) {
  // thread per (site atom, order m): the diagonal R_m^m by m complex steps,
  // then the m column (harmonics.py:62-76), written to its packed slots of
  // the block's rows in shared memory; the block's consecutive atoms' rows
  // then leave as one coalesced run.  Block = (atoms per block) x (p + 1).
  extern __shared__ double rv_rows[];  // [atoms per block][ncp]
  const int apb = blockDim.x / (p + 1);
  const int la = threadIdx.x / (p + 1), m = threadIdx.x % (p + 1);
  const int a0 = blockIdx.x * apb, a = a0 + la;
  const int na_blk = min(apb, n_atoms - a0);
  for (int c = threadIdx.x; c < na_blk * ncp; c += blockDim.x) rv_rows[c] = 0.0;  // padding slots stay zero
  __syncthreads();
  if (la < na_blk) {
  const double invL = 1.0 / box;
  const double x = (site_pos[3 * a] - 0.5 * box) * invL, y = (site_pos[3 * a + 1] - 0.5 * box) * invL,
               z = (site_pos[3 * a + 2] - 0.5 * box) * invL;
  const double r2 = x * x + y * y + z * z;
  double* Rt = rv_rows + (size_t)la * ncp;
  double mr = 1.0, mi = 0.0;
  for (int k = 1; k <= m; ++k) {
    const double c = 1.0 / (2.0 * k);
    const double nr = (mr * x - mi * y) * c, ni = (mr * y + mi * x) * c;
    mr = nr;
    mi = ni;
  }
  auto put = [&](int l, double re, double im) {
    if (m == 0) {
      Rt[l] = re;
    } else {
      const int c = pk_index(p, l, m, 0);
      Rt[c] = re;
      Rt[c + 1] = im;
    }
  };
  put(m, mr, mi);
  if (m + 1 <= p) {
    double p2r = mr, p2i = mi, p1r = z * mr, p1i = z * mi;
    put(m + 1, p1r, p1i);
    for (int l = m + 2; l <= p; ++l) {
      const double c = 1.0 / double((l + m) * (l - m));
      const double nr = ((2 * l - 1) * z * p1r - r2 * p2r) * c, ni = ((2 * l - 1) * z * p1i - r2 * p2i) * c;
      p2r = p1r;
      p2i = p1i;
      p1r = nr;
      p1i = ni;
      put(l, nr, ni);
    }
  }
  }
  __syncthreads();
  double* out = rscratch + (size_t)a0 * ncp;
  for (int c = threadIdx.x; c < na_blk * ncp; c += blockDim.x) out[c] = rv_rows[c];
}

// generic U_t = T1 R_t (any ncp): thread per (site atom, output row)
__global__ void k_hi_umat(const double* __restrict__ lat_t, const double* __restrict__ rscratch, int n_atoms,
                          int nc, int ncp, double* __restrict__ uscratch) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n_atoms * ncp) return;
  const int a = (int)(e / ncp), r = (int)(e % ncp);
  const double* R = rscratch + (size_t)a * ncp;
  double acc = 0.0;
  if (r < nc)
    for (int b = 0; b < nc; ++b) acc = fma(lat_t[(size_t)b * ncp + r], R[b], acc);
  uscratch[(size_t)a * ncp + r] = acc;
}

// Lambda forces from the site-atom potentials and the per-form C_rho of a
// corrections-only k_hi_site pass (assemble_lambda_forces, corrections.py:
// 221-238), warp per site; S_rho and the force sums in exactly k_hi_site's
// order, so splitting the HI step this way changes no bit.
__device__ __forceinline__ void hi_lambda_site(const HiArgs& g, int s, int lane) {
  const int a0 = g.atom_off[s], ns = g.atom_off[s + 1] - a0;
  const int nf = g.nforms[s], nl = g.nlam[s];
  const double* Q = g.form_q + g.form_off[s];
  const double* lam = g.lambdas + 4 * s;
  const bool qi = g.mode == 1;
  double f[4] = {0, 0, 0, 0};
  for (int r = 0; r < nf; ++r) {
    double sv = 0.0;
    for (int i = lane; i < ns; i += 32) sv += Q[r * ns + i] * g.pot_site[a0 + i];
    for (int off = 16; off > 0; off >>= 1) sv += __shfl_down_sync(0xffffffffu, sv, off);
    const int slot = g.fslot_off[s] + r;
    const double cv = qi ? 0.0 : (g.c_p2p[slot] + g.c_lat[slot] + g.c_dip[slot]);
    for (int k = 0; k < nl; ++k) f[k] += hi_wgrad(lam, nl, k, r) * (sv - cv);
  }
  if (lane == 0)
    for (int k = 0; k < 4; ++k) g.forces[4 * s + k] = k < nl ? -f[k] : 0.0;
}

// HI spatial forces: spatial_forces(q~) plus -grad Delta E_site on the site
// atoms (sites never share atoms, system.py:139-143, so no two threads add
// to the same row)
__global__ void k_add_site_forces(double* __restrict__ forces, const int* __restrict__ atom_idx, int n_atoms,
                                  const double* __restrict__ site_force) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3 * n_atoms) return;
  const int a = e / 3, k = e - 3 * a;
  const int i = atom_idx[a];
  if (i >= 0) forces[3 * (size_t)i + k] += site_force[e];
}

// fixed-order sum of per-site offsets (CorrectionSet.energy_offset, :153-154)
__global__ void k_sum_offsets(const double* __restrict__ v, int n, double* __restrict__ out) {
  dd acc[1] = {dd{0.0, 0.0}};
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc[0] = dd_add(acc[0], dd_from(v[i]));
  __shared__ dd res[1];
  block_reduce_dd<1>(acc, res);
  if (threadIdx.x == 0) *out = res[0].hi + res[0].lo;
}

// gather caller positions of site atoms from the raw input positions
__global__ void k_gather_site_pos(const double* __restrict__ pos_in, const int* __restrict__ idx, int n,
                                  double* __restrict__ out) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int i = idx[a];
  out[3 * a] = pos_in[3 * i];
  out[3 * a + 1] = pos_in[3 * i + 1];
  out[3 * a + 2] = pos_in[3 * i + 2];
}

// scale_charges (system.py:179-197): copy, then blend site entries
__global__ void k_scale_charges(const double* __restrict__ q_in, int64_t n, double* __restrict__ q_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) q_out[i] = q_in[i];
}
__global__ void k_blend_sites(HiArgs g, double* __restrict__ q_out) {
  const int s = blockIdx.x;
  if (s >= g.n_sites) return;
  const int a0 = g.atom_off[s], ns = g.atom_off[s + 1] - a0;
  const int nf = g.nforms[s], nl = g.nlam[s];
  const double* Q = g.form_q + g.form_off[s];
  const double* lam = g.lambdas + 4 * s;
  for (int t = threadIdx.x; t < ns; t += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < nf; ++r) acc += hi_weight(lam, nl, r) * Q[r * ns + t];
    const int i = g.atom_idx[a0 + t];
    if (i >= 0) q_out[i] = acc;  // < 0: atom held by another rank (distributed.py)
  }
}

}  // namespace lfmm
