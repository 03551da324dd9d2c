// lfmm_expansions.cuh — P2M, L2P(+gradient) and the gathered-GEMM kernel that
// runs every dense translation (M2M, L2L, M2L, lattice).
//
//   P2M  harmonics.particle_multipole (harmonics.py:206-216), upward_pass
//        leaf loop (solver.py:237-247)
//   L2P  harmonics.eval_local / eval_local_grad (harmonics.py:219-234),
//        evaluate / evaluate_gradient (solver.py:294-324)
//   GEMM upward_pass M2M (solver.py:248-258), lattice root (:364-367),
//        downward_pass L2L + offset-grouped M2L (:262-291)
#pragma once
#include "lfmm_common.cuh"
#include "lfmm_tree.cuh"

namespace lfmm {

constexpr int EXP_WARPS = 4;

// ---------------------------------------------------------------- P2M ----
// One warp per leaf, one lane per atom.  Each lane streams q*R^(a/s) into a
// per-warp 32x33 transpose tile; every 32 coefficients the lanes sum one
// column each (fixed order) and accumulate into the leaf's multipole.
template <class T>
__global__ void __launch_bounds__(EXP_WARPS * 32) k_p2m(const vec4_t<T>* __restrict__ xq,
                                                        const int* __restrict__ leaf_start, int depth,
                                                        int p, T inv_size, int ncp,
                                                        T* __restrict__ mult, int x0) {
  __shared__ T buf[EXP_WARPS][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = (x0 << (2 * depth)) + blockIdx.x * EXP_WARPS + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  T* out = mult + (size_t)b * ncp;
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  const int nc = ncoef(p);
  if (t1 == t0) {
    for (int c = lane; c < nc; c += 32) out[c] = T(0);
    return;
  }
  T(*tb)[33] = buf[w];
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    T x = 0, y = 0, z = 0, q = 0;
    if (i < t1) {
      const vec4_t<T> v = xq[i];
      x = v.x * inv_size;
      y = v.y * inv_size;
      z = v.z * inv_size;
      q = v.w;
    }
    const bool first = (tc == t0);
    int col = 0, sbase = 0;
    auto flush = [&]() {
      __syncwarp();
      if (lane < col) {
        T s = T(0);
#pragma unroll 8
        for (int k = 0; k < 32; ++k) s += tb[lane][k];
        const int g = sbase + lane;
        out[g] = first ? s : out[g] + s;
      }
      __syncwarp();
      sbase += col;
      col = 0;
    };
    regular_stream<T>(x, y, z, p, [&](int m, int l, T re, T im) {
      tb[col][lane] = q * re;
      ++col;
      if (col == 32) flush();
      if (m > 0) {
        tb[col][lane] = q * im;
        ++col;
        if (col == 32) flush();
      }
    });
    if (col > 0) flush();
  }
}

// Compile-time-order P2M: the transpose tile columns are static, so the
// recurrence, the tile stores and the column sums fully unroll.
template <class T, int P>
__global__ void __launch_bounds__(EXP_WARPS * 32) k_p2m_c(const vec4_t<T>* __restrict__ xq,
                                                          const int* __restrict__ leaf_start, int depth,
                                                          T inv_size, int ncp, T* __restrict__ mult, int x0) {
  constexpr int NC = (P + 1) * (P + 1);
  constexpr int NF = (NC + 31) / 32;  // flushes of 32 coefficients
  constexpr int TBS = sizeof(T) == 4 ? 36 : 33;  // row stride: 16-B rows (LDS.128) for fp32
  __shared__ __align__(16) T buf[EXP_WARPS][32][TBS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = (x0 << (2 * depth)) + blockIdx.x * EXP_WARPS + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  T* out = mult + (size_t)b * ncp;
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  T(*tb)[TBS] = buf[w];
  T acc[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f] = T(0);
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    T x = 0, y = 0, z = 0, q = 0;
    if (i < t1) {
      const vec4_t<T> v = xq[i];
      x = v.x * inv_size;
      y = v.y * inv_size;
      z = v.z * inv_size;
      q = v.w;
    }
    int col = 0, fl = 0;
    auto flush = [&]() {
      __syncwarp();
      T s = T(0);
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const float4 v = *reinterpret_cast<const float4*>(&tb[lane][k]);
          s += v.x;
          s += v.y;
          s += v.z;
          s += v.w;
        }
      } else {
#pragma unroll 8
        for (int k = 0; k < 32; ++k) s += tb[lane][k];
      }
      if (lane < col) acc[fl] += s;
      __syncwarp();
      ++fl;
      col = 0;
    };
    regular_stream_c<T, P>(
        x, y, z,
        [&](int m, int l, T re, T im) {
          tb[col][lane] = re;
          if (++col == 32) flush();
          if (m > 0) {
            tb[col][lane] = im;
            if (++col == 32) flush();
          }
        },
        q);
    if (col > 0) flush();
  }
#pragma unroll
  for (int f = 0; f < NF; ++f)
    if (f * 32 + lane < NC) out[f * 32 + lane] = acc[f];
}

// ---------------------------------------------------------------- L2P ----
// Warp per leaf.  The leaf local L^ and its three gradient coefficient
// vectors (order p-1, G_x = (L_{j+1}^{k+1} - L_{j+1}^{k-1})/2,
// G_y = i(L_{j+1}^{k+1} + L_{j+1}^{k-1})/2, G_z = L_{j+1}^k — the
// harmonics.regular_grad ladder, harmonics.py:106-130, moved onto the
// coefficients) are staged in shared memory; each lane streams R^(a/s) of
// its atom and contracts.  V = Re sum L R / s, grad V = Re sum G R / s^2.
template <class T>
__device__ __forceinline__ void ld_full(const T* Lh, int p, int l, int m, T& re, T& im) {
  // full-index read of a conj-symmetric packed vector
  if (m == 0) {
    re = Lh[l];
    im = T(0);
  } else if (m > 0) {
    const int a = pk_base(p, m) + 2 * (l - m);
    re = Lh[a];
    im = Lh[a + 1];
  } else {
    const int mm = -m;
    const int a = pk_base(p, mm) + 2 * (l - mm);
    const T s = (mm & 1) ? T(-1) : T(1);
    re = s * Lh[a];
    im = -s * Lh[a + 1];
  }
}

template <class T, bool GRAD>
__global__ void __launch_bounds__(EXP_WARPS * 32) k_l2p(const vec4_t<T>* __restrict__ xq,
                                                        const int* __restrict__ leaf_start, int depth,
                                                        int p, T size, int ncp,
                                                        const T* __restrict__ loc,
                                                        T* __restrict__ vout, T* __restrict__ gout, int x0, int x1) {
  extern __shared__ unsigned char smem_raw[];
  const int nc = ncoef(p), ng = p * p;
  const int per_warp = nc + 3 * ng;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* Lh = reinterpret_cast<T*>(smem_raw) + w * per_warp;
  T* Gx = Lh + nc;
  T* Gy = Gx + ng;
  T* Gz = Gy + ng;
  const int b = (x0 << (2 * depth)) + blockIdx.x * (blockDim.x >> 5) + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  if ((b >> (2 * depth)) < x0 || (b >> (2 * depth)) >= x1) return;  // leaf outside this rank's slab
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  if (t1 == t0) return;
  const T* src = loc + (size_t)b * ncp;
  for (int c = lane; c < nc; c += 32) Lh[c] = src[c];
  __syncwarp();
  if (GRAD) {
    const int q = p - 1;
    for (int a = lane; a < ng; a += 32) {
      int j, k, part;
      pk_decode(q, a, j, k, part);
      T ar, ai, br, bi, cr, ci;
      ld_full(Lh, p, j + 1, k + 1, ar, ai);
      ld_full(Lh, p, j + 1, k - 1, br, bi);
      ld_full(Lh, p, j + 1, k, cr, ci);
      const T gxr = T(0.5) * (ar - br), gxi = T(0.5) * (ai - bi);
      const T gyr = T(-0.5) * (ai + bi), gyi = T(0.5) * (ar + br);
      Gx[a] = part ? gxi : gxr;
      Gy[a] = part ? gyi : gyr;
      Gz[a] = part ? ci : cr;
    }
    __syncwarp();
  }
  const T inv_s = T(1) / size;
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    const bool act = i < t1;
    T x = 0, y = 0, z = 0;
    if (act) {
      const vec4_t<T> v = xq[i];
      x = v.x * inv_s;
      y = v.y * inv_s;
      z = v.z * inv_s;
    }
    T V = 0, dx = 0, dy = 0, dz = 0;
    int a = 0, g = 0;
    regular_stream<T>(x, y, z, p, [&](int m, int l, T re, T im) {
      if (m == 0) {
        V = fma(Lh[a], re, V);
        ++a;
        if (GRAD && l < p) {
          dx = fma(Gx[g], re, dx);
          dy = fma(Gy[g], re, dy);
          dz = fma(Gz[g], re, dz);
          ++g;
        }
      } else {
        V += T(2) * (Lh[a] * re - Lh[a + 1] * im);
        a += 2;
        if (GRAD && l < p) {
          dx += T(2) * (Gx[g] * re - Gx[g + 1] * im);
          dy += T(2) * (Gy[g] * re - Gy[g + 1] * im);
          dz += T(2) * (Gz[g] * re - Gz[g + 1] * im);
          g += 2;
        }
      }
    });
    if (act) {
      vout[i] = V * inv_s;
      if (GRAD) {
        const T s2 = inv_s * inv_s;
        gout[3 * (size_t)i] = dx * s2;
        gout[3 * (size_t)i + 1] = dy * s2;
        gout[3 * (size_t)i + 2] = dz * s2;
      }
    }
  }
}

// Compile-time-order L2P(+gradient): same contraction as k_l2p with static
// shared-memory offsets (broadcast loads) and an unrolled recurrence.
template <class T, bool GRAD, int P>
__global__ void __launch_bounds__(EXP_WARPS * 32) k_l2p_c(const vec4_t<T>* __restrict__ xq,
                                                          const int* __restrict__ leaf_start, int depth,
                                                          T size, int ncp, const T* __restrict__ loc,
                                                          T* __restrict__ vout, T* __restrict__ gout, int x0, int x1) {
  constexpr int NC = (P + 1) * (P + 1), NG = P * P;
  __shared__ T sh[EXP_WARPS][NC + 3 * NG];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* Lh = sh[w];
  T* Gx = Lh + NC;
  T* Gy = Gx + NG;
  T* Gz = Gy + NG;
  const int b = (x0 << (2 * depth)) + blockIdx.x * (blockDim.x >> 5) + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  if ((b >> (2 * depth)) < x0 || (b >> (2 * depth)) >= x1) return;  // leaf outside this rank's slab
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  if (t1 == t0) return;
  const T* src = loc + (size_t)b * ncp;
  for (int c = lane; c < NC; c += 32) Lh[c] = src[c];
  __syncwarp();
  if (GRAD) {
    constexpr int Q = P - 1;
    for (int a = lane; a < NG; a += 32) {
      int j, k, part;
      pk_decode(Q, a, j, k, part);
      T ar, ai, br, bi, cr, ci;
      ld_full(Lh, P, j + 1, k + 1, ar, ai);
      ld_full(Lh, P, j + 1, k - 1, br, bi);
      ld_full(Lh, P, j + 1, k, cr, ci);
      const T gxr = T(0.5) * (ar - br), gxi = T(0.5) * (ai - bi);
      const T gyr = T(-0.5) * (ai + bi), gyi = T(0.5) * (ar + br);
      Gx[a] = part ? gxi : gxr;
      Gy[a] = part ? gyi : gyr;
      Gz[a] = part ? ci : cr;
    }
    __syncwarp();
  }
  const T inv_s = T(1) / size;
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    const bool act = i < t1;
    T x = 0, y = 0, z = 0;
    if (act) {
      const vec4_t<T> v = xq[i];
      x = v.x * inv_s;
      y = v.y * inv_s;
      z = v.z * inv_s;
    }
    T V = 0, dx = 0, dy = 0, dz = 0;
    int a = 0, g = 0;
    regular_stream_c<T, P>(x, y, z, [&](int m, int l, T re, T im) {
      if (m == 0) {
        V = fma(Lh[a], re, V);
        ++a;
        if (GRAD && l < P) {
          dx = fma(Gx[g], re, dx);
          dy = fma(Gy[g], re, dy);
          dz = fma(Gz[g], re, dz);
          ++g;
        }
      } else {
        V += T(2) * (Lh[a] * re - Lh[a + 1] * im);
        a += 2;
        if (GRAD && l < P) {
          dx += T(2) * (Gx[g] * re - Gx[g + 1] * im);
          dy += T(2) * (Gy[g] * re - Gy[g + 1] * im);
          dz += T(2) * (Gz[g] * re - Gz[g + 1] * im);
          g += 2;
        }
      }
    });
    if (act) {
      vout[i] = V * inv_s;
      if (GRAD) {
        const T s2 = inv_s * inv_s;
        gout[3 * (size_t)i] = dx * s2;
        gout[3 * (size_t)i + 1] = dy * s2;
        gout[3 * (size_t)i + 2] = dz * s2;
      }
    }
  }
}

// fp32 L2P(+gradient) on packed pairs: the complex (m > 0) coefficients are
// staged as (2 Re, -2 Im) float2 so each term is one FFMA2 against the
// (Re R, Im R) pair the recurrence produces (also in packed form); real
// m = 0 terms stay scalar.  V = vs + acc.x + acc.y.
// one (l, m > 0) term of k_l2p_f2: potential and, for l <= Q, the gradient
template <bool GRAD>
__device__ __forceinline__ void l2p_term(const float4* SC, int c, bool grad_term, uint64_t q, uint64_t& va,
                                         uint64_t& gxa, uint64_t& gya, uint64_t& gza) {
  const float4 a = SC[2 * c];
  va = f2fma(f2pack(a.x, a.y), q, va);
  if (GRAD && grad_term) {
    const float4 b = SC[2 * c + 1];
    gxa = f2fma(f2pack(a.z, a.w), q, gxa);
    gya = f2fma(f2pack(b.x, b.y), q, gya);
    gza = f2fma(f2pack(b.z, b.w), q, gza);
  }
}

template <bool GRAD, int P>
__global__ void __launch_bounds__(EXP_WARPS * 32) k_l2p_f2(const float4* __restrict__ xq,
                                                           const int* __restrict__ leaf_start, int depth,
                                                           float size, int ncp, const float* __restrict__ loc,
                                                           float* __restrict__ vout, float* __restrict__ gout, int x0, int x1) {
  constexpr int Q = P - 1;
  constexpr int NCC = P * (P + 1) / 2, NQC = Q * (Q + 1) / 2;  // complex coefficients (m > 0)
  // coefficients interleaved per term so that one 16-B shared load feeds
  // two packed FMAs (the term loop was bound by its 8-B loads):
  //   m = 0, order l:  s0[l] = (L, Gx, Gy, Gz)
  //   m > 0, term c:   sc[2c] = (L | Gx), sc[2c + 1] = (Gy | Gz) (complex)
  __shared__ __align__(16) float4 s0[EXP_WARPS][P + 1];
  __shared__ __align__(16) float4 sc[EXP_WARPS][2 * NCC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = (x0 << (2 * depth)) + blockIdx.x * (blockDim.x >> 5) + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  if ((b >> (2 * depth)) < x0 || (b >> (2 * depth)) >= x1) return;  // leaf outside this rank's slab
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  if (t1 == t0) return;
  // first pass's atom, loaded before the staging so both latencies overlap
  float4 vnext = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t0 + lane < t1) vnext = xq[t0 + lane];
  // ---- stage L (one 16-B vector per lane) and build the gradient ladder G
  // (harmonics.py:106-130) from the shared copy ----
  __shared__ __align__(16) float sL[EXP_WARPS][128];
  if (lane * 4 < ncp) reinterpret_cast<float4*>(sL[w])[lane] = reinterpret_cast<const float4*>(loc + (size_t)b * ncp)[lane];
  __syncwarp();
  const float* Lh = sL[w];
  for (int e = lane; e < (P + 1) + NCC; e += 32) {
    if (e <= P) {
      s0[w][e].x = Lh[e];
    } else {
      const int a = (P + 1) + 2 * (e - (P + 1));
      sc[w][2 * (e - (P + 1))].x = 2.f * Lh[a];
      sc[w][2 * (e - (P + 1))].y = -2.f * Lh[a + 1];
    }
  }
  if (GRAD) {
    for (int e = lane; e < (Q + 1) + NQC; e += 32) {
      int j, k;
      if (e <= Q) {
        j = e;
        k = 0;
      } else {  // m-major packed order of the order-Q complex block
        int r = e - (Q + 1);
        k = 1;
        while (r >= Q + 1 - k) {
          r -= Q + 1 - k;
          ++k;
        }
        j = k + r;
      }
      float ar, ai, br, bi, cr, ci;
      ld_full(Lh, P, j + 1, k + 1, ar, ai);
      ld_full(Lh, P, j + 1, k - 1, br, bi);
      ld_full(Lh, P, j + 1, k, cr, ci);
      const float gxr = 0.5f * (ar - br), gxi = 0.5f * (ai - bi);
      const float gyr = -0.5f * (ai + bi), gyi = 0.5f * (ar + br);
      if (e <= Q) {
        s0[w][e].y = gxr;
        s0[w][e].z = gyr;
        s0[w][e].w = cr;
      } else {
        const int c = (k - 1) * (P + 1) - (k - 1) * k / 2 + (j - k);  // (j, k) in the order-P term order
        sc[w][2 * c].z = 2.f * gxr;
        sc[w][2 * c].w = -2.f * gxi;
        sc[w][2 * c + 1] = make_float4(2.f * gyr, -2.f * gyi, 2.f * cr, -2.f * ci);
      }
    }
  }
  __syncwarp();
  const float4* S0 = s0[w];
  const float4* SC = sc[w];
  const float inv_s = 1.f / size;
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    const bool act = i < t1;
    const float4 v = vnext;
    vnext = (tc + 32 + lane < t1) ? xq[tc + 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);  // next pass
    const float x = v.x * inv_s, y = v.y * inv_s, z = v.z * inv_s;
    const float r2 = x * x + y * y + z * z;
    float vs = 0.f, gxs = 0.f, gys = 0.f, gzs = 0.f;
    uint64_t va = 0, gxa = 0, gya = 0, gza = 0;
    // m = 0 column (real)
    {
      float p2 = 1.f, p1 = z;
      {
        const float4 c0 = S0[0];
        vs = fmaf(c0.x, p2, vs);
        if (GRAD) {
          gxs = fmaf(c0.y, p2, gxs);
          gys = fmaf(c0.z, p2, gys);
          gzs = fmaf(c0.w, p2, gzs);
        }
        const float4 c1 = S0[1];
        vs = fmaf(c1.x, p1, vs);
        if (GRAD && 1 <= Q) {
          gxs = fmaf(c1.y, p1, gxs);
          gys = fmaf(c1.z, p1, gys);
          gzs = fmaf(c1.w, p1, gzs);
        }
      }
#pragma unroll
      for (int l = 2; l <= P; ++l) {
        const float c = 1.f / float(l * l);
        const float nv = (float(2 * l - 1) * z * p1 - r2 * p2) * c;
        p2 = p1;
        p1 = nv;
        const float4 cl = S0[l];
        vs = fmaf(cl.x, nv, vs);
        if (GRAD && l <= Q) {
          gxs = fmaf(cl.y, nv, gxs);
          gys = fmaf(cl.z, nv, gys);
          gzs = fmaf(cl.w, nv, gzs);
        }
      }
    }
    // m > 0 columns (packed complex)
    float mr = 1.f, mi = 0.f;
    int ci = 0;
#pragma unroll
    for (int m = 1; m <= P; ++m) {
      const float c = 1.f / float(2 * m);
      const float nr = (mr * x - mi * y) * c, ni = (mr * y + mi * x) * c;
      mr = nr;
      mi = ni;
      uint64_t q2 = f2pack(mr, mi);
      uint64_t q1 = f2mul(q2, f2pack(z, z));
      l2p_term<GRAD>(SC, ci, m <= Q, q2, va, gxa, gya, gza);
      ++ci;
      if (m + 1 <= P) {
        l2p_term<GRAD>(SC, ci, m + 1 <= Q, q1, va, gxa, gya, gza);
        ++ci;
      }
#pragma unroll
      for (int l = m + 2; l <= P; ++l) {
        const float cc = 1.f / float((l + m) * (l - m));
        const float a = float(2 * l - 1) * z * cc, bcoef = -r2 * cc;
        const uint64_t nq = f2fma(q1, f2pack(a, a), f2mul(q2, f2pack(bcoef, bcoef)));
        q2 = q1;
        q1 = nq;
        l2p_term<GRAD>(SC, ci, l <= Q, nq, va, gxa, gya, gza);
        ++ci;
      }
    }
    if (act) {
      float u0, u1;
      f2unpack(va, u0, u1);
      vout[i] = (vs + (u0 + u1)) * inv_s;
      if (GRAD) {
        const float s2 = inv_s * inv_s;
        f2unpack(gxa, u0, u1);
        gout[3 * (size_t)i] = (gxs + (u0 + u1)) * s2;
        f2unpack(gya, u0, u1);
        gout[3 * (size_t)i + 1] = (gys + (u0 + u1)) * s2;
        f2unpack(gza, u0, u1);
        gout[3 * (size_t)i + 2] = (gzs + (u0 + u1)) * s2;
      }
    }
  }
}

// ------------------------------------------------------- gathered GEMM ----
// dst[:, tile] = sum_terms Op_term (ncp x ncp) * src_term[:, gather(tile)]
//
// Modes (one CTA = one job: a tile of up to GB_N target boxes of one level
// and a contiguous range of terms):
//   UP    M2M: terms are the 8 children (solver.py:248-258)
//   ROOT  lattice operator on the root multipole (solver.py:364-367)
//   M2L   terms are the 189 partners of the tile's parity class, in
//         M2L_OFFSETS row order (octree.py:35-38, :96-111); all targets of a
//         tile share one parity, hence one offset list.  The 189 terms are
//         split over `nsplit` CTAs writing partial slots, which keeps the
//         small levels from serialising 189 terms in a single CTA.
//   L2L   one term (parent local, solver.py:276-281); the epilogue adds the
//         level's M2L partial slots in fixed slot order and writes the local.
// Every output element is produced by exactly one thread with a fixed
// summation order: reruns are bit identical.
enum GemmMode { GEMM_UP = 0, GEMM_ROOT = 1, GEMM_M2L = 2, GEMM_L2L = 3 };

constexpr int GB_M = 128, GB_N = 64, G_THREADS = 256;
constexpr int MAX_SPLIT = 16;

struct GemmArgs {
  int mode;
  int ncp;
  int depth;
  const void* mult;   // all levels, box-major, ncp per box
  void* loc;          // all levels
  void* partial;      // M2L partial slots
  const void* ops_m2l;   // [316][ncp][ncp]
  const void* ops_m2l_t; // fp64, ncp == 128: [316][k][row] (k_m2l_f64)
  const void* ops_m2m;   // [8]
  const void* ops_l2l;   // [8]
  const void* ops_lat;   // [1]
  int64_t level_off[DMAX + 2];  // box offset of each level in mult/loc
  int64_t part_off[DMAX + 2];   // vector offset of each level's partial slots
  int nsplit[DMAX + 2];         // partial slots per level (M2L)
  // job decoding for M2L: cumulative job counts per level
  int job_start[DMAX + 3];
  int level;  // UP / L2L / ROOT: the single target level of this launch
  // UP split: the 8 children over `up_split` CTAs writing partial slots
  // (up_part[slot][box]); the last CTA of a tile to finish reduces the slots
  // in fixed order (counter up_cnt[tile], reset by that CTA)
  int up_split;
  void* up_part;
  int* up_cnt;
};

template <class T>
struct GemmTile {
  static constexpr int BK = sizeof(T) == 4 ? 16 : 8;  // keeps smem double buffer < 48 KB
  static constexpr int AK = BK / 2;                    // A elements per thread per stage
  static constexpr int BKT = BK / 4;                   // B elements per thread per stage
};

__host__ __device__ inline int tiles_per_parity(int level) {
  const int sub = 1 << (level - 1);
  return (sub * sub * sub + GB_N - 1) / GB_N;
}
__host__ __device__ inline int tiles_all(int level) { return ((1 << (3 * level)) + GB_N - 1) / GB_N; }

// vector load of N consecutive T (16-B aligned)
template <class T, int N>
__device__ __forceinline__ void ldv(const T* __restrict__ p, T (&r)[N]) {
  constexpr int VW = 16 / sizeof(T);
  static_assert(N % VW == 0, "vector width");
#pragma unroll
  for (int u = 0; u < N / VW; ++u) {
    if constexpr (sizeof(T) == 4) {
      const float4 v = reinterpret_cast<const float4*>(p)[u];
      r[4 * u] = v.x;
      r[4 * u + 1] = v.y;
      r[4 * u + 2] = v.z;
      r[4 * u + 3] = v.w;
    } else {
      const double2 v = reinterpret_cast<const double2*>(p)[u];
      r[2 * u] = v.x;
      r[2 * u + 1] = v.y;
    }
  }
}

// ldv through L2 only (data written by other CTAs of the same launch)
template <class T, int N>
__device__ __forceinline__ void ldv_cg(const T* __restrict__ p, T (&r)[N]) {
  constexpr int VW = 16 / sizeof(T);
  static_assert(N % VW == 0, "vector width");
#pragma unroll
  for (int u = 0; u < N / VW; ++u) {
    if constexpr (sizeof(T) == 4) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(p) + u);
      r[4 * u] = v.x;
      r[4 * u + 1] = v.y;
      r[4 * u + 2] = v.z;
      r[4 * u + 3] = v.w;
    } else {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(p) + u);
      r[2 * u] = v.x;
      r[2 * u + 1] = v.y;
    }
  }
}

// vector store of N consecutive T (16-B aligned)
template <class T, int N>
__device__ __forceinline__ void stv(T* __restrict__ p, const T (&r)[N]) {
  constexpr int VW = 16 / sizeof(T);
  static_assert(N % VW == 0, "vector width");
#pragma unroll
  for (int u = 0; u < N / VW; ++u) {
    if constexpr (sizeof(T) == 4)
      reinterpret_cast<float4*>(p)[u] = make_float4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
    else
      reinterpret_cast<double2*>(p)[u] = make_double2(r[2 * u], r[2 * u + 1]);
  }
}

// box index of the q-th target of parity `par` at `level`
__device__ __forceinline__ int parity_box(int level, int par, int q) {
  const int lsub = level - 1, sub = 1 << lsub;
  const int qx = q >> (2 * lsub), qy = (q >> lsub) & (sub - 1), qz = q & (sub - 1);
  const int gx = 2 * qx + ((par >> 2) & 1), gy = 2 * qy + ((par >> 1) & 1), gz = 2 * qz + (par & 1);
  return (gx << (2 * level)) | (gy << level) | gz;
}

template <class T>
__global__ void __launch_bounds__(G_THREADS) k_gemm_gather(GemmArgs g) {
  constexpr int BK = GemmTile<T>::BK, AK = GemmTile<T>::AK, BKT = GemmTile<T>::BKT;
  // fp64 runs on the DMMA pipe (mma.sync m8n8k4): rows padded by 8 doubles so
  // a fragment load (4 k-rows x 8 consecutive elements) touches every bank
  // exactly twice
  constexpr bool DMMA = sizeof(T) == 8;
  constexpr int APAD = DMMA ? 8 : 0;
  __shared__ __align__(16) T As[2][BK][GB_M + APAD];
  __shared__ __align__(16) T Bs[2][BK][GB_N + APAD];
  __shared__ int col_dst[GB_N];
  const int tid = threadIdx.x;
  const int ncp = g.ncp;
  const int row0 = blockIdx.y * GB_M;

  // ---- decode the job ----
  int level = g.level, par = 0, t0 = 0, t1 = 1, slot = -1;
  if (g.mode == GEMM_M2L) {
    level = 1;
    while (level < g.depth && (int)blockIdx.x >= g.job_start[level + 1]) ++level;
    const int j = blockIdx.x - g.job_start[level];
    const int ns = g.nsplit[level];
    const int tpp = tiles_per_parity(level);
    slot = j % ns;
    const int tile = j / ns;
    par = tile / tpp;
    const int q0 = (tile % tpp) * GB_N;
    const int sub = 1 << (level - 1);
    if (tid < GB_N) col_dst[tid] = (q0 + tid < sub * sub * sub) ? parity_box(level, par, q0 + tid) : -1;
    t0 = (NM2L * slot) / ns;
    t1 = (NM2L * (slot + 1)) / ns;
  } else if (g.mode == GEMM_L2L) {
    const int tpp = tiles_per_parity(level);
    par = blockIdx.x / tpp;
    const int q0 = (blockIdx.x % tpp) * GB_N;
    const int sub = 1 << (level - 1);
    if (tid < GB_N) col_dst[tid] = (q0 + tid < sub * sub * sub) ? parity_box(level, par, q0 + tid) : -1;
  } else if (g.mode == GEMM_UP) {
    const int ns = g.up_split;
    slot = blockIdx.x % ns;
    const int q0 = (blockIdx.x / ns) * GB_N;
    if (tid < GB_N) col_dst[tid] = (q0 + tid < (1 << (3 * level))) ? q0 + tid : -1;
    t0 = (8 * slot) / ns;
    t1 = (8 * (slot + 1)) / ns;
  } else {  // ROOT
    if (tid < GB_N) col_dst[tid] = tid == 0 ? 0 : -1;
  }
  __syncthreads();

  const int nside = 1 << level, msk = nside - 1;
  const int nk = ncp / BK;
  const int niter = (t1 - t0) * nk;

  // loader mapping (conflict-free smem stores): A: 128 consecutive rows per
  // k-group, B: 64 consecutive target columns per k-group
  const int a_row = tid & (GB_M - 1), a_k = (tid >> 7) * AK;
  const int b_col = tid & (GB_N - 1), b_k = (tid >> 6) * BKT;
  // compute mapping: 16 x 16 threads, 8 rows (two groups of 4) x 4 columns
  const int ty = tid >> 4, tx = tid & 15;

  // SIMT (fp32): acc[i][j] = D[row i of the thread's 8][col tx*4+j].  DMMA
  // (fp64): warp w owns rows (w & 3)*32.., cols (w >> 2)*32..; acc[2*mt +
  // (nt >> 1)][2*(nt & 1) + e] = D[mt*8 + lane/4][nt*8 + 2*(lane%4) + e]
  T acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  const int lane = tid & 31, wm = (tid >> 5) & 3, wn = tid >> 7;

  T ra[AK], rb[BKT];
  const T* Ab = nullptr;
  const T* Bb = nullptr;
  int cur_term = -1, my_src = -1;
  const int tgt = col_dst[b_col];
  const T* mult = reinterpret_cast<const T*>(g.mult);
  const T* loc = reinterpret_cast<const T*>(g.loc);

  auto term_setup = [&](int term) {
    int src_box = -1;
    if (g.mode == GEMM_M2L) {
      const char4 o = c_m2l_off[par * NM2L + term];
      const int row = c_m2l_row[par * NM2L + term];
      Ab = reinterpret_cast<const T*>(g.ops_m2l) + (size_t)row * ncp * ncp;
      Bb = mult + g.level_off[level] * ncp;
      if (tgt >= 0) {
        const int gx = tgt >> (2 * level), gy = (tgt >> level) & msk, gz = tgt & msk;
        src_box = ((((gx + o.x) & msk) << level | ((gy + o.y) & msk)) << level) | ((gz + o.z) & msk);
      }
    } else if (g.mode == GEMM_L2L) {
      Ab = reinterpret_cast<const T*>(g.ops_l2l) + (size_t)par * ncp * ncp;
      Bb = loc + g.level_off[level - 1] * ncp;
      if (tgt >= 0) {
        const int pl = level - 1;
        const int gx = (tgt >> (2 * level)) >> 1, gy = ((tgt >> level) & msk) >> 1, gz = (tgt & msk) >> 1;
        src_box = (gx << (2 * pl)) | (gy << pl) | gz;
      }
    } else if (g.mode == GEMM_UP) {
      Ab = reinterpret_cast<const T*>(g.ops_m2m) + (size_t)term * ncp * ncp;
      Bb = mult + g.level_off[level + 1] * ncp;
      if (tgt >= 0) {
        const int cl = level + 1;
        const int gx = tgt >> (2 * level), gy = (tgt >> level) & msk, gz = tgt & msk;
        const int cx = 2 * gx + ((term >> 2) & 1), cy = 2 * gy + ((term >> 1) & 1), cz = 2 * gz + (term & 1);
        src_box = (cx << (2 * cl)) | (cy << cl) | cz;
      }
    } else {
      Ab = reinterpret_cast<const T*>(g.ops_lat);
      Bb = mult;
      if (tgt >= 0) src_box = 0;
    }
    return src_box;
  };

  auto load_regs = [&](int it) {
    const int tl = it / nk, kc = it - tl * nk;
    const int term = t0 + tl;
    if (term != cur_term) {
      my_src = term_setup(term);
      cur_term = term;
    }
    const int k0 = kc * BK;
    const int r = row0 + a_row;
    if (r < ncp) {
      ldv<T, AK>(Ab + (size_t)r * ncp + k0 + a_k, ra);
    } else {
#pragma unroll
      for (int u = 0; u < AK; ++u) ra[u] = T(0);
    }
    if (my_src >= 0) {
      ldv<T, BKT>(Bb + (size_t)my_src * ncp + k0 + b_k, rb);
    } else {
#pragma unroll
      for (int u = 0; u < BKT; ++u) rb[u] = T(0);
    }
  };
  auto store_smem = [&](int buf) {
#pragma unroll
    for (int u = 0; u < AK; ++u) As[buf][a_k + u][a_row] = ra[u];
#pragma unroll
    for (int u = 0; u < BKT; ++u) Bs[buf][b_k + u][b_col] = rb[u];
  };

  if (niter > 0) {
    load_regs(0);
    store_smem(0);
  }
  __syncthreads();
  for (int it = 0; it < niter; ++it) {
    const int buf = it & 1;
    if (it + 1 < niter) load_regs(it + 1);
    if constexpr (DMMA) {
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          af[u] = As[buf][ks + (lane & 3)][wm * 32 + u * 8 + (lane >> 2)];
          bf[u] = Bs[buf][ks + (lane & 3)][wn * 32 + u * 8 + (lane >> 2)];
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            double& d0 = reinterpret_cast<double&>(acc[2 * mt + (nt >> 1)][2 * (nt & 1)]);
            double& d1 = reinterpret_cast<double&>(acc[2 * mt + (nt >> 1)][2 * (nt & 1) + 1]);
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d0), "+d"(d1)
                         : "d"(af[mt]), "d"(bf[nt]));
          }
      }
    } else {
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[8], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[buf][k][ty * 4 + u];
        a[4 + u] = As[buf][k][64 + ty * 4 + u];
        bv[u] = Bs[buf][k][tx * 4 + u];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
    }
    }
    if (it + 1 < niter) store_smem(buf ^ 1);
    __syncthreads();
  }

  // ---- epilogue, staged through shared memory so that every global
  // access (partial slots, outputs) is a coalesced run along the coefficients
  T* out;
  size_t out_base;
  const size_t nbox_l = (size_t)1 << (3 * level);
  if (g.mode == GEMM_M2L) {
    out = reinterpret_cast<T*>(g.partial);
    out_base = (size_t)(g.part_off[level] + (int64_t)slot * nbox_l);
  } else if (g.mode == GEMM_UP && g.up_split > 1) {
    out = reinterpret_cast<T*>(g.up_part);
    out_base = (size_t)slot * nbox_l;
  } else if (g.mode == GEMM_UP) {
    out = const_cast<T*>(mult);
    out_base = (size_t)g.level_off[level];
  } else {
    out = reinterpret_cast<T*>(g.loc);
    out_base = (size_t)g.level_off[level];
  }
  const T* part = reinterpret_cast<const T*>(g.partial);
  const int nsl = (g.mode == GEMM_L2L) ? g.nsplit[level] : 0;
  T* stage = &As[0][0][0];
  constexpr int CC = (2 * BK * GB_M) / GB_M;  // columns per pass
#pragma unroll 1
  for (int c0 = 0; c0 < GB_N; c0 += CC) {
    if constexpr (DMMA) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int mt = i >> 1, nt = 2 * (i & 1) + (j >> 1), e = j & 1;
          const int col = wn * 32 + nt * 8 + 2 * (lane & 3) + e - c0;
          const int r = wm * 32 + mt * 8 + (lane >> 2);
          if (col >= 0 && col < CC) stage[col * GB_M + r] = acc[i][j];
        }
    } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = tx * 4 + j - c0;
      if (col < 0 || col >= CC) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        stage[col * GB_M + r] = acc[i][j];
      }
    }
    }
    __syncthreads();
    for (int e = tid; e < CC * GB_M; e += G_THREADS) {
      const int col = e / GB_M, rr = e % GB_M, r = row0 + rr;
      const int box = col_dst[c0 + col];
      if (box < 0 || r >= ncp) continue;
      T v = stage[e];
      for (int s2 = 0; s2 < nsl; ++s2)  // M2L partial slots, fixed order
        v += part[((size_t)g.part_off[level] + (size_t)s2 * nbox_l + box) * ncp + r];
      out[(out_base + box) * ncp + r] = v;
    }
    __syncthreads();
  }
  if (g.mode == GEMM_UP && g.up_split > 1) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    const int tile = blockIdx.x / g.up_split;
    if (tid == 0) {
      const int old = atomicAdd(&g.up_cnt[tile * gridDim.y + blockIdx.y], 1);
      last = (old == g.up_split - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const T* up = reinterpret_cast<const T*>(g.up_part);
      T* dst = const_cast<T*>(mult) + (size_t)g.level_off[level] * ncp;
      for (int e = tid; e < GB_N * GB_M; e += G_THREADS) {
        const int col = e / GB_M, r = row0 + e % GB_M;
        const int box = col_dst[col];
        if (box < 0 || r >= ncp) continue;
        T v = T(0);
        for (int s2 = 0; s2 < g.up_split; ++s2) v += __ldcg(up + ((size_t)s2 * nbox_l + box) * ncp + r);
        dst[(size_t)box * ncp + r] = v;
      }
      if (tid == 0) g.up_cnt[tile * gridDim.y + blockIdx.y] = 0;
    }
  }
}

// fp64 M2L (ncp == 128) on the DMMA pipe with a cp.async ring: the same jobs
// as k_gemm_gather's GEMM_M2L (a tile of 64 same-parity targets x a slice of
// the 189 terms, one partial slot), K streamed in 16-deep chunks through a
// 4-stage ring so three chunks are in flight while one is multiplied.
// A = the term's operator, stored transposed ([k][row]) so a chunk is 16
// contiguous 1-KB rows; B = the 64 targets' source multipoles, one 128-B run
// per column (zero-filled for padding columns).  Warp tiles 32 x 32 of
// mma.sync m8n8k4.f64; every output is one thread's fixed-order sum.
#ifndef LFMM_F64_BK
#define LFMM_F64_BK 16
#endif
#ifndef LFMM_F64_S
#define LFMM_F64_S 4
#endif
#ifndef LFMM_F64_MINB
#define LFMM_F64_MINB 2
#endif
constexpr int F64_BK = LFMM_F64_BK, F64_S = LFMM_F64_S, F64_AP = GB_M + 8, F64_BP = F64_BK + 4;
constexpr int F64_STAGE = F64_BK * F64_AP + GB_N * F64_BP;  // doubles per stage
constexpr size_t F64_SMEM = (size_t)F64_S * F64_STAGE * sizeof(double);

__device__ __forceinline__ void cp16_zfill(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(G_THREADS, LFMM_F64_MINB) k_m2l_f64(GemmArgs g) {
  extern __shared__ __align__(16) double f64_smem[];
  __shared__ int col_dst[GB_N];
  const int tid = threadIdx.x, lane = tid & 31, wm = (tid >> 5) & 3, wn = tid >> 7;
  int level = 1;
  while (level < g.depth && (int)blockIdx.x >= g.job_start[level + 1]) ++level;
  const int j = blockIdx.x - g.job_start[level];
  const int ns = g.nsplit[level];
  const int tpp = tiles_per_parity(level);
  const int slot = j % ns, tile = j / ns;
  const int par = tile / tpp, q0 = (tile % tpp) * GB_N;
  const int sub = 1 << (level - 1);
  if (tid < GB_N) col_dst[tid] = (q0 + tid < sub * sub * sub) ? parity_box(level, par, q0 + tid) : -1;
  const int t0 = (NM2L * slot) / ns, t1 = (NM2L * (slot + 1)) / ns;
  __syncthreads();
  const int msk = (1 << level) - 1;
  const int nk = 128 / F64_BK;
  const int niter = (t1 - t0) * nk;
  const double* mult = reinterpret_cast<const double*>(g.mult) + g.level_off[level] * 128;
  const double* ops_t = reinterpret_cast<const double*>(g.ops_m2l_t);
  // this thread's B pieces: column n = c / (BK / 2), 16-B piece u = c % (BK / 2)
  int bt[F64_BK / 8];
#pragma unroll
  for (int h = 0; h < F64_BK / 8; ++h) bt[h] = col_dst[(tid + h * G_THREADS) / (F64_BK / 2)];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(f64_smem);

  auto load = [&](int it, int st) {
    const int term = t0 + it / nk, k0 = (it % nk) * F64_BK;
    const char4 o = c_m2l_off[par * NM2L + term];
    const int row = c_m2l_row[par * NM2L + term];
    const double* A = ops_t + ((size_t)row * 128 + k0) * 128;
    const uint32_t sa = sbase + (uint32_t)(st * F64_STAGE) * 8u;
    const uint32_t sb = sa + (uint32_t)(F64_BK * F64_AP) * 8u;
#pragma unroll
    for (int h = 0; h < F64_BK / 4; ++h) {  // A: F64_BK k-rows x 64 pieces
      const int c = tid + h * G_THREADS, kr = c >> 6, pc = c & 63;
      cp16_zfill(sa + (uint32_t)(kr * F64_AP + 2 * pc) * 8u, A + kr * 128 + 2 * pc, true);
    }
#pragma unroll
    for (int h = 0; h < F64_BK / 8; ++h) {  // B: 64 columns x F64_BK / 2 pieces
      const int c = tid + h * G_THREADS, n = c / (F64_BK / 2), u = c % (F64_BK / 2);
      const int t = bt[h];
      int src = 0;
      if (t >= 0) {
        const int gx = t >> (2 * level), gy = (t >> level) & msk, gz = t & msk;
        src = ((((gx + o.x) & msk) << level | ((gy + o.y) & msk)) << level) | ((gz + o.z) & msk);
      }
      cp16_zfill(sb + (uint32_t)(n * F64_BP + 2 * u) * 8u, mult + (size_t)src * 128 + k0 + 2 * u, t >= 0);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < F64_S - 1; ++s) {
    if (s < niter) load(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < niter; ++it) {
    asm volatile("cp.async.wait_group %0;" ::"n"(F64_S - 2) : "memory");
    __syncthreads();
    const double* As = f64_smem + (size_t)(it % F64_S) * F64_STAGE;
    const double* Bs = As + F64_BK * F64_AP;
#pragma unroll
    for (int ks = 0; ks < F64_BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        af[u] = As[(ks + (lane & 3)) * F64_AP + wm * 32 + u * 8 + (lane >> 2)];
        bf[u] = Bs[(wn * 32 + u * 8 + (lane >> 2)) * F64_BP + ks + (lane & 3)];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(af[mt]), "d"(bf[nt]));
    }
    if (it + F64_S - 1 < niter) load(it + F64_S - 1, (it + F64_S - 1) % F64_S);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // ---- epilogue: stage D column-major through shared memory, then every
  // partial-slot write is a coalesced run along the coefficients ----
  double* stage = f64_smem;  // 64 x 128 doubles = 64 KB < F64_SMEM
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + nt * 8 + 2 * (lane & 3) + e, r = wm * 32 + mt * 8 + (lane >> 2);
        stage[col * GB_M + r] = acc[mt][nt][e];
      }
  __syncthreads();
  const size_t nbox_l = (size_t)1 << (3 * level);
  double* out = reinterpret_cast<double*>(g.partial) + ((size_t)g.part_off[level] + (size_t)slot * nbox_l) * 128;
  for (int e = tid; e < GB_N * GB_M; e += G_THREADS) {
    const int box = col_dst[e / GB_M];
    if (box >= 0) out[(size_t)box * 128 + (e % GB_M)] = stage[e];
  }
}

// dst[:, j] = A src[:, j] for ncols contiguous 128-double columns, fp64 on
// the DMMA pipe (the HI lattice product U = T1 R over all site atoms): the
// k_m2l_f64 tile and ring with one operator (A transposed, [k][row]).
__global__ void __launch_bounds__(G_THREADS, LFMM_F64_MINB) k_cols_f64(const double* __restrict__ ops_t,
                                                                      const double* __restrict__ src,
                                                                      double* __restrict__ dst, int ncols) {
  extern __shared__ __align__(16) double f64_smem[];
  const int tid = threadIdx.x, lane = tid & 31, wm = (tid >> 5) & 3, wn = tid >> 7;
  const int c0 = blockIdx.x * GB_N;
  const int nk = 128 / F64_BK;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(f64_smem);
  auto load = [&](int it, int st) {
    const int k0 = it * F64_BK;
    const uint32_t sa = sbase + (uint32_t)(st * F64_STAGE) * 8u;
    const uint32_t sb = sa + (uint32_t)(F64_BK * F64_AP) * 8u;
#pragma unroll
    for (int h = 0; h < F64_BK / 4; ++h) {
      const int c = tid + h * G_THREADS, kr = c >> 6, pc = c & 63;
      cp16_zfill(sa + (uint32_t)(kr * F64_AP + 2 * pc) * 8u, ops_t + (size_t)(k0 + kr) * 128 + 2 * pc, true);
    }
#pragma unroll
    for (int h = 0; h < F64_BK / 8; ++h) {
      const int c = tid + h * G_THREADS, n = c / (F64_BK / 2), u = c % (F64_BK / 2);
      const bool ok = c0 + n < ncols;
      cp16_zfill(sb + (uint32_t)(n * F64_BP + 2 * u) * 8u, src + (size_t)(ok ? c0 + n : 0) * 128 + k0 + 2 * u, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < F64_S - 1; ++s) {
    if (s < nk) load(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < nk; ++it) {
    asm volatile("cp.async.wait_group %0;" ::"n"(F64_S - 2) : "memory");
    __syncthreads();
    const double* As = f64_smem + (size_t)(it % F64_S) * F64_STAGE;
    const double* Bs = As + F64_BK * F64_AP;
#pragma unroll
    for (int ks = 0; ks < F64_BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        af[u] = As[(ks + (lane & 3)) * F64_AP + wm * 32 + u * 8 + (lane >> 2)];
        bf[u] = Bs[(wn * 32 + u * 8 + (lane >> 2)) * F64_BP + ks + (lane & 3)];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(af[mt]), "d"(bf[nt]));
    }
    if (it + F64_S - 1 < nk) load(it + F64_S - 1, (it + F64_S - 1) % F64_S);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double* stage = f64_smem;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + nt * 8 + 2 * (lane & 3) + e, r = wm * 32 + mt * 8 + (lane >> 2);
        stage[col * GB_M + r] = acc[mt][nt][e];
      }
  __syncthreads();
  for (int e = tid; e < GB_N * GB_M; e += G_THREADS) {
    const int col = c0 + e / GB_M;
    if (col < ncols) dst[(size_t)col * 128 + (e % GB_M)] = stage[e];
  }
}

}  // namespace lfmm

namespace lfmm {

// ---------------------------------------------------- M2M / L2L sweeps ----
// One CTA = (tile of TR_PT target columns, octant o): D = Op_o (ncp x ncp)
// x B (ncp x TR_PT) over the whole K = ncp, K streamed through shared memory
// in TR_KC chunks with cp.async double buffering.  Operators are stored
// transposed ([k][row]) so a K chunk is one contiguous block.
//   UP  (M2M, upward_pass solver.py:248-258): parent tile p, octant o:
//       B = child(p, o) multipoles; D goes to partial slot o; the last of the
//       8 octant CTAs of a tile adds the slots in octant order (fixed-order,
//       deterministic) and writes the parent multipoles.
//   DOWN (L2L, downward_pass solver.py:276-281): parent tile p, octant o:
//       B = parent locals; child(p, o) local = D + the level's M2L partial
//       slots in slot order.
// 256 threads: lane -> 4 consecutive rows (coefficients), warp -> 2 columns.
constexpr int TR_KC = 32, TR_THREADS = 256;  // columns per CTA: 8 warps x CPW (template)

struct TrArgs {
  int mode;            // 0 UP (M2M), 1 DOWN (L2L), 2 plain columns (dst[:, c] = Op src[:, c])
  int ncols;           // mode 2: number of columns
  int level;           // UP: parent level; DOWN: child level
  int ncp;
  const void* ops_t;   // [8][ncp (k)][ncp (row)]
  const void* src;     // UP: child-level multipoles; DOWN: parent-level locals
  void* dst;           // UP: parent-level multipoles; DOWN: child-level locals
  void* slots;         // UP: [8][nparents][ncp] scratch
  int* cnt;            // UP: one counter per tile
  const void* partial; // DOWN: M2L partial slots of the child level ([nsplit][nchild][ncp])
  int nsplit;
  int p0, pend;        // UP/DOWN: parent columns [p0, pend) (pend == 0: the whole level; a
                       // slab decomposition restricts the owned levels to its x-slab)
};

template <class T>
__device__ __forceinline__ void tr_cp16(T* sdst, const T* gsrc) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}

template <class T, int CPW, int NS>
__global__ void __launch_bounds__(TR_THREADS) k_translate(TrArgs g) {
  constexpr int VW = 16 / sizeof(T);  // elements per 16-B copy
  constexpr int PT = 8 * CPW;         // target columns per CTA (8 warps x CPW)
  extern __shared__ __align__(16) unsigned char tr_smem[];
  T* As = reinterpret_cast<T*>(tr_smem);              // [NS][TR_KC][ncp]
  const int ncp = g.ncp;
  T* Bs = As + NS * TR_KC * ncp;                       // [NS][PT][TR_KC]
  __shared__ int col_src[PT], col_dst[PT];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int o = blockIdx.y;
  const int tile = blockIdx.x;
  const int pl = g.mode == 0 ? g.level : g.level - 1;  // parent level
  const int np = 1 << (3 * pl), pn = 1 << pl, cn = 2 * pn;
  if (tid < PT) {
    const int p = g.p0 + tile * PT + tid;
    int s = -1, d = -1;
    if (g.mode == 2) {
      if (p < g.ncols) s = d = p;
    } else if (p < (g.pend ? g.pend : np)) {
      const int px = p >> (2 * pl), py = (p >> pl) & (pn - 1), pz = p & (pn - 1);
      const int c = ((((2 * px + ((o >> 2) & 1)) * cn) + 2 * py + ((o >> 1) & 1)) * cn) + 2 * pz + (o & 1);
      if (g.mode == 0) {
        s = c;
        d = p;
      } else {
        s = p;
        d = c;
      }
    }
    col_src[tid] = s;
    col_dst[tid] = d;
  }
  __syncthreads();
  const T* ops = reinterpret_cast<const T*>(g.ops_t) + (size_t)o * ncp * ncp;
  const T* src = reinterpret_cast<const T*>(g.src);
  const int nk = ncp / TR_KC;
  auto stage = [&](int kc, int buf) {
    T* a = As + (size_t)buf * TR_KC * ncp;
    const T* ga = ops + (size_t)kc * TR_KC * ncp;
    for (int e = tid; e < TR_KC * ncp / VW; e += TR_THREADS) tr_cp16(a + e * VW, ga + e * VW);
    T* b = Bs + (size_t)buf * PT * TR_KC;
    for (int e = tid; e < PT * TR_KC / VW; e += TR_THREADS) {
      const int c = e / (TR_KC / VW), u = e % (TR_KC / VW);
      const int sb = col_src[c];
      if (sb >= 0)
        tr_cp16(b + c * TR_KC + u * VW, src + (size_t)sb * ncp + kc * TR_KC + u * VW);
      else
#pragma unroll
        for (int v = 0; v < VW; ++v) b[c * TR_KC + u * VW + v] = T(0);
    }
  };
  T acc[4][CPW];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < CPW; ++j) acc[i][j] = T(0);
  const int r0 = 4 * lane;  // rows r0..r0+3 (the plan routes only ncp == 128 here)
  // NS-stage cp.async ring: NS - 1 chunks in flight ahead of the one in use
  // (small levels use NS = nk: the whole K extent is requested at once)
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) stage(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + NS - 1 < nk) stage(kc + NS - 1, (kc + NS - 1) % NS);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
    __syncthreads();
    const T* a = As + (size_t)(kc % NS) * TR_KC * ncp;
    const T* b = Bs + (size_t)(kc % NS) * PT * TR_KC + (size_t)(CPW * w) * TR_KC;
#pragma unroll 2
    for (int k = 0; k < TR_KC; k += 4) {
      T av[4][4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ldv<T, 4>(a + (k + kk) * ncp + r0, av[kk]);
#pragma unroll
      for (int j = 0; j < CPW; ++j) {
        T bv[4];
        ldv<T, 4>(b + j * TR_KC + k, bv);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u][j] = fma(av[kk][u], bv[kk], acc[u][j]);
      }
    }
    __syncthreads();
  }
  // ---- epilogue ----
  if (g.mode == 2) {
    T* dst = reinterpret_cast<T*>(g.dst);
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int d = col_dst[CPW * w + j];
      if (d < 0) continue;
      T v4[4] = {acc[0][j], acc[1][j], acc[2][j], acc[3][j]};
      stv<T, 4>(dst + (size_t)d * ncp + r0, v4);
    }
  } else if (g.mode == 0) {
    T* slots = reinterpret_cast<T*>(g.slots);
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int d = col_dst[CPW * w + j];
      if (d < 0) continue;
      T v4[4] = {acc[0][j], acc[1][j], acc[2][j], acc[3][j]};
      stv<T, 4>(slots + ((size_t)o * np + d) * ncp + r0, v4);
    }
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = (atomicAdd(&g.cnt[tile], 1) == 7);
    __syncthreads();
    if (!last) return;
    __threadfence();
    T* dst = reinterpret_cast<T*>(g.dst);
    // 4-row vectors, two per thread per round: 16 independent loads in flight
    const int nv = PT * ncp / 4;
    for (int e0 = tid; e0 < nv; e0 += 2 * TR_THREADS) {
      T q[2][8][4];
      int dd[2], rr[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = e0 + u * TR_THREADS;
        dd[u] = e < nv ? col_dst[e / (ncp / 4)] : -1;
        rr[u] = 4 * (e % (ncp / 4));
        if (dd[u] >= 0)
#pragma unroll
          for (int s = 0; s < 8; ++s) ldv_cg<T, 4>(slots + ((size_t)s * np + dd[u]) * ncp + rr[u], q[u][s]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (dd[u] < 0) continue;
        T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int s = 0; s < 8; ++s)
#pragma unroll
          for (int x = 0; x < 4; ++x) v[x] += q[u][s][x];
        stv<T, 4>(dst + (size_t)dd[u] * ncp + rr[u], v);
      }
    }
    if (tid == 0) g.cnt[tile] = 0;
  } else {
    const T* part = reinterpret_cast<const T*>(g.partial);
    T* dst = reinterpret_cast<T*>(g.dst);
    const size_t nchild = (size_t)np * 8;
    // M2L partial slots added in fixed slot order; all CPW columns of one
    // slot loaded together (loads issued before any store)
    int dcol[CPW];
#pragma unroll
    for (int j = 0; j < CPW; ++j) dcol[j] = col_dst[CPW * w + j];
    for (int s = 0; s < g.nsplit; ++s) {
      T q4[CPW][4];
#pragma unroll
      for (int j = 0; j < CPW; ++j)
        if (dcol[j] >= 0) ldv<T, 4>(part + ((size_t)s * nchild + dcol[j]) * ncp + r0, q4[j]);
#pragma unroll
      for (int j = 0; j < CPW; ++j)
        if (dcol[j] >= 0)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u][j] += q4[j][u];
    }
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      if (dcol[j] < 0) continue;
      T v4[4] = {acc[0][j], acc[1][j], acc[2][j], acc[3][j]};
      stv<T, 4>(dst + (size_t)dcol[j] * ncp + r0, v4);
    }
  }
}

}  // namespace lfmm
