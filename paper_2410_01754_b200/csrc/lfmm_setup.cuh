// lfmm_setup.cuh — plan-time construction of every translation operator on
// the device, in the packed normalised form the hot kernels consume.
//
//   M2L  harmonics.m2l_from_irregular (harmonics.py:143-152, :196-203) on
//        irregular(o, 2p) of the 316 unit offsets (solver.py:120-123)
//   M2M  harmonics.m2m_matrix (harmonics.py:133-159), d=(0.5-oct)*child.size
//        (solver.py:251)
//   L2L  harmonics.l2l_matrix (harmonics.py:162-166), d=(oct-0.5)*size
//        (solver.py:278)
//   lattice converged_operator (lattice.py:124-155) / shell_sum_operator
//        (lattice.py:109-121), unit box; scaled() (lattice.py:95-100) is the
//        identity in normalised form.
//
// "Realification": a complex operator O acting on conjugate-symmetric
// vectors is turned into the real (p+1)^2 x (p+1)^2 matrix acting on the
// packed layout (lfmm_common.cuh).  For input (j,k>0):
//   Re part  -> O[:,(j,k)] + (-1)^k O[:,(j,-k)]
//   Im part  -> i (O[:,(j,k)] - (-1)^k O[:,(j,-k)])
// and the output row takes Re / Im of Y_(n,mu), mu >= 0.
#pragma once
#include "lfmm_common.cuh"

namespace lfmm {

enum OpKind { OP_M2L = 0, OP_M2M = 1, OP_L2L = 2, OP_DENSE = 3 };

// full complex entry O[(n,mu),(j,k)] of operator `kind`
__device__ inline double2 op_entry(int kind, const double2* __restrict__ v, int p, int n, int mu, int j,
                                   int k) {
  if (kind == OP_M2L) {
    // B[(n,mu),(j,k)] = (-1)^(j+mu+k) I_{n+j}^{-(mu+k)}     (harmonics.py:143-152)
    const int L = n + j, M = -(mu + k);
    if (M < -L || M > L) return make_double2(0.0, 0.0);  // never for |mu|<=n, |k|<=j
    const double2 iv = v[cidx(L, M)];
    const double s = ((j + mu + k) & 1) ? -1.0 : 1.0;
    return make_double2(s * iv.x, s * iv.y);
  }
  if (kind == OP_M2M) {
    // A[(l,m),(j,k)] = R_{l-j}^{m-k}(-d), |m-k| <= l-j   (harmonics.py:133-159)
    const int dl = n - j, dm = mu - k;
    if (dl < 0 || dm < -dl || dm > dl) return make_double2(0.0, 0.0);
    return v[cidx(dl, dm)];
  }
  if (kind == OP_L2L) {
    // C = gather(R(d))^T: C[(n,mu),(j,k)] = R_{j-n}^{k-mu}(d)
    const int dl = j - n, dm = k - mu;
    if (dl < 0 || dm < -dl || dm > dl) return make_double2(0.0, 0.0);
    return v[cidx(dl, dm)];
  }
  // dense complex (nc x nc, row-major)
  return v[(size_t)cidx(n, mu) * ncoef(p) + cidx(j, k)];
}

// out[mat][a][b] (ncp x ncp, zero padded) for mat in [0, nmat)
//   scale: out_pow^(l_a + out_add) * in_pow^(l_b)
template <class T>
__global__ void k_realify(int kind, int p, int nmat, const double2* __restrict__ data, int64_t data_stride,
                          double out_pow, int out_add, double in_pow, T* __restrict__ out, int ncp) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)ncp * ncp;
  if (idx >= per * nmat) return;
  const int mat = (int)(idx / per);
  const int a = (int)((idx % per) / ncp), b = (int)(idx % ncp);
  const int nc = ncoef(p);
  if (a >= nc || b >= nc) {
    out[idx] = T(0);
    return;
  }
  const double2* v = data + (size_t)mat * data_stride;
  int n, mu, pa, j, k, pb;
  pk_decode(p, a, n, mu, pa);
  pk_decode(p, b, j, k, pb);
  double2 y;
  if (k == 0) {
    y = op_entry(kind, v, p, n, mu, j, 0);
  } else {
    const double2 c1 = op_entry(kind, v, p, n, mu, j, k);
    const double2 c2 = op_entry(kind, v, p, n, mu, j, -k);
    const double s = (k & 1) ? -1.0 : 1.0;
    if (pb == 0)
      y = make_double2(c1.x + s * c2.x, c1.y + s * c2.y);
    else
      y = make_double2(-(c1.y - s * c2.y), c1.x - s * c2.x);
  }
  double val = pa ? y.y : y.x;
  val *= pow(out_pow, double(n + out_add)) * pow(in_pow, double(j));
  out[idx] = (T)val;
}

// irregular / regular harmonics of a list of vectors, full complex layout
__global__ void k_harmonics_full(const double* __restrict__ vecs, int nvec, int order, int irregular,
                                 double2* __restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvec) return;
  const int stride = ncoef(order);
  if (irregular)
    irregular_full(vecs[3 * v], vecs[3 * v + 1], vecs[3 * v + 2], order, out + (size_t)v * stride);
  else
    regular_full(vecs[3 * v], vecs[3 * v + 1], vecs[3 * v + 2], order, out + (size_t)v * stride);
}

// acc[c] += sum_v vals[v][c], fixed order over v (deterministic)
__global__ void k_sum_vectors(const double2* __restrict__ vals, int nvec, int ncoefs, double2* __restrict__ acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncoefs) return;
  double2 s = acc[c];
  for (int v = 0; v < nvec; ++v) {
    const double2 x = vals[(size_t)v * ncoefs + c];
    s.x += x.x;
    s.y += x.y;
  }
  acc[c] = s;
}

// dense complex operator (nc x nc) from a vector, kind M2L (order-2p irregular
// sum) or M2M (order-p regular sum); optional row scaling 3^-l (S_hat)
__global__ void k_dense_from_vector(int kind, const double2* __restrict__ v, int p, double row_pow,
                                    double2* __restrict__ out) {
  const int nc = ncoef(p);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nc * nc) return;
  const int r = idx / nc, c = idx % nc;
  const int n = (int)sqrt((double)r), j = (int)sqrt((double)c);
  const int mu = r - n * n - n, k = c - j * j - j;
  double2 e = op_entry(kind, v, p, n, mu, j, k);
  const double sc = pow(row_pow, double(n));
  out[idx] = make_double2(e.x * sc, e.y * sc);
}

// C = A @ B, complex row-major n x n (setup only)
__global__ void k_zgemm(const double2* __restrict__ A, const double2* __restrict__ B, double2* __restrict__ C,
                        int n) {
  __shared__ double2 As[16][17], Bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double cr = 0.0, ci = 0.0;
  for (int k0 = 0; k0 < n; k0 += 16) {
    As[ty][tx] = (row < n && k0 + tx < n) ? A[(size_t)row * n + k0 + tx] : make_double2(0.0, 0.0);
    Bs[ty][tx] = (k0 + ty < n && col < n) ? B[(size_t)(k0 + ty) * n + col] : make_double2(0.0, 0.0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 a = As[ty][k], b = Bs[k][tx];
      cr += a.x * b.x - a.y * b.y;
      ci += a.x * b.y + a.y * b.x;
    }
    __syncthreads();
  }
  if (row < n && col < n) C[(size_t)row * n + col] = make_double2(cr, ci);
}

// total += diag(3^(-k(n+1))) * P   (telescoping step, lattice.py:150-151)
__global__ void k_lattice_accum(double2* __restrict__ total, const double2* __restrict__ P, int p, int kstep) {
  const int nc = ncoef(p);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nc * nc) return;
  const int n = (int)sqrt((double)(idx / nc));
  const double sc = pow(3.0, -double(kstep) * (n + 1.0));
  total[idx].x += sc * P[idx].x;
  total[idx].y += sc * P[idx].y;
}

// zero entries with l_row + l_col < min_order (converged mode: keep >= 4),
// then symmetrise 0.5 (T + T^T)  (lattice.py:103-106, :154)
__global__ void k_lattice_finish(const double2* __restrict__ in, double2* __restrict__ out, int p, int min_order) {
  const int nc = ncoef(p);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nc * nc) return;
  const int r = idx / nc, c = idx % nc;
  const int lr = (int)sqrt((double)r), lc = (int)sqrt((double)c);
  double2 a = in[idx], b = in[(size_t)c * nc + r];
  if (lr + lc < min_order) {
    a = make_double2(0.0, 0.0);
    b = a;
  }
  out[idx] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
}

__global__ void k_identity(double2* __restrict__ m, int n) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  m[idx] = make_double2((idx / n) == (idx % n) ? 1.0 : 0.0, 0.0);
}

}  // namespace lfmm
