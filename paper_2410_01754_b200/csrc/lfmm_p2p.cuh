// lfmm_p2p.cuh — near field: potentials and gradients from the 27 periodic
// neighbour images (fmm/solver.py:126-224, numba loop :166-195).
//
// One warp per target leaf, one lane per target atom; source atoms of each
// neighbour image are staged 32 at a time in a per-warp shared tile as
// (x,y,z,q) vectors (one 16-B (fp32) / 32-B (fp64) load per atom) and
// broadcast to the lanes.  Coordinates are leaf-relative: for target leaf
// b and neighbour offset o, disp = a_i - (a_j + o*size), which equals the
// reference x_i - x_j - shift*L (the image centre of the wrapped neighbour is
// c_b + o*size) while keeping every fp32 coordinate below 1.5 leaf edges.
// Potential and gradient come from the same pair pass; the home-image self
// pair (same box, zero shift, j == i) is skipped exactly like :182-189.
#pragma once
#include "lfmm_common.cuh"
#include "lfmm_tree.cuh"

namespace lfmm {

constexpr int P2P_WARPS = 4;

template <class T, bool GRAD, bool SELF>
__device__ __forceinline__ void p2p_tile(const vec4_t<T>* __restrict__ tile, int cnt, int jbase, int i,
                                         T xi, T yi, T zi, T& v, T& gx, T& gy, T& gz) {
#pragma unroll 4
  for (int jj = 0; jj < cnt; ++jj) {
    const vec4_t<T> s = tile[jj];
    const T dx = xi - s.x, dy = yi - s.y, dz = zi - s.z;
    const T r2 = dx * dx + dy * dy + dz * dz;
    T inv = rsqrt_t(r2);
    if (SELF) inv = (jbase + jj == i) ? T(0) : inv;
    const T qi = s.w * inv;
    v += qi;
    if (GRAD) {
      const T q3 = qi * inv * inv;
      gx = fma(dx, q3, gx);
      gy = fma(dy, q3, gy);
      gz = fma(dz, q3, gz);
    }
  }
}

template <class T, bool GRAD>
__global__ void __launch_bounds__(P2P_WARPS * 32) k_p2p(const vec4_t<T>* __restrict__ xq,
                                                        const int* __restrict__ leaf_start, int depth,
                                                        T size, int periodic, T* __restrict__ vout,
                                                        T* __restrict__ gout) {
  __shared__ vec4_t<T> tiles[P2P_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * P2P_WARPS + w;
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  vec4_t<T>* tile = tiles[w];
  const int t0 = leaf_start[b], t1 = leaf_start[b + 1];
  const int tlo = periodic ? 0 : 13, thi = periodic ? 27 : 14;
  for (int tc = t0; tc < t1; tc += 32) {
    const int i = tc + lane;
    const bool act = i < t1;
    vec4_t<T> me;
    if (act) me = xq[i];
    else me.x = me.y = me.z = me.w = T(0);
    T v = 0, gx = 0, gy = 0, gz = 0;
    for (int t = tlo; t < thi; ++t) {
      int nb, sx, sy, sz;
      neighbor(b, t, depth, nb, sx, sy, sz);
      const T ox = T(t / 9 - 1) * size, oy = T((t / 3) % 3 - 1) * size, oz = T(t % 3 - 1) * size;
      const int s0 = leaf_start[nb], s1 = leaf_start[nb + 1];
      for (int sc = s0; sc < s1; sc += 32) {
        const int j = sc + lane;
        vec4_t<T> s;
        if (j < s1) {
          s = xq[j];
          s.x += ox;
          s.y += oy;
          s.z += oz;
        } else {
          s.x = s.y = s.z = T(1);
          s.w = T(0);
        }
        __syncwarp();
        tile[lane] = s;
        __syncwarp();
        const int cnt = min(32, s1 - sc);
        if (t == 13)
          p2p_tile<T, GRAD, true>(tile, cnt, sc, i, me.x, me.y, me.z, v, gx, gy, gz);
        else
          p2p_tile<T, GRAD, false>(tile, cnt, sc, i, me.x, me.y, me.z, v, gx, gy, gz);
      }
    }
    if (act) {
      vout[i] = v;
      if (GRAD) {  // grad V = -sum q d / r^3
        gout[3 * (size_t)i] = -gx;
        gout[3 * (size_t)i + 1] = -gy;
        gout[3 * (size_t)i + 2] = -gz;
      }
    }
  }
}

}  // namespace lfmm
