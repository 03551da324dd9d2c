// lfmm_tree.cuh — uniform periodic octree on the device, bit-exact with
// octree.build_octree (fmm/octree.py:114-163):
//   wrap    : np.mod(x, L), then x >= L -> 0          (system.py:103-108)
//   cell    : clip(int64(x / (L / 2^d)), 0, 2^d - 1)    (octree.py:121-123)
//   leaf    : (ix*n + iy)*n + iz                        (octree.py:48-49)
//   order   : lexsort((z, y, x, leaf)) — leaf, x, y, z, then input index
//             (numpy's lexsort is stable)               (octree.py:125)
// Counting sort into leaf buckets (integer atomics only: the histogram is
// order independent), then a per-leaf rank sort on the full fp64 key makes
// the canonical permutation independent of scheduling.
#pragma once
#include "lfmm_common.cuh"

namespace lfmm {

// numpy float remainder (npy_divmod): fmod, shifted into the divisor's sign,
// and +0.0 for an exact zero.
__device__ __forceinline__ double np_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0.0) != (m < 0.0)) m += b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}

// wrap_positions (system.py:103-108): np.mod(x, L), then x >= L -> 0.  The
// common case 0 <= x < L is fmod's identity (and +0.0 for either zero).
__device__ __forceinline__ double wrap_coord(double x, double box) {
  const double w = (x >= 0.0 && x < box) ? x + 0.0 : np_mod(x, box);
  return w >= box ? 0.0 : w;
}
// all three coordinates, the in-box case without any fmod code on its path
__device__ __forceinline__ void wrap_xyz(const double* p, double box, double& x, double& y, double& z) {
  x = p[0];
  y = p[1];
  z = p[2];
  if (x >= 0.0 && x < box && y >= 0.0 && y < box && z >= 0.0 && z < box) {
    x += 0.0;
    y += 0.0;
    z += 0.0;
  } else {
    x = wrap_coord(x, box);
    y = wrap_coord(y, box);
    z = wrap_coord(z, box);
  }
}

// The wrapped coordinates are not stored (one 24 MB write less per
// rebuild): k_leaf_rank recomputes them from the raw positions (wrap_coord);
// only the wrapped x rounded to fp32, its fast-path sort key, is kept.
// pos_copy (device-resident caller positions): also written to pos_copy,
// the plan's copy of the raw positions (one pass instead of a memcpy first)
__global__ void k_wrap_cell(const double* __restrict__ pos_in, int64_t n, double box, double size,
                            int depth, int* __restrict__ leaf_of,
                            int* __restrict__ counts, int* __restrict__ slot_of, double* __restrict__ pos_copy,
                            float* __restrict__ key32) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = i < n;
  const int nside = 1 << depth;
  int leaf = -1;
  if (ok) {
    int cell[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x = pos_in[3 * i + a];
      if (pos_copy) pos_copy[3 * i + a] = x;
      const double w = wrap_coord(x, box);
      if (a == 0) key32[i] = (float)w;  // k_leaf_rank's fast-path sort key
      double t = w / size;  // IEEE division, like positions / size
      long long c = (long long)t;  // astype(int64): truncation
      c = c < 0 ? 0 : (c > nside - 1 ? nside - 1 : c);
      cell[a] = (int)c;
    }
    leaf = (cell[0] * nside + cell[1]) * nside + cell[2];
    leaf_of[i] = leaf;
  }
  // the counter's old value is the atom's slot in its leaf bucket (bucket
  // order is arbitrary: k_leaf_rank orders each leaf by the exact key); one
  // atomic per distinct leaf of the warp (neighbouring atoms share leaves)
  const unsigned act = __ballot_sync(0xffffffffu, ok);
  if (!ok) return;
  const unsigned peers = __match_any_sync(act, leaf);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&counts[leaf], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  slot_of[i] = base + __popc(peers & ((1u << lane) - 1u));
}

// Exclusive scan of one block's values (warp shuffles, then the warp totals).
__device__ __forceinline__ int block_scan_excl(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  total = warp_tot[nw - 1];
  const int base = w > 0 ? warp_tot[w - 1] : 0;
  return base + x - v;
}

// One block (1024 threads) scans all n leaf counts in tiles of 8 x 1024:
// each thread loads 8 consecutive counts (two int4, coalesced across the
// warp), the block scans the per-thread sums, and a running carry links the
// tiles (one launch instead of block scans + total scan + add; n = 32,768 at
// depth 5: 4 tiles, 262,144 at depth 6: 32 tiles).  n is a multiple of 8.
__global__ void __launch_bounds__(1024) k_scan_single(const int* __restrict__ counts, int n,
                                                      int* __restrict__ start) {
  __shared__ int wt[32];
  if (n & 7) {  // depth 0: one leaf
    if (threadIdx.x == 0) {
      int run = 0;
      for (int i = 0; i < n; ++i) {
        start[i] = run;
        run += counts[i];
      }
      start[n] = run;
    }
    return;
  }
  const int tile = blockDim.x * 8;
  int carry = 0;
  for (int base = 0; base < n; base += tile) {
    const int i0 = base + 8 * threadIdx.x;
    int4 a = make_int4(0, 0, 0, 0), b = make_int4(0, 0, 0, 0);
    if (i0 < n) {
      a = reinterpret_cast<const int4*>(counts + i0)[0];
      b = reinterpret_cast<const int4*>(counts + i0)[1];
    }
    const int sum = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
    int total;
    int ex = carry + block_scan_excl(sum, wt, total);
    if (i0 < n) {
      int4 oa, ob;
      oa.x = ex;
      oa.y = oa.x + a.x;
      oa.z = oa.y + a.y;
      oa.w = oa.z + a.z;
      ob.x = oa.w + a.w;
      ob.y = ob.x + b.x;
      ob.z = ob.y + b.y;
      ob.w = ob.z + b.z;
      reinterpret_cast<int4*>(start + i0)[0] = oa;
      reinterpret_cast<int4*>(start + i0)[1] = ob;
    }
    carry += total;
    __syncthreads();  // wt is reused by the next tile's scan
  }
  if (threadIdx.x == 0) start[n] = carry;
}

// Multi-block exclusive scan with decoupled look-back: block b scans 4096
// counts (8 per thread, two int4), publishes its aggregate, then takes the
// prefix of the blocks before it from their published aggregates / inclusive
// prefixes (status zeroed before the launch; the grid is at most a few dozen
// blocks, all resident, so the waits cannot starve).  Same result as
// k_scan_single (integer sums), one launch of n / 4096 blocks.
constexpr int SCAN_THREADS = 512, SCAN_TILE = 8 * SCAN_THREADS;
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(const int* __restrict__ counts, int n,
                                                                int* __restrict__ start,
                                                                unsigned long long* __restrict__ status) {
  __shared__ int wt[32];
  __shared__ int s_prefix;
  const int b = blockIdx.x;
  const int i0 = b * SCAN_TILE + 8 * threadIdx.x;
  int4 a = make_int4(0, 0, 0, 0), c = make_int4(0, 0, 0, 0);
  if (i0 < n) {
    a = reinterpret_cast<const int4*>(counts + i0)[0];
    c = reinterpret_cast<const int4*>(counts + i0)[1];
  }
  const int sum = a.x + a.y + a.z + a.w + c.x + c.y + c.z + c.w;
  int total;
  const int ex = block_scan_excl(sum, wt, total);
  if (threadIdx.x == 0) {
    volatile unsigned long long* st = status;
    int prefix = 0;
    if (b == 0) {
      st[0] = (2ull << 32) | (unsigned)total;
    } else {
      st[b] = (1ull << 32) | (unsigned)total;
      for (int j = b - 1; j >= 0; --j) {
        unsigned long long v;
        do {
          v = st[j];
        } while ((v >> 32) == 0);
        prefix += (int)(unsigned)v;
        if ((v >> 32) == 2) break;
      }
      __threadfence();
      st[b] = (2ull << 32) | (unsigned)(prefix + total);
    }
    s_prefix = prefix;
    if (b == gridDim.x - 1) start[n] = prefix + total;
  }
  __syncthreads();
  if (i0 < n) {
    int4 oa, ob;
    oa.x = s_prefix + ex;
    oa.y = oa.x + a.x;
    oa.z = oa.y + a.y;
    oa.w = oa.z + a.z;
    ob.x = oa.w + a.w;
    ob.y = ob.x + c.x;
    ob.z = ob.y + c.y;
    ob.w = ob.z + c.z;
    reinterpret_cast<int4*>(start + i0)[0] = oa;
    reinterpret_cast<int4*>(start + i0)[1] = ob;
  }
}

__global__ void k_scatter_leaf(const int* __restrict__ leaf_of, int64_t n, const int* __restrict__ start,
                               const int* __restrict__ slot_of, int* __restrict__ bucket) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bucket[start[leaf_of[i]] + slot_of[i]] = (int)i;
}

__device__ __forceinline__ bool key_less(double ax, double ay, double az, int ai, double bx, double by,
                                         double bz, int bi) {
  if (ax != bx) return ax < bx;
  if (ay != by) return ay < by;
  if (az != bz) return az < bz;
  return ai < bi;
}

// One warp per leaf: rank of every bucket entry under (x, y, z, index).
// Fast path: x rounded to fp32 is monotone, so x32_j < x32_i (or >) decides
// the fp64 order; the rank is the count of strictly smaller x32 in the leaf,
// read as shared-memory broadcasts.  If any lane sees an x32 tie with another
// entry (rare: fp32 resolves ~1e-6 nm), the warp recomputes that pass with
// the exact (x, y, z, index) comparison, keys broadcast by shuffles.
// The ranked entry also writes its canonical-order arrays (fp64 sorted
// positions, leaf-relative coordinates x - c_leaf with c_leaf = (grid + 0.5)
// size (octree.py:65-66) in T, leaf index), which it holds in registers.
constexpr int RANK_WARPS = 4;
template <class T>
__global__ void __launch_bounds__(RANK_WARPS * 32) k_leaf_rank(const double* __restrict__ pos, double box,
                                                              const float* __restrict__ key32,
                                                              const int* __restrict__ start,
                                                              const int* __restrict__ bucket, int nleaf,
                                                              int* __restrict__ perm, int* __restrict__ inv_perm,
                                                              int depth, double size, double* __restrict__ pos_sorted,
                                                              vec4_t<T>* __restrict__ xq,
                                                              int* __restrict__ leaf_sorted, float4* __restrict__ pa,
                                                              float4* __restrict__ pb) {
  __shared__ float kx[RANK_WARPS][32];
  const int wl = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nleaf) return;
  const int s0 = start[warp], s1 = start[warp + 1];
  for (int e0 = s0; e0 < s1; e0 += 32) {
    const int e = e0 + lane;
    int i = -1;
    double x = 0, y = 0, z = 0;
    if (e < s1) {
      i = bucket[e];
      wrap_xyz(pos + 3 * (size_t)i, box, x, y, z);
    }
    const float x32 = (float)x;
    int rank = 0, eq = 0;
    for (int f0 = s0; f0 < s1; f0 += 32) {
      const int f = f0 + lane;
      __syncwarp();
      kx[wl][lane] = f < s1 ? key32[bucket[f]] : 0.f;
      __syncwarp();
      const int cnt = min(32, s1 - f0);
      for (int k = 0; k < cnt; ++k) {
        const float xj = kx[wl][k];
        rank += xj < x32;
        eq += xj == x32;
      }
    }
    if (__any_sync(0xffffffffu, e < s1 && eq > 1)) {
      rank = 0;
      for (int f0 = s0; f0 < s1; f0 += 32) {
        const int f = f0 + lane;
        int jf = -1;
        double xf = 0, yf = 0, zf = 0;
        if (f < s1) {
          jf = bucket[f];
          wrap_xyz(pos + 3 * (size_t)jf, box, xf, yf, zf);
        }
        const int cnt = min(32, s1 - f0);
        for (int k = 0; k < cnt; ++k) {
          const int j = __shfl_sync(0xffffffffu, jf, k);
          const double xj = __shfl_sync(0xffffffffu, xf, k), yj = __shfl_sync(0xffffffffu, yf, k),
                       zj = __shfl_sync(0xffffffffu, zf, k);
          rank += key_less(xj, yj, zj, j, x, y, z, i);
        }
      }
    }
    if (e < s1) {
      const int k = s0 + rank;
      perm[k] = i;
      inv_perm[i] = k;
      const int nside = 1 << depth, msk = nside - 1;
      const int leaf = warp;
      pos_sorted[3 * (size_t)k] = x;
      pos_sorted[3 * (size_t)k + 1] = y;
      pos_sorted[3 * (size_t)k + 2] = z;
      vec4_t<T> v;
      v.x = (T)(x - ((leaf >> (2 * depth)) + 0.5) * size);
      v.y = (T)(y - (((leaf >> depth) & msk) + 0.5) * size);
      v.z = (T)(z - ((leaf & msk) + 0.5) * size);
      v.w = T(0);
      xq[k] = v;
      leaf_sorted[k] = leaf;
      if (pa) {  // fp32 source pairs for k_p2p2 (charges written by k_stage_q)
        const int pp = ((s0 + leaf + 1) >> 1) + (rank >> 1), h = rank & 1;
        reinterpret_cast<float*>(pa + pp)[h] = (float)v.x;
        reinterpret_cast<float*>(pa + pp)[2 + h] = (float)v.y;
        reinterpret_cast<float*>(pb + pp)[h] = (float)v.z;
      }
    }
  }
  // odd leaf: the last pair's second half is a far, chargeless pad
  if (pa && lane == 0 && ((s1 - s0) & 1)) {
    const int pp = ((s0 + warp + 1) >> 1) + ((s1 - s0) >> 1);
    reinterpret_cast<float*>(pa + pp)[1] = 1.0e4f;
    reinterpret_cast<float*>(pa + pp)[3] = 1.0e4f;
    reinterpret_cast<float*>(pb + pp)[1] = 1.0e4f;
    reinterpret_cast<float*>(pb + pp)[3] = 0.f;
  }
}

// Neighbour enumeration shared by P2P and the list export (octree.py:136-139):
// row t of NEIGHBOR_OFFSETS is ((t/9)-1, (t/3)%3-1, t%3-1).
__host__ __device__ inline void neighbor(int b, int t, int depth, int& nb, int& shx, int& shy, int& shz) {
  const int nside = 1 << depth, msk = nside - 1;
  const int bx = b >> (2 * depth), by = (b >> depth) & msk, bz = b & msk;
  const int rx = bx + t / 9 - 1, ry = by + (t / 3) % 3 - 1, rz = bz + t % 3 - 1;
  // floor_divide by a power of two == arithmetic shift
  shx = rx >> depth;
  shy = ry >> depth;
  shz = rz >> depth;
  nb = (((rx & msk) << depth | (ry & msk)) << depth) | (rz & msk);
}

__global__ void k_export_nb(int depth, int64_t* __restrict__ nb_box, int64_t* __restrict__ nb_shift) {
  const int nleaf = 1 << (3 * depth);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nleaf * 27) return;
  const int b = idx / 27, t = idx % 27;
  int nb, sx, sy, sz;
  neighbor(b, t, depth, nb, sx, sy, sz);
  if (nb_box) nb_box[idx] = nb;
  if (nb_shift) {
    nb_shift[3 * idx] = sx;
    nb_shift[3 * idx + 1] = sy;
    nb_shift[3 * idx + 2] = sz;
  }
}

// M2L partner of target box b at level l, slot s (0..188), as the M2L
// kernels gather it: sources = wrap(grid + offset) (octree.py:109).
__device__ __forceinline__ int m2l_source(int b, int s, int level, int& row) {
  const int nside = 1 << level, msk = nside - 1;
  const int gx = b >> (2 * level), gy = (b >> level) & msk, gz = b & msk;
  const int par = ((gx & 1) << 2) | ((gy & 1) << 1) | (gz & 1);
  const char4 o = c_m2l_off[par * NM2L + s];
  row = c_m2l_row[par * NM2L + s];
  return ((((gx + o.x) & msk) << level | ((gy + o.y) & msk)) << level) | ((gz + o.z) & msk);
}

__global__ void k_export_m2l(int level, int64_t* __restrict__ src, int64_t* __restrict__ rows) {
  const int nbox = 1 << (3 * level);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nbox * NM2L) return;
  int row;
  const int s = m2l_source(idx / NM2L, idx % NM2L, level, row);
  if (src) src[idx] = s;
  if (rows) rows[idx] = row;
}

}  // namespace lfmm
