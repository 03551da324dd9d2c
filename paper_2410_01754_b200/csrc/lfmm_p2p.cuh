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
#include "lfmm_sm100.cuh"
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
                                                        T* __restrict__ gout, int x0, int x1) {
  __shared__ vec4_t<T> tiles[P2P_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = (x0 << (2 * depth)) + blockIdx.x * P2P_WARPS + w;  // grid from the rank's first leaf plane
  const int nleaf = 1 << (3 * depth);
  if (b >= nleaf) return;
  if ((b >> (2 * depth)) < x0 || (b >> (2 * depth)) >= x1) return;  // leaf outside this rank's slab
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


// ------------------------------------------------------------------------
// fp32 near field on packed f32x2 arithmetic (FADD2/FMUL2/FFMA2, sm_100).
//
// One warp per target leaf.  The leaf's whole 27-image neighbourhood is
// staged once in shared memory, shifted into the target leaf's frame, as
// pairs of sources in SoA form (x_k, x_k+1, y_k, y_k+1 | z_k, z_k+1, q_k,
// q_k+1), so one lane processes two sources per step with packed
// instructions (two MUFU.RSQ).  Staged order: the home image first (the only
// one where the self pair can occur, masked there), then the 26 others.
// Lane use: a leaf's targets run in passes of up to 32; a pass with r < 32
// targets splits the sources over P = 2^k <= 32 / r lane groups, which are
// reduced with xor shuffles at the end (keeps ~91% of lanes busy on water,
// where leaves hold 9..55 atoms).  Neighbourhoods longer than one staging
// buffer are processed in chunks.  Every output is the sum of a fixed
// sequence of operations: reruns are bit identical.
#ifndef LFMM_P2P2_WARPS
#define LFMM_P2P2_WARPS 4
#endif
#ifndef LFMM_P2P2_MINB
#define LFMM_P2P2_MINB 5  // <= 102 registers: 5 CTAs (20 warps) per SM; measured 0.525 vs 0.543 ms at 4 CTAs
#endif
#ifndef LFMM_P2P2_SMAX
#define LFMM_P2P2_SMAX 512
#endif
constexpr int P2P2_WARPS = LFMM_P2P2_WARPS;
constexpr int P2P2_SMAX = LFMM_P2P2_SMAX;  // staged sources per warp and chunk (even): 32 KB per CTA, 6 CTAs/SM
constexpr int P2P2_SMEM = P2P2_WARPS * P2P2_SMAX * 16;  // dynamic shared memory per CTA

__device__ __forceinline__ float rsqrt_fast(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// two sources (pair index k) against one target; MASK: zero the pair halves
// whose staged index equals `self`
template <bool GRAD, bool MASK>
__device__ __forceinline__ void p2p2_step(const float4* __restrict__ A, const float4* __restrict__ B, int k,
                                          uint64_t x2, uint64_t y2, uint64_t z2, int self, uint64_t& v2,
                                          uint64_t& gx2, uint64_t& gy2, uint64_t& gz2) {
  const float4 a = A[k], b = B[k];
  const uint64_t dx = f2sub(x2, f2pack(a.x, a.y));
  const uint64_t dy = f2sub(y2, f2pack(a.z, a.w));
  const uint64_t dz = f2sub(z2, f2pack(b.x, b.y));
  uint64_t r2 = f2mul(dx, dx);
  r2 = f2fma(dy, dy, r2);
  r2 = f2fma(dz, dz, r2);
  float ra, rb;
  f2unpack(r2, ra, rb);
  float ia = rsqrt_fast(ra), ib = rsqrt_fast(rb);
  if (MASK) {
    ia = (2 * k == self) ? 0.f : ia;
    ib = (2 * k + 1 == self) ? 0.f : ib;
  }
  const uint64_t inv = f2pack(ia, ib);
  const uint64_t qi = f2mul(f2pack(b.z, b.w), inv);
  v2 = f2add(v2, qi);
  if (GRAD) {
    const uint64_t q3 = f2mul(qi, f2mul(inv, inv));
    gx2 = f2fma(dx, q3, gx2);
    gy2 = f2fma(dy, q3, gy2);
    gz2 = f2fma(dz, q3, gz2);
  }
}

// The potential is summed in two levels: blocks of <= 32 pair terms into a
// fresh fp32 partial, partials into a Kahan-compensated total.  A leaf's
// ~1800 terms summed into one fp32 running sum leave ~1e-5 absolute error,
// which small near-neutral systems turn into ~3e-4 relative energy error (the
// reference's "single" mode rounds only once per stage, solver.py:95-102).
__device__ __forceinline__ void kahan_fold(uint64_t& v2, uint64_t& c2, uint64_t p2) {
  const uint64_t y = f2sub(p2, c2);
  const uint64_t t = f2add(v2, y);
  c2 = f2sub(f2sub(t, v2), y);
  v2 = t;
}

// One target leaf b for the calling warp (staging buffers A/B, per-warp
// tables, mbarrier `bar` whose parity `phase` carries over between leaves).
template <bool GRAD>
__device__ __forceinline__ void p2p2_leaf(int b, const float4* __restrict__ xq, const float4* __restrict__ pair_a,
                                          const float4* __restrict__ pair_b, const int* __restrict__ leaf_start,
                                          int depth, float size, int periodic, float* __restrict__ vout,
                                          float* __restrict__ gout, float4* A, float4* B, int2* s_imgw,
                                          float4* s_shiftw, unsigned char* s_imgof, uint32_t bar,
                                          uint32_t& phase) {
  const int lane = threadIdx.x & 31;
  const int t0 = leaf_start[b], n = leaf_start[b + 1] - t0;
  if (n == 0) return;
  // images: lane t < nimg holds image t (home = lane 0): its leaf's first
  // source pair, pair count, shift into the target leaf's frame
  const int nimg = periodic ? 27 : 1;
  int i_pair = 0, i_np = 0;
  float i_ox = 0.f, i_oy = 0.f, i_oz = 0.f;
  if (lane < nimg) {
    // lane 0 = home image (row 13); lanes 1..26 = rows 0..12, 14..26
    const int t = (lane == 0 || !periodic) ? 13 : (lane <= 13 ? lane - 1 : lane);
    int nb, sx, sy, sz;
    neighbor(b, t, depth, nb, sx, sy, sz);
    const int st = leaf_start[nb];
    i_pair = (st + nb + 1) >> 1;  // leaf nb's pairs (lfmm_tree.cuh k_leaf_rank)
    i_np = (leaf_start[nb + 1] - st + 1) >> 1;
    i_ox = (float)(t / 9 - 1) * size;
    i_oy = (float)((t / 3) % 3 - 1) * size;
    i_oz = (float)(t % 3 - 1) * size;
  }
  // staged pair offsets: home [0, hp), the others packed after it
  const int hp = (n + 1) >> 1;
  int excl = i_np;  // inclusive scan of pair counts over the images
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, excl, o);
    if (lane >= o) excl += y;
  }
  const int i_off = excl - i_np;                        // staged pair offset of my image
  const int tp = __shfl_sync(0xffffffffu, excl, 31);  // total staged pairs
  if (lane < nimg) {
    s_imgw[lane] = make_int2(i_off, i_np);
    s_shiftw[lane] = make_float4(i_ox, i_oy, i_oz, 0.f);
  }
  if (lane == nimg) s_imgw[lane] = make_int2(0x7fffffff, 0);
  constexpr int CH = P2P2_SMAX / 2;  // pairs per staging chunk
  const int nchunk = (tp + CH - 1) / CH;
  __syncwarp();

  for (int pb = 0; pb < n; pb += 32) {
    const int nt = min(32, n - pb);
    int P = 1;
    while (P < 32 && nt * (2 * P) <= 32) P *= 2;
    const int lp = __ffs(P) - 1;  // P = 2^lp: shifts, not integer divisions
    const int W = 32 >> lp, slot = lane & (W - 1), part = lane >> (5 - lp);
    const bool act = slot < nt;
    const int ti = t0 + pb + (act ? slot : 0);
    const float4 me = xq[ti];
    const uint64_t x2 = f2pack(me.x, me.x), y2 = f2pack(me.y, me.y), z2 = f2pack(me.z, me.z);
    const int self = pb + slot;  // staged index of my target in the home block
    uint64_t v2 = 0, c2 = 0, gx2 = 0, gy2 = 0, gz2 = 0;
    for (int c = 0; c < nchunk; ++c) {
      const int cb = c * CH, ce = min(tp, cb + CH);  // pairs [cb, ce)
      if (nchunk > 1 || pb == 0) {
        // ---- stage pairs [cb, ce): one bulk copy per image and half (TMA
        // engine, no registers), then the images' frame shifts in place ----
        __syncwarp();  // every lane is done reading the previous contents
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"((uint32_t)(ce - cb) * 32u)
                       : "memory");
        __syncwarp();
        {
          const int lo = max(i_off, cb), hi = min(i_off + i_np, ce);
          if (lane < nimg && hi > lo) {
            const uint32_t bytes = (uint32_t)(hi - lo) * 16u;
            const int src = i_pair + (lo - i_off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(A + (lo - cb))),
                "l"(pair_a + src), "r"(bytes), "r"(bar)
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(B + (lo - cb))),
                "l"(pair_b + src), "r"(bytes), "r"(bar)
                : "memory");
          }
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        if (nimg > 1) {
          // each image lane marks its pairs of the chunk in a byte table,
          // then every lane shifts its pairs (two dependent shared loads
          // per pair instead of a per-lane search over the image table)
          const int qlo = max(cb, hp);
          if (lane >= 1 && lane < nimg) {
            const int hi = min(i_off + i_np, ce);
            for (int q = max(i_off, qlo); q < hi; ++q) s_imgof[q - cb] = (unsigned char)lane;
          }
          __syncwarp();
          for (int q = qlo + lane; q < ce; q += 32) {
            const float4 sh = s_shiftw[s_imgof[q - cb]];
            float4 av = A[q - cb];
            float4 bv = B[q - cb];
            av.x += sh.x;
            av.y += sh.x;
            av.z += sh.y;
            av.w += sh.y;
            bv.x += sh.z;
            bv.y += sh.z;
            A[q - cb] = av;
            B[q - cb] = bv;
          }
        }
        __syncwarp();
      }
      // ---- home block (self masked): pairs [cb, min(ce, hp)) ----
      {
        const int lo = cb, hi = max(lo, min(ce, hp));
        const int np = hi - lo;
        const int k0 = lo + ((np * part) >> lp), k1 = lo + ((np * (part + 1)) >> lp);
        uint64_t p2 = 0;
        for (int k = k0; k < k1; ++k)
          p2p2_step<GRAD, true>(A - cb, B - cb, k, x2, y2, z2, self, p2, gx2, gy2, gz2);
        kahan_fold(v2, c2, p2);
      }
      // ---- other images: pairs [max(cb, hp), ce) ----
      {
        const int lo = max(cb, hp), hi = max(lo, ce);
        const int np = hi - lo;
        const int k0 = lo + ((np * part) >> lp), k1 = lo + ((np * (part + 1)) >> lp);
        const float4* Ab = A - cb;
        const float4* Bb = B - cb;
        // two independent accumulator sets per step pair (ILP); potential
        // partials folded every 16 steps
        uint64_t hx2 = 0, hy2 = 0, hz2 = 0;
        int k = k0;
#pragma unroll 1
        for (; k + 16 <= k1; k += 16) {
          uint64_t p2 = 0, q2 = 0;
#pragma unroll
          for (int u = 0; u < 16; u += 2) {
            p2p2_step<GRAD, false>(Ab, Bb, k + u, x2, y2, z2, 0, p2, gx2, gy2, gz2);
            p2p2_step<GRAD, false>(Ab, Bb, k + u + 1, x2, y2, z2, 0, q2, hx2, hy2, hz2);
          }
          kahan_fold(v2, c2, f2add(p2, q2));
        }
        {
          uint64_t p2 = 0, q2 = 0;
#pragma unroll 1
          for (; k + 2 <= k1; k += 2) {
            p2p2_step<GRAD, false>(Ab, Bb, k, x2, y2, z2, 0, p2, gx2, gy2, gz2);
            p2p2_step<GRAD, false>(Ab, Bb, k + 1, x2, y2, z2, 0, q2, hx2, hy2, hz2);
          }
          if (k < k1) p2p2_step<GRAD, false>(Ab, Bb, k, x2, y2, z2, 0, q2, hx2, hy2, hz2);
          kahan_fold(v2, c2, f2add(p2, q2));
        }
        if (GRAD) {
          gx2 = f2add(gx2, hx2);
          gy2 = f2add(gy2, hy2);
          gz2 = f2add(gz2, hz2);
        }
      }
    }
    float v, gx, gy, gz, u;
    {
      float ca, cb2;
      f2unpack(c2, ca, cb2);
      f2unpack(v2, v, u);
      v = (v - ca) + (u - cb2);
    }
    f2unpack(gx2, gx, u);
    gx += u;
    f2unpack(gy2, gy, u);
    gy += u;
    f2unpack(gz2, gz, u);
    gz += u;
    for (int m = 16; m >= W; m >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, m);
      if (GRAD) {
        gx += __shfl_xor_sync(0xffffffffu, gx, m);
        gy += __shfl_xor_sync(0xffffffffu, gy, m);
        gz += __shfl_xor_sync(0xffffffffu, gz, m);
      }
    }
    if (act && part == 0) {
      const int i = t0 + pb + slot;
      vout[i] = v;
      if (GRAD) {
        gout[3 * (size_t)i] = -gx;
        gout[3 * (size_t)i + 1] = -gy;
        gout[3 * (size_t)i + 2] = -gz;
      }
    }
  }
  __syncwarp();  // the staging buffers are reused by the warp's next leaf
}

// ctl == nullptr: one warp per leaf of the grid.  ctl != nullptr: persistent
// and preemptible: warps fetch leaves from the counter *ctl (relative to the
// rank's first leaf) until every leaf is taken or the flag *stop is raised; a fetched leaf is always finished, so a later launch over the
// same counter picks up exactly the leaves not done yet (the near field then
// fills the SMs the latency-bound far-field chains leave idle, and yields them
// to the tensor-core M2L, lfmm_api.cu issue_p2p).
template <bool GRAD>
__global__ void __launch_bounds__(P2P2_WARPS * 32, LFMM_P2P2_MINB) k_p2p2(const float4* __restrict__ xq,
                                                          const float4* __restrict__ pair_a,
                                                          const float4* __restrict__ pair_b,
                                                          const int* __restrict__ leaf_start, int depth,
                                                          float size, int periodic, float* __restrict__ vout,
                                                          float* __restrict__ gout, int x0, int x1,
                                                          int* __restrict__ ctl, const int* __restrict__ stop) {
  extern __shared__ float4 p2p2_smem[];  // [warp][A | B][SMAX / 2]
  __shared__ __align__(8) uint64_t s_bar[P2P2_WARPS];
  __shared__ int2 s_img[P2P2_WARPS][28];  // {first staged pair, pair count}; sentinel at nimg
  __shared__ float4 s_shift[P2P2_WARPS][27];
  __shared__ unsigned char s_imgof_all[P2P2_WARPS][P2P2_SMAX / 2];  // image of each staged pair (shift pass)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nleaf = 1 << (3 * depth);
  const int first = x0 << (2 * depth);  // the rank's first leaf plane
  const int own = (min(x1, 1 << depth) - x0) << (2 * depth);
  float4* A = p2p2_smem + (size_t)w * P2P2_SMAX;
  float4* B = A + P2P2_SMAX / 2;
  const uint32_t bar = smem_u32(&s_bar[w]);
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  if (ctl == nullptr) {
    const int b = first + blockIdx.x * P2P2_WARPS + w;
    if (b >= nleaf || (b >> (2 * depth)) >= x1) return;
    p2p2_leaf<GRAD>(b, xq, pair_a, pair_b, leaf_start, depth, size, periodic, vout, gout, A, B, s_img[w],
                    s_shift[w], s_imgof_all[w], bar, phase);
    return;
  }
  for (;;) {
    int v = 0;
    if (lane == 0) v = *reinterpret_cast<const volatile int*>(stop) ? own : atomicAdd(ctl, 1);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v >= own) break;
    p2p2_leaf<GRAD>(first + v, xq, pair_a, pair_b, leaf_start, depth, size, periodic, vout, gout, A, B, s_img[w],
                    s_shift[w], s_imgof_all[w], bar, phase);
  }
}

}  // namespace lfmm
