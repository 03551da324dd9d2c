// lfmm_translate_tc.cuh — the fp32 M2M / L2L sweeps on the tensor cores
// (tcgen05 kind::tf32, TMEM accumulator), 3xTF32.
//
// Same translations and the same CTA decomposition as k_translate
// (lfmm_expansions.cuh; upward_pass solver.py:248-258, downward_pass
// solver.py:276-281): CTA = (tile of TT columns, octant o),
//
//   D[128 coeff x TN columns] (TMEM fp32) = Op_o[128 x 128] B[128 x TN]
//
// with B the child multipoles of the tile's parents (UP) or the parents'
// locals (DOWN).  Operands are split hi + lo, each rounded to tf32 (10-bit
// mantissa, 8-bit exponent: no scaling), and the three products hi*hi +
// hi*lo + lo*hi carry 22 operand bits, the fp32 SIMT kernel's precision at
// the tensor rate.  Each K chunk accumulates into its own TMEM columns (a
// chain of 12 MMAs: 3 products x 4 K steps) and the chunks are added in fp32
// registers: the tensor core's accumulation truncates, and one 48-MMA chain
// per tile doubled the fp32 parity error.
//
// K is streamed in chunks of 32 (one 128-B row of fp32) through an NSTG-stage
// ring: the operator chunk (hi | lo, 32 KB, pre-split in its shared-memory
// image at plan setup) by cp.async.bulk, the B chunk by the 128 threads (LDG,
// split, STS into the K-major core-matrix layout).  At 96 KB (NSTG = 2) a CTA
// fits beside the near-field launch that shares the SMs with the far chain.
// Epilogues as k_translate: UP writes the octant's partial slot and the last
// of the 8 octant CTAs of a tile adds them in octant order; DOWN adds the
// level's M2L partial slots in slot order.
#pragma once
#include <cstdint>

#include "lfmm_expansions.cuh"
#include "lfmm_sm100.cuh"

namespace lfmm {

constexpr int TT_THREADS = 128;
constexpr int TT_KC = 32;                           // K per chunk
constexpr int TT_NCH = 4;                           // chunks (K = 128)
constexpr int TT_APLANE = 128 * TT_KC * 4;          // one operator chunk, one plane: 16 KB
constexpr int TT_ACHUNK = 2 * TT_APLANE;            // hi | lo: 32 KB
constexpr int TT_OPBYTES = TT_NCH * TT_ACHUNK;      // one octant's operator image: 128 KB

template <int TN, int NSTG>
constexpr size_t tt_smem_bytes() {
  return (size_t)NSTG * (TT_ACHUNK + 2 * TN * TT_KC * 4) + 1024;  // + alignment slack
}

// byte offset of (row r, k in chunk) in a K-major, no-swizzle operand tile:
// core matrices of 8 rows x 16 B; K-adjacent ones 128 B apart (LBO), 8-row
// groups 1024 B apart (SBO)
__device__ __forceinline__ uint32_t tt_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
// round to tf32 (10-bit mantissa), to nearest, ties away from zero
__device__ __forceinline__ float tt_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ uint64_t tt_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;   // LBO
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void tt_mma_w(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tt_commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tt_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Operator images for k_translate_tc: ops [8][128 rows][128 k] fp32 ->
// img [8][chunk][hi | lo][16 KB core-matrix layout]
__global__ void k_tt_ops(const float* __restrict__ ops, unsigned char* __restrict__ img) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 8 * 128 * 128) return;
  const int o = i >> 14, r = (i >> 7) & 127, k = i & 127;
  const float x = ops[i];
  const float hi = tt_rna(x), lo = tt_rna(x - hi);
  unsigned char* base = img + (size_t)(o * TT_NCH + (k >> 5)) * TT_ACHUNK;
  *reinterpret_cast<float*>(base + tt_off(r, k & 31)) = hi;
  *reinterpret_cast<float*>(base + TT_APLANE + tt_off(r, k & 31)) = lo;
}

// Per-CTA state of the translation kernels (barriers, TMEM, tables).
template <int TN, int NSTG>
struct TtCta {
  uint64_t a_full[NSTG], mma_done[NSTG];
  uint32_t tmem_sh;
  int col_src[TN], col_dst[TN];
  int last;
};

template <int TN, int NSTG>
__device__ __forceinline__ uint32_t tt_cta_init(TtCta<TN, NSTG>& st) {
  constexpr uint32_t TCOLS = TT_NCH * TN < 32 ? 32 : TT_NCH * TN;  // one accumulator per K chunk
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(smem_u32(&st.a_full[s]), 2);
      mbar_init(smem_u32(&st.mma_done[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&st.tmem_sh)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return st.tmem_sh;
}
template <int TN, int NSTG>
__device__ __forceinline__ void tt_cta_exit(uint32_t tmem) {
  constexpr uint32_t TCOLS = TT_NCH * TN < 32 ? 32 : TT_NCH * TN;  // one accumulator per K chunk
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// One (column tile, octant) of one level.  Every call runs all TT_NCH
// chunks, so each barrier completes an even number of phases per call and
// the parity arithmetic below holds for any number of calls per CTA.
template <int TN, int NSTG>
__device__ __forceinline__ void tt_tile(const TrArgs& g, const unsigned char* __restrict__ img, int tile, int o,
                                        unsigned char* sm, uint32_t sbase, uint32_t tmem, TtCta<TN, NSTG>& st) {
  constexpr int BPLANE = TN * TT_KC * 4;        // one B chunk, one plane
  constexpr int STAGE = TT_ACHUNK + 2 * BPLANE;  // A hi | A lo | B hi | B lo
  constexpr int PPT = TN * 8 / TT_THREADS;      // 16-B B pieces per thread per chunk
  uint64_t* a_full = st.a_full;
  uint64_t* mma_done = st.mma_done;
  int* col_src = st.col_src;
  int* col_dst = st.col_dst;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  (void)lane;
  const int pl = g.mode == 0 ? g.level : g.level - 1;  // parent level
  const int np = 1 << (3 * pl), pn = 1 << pl, cn = 2 * pn;
  // the previous call's epilogue is done with the tables, the stages and
  // (its TMEM loads ordered before this call's MMAs) the accumulator
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < TN) {
    const int p = g.p0 + tile * TN + tid;
    int s = -1, d = -1;
    if (p < (g.pend ? g.pend : np)) {
      const int px = p >> (2 * pl), py = (p >> pl) & (pn - 1), pz = p & (pn - 1);
      const int c = ((((2 * px + ((o >> 2) & 1)) * cn) + 2 * py + ((o >> 1) & 1)) * cn) + 2 * pz + (o & 1);
      s = g.mode == 0 ? c : p;
      d = g.mode == 0 ? p : c;
    }
    col_src[tid] = s;
    col_dst[tid] = d;
  }
  __syncthreads();
  const unsigned char* opimg = img + (size_t)o * TT_OPBYTES;
  auto load_a = [&](int c) {
    const int s = c % NSTG;
    const uint32_t dst = sbase + (uint32_t)(s * STAGE), bar = smem_u32(&a_full[s]);
    bulk_load(dst, opimg + (size_t)c * TT_ACHUNK, TT_APLANE, bar);
    bulk_load(dst + TT_APLANE, opimg + (size_t)c * TT_ACHUNK + TT_APLANE, TT_APLANE, bar);
  };
  if (tid == 0)
    for (int c = 0; c < NSTG && c < TT_NCH; ++c) load_a(c);
  // every B piece of the tile in flight at once (L2 loads: in the chained
  // small levels the sources were written earlier in the same launch): piece e -> column
  // n = 8 (e / 64) + e % 8, k quad (e / 8) % 8 (8 lanes fill one 128-B core
  // matrix row group: conflict-free stores)
  const float* src = reinterpret_cast<const float*>(g.src);
  float4 raw[TT_NCH][PPT];
#pragma unroll
  for (int i = 0; i < PPT; ++i) {
    const int e = tid + i * TT_THREADS, n = ((e >> 6) << 3) | (e & 7), kq = (e >> 3) & 7;
    const int sb = col_src[n];
#pragma unroll
    for (int c = 0; c < TT_NCH; ++c)
      raw[c][i] = sb >= 0 ? __ldcg(reinterpret_cast<const float4*>(src + (size_t)sb * 128 + c * TT_KC + kq * 4))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
#pragma unroll
  for (int c = 0; c < TT_NCH; ++c) {
    const int s = c % NSTG;
    if (c >= NSTG) {  // stage s is free once chunk c - NSTG's MMAs completed
      mbar_wait(smem_u32(&mma_done[s]), ((c - NSTG) / NSTG) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tid == 0) load_a(c);
    }
    unsigned char* bst = sm + s * STAGE + TT_ACHUNK;
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int e = tid + i * TT_THREADS, n = ((e >> 6) << 3) | (e & 7), kq = (e >> 3) & 7;
      const float4 v = raw[c][i];
      float4 h, l;
      h.x = tt_rna(v.x);
      h.y = tt_rna(v.y);
      h.z = tt_rna(v.z);
      h.w = tt_rna(v.w);
      l.x = tt_rna(v.x - h.x);
      l.y = tt_rna(v.y - h.y);
      l.z = tt_rna(v.z - h.z);
      l.w = tt_rna(v.w - h.w);
      const uint32_t off = tt_off(n, 4 * kq);
      *reinterpret_cast<float4*>(bst + off) = h;
      *reinterpret_cast<float4*>(bst + BPLANE + off) = l;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      mbar_wait(smem_u32(&a_full[s]), (c / NSTG) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = sbase + (uint32_t)(s * STAGE), b0 = a0 + TT_ACHUNK;
#pragma unroll
      for (int j = 0; j < TT_KC / 8; ++j) {
        const uint64_t ah = tt_desc(a0 + 256 * j), al = tt_desc(a0 + TT_APLANE + 256 * j);
        const uint64_t bh = tt_desc(b0 + 256 * j), bl = tt_desc(b0 + BPLANE + 256 * j);
        // chunk c into its own accumulator: chains of 12 MMAs (the tensor
        // core's fp32 accumulation truncates), chunks added in fp32 below
        const uint32_t dacc = tmem + (uint32_t)(c * TN);
        tt_mma_w(dacc, ah, bh, idesc, j > 0 ? 1u : 0u);
        tt_mma_w(dacc, ah, bl, idesc, 1u);
        tt_mma_w(dacc, al, bh, idesc, 1u);
      }
      tt_commit_w(smem_u32(&mma_done[s]));
    }
  }
  // the last commit tracks every MMA of the CTA; every stage's last phase
  // is still waited on, so that each phase of each barrier has a waiter
  // before its next arrival (a CTA of the chained kernel runs several tiles)
#pragma unroll
  for (int c = TT_NCH - NSTG; c < TT_NCH; ++c) mbar_wait(smem_u32(&mma_done[c % NSTG]), (c / NSTG) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // drain D into shared memory as [column][128 rows] (the stages are free
  // now), then a vector epilogue: thread -> (column e / 32, rows 4 (e % 32)),
  // a warp one contiguous 512-B row
  float* dsm = reinterpret_cast<float*>(sm);
  {
    const int m = 32 * warp + lane;  // TMEM lane = output coefficient
    const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
    for (int cb = 0; cb < TN; cb += 16) {
      float v[16], u[16];
      tt_ld16(trow + cb, v);
#pragma unroll
      for (int c = 1; c < TT_NCH; ++c) {
        tt_ld16(trow + (uint32_t)(c * TN) + cb, u);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += u[j];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) dsm[(cb + j) * 128 + m] = v[j];
    }
  }
  __syncthreads();
  constexpr int NV = TN * 32 / TT_THREADS;  // 16-B vectors per thread
  // fixed-order sums of nadd slot vectors onto base (base == nullptr: 0),
  // (vector, slot) pairs flattened so that 16 loads are in flight per thread
  auto add_slots = [&](const float* base_sm, const float* slots, size_t slot_stride, int nadd, float* out) {
    const int F = NV * nadd;
    float4 run = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int f0 = 0; f0 < F; f0 += 16) {
      float4 q[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int f = f0 + u, vi = f / nadd, s = f - vi * nadd;
        const int e = tid + vi * TT_THREADS, d = f < F ? col_dst[e >> 5] : -1;
        q[u] = d >= 0 ? __ldcg(reinterpret_cast<const float4*>(slots + (size_t)s * slot_stride + (size_t)d * 128 +
                                                              4 * (e & 31)))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int f = f0 + u, vi = f / nadd, s = f - vi * nadd;
        if (f >= F) break;
        const int e = tid + vi * TT_THREADS;
        if (s == 0)
          run = base_sm ? *reinterpret_cast<const float4*>(base_sm + (e >> 5) * 128 + 4 * (e & 31))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        run.x += q[u].x;
        run.y += q[u].y;
        run.z += q[u].z;
        run.w += q[u].w;
        const int d = col_dst[e >> 5];
        if (s == nadd - 1 && d >= 0) *reinterpret_cast<float4*>(out + (size_t)d * 128 + 4 * (e & 31)) = run;
      }
    }
  };
  if (g.mode == 0) {
    float* slots = reinterpret_cast<float*>(g.slots);
    float* myslot = slots + (size_t)o * np * 128;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int e = tid + i * TT_THREADS, d = col_dst[e >> 5];
      if (d >= 0)
        *reinterpret_cast<float4*>(myslot + (size_t)d * 128 + 4 * (e & 31)) =
            *reinterpret_cast<const float4*>(dsm + (e >> 5) * 128 + 4 * (e & 31));
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st.last = (atomicAdd(&g.cnt[tile], 1) == 7);
    __syncthreads();
    if (st.last) {
      __threadfence();
      add_slots(nullptr, slots, (size_t)np * 128, 8, reinterpret_cast<float*>(g.dst));
      if (tid == 0) g.cnt[tile] = 0;
    }
  } else {
    const size_t nchild = (size_t)np * 8;
    if (g.nsplit > 0) {
      add_slots(dsm, reinterpret_cast<const float*>(g.partial), nchild * 128, g.nsplit, reinterpret_cast<float*>(g.dst));
    } else {
      float* dst = reinterpret_cast<float*>(g.dst);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int e = tid + i * TT_THREADS, d = col_dst[e >> 5];
        if (d >= 0)
          *reinterpret_cast<float4*>(dst + (size_t)d * 128 + 4 * (e & 31)) =
              *reinterpret_cast<const float4*>(dsm + (e >> 5) * 128 + 4 * (e & 31));
      }
    }
  }
}

template <int TN, int NSTG>
__global__ void __launch_bounds__(TT_THREADS) k_translate_tc(TrArgs g, const unsigned char* __restrict__ img) {
  static_assert(TN % 16 == 0 && TN >= 16 && TN <= 64, "MMA N");
  extern __shared__ __align__(16) unsigned char tt_raw[];
  __shared__ __align__(8) TtCta<TN, NSTG> st;
  const uint32_t sbase = (smem_u32(tt_raw) + 1023u) & ~1023u;
  unsigned char* sm = tt_raw + (sbase - smem_u32(tt_raw));
  const uint32_t tmem = tt_cta_init<TN, NSTG>(st);
  tt_tile<TN, NSTG>(g, img, blockIdx.x, blockIdx.y, sm, sbase, tmem, st);
  tt_cta_exit<TN, NSTG>(tmem);
}

// The small levels (at most TN * gridDim.x / 8 parents) in one launch: the
// levels in order, a grid-wide barrier between them (every CTA of this small
// grid is resident beside the near field; the counter is zeroed before the
// launch).  Same tiles and arithmetic as one k_translate_tc launch per level.
struct TtChain {
  TrArgs lev[4];
  int nlev;
  unsigned* bar;
};
template <int TN, int NSTG>
__global__ void __launch_bounds__(TT_THREADS) k_translate_tc_chain(TtChain ch, const unsigned char* __restrict__ img) {
  extern __shared__ __align__(16) unsigned char tt_raw[];
  __shared__ __align__(8) TtCta<TN, NSTG> st;
  const uint32_t sbase = (smem_u32(tt_raw) + 1023u) & ~1023u;
  unsigned char* sm = tt_raw + (sbase - smem_u32(tt_raw));
  const uint32_t tmem = tt_cta_init<TN, NSTG>(st);
  const int o = blockIdx.x & 7, tile = blockIdx.x >> 3;
  const unsigned nblk = gridDim.x;
  for (int l = 0; l < ch.nlev; ++l) {
    const TrArgs& g = ch.lev[l];
    const int pl = g.mode == 0 ? g.level : g.level - 1;
    const int ntile = ((1 << (3 * pl)) + TN - 1) / TN;
    if (tile < ntile) tt_tile<TN, NSTG>(g, img, tile, o, sm, sbase, tmem, st);
    if (l + 1 < ch.nlev) {  // grid barrier: this level's outputs are the next level's inputs
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ch.bar, 1u);
        const unsigned target = (unsigned)(l + 1) * nblk;
        while (*reinterpret_cast<volatile unsigned*>(ch.bar) < target) {
        }
        __threadfence();
      }
      __syncthreads();
    }
  }
  tt_cta_exit<TN, NSTG>(tmem);
}

}  // namespace lfmm
