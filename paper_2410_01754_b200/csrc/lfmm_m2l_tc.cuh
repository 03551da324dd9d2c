// lfmm_m2l_tc.cuh — M2L on the 5th-generation tensor cores (tcgen05, TMEM).
//
// Same math and the same interaction lists as the GEMM_M2L mode of
// k_gemm_gather (downward_pass M2L, fmm/solver.py:282-287; lists
// octree.py:96-111), for the fp32 path with (p+1)^2 <= 128:
//
//   D[128 coeff x 128 targets] (TMEM, fp32) += sum_terms A_term * B_term
//   A_term  = packed M2L operator of the term's offset (128 x 128)
//   B_term  = the 128 targets' source multipoles for that offset (gathered)
//
// fp32 accuracy from TF32 units by the 3xTF32 split: a = a_hi + a_lo with
// a_hi = rna_tf32(a); D += A_hi B_hi + A_hi B_lo + A_lo B_hi (error ~2^-22).
// A is pre-split and pre-arranged on the device at plan time in the
// no-swizzle K-major core-matrix layout (8 rows x 16 B atoms), one 32 KB
// block (hi | lo) per (operator, 32-wide k chunk), so each stage is ONE
// cp.async.bulk copy.  B is loaded to registers (one 128-B line per target
// per chunk, prefetched one iteration ahead), split, and stored to shared
// memory in the same layout.  One thread issues the MMAs
// (tcgen05.mma.cta_group::1.kind::tf32, M=128, N=128, K=8) and commits them
// to an mbarrier; the epilogue reads D with tcgen05.ld and writes the M2L
// partial slot consumed by the L2L sweep.
#pragma once
#include <cstdint>

#include "lfmm_common.cuh"
#include "lfmm_expansions.cuh"

namespace lfmm {

constexpr int TC_N = 128;          // targets per CTA (MMA N)
constexpr int TC_M = 128;          // output coefficients (MMA M), = ncp
constexpr int TC_BK = 32;          // k per stage
constexpr int TC_NCHUNK = 4;       // 128 / 32
constexpr int TC_TILE = TC_M * TC_BK * 4;  // 16 KB: one operand half (hi or lo)
constexpr int TC_STAGE = 2 * TC_TILE;      // 32 KB: hi | lo
constexpr int TC_ASTAGES = 3, TC_BSTAGES = 2;
constexpr int TC_SMEM = (TC_ASTAGES + TC_BSTAGES) * TC_STAGE + 1024;
// accumulators rotate over terms: shorter fp32 accumulation chains inside
// the tensor core (its accumulator adds are not round-to-nearest), summed
// with round-to-nearest fp32 adds in the epilogue
constexpr int TC_NACC = 4;
constexpr int TC_TMEM_COLS = TC_N * TC_NACC;  // 512

struct TcArgs {
  const float* mult;     // multipoles, all levels, 128 per box
  float* partial;        // M2L partial slots (same layout as GemmArgs)
  const float* ops_tc;   // [316][4 chunks][hi|lo][core layout 128 x 32]
  int depth;
  int64_t level_off[DMAX + 2];
  int64_t part_off[DMAX + 2];
  int nsplit[DMAX + 2];
  int job_start[DMAX + 3];
};

__host__ __device__ inline int tc_tiles_per_parity(int level) {
  const int sub = 1 << (level - 1);
  return (sub * sub * sub + TC_N - 1) / TC_N;
}

// byte offset of element (r, k) of a 128 x 32 fp32 tile in the K-major
// SWIZZLE_NONE core-matrix layout: LBO (next 16 B along k) = 128 B,
// SBO (next 8-row group) = 1024 B
__host__ __device__ inline uint32_t tc_core_off(int r, int k) {
  return (uint32_t)((((r >> 3) * 8 + (k >> 2)) * 128) + ((r & 7) * 16) + ((k & 3) * 4));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);        // start address
  d |= (uint64_t)(128 >> 4) << 16;                 // LBO: next k core matrix
  d |= (uint64_t)(1024 >> 4) << 32;                // SBO: next 8-row group
  d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
  return d;                                        // base offset 0, SWIZZLE_NONE
}

// kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(bar),
      "r"(phase));
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Plan-time: ops_m2l (fp32, [316][128][128] row-major) -> ops_tc layout.
__global__ void k_tc_arrange_ops(const float* __restrict__ ops, float* __restrict__ out, int nops) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over nops*128*128
  if (idx >= (int64_t)nops * TC_M * TC_M) return;
  const int op = (int)(idx / (TC_M * TC_M));
  const int r = (int)((idx / TC_M) % TC_M), k = (int)(idx % TC_M);
  const float v = ops[idx];
  const float hi = tf32_rna(v);
  const float lo = v - hi;
  const int chunk = k / TC_BK, kk = k % TC_BK;
  char* base = reinterpret_cast<char*>(out) + ((size_t)op * TC_NCHUNK + chunk) * TC_STAGE;
  *reinterpret_cast<float*>(base + tc_core_off(r, kk)) = hi;
  *reinterpret_cast<float*>(base + TC_TILE + tc_core_off(r, kk)) = lo;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Warp-specialised pipeline over TC_STAGES stages of (A 32 KB | B 32 KB):
//   warps 0-3  B producers: one target row per thread; register prefetch of
//              the next chunk, tf32 split, st.shared, fence.proxy.async,
//              arrive on full_b[s]; afterwards the TMEM epilogue
//   warp 4     MMA issuer (one lane): waits full_a/full_b, 12 MMAs per
//              stage, tcgen05.commit -> empty[s]
//   warp 5     A loader (one lane): waits empty[s], one cp.async.bulk of
//              the pre-arranged operator chunk -> full_a[s]
constexpr int TC_STAGES = 3;
constexpr int TC_SMEM_WS = TC_STAGES * 2 * TC_STAGE + 1024;
constexpr int TC_THREADS = 192;

__global__ void __launch_bounds__(TC_THREADS, 1) k_m2l_tc(TcArgs g) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_a[TC_STAGES], full_b[TC_STAGES], empty_bar[TC_STAGES], done_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int col_dst[TC_N];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- job: (level, parity, tile, slot) ----
  int level = 1;
  while (level < g.depth && (int)blockIdx.x >= g.job_start[level + 1]) ++level;
  const int j = blockIdx.x - g.job_start[level];
  const int ns = g.nsplit[level];
  const int tpp = tc_tiles_per_parity(level);
  const int slot = j % ns;
  const int tile = j / ns;
  const int par = tile / tpp;
  const int q0 = (tile % tpp) * TC_N;
  const int sub = 1 << (level - 1);
  const int nside = 1 << level, msk = nside - 1;
  const int t0 = (NM2L * slot) / ns, t1 = (NM2L * (slot + 1)) / ns;
  const int niter = (t1 - t0) * TC_NCHUNK;
  int my_box = -1;
  if (tid < TC_N) {
    my_box = (q0 + tid < sub * sub * sub) ? parity_box(level, par, q0 + tid) : -1;
    col_dst[tid] = my_box;
  }
  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(smem_u32(&full_a[s]), 1);
      mbar_init(smem_u32(&full_b[s]), TC_N);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&done_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  if (warp < 4) {
    // ------------------------------------------------ B producers ----
    const int gx = my_box >= 0 ? my_box >> (2 * level) : 0;
    const int gy = my_box >= 0 ? (my_box >> level) & msk : 0;
    const int gz = my_box >= 0 ? my_box & msk : 0;
    const float* mult_l = g.mult + g.level_off[level] * TC_M;
    auto b_load = [&](int it, float4 (&r)[8]) {
      if (my_box < 0 || it >= niter) {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
      }
      const int term = t0 + it / TC_NCHUNK, chunk = it % TC_NCHUNK;
      const char4 o = c_m2l_off[par * NM2L + term];
      const int src = ((((gx + o.x) & msk) << level | ((gy + o.y) & msk)) << level) | ((gz + o.z) & msk);
      const float4* p = reinterpret_cast<const float4*>(mult_l + (size_t)src * TC_M + chunk * TC_BK);
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = __ldg(p + u);
    };
    float4 rb[8], rn[8];
    b_load(0, rb);
    for (int it = 0; it < niter; ++it) {
      const int st = it % TC_STAGES, use = it / TC_STAGES;
      b_load(it + 1, rn);
      if (use >= 1) mbar_wait(smem_u32(&empty_bar[st]), (use - 1) & 1);
      unsigned char* bh = smem + st * 2 * TC_STAGE + TC_STAGE;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 v = rb[u];
        float4 h, l;
        h.x = tf32_rna(v.x);
        h.y = tf32_rna(v.y);
        h.z = tf32_rna(v.z);
        h.w = tf32_rna(v.w);
        l.x = v.x - h.x;
        l.y = v.y - h.y;
        l.z = v.z - h.z;
        l.w = v.w - h.w;
        const uint32_t off = tc_core_off(tid, 4 * u);
        *reinterpret_cast<float4*>(bh + off) = h;
        *reinterpret_cast<float4*>(bh + TC_TILE + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(smem_u32(&full_b[st]));
#pragma unroll
      for (int u = 0; u < 8; ++u) rb[u] = rn[u];
    }
    // ------------------------------------------------ epilogue ----
    if (niter > 0) mbar_wait(smem_u32(&done_bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* out = g.partial + ((size_t)g.part_off[level] + (size_t)slot * (1u << (3 * level))) * TC_M;
    const int coef = warp * 32 + lane;
    const int nterm_cta = t1 - t0;
    const int nacc = nterm_cta < TC_NACC ? nterm_cta : TC_NACC;
#pragma unroll 1
    for (int c0 = 0; c0 < TC_N; c0 += 32) {
      float sum[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) sum[jj] = 0.f;
#pragma unroll 1
      for (int a = 0; a < nacc; ++a) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c0 + a * TC_N);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) sum[jj] += __uint_as_float(v[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int box = col_dst[c0 + jj];
        if (box >= 0) out[(size_t)box * TC_M + coef] = sum[jj];
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer ----
    if (lane == 0) {
      for (int it = 0; it < niter; ++it) {
        const int st = it % TC_STAGES, ph = (it / TC_STAGES) & 1;
        mbar_wait(smem_u32(&full_a[st]), ph);
        mbar_wait(smem_u32(&full_b[st]), ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(smem + st * 2 * TC_STAGE), b0 = a0 + TC_STAGE;
        const int tl = it / TC_NCHUNK;
        const uint32_t dacc = tmem + (uint32_t)((tl % TC_NACC) * TC_N);
        const bool fresh = tl < TC_NACC && (it % TC_NCHUNK) == 0;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          const uint32_t ko = kk * 256;
          const uint64_t ah = tc_desc(a0 + ko), al = tc_desc(a0 + TC_TILE + ko);
          const uint64_t bhd = tc_desc(b0 + ko), bld = tc_desc(b0 + TC_TILE + ko);
          tc_mma(dacc, ah, bhd, (fresh && kk == 0) ? 0u : 1u);
          tc_mma(dacc, ah, bld, 1u);
          tc_mma(dacc, al, bhd, 1u);
        }
        tc_commit(smem_u32(&empty_bar[st]));
      }
      if (niter > 0) tc_commit(smem_u32(&done_bar));
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ A loader ----
    if (lane == 0) {
      for (int it = 0; it < niter; ++it) {
        const int st = it % TC_STAGES, use = it / TC_STAGES;
        if (use >= 1) mbar_wait(smem_u32(&empty_bar[st]), (use - 1) & 1);
        const int term = t0 + it / TC_NCHUNK, chunk = it % TC_NCHUNK;
        const int row = c_m2l_row[par * NM2L + term];
        const char* src = reinterpret_cast<const char*>(g.ops_tc) + ((size_t)row * TC_NCHUNK + chunk) * TC_STAGE;
        bulk_load(smem_u32(smem + st * 2 * TC_STAGE), src, TC_STAGE, smem_u32(&full_a[st]));
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
}

}  // namespace lfmm
