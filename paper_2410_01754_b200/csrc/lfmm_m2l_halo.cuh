// lfmm_m2l_halo.cuh — M2L as shifted-window tensor-core GEMMs (tcgen05, TMEM).
//
// Same translations as downward_pass M2L (fmm/solver.py:282-287) over the
// same interaction lists (octree.py:96-111): target box T = 2i + tc (tc its
// parity class), offset o (189 per tc), source S = T + o = 2(i + d) + sc with
// tc + o = 2d + sc, d in {-1,0,1}^3.  For a fixed (tc, sc) the sources of all
// targets of class tc are the class-sc grid SHIFTED by d, so with the class
// grids laid out in a padded linear order (strides Z^2, Z, 1, Z = h + 2, one
// halo box per side, periodic wrap) the B operand of term o is a window of a
// halo array at a constant row offset: the tcgen05 descriptor start address
// moves by 16 B per row and nothing is gathered per term.
//
//   D[128 coeff x N rows] (TMEM fp32) += A_o[128 x 16] B_{sc,d}[16 x N]
//
// Operands are fp16 "hi/lo" pairs after power-of-two equilibration
// (A' = diag(r) A diag(c), M' = gl M / c): three products hi*hi + hi*lo +
// lo*hi carry the same 22-bit operand precision as 3xTF32 (tools/
// m2l_fp16_study.py) at twice the tensor rate and half the shared-memory
// bytes.  Accumulation chains inside the tensor core are kept to one
// (sc, 16-coefficient chunk) iteration (<= 78 MMAs; tools/tc_probe.cu shows the
// truncation bias grows with chain length) and drained into fp32 registers.
//
// Before the M2L launch k_pack_mult16 writes every level's multipoles, scaled
// and split, as fp16 "planes" in exactly the padded linear class-grid order
// (periodic halo boxes duplicated), one plane per (source class, 16-coeff
// chunk, hi/lo, 8-wide k group); a halo window is then one contiguous
// cp.async.bulk per plane.
//
// Roles (384 threads, one CTA per SM):
//   warps 0-7  workers: drain the accumulator of each iteration (tcgen05.ld)
//              into fp32 register sums; final epilogue (partial slot)
//   warps 8, 9 MMA issuers (one lane each): even / odd iterations into TMEM
//              accumulators 0 / 1.  One issuing thread sustains only one
//              MMA per ~130-190 clk (tools/tc_rate.cu), less than the 128
//              clk an N = 256 MMA occupies the tensor core; two issuers reach
//              it, and one issuer's MMAs overlap the other accumulator's drain.
//              Each accumulator still sees its MMAs in one fixed order.
//   warp 10    A loader (one lane): one 8 KB cp.async.bulk per term, the two
//              iterations of a pair interleaved term by term in the ring
//   warp 11    halo loader (one lane): 12 cp.async.bulk per iteration
// Pipelines: halo buffers x2 (full/empty), TMEM accumulators x2 (full/empty),
// A stages x HM_ASTAGES (full/empty).
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "lfmm_common.cuh"
#include "lfmm_sm100.cuh"

namespace lfmm {

constexpr int HM_NMAX = 256;       // target rows per job (MMA N)
constexpr int HM_KC = 16;          // coefficients per iteration (one f16 MMA K)
constexpr int HM_NKC = 8;          // 128 / 16
constexpr int HM_ATILE = 8192;     // one operator chunk: hi 4 KB | lo 4 KB
constexpr int HM_ASTAGES = 14;   // A-ring stages (10 when the level-6 halo windows need the room)
constexpr int HM_ASTAGES_SMALL = 10;
constexpr int HM_THREADS = 384;
constexpr int HM_WORKERS = 256;

// (tc, sc) term tables: count and {operator row, dx, dy, dz}
__constant__ int c_hterm_n[64];
__constant__ short c_hterm_row[64 * 27];
__constant__ char4 c_hterm_d[64 * 27];

struct HaloArgs {
  const float* mult;                 // multipoles, all levels, 128 per box
  float* partial;                    // M2L partial slots
  const unsigned char* ops16;        // [316][8][hi 4 KB | lo 4 KB]
  unsigned char* mult16;             // packed fp16 planes, all levels
  int64_t m16_off[DMAX + 2];         // byte offset of each level's planes
  const int4* jobs;                  // {level | tc<<4 | grp<<8 | G<<12, t0, N, 0}
  const unsigned int* level_max;     // per level: float bits of max |M^/c|
  const float* inv_r;                // 1 / row scale (128)
  const float* inv_c;                // 1 / column scale (128)
  int64_t level_off[DMAX + 2];
  int64_t part_off[DMAX + 2];
  int rw_cap;                        // rows per window the buffers were sized for
  int lvl0;                          // first level of a k_level_absmax / k_pack_mult16 launch (grid.y = levels)
  int own_x0, own_x1, own_depth;     // k_level_absmax over one rank's leaf x-slab (own_x1 == 0: whole level)
  int stagger;                       // terms issuer 1 runs behind issuer 0 (A-ring order, see hm_aseq)
  int pk_r0[DMAX + 2], pk_r1[DMAX + 2];  // k_pack_mult16: padded rows [r0, r1) per level (r1 == 0: all)
  int njobs;                         // jobs of this launch (k_m2l_halo is persistent)
  int* counter;                      // next job to fetch; zeroed before each launch
};

// A-ring slot sequence of issuer par's u-th term (u counts its terms over all
// its iterations; both issuers own T terms).  The loader walks steps s = 0,
// 1, ...: issuer 0's term s, then issuer 1's term s - D.  Issuer 1 thus runs
// D terms behind issuer 0, so the two never finish an iteration together
// (an iteration's end waits for its next halo window, and in phase both
// issuers would wait at once and leave the tensor core idle).  D is capped at
// AS - 6; soundness needs D + 1 < AS (the ring invariant in k_m2l_halo).
__device__ __forceinline__ int hm_aseq(int par, int u, int D, int T) {
  return par == 0 ? u + min(max(u - D, 0), T) : min(u + D + 1, T) + u;
}

__host__ __device__ inline int hm_rw(int N, int Z) { return N + 2 * Z + 2; }
__host__ __device__ inline size_t hm_buf_bytes(int rw) { return (size_t)192 * rw; }  // 2 parts x 2 kgroups x 3 windows x 16 B
__host__ inline size_t hm_smem_bytes(int rw_cap, int astages = HM_ASTAGES) {
  return 2 * hm_buf_bytes(rw_cap) + (size_t)astages * HM_ATILE + 1024;
}

// group g of G: relative parities (tc ^ sc) it covers
// (G = 8: one class per job; 4: the pairs (0,7) (1,6) (2,5) (4,3); 2: two
// pairs per job)
__device__ __forceinline__ int hm_group_rel(int G, int g, int k) {
  if (G == 8) return g;
  const int pi = (G == 4) ? g : 2 * g + (k >> 1);
  const int r = (pi == 3) ? 4 : pi;
  return (k & 1) == 0 ? r : (r ^ 7);
}

__device__ __forceinline__ uint64_t hm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// warp-wide issue: every lane of the issuer warp runs the loop (operands are
// warp-uniform), one elected lane issues the instruction
__device__ __forceinline__ void hm_mma_w(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void hm_commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ uint32_t hm_idesc(int N) {
  // kind::f16: D f32, A/B f16, K-major both, N, M = 128
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void hm_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void hm_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Plan-time: ops_m2l fp32 [316][128][128] (row = output coeff a, col = input
// coeff b) -> equilibrated fp16 hi/lo chunks in the K-major core layout
// (8 rows x 16 B atoms, LBO 128 B between the two 8-wide k groups, SBO 256 B
// between 8-row groups).
__global__ void k_h16_arrange(const float* __restrict__ ops, const float* __restrict__ rs,
                              const float* __restrict__ cs, unsigned char* __restrict__ out, int nops) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nops * 128 * 128) return;
  const int op = (int)(idx >> 14), a = (int)((idx >> 7) & 127), b = (int)(idx & 127);
  const float v = ops[idx] * rs[a] * cs[b];
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  const int kc = b >> 4, k = b & 15;
  unsigned char* base = out + ((size_t)op * HM_NKC + kc) * HM_ATILE;
  const uint32_t off = (a >> 3) * 256 + (k >> 3) * 128 + (a & 7) * 16 + (k & 7) * 2;
  *reinterpret_cast<__half*>(base + off) = hi;
  *reinterpret_cast<__half*>(base + 4096 + off) = lo;
}

// per level (blockIdx.y + lvl0): max over boxes and coefficients of |M^ / c|
__global__ void k_level_absmax(const float* __restrict__ mult, HaloArgs g, unsigned int* __restrict__ out) {
  const int level = blockIdx.y + g.lvl0;
  const int nbox = 1 << (3 * level);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4 ic = reinterpret_cast<const float4*>(g.inv_c)[lane];
  float m = 0.f;
  int b0 = 0, b1 = nbox;
  if (g.own_x1 > 0) {  // slab decomposition: the boxes of x-planes [x0, x1) at this level are contiguous
    const int sh = g.own_depth - level;
    b0 = (g.own_x0 >> sh) << (2 * level);
    b1 = (g.own_x1 >> sh) << (2 * level);
  }
  for (int b = b0 + blockIdx.x * 64 + warp; b < min(b1, b0 + (int)blockIdx.x * 64 + 64); b += 8) {
    const float4 v = reinterpret_cast<const float4*>(mult + (g.level_off[level] + b) * 128)[lane];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x * ic.x), fabsf(v.y * ic.y)), fmaxf(fabsf(v.z * ic.z), fabsf(v.w * ic.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[8];
  if (lane == 0) wm[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float x = wm[0];
    for (int w = 1; w < 8; ++w) x = fmaxf(x, wm[w]);
    atomicMax(out + level, __float_as_uint(x));
  }
}

// power-of-two level scale: max |M'| = gl max|M^/c| in [2^11, 2^12)
__device__ __forceinline__ float hm_level_scale(const unsigned int* level_max, int level) {
  const float mmax = __uint_as_float(level_max[level]);
  if (!(mmax > 0.f)) return 1.f;
  int ex = 0;
  frexpf(mmax, &ex);
  return ldexpf(1.f, 12 - ex);
}

// rows of one level's padded class grid (+16 rows of slack for the last tile)
__host__ __device__ inline int hm_plane_rows(int level) {
  const int Z = (1 << (level - 1)) + 2;
  return Z * Z * Z + 16;
}

// multipoles -> fp16 planes: thread per (level, source class, padded row)
__global__ void k_pack_mult16(HaloArgs g) {
  // thread per (padded row, 16-coefficient chunk kc): 8 threads read one
  // box's 512 B contiguously, every plane store is a coalesced row run
  const int level = blockIdx.y + g.lvl0, sc = blockIdx.z;
  const int prow = hm_plane_rows(level);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // a slab decomposition packs only the x-rows its owned targets' windows read
  const int r = (t >> 3) + g.pk_r0[level], kc = t & 7;
  if (r >= (g.pk_r1[level] ? g.pk_r1[level] : prow)) return;
  const int h = 1 << (level - 1), Z = h + 2, YZ = Z * Z;
  const int x = ((r / YZ - 1) + h) & (h - 1), y = (((r / Z) % Z - 1) + h) & (h - 1), z = ((r % Z - 1) + h) & (h - 1);
  const int box = ((((2 * x + ((sc >> 2) & 1)) << level) | (2 * y + ((sc >> 1) & 1))) << level) |
                  (2 * z + (sc & 1));
  const float gl = hm_level_scale(g.level_max, level);
  const float4* src = reinterpret_cast<const float4*>(g.mult + (g.level_off[level] + box) * 128) + kc * 4;
  const float4* icv = reinterpret_cast<const float4*>(g.inv_c) + kc * 4;
  unsigned char* base = g.mult16 + g.m16_off[level];
  float4 v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = __ldg(src + u);
  uint4 hv[2], lv[2];
#pragma unroll
  for (int kg = 0; kg < 2; ++kg) {
    float a[8];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float4 w = v[kg * 2 + u];
      const float4 c = icv[kg * 2 + u];
      a[4 * u] = w.x * c.x * gl;
      a[4 * u + 1] = w.y * c.y * gl;
      a[4 * u + 2] = w.z * c.z * gl;
      a[4 * u + 3] = w.w * c.w * gl;
    }
    float hf[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) hf[j] = __half2float(__float2half_rn(a[j]));
    hv[kg] = make_uint4(pack_h2(hf[0], hf[1]), pack_h2(hf[2], hf[3]), pack_h2(hf[4], hf[5]), pack_h2(hf[6], hf[7]));
    lv[kg] = make_uint4(pack_h2(a[0] - hf[0], a[1] - hf[1]), pack_h2(a[2] - hf[2], a[3] - hf[3]),
                        pack_h2(a[4] - hf[4], a[5] - hf[5]), pack_h2(a[6] - hf[6], a[7] - hf[7]));
  }
#pragma unroll
  for (int part = 0; part < 2; ++part)
#pragma unroll
    for (int kg = 0; kg < 2; ++kg) {
      const size_t plane = (((size_t)sc * HM_NKC + kc) * 2 + part) * 2 + kg;
      *reinterpret_cast<uint4*>(base + (plane * prow + r) * 16) = part == 0 ? hv[kg] : lv[kg];
    }
}

#ifdef LFMM_HM_PROF
// profiling build only (tools/hm_prof.py): per CTA {start, end, wait halo,
// wait acc_empty, wait a_full, terms, MMA issue end, smid}
__device__ unsigned long long g_hm_prof[8192][8];
#define HM_T0() const unsigned long long _t0 = clock64()
#define HM_ACC(slot) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_hm_prof[blockIdx.x][slot], clock64() - _t0)
#else
#define HM_T0()
#define HM_ACC(slot)
#endif

// Persistent CTAs (one per SM): jobs are fetched from a global counter by
// the halo-loader warp and handed to the other roles through a JQ-slot ring in
// shared memory (job descriptor + its term tables, job_full / job_empty
// mbarriers).  Every role walks the same job sequence; iteration, A-ring and
// accumulator counters run on across jobs, so the next job's MMAs start while
// the workers drain and write out the previous one (no per-job pipeline
// fill / drain tail).
constexpr int HM_JQ = 2;
constexpr int HM_JOB_CONSUMERS = 1 + 2 + 8;  // A loader lane, 2 issuer warps, 8 worker warps

template <int AS>
__global__ void __launch_bounds__(HM_THREADS, 1) k_m2l_halo(HaloArgs g) {
#ifdef LFMM_HM_PROF
  unsigned long long _tstart = 0;
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_tstart));
    g_hm_prof[blockIdx.x][0] = _tstart;
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_hm_prof[blockIdx.x][7] = sm;
    for (int i = 2; i < 7; ++i) g_hm_prof[blockIdx.x][i] = 0;
  }
#endif
  extern __shared__ __align__(1024) unsigned char hm_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)hm_smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t halo_full[2], halo_empty[2], acc_full[2], acc_empty[2];
  __shared__ __align__(8) uint64_t a_full[AS], a_empty[AS];
  __shared__ __align__(8) uint64_t job_full[HM_JQ], job_empty[HM_JQ];
  __shared__ uint32_t tmem_base_sh;
  // per job slot: the descriptor and the (tc, sc) term lists (B row offset in
  // 16-B units, operator row, term count per source class)
  __shared__ int4 s_job[HM_JQ];
  __shared__ uint32_t s_boff[HM_JQ][4][27];
  __shared__ int s_orow[HM_JQ][4][27];
  __shared__ int s_nt[HM_JQ][4];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t bufb = hm_buf_bytes(g.rw_cap);
  unsigned char* abase = smem + 2 * bufb;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&halo_full[s]), 12);
      mbar_init(smem_u32(&halo_empty[s]), 1);
      mbar_init(smem_u32(&acc_full[s]), 1);
      mbar_init(smem_u32(&acc_empty[s]), HM_WORKERS);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(smem_u32(&a_full[s]), 1);
      mbar_init(smem_u32(&a_empty[s]), 1);
    }
    for (int s = 0; s < HM_JQ; ++s) {
      mbar_init(smem_u32(&job_full[s]), 1);
      mbar_init(smem_u32(&job_empty[s]), HM_JOB_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  if (warp < 8) {
    // ================================================= workers =========
    const int quad = warp & 3, hcol = warp >> 2;
    int it_g = 0;
    for (int jq = 0;; ++jq) {
      const int slot = jq % HM_JQ;
      mbar_wait(smem_u32(&job_full[slot]), (jq / HM_JQ) & 1);
      const int4 job = s_job[slot];
      if (job.x == 0) break;
      const int level = job.x & 15, tc = (job.x >> 4) & 7, grp = (job.x >> 8) & 15, G = (job.x >> 12) & 15;
      const int t0 = job.y, N = job.z;
      const int h = 1 << (level - 1), Z = h + 2, YZ = Z * Z;
      const int niter = (8 / G) * HM_NKC;
      const int ncol = min(128, N - 128 * hcol);  // columns this thread drains (may be <= 0)
      float sum[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) sum[j] = 0.f;
      for (int it = 0; it < niter; ++it, ++it_g) {
        mbar_wait(smem_u32(&acc_full[it_g & 1]), (it_g >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (ncol > 0) {
          const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)((it_g & 1) * 256 + hcol * 128);
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c * 8 < ncol) {
              float v[8];
              hm_ld8(tb + c * 8, v);
#pragma unroll
              for (int j = 0; j < 8; ++j) sum[c * 8 + j] += v[j];
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(smem_u32(&acc_empty[it_g & 1]));
      }
      // ---- epilogue: partial slot grp of this level (overlaps the next job's MMAs) ----
      const int coef = quad * 32 + lane;
      const float scale = g.inv_r[coef] / hm_level_scale(g.level_max, level);
      float* out = g.partial + ((size_t)g.part_off[level] + (size_t)grp * ((size_t)1 << (3 * level))) * 128;
      const int tcx = (tc >> 2) & 1, tcy = (tc >> 1) & 1, tcz = tc & 1;
      const int gi = t0 + hcol * 128;
      int x = gi / YZ - 1, y = (gi / Z) % Z - 1, z = gi % Z - 1;
#pragma unroll
      for (int j = 0; j < 128; ++j) {
        if (hcol * 128 + j < N && x >= 0 && x < h && y >= 0 && y < h && z >= 0 && z < h) {
          const int box = ((((2 * x + tcx) << level) | (2 * y + tcy)) << level) | (2 * z + tcz);
          out[(size_t)box * 128 + coef] = sum[j] * scale;
        }
        if (++z == Z - 1) {  // next padded row: z, y in [-1, Z - 1)
          z = -1;
          if (++y == Z - 1) {
            y = -1;
            ++x;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&job_empty[slot]));
    }
  } else if (warp == 8 || warp == 9) {
    // ================================================= MMA issuers =====
    // (whole warp; hm_mma_w / hm_commit_w elect one lane).  Issuer par runs
    // the global iterations of its parity, so it always fills accumulator par
    // and reads halo buffer par (every job has an even iteration count).
    const int par = __shfl_sync(0xffffffffu, warp - 8, 0);
    const uint64_t a_desc0 = hm_desc(smem_u32(abase), 128, 256);
    int it_base = 0, seq_base = 0;
    for (int jq = 0;; ++jq) {
      const int slot = jq % HM_JQ;
      mbar_wait(smem_u32(&job_full[slot]), (jq / HM_JQ) & 1);
      const int4 job = s_job[slot];
      if (job.x == 0) break;
      const int level = job.x & 15, G = (job.x >> 12) & 15, N = job.z;
      const int Z = (1 << (level - 1)) + 2;
      const int rw = hm_rw(N, Z);
      const int nsc = 8 / G, niter = nsc * HM_NKC;
      const uint32_t idesc = hm_idesc(N);
      const uint32_t lbo = 3u * rw * 16u;
      int T = 0;
      for (int k = 0; k < nsc; ++k) T += (HM_NKC / 2) * s_nt[slot][k];
      // Ring invariant: an issuer's wait on sequence j (stage j % AS, parity
      // (j / AS) & 1) is only sound if fill j - AS of that stage has completed
      // (else the parity test sees the phase two behind and passes early).
      // Fills complete in issue order and an issuer's consumed sequence m
      // orders every fill <= m before it, so the largest jump between an
      // issuer's consecutive sequence numbers must stay <= AS; issuer 1
      // starts a job at j = D + 1 after its previous job's last term (a jump
      // of D + 2), so D + 2 <= AS (tests/test_m2l_schedule.py checks every
      // term count, across job boundaries).  The cap keeps 4 stages spare.
      const int D = min(min(g.stagger, AS - 6), T);
      int u = 0;  // this issuer's terms so far in this job
      for (int it0 = 0; it0 < niter; it0 += 2) {
        const int k = it0 / HM_NKC;
        const int nt = s_nt[slot][k];
        const int itg = it_base + it0 + par;
        {
          HM_T0();
          mbar_wait(smem_u32(&halo_full[par]), (itg >> 1) & 1);
          HM_ACC(2);
        }
        {
          HM_T0();
          if (itg >= 2) mbar_wait(smem_u32(&acc_empty[par]), ((itg - 2) >> 1) & 1);
          HM_ACC(3);
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // descriptors are advanced by adding (bytes >> 4) to the start-address
        // field (shared addresses < 256 KB: no carry out of its 14 bits)
        const uint64_t b_desc0 = hm_desc(smem_u32(smem + par * bufb), lbo, 128);
        const uint64_t b_lo = (2u * lbo) >> 4;
        const uint32_t dacc = tmem + (uint32_t)(par * 256);
        uint32_t boff = s_boff[slot][k][0];
        for (int t = 0; t < nt; ++t) {
          const int sq = seq_base + hm_aseq(par, u + t, D, T);
          const int stage = sq % AS;
          const uint64_t dbh = b_desc0 + boff;
          if (t + 1 < nt) boff = s_boff[slot][k][t + 1];
          const uint64_t dah = a_desc0 + (uint64_t)(stage * (HM_ATILE >> 4));
          {
            HM_T0();
            mbar_wait(smem_u32(&a_full[stage]), (sq / AS) & 1);
            HM_ACC(4);
          }
#ifdef LFMM_HM_PROF
          if (lane == 0) atomicAdd(&g_hm_prof[blockIdx.x][5], 1ull);
#endif
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          hm_mma_w(dacc, dah, dbh, idesc, t > 0 ? 1u : 0u);
          hm_mma_w(dacc, dah, dbh + b_lo, idesc, 1u);
          hm_mma_w(dacc, dah + (4096 >> 4), dbh, idesc, 1u);
          hm_commit_w(smem_u32(&a_empty[stage]));
        }
        hm_commit_w(smem_u32(&acc_full[par]));
        hm_commit_w(smem_u32(&halo_empty[par]));
        u += nt;
      }
      it_base += niter;
      seq_base += 2 * T;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&job_empty[slot]));
    }
#ifdef LFMM_HM_PROF
    unsigned long long te;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
    g_hm_prof[blockIdx.x][6] = te;
#endif
    __syncwarp();
  } else if (warp == 10) {
    // ================================================= A loader ========
    if (lane == 0) {
      int seq = 0;
      for (int jq = 0;; ++jq) {
        const int slot = jq % HM_JQ;
        mbar_wait(smem_u32(&job_full[slot]), (jq / HM_JQ) & 1);
        const int4 job = s_job[slot];
        if (job.x == 0) break;
        const int G = (job.x >> 12) & 15, nsc = 8 / G;
        int T = 0;
        for (int k = 0; k < nsc; ++k) T += (HM_NKC / 2) * s_nt[slot][k];
        const int D = min(min(g.stagger, AS - 6), T);  // same lag as the issuers (ring invariant above)
        // one cursor per issuer: (iteration pair it0, term t)
        int c_it0[2] = {0, 0}, c_t[2] = {0, 0};
        for (int s = 0; s < T + D; ++s) {
#pragma unroll
          for (int par = 0; par < 2; ++par) {
            const int u = s - par * D;
            if (u < 0 || u >= T) continue;
            const int k = c_it0[par] / HM_NKC;
            const int row = s_orow[slot][k][c_t[par]];
            const int kc = (c_it0[par] + par) % HM_NKC;
            if (++c_t[par] == s_nt[slot][k]) {
              c_t[par] = 0;
              c_it0[par] += 2;
            }
            const int stage = seq % AS, use = seq / AS;
            if (use >= 1) mbar_wait(smem_u32(&a_empty[stage]), (use - 1) & 1);
            bulk_load(smem_u32(abase + stage * HM_ATILE), g.ops16 + ((size_t)row * HM_NKC + kc) * HM_ATILE,
                      HM_ATILE, smem_u32(&a_full[stage]));
            ++seq;
          }
        }
        mbar_arrive(smem_u32(&job_empty[slot]));
      }
    }
    __syncwarp();
  } else {
    // ========================================= job fetch + halo loader =====
    int it_g = 0;
    for (int jq = 0;; ++jq) {
      const int slot = jq % HM_JQ;
      if (jq >= HM_JQ) mbar_wait(smem_u32(&job_empty[slot]), ((jq / HM_JQ) - 1) & 1);
      int j = 0;
      if (lane == 0) j = atomicAdd(g.counter, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      const int4 job = j < g.njobs ? g.jobs[j] : make_int4(0, 0, 0, 0);
      if (job.x != 0) {
        const int level = job.x & 15, tc = (job.x >> 4) & 7, grp = (job.x >> 8) & 15, G = (job.x >> 12) & 15;
        const int Z = (1 << (level - 1)) + 2;
        const int rw = hm_rw(job.z, Z);
        for (int e = lane; e < 4 * 27; e += 32) {
          const int k = e / 27, t = e % 27;
          if (k < 8 / G) {
            const int sc = tc ^ hm_group_rel(G, grp, k);
            const int tab = tc * 8 + sc;
            if (t == 0) s_nt[slot][k] = c_hterm_n[tab];
            if (t < c_hterm_n[tab]) {
              const char4 d = c_hterm_d[tab * 27 + t];
              s_boff[slot][k][t] = (uint32_t)((d.x + 1) * rw + (Z + 1) + d.y * Z + d.z);
              s_orow[slot][k][t] = c_hterm_row[tab * 27 + t];
            }
          }
        }
      }
      if (lane == 0) s_job[slot] = job;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&job_full[slot]));  // release: tables and descriptor
      if (job.x == 0) break;
      if (lane == 0) {
        const int level = job.x & 15, tc = (job.x >> 4) & 7, grp = (job.x >> 8) & 15, G = (job.x >> 12) & 15;
        const int t0 = job.y, N = job.z;
        const int Z = (1 << (level - 1)) + 2, YZ = Z * Z;
        const int rw = hm_rw(N, Z);
        const int niter = (8 / G) * HM_NKC;
        const int prow = hm_plane_rows(level);
        const unsigned char* base = g.mult16 + g.m16_off[level];
        const uint32_t bytes = (uint32_t)rw * 16u;
        for (int it = 0; it < niter; ++it, ++it_g) {
          const int sc = tc ^ hm_group_rel(G, grp, it / HM_NKC);
          const int kc = it % HM_NKC;
          if (it_g >= 2) mbar_wait(smem_u32(&halo_empty[it_g & 1]), ((it_g - 2) >> 1) & 1);
          unsigned char* buf = smem + (it_g & 1) * bufb;
          const uint32_t bar = smem_u32(&halo_full[it_g & 1]);
#pragma unroll
          for (int pk = 0; pk < 4; ++pk) {  // (part, kgroup)
            const size_t plane = ((size_t)sc * HM_NKC + kc) * 4 + pk;
#pragma unroll
            for (int w = 0; w < 3; ++w) {
              const int r0 = t0 + (w - 1) * YZ - (Z + 1);
              bulk_load(smem_u32(buf + (size_t)(pk * 3 + w) * bytes), base + (plane * prow + r0) * 16, bytes, bar);
            }
          }
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
#ifdef LFMM_HM_PROF
  if (threadIdx.x == 0) {
    unsigned long long te;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
    g_hm_prof[blockIdx.x][1] = te;
  }
#endif
}

}  // namespace lfmm
