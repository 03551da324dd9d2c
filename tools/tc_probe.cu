// tc_probe.cu — one-off hardware probe for the M2L redesign (not product code).
//
// Checks, on the B200, the three tcgen05 facts the halo M2L kernel relies on:
//  1. kind::f16 with fp16 operands, M=128, N=256, K=16, fp32 accumulator;
//  2. a "linear-row" K-major SWIZZLE_NONE descriptor for B (SBO = 128 B, so
//     8-row groups are contiguous, LBO = R*16 B between 8-wide k groups): a
//     shift of the B start address by s*16 B selects rows s..s+N-1, i.e. a
//     spatially shifted window of a halo array is just a descriptor change;
//  3. the error of long accumulation chains inside the tensor core (T MMAs
//     into one accumulator) and of the 3-product fp16 split
//     a*b ~ ah*bh + ah*bl + al*bh (a = ah + al, fp16 each).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 128, N = 256, K = 16;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

// A parts: NA x (128 x 16) row-major fp16 in global; B parts: NB x (R x 16).
// Product i uses A part pa[i] and B part pb[i]; iteration t shifts B rows by t.
__global__ void k_probe(const __half* __restrict__ A, int NA, const __half* __restrict__ B, int NB, int R,
                        int T, int NP, const int* __restrict__ pa, const int* __restrict__ pb, float* __restrict__ D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A: standard core layout, LBO = 128 (k groups), SBO = 256 (8-row groups)
  const uint32_t a_bytes = M * K * 2;
  for (int e = tid; e < NA * M * K; e += blockDim.x) {
    const int part = e / (M * K), r = (e / K) % M, k = e % K;
    const uint32_t off = part * a_bytes + (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
    *reinterpret_cast<__half*>(sm + off) = A[e];
  }
  // B: linear rows, LBO = R*16, SBO = 128
  unsigned char* bs = sm + NA * a_bytes;
  const uint32_t b_bytes = (uint32_t)R * K * 2;
  for (int e = tid; e < NB * R * K; e += blockDim.x) {
    const int part = e / (R * K), r = (e / K) % R, k = e % K;
    const uint32_t off = part * b_bytes + (k >> 3) * (R * 16) + r * 16 + (k & 7) * 2;
    *reinterpret_cast<__half*>(bs + off) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < NP; ++i) {
        const uint64_t da = desc(su32(sm + pa[i] * a_bytes), 128, 256);
        const uint64_t db = desc(su32(bs + pb[i] * b_bytes + t * 16), R * 16, 128);
        const uint32_t acc = (t > 0 || i > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(IDESC), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

struct Run {
  double max_rel, bias;
};

// mode 0: single fp16 product; mode 1: 3-product split of fp32 data
Run run(int T, int mode, std::mt19937& rng, bool print_layout) {
  const int R = N + T;
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> a32(M * K), b32((size_t)R * K);
  for (auto& x : a32) x = U(rng);
  for (auto& x : b32) x = U(rng);
  int NA = 1, NB = 1, NP = 1;
  std::vector<__half> ha, hb;
  std::vector<int> pa = {0}, pb = {0};
  std::vector<double> ad(M * K), bd((size_t)R * K);
  if (mode == 0) {
    for (int i = 0; i < M * K; ++i) {
      ha.push_back(__float2half_rn(a32[i]));
      ad[i] = (double)__half2float(ha.back());
    }
    for (size_t i = 0; i < (size_t)R * K; ++i) {
      hb.push_back(__float2half_rn(b32[i]));
      bd[i] = (double)__half2float(hb.back());
    }
  } else {
    NA = NB = 2;
    NP = 3;
    pa = {0, 0, 1};
    pb = {0, 1, 0};
    ha.resize(2 * M * K);
    hb.resize(2 * (size_t)R * K);
    for (int i = 0; i < M * K; ++i) {
      __half h = __float2half_rn(a32[i]);
      ha[i] = h;
      ha[M * K + i] = __float2half_rn(a32[i] - __half2float(h));
      ad[i] = a32[i];
    }
    for (size_t i = 0; i < (size_t)R * K; ++i) {
      __half h = __float2half_rn(b32[i]);
      hb[i] = h;
      hb[(size_t)R * K + i] = __float2half_rn(b32[i] - __half2float(h));
      bd[i] = b32[i];
    }
  }
  __half *dA, *dB;
  float* dD;
  int *dpa, *dpb;
  CK(cudaMalloc(&dA, ha.size() * 2));
  CK(cudaMalloc(&dB, hb.size() * 2));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMalloc(&dpa, 16));
  CK(cudaMalloc(&dpb, 16));
  CK(cudaMemcpy(dA, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpa, pa.data(), pa.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpb, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)NA * M * K * 2 + (size_t)NB * R * K * 2;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_probe<<<1, 128, smem>>>(dA, NA, dB, NB, R, T, NP, dpa, dpb, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> D(M * N);
  CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
  double maxref = 0, maxerr = 0, bias = 0;
  std::vector<double> ref(M * N, 0.0);
  for (int t = 0; t < T; ++t)
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += ad[m * K + k] * bd[(size_t)(n + t) * K + k];
        ref[m * N + n] += s;
      }
  for (int i = 0; i < M * N; ++i) {
    maxref = std::max(maxref, std::fabs(ref[i]));
    const double e = (double)D[i] - ref[i];
    maxerr = std::max(maxerr, std::fabs(e));
    bias += (ref[i] >= 0 ? e : -e);  // >0: away from zero on average
  }
  if (print_layout) printf("D[0][0]=%g ref=%g  D[77][201]=%g ref=%g\n", D[0], ref[0], D[77 * N + 201], ref[77 * N + 201]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dpa);
  cudaFree(dpb);
  return {maxerr / maxref, bias / (M * N) / maxref};
}

int main() {
  std::mt19937 rng(1234);
  printf("tcgen05 kind::f16 M=128 N=256 K=16, linear-row B descriptor, row shift t per MMA\n");
  for (int mode = 0; mode < 2; ++mode)
    for (int T : {1, 4, 32, 256, 1024, 2048}) {
      Run r = run(T, mode, rng, T == 4 && mode == 0);
      printf("mode=%s T=%5d  max|err|/max|ref| = %.3e   mean signed err/max|ref| = %+.3e  (2^-24=%.2e)\n",
             mode == 0 ? "fp16x1" : "fp16x3", T, r.max_rel, r.bias, std::ldexp(1.0, -24));
    }
  return 0;
}
