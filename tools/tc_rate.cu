// tc_rate.cu — one-off probe (not product code): cost per tcgen05.mma
// kind::f16 M=128, K=16 as a function of N, of accumulator interleaving
// (one chain vs two/four independent TMEM accumulators) and of a
// tcgen05.commit + mbarrier round per 3 MMAs (the M2L term loop).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_rate tools/tc_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(bar),
               "r"(ph));
}

// mode bit0: commit+wait-on-previous-commit per term (3 MMAs); nacc chains
__global__ void k_rate(int N, int terms, int nacc, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // mode bit1: the whole warp 0 runs the loop (converged); bit2: warps 0 and 1
  // each issue half of the terms into their own accumulators
  // bit3: issuers are lane 0 of warps 0..(1 << (mode >> 4)) - 1 (one thread each)
  const int nw_iss = (mode & 8) ? (1 << (mode >> 4)) : 1;
  const bool issuer = (mode & 8) ? ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < nw_iss)
                                 : ((mode & 6) ? ((mode & 4) ? threadIdx.x < 64 : threadIdx.x < 32) : threadIdx.x == 0);
  if (issuer) {
    const int wsplit = (mode & 8) ? nw_iss : ((mode & 4) ? 2 : 1), wid = threadIdx.x >> 5;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t da = desc(su32(sm), 128, 256);
    const uint64_t db = desc(su32(sm + 8192), 300 * 16, 128);
    const int step = 512 / nacc;
    unsigned long long t0 = clock64();
    for (int t = wid; t < terms; t += wsplit) {
      const uint32_t d = tb + (uint32_t)((t % nacc) * step);
      if ((mode & 1) && t >= 8) wait(su32(&bars[t % 8]), ((t - 8) / 8) & 1);
      mma(d, da, db, idesc, t >= nacc ? 1u : 0u);
      mma(d, da, db + 1, idesc, 1u);
      mma(d, da + 256, db, idesc, 1u);
      if (mode & 1) commit(su32(&bars[t % 8]));
    }
    if (mode & 4) __syncwarp();
    unsigned long long t1 = clock64();
    __syncwarp(__activemask());
    if ((threadIdx.x & 31) == 0) {
      commit(su32(&bars[14 + wid]));
      wait(su32(&bars[14 + wid]), 0);
    }
    __syncwarp(__activemask());
    unsigned long long t2 = clock64();
    if ((threadIdx.x & 31) == 0 && wid == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int terms = 2000;
  printf("clk per MMA (3 MMAs per term, %d terms): issue-loop / until-complete\n", terms);
  for (int mode : {0, 8 + 16, 8 + 32})
    for (int N : {16, 128, 256})
      for (int nacc : {4}) {
        if (N * nacc > 512) continue;
        k_rate<<<1, 128, 64 * 1024>>>(N, terms, nacc, mode, d);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("mode=%d N=%3d chains=%d : issue %.1f  total %.1f  (ideal work %.1f)\n", mode,
               N, nacc, h[0] / (3.0 * terms), h[1] / (3.0 * terms), N / 2.0);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
