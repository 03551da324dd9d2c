// Microbenchmark of the pipe peaks the FMM stages are bounded by (FFMA, DFMA,
// MUFU rsqrt, legacy mma.sync TF32 / DMMA). Measured once per box; the numbers
// go into DESIGN.md as roofline denominators for the non-GEMM pipes.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void ffma_k(float* out, float a, float b) {
  float x0=threadIdx.x,x1=x0+1,x2=x0+2,x3=x0+3,x4=x0+4,x5=x0+5,x6=x0+6,x7=x0+7;
  float y0=b, y1=b*2;
  for (int i=0;i<ITERS;i++){
    x0=fmaf(x0,y0,y1);x1=fmaf(x1,y0,y1);x2=fmaf(x2,y0,y1);x3=fmaf(x3,y0,y1);
    x4=fmaf(x4,y0,y1);x5=fmaf(x5,y0,y1);x6=fmaf(x6,y0,y1);x7=fmaf(x7,y0,y1);
    y1 = y1 + a;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void dfma_k(double* out, double a, double b) {
  double x0=threadIdx.x,x1=x0+1,x2=x0+2,x3=x0+3,x4=x0+4,x5=x0+5,x6=x0+6,x7=x0+7;
  double y0=b, y1=b*2;
  for (int i=0;i<ITERS/4;i++){
    x0=fma(x0,y0,y1);x1=fma(x1,y0,y1);x2=fma(x2,y0,y1);x3=fma(x3,y0,y1);
    x4=fma(x4,y0,y1);x5=fma(x5,y0,y1);x6=fma(x6,y0,y1);x7=fma(x7,y0,y1);
    y1 = y1 + a;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void rsqrt_k(float* out, float a) {
  float x0=threadIdx.x+1,x1=x0+1,x2=x0+2,x3=x0+3;
  for (int i=0;i<ITERS;i++){
    x0=rsqrtf(x0)+a;x1=rsqrtf(x1)+a;x2=rsqrtf(x2)+a;x3=rsqrtf(x3)+a;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3;
}
__global__ void mma_tf32_k(float* out) {
  // four independent chains with distinct operands and initial values, so
  // ptxas cannot merge them (cuobjdump -sass: 4 HMMA per inner iteration)
  unsigned a0=threadIdx.x,a1=a0+1,a2=a0+2,a3=a0+3,b0=a0*3,b1=a0*5;
  float c[4][4];
  for(int j=0;j<4;j++) for(int r=0;r<4;r++) c[j][r]=j+0.25f*r;
  for (int i=0;i<ITERS/4;i++){
#pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
      : "+f"(c[j][0]),"+f"(c[j][1]),"+f"(c[j][2]),"+f"(c[j][3]) : "r"(a0+j),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1+j));
  }
  float s=0; for(int j=0;j<4;j++) s+=c[j][0]+c[j][1]+c[j][2]+c[j][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void dmma_k(double* out) {
  // four independent chains with distinct operands and initial values (the
  // round-1 version fed four identical chains and ptxas merged them into one,
  // overstating the rate 4x)
  double a=threadIdx.x, b=a*0.5;
  double c[4][2];
  for(int j=0;j<4;j++){ c[j][0]=j; c[j][1]=-j; }
  for (int i=0;i<ITERS/16;i++){
#pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
      : "+d"(c[j][0]),"+d"(c[j][1]) : "d"(a+j),"d"(b-j));
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=c[0][0]+c[1][1]+c[2][0]+c[3][1];
}
template <class F> float timeit(F f){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best=1e30;
  for(int r=0;r<5;r++){ cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best) best=ms; }
  return best;
}
int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks=nsm*8, threads=256; long nt=(long)blocks*threads;
  float* fo; double* dout; cudaMalloc(&fo, nt*4); cudaMalloc(&dout, nt*8);
  float t;
  t=timeit([&]{ffma_k<<<blocks,threads>>>(fo,1e-7f,0.999f);});
  printf("FFMA   %.2f TFLOP/s (2 flop/FMA)\n", 2.0*8*ITERS*nt/t/1e9);
  t=timeit([&]{dfma_k<<<blocks,threads>>>(dout,1e-7,0.999);});
  printf("DFMA   %.2f TFLOP/s\n", 2.0*8*(ITERS/4)*nt/t/1e9);
  t=timeit([&]{rsqrt_k<<<blocks,threads>>>(fo,1e-7f);});
  printf("MUFU.RSQ %.3f Tops/s\n", 4.0*ITERS*nt/t/1e9);
  t=timeit([&]{mma_tf32_k<<<blocks,threads>>>(fo);});
  printf("mma.sync tf32 m16n8k8 %.1f TFLOP/s\n", 2.0*16*8*8*4*(ITERS/4)*(nt/32)/t/1e9);
  t=timeit([&]{dmma_k<<<blocks,threads>>>(dout);});
  printf("mma.sync f64 m8n8k4 %.2f TFLOP/s\n", 2.0*8*8*4*4*(ITERS/16)*(nt/32)/t/1e9);
  cudaError_t e=cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
