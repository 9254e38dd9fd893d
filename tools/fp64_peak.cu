// FP64 peak probes for the roofline denominators: DFMA loop and DMMA (mma.sync m8n8k4 f64) loop.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, bb = 1.0 - threadIdx.x * 1e-9;
  double c0[4] = {0,0,0,0}, c1[4] = {0,0,0,0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[u]), "+d"(c1[u]) : "d"(a), "d"(bb));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c1[0] + c0[1] + c1[1] + c0[2] + c1[2] + c0[3] + c1[3];
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    int threads = 512, blocks = sms * 4, iters = 20000;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)threads * blocks;
    printf("{\"probe\":\"dfma\",\"tflops\":%.3f,\"ms\":%.3f}\n", fl / ms * 1e-9, ms);
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * (threads / 32) * blocks;
    printf("{\"probe\":\"dmma_m8n8k4\",\"tflops\":%.3f,\"ms\":%.3f}\n", fl / ms * 1e-9, ms);
  }
  printf("sms=%d clock_khz=%d l2=%d smem_optin=%zu\n", sms, p.clockRate, p.l2CacheSize, p.sharedMemPerBlockOptin);
  cudaError_t err = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
