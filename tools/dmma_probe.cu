#include <cstdio>
#include <cuda_runtime.h>
template <int NA>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, bb = 1.0 - threadIdx.x * 1e-9;
  double c0[NA], c1[NA];
  for (int u = 0; u < NA; ++u) c0[u] = c1[u] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < NA; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[u]), "+d"(c1[u]) : "d"(a), "d"(bb));
  }
  double s = 0; for (int u = 0; u < NA; ++u) s += c0[u] + c1[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NA> void run(int sms, int bps, int threads, double* out) {
  int iters = 20000 * 4 / NA;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_loop<NA><<<sms * bps, threads>>>(out, 10);
  cudaEventRecord(e0); dmma_loop<NA><<<sms * bps, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * NA * iters * (threads / 32) * (double)sms * bps;
  printf("{\"acc_per_warp\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", NA, bps * threads / 32, fl / ms * 1e-9);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  for (int bps : {1, 2, 4}) { run<4>(sms, bps, 512, out); run<8>(sms, bps, 512, out); run<16>(sms, bps, 512, out); }
  run<8>(sms, 1, 256, out); run<16>(sms, 1, 256, out);  run<16>(sms, 1, 128, out);
  return 0;
}
