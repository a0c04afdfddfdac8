// tools/fp64_probe.cu -- DFMA throughput vs occupancy and ILP on this GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-7 + c;
  const double b = 0.999999, d = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) a[c] = fma(a[c], b, d);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
void run(int warps_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int threads = 32 * warps_per_sm;  // one block per SM
  const int iters = 4096 / CH;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH><<<sms, threads>>>(out, 16);
  cudaEventRecord(e0);
  k<CH><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 16 * CH * (double)iters * threads * sms;
  printf("warps/SM %2d chains %d : %6.2f TFLOP/s\n", warps_per_sm, CH, flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}
int main() {
  for (int w : {4, 8, 12, 16, 32}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
