// tools/dmma_probe.cu -- FP64 tensor-core MMA (mma.sync m8n8k4 f64) vs DFMA
// throughput on this GPU, alone and mixed in the same warps (are they
// separate pipes?). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// MODE 0: DMMA only (CH independent accumulators); 1: DFMA only (CH chains);
// 2: per iteration CH DMMA + DF DFMA-chains x 8 in the same warp
template <int MODE, int CH, int DF>
__global__ void k(double* out, int iters) {
  double acc[CH][2], f[DF];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = c;
#pragma unroll
  for (int c = 0; c < DF; ++c) f[c] = c + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (MODE != 1) dmma(acc[c][0], acc[c][1], a, b);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < DF; ++c)
        if (MODE != 0) f[c] = fma(f[c], b, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int c = 0; c < DF; ++c) s += f[c];
  if (s == 1.2345) out[0] = s;
}

template <int MODE, int CH, int DF>
void run(int warps_per_sm, const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 32 * warps_per_sm, iters = 4096;
  k<MODE, CH, DF><<<sms, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE, CH, DF><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(sms) * warps_per_sm;
  // m8n8k4: 8*8*4 FMA = 256 FMA = 512 flop per warp instruction
  const double mma_flop = (MODE != 1) ? 512.0 * CH * iters * warps : 0.0;
  const double fma_flop = (MODE != 0) ? 2.0 * 32 * 8 * DF * iters * warps : 0.0;
  printf("%-28s warps/SM %2d : DMMA %6.2f TF/s  DFMA %6.2f TF/s  total %6.2f TF/s\n", name, warps_per_sm,
         mma_flop / (ms * 1e-3) / 1e12, fma_flop / (ms * 1e-3) / 1e12, (mma_flop + fma_flop) / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0, 4, 1>(w, "DMMA x4 chains");
    run<0, 8, 1>(w, "DMMA x8 chains");
    run<1, 1, 4>(w, "DFMA x4 chains");
    run<2, 4, 2>(w, "mixed 4 DMMA + 2x8 DFMA");
    run<2, 4, 4>(w, "mixed 4 DMMA + 4x8 DFMA");
    run<2, 2, 4>(w, "mixed 2 DMMA + 4x8 DFMA");
  }
  return 0;
}
