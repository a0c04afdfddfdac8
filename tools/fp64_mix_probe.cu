// tools/fp64_mix_probe.cu -- FP64 pipe throughput per instruction form on
// this GPU: DFMA / DADD / DMUL chains, and DFMA whose three operands are all
// distinct live registers (no operand reuse), at 12 warps/SM with 8
// independent chains per thread. Tells whether the K3 body's DADD / DMUL or
// its operand pattern costs more than the DFMA-chain peak.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix_probe fp64_mix_probe.cu
#include <cstdio>

#include <cuda_runtime.h>

constexpr int CH = 8;

template <int MODE>
__global__ void __launch_bounds__(128, 3) k(double* out, int iters, double b, double d) {
  double a[CH], c[CH], e[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = threadIdx.x * 1e-7 + i;
    c[i] = 1.0 + 1e-9 * i;
    e[i] = 1e-12 * (i + 1);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (MODE == 0) a[i] = fma(a[i], b, d);                    // DFMA, reused operands
        if (MODE == 1) a[i] = a[i] + d;                           // DADD
        if (MODE == 2) a[i] = a[i] * b;                           // DMUL
        if (MODE == 3) a[i] = fma(a[i], c[(i + u) % CH], e[(i + 3 * u) % CH]);  // DFMA, distinct regs
        if (MODE == 4) {                                          // 4 DFMA : 1 DADD : 1 DMUL
          if (u % 6 == 4) a[i] = a[i] + e[(i + u) % CH];
          else if (u % 6 == 5) a[i] = a[i] * c[(i + u) % CH];
          else a[i] = fma(a[i], c[(i + u) % CH], e[(i + 3 * u) % CH]);
        }
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

template <int MODE>
void run(const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = 3 * sms, iters = 2048;
  k<MODE><<<blocks, 128>>>(out, 8, 0.999999, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 128>>>(out, iters, 0.999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double inst = 8.0 * CH * iters * 128.0 * blocks;  // FP64 thread instructions
  printf("%-36s %6.2f T FP64 instr/s (x2 = %6.2f TFLOP/s if all were DFMA)\n", name, inst / (ms * 1e-3) / 1e12,
         2 * inst / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  run<0>("DFMA chains (reused b, d)");
  run<1>("DADD chains");
  run<2>("DMUL chains");
  run<3>("DFMA, distinct register operands");
  run<4>("mix 4 DFMA : 1 DADD : 1 DMUL");
  return 0;
}
