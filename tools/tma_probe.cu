// tools/tma_probe.cu -- cp.async.bulk (1D TMA) global->shared throughput vs
// copy size and copies in flight per CTA. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const double* __restrict__ g, long total, int chunk_bytes, int inflight, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const long nchunks = total * 8 / chunk_bytes;
  unsigned phase = 0;
  double acc = 0;
  long c = blockIdx.x;
  int slot = 0;
  // prologue
  long issued = c;
  for (int i = 0; i < inflight && issued < nchunks; ++i, issued += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(chunk_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + i * chunk_bytes)),
                   "l"((const char*)g + issued * chunk_bytes), "r"(chunk_bytes), "r"(sa(&bar[i])) : "memory");
    }
  }
  for (; c < nchunks; c += gridDim.x) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar[slot])),
                 "r"((phase >> slot) & 1u) : "memory");
    phase ^= 1u << slot;
    acc += ((const double*)(sm + slot * chunk_bytes))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && issued < nchunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[slot])), "r"(chunk_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + slot * chunk_bytes)),
                   "l"((const char*)g + issued * chunk_bytes), "r"(chunk_bytes), "r"(sa(&bar[slot])) : "memory");
    }
    issued += gridDim.x;
    slot = (slot + 1) % inflight;
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  const long total = 1L << 28;  // 2 GB of doubles
  double* g; cudaMalloc(&g, total * 8); cudaMemset(g, 0, total * 8);
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int chunk : {4096, 16384, 32768}) for (int inflight : {1, 2, 4, 6}) for (int cps : {1, 2}) {
    size_t smem = (size_t)chunk * inflight;
    if (smem * cps > 200 * 1024) continue;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<sms * cps, 256, smem>>>(g, total, chunk, inflight, out);
    cudaEventRecord(a);
    k<<<sms * cps, 256, smem>>>(g, total, chunk, inflight, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("chunk %6d B inflight %d ctas/SM %d : %7.1f GB/s  (%s)\n", chunk, inflight, cps, total * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
