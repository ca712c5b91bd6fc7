// Microbenchmark: do fp64 mma.sync (DMMA) and DFMA share the B200 fp64 datapath?
// Times DFMA-only, DMMA-only and interleaved kernels with the same per-thread op counts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma dmma_dfma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <bool FMA, bool MMA>
__global__ void kern(int iters, double seed, double* sink) {
  double f[8], m0[4], m1[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = seed + threadIdx.x * 1e-9 + k * 1e-7;
#pragma unroll
  for (int k = 0; k < 4; ++k) { m0[k] = f[k]; m1[k] = f[k + 4]; }
  const double a = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) if (FMA) f[k] = fma(f[k], a, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) if (MMA) dmma(m0[k], m1[k], a, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += f[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) s += m0[k] + m1[k];
  if (s == 1234.5) sink[0] = s;
}

template <bool F, bool M>
float run(int iters, int blocks, int threads, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<F, M><<<blocks, threads>>>(iters, 1.0, sink);
  cudaEventRecord(e0);
  kern<F, M><<<blocks, threads>>>(iters, 2.0, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 256;
  for (int occ : {4, 8}) {
    const int blocks = sms * occ;
    const float tf = run<true, false>(iters, blocks, threads, sink);
    const float tm = run<false, true>(iters, blocks, threads, sink);
    const float tb = run<true, true>(iters, blocks, threads, sink);
    const double nthr = double(blocks) * threads;
    const double dfma_flops = 2.0 * 8 * iters * nthr;
    const double dmma_flops = 512.0 * 4 * iters * (nthr / 32);
    printf("blocks/SM %d: DFMA only %.3f ms (%.1f TF)  DMMA only %.3f ms (%.1f TF)  both %.3f ms (sum %.3f, max %.3f)\n",
           occ, tf, dfma_flops / tf / 1e9, tm, dmma_flops / tm / 1e9, tb, tf + tm, tf > tm ? tf : tm);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
