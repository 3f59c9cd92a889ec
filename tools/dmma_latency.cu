// DMMA.8x8x4 (FP64 mma.sync m8n8k4) latency and per-SMSP issue rate on sm_100a: one CTA of W warps
// on one SM, each warp running K independent accumulator chains of length L; cycles per DMMA from
// clock64.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dmma_latency tools/dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void k_chain(int iters, double* out, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[K], c1[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { c0[k] = k; c1[k] = -k; }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[k]), "+d"(c1[k]) : "d"(a), "d"(b));
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += c0[k] + c1[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(int warps) {
  const int iters = 4096;
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  k_chain<K><<<1, 32 * warps>>>(iters, out, cyc);
  k_chain<K><<<1, 32 * warps>>>(iters, out, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp_dmma = (double)c / (iters * K);        // cycles per DMMA of one warp
  const double sm_dmma_per_cyc = (double)iters * K * warps / c;  // DMMAs per cycle per SM
  printf("K=%d chains/warp, %2d warps: %7.2f cyc per dependent step, SM %.4f DMMA/cyc (%.1f flop/cyc)\n", K, warps,
         (double)c / iters, sm_dmma_per_cyc, sm_dmma_per_cyc * 512);
  (void)per_warp_dmma;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
  }
  return 0;
}
