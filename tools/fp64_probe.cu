// Early microbenchmark: FP64 DFMA vs DMMA.8x8x4 throughput on sm_100a, and a
// shared-memory-fed 64x64 complex product loop.  Standalone; not the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[8], b = 1.0000001, c = 1e-9;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  double a = 1e-3 * threadIdx.x, b = 1.0 + 1e-6 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

// 8 warps; warp w owns rows 8w..8w+7 of C = A B (64x64 complex, planar).  A strip in
// registers (A-layout), B in smem (LD = 68).  Repeats the product `reps` times.
constexpr int LD = 68;
__global__ void __launch_bounds__(256, 1) zmm_loop(double* out, int reps) {
  extern __shared__ double sm[];
  double* Br = sm; double* Bi = sm + 64 * LD;
  for (int e = threadIdx.x; e < 64 * LD; e += 256) { Br[e] = 1e-3 * (e % 97); Bi[e] = 1e-3 * (e % 89); }
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double ar[16], ai[16];
  for (int k = 0; k < 16; ++k) { ar[k] = 1e-2 * (w + k + g); ai[k] = 1e-2 * (t - k); }
  double cr[16], ci[16];
  for (int i = 0; i < 16; ++i) { cr[i] = 0; ci[i] = 0; }
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a_r = ar[k], a_i = ai[k], na_i = -ai[k];
      const double* br = Br + (4 * k + t) * LD + g;
      const double* bi = Bi + (4 * k + t) * LD + g;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double b_r = br[8 * j], b_i = bi[8 * j];
        dmma(cr[2 * j], cr[2 * j + 1], a_r, b_r);
        dmma(cr[2 * j], cr[2 * j + 1], na_i, b_i);
        dmma(ci[2 * j], ci[2 * j + 1], a_r, b_i);
        dmma(ci[2 * j], ci[2 * j + 1], a_i, b_r);
      }
    }
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += cr[i] + ci[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d kHz\n", sms, clk);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    for (int blocksPerSM : {1, 2, 4}) {
      int iters = 20000;
      cudaEventRecord(e0);
      dfma_loop<<<sms * blocksPerSM, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * 256.0 * sms * blocksPerSM;
      printf("DFMA  %d blk/SM x256: %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
      cudaEventRecord(e0);
      dmma_loop<<<sms * blocksPerSM, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * 8.0 * sms * blocksPerSM;
      printf("DMMA  %d blk/SM x256: %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
    }
    size_t smem = 2 * 64 * LD * 8;
    cudaFuncSetAttribute(zmm_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int reps = 400;
    cudaEventRecord(e0);
    zmm_loop<<<sms, 256, smem>>>(out, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 8.0 * 64 * 64 * 64 * reps * sms;
    printf("ZMM64 smem-B, 1 CTA/SM: %.2f TFLOP/s (%.2f us per 64x64 complex product per SM)\n",
           fl / ms / 1e9, ms * 1e3 / reps);
    cudaError_t err = cudaGetLastError();
    if (err) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
  }
  return 0;
}
