// Microbenchmark: throughput of every FP64 mma.sync shape sm_100a accepts
// (m8n8k4, m16n8k4, m16n8k8, m16n8k16) and of DFMA, with 8 or 16 warps per SM and
// NACC independent accumulators per warp.  Standalone; not the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes_probe tools/dmma_shapes_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_m8n8k4(double* out, int iters) {
  double acc[NACC][2] = {};
  double a = 1e-3 * threadIdx.x, b = 1.0 + 1e-6 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void k_m16n8k4(double* out, int iters) {
  double acc[NACC][4] = {};
  double a0 = 1e-3 * threadIdx.x, a1 = a0 + 1, b = 1.0 + 1e-6 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void k_m16n8k8(double* out, int iters) {
  double acc[NACC][4] = {};
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 1e-3 * threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 1.0 + 1e-6 * threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void k_m16n8k16(double* out, int iters) {
  double acc[NACC][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * threadIdx.x + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + 1e-6 * threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a[16], b = 1.0000001, c = 1e-9;
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
static void run(const char* name, K kern, double flop_per_warp_iter, int warps, int iters, int sms) {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms;
  kern<<<blocks, 32 * warps>>>(out, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = flop_per_warp_iter * warps * (double)blocks * iters;
  printf("%-22s warps/SM %2d : %8.2f TFLOP/s (%.3f ms)  err=%s\n", name, warps, flops / (best * 1e-3) / 1e12, best,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  const int it = 20000;
  for (int w : {4, 8, 16}) {
    run("dfma x16", k_dfma, 2.0 * 32 * 16, w, it, sms);
    run("m8n8k4 x4", k_m8n8k4<4>, 2.0 * 8 * 8 * 4 * 4, w, it, sms);
    run("m8n8k4 x8", k_m8n8k4<8>, 2.0 * 8 * 8 * 4 * 8, w, it, sms);
    run("m8n8k4 x16", k_m8n8k4<16>, 2.0 * 8 * 8 * 4 * 16, w, it, sms);
    run("m16n8k4 x4", k_m16n8k4<4>, 2.0 * 16 * 8 * 4 * 4, w, it, sms);
    run("m16n8k4 x8", k_m16n8k4<8>, 2.0 * 16 * 8 * 4 * 8, w, it, sms);
    run("m16n8k8 x4", k_m16n8k8<4>, 2.0 * 16 * 8 * 8 * 4, w, it / 2, sms);
    run("m16n8k8 x8", k_m16n8k8<8>, 2.0 * 16 * 8 * 8 * 8, w, it / 2, sms);
    run("m16n8k16 x4", k_m16n8k16<4>, 2.0 * 16 * 8 * 16 * 4, w, it / 4, sms);
    run("m16n8k16 x8", k_m16n8k16<8>, 2.0 * 16 * 8 * 16 * 8, w, it / 4, sms);
  }
  return 0;
}
