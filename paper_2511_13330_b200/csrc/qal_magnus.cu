// qal_magnus.cu -- K2+K3: per-slice Magnus generator, expm and in-CTA ordered fold.
//
// PAPER.md P:125-141 (Eqs. 13-15) generalised to 4th order (A1, A2):
//   Omega_k = (h/2)(A_1 + A_2) - (sqrt(3) h^2/12)[A_1, A_2],  A_a = L(tau_{k,a}),
// expanded through the bilinear basis (a3): the commutator of the two node
// generators is a linear combination of [L0, L_j] and [L_a, L_c], so Omega_k costs
// no matrix product.  U_k = expm(Omega_k) by scaling and squaring around a
// Paterson-Stockmeyer Taylor polynomial of degree m in {8, 12, 16} (A15), then the
// CTA folds its chunk of slices, later slice on the LEFT (Eq. 15, A4).
//
// One persistent CTA (8 warps) per SM; work item = (pulse, chunk).  Shared memory:
// three 64 KB matrix images (X = Omega/2^s, X^4 / squaring buffer, running chunk
// product P).  TMEM: X^2 and X^3 strips.  Products: DMMA.8x8x4 (qal_dev.cuh).
#include "qal_dev.cuh"
#include "qal_internal.h"
#include "qal_slice.cuh"

namespace qal {

constexpr int FWD_SMEM_BYTES = 3 * IMG * 8 + (8 * 64 + 16) * 8;

// U = expm(X 2^s) given X's strip in `A` and its image in SX; result left in A.
// Uses SX4 as scratch; TMEM slots 0, 1.  Returns number of 64x64 products done.
__device__ __forceinline__ int expm_ps(Strip& A, Strip& acc, int m, int s, double* SX, double* SX4, uint32_t tm,
                                       const Lane& L) {
  // powers
  zero(acc); mma_acc(acc, A, SX, L);        // X^2
  tmem_store(tm, acc);
  copy(A, acc);
  zero(acc); mma_acc(acc, A, SX, L);        // X^3
  tmem_store(tm + 128, acc);
  copy(A, acc);
  zero(acc); mma_acc(acc, A, SX, L);        // X^4 (in acc)
  store_img(SX4, acc, L);
  const int tb = m / 4;                     // top block index: H = B_{tb-1} + c_m X^4
  ps_block(A, tb - 1, SX, tm, L);
  const double cm = inv_fact(m);
#pragma unroll
  for (int i = 0; i < 16; ++i) { A.re[i] = fma(cm, acc.re[i], A.re[i]); A.im[i] = fma(cm, acc.im[i], A.im[i]); }
  __syncthreads();                          // X^4 image complete
  int prods = 3;
  for (int blk = tb - 2; blk >= 0; --blk) {  // Horner in X^4
    ps_block(acc, blk, SX, tm, L);
    mma_acc(acc, A, SX4, L);
    copy(A, acc);
    ++prods;
  }
  for (int q = 0; q < s; ++q) {             // squarings
    __syncthreads();                        // all reads of SX4 done
    store_img(SX4, A, L);
    __syncthreads();
    zero(acc); mma_acc(acc, A, SX4, L);
    copy(A, acc);
    ++prods;
  }
  return prods;
}

__global__ void __launch_bounds__(NT, 1) k_expm_fold(int batch, Basis B, SliceGrid G, FwdOut O,
                                                    unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  double* SX = smem;
  double* SX4 = smem + IMG;
  double* SP = smem + 2 * IMG;
  double* red = smem + 3 * IMG;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int bad_sh;
  const Lane L = lane_id();
  if (L.w == 0) tmem_alloc512(&tmem_base_sh);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = tmem_slot_addr(tmem_base_sh, L, 0);

  const int nchunk = G.count / O.chunk;
  const int items = batch * nchunk;
  Strip A, acc;
  unsigned long long nprod = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = item / nchunk, c = item % nchunk;
    if (threadIdx.x == 0) bad_sh = 0;
    for (int kk = 0; kk < O.chunk; ++kk) {
      const int k = c * O.chunk + kk;
      build_omega(A, B, G, b, k, L);
      const double nrm = norm1(A, red, L);  // 2 syncs
      int m, s;
      choose_ms(nrm, m, s);
      if (!(nrm <= 1e300) && threadIdx.x == 0) bad_sh = 1;
      const double sc = ldexp(1.0, -s);
#pragma unroll
      for (int i = 0; i < 16; ++i) { A.re[i] *= sc; A.im[i] *= sc; }
      store_img(SX, A, L);
      __syncthreads();
      nprod += expm_ps(A, acc, m, s, SX, SX4, tm, L);
      const size_t slot = (size_t)b * G.count + k;
      if (O.U_nat) store_nat(O.U_nat + slot * PLANE, A, L);
      if (O.U_img) store_img(O.U_img + slot * IMG, A, L);
      if (O.chunk_nat) {
        if (kk == 0) {
          store_img(SP, A, L);             // P = U_k (no reader of SP is in flight)
        } else {
          zero(acc); mma_acc(acc, A, SP, L);  // P <- U_k P
          copy(A, acc);
          ++nprod;
          __syncthreads();
          store_img(SP, A, L);
        }
      }
    }
    if (O.chunk_nat) store_nat(O.chunk_nat + ((size_t)b * nchunk + c) * PLANE, A, L);
    __syncthreads();
    // status[] is zeroed by the host API before the launch; only failures are written
    if (O.status && threadIdx.x == 0 && bad_sh) O.status[b] = -4;
  }
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, nprod);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (L.w == 0) tmem_dealloc512(tmem_base_sh);
}

cudaError_t launch_expm_fold(int batch, const Basis& B, const SliceGrid& G, const FwdOut& O, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_expm_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, FWD_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = batch * (G.count / O.chunk);
  const int grid = items < num_sms() ? items : num_sms();
  prof_pre(ST_EXPM, st);
  k_expm_fold<<<grid, NT, FWD_SMEM_BYTES, st>>>(batch, B, G, O, prof_counter(ST_EXPM));
  prof_post(ST_EXPM, st);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace qal
