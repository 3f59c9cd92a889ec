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
// three 64 KB matrix images (X = Omega/2^s, the shared operand of the Taylor scheme /
// squarings, running chunk product P).  TMEM: the powers X^2, X^3, X^6 as strips.
// Products: DMMA.8x8x4 (qal_dev.cuh).
#include "qal_dev.cuh"
#include "qal_internal.h"
#include "qal_slice.cuh"

namespace qal {

constexpr int FWD_SMEM_BYTES = 3 * IMG * 8 + (8 * 64 + 16) * 8;

// U = expm(X 2^s) given X's strip in `A` and its image in SX; result left in A.
// m = 8: T8 in 3 products; m = 18: T18 in 5 products (qal_slice.cuh); then s squarings.
// Uses SX4 as the shared operand buffer and TMEM slots 0..2.  Returns the products done.
__device__ __forceinline__ int expm_fast(Strip& A, Strip& acc, int m, int s, double* SX, double* SX4, uint32_t tm,
                                         const Lane& L) {
  const uint32_t T0 = tm, T1 = tm + 128, T2 = tm + 256;
  int prods;
  zero(acc); mma_acc(acc, A, SX, L);                   // A2 = X X
  tmem_store(T0, acc);
  if (m == 8) {
    // W = c1 X + c2 A2 (shared), Y = A2 W
    copy(A, acc);
    zero(acc);
    add_strip(acc, c_t8[1], A);
    add_img(acc, c_t8[0], SX, L);
    store_img(SX4, acc, L);                            // no reader of SX4 is in flight
    __syncthreads();
    zero(acc); mma_acc(acc, A, SX4, L);                // Y
    tmem_store(T1, acc);
    __syncthreads();                                   // all reads of SX4 (W) done
    // R = Y + c5 A2 (shared);  L = Y + c3 A2 + c4 X (registers, in place over A2)
    store_img_axpy(SX4, acc, c_t8[4], A, L);
#pragma unroll
    for (int i = 0; i < 16; ++i) { A.re[i] = fma(c_t8[2], A.re[i], acc.re[i]); A.im[i] = fma(c_t8[2], A.im[i], acc.im[i]); }
    add_img(A, c_t8[3], SX, L);
    __syncthreads();
    zero(acc);                                         // T8 = c6 Y + c7 A2 + X + I + L R
    add_tm(acc, c_t8[5], T1);
    add_tm(acc, c_t8[6], T0);
    add_img(acc, 1.0, SX, L);
    add_diag(acc, 1.0, L);
    mma_acc(acc, A, SX4, L);
    copy(A, acc);
    prods = 3;
  } else {
    copy(A, acc);
    zero(acc); mma_acc(acc, A, SX, L);                 // A3 = A2 X
    tmem_store(T1, acc);
    store_img(SX4, acc, L);                            // A3 shared (no reader of SX4 in flight)
    copy(A, acc);
    __syncthreads();
    zero(acc); mma_acc(acc, A, SX4, L);                // A6 = A3 A3
    tmem_store(T2, acc);
    // B5 = e1 X + e2 A2 + A6 (shared)
    add_img(acc, c_t18[T18_B5][1], SX, L);
    add_tm(acc, c_t18[T18_B5][2], T0);
    __syncthreads();                                   // reads of SX4 (A3) done
    store_img(SX4, acc, L);
    // B1 = a1 X + a2 A2 + a3 A3 -> A
    zero(A);
    add_img(A, c_t18[T18_B1][1], SX, L);
    add_tm(A, c_t18[T18_B1][2], T0);
    add_tm(A, c_t18[T18_B1][3], T1);
    // acc = B4
    zero(acc);
    add_diag(acc, c_t18[T18_B4][0], L);
    add_img(acc, c_t18[T18_B4][1], SX, L);
    add_tm(acc, c_t18[T18_B4][2], T0);
    add_tm(acc, c_t18[T18_B4][3], T1);
    add_tm(acc, c_t18[T18_B4][4], T2);
    __syncthreads();                                   // B5 image complete
    mma_acc(acc, A, SX4, L);                           // A9 = B4 + B1 B5
    __syncthreads();                                   // reads of SX4 (B5) done
    store_img(SX4, acc, L);                            // A9 shared
    // L = B3 + A9 -> A
    copy(A, acc);
    add_diag(A, c_t18[T18_B3][0], L);
    add_img(A, c_t18[T18_B3][1], SX, L);
    add_tm(A, c_t18[T18_B3][2], T0);
    add_tm(A, c_t18[T18_B3][3], T1);
    add_tm(A, c_t18[T18_B3][4], T2);
    zero(acc);                                         // T18 = B2 + L A9
    add_diag(acc, c_t18[T18_B2][0], L);
    add_img(acc, c_t18[T18_B2][1], SX, L);
    add_tm(acc, c_t18[T18_B2][2], T0);
    add_tm(acc, c_t18[T18_B2][3], T1);
    add_tm(acc, c_t18[T18_B2][4], T2);
    __syncthreads();                                   // A9 image complete
    mma_acc(acc, A, SX4, L);
    copy(A, acc);
    prods = 5;
  }
  for (int q = 0; q < s; ++q) {                        // squarings
    __syncthreads();                                   // all reads of SX4 done
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
      choose_scheme(nrm, m, s);
      if (!(nrm <= 1e300) && threadIdx.x == 0) bad_sh = 1;
      const double sc = ldexp(1.0, -s);
#pragma unroll
      for (int i = 0; i < 16; ++i) { A.re[i] *= sc; A.im[i] *= sc; }
      store_img(SX, A, L);
      __syncthreads();
      nprod += expm_fast(A, acc, m, s, SX, SX4, tm, L);
      const size_t slot = (size_t)b * G.count + k;
      if (O.U_nat) store_nat(O.U_nat + slot * PLANE, A, L);
      if (O.U_img) store_img_l2(O.U_img + slot * IMG, A, L, l2_evict_first());
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
  {
    const cudaError_t e = ensure_smem((const void*)k_expm_fold, FWD_SMEM_BYTES);
    if (e != cudaSuccess) return e;
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
