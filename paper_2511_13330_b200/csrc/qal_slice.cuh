// qal_slice.cuh -- per-slice generator assembly (a1-a3) and Paterson-Stockmeyer
// blocks shared by the forward (qal_magnus.cu) and gradient (qal_grad.cu) kernels.
#pragma once
#include "qal_dev.cuh"
#include "qal_internal.h"

namespace qal {

// X += a * M (natural layout, strip of lane L)
__device__ __forceinline__ void axpy_nat(Strip& X, double a, const double2* __restrict__ M, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double2 v = __ldg(M + L.r * 64 + 4 * i + L.t);
    X.re[i] = fma(a, v.x, X.re[i]);
    X.im[i] = fma(a, v.y, X.im[i]);
  }
}

// Omega_k (strip) from the generator basis and the control values of slice k (a1-a3)
__device__ __forceinline__ void build_omega(Strip& X, const Basis& B, const SliceGrid& G, int b, int k,
                                            const Lane& L) {
  const int J = B.J;
  const int nodes = (G.mode == 1) ? 2 : 1;
  const double* u = G.u + ((size_t)b * G.count + k) * nodes * J;
  zero(X);
  axpy_nat(X, G.h, B.L0 + (size_t)b * B.L0_stride, L);
  for (int j = 0; j < J; ++j) {
    const double v1 = __ldg(u + j), v2 = __ldg(u + (nodes - 1) * J + j);
    axpy_nat(X, 0.5 * G.h * (v1 + v2), B.Lc + (size_t)j * PLANE, L);
  }
  if (B.ncomm > 0) {
    const double2* Cb = B.Lcomm + (size_t)b * B.Lcomm_stride;
    for (int j = 0; j < J; ++j) {
      const double v1 = __ldg(u + j), v2 = __ldg(u + J + j);
      axpy_nat(X, -G.c4 * (v2 - v1), Cb + (size_t)j * PLANE, L);
    }
    int p = J;
    for (int a = 0; a < J; ++a)
      for (int c = a + 1; c < J; ++c, ++p) {
        const double coef = -G.c4 * (__ldg(u + a) * __ldg(u + J + c) - __ldg(u + c) * __ldg(u + J + a));
        axpy_nat(X, coef, Cb + (size_t)p * PLANE, L);
      }
  }
}

// acc = c0 I + c1 X + c2 X^2 + c3 X^3  (Paterson-Stockmeyer block, c_i = 1/i!), X
// from an image (shared or global), X^2 / X^3 from TMEM at tm / tm + 128.
__device__ __forceinline__ void ps_block(Strip& acc, int blk, const double* SX, uint32_t tm, const Lane& L) {
  const double c0 = inv_fact(4 * blk), c1 = inv_fact(4 * blk + 1);
  const double c2 = inv_fact(4 * blk + 2), c3 = inv_fact(4 * blk + 3);
  load_img(acc, SX, L);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    acc.re[i] = c1 * acc.re[i] + (is_diag(L, i) ? c0 : 0.0);
    acc.im[i] = c1 * acc.im[i];
  }
  tmem_axpy(acc, c2, tm);
  tmem_axpy(acc, c3, tm + 128);
}

// derivative of a Paterson-Stockmeyer block: acc = c1 dX + c2 dX^2 + c3 dX^3
__device__ __forceinline__ void dps_block(Strip& acc, int blk, const double* dX, uint32_t tm2, const Lane& L) {
  const double c1 = inv_fact(4 * blk + 1), c2 = inv_fact(4 * blk + 2), c3 = inv_fact(4 * blk + 3);
  load_img(acc, dX, L);
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc.re[i] *= c1; acc.im[i] *= c1; }
  tmem_axpy(acc, c2, tm2);
  tmem_axpy(acc, c3, tm2 + 128);
}

__device__ __forceinline__ void tmem_load(Strip& s, uint32_t addr) {
  tmem_load_half(addr, s.re);
  tmem_load_half(addr + 32, s.im);
}

}  // namespace qal
