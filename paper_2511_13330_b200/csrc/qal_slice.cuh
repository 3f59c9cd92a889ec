// qal_slice.cuh -- per-slice generator assembly (a1-a3) and Paterson-Stockmeyer
// blocks shared by the forward (qal_magnus.cu) and gradient (qal_grad.cu) kernels.
#pragma once
#include "qal_dev.cuh"
#include "qal_internal.h"

namespace qal {

// X += a * M (natural layout, strip of lane L)
__device__ __forceinline__ void axpy_nat(Strip& X, double a, const double2* __restrict__ M, const Lane& L) {
  const uint64_t keep = l2_evict_last();   // the basis is shared by every CTA and slice
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double vx, vy;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(vx), "=d"(vy)
                 : "l"(M + L.r * 64 + 4 * i + L.t), "l"(keep));
    X.re[i] = fma(a, vx, X.re[i]);
    X.im[i] = fma(a, vy, X.im[i]);
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
  uint32_t v[32], w[32];
  tmem_ld32(addr, v);
  tmem_ld32(addr + 32, w);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    s.re[i] = __hiloint2double(static_cast<int>(v[2 * i + 1]), static_cast<int>(v[2 * i]));
    s.im[i] = __hiloint2double(static_cast<int>(w[2 * i + 1]), static_cast<int>(w[2 * i]));
  }
}

// ---------------------------------------------------------------------------------------------
// Taylor evaluation schemes with fewer products than Paterson-Stockmeyer (A15; the coefficients
// were solved in 50-digit arithmetic by tools/derive_taylor18.py / derive_taylor8.py, match
// sum_k A^k/k! exactly as polynomials, and were checked for rounding stability):
//   T8  (3 products):  A2 = A^2, Y = A2 (c1 A + c2 A2),
//                      T8 = (Y + c3 A2 + c4 A)(Y + c5 A2) + c6 Y + c7 A2 + A + I
//   T18 (5 products):  A2 = A^2, A3 = A2 A, A6 = A3^2,
//                      A9 = B1 B5 + B4,  T18 = B2 + (B3 + A9) A9,
//                      B_i = x0 I + x1 A + x2 A2 + x3 A3 + x6 A6 (table below, columns I, A, A2, A3, A6)
// theta_m: sum_{k>m} theta^k/k! <= 2^-53 e^-theta.
constexpr double THETA_T8 = 0.06939604586390902;
constexpr double THETA_T18 = 1.0802931244608445;
__constant__ double c_t8[7] = {0.019920476822239894, 0.004980119205559973, 0.07665265321119147,
                               0.8765009801785554,   0.12255211501120747,  2.9743072048476265, 0.5};
enum { T18_B1 = 0, T18_B5, T18_B4, T18_B3, T18_B2 };
__constant__ double c_t18[5][5] = {
    {0.0, 1.4059892894192667e-06, 1.1247914315354133e-07, 1.2497682572615703e-08, 0.0},           // B1
    {0.0, 38083.5, 17472.375, 0.0, 1.0},                                                          // B5
    {0.0, 1.6125176868819238, 0.07122912172133387, 0.0029909869115921006, 3.4689174187293366e-05},  // B4
    {-11.148502971774368, -1.680158138789062, -0.05717798464788655, 0.0069821012248805206,
     -3.3497501708607054e-05},                                                                    // B3
    {1.0, 18.977158224241858, 2.000116014975223, 0.42108104943688435, -0.00026748043271311394}};   // B2

// scheme (8 or 18) and squarings s for ||Omega||_1 = nrm: the cheaper of 3 + s8 and 5 + s18
__device__ __forceinline__ void choose_scheme(double nrm, int& m, int& s) {
  if (!(nrm <= 1e300)) { m = 18; s = 0; return; }
  int s8 = 0, s18 = 0;
  double a = nrm;
  while (a > THETA_T8 && s8 < 1100) { a *= 0.5; ++s8; }
  a = nrm;
  while (a > THETA_T18 && s18 < 1100) { a *= 0.5; ++s18; }
  if (3 + s8 < 5 + s18) { m = 8; s = s8; } else { m = 18; s = s18; }
}

// strip accumulation helpers (acc += a * source)
__device__ __forceinline__ void add_diag(Strip& acc, double a, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (is_diag(L, i)) acc.re[i] += a;
}
__device__ __forceinline__ void add_img(Strip& acc, double a, const double* img, const Lane& L) {
  if (a == 0.0) return;
  Strip x;
  load_img(x, img, L);
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc.re[i] = fma(a, x.re[i], acc.re[i]); acc.im[i] = fma(a, x.im[i], acc.im[i]); }
}
__device__ __forceinline__ void add_img_l2(Strip& acc, double a, const double* img, const Lane& L, uint64_t pol) {
  if (a == 0.0) return;
  Strip x;
  load_img_l2(x, img, L, pol);
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc.re[i] = fma(a, x.re[i], acc.re[i]); acc.im[i] = fma(a, x.im[i], acc.im[i]); }
}
__device__ __forceinline__ void add_tm(Strip& acc, double a, uint32_t addr) {
  if (a == 0.0) return;
  tmem_axpy(acc, a, addr);
}
__device__ __forceinline__ void add_strip(Strip& acc, double a, const Strip& x) {
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc.re[i] = fma(a, x.re[i], acc.re[i]); acc.im[i] = fma(a, x.im[i], acc.im[i]); }
}

}  // namespace qal
