// qal_product.cu -- K1 (Liouvillian + commutator basis), K4 (ordered-product tree
// level), K5 (fidelity), K0 (FP64 peak probe).
#include "qal_dev.cuh"
#include "qal_internal.h"

namespace qal {

// ------------------------------------------------------------------ K4
// One tree level of Eq. 15: out[b][i] = in[b][2i+1] in[b][2i] (later factor
// on the LEFT); an odd last element is carried up unchanged.  One CTA per output.
__global__ void __launch_bounds__(NT, 2) k_tree_level(int batch, int cnt, const double2* __restrict__ in,
                                                      double2* __restrict__ out, unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  const Lane L = lane_id();
  const int half = (cnt + 1) / 2;
  const int b = blockIdx.x / half, i = blockIdx.x % half;
  const double2* src = in + (size_t)b * cnt * PLANE;
  double2* dst = out + ((size_t)b * half + i) * PLANE;
  if (2 * i + 1 == cnt) {  // carry
    for (int e = threadIdx.x; e < PLANE; e += NT) dst[e] = src[(size_t)(cnt - 1) * PLANE + e];
    return;
  }
  block_nat_to_img(smem, src + (size_t)(2 * i) * PLANE);
  Strip A, acc;
  load_nat(A, src + (size_t)(2 * i + 1) * PLANE, L);
  __syncthreads();
  zero(acc);
  mma_acc(acc, A, smem, L);
  store_nat(dst, acc, L);
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, 1ull);
}

cudaError_t launch_tree_level(int batch, int cnt, const double2* in, double2* out, cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_tree_level, IMG * 8);
    if (e != cudaSuccess) return e;
  }
  const int half = (cnt + 1) / 2;
  prof_pre(ST_TREE, st);
  k_tree_level<<<batch * half, NT, IMG * 8, st>>>(batch, cnt, in, out, prof_counter(ST_TREE));
  prof_post(ST_TREE, st);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ scans (log-depth prefix/suffix)
// One Hillis-Steele level over per-pulse sequences of `cnt` matrices (later factor on the LEFT):
//   prefix (dir 0): out[s] = in[s] in[s-d]  (s >= d), else copy  -> after all levels: U_s ... U_0
//   suffix (dir 1): out[s] = in[s+d] in[s]  (s+d < cnt), else copy -> U_{cnt-1} ... U_s
__global__ void __launch_bounds__(NT, 2) k_scan_level(int cnt, int d, int dir, const double2* __restrict__ in,
                                                      double2* __restrict__ out, unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  const Lane L = lane_id();
  const int b = blockIdx.x / cnt, s = blockIdx.x % cnt;
  const double2* src = in + (size_t)b * cnt * PLANE;
  double2* dst = out + ((size_t)b * cnt + s) * PLANE;
  const int partner = dir == 0 ? s - d : s + d;
  if (partner < 0 || partner >= cnt) {
    for (int e = threadIdx.x; e < PLANE; e += NT) dst[e] = src[(size_t)s * PLANE + e];
    return;
  }
  const int later = dir == 0 ? s : partner, earlier = dir == 0 ? partner : s;
  block_nat_to_img(smem, src + (size_t)earlier * PLANE);
  Strip A, acc;
  load_nat(A, src + (size_t)later * PLANE, L);
  __syncthreads();
  zero(acc);
  mma_acc(acc, A, smem, L);
  store_nat(dst, acc, L);
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, 1ull);
}

// exclusive outputs from the inclusive scans: pre[s] = incl_pre[s-1] (I at s = 0),
// suf[s] = incl_suf[s+1] (I at s = cnt-1)
__global__ void __launch_bounds__(NT) k_scan_shift(int cnt, const double2* __restrict__ ip, const double2* __restrict__ is,
                                                   double2* __restrict__ pre, double2* __restrict__ suf) {
  const int b = blockIdx.x / cnt, s = blockIdx.x % cnt;
  double2* p = pre + ((size_t)b * cnt + s) * PLANE;
  double2* q = suf + ((size_t)b * cnt + s) * PLANE;
  const double2* ps = s > 0 ? ip + ((size_t)b * cnt + s - 1) * PLANE : nullptr;
  const double2* qs = s + 1 < cnt ? is + ((size_t)b * cnt + s + 1) * PLANE : nullptr;
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const double2 id = make_double2((e >> 6) == (e & 63) ? 1.0 : 0.0, 0.0);
    if (pre) p[e] = ps ? ps[e] : id;
    if (suf) q[e] = qs ? qs[e] : id;
  }
}

cudaError_t launch_scan(int batch, int cnt, const double2* U, double2* pre, double2* suf, double2* ws,
                        cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_scan_level, IMG * 8);
    if (e != cudaSuccess) return e;
  }
  const size_t seq = (size_t)batch * cnt * PLANE;
  double2* buf[2][2] = {{ws, ws + seq}, {ws + 2 * seq, ws + 3 * seq}};   // [dir][ping-pong]
  const double2* res[2] = {U, U};
  for (int dir = 0; dir < 2; ++dir) {
    if ((dir == 0 && !pre) || (dir == 1 && !suf)) continue;
    const double2* in = U;
    int pp = 0;
    for (int d = 1; d < cnt; d <<= 1) {
      prof_pre(ST_TREE, st);
      k_scan_level<<<batch * cnt, NT, IMG * 8, st>>>(cnt, d, dir, in, buf[dir][pp], prof_counter(ST_TREE));
      prof_post(ST_TREE, st);
      ++launch_counter();
      in = buf[dir][pp];
      pp ^= 1;
    }
    res[dir] = in;
  }
  k_scan_shift<<<batch * cnt, NT, 0, st>>>(cnt, res[0], res[1], pre, suf);
  ++launch_counter();
  return cudaGetLastError();
}

// out[i] = A[i] B[i] with element strides (0 = broadcast); one CTA per product
__global__ void __launch_bounds__(NT, 2) k_batched_mm(const double2* __restrict__ A, long long sa,
                                                      const double2* __restrict__ B, long long sb,
                                                      double2* __restrict__ C, unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  const Lane L = lane_id();
  const size_t i = blockIdx.x;
  block_nat_to_img(smem, B + i * sb);
  Strip a, acc;
  load_nat(a, A + i * sa, L);
  __syncthreads();
  zero(acc);
  mma_acc(acc, a, smem, L);
  store_nat(C + i * PLANE, acc, L);
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, 1ull);
}

cudaError_t launch_batched_mm(int count, const double2* A, long long sa, const double2* B, long long sb, double2* C,
                              cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_batched_mm, IMG * 8);
    if (e != cudaSuccess) return e;
  }
  prof_pre(ST_TREE, st);
  k_batched_mm<<<count, NT, IMG * 8, st>>>(A, sa, B, sb, C, prof_counter(ST_TREE));
  prof_post(ST_TREE, st);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K5
// F[b] = Re Tr(S_V^dag Lambda_b) / d^2 with S_V[i+dj, k+dl] = conj(V[j][l]) V[i][k] (A8):
// F = Re sum V[j][l] conj(V[i][k]) Lambda[i+dj][k+dl] / d^2.  d = 8.  One CTA per pulse.
__global__ void __launch_bounds__(NT) k_fidelity(const double2* __restrict__ Lam, const double2* __restrict__ V,
                                                 double* __restrict__ F) {
  __shared__ double2 Vs[64];
  __shared__ double red[16];
  const Lane L = lane_id();
  if (threadIdx.x < 64) Vs[threadIdx.x] = V[threadIdx.x];
  __syncthreads();
  const double2* M = Lam + (size_t)blockIdx.x * PLANE;
  double acc = 0.0;
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int a = e >> 6, c = e & 63;
    const int i = a & 7, j = a >> 3, k = c & 7, l = c >> 3;
    const double2 vjl = Vs[j * 8 + l], vik = Vs[i * 8 + k], x = M[e];
    // w = vjl * conj(vik)
    const double wr = vjl.x * vik.x + vjl.y * vik.y;
    const double wi = vjl.y * vik.x - vjl.x * vik.y;
    acc += wr * x.x - wi * x.y;
  }
  const double s = block_sum(acc, red, L);
  if (threadIdx.x == 0) F[blockIdx.x] = s / 64.0;
}

cudaError_t launch_fidelity(int batch, const double2* Lam, const double2* V, double* F, cudaStream_t st) {
  prof_pre(ST_FID, st);
  k_fidelity<<<batch, NT, 0, st>>>(Lam, V, F);
  prof_post(ST_FID, st);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1
// Eq. 8, column stacking (A5): with a = p d + r, c = s d + q (p, s: column index of
// rho; r, q: row index),
//   (I (x) H)[a][c] = delta_ps H[r][q],   (H^T (x) I)[a][c] = H[s][p] delta_rq,
//   (conj(C) (x) C)[a][c] = conj(C[p][s]) C[r][q].
// blockIdx.y = 0 -> L0 of pulse blockIdx.z (drift + all dissipators); y = 1 + j -> L_j.
__global__ void __launch_bounds__(NT) k_liouvillian(const double2* __restrict__ H0, const double2* __restrict__ Hc,
                                                    int ncops, const double2* __restrict__ C,
                                                    double2* __restrict__ L0, double2* __restrict__ Lc, int yoff) {
  constexpr int d = 8;
  __shared__ double2 H[64], S[64];   // H and S = sum_c C^dag C
  __shared__ double2 Cs[64];
  const int y = blockIdx.y + yoff, b = blockIdx.z;
  const bool drift = (y == 0);
  const double2* Hsrc = drift ? H0 + (size_t)b * 64 : Hc + (size_t)(y - 1) * 64;
  if (threadIdx.x < 64) {
    H[threadIdx.x] = Hsrc[threadIdx.x];
    S[threadIdx.x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (drift) {
    for (int cc = 0; cc < ncops; ++cc) {
      if (threadIdx.x < 64) Cs[threadIdx.x] = C[(size_t)cc * 64 + threadIdx.x];
      __syncthreads();
      if (threadIdx.x < 64) {  // S[r][q] += sum_m conj(C[m][r]) C[m][q]
        const int r = threadIdx.x >> 3, q = threadIdx.x & 7;
        double sr = 0.0, si = 0.0;
        for (int m = 0; m < d; ++m) {
          const double2 x = Cs[m * 8 + r], z = Cs[m * 8 + q];
          sr += x.x * z.x + x.y * z.y;
          si += x.x * z.y - x.y * z.x;
        }
        S[threadIdx.x].x += sr;
        S[threadIdx.x].y += si;
      }
      __syncthreads();
    }
  }
  double2* out = drift ? L0 + (size_t)b * PLANE : Lc + (size_t)(y - 1) * PLANE;
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int a = e >> 6, c = e & 63;
    const int p = a >> 3, r = a & 7, s = c >> 3, q = c & 7;
    // Hamiltonian part: -i (delta_ps H[r][q] - H[s][p] delta_rq)
    double hr = 0.0, hi = 0.0;
    if (p == s) { hr += H[r * 8 + q].x; hi += H[r * 8 + q].y; }
    if (r == q) { hr -= H[s * 8 + p].x; hi -= H[s * 8 + p].y; }
    double vr = hi, vi = -hr;  // -i (hr + i hi) = hi - i hr
    if (drift) {
      for (int cc = 0; cc < ncops; ++cc) {
        const double2 cps = C[(size_t)cc * 64 + p * 8 + s], crq = C[(size_t)cc * 64 + r * 8 + q];
        // conj(cps) * crq
        vr += cps.x * crq.x + cps.y * crq.y;
        vi += cps.x * crq.y - cps.y * crq.x;
      }
      if (p == s) { vr -= 0.5 * S[r * 8 + q].x; vi -= 0.5 * S[r * 8 + q].y; }
      if (r == q) { vr -= 0.5 * S[s * 8 + p].x; vi -= 0.5 * S[s * 8 + p].y; }
    }
    out[e] = make_double2(vr, vi);
  }
}

cudaError_t launch_liouvillian(int batch, const double2* H0, int J, const double2* Hc, int ncops, const double2* C,
                               double2* L0, double2* Lc, cudaStream_t st) {
  // drift part of every pulse (y = 0, z = pulse), then the J control parts once
  prof_pre(ST_LIOUV, st);
  k_liouvillian<<<dim3(1, 1, batch), NT, 0, st>>>(H0, Hc, ncops, C, L0, Lc, 0);
  prof_post(ST_LIOUV, st);
  ++launch_counter();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || J == 0) return e;
  prof_pre(ST_LIOUV, st);
  k_liouvillian<<<dim3(1, J, 1), NT, 0, st>>>(H0, Hc, ncops, C, L0, Lc, 1);
  prof_post(ST_LIOUV, st);
  ++launch_counter();
  return cudaGetLastError();
}

// [X, Y] = X Y - Y X for the commutator basis of the order-4 generator (a3, A2):
// blockIdx.y = j < J:   [L0_b, L_j];   j >= J: pair (a, c), a < c, lexicographic.
__global__ void __launch_bounds__(NT, 1) k_commutators(int J, const double2* __restrict__ L0,
                                                       const double2* __restrict__ Lc,
                                                       double2* __restrict__ Lcomm, unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  double* SX = smem;
  double* SY = smem + IMG;
  const Lane L = lane_id();
  const int b = blockIdx.x, m = blockIdx.y;
  const int ncomm = J + J * (J - 1) / 2;
  const double2 *Xp, *Yp;
  if (m < J) {
    Xp = L0 + (size_t)b * PLANE;
    Yp = Lc + (size_t)m * PLANE;
  } else {
    int p = J, a = 0, c = 1;
    for (int aa = 0; aa < J; ++aa)
      for (int cc = aa + 1; cc < J; ++cc, ++p)
        if (p == m) { a = aa; c = cc; }
    Xp = Lc + (size_t)a * PLANE;
    Yp = Lc + (size_t)c * PLANE;
  }
  block_nat_to_img(SX, Xp);
  block_nat_to_img(SY, Yp);
  Strip A, acc;
  __syncthreads();
  zero(acc);
  load_nat(A, Xp, L);
  mma_acc(acc, A, SY, L);  // X Y
  load_nat(A, Yp, L);
#pragma unroll
  for (int i = 0; i < 16; ++i) { A.re[i] = -A.re[i]; A.im[i] = -A.im[i]; }
  mma_acc(acc, A, SX, L);  // - Y X
  store_nat(Lcomm + ((size_t)b * ncomm + m) * PLANE, acc, L);
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, 2ull);
}

cudaError_t launch_commutators(int batch, int J, const double2* L0, const double2* Lc, double2* Lcomm,
                               cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_commutators, 2 * IMG * 8);
    if (e != cudaSuccess) return e;
  }
  const int ncomm = J + J * (J - 1) / 2;
  prof_pre(ST_COMM, st);
  k_commutators<<<dim3(batch, ncomm), NT, 2 * IMG * 8, st>>>(J, L0, Lc, Lcomm, prof_counter(ST_COMM));
  prof_post(ST_COMM, st);
  ++launch_counter();
  return cudaGetLastError();
}

// cotangent of the fidelity (A8): C = S_V^dag / d^2, C[a][c] = V[j][l] conj(V[i][k]) / d^2 with
// a = k + d l, c = i + d j (so that dF = Re Tr(C dLambda)).  d = 8.
__global__ void __launch_bounds__(NT) k_fidelity_cotangent(const double2* __restrict__ V, double2* __restrict__ C) {
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int a = e >> 6, c = e & 63;
    const int k = a & 7, l = a >> 3, i = c & 7, j = c >> 3;
    const double2 vjl = V[j * 8 + l], vik = V[i * 8 + k];
    C[e] = make_double2((vjl.x * vik.x + vjl.y * vik.y) / 64.0, (vjl.y * vik.x - vjl.x * vik.y) / 64.0);
  }
}
cudaError_t launch_fidelity_cotangent(const double2* V, double2* C, cudaStream_t st) {
  k_fidelity_cotangent<<<1, NT, 0, st>>>(V, C);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Eqs. 16-17
// Logical projection Pi = P^dag Lambda P (P = [vec(rho_0) vec(rho_1)], n x 2), the mean squared
// error loss = 1/4 ||Pi - G||_F^2 (Frobenius via A^dag A, A22), and its cotangent
// C = 1/2 P (Pi - G)^dag P^dag, so that d loss = Re Tr(C dLambda).  One CTA per pulse.
__global__ void __launch_bounds__(NT) k_logical_loss(const double2* __restrict__ Lam, const double2* __restrict__ Pp,
                                                     const double2* __restrict__ Gt, double* __restrict__ loss,
                                                     double2* __restrict__ C) {
  __shared__ double red[8][9];
  __shared__ double2 Ash[4];
  const Lane L = lane_id();
  const double2* M = Lam + (size_t)blockIdx.x * PLANE;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // Pi_ab re/im, ab = 00, 01, 10, 11
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int i = e >> 6, j = e & 63;
    const double2 x = M[e];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const double2 pia = __ldg(Pp + i * 2 + a);   // conj(P_ia) Lambda_ij P_jb
      const double tr = pia.x * x.x + pia.y * x.y, ti = pia.x * x.y - pia.y * x.x;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double2 pjb = __ldg(Pp + j * 2 + b);
        acc[2 * (2 * a + b)] += tr * pjb.x - ti * pjb.y;
        acc[2 * (2 * a + b) + 1] += tr * pjb.y + ti * pjb.x;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
  if (L.lane == 0)
    for (int q = 0; q < 8; ++q) red[L.w][q] = acc[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int ab = 0; ab < 4; ++ab) {
      double pr = 0.0, pi = 0.0;
      for (int w = 0; w < 8; ++w) { pr += red[w][2 * ab]; pi += red[w][2 * ab + 1]; }
      const double2 g = Gt[ab];
      Ash[ab] = make_double2(pr - g.x, pi - g.y);
      l += (pr - g.x) * (pr - g.x) + (pi - g.y) * (pi - g.y);
    }
    loss[blockIdx.x] = 0.25 * l;
  }
  __syncthreads();
  if (!C) return;
  double2* Cb = C + (size_t)blockIdx.x * PLANE;
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int i = e >> 6, j = e & 63;
    double cr = 0.0, ci = 0.0;   // 1/2 sum_ab P_ia conj(A_ba) conj(P_jb)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double2 pia = __ldg(Pp + i * 2 + a), pjb = __ldg(Pp + j * 2 + b), A = Ash[2 * b + a];
        // w = P_ia * conj(A_ba)
        const double wr = pia.x * A.x + pia.y * A.y, wi = pia.y * A.x - pia.x * A.y;
        // w * conj(P_jb)
        cr += wr * pjb.x + wi * pjb.y;
        ci += wi * pjb.x - wr * pjb.y;
      }
    Cb[e] = make_double2(0.5 * cr, 0.5 * ci);
  }
}

cudaError_t launch_logical_loss(int batch, const double2* Lam, const double2* Pproj, const double2* Gt, double* loss,
                                double2* C, cudaStream_t st) {
  k_logical_loss<<<batch, NT, 0, st>>>(Lam, Pproj, Gt, loss, C);
  ++launch_counter();
  return cudaGetLastError();
}

// Adam (ref [13]): m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2; theta <- theta - lr mhat/(sqrt(vhat)+eps)
__global__ void __launch_bounds__(NT) k_adam(int n, double* __restrict__ th, const double* __restrict__ g,
                                             double* __restrict__ m, double* __restrict__ v, double c1, double c2,
                                             double lr, double b1, double b2, double eps) {
  const int i = blockIdx.x * NT + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const double mi = b1 * m[i] + (1.0 - b1) * gi;
  const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  th[i] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
}

cudaError_t launch_adam(int n, double* theta, const double* g, double* m, double* v, int t, double lr, double b1,
                        double b2, double eps, cudaStream_t st) {
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  k_adam<<<(n + NT - 1) / NT, NT, 0, st>>>(n, theta, g, m, v, c1, c2, lr, b1, b2, eps);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a1 (NODES controls)
// configs[3] controls (A11) at the Gauss-Legendre nodes of slices k0..k0+count-1.
__global__ void __launch_bounds__(NT) k_sample_sines(int J, int nterm, const double* __restrict__ prm, double umax,
                                                     double h, int k0, int count, double* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * NT + threadIdx.x;
  if (idx >= (long long)count * 2 * J) return;
  const int j = (int)(idx % J);
  const int a = (int)((idx / J) % 2);
  const long long k = idx / (2 * J) + k0;
  // explicit round-to-nearest operations (no FMA contraction): the phase 2 pi f t reaches
  // ~3e3 rad at t = 10 us, where a contracted multiply-add would move u by ~1e-13
  const double c = __ddiv_rn(__dsqrt_rn(3.0), 6.0);
  const double tk = __dmul_rn((double)k, h);
  const double t = __dadd_rn(tk, __dmul_rn(a == 0 ? __dsub_rn(0.5, c) : __dadd_rn(0.5, c), h));
  const double* p = prm + (size_t)j * nterm * 3;
  double s = 0.0, a2 = 0.0;
  for (int m = 0; m < nterm; ++m) {
    const double arg = __dadd_rn(__dmul_rn(__dmul_rn(2.0 * 3.141592653589793, p[3 * m + 1]), t), p[3 * m + 2]);
    s = __dadd_rn(s, __dmul_rn(p[3 * m], sin(arg)));
    a2 = __dadd_rn(a2, __dmul_rn(p[3 * m], p[3 * m]));
  }
  s = __ddiv_rn(s, __dsqrt_rn(__ddiv_rn(a2, 2.0)));
  const double v = __dmul_rn(__dmul_rn(0.5, umax), __dadd_rn(1.0, __dmul_rn(0.5, s)));
  out[idx] = v < 0.0 ? 0.0 : (v > umax ? umax : v);
}

cudaError_t launch_sample_sines(int J, int nterm, const double* prm, double umax, double h, int k0, int count,
                               double* out, cudaStream_t st) {
  const long long total = (long long)count * 2 * J;
  const int grid = (int)((total + NT - 1) / NT);
  k_sample_sines<<<grid, NT, 0, st>>>(J, nterm, prm, umax, h, k0, count, out);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K0
__global__ void __launch_bounds__(NT) k_probe_dmma(double* sink, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 1.0 + 1e-6 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5) *sink = s;
}
__global__ void __launch_bounds__(NT) k_probe_dfma(double* sink, int iters) {
  double a[8];
  const double b = 1.0000001, c = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5) *sink = s;
}

cudaError_t launch_fp64_probe(int kind, int blocks, int iters, double* sink, cudaStream_t st) {
  if (kind == 0) k_probe_dmma<<<blocks, NT, 0, st>>>(sink, iters);
  else k_probe_dfma<<<blocks, NT, 0, st>>>(sink, iters);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace qal
