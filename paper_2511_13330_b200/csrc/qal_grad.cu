// qal_grad.cu -- K6: fidelity gradient by prefix/suffix products and one adjoint
// Frechet derivative of expm per slice (BASELINE north_star; P:185 is the memory
// wall of the paper's reverse-mode autodiff that this avoids).
//
//   F = Re Tr(S_V^dag U_{N-1} ... U_0) / d^2                        (A8)
//   dF/du_{k,j} = Re Tr(G_k dU_k) / d^2,  G_k = P_k X_{k+1},
//   P_k = U_{k-1} ... U_0,  X_{k+1} = S_V^dag U_{N-1} ... U_{k+1}.
// For a matrix function f given by a power series, Tr(G L_f(X, E)) = Tr(L_f(X, G) E),
// so with W_k = L_exp(Omega_k, G_k) (one Frechet derivative per slice, independent of
// the number of controls):  dF/du_{k,j} = Re Tr(W_k dOmega_k/du_{k,j}) / d^2.
// W_k is computed by differentiating the very Paterson-Stockmeyer / squaring
// evaluation of the forward pass (chain rule on every product), i.e. the top-right
// block of the block-triangular augmented exponential of [[Omega, G], [0, Omega]].
//
// Kernels: k_prefix_chain / k_suffix_chain (one CTA per pulse, the per-slice U_k
// images streamed into shared memory by TMA bulk copies, double-buffered) and
// k_grad_slices (persistent, one (pulse, slice) item per CTA iteration).
#include "qal_dev.cuh"
#include "qal_internal.h"
#include "qal_slice.cuh"

namespace qal {

constexpr int CHAIN_SMEM_BYTES = 3 * IMG * 8 + 64;
constexpr int GRAD_SMEM_BYTES = 3 * IMG * 8 + (8 * 64 + 16) * 8 + 64;
constexpr int GRAD_SCRATCH_STRIPS = 6;
constexpr int QAL_TR_MAX = MAXJ + MAXJ + MAXJ * (MAXJ - 1) / 2;   // traces per slice (<= 44)
static_assert(9 * QAL_TR_MAX <= 8 * 64 + 16, "trace reduction buffer");

__device__ __forceinline__ void set_identity(Strip& s, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i) { s.re[i] = is_diag(L, i) ? 1.0 : 0.0; s.im[i] = 0.0; }
}

// ------------------------------------------------------------------ prefix chain
// P_0 = P_init (default I), P_{k+1} = U_k P_k; writes P_img[b][k] = P_k (k < N) and Lam[b] = P_N.
__global__ void __launch_bounds__(NT, 1) k_prefix_chain(int N, const double* __restrict__ U_img,
                                                        double* __restrict__ P_img, double2* __restrict__ Lam,
                                                        const double2* __restrict__ P_init,
                                                        unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  double* SP = smem;
  double* SU[2] = {smem + IMG, smem + 2 * IMG};
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * IMG);
  const Lane L = lane_id();
  const int b = blockIdx.x;
  const double* U = U_img + (size_t)b * N * IMG;
  double* P = P_img + (size_t)b * N * IMG;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) tma_load_img_stream(SU[0], U, &bar[0]);
  Strip A, acc;
  if (P_init) load_nat(A, P_init + (size_t)b * PLANE, L);   // time-sharded: prefix of earlier ranks
  else set_identity(A, L);
  store_img(SP, A, L);
  store_img(P, A, L);
  uint32_t ph[2] = {0, 0};
  for (int k = 0; k < N; ++k) {
    const int cur = k & 1;
    __syncthreads();  // SP written; buffer cur^1 (read at step k-1) is free
    if (threadIdx.x == 0 && k + 1 < N) {
      fence_proxy_async();
      tma_load_img_stream(SU[cur ^ 1], U + (size_t)(k + 1) * IMG, &bar[cur ^ 1]);
    }
    mbar_wait(&bar[cur], ph[cur]);
    ph[cur] ^= 1;
    load_img(A, SU[cur], L);  // U_k strip (own rows)
    zero(acc);
    mma_acc(acc, A, SP, L);   // U_k P_k
    __syncthreads();          // all reads of SP done
    store_img(SP, acc, L);
    if (k + 1 < N) store_img_l2(P + (size_t)(k + 1) * IMG, acc, L, l2_evict_first());
    else store_nat(Lam + (size_t)b * PLANE, acc, L);
  }
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, (unsigned long long)N);
}

// ------------------------------------------------------------------ suffix chain
// X_N = C (default S_V^dag), X_k = X_{k+1} U_k; writes X_img[b][k-1] = X_k for k = 1..N.
// S_V^dag[a][c] = V[j][l] conj(V[i][k]) with a = k + 8 l, c = i + 8 j (A8, column stacking).
__global__ void __launch_bounds__(NT, 1) k_suffix_chain(int N, const double* __restrict__ U_img,
                                                        const double2* __restrict__ V,
                                                        const double2* __restrict__ Cseed, double* __restrict__ X_img,
                                                        unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  double* SU[2] = {smem, smem + IMG};
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * IMG);
  const Lane L = lane_id();
  const int b = blockIdx.x;
  const double* U = U_img + (size_t)b * N * IMG;
  double* X = X_img + (size_t)b * N * IMG;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && N > 1) tma_load_img_stream(SU[(N - 1) & 1], U + (size_t)(N - 1) * IMG, &bar[(N - 1) & 1]);
  Strip A, acc;
  if (Cseed) {
    load_nat(A, Cseed + (size_t)b * PLANE, L);       // general cotangent: dL = Re Tr(C dLambda)
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int a = L.r, c = 4 * i + L.t;
      const int kk = a & 7, l = a >> 3, ii = c & 7, j = c >> 3;
      const double2 vjl = __ldg(V + j * 8 + l), vik = __ldg(V + ii * 8 + kk);
      A.re[i] = vjl.x * vik.x + vjl.y * vik.y;
      A.im[i] = vjl.y * vik.x - vjl.x * vik.y;
    }
  }
  store_img(X + (size_t)(N - 1) * IMG, A, L);
  uint32_t ph[2] = {0, 0};
  for (int k = N - 1; k >= 1; --k) {
    const int cur = k & 1;
    __syncthreads();  // buffer cur^1 (read at step k+1) is free
    if (threadIdx.x == 0 && k - 1 >= 1) {
      fence_proxy_async();
      tma_load_img_stream(SU[cur ^ 1], U + (size_t)(k - 1) * IMG, &bar[cur ^ 1]);
    }
    mbar_wait(&bar[cur], ph[cur]);
    ph[cur] ^= 1;
    zero(acc);
    mma_acc(acc, A, SU[cur], L);  // X_{k+1} U_k
    copy(A, acc);
    store_img_l2(X + (size_t)(k - 1) * IMG, A, L, l2_evict_first());
  }
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, (unsigned long long)(N - 1));
}

// ------------------------------------------------------------------ gradient slices
// Number of generator-basis traces per slice and their combination into dF/du.
__device__ __forceinline__ int n_traces(const Basis& B) { return B.J + B.ncomm; }

__global__ void __launch_bounds__(NT, 1) k_grad_slices(int batch, Basis B, SliceGrid G,
                                                       const double* __restrict__ P_img,
                                                       const double* __restrict__ X_img, double* __restrict__ grad,
                                                       int* __restrict__ status, double* __restrict__ scratch,
                                                       double gscale, unsigned long long* ctr) {
  // Dual-number evaluation of the forward Taylor scheme (T8 / T18 + s squarings) at X = Omega/2^s
  // in the direction dX = G/2^s: every product (P, dP)(Q, dQ) = (PQ, dP Q + P dQ) with the
  // right factors Q, dQ as shared images (SV = values, SD = derivatives) and the left factors
  // as strips (TMEM slots / L2 scratch).  The result dE is W = L_exp(Omega, G).
  extern __shared__ __align__(128) double smem[];
  double* SD = smem;            // P_k (TMA), then dX, dA3 / dW, dB5 / dR, dA9, dE
  double* SV = smem + IMG;      // X, A3 / W, B5 / R, A9, E
  double* SN = smem + 2 * IMG;  // X_{k+1} of this item (TMA, prefetched during the previous item)
  double* red = smem + 3 * IMG;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 8 * 64 + 16);   // [0] = P_k -> SD, [1] = X_{k+1} -> SN
  __shared__ uint32_t tmem_base_sh;
  const Lane L = lane_id();
  if (L.w == 0) tmem_alloc512(&tmem_base_sh);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = tmem_slot_addr(tmem_base_sh, L, 0);
  const uint32_t T0 = tm, T1 = tm + 128, T2 = tm + 256, T3 = tm + 384;   // A2, dA2, A3|Y, dA3|dY
  double* scr = scratch + (size_t)blockIdx.x * GRAD_SCRATCH_STRIPS * IMG;
  double* gX = scr;
  double* gdX = scr + IMG;
  double* gA6 = scr + 2 * IMG;
  double* gdA6 = scr + 3 * IMG;
  double* gE = scr + 4 * IMG;     // squarings only (s > 0)
  double* gdE = scr + 5 * IMG;
  const int N = G.count;
  const int items = batch * N;
  const int K = n_traces(B);
  const uint64_t keep = l2_evict_last();
  uint32_t ph0 = 0, ph1 = 0;
  unsigned long long nprod = 0;
  Strip A, acc;
  if (threadIdx.x == 0 && blockIdx.x < items) tma_load_img_stream(SN, X_img + (size_t)blockIdx.x * IMG, &bar[1]);
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = item / N, k = item % N;
    __syncthreads();  // previous item done with SD, SV
    if (threadIdx.x == 0) {
      fence_proxy_async();
      tma_load_img_stream(SD, P_img + ((size_t)b * N + k) * IMG, &bar[0]);
    }
    // X = Omega_k / 2^s
    build_omega(A, B, G, b, k, L);
    const double nrm = norm1(A, red, L);
    int m, s;
    choose_scheme(nrm, m, s);
    if (!(nrm <= 1e300) && threadIdx.x == 0 && status) status[b] = -4;
    const double sc = ldexp(1.0, -s);
#pragma unroll
    for (int i = 0; i < 16; ++i) { A.re[i] *= sc; A.im[i] *= sc; }
    store_img(SV, A, L);
    store_img_l2(gX, A, L, keep);
    // G = P_k X_{k+1};  dX = G / 2^s
    mbar_wait(&bar[0], ph0);
    ph0 ^= 1;
    load_img(A, SD, L);
    mbar_wait(&bar[1], ph1);
    ph1 ^= 1;
    zero(acc);
    mma_acc(acc, A, SN, L);
#pragma unroll
    for (int i = 0; i < 16; ++i) { acc.re[i] *= sc; acc.im[i] *= sc; }
    __syncthreads();  // reads of SD (P_k), SN (X_{k+1}) done; SV (X) complete
    store_img(SD, acc, L);
    store_img_l2(gdX, acc, L, keep);
    __syncthreads();  // SD = dX complete
    // (A2, dA2)
    load_img(A, SV, L);
    zero(acc); mma_acc(acc, A, SV, L);                 // A2 = X X
    tmem_store(T0, acc);
    zero(acc); mma_acc(acc, A, SD, L);                 // X dX
    load_img(A, SD, L);
    mma_acc(acc, A, SV, L);                            // + dX X
    tmem_store(T1, acc);
    int np = 1 + 1 + 2;
    if (m == 8) {
      // (W, dW) = c1 (X, dX) + c2 (A2, dA2) shared;  (Y, dY) = (A2, dA2)(W, dW)
      __syncthreads();                                 // reads of SV (X), SD (dX) done
      zero(acc); add_img_l2(acc, c_t8[0], gX, L, keep); add_tm(acc, c_t8[1], T0); store_img(SV, acc, L);
      zero(acc); add_img_l2(acc, c_t8[0], gdX, L, keep); add_tm(acc, c_t8[1], T1); store_img(SD, acc, L);
      __syncthreads();
      tmem_load(A, T0);
      zero(acc); mma_acc(acc, A, SV, L);               // Y = A2 W
      tmem_store(T2, acc);
      zero(acc); mma_acc(acc, A, SD, L);               // A2 dW
      tmem_load(A, T1);
      mma_acc(acc, A, SV, L);                          // + dA2 W = dY
      tmem_store(T3, acc);
      __syncthreads();                                 // reads of SV (W), SD (dW) done
      // (R, dR) = (Y, dY) + c5 (A2, dA2) shared
      zero(acc); add_tm(acc, 1.0, T2); add_tm(acc, c_t8[4], T0); store_img(SV, acc, L);
      zero(acc); add_tm(acc, 1.0, T3); add_tm(acc, c_t8[4], T1); store_img(SD, acc, L);
      __syncthreads();
      // dT = c6 dY + c7 dA2 + dX + dL R + L dR,   L = Y + c3 A2 + c4 X
      zero(acc);
      add_tm(acc, c_t8[5], T3); add_tm(acc, c_t8[6], T1); add_img_l2(acc, 1.0, gdX, L, keep);
      zero(A); add_tm(A, 1.0, T3); add_tm(A, c_t8[2], T1); add_img_l2(A, c_t8[3], gdX, L, keep);   // dL
      mma_acc(acc, A, SV, L);
      zero(A); add_tm(A, 1.0, T2); add_tm(A, c_t8[2], T0); add_img_l2(A, c_t8[3], gX, L, keep);    // L
      mma_acc(acc, A, SD, L);
      if (s > 0) store_img_l2(gdE, acc, L, keep);
      np += 1 + 2 + 2;
      if (s > 0) {                                     // T = c6 Y + c7 A2 + X + I + L R
        zero(acc);
        add_tm(acc, c_t8[5], T2); add_tm(acc, c_t8[6], T0); add_img_l2(acc, 1.0, gX, L, keep); add_diag(acc, 1.0, L);
        mma_acc(acc, A, SV, L);
        store_img_l2(gE, acc, L, keep);
        ++np;
      }
    } else {
      // (A3, dA3) = (A2, dA2)(X, dX)
      tmem_load(A, T0);
      zero(acc); mma_acc(acc, A, SV, L);               // A3
      tmem_store(T2, acc);
      zero(acc); mma_acc(acc, A, SD, L);               // A2 dX
      tmem_load(A, T1);
      mma_acc(acc, A, SV, L);                          // + dA2 X = dA3
      tmem_store(T3, acc);
      __syncthreads();                                 // reads of SV (X), SD (dX) done
      tmem_load(A, T2); store_img(SV, A, L);
      tmem_load(A, T3); store_img(SD, A, L);
      __syncthreads();
      // (A6, dA6) = (A3, dA3)(A3, dA3)
      tmem_load(A, T2);
      zero(acc); mma_acc(acc, A, SV, L);               // A6
      store_img_l2(gA6, acc, L, keep);
      zero(acc); mma_acc(acc, A, SD, L);               // A3 dA3
      tmem_load(A, T3);
      mma_acc(acc, A, SV, L);                          // + dA3 A3
      store_img_l2(gdA6, acc, L, keep);
      __syncthreads();                                 // reads of SV (A3), SD (dA3) done
      // (B5, dB5) shared
      zero(acc);
      add_img_l2(acc, c_t18[T18_B5][1], gX, L, keep); add_tm(acc, c_t18[T18_B5][2], T0); add_img_l2(acc, 1.0, gA6, L, keep);
      store_img(SV, acc, L);
      zero(acc);
      add_img_l2(acc, c_t18[T18_B5][1], gdX, L, keep); add_tm(acc, c_t18[T18_B5][2], T1); add_img_l2(acc, 1.0, gdA6, L, keep);
      store_img(SD, acc, L);
      __syncthreads();
      // dA9 = dB4 + dB1 B5 + B1 dB5
      zero(acc);
      add_img_l2(acc, c_t18[T18_B4][1], gdX, L, keep); add_tm(acc, c_t18[T18_B4][2], T1);
      add_tm(acc, c_t18[T18_B4][3], T3); add_img_l2(acc, c_t18[T18_B4][4], gdA6, L, keep);
      zero(A);
      add_img_l2(A, c_t18[T18_B1][1], gdX, L, keep); add_tm(A, c_t18[T18_B1][2], T1); add_tm(A, c_t18[T18_B1][3], T3);
      mma_acc(acc, A, SV, L);
      zero(A);
      add_img_l2(A, c_t18[T18_B1][1], gX, L, keep); add_tm(A, c_t18[T18_B1][2], T0); add_tm(A, c_t18[T18_B1][3], T2);
      mma_acc(acc, A, SD, L);
      store_img(SN, acc, L);                           // dA9 (SN idle since G)
      // A9 = B4 + B1 B5   (A still holds B1)
      zero(acc);
      add_diag(acc, c_t18[T18_B4][0], L);
      add_img_l2(acc, c_t18[T18_B4][1], gX, L, keep); add_tm(acc, c_t18[T18_B4][2], T0);
      add_tm(acc, c_t18[T18_B4][3], T2); add_img_l2(acc, c_t18[T18_B4][4], gA6, L, keep);
      mma_acc(acc, A, SV, L);
      __syncthreads();                                 // reads of SV (B5), SD (dB5) done
      store_img(SV, acc, L);                           // A9
      __syncthreads();                                 // A9 (SV), dA9 (SN) complete
      // dT = dB2 + dL A9 + L dA9,  L = B3 + A9
      zero(acc);
      add_img_l2(acc, c_t18[T18_B2][1], gdX, L, keep); add_tm(acc, c_t18[T18_B2][2], T1);
      add_tm(acc, c_t18[T18_B2][3], T3); add_img_l2(acc, c_t18[T18_B2][4], gdA6, L, keep);
      load_img(A, SN, L);                              // dL = dB3 + dA9
      add_img_l2(A, c_t18[T18_B3][1], gdX, L, keep); add_tm(A, c_t18[T18_B3][2], T1);
      add_tm(A, c_t18[T18_B3][3], T3); add_img_l2(A, c_t18[T18_B3][4], gdA6, L, keep);
      mma_acc(acc, A, SV, L);
      load_img(A, SV, L);                              // L = B3 + A9
      add_diag(A, c_t18[T18_B3][0], L);
      add_img_l2(A, c_t18[T18_B3][1], gX, L, keep); add_tm(A, c_t18[T18_B3][2], T0);
      add_tm(A, c_t18[T18_B3][3], T2); add_img_l2(A, c_t18[T18_B3][4], gA6, L, keep);
      mma_acc(acc, A, SN, L);
      if (s > 0) store_img_l2(gdE, acc, L, keep);
      np += 1 + 2 + 1 + 2 + 2 + 1 + 2;
      if (s > 0) {                                     // T = B2 + L A9
        zero(acc);
        add_diag(acc, c_t18[T18_B2][0], L);
        add_img_l2(acc, c_t18[T18_B2][1], gX, L, keep); add_tm(acc, c_t18[T18_B2][2], T0);
        add_tm(acc, c_t18[T18_B2][3], T2); add_img_l2(acc, c_t18[T18_B2][4], gA6, L, keep);
        mma_acc(acc, A, SV, L);
        store_img_l2(gE, acc, L, keep);
        ++np;
      }
    }
    // squarings: (E, dE) <- (E E, dE E + E dE)
    for (int q = 0; q < s; ++q) {
      __syncthreads();
      load_img_l2(A, gE, L, keep);
      store_img(SV, A, L);
      load_img_l2(acc, gdE, L, keep);
      store_img(SD, acc, L);
      __syncthreads();
      zero(acc); mma_acc(acc, A, SD, L);               // E dE
      load_img_l2(A, gdE, L, keep);
      mma_acc(acc, A, SV, L);                          // + dE E
      store_img_l2(gdE, acc, L, keep);
      load_img_l2(A, gE, L, keep);
      zero(acc); mma_acc(acc, A, SV, L);               // E E
      store_img_l2(gE, acc, L, keep);
      np += 3;
    }
    nprod += np;
    // W = dE = L(Omega, G).  traces T_m = Re Tr(W B_m) = sum_{r,c} Re(W[r][c] B_m[c][r])
    if (s > 0) load_img_l2(A, gdE, L, keep);
    else copy(A, acc);
    for (int mm = 0; mm < K; ++mm) {
      const double2* Bm = (mm < B.J) ? B.Lc + (size_t)mm * PLANE
                                     : B.Lcomm + (size_t)b * B.Lcomm_stride + (size_t)(mm - B.J) * PLANE;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double2 x = __ldg(Bm + (4 * i + L.t) * 64 + L.r);
        v = fma(A.re[i], x.x, v);
        v = fma(-A.im[i], x.y, v);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (L.lane == 0) red[L.w * QAL_TR_MAX + mm] = v;
    }
    __syncthreads();  // also: every product of this item is done -> SN is free
    if (threadIdx.x == 0 && item + (int)gridDim.x < items) {
      fence_proxy_async();
      tma_load_img_stream(SN, X_img + (size_t)(item + gridDim.x) * IMG, &bar[1]);   // next item's X_{k+1}
    }
    if (threadIdx.x < K) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w * QAL_TR_MAX + threadIdx.x];
      red[8 * QAL_TR_MAX + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double* T = red + 8 * QAL_TR_MAX;
      const int J = B.J;
      const double inv_d2 = gscale;   // 1/d^2 for the fidelity, 1 for a general cotangent
      if (G.mode == 0) {
        double* g = grad + ((size_t)b * N + k) * J;
        for (int j = 0; j < J; ++j) g[j] = G.h * T[j] * inv_d2;
      } else {
        const int nodes = 2;
        const double* u = G.u + ((size_t)b * N + k) * nodes * J;
        double* g = grad + ((size_t)b * N + k) * nodes * J;
        for (int j = 0; j < J; ++j) {
          double g1 = 0.5 * G.h * T[j], g2 = 0.5 * G.h * T[j];
          if (B.ncomm > 0) {
            // dOmega/dv1_j = (h/2) L_j - c4 [L_j, A_2];  [L_j, A_2] = -C0j + sum_{c>j} v2_c C_jc - sum_{c<j} v2_c C_cj
            // dOmega/dv2_j = (h/2) L_j - c4 [A_1, L_j];  [A_1, L_j] =  C0j + sum_{a<j} v1_a C_aj - sum_{a>j} v1_a C_ja
            double c1 = -T[J + j], c2 = T[J + j];
            int p = 2 * J;
            for (int a = 0; a < J; ++a)
              for (int c = a + 1; c < J; ++c, ++p) {
                const double Tp = T[p];
                if (a == j) { c1 += u[J + c] * Tp; c2 -= u[c] * Tp; }
                if (c == j) { c1 -= u[J + a] * Tp; c2 += u[a] * Tp; }
              }
            g1 -= G.c4 * c1;
            g2 -= G.c4 * c2;
          }
          g[j] = g1 * inv_d2;
          g[J + j] = g2 * inv_d2;
        }
      }
    }
  }
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, nprod);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (L.w == 0) tmem_dealloc512(tmem_base_sh);
}

size_t grad_scratch_bytes() { return (size_t)num_sms() * GRAD_SCRATCH_STRIPS * MAT_BYTES; }

cudaError_t launch_prefix_chain(int batch, int N, const double* U_img, double* P_img, double2* Lam,
                                const double2* P_init, cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_prefix_chain, CHAIN_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  prof_pre(ST_PREFIX, st);
  k_prefix_chain<<<batch, NT, CHAIN_SMEM_BYTES, st>>>(N, U_img, P_img, Lam, P_init, prof_counter(ST_PREFIX));
  prof_post(ST_PREFIX, st);
  ++launch_counter();
  return cudaGetLastError();
}

cudaError_t launch_suffix_chain(int batch, int N, const double* U_img, const double2* V, const double2* Cseed,
                                double* X_img, cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_suffix_chain, CHAIN_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  prof_pre(ST_SUFFIX, st);
  k_suffix_chain<<<batch, NT, CHAIN_SMEM_BYTES, st>>>(N, U_img, V, Cseed, X_img, prof_counter(ST_SUFFIX));
  prof_post(ST_SUFFIX, st);
  ++launch_counter();
  return cudaGetLastError();
}

cudaError_t launch_grad_slices(int batch, const Basis& B, const SliceGrid& G, const double* P_img,
                               const double* X_img, double* grad, int* status, double* scratch, double gscale,
                               cudaStream_t st) {
  {
    const cudaError_t e = ensure_smem((const void*)k_grad_slices, GRAD_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  const int items = batch * G.count;
  const int grid = items < num_sms() ? items : num_sms();
  prof_pre(ST_GRAD, st);
  k_grad_slices<<<grid, NT, GRAD_SMEM_BYTES, st>>>(batch, B, G, P_img, X_img, grad, status, scratch, gscale,
                                                    prof_counter(ST_GRAD));
  prof_post(ST_GRAD, st);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace qal
