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
constexpr int GRAD_SCRATCH_STRIPS = 4;
constexpr int QAL_TR_MAX = MAXJ + MAXJ + MAXJ * (MAXJ - 1) / 2;   // traces per slice (<= 44)
static_assert(9 * QAL_TR_MAX <= 8 * 64 + 16, "trace reduction buffer");

__device__ __forceinline__ void set_identity(Strip& s, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i) { s.re[i] = is_diag(L, i) ? 1.0 : 0.0; s.im[i] = 0.0; }
}

// ------------------------------------------------------------------ prefix chain
// P_0 = I, P_{k+1} = U_k P_k; writes P_img[b][k] = P_k (k < N) and Lam[b] = P_N.
__global__ void __launch_bounds__(NT, 1) k_prefix_chain(int N, const double* __restrict__ U_img,
                                                        double* __restrict__ P_img, double2* __restrict__ Lam,
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
  if (threadIdx.x == 0) tma_load_img(SU[0], U, &bar[0]);
  Strip A, acc;
  set_identity(A, L);
  store_img(SP, A, L);
  store_img(P, A, L);
  uint32_t ph[2] = {0, 0};
  for (int k = 0; k < N; ++k) {
    const int cur = k & 1;
    __syncthreads();  // SP written; buffer cur^1 (read at step k-1) is free
    if (threadIdx.x == 0 && k + 1 < N) {
      fence_proxy_async();
      tma_load_img(SU[cur ^ 1], U + (size_t)(k + 1) * IMG, &bar[cur ^ 1]);
    }
    mbar_wait(&bar[cur], ph[cur]);
    ph[cur] ^= 1;
    load_img(A, SU[cur], L);  // U_k strip (own rows)
    zero(acc);
    mma_acc(acc, A, SP, L);   // U_k P_k
    __syncthreads();          // all reads of SP done
    store_img(SP, acc, L);
    if (k + 1 < N) store_img(P + (size_t)(k + 1) * IMG, acc, L);
    else store_nat(Lam + (size_t)b * PLANE, acc, L);
  }
  if (ctr && threadIdx.x == 0) atomicAdd(ctr, (unsigned long long)N);
}

// ------------------------------------------------------------------ suffix chain
// X_N = S_V^dag, X_k = X_{k+1} U_k; writes X_img[b][k-1] = X_k for k = 1..N.
// S_V^dag[a][c] = V[j][l] conj(V[i][k]) with a = k + 8 l, c = i + 8 j (A8, column stacking).
__global__ void __launch_bounds__(NT, 1) k_suffix_chain(int N, const double* __restrict__ U_img,
                                                        const double2* __restrict__ V, double* __restrict__ X_img,
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
  if (threadIdx.x == 0 && N > 1) tma_load_img(SU[(N - 1) & 1], U + (size_t)(N - 1) * IMG, &bar[(N - 1) & 1]);
  Strip A, acc;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int a = L.r, c = 4 * i + L.t;
    const int kk = a & 7, l = a >> 3, ii = c & 7, j = c >> 3;
    const double2 vjl = __ldg(V + j * 8 + l), vik = __ldg(V + ii * 8 + kk);
    A.re[i] = vjl.x * vik.x + vjl.y * vik.y;
    A.im[i] = vjl.y * vik.x - vjl.x * vik.y;
  }
  store_img(X + (size_t)(N - 1) * IMG, A, L);
  uint32_t ph[2] = {0, 0};
  for (int k = N - 1; k >= 1; --k) {
    const int cur = k & 1;
    __syncthreads();  // buffer cur^1 (read at step k+1) is free
    if (threadIdx.x == 0 && k - 1 >= 1) {
      fence_proxy_async();
      tma_load_img(SU[cur ^ 1], U + (size_t)(k - 1) * IMG, &bar[cur ^ 1]);
    }
    mbar_wait(&bar[cur], ph[cur]);
    ph[cur] ^= 1;
    zero(acc);
    mma_acc(acc, A, SU[cur], L);  // X_{k+1} U_k
    copy(A, acc);
    store_img(X + (size_t)(k - 1) * IMG, A, L);
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
                                                       unsigned long long* ctr) {
  extern __shared__ __align__(128) double smem[];
  double* S1 = smem;            // X_{k+1}, then dX = G / 2^s, then dX^4, then dE
  double* S2 = smem + IMG;      // X = Omega / 2^s
  double* S3 = smem + 2 * IMG;  // X^4, then E (squarings)
  double* red = smem + 3 * IMG;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 8 * 64 + 16);
  __shared__ uint32_t tmem_base_sh;
  const Lane L = lane_id();
  if (L.w == 0) tmem_alloc512(&tmem_base_sh);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = tmem_slot_addr(tmem_base_sh, L, 0);   // slots: X^2, X^3, dX^2, dX^3
  double* scr = scratch + (size_t)blockIdx.x * GRAD_SCRATCH_STRIPS * IMG;
  double* sX = scr;             // strips parked in global (L2): X, dX, H, dH
  double* sdX = scr + IMG;
  double* sH = scr + 2 * IMG;
  double* sdH = scr + 3 * IMG;
  const int N = G.count;
  const int items = batch * N;
  const int K = n_traces(B);
  uint32_t phase = 0;
  unsigned long long nprod = 0;
  Strip A, acc;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = item / N, k = item % N;
    __syncthreads();  // previous item done with S1
    if (threadIdx.x == 0) {
      fence_proxy_async();
      tma_load_img(S1, X_img + ((size_t)b * N + k) * IMG, bar);
    }
    // X = Omega_k / 2^s
    build_omega(A, B, G, b, k, L);
    const double nrm = norm1(A, red, L);
    int m, s;
    choose_ms(nrm, m, s);
    if (!(nrm <= 1e300) && threadIdx.x == 0 && status) status[b] = -4;
    const double sc = ldexp(1.0, -s);
#pragma unroll
    for (int i = 0; i < 16; ++i) { A.re[i] *= sc; A.im[i] *= sc; }
    store_img(S2, A, L);
    store_img(sX, A, L);
    // G = P_k X_{k+1}
    load_img(A, P_img + ((size_t)b * N + k) * IMG, L);
    mbar_wait(bar, phase);
    phase ^= 1;
    zero(acc);
    mma_acc(acc, A, S1, L);
#pragma unroll
    for (int i = 0; i < 16; ++i) { acc.re[i] *= sc; acc.im[i] *= sc; }
    __syncthreads();  // all reads of S1 (X_{k+1}) done; S2 complete
    store_img(S1, acc, L);
    store_img(sdX, acc, L);
    __syncthreads();  // dX complete
    // powers and their derivatives
    load_img(A, sX, L);
    zero(acc); mma_acc(acc, A, S2, L);            // X^2
    tmem_store(tm, acc);
    zero(acc); mma_acc(acc, A, S1, L);            // X dX
    load_img(A, sdX, L);
    mma_acc(acc, A, S2, L);                       // + dX X = dX^2
    tmem_store(tm + 256, acc);
    tmem_load(A, tm);
    zero(acc); mma_acc(acc, A, S2, L);            // X^3
    tmem_store(tm + 128, acc);
    zero(acc); mma_acc(acc, A, S1, L);            // X^2 dX
    tmem_load(A, tm + 256);
    mma_acc(acc, A, S2, L);                       // + dX^2 X = dX^3
    tmem_store(tm + 384, acc);
    tmem_load(A, tm + 128);
    zero(acc); mma_acc(acc, A, S2, L);            // X^4
    store_img(S3, acc, L);
    zero(acc); mma_acc(acc, A, S1, L);            // X^3 dX
    tmem_load(A, tm + 384);
    mma_acc(acc, A, S2, L);                       // + dX^3 X = dX^4
    __syncthreads();                              // all reads of S1, S2 done; S3 = X^4
    store_img(S1, acc, L);                        // S1 = dX^4
    // Horner with derivative: H = B_{tb-1} + c_m X^4, dH = dB_{tb-1} + c_m dX^4
    const int tb = m / 4;
    nprod += 1 + 3 + 6 + 3 * (tb - 1) + 3 * s;   // G, powers, their derivatives, Horner, squarings
    const double cm = inv_fact(m);
    ps_block(A, tb - 1, sX, tm, L);
    load_img(acc, S3, L);
#pragma unroll
    for (int i = 0; i < 16; ++i) { A.re[i] = fma(cm, acc.re[i], A.re[i]); A.im[i] = fma(cm, acc.im[i], A.im[i]); }
    store_img(sH, A, L);
    dps_block(A, tb - 1, sdX, tm + 256, L);
    {
      Strip d4;
      load_img(d4, S1, L);  // own rows of dX^4 (written by this thread)
#pragma unroll
      for (int i = 0; i < 16; ++i) { A.re[i] = fma(cm, d4.re[i], A.re[i]); A.im[i] = fma(cm, d4.im[i], A.im[i]); }
    }
    store_img(sdH, A, L);
    __syncthreads();                              // S1 = dX^4 complete
    for (int blk = tb - 2; blk >= 0; --blk) {
      dps_block(acc, blk, sdX, tm + 256, L);      // dH <- dB + dH X^4 + H dX^4
      load_img(A, sdH, L);
      mma_acc(acc, A, S3, L);
      load_img(A, sH, L);
      mma_acc(acc, A, S1, L);
      store_img(sdH, acc, L);
      ps_block(acc, blk, sX, tm, L);              // H <- B + H X^4
      mma_acc(acc, A, S3, L);
      store_img(sH, acc, L);
    }
    // squarings: E <- E^2, dE <- dE E + E dE
    for (int q = 0; q < s; ++q) {
      __syncthreads();
      load_img(A, sH, L);
      store_img(S3, A, L);
      load_img(acc, sdH, L);
      store_img(S1, acc, L);
      __syncthreads();
      zero(acc); mma_acc(acc, A, S1, L);          // E dE
      load_img(A, sdH, L);
      mma_acc(acc, A, S3, L);                     // + dE E
      store_img(sdH, acc, L);
      load_img(A, sH, L);
      zero(acc); mma_acc(acc, A, S3, L);          // E^2
      store_img(sH, acc, L);
    }
    // W = dE = L(Omega, G).  traces T_m = Re Tr(W B_m) = sum_{r,c} Re(W[r][c] B_m[c][r])
    load_img(A, sdH, L);
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
    __syncthreads();
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
      const double inv_d2 = 1.0 / 64.0;
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

cudaError_t launch_prefix_chain(int batch, int N, const double* U_img, double* P_img, double2* Lam, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_prefix_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, CHAIN_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  prof_pre(ST_PREFIX, st);
  k_prefix_chain<<<batch, NT, CHAIN_SMEM_BYTES, st>>>(N, U_img, P_img, Lam, prof_counter(ST_PREFIX));
  prof_post(ST_PREFIX, st);
  ++launch_counter();
  return cudaGetLastError();
}

cudaError_t launch_suffix_chain(int batch, int N, const double* U_img, const double2* V, double* X_img,
                                cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_suffix_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, CHAIN_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  prof_pre(ST_SUFFIX, st);
  k_suffix_chain<<<batch, NT, CHAIN_SMEM_BYTES, st>>>(N, U_img, V, X_img, prof_counter(ST_SUFFIX));
  prof_post(ST_SUFFIX, st);
  ++launch_counter();
  return cudaGetLastError();
}

cudaError_t launch_grad_slices(int batch, const Basis& B, const SliceGrid& G, const double* P_img,
                               const double* X_img, double* grad, int* status, double* scratch, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_grad_slices, cudaFuncAttributeMaxDynamicSharedMemorySize, GRAD_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = batch * G.count;
  const int grid = items < num_sms() ? items : num_sms();
  prof_pre(ST_GRAD, st);
  k_grad_slices<<<grid, NT, GRAD_SMEM_BYTES, st>>>(batch, B, G, P_img, X_img, grad, status, scratch,
                                                    prof_counter(ST_GRAD));
  prof_post(ST_GRAD, st);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace qal
