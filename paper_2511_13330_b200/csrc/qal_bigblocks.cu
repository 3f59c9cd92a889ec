// qal_bigblocks.cu -- the coherence-block structure on the n = 4096 path (d = 64: two exchange-only
// qubits, six spins; BASELINE configs[4]; the 3-dot Hubbard model, NEXT f3).
//
// As for d = 8 (qal_blocks.cu), every operator conserves total S_z, so the Liouvillian of
// Eq. 8 and everything built from it by Eqs. 13-15 is block diagonal by coherence order; for six
// spins the blocks q = 0..6 have 924, 792, 495, 220, 66, 12, 1 rows, and Hermiticity preservation ties q
// to -q (pin P-5), so with the mirror 2.1% of the dense product flops remain.  These blocks are far larger
// than the d = 8 ones: each is stored as its own grid of 64 x 64 TILE IMAGES (the K7 layout of
// qal_dense.cu) and every product is a block-diagonal tiled GEMM -- one persistent launch over the output
// tiles of all blocks, each tile the DMMA.8x8x4 K loop of k_dense_gemm with TMA-streamed A / B tiles.
// The expm scheme (Paterson-Stockmeyer m = 16, s squarings) is chosen per block on the device.
//
// The structure is detected on the device (union of the non-zero patterns of the basis matrices,
// k_bb_nzmask) and the components found on the host; k_bb_check re-verifies every call that no basis
// entry couples two blocks.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/qal.h"
#include "qal_dev.cuh"
#include "qal_internal.h"

namespace qal {

constexpr int BBN = 4096;   // superoperator dimension of this path
constexpr int BBW = BBN / 64;   // 64-bit words per row of the non-zero mask

// device view of a big-block plan (tables in device memory)
struct BBDev {
  int nb, ntiles, nrows;
  int nt[QAL_BB_MAX_BLOCKS];           // tiles per dimension of block b
  int tstart[QAL_BB_MAX_BLOCKS + 1];   // prefix of nt^2 (output tiles)
  int row0[QAL_BB_MAX_BLOCKS];         // first packed row (64-aligned)
  long long toff[QAL_BB_MAX_BLOCKS];   // double offset of block b's tiles in a tiled-block matrix
  long long total;                     // doubles per tiled-block matrix
  const int* perm;                     // [nrows] packed row -> natural index (-1 padding)
  const int* inv;                      // [4096] natural -> packed row (-1: mirrored / not stored)
  const int* comp;                     // [4096] natural -> component
  const int* rtype;                    // [nrows] 0 complex, 1 real diagonal, 2 pair a, 3 pair b
  const int* ncode;                    // [4096] 0 complex, 1 real diagonal, 2 pair rep, 3 pair mirror
  int real[QAL_BB_MAX_BLOCKS];         // block b in the real Hermitian basis (qal_blocks.cu A29)
  int used[QAL_BB_MAX_BLOCKS];         // stored rows of block b (the rest of its 64-multiple is padding)
};

struct BBPlanRec {   // per block, written on the device
  int m, s, bad, pad;
  double nrm;
};
constexpr int BB_PLAN_STRIDE = 64;
#ifndef QAL_BB_TRIM
#define QAL_BB_TRIM 1
#endif
constexpr bool BB_TRIM = QAL_BB_TRIM != 0;   // skip the padding k-steps / column tiles / row strips   // plan records per slice of a batch (>= QAL_BB_MAX_BLOCKS)
// slices per batch (every launch covers the tiles of a whole batch): as many as ~4 GB of batch
// workspace holds, at most 64 (configs[4]: 16; the Hubbard blocks: 64)
#ifndef QAL_BB_SB_MAX
#define QAL_BB_SB_MAX 64
#endif
inline int bb_sb(const qal_bigblock_plan& p) {
  const size_t per = 6 * (size_t)p.total_doubles * 8;
  const size_t n = ((size_t)4 << 30) / std::max<size_t>(per, 1);
  return (int)std::min<size_t>(QAL_BB_SB_MAX, std::max<size_t>(1, n));
}

__device__ __forceinline__ int bb_block_of_tile(const BBDev& D, int t) {
  int b = 0;
  for (int q = 1; q < D.nb; ++q)
    if (t >= D.tstart[q]) b = q;
  return b;
}
// flat double index e of a tiled-block matrix -> block, tile (I, J), logical (r, c) within the tile, plane
struct BBPos {
  int b, I, J, r, c, plane;
};
__device__ __forceinline__ BBPos bb_decode(const BBDev& D, size_t e) {
  BBPos p;
  const int t = (int)(e / IMG);
  const int within = (int)(e % IMG);
  p.b = bb_block_of_tile(D, t);
  const int tl = t - D.tstart[p.b];
  p.I = tl / D.nt[p.b];
  p.J = tl % D.nt[p.b];
  p.plane = within >= PLANE;
  const int w = within - p.plane * PLANE;
  p.r = w >> 6;
  const int pc = (w & 63) ^ ((p.r & 1) << 3);
  const int q = pc & 7;
  p.c = (pc & ~7) | (4 * (q & 1) + (q >> 1));
  return p;
}
__device__ __forceinline__ double* bb_tile(const BBDev& D, double* M, int b, int I, int J) {
  return M + D.toff[b] + ((size_t)I * D.nt[b] + J) * IMG;
}
__device__ __forceinline__ const double* bb_tile(const BBDev& D, const double* M, int b, int I, int J) {
  return M + D.toff[b] + ((size_t)I * D.nt[b] + J) * IMG;
}

// ------------------------------------------------------------------ structure detection
// mask[r][w] bit c: some matrix has a non-zero at (r, 64 w + c)
__global__ void __launch_bounds__(64) k_bb_nzmask(int nmat, const double2* __restrict__ mats,
                                                  unsigned long long* __restrict__ mask) {
  const int r = blockIdx.x, w = threadIdx.x;
  unsigned long long bits = 0;
  for (int m = 0; m < nmat; ++m) {
    const double2* row = mats + ((size_t)m * BBN + r) * BBN + 64 * w;
    for (int c = 0; c < 64; ++c) {
      const double2 v = __ldg(row + c);
      if (v.x != 0.0 || v.y != 0.0) bits |= 1ull << c;
    }
  }
  mask[(size_t)r * BBW + w] = bits;
}

// every entry coupling two components must be exactly zero
__global__ void __launch_bounds__(256) k_bb_check(BBDev D, const double2* __restrict__ M, int* __restrict__ flag) {
  int bad = 0;
  const size_t n2 = (size_t)BBN * BBN;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (size_t)gridDim.x * blockDim.x) {
    const int R = (int)(e >> 12), C = (int)(e & 4095);
    if (D.comp[R] != D.comp[C]) {
      const double2 v = M[e];
      if (v.x != 0.0 || v.y != 0.0) bad = 1;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = QAL_ERR_STRUCTURE;
}

// T[natural][packed row] of a real block row (the Hermitian basis of qal_blocks.cu, A29)
__device__ __forceinline__ int bb_row_terms(const BBDev& D, int grow, int* R, double* tr, double* ti) {
  const int r0 = D.perm[grow];
  const double h = 0.70710678118654752440;
  if (r0 < 0) return 0;
  const int t = D.rtype[grow];
  R[0] = r0;
  if (t <= 1) { tr[0] = 1.0; ti[0] = 0.0; return 1; }
  R[1] = (r0 >> 6) + 64 * (r0 & 63);
  if (t == 2) { tr[0] = h; ti[0] = 0.0; tr[1] = h; ti[1] = 0.0; }
  else { tr[0] = 0.0; ti[0] = h; tr[1] = 0.0; ti[1] = -h; }
  return 2;
}

// ------------------------------------------------------------------ elementwise
// X = h (L0 + sum_j u_j L_j) gathered into the tiled blocks (a3, PWC)
// batched over slices: blockIdx.y = slice i of the batch (u row i, X + i * total)
__global__ void __launch_bounds__(NT) k_bb_omega(BBDev D, const double2* __restrict__ L0,
                                                 const double2* __restrict__ Lc, int J, const double* __restrict__ u,
                                                 double h, double* __restrict__ X) {
  u += (size_t)blockIdx.y * J;
  X += (size_t)blockIdx.y * D.total;
  __shared__ double cf[MAXJ + 1];
  if (threadIdx.x <= J) cf[threadIdx.x] = threadIdx.x == 0 ? h : h * u[threadIdx.x - 1];
  __syncthreads();
  const size_t n2 = (size_t)BBN * BBN;
  const size_t half = (size_t)D.ntiles * PLANE;   // complex entries
  for (size_t e = (size_t)blockIdx.x * NT + threadIdx.x; e < half; e += (size_t)gridDim.x * NT) {
    const int t = (int)(e / PLANE), w = (int)(e % PLANE);
    const int b = bb_block_of_tile(D, t);
    const int tl = t - D.tstart[b];
    const int I = tl / D.nt[b], Jt = tl % D.nt[b];
    const int r = w >> 6, c = w & 63;
    const int R = D.perm[D.row0[b] + 64 * I + r], Cc = D.perm[D.row0[b] + 64 * Jt + c];
    double re = 0.0, im = 0.0;
    if (R >= 0 && Cc >= 0 && D.real[b]) {
      // M'[r][c] = Re sum conj(T[Ri][r]) M[Ri][Cj] T[Cj][c] for M = h (L0 + sum_j u_j L_j)
      int Ra[2], Cb[2];
      double ar[2], ai[2], br[2], bi[2];
      const int na = bb_row_terms(D, D.row0[b] + 64 * I + r, Ra, ar, ai);
      const int nb = bb_row_terms(D, D.row0[b] + 64 * Jt + c, Cb, br, bi);
      for (int i1 = 0; i1 < na; ++i1)
        for (int j1 = 0; j1 < nb; ++j1) {
          const size_t idx = (size_t)Ra[i1] * BBN + Cb[j1];
          const double2 x0 = __ldg(L0 + idx);
          double mr = cf[0] * x0.x, mi = cf[0] * x0.y;
          for (int j = 0; j < J; ++j) {
            const double2 x = __ldg(Lc + (size_t)j * n2 + idx);
            mr = fma(cf[j + 1], x.x, mr);
            mi = fma(cf[j + 1], x.y, mi);
          }
          const double xr = ar[i1] * mr + ai[i1] * mi, xi = ar[i1] * mi - ai[i1] * mr;   // conj(ta) m
          re += xr * br[j1] - xi * bi[j1];                                              // ... tb
        }
    } else if (R >= 0 && Cc >= 0) {
      const size_t idx = (size_t)R * BBN + Cc;
      const double2 x0 = __ldg(L0 + idx);
      re = cf[0] * x0.x;
      im = cf[0] * x0.y;
      for (int j = 0; j < J; ++j) {
        const double2 x = __ldg(Lc + (size_t)j * n2 + idx);
        re = fma(cf[j + 1], x.x, re);
        im = fma(cf[j + 1], x.y, im);
      }
    }
    double* T = X + D.toff[b] + (size_t)tl * IMG;
    const int o = img_off(r, c);
    T[o] = re;
    T[PLANE + o] = im;
  }
}

// part[t][c] = sum over the 64 rows of tile t of |X[r][c]|
__global__ void __launch_bounds__(64) k_bb_colsum(BBDev D, const double* __restrict__ X, double* __restrict__ part) {
  X += (size_t)blockIdx.y * D.total;
  part += (size_t)blockIdx.y * D.ntiles * 64;
  const int t = blockIdx.x, c = threadIdx.x;
  const int b = bb_block_of_tile(D, t);
  const double* T = X + D.toff[b] + (size_t)(t - D.tstart[b]) * IMG;
  double s = 0.0;
  for (int r = 0; r < 64; ++r) {
    const int o = img_off(r, c);
    s += hypot(T[o], T[PLANE + o]);
  }
  part[(size_t)t * 64 + c] = s;
}

// per block: ||X_b||_1 = max_c sum_I part[(I, c / 64)][c % 64]; m = 16, s from theta_16 (A15)
__global__ void __launch_bounds__(1024) k_bb_plan(BBDev D, const double* __restrict__ part, BBPlanRec* plan,
                                                  int smax, int* status) {
  part += (size_t)blockIdx.y * D.ntiles * 64;
  plan += (size_t)blockIdx.y * BB_PLAN_STRIDE;
  __shared__ double red[32];
  const int b = blockIdx.x, nt = D.nt[b];
  double m = 0.0;
  bool nan = false;
  for (int c = threadIdx.x; c < 64 * nt; c += 1024) {
    double s = 0.0;
    for (int I = 0; I < nt; ++I) s += part[(size_t)(D.tstart[b] + I * nt + c / 64) * 64 + (c % 64)];
    if (!(s == s)) nan = true;
    m = fmax(m, s);
  }
  if (nan) m = __longlong_as_double(0x7ff8000000000000LL);
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, m, off);
    m = (o != o || o > m) ? o : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int w = 1; w < 32; ++w) v = (red[w] != red[w] || red[w] > v) ? red[w] : v;
    int mm, s;
    choose_ms(v, mm, s);
    const int bad = !(v <= 1e300) || s > smax;
    if (bad) s = 0;
    plan[b].m = 16;
    plan[b].s = s;
    plan[b].bad = bad;
    plan[b].nrm = v;
    if (bad && status) *status = QAL_ERR_NONFINITE;
  }
}

__global__ void __launch_bounds__(NT) k_bb_scale(BBDev D, double* X, const BBPlanRec* plan) {
  X += (size_t)blockIdx.y * D.total;
  plan += (size_t)blockIdx.y * BB_PLAN_STRIDE;
  for (size_t e = (size_t)blockIdx.x * NT + threadIdx.x; e < (size_t)D.total; e += (size_t)gridDim.x * NT) {
    const int b = bb_block_of_tile(D, (int)(e / IMG));
    const int s = plan[b].s;
    if (s) X[e] *= ldexp(1.0, -s);
  }
}

// out = cid I + sum_q coef[q] src[q]
struct BBCombo {
  const double* src[5];
  double coef[5];
  int nsrc;
  double cid;
  double* out;
};
__global__ void __launch_bounds__(NT) k_bb_combo(BBDev D, BBCombo g) {
  const size_t sl = (size_t)blockIdx.y * D.total;   // slice of the batch
  g.out += sl;
  for (size_t e = (size_t)blockIdx.x * NT + threadIdx.x; e < (size_t)D.total; e += (size_t)gridDim.x * NT) {
    double v = 0.0;
    for (int q = 0; q < g.nsrc; ++q) v = fma(g.coef[q], g.src[q][sl + e], v);
    if (g.cid != 0.0) {
      const BBPos p = bb_decode(D, e);
      if (!p.plane && p.I == p.J && p.r == p.c) v += g.cid;
    }
    g.out[e] = v;
  }
}

// dst = per block (s odd ? b : a)
__global__ void __launch_bounds__(NT) k_bb_copy_sel(BBDev D, double* dst, const double* a, const double* bsrc,
                                                    const BBPlanRec* plan) {
  const size_t sl = (size_t)blockIdx.y * D.total;
  dst += sl;
  a += sl;
  bsrc += sl;
  plan += (size_t)blockIdx.y * BB_PLAN_STRIDE;
  for (size_t e = (size_t)blockIdx.x * NT + threadIdx.x; e < (size_t)D.total; e += (size_t)gridDim.x * NT) {
    const int b = bb_block_of_tile(D, (int)(e / IMG));
    dst[e] = (plan[b].s & 1) ? bsrc[e] : a[e];
  }
}

// rows of natural index R in a real block and T[R][row]
__device__ __forceinline__ int bb_nat_terms(const BBDev& D, int R, int* rows, double* tr, double* ti) {
  const int code = D.ncode[R];
  const double h = 0.70710678118654752440;
  if (code == 1) { rows[0] = D.inv[R]; tr[0] = 1.0; ti[0] = 0.0; return 1; }
  const int a = (code == 2) ? D.inv[R] : D.inv[(R >> 6) + 64 * (R & 63)];
  if (a < 0) return 0;
  rows[0] = a; tr[0] = h; ti[0] = 0.0;
  rows[1] = a + 1; tr[1] = 0.0; ti[1] = (code == 2) ? h : -h;
  return 2;
}

// natural from the tiled blocks: stored component -> value, mirrored component -> conj of the stored
// mirror entry (Lambda[s(R), s(C)] = conj(Lambda[R, C]), s(i + d j) = j + d i), else 0
__global__ void __launch_bounds__(NT) k_bb_unpack(BBDev D, const double* __restrict__ X, double2* __restrict__ M) {
  const size_t n2 = (size_t)BBN * BBN;
  for (size_t e = (size_t)blockIdx.x * NT + threadIdx.x; e < n2; e += (size_t)gridDim.x * NT) {
    const int R = (int)(e >> 12), C = (int)(e & 4095);
    double2 v = make_double2(0.0, 0.0);
    if (D.comp[R] == D.comp[C] && D.ncode[R] != 0) {   // real block: M = T M' T^dag
      int rr[2], cc[2];
      double ar[2], ai[2], br[2], bi[2];
      const int na = bb_nat_terms(D, R, rr, ar, ai), nb = bb_nat_terms(D, C, cc, br, bi);
      double re = 0.0, im = 0.0;
      for (int i1 = 0; i1 < na; ++i1)
        for (int j1 = 0; j1 < nb; ++j1) {
          int b = 0;
          for (int q = 1; q < D.nb; ++q)
            if (rr[i1] >= D.row0[q]) b = q;
          const int lr = rr[i1] - D.row0[b], lc = cc[j1] - D.row0[b];
          const double m = bb_tile(D, X, b, lr >> 6, lc >> 6)[img_off(lr & 63, lc & 63)];
          const double xr = ar[i1] * m, xi = ai[i1] * m;
          re += xr * br[j1] + xi * bi[j1];
          im += xi * br[j1] - xr * bi[j1];
        }
      v = make_double2(re, im);
    } else if (D.comp[R] == D.comp[C]) {
      int r = D.inv[R], c = D.inv[C];
      bool cj = false;
      if (r < 0) {
        r = D.inv[(R >> 6) + 64 * (R & 63)];
        c = D.inv[(C >> 6) + 64 * (C & 63)];
        cj = true;
      }
      if (r >= 0 && c >= 0) {
        int b = 0;
        for (int q = 1; q < D.nb; ++q)
          if (r >= D.row0[q]) b = q;
        const int lr = r - D.row0[b], lc = c - D.row0[b];
        const double* T = bb_tile(D, X, b, lr >> 6, lc >> 6);
        const int o = img_off(lr & 63, lc & 63);
        v = make_double2(T[o], cj ? -T[PLANE + o] : T[PLANE + o]);
      }
    }
    M[e] = v;
  }
}

// ------------------------------------------------------------------ block-diagonal tiled GEMM
// C = A B block by block (C_b = A_b B_b), accumulator initialised to cid I + sum coef[q] src[q];
// slot >= 0: a squaring, active for block b only when slot < plan[b].s; A_alt is used for blocks with
// odd plan[b].s (the result of their squarings).
// acc.re += a.re * B.re (a real block: 1 DMMA per 8x8x4 step)
__device__ __forceinline__ void mma_acc_re(Strip& acc, const Strip& a, const double* __restrict__ Bs,
                                           const Lane& L) {
  const int todd = L.t & 1;
  const uint32_t bE = smem_u32(Bs + L.t * 64 + L.g + 8 * todd);
  const uint32_t bO = smem_u32(Bs + L.t * 64 + L.g - 8 * todd);
  double br[2][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) br[0][j] = lds_v(((j & 1) ? bO : bE) + 8u * (8 * j));
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int cur = q & 1;
    if (q + 1 < 16) {
#pragma unroll
      for (int j = 0; j < 8; ++j) br[cur ^ 1][j] = lds_v(((j & 1) ? bO : bE) + 8u * ((q + 1) * 256 + 8 * j));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc.re[2 * j], acc.re[2 * j + 1], a.re[q], br[cur][j]);
  }
  QAL_FENCE();
}
// The same products restricted to the first qmax k-steps and the first jmax output column tiles (the
// rest of the tile is block padding: zero rows of B / columns nobody reads).  Exact for the stored
// entries: the padding rows and columns of every block matrix are decoupled from the stored ones.
__device__ __forceinline__ void mma_acc_trim(Strip& acc, const Strip& a, const double* __restrict__ Bs, const Lane& L,
                                             int qmax, int jmax) {
  const int todd = L.t & 1;
  const uint32_t bE = smem_u32(Bs + L.t * 64 + L.g + 8 * todd);
  const uint32_t bO = smem_u32(Bs + L.t * 64 + L.g - 8 * todd);
  double br[2][8], bi[2][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t p = ((j & 1) ? bO : bE) + 8u * (8 * j);
    br[0][j] = lds_v(p);
    bi[0][j] = lds_v(p + 8u * PLANE);
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q >= qmax) break;
    const int cur = q & 1;
    if (q + 1 < qmax) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t p = ((j & 1) ? bO : bE) + 8u * ((q + 1) * 256 + 8 * j);
        br[cur ^ 1][j] = lds_v(p);
        bi[cur ^ 1][j] = lds_v(p + 8u * PLANE);
      }
    }
    const double ar = a.re[q], ai = a.im[q], nai = -a.im[q];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < jmax) {
        dmma(acc.re[2 * j], acc.re[2 * j + 1], ar, br[cur][j]);
        dmma(acc.re[2 * j], acc.re[2 * j + 1], nai, bi[cur][j]);
        dmma(acc.im[2 * j], acc.im[2 * j + 1], ar, bi[cur][j]);
        dmma(acc.im[2 * j], acc.im[2 * j + 1], ai, br[cur][j]);
      }
    }
  }
  QAL_FENCE();
}
__device__ __forceinline__ void mma_acc_re_trim(Strip& acc, const Strip& a, const double* __restrict__ Bs,
                                                const Lane& L, int qmax, int jmax) {
  const int todd = L.t & 1;
  const uint32_t bE = smem_u32(Bs + L.t * 64 + L.g + 8 * todd);
  const uint32_t bO = smem_u32(Bs + L.t * 64 + L.g - 8 * todd);
  double br[2][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) br[0][j] = lds_v(((j & 1) ? bO : bE) + 8u * (8 * j));
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q >= qmax) break;
    const int cur = q & 1;
    if (q + 1 < qmax) {
#pragma unroll
      for (int j = 0; j < 8; ++j) br[cur ^ 1][j] = lds_v(((j & 1) ? bO : bE) + 8u * ((q + 1) * 256 + 8 * j));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < jmax) dmma(acc.re[2 * j], acc.re[2 * j + 1], a.re[q], br[cur][j]);
  }
  QAL_FENCE();
}
__device__ __forceinline__ void load_img_re(Strip& s, const double* __restrict__ img, const Lane& L) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 a = *reinterpret_cast<const double2*>(img + pair_off(L, j));
    s.re[2 * j] = a.x; s.re[2 * j + 1] = a.y;
    s.im[2 * j] = 0.0; s.im[2 * j + 1] = 0.0;
  }
}

__device__ __forceinline__ void store_img_re(double* __restrict__ img, const Strip& s, const Lane& L) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<double2*>(img + pair_off(L, j)) = make_double2(s.re[2 * j], s.re[2 * j + 1]);
}

// C_i = A_i B_i for i < nbatch (A_i = A + i sA, ...; the accumulator is initialised to
// cid I + sum coef[q] src[q]_i, src_i = src + i sSrc); plan_i = plan + i pstride.
struct BBGemm {
  const double* A;
  const double* A_alt;
  const double* B;
  double* C;
  const double* src[3];
  double coef[3];
  double cid;
  int nsrc;
  int slot;
  int nbatch;
  long long sA, sB, sC, sSrc;   // doubles between batch members
  int pstride;                  // plan records between batch members
  const BBPlanRec* plan;
  unsigned long long* ctr;   // profiling: algorithmic flops of the executed block products
  unsigned long long bflops[QAL_BB_MAX_BLOCKS];
};

__device__ __forceinline__ bool bb_active(const BBDev& D, const BBGemm& g, int i, int b) {
  return g.slot < 0 || g.slot < g.plan[(size_t)i * g.pstride + b].s;
}
// virtual tile v = i * ntiles + t: batch member i, output tile t
struct BBVT {
  int i, b, I, J;
};
__device__ __forceinline__ BBVT bb_vt(const BBDev& D, int v) {
  BBVT r;
  r.i = v / D.ntiles;
  const int t = v - r.i * D.ntiles;
  r.b = bb_block_of_tile(D, t);
  const int tl = t - D.tstart[r.b];
  r.I = tl / D.nt[r.b];
  r.J = tl % D.nt[r.b];
  return r;
}
// next active virtual tile >= v (or nv)
__device__ __forceinline__ int bb_next_vt(const BBDev& D, const BBGemm& g, int v, int stride, int nv) {
  while (v < nv) {
    const int i = v / D.ntiles;
    if (bb_active(D, g, i, bb_block_of_tile(D, v - i * D.ntiles))) break;
    v += stride;
  }
  return v;
}

__global__ void __launch_bounds__(NT, 1) k_bb_gemm(BBDev D, BBGemm g) {
  extern __shared__ __align__(128) double smem[];
  double* SA = smem;
  double* SB[2] = {smem + IMG, smem + 2 * IMG};
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * IMG);
  const Lane L = lane_id();
  const int nv = g.nbatch * D.ntiles;
  if (g.ctr && blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < g.nbatch; ++i)
      for (int b = 0; b < D.nb; ++b)
        if (bb_active(D, g, i, b)) atomicAdd(g.ctr, g.bflops[b]);
  int v = bb_next_vt(D, g, blockIdx.x, gridDim.x, nv);
  if (v >= nv) return;
  // the first `rows` rows of each plane of a tile image (rows are contiguous 64-double lines of the
  // plane; a real block's tiles carry only their re plane, the im plane is zero and never read).  The
  // GEMM reads A rows of the used row strips and B rows of the used k-steps only (BB_TRIM), so the
  // padding rows of a block's last tile row / column are not moved.
  auto tma_tile = [&](double* dst, const double* src, uint64_t* br, bool real, int rows) {
    const uint32_t bytes = (uint32_t)rows * 64 * 8;   // per plane, <= 32 KB
    mbar_expect_tx(br, real ? bytes : 2 * bytes);
    const int np = real ? 1 : 2;
    for (int pl = 0; pl < np; ++pl) {
      if (bytes > 16384) {
        bulk_g2s(dst + pl * PLANE, src + pl * PLANE, 16384, br);
        bulk_g2s(dst + pl * PLANE + 2048, src + pl * PLANE + 2048, bytes - 16384, br);
      } else {
        bulk_g2s(dst + pl * PLANE, src + pl * PLANE, bytes, br);
      }
    }
  };
  // rows of A tile (I, .) = the used row strips, of B tile (K, .) = the used k-steps
  auto rowsA = [&](int b, int I) { return BB_TRIM ? std::min(64, (D.used[b] - 64 * I + 7) & ~7) : 64; };
  auto rowsB = [&](int b, int K) { return BB_TRIM ? std::min(64, (D.used[b] - 64 * K + 3) & ~3) : 64; };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto Aof = [&](const BBVT& x) {
    const double* a = (g.A_alt && (g.plan[(size_t)x.i * g.pstride + x.b].s & 1)) ? g.A_alt : g.A;
    return a + x.i * g.sA;
  };
  auto Bof = [&](const BBVT& x) { return g.B + x.i * g.sB; };
  BBVT x = bb_vt(D, v);
  if (threadIdx.x == 0) {
    tma_tile(SA, bb_tile(D, Aof(x), x.b, x.I, 0), &bar[0], D.real[x.b], rowsA(x.b, x.I));
    tma_tile(SB[0], bb_tile(D, Bof(x), x.b, 0, x.J), &bar[1], D.real[x.b], rowsB(x.b, 0));
  }
  uint32_t phA = 0, phB[2] = {0, 0};
  int step = 0;
  Strip a, acc;
  while (v < nv) {
    x = bb_vt(D, v);
    const int nt = D.nt[x.b];
    const bool re_only = D.real[x.b] != 0;
    // a warp whose 8 rows lie wholly in the block's padding neither reads the accumulator sources nor
    // writes its strip of C: no kernel ever reads those rows (the GEMM reads A rows of the used strips
    // and B rows of the used k-steps, the unpack the stored entries, the norms only the Omega images)
    const bool live = !BB_TRIM || 64 * x.I + 8 * L.w < D.used[x.b];
    zero(acc);
    for (int q = 0; live && q < g.nsrc; ++q) {
      Strip y;
      const double* st = bb_tile(D, g.src[q] + x.i * g.sSrc, x.b, x.I, x.J);
      if (re_only) load_img_re(y, st, L);   // a real block's im plane is never read
      else load_img(y, st, L);
      const double c = g.coef[q];
#pragma unroll
      for (int i = 0; i < 16; ++i) { acc.re[i] = fma(c, y.re[i], acc.re[i]); acc.im[i] = fma(c, y.im[i], acc.im[i]); }
    }
    if (x.I == x.J && g.cid != 0.0) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (is_diag(L, i)) acc.re[i] += g.cid;
    }
    const int vnext = bb_next_vt(D, g, v + gridDim.x, gridDim.x, nv);
    for (int K = 0; K < nt; ++K, ++step) {
      const int cur = step & 1;
      mbar_wait(&bar[0], phA);
      phA ^= 1;
      mbar_wait(&bar[1 + cur], phB[cur]);
      phB[cur] ^= 1;
      if (D.real[x.b]) load_img_re(a, SA, L);
      else load_img(a, SA, L);
      __syncthreads();   // SA drained by every warp; SB[cur^1] no longer read
      if (threadIdx.x == 0) {
        BBVT xn = x;
        int Kn = K + 1;
        bool more = true;
        if (Kn == nt) {
          Kn = 0;
          more = vnext < nv;
          if (more) xn = bb_vt(D, vnext);
        }
        if (more) {
          fence_proxy_async();
          tma_tile(SA, bb_tile(D, Aof(xn), xn.b, xn.I, Kn), &bar[0], D.real[xn.b], rowsA(xn.b, xn.I));
          tma_tile(SB[cur ^ 1], bb_tile(D, Bof(xn), xn.b, Kn, xn.J), &bar[1 + (cur ^ 1)], D.real[xn.b],
                   rowsB(xn.b, Kn));
        }
      }
      // padding: k-steps past the block's stored rows (last K tile), output column tiles past them
      // (last column tile), and whole strips of padding rows (last row tile) are skipped
      const int ub = D.used[x.b];
      const int qmax = BB_TRIM ? std::min(16, (ub - 64 * K + 3) >> 2) : 16;
      const int jmax = BB_TRIM ? std::min(8, (ub - 64 * x.J + 7) >> 3) : 8;
      const bool rows = !BB_TRIM || 64 * x.I + 8 * L.w < ub;
      if (rows && qmax == 16 && jmax == 8) {
        if (D.real[x.b]) mma_acc_re(acc, a, SB[cur], L);
        else mma_acc(acc, a, SB[cur], L);
      } else if (rows) {
        if (D.real[x.b]) mma_acc_re_trim(acc, a, SB[cur], L, qmax, jmax);
        else mma_acc_trim(acc, a, SB[cur], L, qmax, jmax);
      }
    }
    if (live) {
      double* ct = bb_tile(D, g.C + x.i * g.sC, x.b, x.I, x.J);
      if (re_only) store_img_re(ct, acc, L);   // the im plane of a real block's tile is never read
      else store_img(ct, acc, L);
    }
    v = vnext;
  }
}

// ------------------------------------------------------------------ host
namespace {
constexpr int BB_GEMM_SMEM = 3 * IMG * 8 + 64;
int bb_grid_ew() { return 4 * num_sms(); }
}  // namespace

size_t bb_ws_bytes(const qal_bigblock_plan& p) {
  // 6 batches of SB tiled-block matrices (X, X2, X3, X4, T0, T1) + the running products P[2] +
  // column partials and plan records per slice of a batch + device tables
  const size_t SB = bb_sb(p);
  return (6 * SB + 2) * (size_t)p.total_doubles * 8 + SB * p.ntiles * 64 * 8 + SB * BB_PLAN_STRIDE * sizeof(BBPlanRec) +
         (size_t)(2 * p.nrows + 3 * BBN) * sizeof(int) + 1024;
}

// device view; copies the index tables into `tab` (device, inside the workspace) on `st`
static cudaError_t bb_dev(const qal_bigblock_plan& p, int* tab, BBDev& D, cudaStream_t st) {
  memset(&D, 0, sizeof(D));
  D.nb = p.nb;
  D.ntiles = p.ntiles;
  D.nrows = p.nrows;
  D.total = p.total_doubles;
  int ts = 0;
  for (int b = 0; b < p.nb; ++b) {
    D.nt[b] = p.nt[b];
    D.row0[b] = p.row0[b];
    D.toff[b] = (long long)ts * IMG;
    D.tstart[b] = ts;
    ts += p.nt[b] * p.nt[b];
  }
  D.tstart[p.nb] = ts;
  std::vector<int> h(2 * p.nrows + 3 * BBN);
  for (int r = 0; r < p.nrows; ++r) { h[r] = p.perm[r]; h[p.nrows + 3 * BBN + r] = p.rtype[r]; }
  for (int i = 0; i < BBN; ++i) {
    h[p.nrows + i] = p.inv[i];
    h[p.nrows + BBN + i] = p.comp[i];
    h[p.nrows + 2 * BBN + i] = p.ncode[i];
  }
  for (int b = 0; b < p.nb; ++b) D.real[b] = p.real[b];
  for (int b = 0; b < p.nb; ++b) D.used[b] = p.size[b];
  // pageable source: the runtime stages it before returning, so `h` may die with this frame
  const cudaError_t e = cudaMemcpyAsync(tab, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, st);
  D.perm = tab;
  D.inv = tab + p.nrows;
  D.comp = tab + p.nrows + BBN;
  D.ncode = tab + p.nrows + 2 * BBN;
  D.rtype = tab + p.nrows + 3 * BBN;
  return e;
}

size_t bb_plan_ws_bytes() { return (size_t)BBN * BBW * 8; }

int build_bigblock_plan(int nmat, const double2* mats, int mirror, qal_bigblock_plan* out, void* ws, cudaStream_t st) {
  // non-zero pattern on the device (2 MB bitmask in the caller's workspace), components on the host
  unsigned long long* dmask = reinterpret_cast<unsigned long long*>(ws);
  k_bb_nzmask<<<BBN, BBW, 0, st>>>(nmat, mats, dmask);
  ++launch_counter();
  std::vector<unsigned long long> mask((size_t)BBN * BBW);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(mask.data(), dmask, mask.size() * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return QAL_ERR_CUDA;
  std::vector<int> par(BBN);
  for (int i = 0; i < BBN; ++i) par[i] = i;
  auto find = [&](int a) {
    while (par[a] != a) a = par[a] = par[par[a]];
    return a;
  };
  for (int r = 0; r < BBN; ++r)
    for (int w = 0; w < BBW; ++w) {
      unsigned long long bits = mask[(size_t)r * BBW + w];
      while (bits) {
        const int c = 64 * w + __builtin_ctzll(bits);
        bits &= bits - 1;
        const int a = find(r), b = find(c);
        if (a != b) par[std::max(a, b)] = std::min(a, b);
      }
    }
  std::vector<int> cid(BBN), root(BBN, -1);
  int ncomp = 0;
  for (int i = 0; i < BBN; ++i) {
    const int r = find(i);
    if (root[r] < 0) root[r] = ncomp++;
    cid[i] = root[r];
  }
  std::vector<std::vector<int>> members(ncomp);
  for (int i = 0; i < BBN; ++i) members[cid[i]].push_back(i);
  std::vector<int> mir(ncomp);
  for (int k = 0; k < ncomp; ++k) {
    const int i0 = members[k][0];
    mir[k] = cid[(i0 >> 6) + 64 * (i0 & 63)];
    for (int i : members[k])
      if (cid[(i >> 6) + 64 * (i & 63)] != mir[k]) return QAL_ERR_STRUCTURE;
  }
  std::vector<int> keep;
  for (int k = 0; k < ncomp; ++k)
    if (!mirror || k <= mir[k]) keep.push_back(k);
  std::stable_sort(keep.begin(), keep.end(), [&](int a, int b) { return members[a].size() > members[b].size(); });
  // best-fit-decreasing packing of the components into blocks of 64-multiple width (components that
  // share a block are multiplied densely together -- their cross terms are zero).  Measured against a
  // packing that keeps the components apart (each in its own trimmed block, by a modelled DMMA-time
  // rule): Hubbard 7.8k -> 5.5k slices/s, configs[4] 548 -> 538 -- more, shorter (tile, K) steps whose TMA
  // wait and per-tile source loads are no longer hidden behind a full tile's DMMAs cost more than the zero
  // cross terms of the packed tiles (DESIGN 5d)
  struct Bin { int width, used, real; std::vector<int> comps; };
  std::vector<Bin> bins;
  for (int k : keep) {
    const int sz = (int)members[k].size();
    const int rl = (mir[k] == k);   // self-mirrored: real in the Hermitian basis
    int best = -1;
    for (int i = 0; i < (int)bins.size(); ++i)
      if (bins[i].real == rl && bins[i].used + sz <= bins[i].width &&
          (best < 0 || bins[i].width - bins[i].used < bins[best].width - bins[best].used))
        best = i;
    if (best >= 0) { bins[best].used += sz; bins[best].comps.push_back(k); }
    else bins.push_back({(sz + 63) / 64 * 64, sz, rl, {k}});
  }
  if ((int)bins.size() > QAL_BB_MAX_BLOCKS) return QAL_ERR_UNSUPPORTED;
  qal_bigblock_plan p;
  memset(&p, 0, sizeof(p));
  p.n = BBN;
  p.d = 64;
  p.mirror = mirror ? 1 : 0;
  p.nb = (int)bins.size();
  p.n_components = ncomp;
  for (int i = 0; i < QAL_BB_MAX_ROWS; ++i) { p.perm[i] = -1; p.rtype[i] = 0; }
  for (int i = 0; i < BBN; ++i) { p.inv[i] = -1; p.comp[i] = cid[i]; p.ncode[i] = 0; }
  int row = 0, tiles = 0;
  double flops = 0.0;
  for (int b = 0; b < p.nb; ++b) {
    p.size[b] = bins[b].used;
    const int width = bins[b].width;
    p.nt[b] = width / 64;
    p.row0[b] = row;
    p.weight[b] = 1;
    if (row + width > QAL_BB_MAX_ROWS) return QAL_ERR_UNSUPPORTED;
    p.real[b] = bins[b].real;
    int r = row;
    double fl = 0.0;
    for (int k : bins[b].comps) {
      for (int i : members[k]) {
        const int si = (i >> 6) + 64 * (i & 63);
        if (!bins[b].real) {
          p.perm[r] = i; p.inv[i] = r; ++r;
        } else if (si == i) {
          p.perm[r] = i; p.rtype[r] = 1; p.inv[i] = r; p.ncode[i] = 1; ++r;
        } else if (i < si) {
          p.perm[r] = i; p.rtype[r] = 2; p.inv[i] = r; p.ncode[i] = 2;
          p.perm[r + 1] = i; p.rtype[r + 1] = 3;
          p.ncode[si] = 3;
          r += 2;
        }
      }
      const double sz = (double)members[k].size();
      fl += (bins[b].real ? 2.0 : 2.0 * QAL_REAL_MMAS_PER_CMMA) * sz * sz * sz;
    }
    p.flops[b] = fl;
    flops += fl;
    row += width;
    tiles += p.nt[b] * p.nt[b];
  }
  p.nrows = row;
  p.ntiles = tiles;
  p.total_doubles = (long long)tiles * IMG;
  p.flops_per_product = flops;
  *out = p;
  return QAL_OK;
}

static cudaError_t bb_gemm(const BBDev& D, const BBGemm& g0, const qal_bigblock_plan& p, cudaStream_t st) {
  BBGemm g = g0;
  if (g.nbatch < 1) g.nbatch = 1;
  g.ctr = prof_counter(ST_BLK_GEMM);
  for (int b = 0; b < p.nb; ++b) g.bflops[b] = (unsigned long long)p.flops[b];
  {
    const cudaError_t e = ensure_smem((const void*)k_bb_gemm, BB_GEMM_SMEM);
    if (e != cudaSuccess) return e;
  }
  prof_pre(ST_BLK_GEMM, st);
  k_bb_gemm<<<num_sms(), NT, BB_GEMM_SMEM, st>>>(D, g);
  prof_post(ST_BLK_GEMM, st);
  ++launch_counter();
  return cudaGetLastError();
}

// Propagator of `count` PWC slices of one pulse on the tiled blocks: chunk folds -> chunk_nat (natural,
// mirror-filled).  Slices go in batches of up to bb_sb(p) (never across a chunk boundary): every launch
// covers the tiles of the whole batch (the per-slice Paterson-Stockmeyer / squaring schedule of
// launch_dense_expm_fold, per slice and block), the batch's U_k are multiplied by a balanced tree
// (later slice on the left, Eq. 15) and folded into the chunk's running product.
cudaError_t launch_bb_expm_fold(const qal_bigblock_plan& p, const double2* L0, const double2* Lc, int J,
                                const double* u, int count, double h, int chunk, double2* chunk_nat, int* status,
                                int* flag, double* ws, cudaStream_t st) {
  const size_t M = (size_t)p.total_doubles;
  const int SB = bb_sb(p);
  const size_t MB = (size_t)SB * M;
  double* X = ws;
  double* X2 = X + MB;
  double* X3 = X2 + MB;
  double* X4 = X3 + MB;
  double* T0 = X4 + MB;
  double* T1 = T0 + MB;
  double* P[2] = {T1 + MB, T1 + MB + M};
  double* part = P[1] + M;
  BBPlanRec* plan = reinterpret_cast<BBPlanRec*>(part + (size_t)SB * p.ntiles * 64);
  int* tab = reinterpret_cast<int*>(plan + (size_t)SB * BB_PLAN_STRIDE);
  BBDev D;
  cudaError_t e = bb_dev(p, tab, D, st);
  if (e != cudaSuccess) return e;
  if (flag) {   // structure check of the basis of this call
    k_bb_check<<<bb_grid_ew(), 256, 0, st>>>(D, L0, flag);
    for (int j = 0; j < J; ++j) k_bb_check<<<bb_grid_ew(), 256, 0, st>>>(D, Lc + (size_t)j * BBN * BBN, flag);
    launch_counter() += 1 + J;
  }
  constexpr int SMAX = 8;
  static const double ifac[17] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,
                                  0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05,
                                  2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08,
                                  2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11,
                                  7.647163731819816e-13, 4.779477332387385e-14};
  // a batch GEMM over S slices with the per-slice plans
  auto batch = [&](BBGemm g, int S) {
    g.nbatch = S;
    g.sA = g.sB = g.sC = g.sSrc = (long long)M;
    g.pstride = BB_PLAN_STRIDE;
    g.plan = plan;
    return bb_gemm(D, g, p, st);
  };
  int pc = 0;
  for (int k = 0; k < count && e == cudaSuccess;) {
    const int S = std::min(SB, std::min(chunk - k % chunk, count - k));
    const dim3 gew((unsigned)std::max(1, bb_grid_ew() / S), (unsigned)S);
    k_bb_omega<<<gew, NT, 0, st>>>(D, L0, Lc, J, u + (size_t)k * J, h, X);
    k_bb_colsum<<<dim3(p.ntiles, S), 64, 0, st>>>(D, X, part);
    k_bb_plan<<<dim3(p.nb, S), 1024, 0, st>>>(D, part, plan, SMAX, status);
    k_bb_scale<<<gew, NT, 0, st>>>(D, X, plan);
    launch_counter() += 4;
    BBGemm g{};
    g.slot = -1;
    g.A = X; g.B = X; g.C = X2;
    if ((e = batch(g, S)) != cudaSuccess) break;
    g.A = X2; g.C = X3;
    if ((e = batch(g, S)) != cudaSuccess) break;
    g.A = X3; g.C = X4;
    if ((e = batch(g, S)) != cudaSuccess) break;
    BBCombo cb{};
    cb.src[0] = X; cb.src[1] = X2; cb.src[2] = X3; cb.src[3] = X4;
    cb.coef[0] = ifac[13]; cb.coef[1] = ifac[14]; cb.coef[2] = ifac[15]; cb.coef[3] = ifac[16];
    cb.nsrc = 4;
    cb.cid = ifac[12];
    cb.out = T0;
    k_bb_combo<<<gew, NT, 0, st>>>(D, cb);
    ++launch_counter();
    double* Hin = T0;
    double* Hout = T1;
    for (int blk = 2; blk >= 0 && e == cudaSuccess; --blk) {   // H <- B_blk + H X^4
      BBGemm h2{};
      h2.A = Hin; h2.B = X4; h2.C = Hout; h2.slot = -1;
      h2.src[0] = X; h2.src[1] = X2; h2.src[2] = X3;
      h2.coef[0] = ifac[4 * blk + 1]; h2.coef[1] = ifac[4 * blk + 2]; h2.coef[2] = ifac[4 * blk + 3];
      h2.nsrc = 3;
      h2.cid = ifac[4 * blk];
      e = batch(h2, S);
      double* tmp = Hin; Hin = Hout; Hout = tmp;
    }
    if (e != cudaSuccess) break;
    double* E[2] = {Hin, Hout};
    for (int q = 0; q < SMAX && e == cudaSuccess; ++q) {   // squarings, per slice and block only while q < s
      BBGemm sq{};
      sq.A = E[q & 1]; sq.B = E[q & 1]; sq.C = E[(q + 1) & 1]; sq.slot = q;
      e = batch(sq, S);
    }
    if (e != cudaSuccess) break;
    // U_k of the batch, contiguous in X (free since the Horner step)
    k_bb_copy_sel<<<gew, NT, 0, st>>>(D, X, E[0], E[1], plan);
    ++launch_counter();
    // balanced tree over the batch: level (2i+1, 2i) -> i, an odd last member carried
    double* in = X;
    double* outb[2] = {X2, X3};
    int cnt = S, ob = 0;
    while (cnt > 1 && e == cudaSuccess) {
      const int half = cnt / 2;
      BBGemm t{};
      t.slot = -1; t.plan = plan; t.pstride = 0;
      t.A = in + M; t.B = in; t.C = outb[ob];
      t.nbatch = half;
      t.sA = t.sB = 2 * (long long)M; t.sC = (long long)M;
      if ((e = bb_gemm(D, t, p, st)) != cudaSuccess) break;
      if (cnt & 1) {
        e = cudaMemcpyAsync(outb[ob] + (size_t)half * M, in + (size_t)(cnt - 1) * M, M * 8, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) break;
      }
      in = outb[ob];
      ob ^= 1;
      cnt = half + (cnt & 1);
    }
    if (e != cudaSuccess) break;
    if (k % chunk == 0) {   // first batch of a chunk: P = Q
      e = cudaMemcpyAsync(P[pc], in, M * 8, cudaMemcpyDeviceToDevice, st);
    } else {                 // P <- Q P
      BBGemm f{};
      f.A = in; f.B = P[pc]; f.C = P[pc ^ 1]; f.slot = -1; f.plan = plan; f.pstride = 0; f.nbatch = 1;
      e = bb_gemm(D, f, p, st);
      pc ^= 1;
    }
    if (e != cudaSuccess) break;
    k += S;
    if (k % chunk == 0) {
      k_bb_unpack<<<bb_grid_ew(), NT, 0, st>>>(D, P[pc], chunk_nat + (size_t)(k / chunk - 1) * BBN * BBN);
      ++launch_counter();
    }
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace qal
