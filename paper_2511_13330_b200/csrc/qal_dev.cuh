// qal_dev.cuh -- device building blocks of libqal.so (sm_100a only).
//
// One CTA of 8 warps owns one 64x64 complex128 matrix product at a time:
//   * warp w owns the 8-row STRIP r = 8w..8w+7 of every operand and result;
//     lane (g = lane/4, t = lane%4) holds the 16 complex entries
//         strip[i] = M[8w + g][4i + t],   i = 0..15.
//   * C = A B is evaluated with FP64 tensor-core MMAs (mma.sync m8n8k4 f64 ->
//     SASS DMMA.8x8x4), 4 real MMAs per complex 8x8x4 step (planar re/im).
//     A comes from registers (the strip layout IS the m8n8k4 A-fragment layout
//     for k-step i), B from a shared-memory IMAGE of the whole matrix.
//   * The image stores the columns of every 8-column tile permuted,
//         phys(c) = (c & ~7) | ((c & 3) << 1) | ((c >> 2) & 1),
//     so that the accumulator of a product comes out in the strip layout: a
//     result feeds the next product as its A operand with no shuffles.  Rows
//     alternate an XOR-8 swizzle of the physical column, which makes the
//     B-fragment loads (LDS.64) and strip loads/stores (LDS/STS.128) free of
//     bank conflicts without padding (image = 2 x 32 KB, re plane then im plane).
//   * Strips that only their owner thread needs again (powers X^2, X^3 in the
//     Taylor evaluation) are parked in Tensor Memory with tcgen05.st / tcgen05.ld:
//     TMEM is 256 KB/SM of otherwise idle on-chip storage on this FP64 path.
#pragma once
#include <cassert>
#include <cuda_runtime.h>
#include <stdint.h>

namespace qal {

constexpr int NT = 256;           // threads per CTA (8 warps)
constexpr int PLANE = 64 * 64;    // doubles per re / im plane
constexpr int IMG = 2 * PLANE;    // doubles per matrix image (64 KB)

struct Lane {
  int w, g, t, r, lane;
};

__device__ __forceinline__ Lane lane_id() {
  Lane L;
  L.lane = threadIdx.x & 31;
  L.w = threadIdx.x >> 5;
  L.g = L.lane >> 2;
  L.t = L.lane & 3;
  L.r = 8 * L.w + L.g;
  return L;
}

struct Strip {
  double re[16], im[16];
};

// Compiler-only fence: keeps the operand loads of the NEXT product from being hoisted
// into the current DMMA loop (they would need another 64 live registers).
#define QAL_FENCE() asm volatile("" ::: "memory")

// Race stress (experiment build -DQAL_RACE_JITTER, tools/stress_check.py): a pseudo-random per-warp delay
// of 0-2 us in front of every shared-memory image access, product and TMEM access changes the interleaving
// of the warps that share images.  Every reduction in the library has a fixed order, so a build with the
// jitter must reproduce the default build bit for bit; a missing barrier would show as a difference.
// (compute-sanitizer is not available on this pool.)  Bounds mode (-DQAL_CHECKED): device asserts on the
// shared-memory regions and item indices of the block kernels.
#ifdef QAL_RACE_JITTER
__device__ __forceinline__ void qal_jitter() {
  const unsigned long long t = clock64();
  unsigned h = static_cast<unsigned>(t ^ (t >> 13)) * 2654435761u;
  h ^= (threadIdx.x >> 5) * 40503u + blockIdx.x * 9973u;
  h *= 2246822519u;
  if ((h >> 29) == 0) __nanosleep((h >> 8) & 2047);
}
#define QAL_JITTER() qal_jitter()
#else
#define QAL_JITTER() ((void)0)
#endif
#ifdef QAL_CHECKED
#define QAL_DCHECK(c) assert(c)
#else
#define QAL_DCHECK(c) ((void)0)
#endif

// ---------------------------------------------------------------- layout
__device__ __forceinline__ int phys_col(int r, int c) {
  return ((c & ~7) | ((c & 3) << 1) | ((c >> 2) & 1)) ^ ((r & 1) << 3);
}
__device__ __forceinline__ int img_off(int r, int c) { return r * 64 + phys_col(r, c); }

// offset of the (even) strip pair (2j, 2j+1) of lane L in an image plane
__device__ __forceinline__ int pair_off(const Lane& L, int j) {
  return L.r * 64 + ((8 * j + 2 * L.t) ^ ((L.g & 1) << 3));
}

__device__ __forceinline__ void zero(Strip& s) {
#pragma unroll
  for (int i = 0; i < 16; ++i) { s.re[i] = 0.0; s.im[i] = 0.0; }
}

__device__ __forceinline__ void copy(Strip& d, const Strip& s) {
#pragma unroll
  for (int i = 0; i < 16; ++i) { d.re[i] = s.re[i]; d.im[i] = s.im[i]; }
}

// strip <-> image (shared or global; generic pointers, 16-byte accesses)
__device__ __forceinline__ void load_img(Strip& s, const double* __restrict__ img, const Lane& L) {
  QAL_JITTER();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int o = pair_off(L, j);
    double2 a = *reinterpret_cast<const double2*>(img + o);
    double2 b = *reinterpret_cast<const double2*>(img + PLANE + o);
    s.re[2 * j] = a.x; s.re[2 * j + 1] = a.y;
    s.im[2 * j] = b.x; s.im[2 * j + 1] = b.y;
  }
}
__device__ __forceinline__ void store_img(double* __restrict__ img, const Strip& s, const Lane& L) {
  QAL_JITTER();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int o = pair_off(L, j);
    *reinterpret_cast<double2*>(img + o) = make_double2(s.re[2 * j], s.re[2 * j + 1]);
    *reinterpret_cast<double2*>(img + PLANE + o) = make_double2(s.im[2 * j], s.im[2 * j + 1]);
  }
}

// img <- x + a * y (strip-wise, no temporary strip)
__device__ __forceinline__ void store_img_axpy(double* __restrict__ img, const Strip& x, double a, const Strip& y,
                                               const Lane& L) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int o = pair_off(L, j);
    *reinterpret_cast<double2*>(img + o) =
        make_double2(fma(a, y.re[2 * j], x.re[2 * j]), fma(a, y.re[2 * j + 1], x.re[2 * j + 1]));
    *reinterpret_cast<double2*>(img + PLANE + o) =
        make_double2(fma(a, y.im[2 * j], x.im[2 * j]), fma(a, y.im[2 * j + 1], x.im[2 * j + 1]));
  }
}

// ---------------------------------------------------------------- L2 residency hints
// Per-CTA scratch strips are re-read within microseconds: keep them in L2 (evict_last);
// the per-slice operand images are streamed once (evict_first).
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void load_img_l2(Strip& s, const double* __restrict__ img, const Lane& L, uint64_t pol) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int o = pair_off(L, j);
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(s.re[2 * j]), "=d"(s.re[2 * j + 1])
                 : "l"(img + o), "l"(pol));
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(s.im[2 * j]), "=d"(s.im[2 * j + 1])
                 : "l"(img + PLANE + o), "l"(pol));
  }
}
__device__ __forceinline__ void store_img_l2(double* __restrict__ img, const Strip& s, const Lane& L, uint64_t pol) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int o = pair_off(L, j);
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(img + o), "d"(s.re[2 * j]),
                 "d"(s.re[2 * j + 1]), "l"(pol)
                 : "memory");
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(img + PLANE + o), "d"(s.im[2 * j]),
                 "d"(s.im[2 * j + 1]), "l"(pol)
                 : "memory");
  }
}

// strip <-> natural row-major complex128 matrix in global memory
__device__ __forceinline__ void load_nat(Strip& s, const double2* __restrict__ M, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double2 v = __ldg(M + L.r * 64 + 4 * i + L.t);
    s.re[i] = v.x; s.im[i] = v.y;
  }
}
__device__ __forceinline__ void store_nat(double2* __restrict__ M, const Strip& s, const Lane& L) {
#pragma unroll
  for (int i = 0; i < 16; ++i) M[L.r * 64 + 4 * i + L.t] = make_double2(s.re[i], s.im[i]);
}

// whole natural matrix -> shared image (cooperative, all 256 threads)
__device__ __forceinline__ void block_nat_to_img(double* __restrict__ img, const double2* __restrict__ M) {
#pragma unroll 4
  for (int e = threadIdx.x; e < PLANE; e += NT) {
    const int r = e >> 6, c = e & 63;
    double2 v = __ldg(M + e);
    const int o = img_off(r, c);
    img[o] = v.x;
    img[PLANE + o] = v.y;
  }
}
// whole image (global) -> shared image (cooperative 16-byte copy)
__device__ __forceinline__ void block_img_copy(double* __restrict__ dst, const double* __restrict__ src) {
  const double2* s = reinterpret_cast<const double2*>(src);
  double2* d = reinterpret_cast<double2*>(dst);
#pragma unroll 4
  for (int e = threadIdx.x; e < IMG / 2; e += NT) d[e] = s[e];
}

__device__ __forceinline__ bool is_diag(const Lane& L, int i) { return L.r == 4 * i + L.t; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- FP64 tensor core
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// acc += A * B, A = strip (registers, A-fragment layout), B = shared image.
// B fragments are fetched one k-step ahead with volatile shared loads (explicit 2-stage
// software pipeline, 32 registers): ptxas keeps them in program order instead of hoisting
// the whole 256-load stream and spilling (the kernels run at 255 registers).
__device__ __forceinline__ double lds_v(uint32_t a) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void mma_acc_4m(Strip& acc, const Strip& a, const double* __restrict__ Bs,
                                           const Lane& L) {
  QAL_JITTER();
  const int todd = L.t & 1;
  // row 4q+t of B; physical tile of output tile j is j ^ (t & 1)
  const uint32_t bE = smem_u32(Bs + L.t * 64 + L.g + 8 * todd);  // even j: tile j + todd
  const uint32_t bO = smem_u32(Bs + L.t * 64 + L.g - 8 * todd);  // odd  j: tile j - todd
  double br[2][8], bi[2][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t p = ((j & 1) ? bO : bE) + 8u * (8 * j);
    br[0][j] = lds_v(p);
    bi[0][j] = lds_v(p + 8u * PLANE);
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int cur = q & 1;
    if (q + 1 < 16) {
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
      dmma(acc.re[2 * j], acc.re[2 * j + 1], ar, br[cur][j]);
      dmma(acc.re[2 * j], acc.re[2 * j + 1], nai, bi[cur][j]);
      dmma(acc.im[2 * j], acc.im[2 * j + 1], ar, bi[cur][j]);
      dmma(acc.im[2 * j], acc.im[2 * j + 1], ai, br[cur][j]);
    }
  }
  QAL_FENCE();
}

// Same product with 3 real MMAs per complex 8x8x4 step (Gauss / "3M"):
//   P = Ar Br,  Q = Ai Bi,  R = (Ar + Ai)(Br + Bi);   Re = P - Q,  Im = R - P - Q.
// The existing accumulator is folded in by initialising P = acc.re, R = acc.re + acc.im
// (so P and R live in the acc registers; only Q is extra).  The output columns are done in
// two halves of 4 tiles, which keeps Q and the B prefetch at 8 + 16 doubles.  The operand
// sums Ar + Ai (once per k-step) and Br + Bi (per tile) are DADDs: 160 per product per
// thread against 384 DMMAs (each 16 pipe cycles per warp), i.e. 25% fewer tensor-pipe
// cycles than mma_acc_4m.  Normwise the rounding error stays O(u |A| |B|).

// an add the compiler may not CSE across the two column halves (it would keep 16 sums
// live through the first half and spill them)
__device__ __forceinline__ double dadd_opaque(double x, double y) {
  double z;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(z) : "d"(x), "d"(y));
  return z;
}
__device__ __forceinline__ void mma_acc_3m(Strip& acc, const Strip& a, const double* __restrict__ Bs,
                                           const Lane& L) {
  const int todd = L.t & 1;
  const uint32_t bE = smem_u32(Bs + L.t * 64 + L.g + 8 * todd);
  const uint32_t bO = smem_u32(Bs + L.t * 64 + L.g - 8 * todd);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double Q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      Q[i] = 0.0;
      acc.im[8 * h + i] += acc.re[8 * h + i];  // R = acc.re + acc.im
    }
    double br[2][4], bi[2][4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * h + jj;
      const uint32_t p = ((j & 1) ? bO : bE) + 8u * (8 * j);
      br[0][jj] = lds_v(p);
      bi[0][jj] = lds_v(p + 8u * PLANE);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int cur = q & 1;
      if (q + 1 < 16) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = 4 * h + jj;
          const uint32_t p = ((j & 1) ? bO : bE) + 8u * ((q + 1) * 256 + 8 * j);
          br[cur ^ 1][jj] = lds_v(p);
          bi[cur ^ 1][jj] = lds_v(p + 8u * PLANE);
        }
      }
      const double ar = a.re[q], ai = a.im[q], as = dadd_opaque(ar, ai);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = 4 * h + jj;
        const double bs = br[cur][jj] + bi[cur][jj];
        dmma(acc.re[2 * j], acc.re[2 * j + 1], ar, br[cur][jj]);   // P
        dmma(Q[2 * jj], Q[2 * jj + 1], ai, bi[cur][jj]);           // Q
        dmma(acc.im[2 * j], acc.im[2 * j + 1], as, bs);            // R
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double p = acc.re[8 * h + i], s = p + Q[i];
      acc.re[8 * h + i] = p - Q[i];
      acc.im[8 * h + i] -= s;
    }
  }
  QAL_FENCE();
}

// The product every kernel uses.  Default: the 4-MMA form.  -DQAL_USE_3M selects the Gauss
// form; measured on B200 (cfg2 fwd+grad): 661k -> 736k slices/s (+11%, not the 25% the DMMA
// count promises: the operand DADDs share the FP64 pipe and the extra live values spill), with
// ~10x larger rounding in the invariants (Hermiticity defect 2.4e-13 after 256 slices).  Kept
// as an option, not the default.
#ifdef QAL_USE_3M
constexpr int QAL_REAL_MMAS_PER_CMMA = 3;
#define mma_acc mma_acc_3m
#else
constexpr int QAL_REAL_MMAS_PER_CMMA = 4;
#define mma_acc mma_acc_4m
#endif

// ---------------------------------------------------------------- Tensor Memory scratch
// 512 columns x 128 lanes x 32 bit.  Warp w reaches lanes 32(w%4)..+31; warps w and
// w+4 use different column halves.  Slot s (0..3) of a warp: 64 columns (re 32, im 32).

__device__ __forceinline__ void tmem_alloc512(uint32_t* slot_smem) {
  // whole warp 0 executes
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot_smem)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t tmem_slot_addr(uint32_t base, const Lane& L, int slot) {
  return base + (static_cast<uint32_t>(32 * (L.w & 3)) << 16) + static_cast<uint32_t>(slot * 128 + (L.w >> 2) * 64);
}

#define QAL_R32(v)                                                                                   \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), \
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),  \
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), \
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define QAL_W32(v)                                                                                       \
  "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
      "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),           \
      "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),           \
      "=r"(v[30]), "=r"(v[31])

__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      QAL_R32(v)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : QAL_W32(v)
      : "r"(addr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_store_half(uint32_t addr, const double (&x)[16]) {
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[2 * i] = static_cast<uint32_t>(__double2loint(x[i]));
    v[2 * i + 1] = static_cast<uint32_t>(__double2hiint(x[i]));
  }
  tmem_st32(addr, v);
}
__device__ __forceinline__ void tmem_load_half(uint32_t addr, double (&x)[16]) {
  uint32_t v[32];
  tmem_ld32(addr, v);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = __hiloint2double(static_cast<int>(v[2 * i + 1]), static_cast<int>(v[2 * i]));
}
__device__ __forceinline__ void tmem_store(uint32_t addr, const Strip& s) {
  QAL_JITTER();
  tmem_store_half(addr, s.re);
  tmem_store_half(addr + 32, s.im);
  tmem_wait_st();
}

// acc += a * M  where M is a strip parked in TMEM (both halves in flight, one wait)
__device__ __forceinline__ void tmem_axpy(Strip& acc, double a, uint32_t addr) {
  QAL_JITTER();
  uint32_t v[32], w[32];
  tmem_ld32(addr, v);
  tmem_ld32(addr + 32, w);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    acc.re[i] = fma(a, __hiloint2double(static_cast<int>(v[2 * i + 1]), static_cast<int>(v[2 * i])), acc.re[i]);
    acc.im[i] = fma(a, __hiloint2double(static_cast<int>(w[2 * i + 1]), static_cast<int>(w[2 * i])), acc.im[i]);
  }
}

// ---------------------------------------------------------------- TMA bulk copies
// 1-D bulk tensor copies (cp.async.bulk, the TMA engine) global -> shared, completion
// tracked by an mbarrier transaction count.
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  QAL_JITTER();
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// one thread: copy a 64 KB matrix image global -> shared, arriving on `bar`
__device__ __forceinline__ void tma_load_img(double* dst, const double* src, uint64_t* bar) {
  mbar_expect_tx(bar, IMG * 8);
#pragma unroll
  for (int p = 0; p < 4; ++p) bulk_g2s(dst + p * (IMG / 4), src + p * (IMG / 4), IMG * 2, bar);
}
// same for an image that is read exactly once (streamed; L2 evict_first)
__device__ __forceinline__ void tma_load_img_stream(double* dst, const double* src, uint64_t* bar) {
  const uint64_t pol = l2_evict_first();
  mbar_expect_tx(bar, IMG * 8);
#pragma unroll
  for (int p = 0; p < 4; ++p) bulk_g2s_hint(dst + p * (IMG / 4), src + p * (IMG / 4), IMG * 2, bar, pol);
}

// ---------------------------------------------------------------- reductions
// max over columns of sum_r |M[r][c]| (the induced 1-norm) of the CTA's matrix given
// by its strips.  Fixed order; two __syncthreads.  red: >= 8*64 + 8 doubles of smem.
__device__ __forceinline__ double norm1(const Strip& s, double* red, const Lane& L) {
  double cs[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) cs[i] = hypot(s.re[i], s.im[i]);
#pragma unroll
  for (int off = 4; off < 32; off <<= 1)
#pragma unroll
    for (int i = 0; i < 16; ++i) cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], off);
  if (L.g == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) red[L.w * 64 + 4 * i + L.t] = cs[i];
  }
  __syncthreads();
  if (L.w == 0) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { a += red[w * 64 + L.lane]; b += red[w * 64 + 32 + L.lane]; }
    double m = fmax(a, b);
    if (!(a == a) || !(b == b)) m = __longlong_as_double(0x7ff8000000000000LL);  // keep NaN
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double o = __shfl_xor_sync(0xffffffffu, m, off);
      m = (o != o || o > m) ? o : m;
    }
    if (L.lane == 0) red[512] = m;
  }
  __syncthreads();
  return red[512];
}

// sum over the CTA of one double per thread, fixed order (warp tree, then warps in
// order).  red: >= 8 doubles of smem + 1; two __syncthreads.
__device__ __forceinline__ double block_sum(double v, double* red, const Lane& L) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (L.lane == 0) red[L.w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w];
    red[8] = s;
  }
  __syncthreads();
  return red[8];
}

// ---------------------------------------------------------------- expm helpers
// Taylor degree / scaling choice (A15): the truncation bound
//   sum_{k>m} theta^k / k! <= 2^-53 e^-theta
// holds for ||X||_1 <= theta_m (thresholds computed offline).
constexpr double THETA8 = 0.0693960458639;
constexpr double THETA12 = 0.3269045734215;
constexpr double THETA16 = 0.7873811561929;

__device__ __forceinline__ void choose_ms(double nrm, int& m, int& s) {
  s = 0;
  if (!(nrm <= 1e300)) { m = 16; s = 0; return; }  // non-finite: flagged by caller
  if (nrm <= THETA8) { m = 8; return; }
  if (nrm <= THETA12) { m = 12; return; }
  m = 16;
  while (nrm > THETA16 && s < 1000) { nrm *= 0.5; ++s; }
}

// Taylor coefficients 1/i!, correctly rounded (Fraction(1, i!) -> double)
__constant__ double c_inv_fact[19] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,
                                      0.008333333333333333, 0.001388888888888889, 0.0001984126984126984,
                                      2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07,
                                      2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10,
                                      1.1470745597729725e-11, 7.647163731819816e-13, 4.779477332387385e-14,
                                      2.8114572543455206e-15, 1.5619206968586225e-16};
__device__ __forceinline__ double inv_fact(int i) { return c_inv_fact[i]; }

}  // namespace qal
