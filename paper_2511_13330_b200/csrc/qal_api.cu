// qal_api.cu -- the C ABI of libqal.so (include/qal.h): synchronous argument
// validation, then kernel launches on the caller's stream.  No allocation.
#include <cmath>
#include <cstdint>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: no-op unless a profiler injects itself

#include "../../include/qal.h"
#include "qal_dev.cuh"
#include "qal_internal.h"

namespace qal {

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

// dynamic shared-memory opt-in (and the all-shared carveout) of a kernel, once per (device, kernel):
// the attribute is per device, so a process driving several GPUs sets it on each; callers on several
// host threads are serialised here.  Raising the size later re-applies the attribute.
cudaError_t ensure_smem(const void* fn, size_t bytes) {
  struct Rec {
    int dev;
    const void* fn;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Rec> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (Rec& r : done)
    if (r.dev == dev && r.fn == fn) {
      if (bytes <= r.bytes) return cudaSuccess;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e == cudaSuccess) r.bytes = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  done.push_back({dev, fn, bytes});
  return cudaSuccess;
}

int& launch_counter() {
  static thread_local int c = 0;
  return c;
}

namespace {
struct ProfRec {
  int stage;
  cudaEvent_t e0, e1;
};
struct ProfState {
  bool on = false;
  unsigned long long* ctr = nullptr;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<ProfRec> recs;
  cudaEvent_t pending = nullptr;
};
ProfState& prof() {
  static ProfState p;
  return p;
}
cudaEvent_t prof_event() {
  ProfState& P = prof();
  if (P.used == P.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    P.pool.push_back(e);
  }
  return P.pool[P.used++];
}
}  // namespace

unsigned long long* prof_counter(int stage) {
  ProfState& P = prof();
  return (P.on && P.ctr) ? P.ctr + stage : nullptr;
}
// NVTX range names of the stages (host-side ranges around every stage launch; nsys / ncu --nvtx)
static const char* const kStageNames[NSTAGE] = {
    "qal:liouvillian", "qal:commutators", "qal:expm_fold", "qal:tree", "qal:fidelity", "qal:prefix_chain",
    "qal:suffix_chain", "qal:grad_slices", "qal:dense_gemm", "qal:blk_expm_fold", "qal:blk_tree",
    "qal:blk_prefix", "qal:blk_suffix_chain", "qal:blk_grad_slices", "qal:blk_gemm", "qal:blk_fold"};
void prof_pre(int stage, cudaStream_t st) {
  nvtxRangePushA(stage >= 0 && stage < NSTAGE ? kStageNames[stage] : "qal");
  ProfState& P = prof();
  if (!P.on) return;
  P.pending = prof_event();
  cudaEventRecord(P.pending, st);
}
void prof_post(int stage, cudaStream_t st) {
  nvtxRangePop();
  ProfState& P = prof();
  if (!P.on || !P.pending) return;
  cudaEvent_t e1 = prof_event();
  cudaEventRecord(e1, st);
  P.recs.push_back({stage, P.pending, e1});
  P.pending = nullptr;
}

}  // namespace qal

using namespace qal;

namespace {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
thread_local cudaError_t g_last_cuda_error = cudaSuccess;   // per host thread, for qal_last_cuda_error
inline int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return QAL_OK;
  g_last_cuda_error = e;
  return QAL_ERR_CUDA;
}
// a failing runtime call or launcher: record its error and return QAL_ERR_CUDA
#define QAL_TRY(expr)                                  \
  do {                                                 \
    const cudaError_t qal_e_ = (expr);                 \
    if (qal_e_ != cudaSuccess) return cuda_rc(qal_e_); \
  } while (0)
inline const double2* D2(const qal_c128* p) { return reinterpret_cast<const double2*>(p); }
inline double2* D2(qal_c128* p) { return reinterpret_cast<double2*>(p); }
inline int ncomm_of(int J) { return J + J * (J - 1) / 2; }

size_t tree_ws_bytes(int batch, int count) {
  if (count <= 2) return 0;
  const size_t c1 = (size_t)(count + 1) / 2, c2 = (c1 + 1) / 2;
  return (size_t)batch * (c1 + c2) * MAT_BYTES;
}

constexpr size_t BIG = (size_t)4096 * 4096;      // complex elements of an n = 4096 matrix
constexpr size_t BIG_BYTES = BIG * 16;

size_t dense_tree_ws_bytes(int batch, int count) {
  const size_t c1 = (size_t)(count + 1) / 2, c2 = (c1 + 1) / 2;
  return (count <= 2 ? 0 : (size_t)batch * (c1 + c2) * BIG_BYTES) + 3 * BIG_BYTES;
}

// n = 4096 balanced tree: level by level, one dense product per pair (each fills the GPU)
int run_dense_tree(int batch, int count, const double2* U, double2* out, void* ws, cudaStream_t st) {
  if (count == 1) return cuda_rc(cudaMemcpyAsync(out, U, (size_t)batch * BIG_BYTES, cudaMemcpyDeviceToDevice, st));
  const size_t c1 = (size_t)(count + 1) / 2, c2 = (c1 + 1) / 2;
  double* tiles = reinterpret_cast<double*>(ws);
  double2* bufA = reinterpret_cast<double2*>(tiles + 3 * BIG * 2);
  double2* bufB = bufA + (size_t)batch * c1 * BIG;
  (void)c2;
  const double2* in = U;
  int cnt = count, lvl = 0;
  while (cnt > 1) {
    const int half = (cnt + 1) / 2;
    double2* dst = (half == 1) ? out : ((lvl & 1) ? bufB : bufA);
    for (int b = 0; b < batch; ++b)
      for (int i = 0; i < half; ++i) {
        const double2* src = in + ((size_t)b * cnt) * BIG;
        double2* d = dst + ((size_t)b * half + i) * BIG;
        if (2 * i + 1 == cnt) {
          if (cudaMemcpyAsync(d, src + (size_t)(cnt - 1) * BIG, BIG_BYTES, cudaMemcpyDeviceToDevice, st) !=
              cudaSuccess)
            return QAL_ERR_CUDA;
        } else if (launch_dense_tree_pair(src + (size_t)(2 * i + 1) * BIG, src + (size_t)(2 * i) * BIG, d, tiles,
                                          st) != cudaSuccess) {
          return QAL_ERR_CUDA;
        }
      }
    in = dst;
    cnt = half;
    ++lvl;
  }
  return QAL_OK;
}

// Balanced tree over `count` natural matrices per pulse -> out.
int run_tree(int batch, int count, const double2* U, double2* out, void* ws, cudaStream_t st) {
  if (count == 1) return cuda_rc(cudaMemcpyAsync(out, U, (size_t)batch * MAT_BYTES, cudaMemcpyDeviceToDevice, st));
  const size_t c1 = (size_t)(count + 1) / 2;
  double2* bufA = reinterpret_cast<double2*>(ws);
  double2* bufB = bufA ? bufA + (size_t)batch * c1 * PLANE_C : nullptr;
  const double2* in = U;
  int cnt = count;
  int lvl = 0;
  while (cnt > 1) {
    const int half = (cnt + 1) / 2;
    double2* dst = (half == 1) ? out : ((lvl & 1) ? bufB : bufA);
    cudaError_t e = launch_tree_level(batch, cnt, in, dst, st);
    QAL_TRY(e);
    in = dst;
    cnt = half;
    ++lvl;
  }
  return QAL_OK;
}

bool is_fin(double x) { return std::isfinite(x); }

struct Common {
  Basis B;
  SliceGrid G;
};

// ------------------------------------------------------------------ coherence-block path
int check_plan(const qal_block_plan* p) {
  if (!p) return QAL_ERR_NULL;
  if (p->n != 64 || p->d != 8 || p->ngroups < 1 || p->ngroups > QAL_BLK_MAX_GROUPS) return QAL_ERR_UNSUPPORTED;
  if (p->nrows < 8 || p->nrows > QAL_BLK_MAX_ROWS || p->nrows % 8) return QAL_ERR_DIM;
  if (p->launch_sets < QAL_BLK_SETS_DEFAULT || p->launch_sets > QAL_BLK_SETS_PAIRS) return QAL_ERR_UNSUPPORTED;
  int row = 0, off = 0;
  for (int g = 0; g < p->ngroups; ++g) {
    const int w = p->width[g];
    if (w < 8 || w > 24 || w % 8 || p->row0[g] != row || p->off[g] != off) return QAL_ERR_DIM;
    row += w;
    off += w * w;
  }
  if (row != p->nrows || off != p->packed) return QAL_ERR_DIM;
  for (int r = 0; r < p->nrows; ++r)
    if (p->perm[r] < -1 || p->perm[r] >= 64 || p->weight[r] < 0 || p->weight[r] > 2) return QAL_ERR_DIM;
  return QAL_OK;
}

struct BlkCommon {
  BlkBasis B;
  SliceGrid G;
};
int check_block_basis(const qal_block_plan* p, int batch, int n_slices, double T, int order, int mode, int J,
                      const double* u, const qal_c128* L0, long long L0s, const qal_c128* Lc, const qal_c128* Lcomm,
                      long long Lcs, BlkCommon& c) {
  int rc = check_plan(p);
  if (rc != QAL_OK) return rc;
  if (batch < 1 || n_slices < 1) return QAL_ERR_EMPTY;
  if (!is_fin(T) || T <= 0.0) return QAL_ERR_NONFINITE;
  if (order != 2 && order != 4) return QAL_ERR_UNSUPPORTED;
  if (mode != QAL_CTRL_PWC && mode != QAL_CTRL_NODES) return QAL_ERR_UNSUPPORTED;
  if (J < 1 || J > QAL_MAX_CTRL) return QAL_ERR_UNSUPPORTED;
  if (!u || !L0 || !Lc) return QAL_ERR_NULL;
  if (L0s != 0 && L0s != (long long)p->packed) return QAL_ERR_DIM;
  const bool comm = (mode == QAL_CTRL_NODES && order == 4);
  if (comm && !Lcomm) return QAL_ERR_NULL;
  if (comm && Lcs != 0 && Lcs != (long long)ncomm_of(J) * p->packed) return QAL_ERR_DIM;
  const double h = T / n_slices;
  c.B.L0 = D2(L0);
  c.B.L0_stride = L0s;
  c.B.Lc = D2(Lc);
  c.B.Lcomm = comm ? D2(Lcomm) : nullptr;
  c.B.Lcomm_stride = comm ? Lcs : 0;
  c.B.J = J;
  c.B.ncomm = comm ? ncomm_of(J) : 0;
  c.B.packed = p->packed;
  c.G.h = h;
  c.G.c4 = (order == 4) ? std::sqrt(3.0) * h * h / 12.0 : 0.0;
  c.G.mode = mode;
  c.G.u = u;
  c.G.count = n_slices;
  return QAL_OK;
}

size_t blk_mat_bytes(const qal_block_plan* p) { return (size_t)p->packed * 16; }

size_t blk_tree_ws_bytes(const qal_block_plan* p, int batch, int count) {
  if (count <= 2) return 0;
  const size_t c1 = (size_t)(count + 1) / 2, c2 = (c1 + 1) / 2;
  return (size_t)batch * (c1 + c2) * blk_mat_bytes(p);
}

int run_blk_tree(const qal_block_plan* p, int batch, int count, const double2* U, double2* out, void* ws,
                 cudaStream_t st) {
  const size_t mb = blk_mat_bytes(p);
  if (count == 1) return cuda_rc(cudaMemcpyAsync(out, U, (size_t)batch * mb, cudaMemcpyDeviceToDevice, st));
  const size_t c1 = (size_t)(count + 1) / 2;
  double2* bufA = reinterpret_cast<double2*>(ws);
  double2* bufB = bufA ? bufA + (size_t)batch * c1 * p->packed : nullptr;
  const double2* in = U;
  int cnt = count, lvl = 0;
  while (cnt > 1) {
    const int half = (cnt + 1) / 2;
    double2* dst = (half == 1) ? out : ((lvl & 1) ? bufB : bufA);
    QAL_TRY(launch_blk_tree_level(*p, batch, cnt, in, dst, st));
    in = dst;
    cnt = half;
    ++lvl;
  }
  return QAL_OK;
}

size_t blk_grad_ws_bytes(const qal_block_plan* p, int batch, int n_slices);
int blk_fidelity_grad_impl(const qal_block_plan* p, int batch, const BlkCommon& c, const double2* V, double* F,
                           double* grad, double2* Lam, int* status, void* ws, cudaStream_t st,
                           const double2* Cseed = nullptr);
int blk_forward_impl(const qal_block_plan* p, int batch, const BlkCommon& c, double2* Lam, int* status, void* ws,
                     cudaStream_t st, bool with_suffix, const double2* V);
int blk_backward_impl(const qal_block_plan* p, int batch, const BlkCommon& c, const double2* V, double* grad,
                      int* status, void* ws, cudaStream_t st, const double2* Cseed, bool suffix_done);

// chunk of the block forward fold: keep >= ~4 CTAs per SM busy, chunk | n_slices
int blk_default_chunk(int batch, int n_slices) {
  const long long want = 4LL * num_sms();
  int ch = n_slices;
  while (ch > 1 && (long long)batch * (n_slices / ch) < want && (ch % 2) == 0) ch /= 2;
  return ch;
}


int check_basis(int n_or_d_ok, int batch, int n_slices, double T, int order, int mode, int J, const double* u,
                const qal_c128* L0, long long L0s, const qal_c128* Lc, const qal_c128* Lcomm, long long Lcs,
                Common& c, bool dense = false) {
  if (!n_or_d_ok) return QAL_ERR_UNSUPPORTED;
  if (batch < 1 || n_slices < 1) return QAL_ERR_EMPTY;
  if (!is_fin(T) || T <= 0.0) return QAL_ERR_NONFINITE;
  if (order != 2 && order != 4) return QAL_ERR_UNSUPPORTED;
  if (mode != QAL_CTRL_PWC && mode != QAL_CTRL_NODES) return QAL_ERR_UNSUPPORTED;
  if (J < 1 || J > QAL_MAX_CTRL) return QAL_ERR_UNSUPPORTED;
  if (!u || !L0 || !Lc) return QAL_ERR_NULL;
  if (L0s != 0 && L0s != (long long)(dense ? BIG : PLANE_C)) return QAL_ERR_DIM;
  if (dense && mode != QAL_CTRL_PWC) return QAL_ERR_UNSUPPORTED;
  const bool comm = (mode == QAL_CTRL_NODES && order == 4);
  if (comm && !Lcomm) return QAL_ERR_NULL;
  if (comm && Lcs != 0 && Lcs != (long long)ncomm_of(J) * PLANE_C) return QAL_ERR_DIM;
  const double h = T / n_slices;
  c.B.L0 = D2(L0);
  c.B.L0_stride = L0s;
  c.B.Lc = D2(Lc);
  c.B.Lcomm = comm ? D2(Lcomm) : nullptr;
  c.B.Lcomm_stride = comm ? Lcs : 0;
  c.B.J = J;
  c.B.ncomm = comm ? ncomm_of(J) : 0;
  c.G.h = h;
  c.G.c4 = (order == 4) ? std::sqrt(3.0) * h * h / 12.0 : 0.0;
  c.G.mode = mode;
  c.G.u = u;
  c.G.count = n_slices;
  return QAL_OK;
}

// workspace of the gradient path: U_img, P_img, X_img [batch][count] images + scratch
struct GradWs {
  double *U, *P, *X, *scratch;
};
GradWs grad_ws(void* ws, int batch, int count) {
  const size_t seq = (size_t)batch * count * IMG;
  GradWs g;
  g.U = reinterpret_cast<double*>(ws);
  g.P = g.U + seq;
  g.X = g.P + seq;
  g.scratch = g.X + seq + (size_t)batch * IMG;   // leaves room for one [batch][n][n] complex temp (Lambda)
  return g;
}

int forward_impl(int batch, const Common& c, const double2* P_init, double2* Lam, int* status, void* ws,
                 cudaStream_t st) {
  GradWs g = grad_ws(ws, batch, c.G.count);
  FwdOut O{nullptr, g.U, nullptr, 1, status};
  QAL_TRY(launch_expm_fold(batch, c.B, c.G, O, st));
  QAL_TRY(launch_prefix_chain(batch, c.G.count, g.U, g.P, Lam, P_init, st));
  return QAL_OK;
}

int vjp_impl(int batch, const Common& c, const double2* V, const double2* C, double gscale, double* grad, int* status,
             void* ws, cudaStream_t st) {
  GradWs g = grad_ws(ws, batch, c.G.count);
  QAL_TRY(launch_suffix_chain(batch, c.G.count, g.U, V, C, g.X, st));
  QAL_TRY(launch_grad_slices(batch, c.B, c.G, g.P, g.X, grad, status, g.scratch, gscale, st));
  return QAL_OK;
}

}  // namespace

extern "C" {

int qal_abi_version(void) { return QAL_ABI_VERSION; }

const char* qal_last_cuda_error(void) {
  // the CUDA error behind the last QAL_ERR_CUDA of this host thread (or the runtime's pending one)
  const cudaError_t e = g_last_cuda_error != cudaSuccess ? g_last_cuda_error : cudaPeekAtLastError();
  return cudaGetErrorString(e);
}

int qal_real_mults_per_complex_product(void) { return qal::QAL_REAL_MMAS_PER_CMMA; }

const char* qal_status_string(int code) {
  switch (code) {
    case QAL_OK: return "ok";
    case QAL_ERR_NULL: return "required pointer is NULL";
    case QAL_ERR_DIM: return "inconsistent dimensions";
    case QAL_ERR_EMPTY: return "empty input";
    case QAL_ERR_NONFINITE: return "non-finite value";
    case QAL_ERR_UNSUPPORTED: return "unsupported size or mode";
    case QAL_ERR_WORKSPACE: return "workspace too small";
    case QAL_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

int qal_last_launch_count(void) { return launch_counter(); }

int qal_default_chunk(int batch, int n_slices) {
  if (batch < 1 || n_slices < 1) return 1;
  int c = 1;
  while (c * 2 <= 64 && n_slices % (c * 2) == 0) c *= 2;
  const long long want = 4LL * num_sms();
  while (c > 1 && (long long)batch * (n_slices / c) < want) c /= 2;
  return c;
}

size_t qal_workspace_bytes(int op, int n, int batch, int n_slices, int n_ctrl, int flags) {
  (void)n_ctrl;
  (void)flags;
  if (batch < 1 || n_slices < 1) return 0;
  if (n == 4096) {
    switch (op) {
      case QAL_OP_EXPM_SLICES: return dense_expm_ws_bytes();
      case QAL_OP_ORDERED_PRODUCT: return dense_tree_ws_bytes(batch, n_slices);
      case QAL_OP_FIDELITY: return dense_expm_ws_bytes() + (size_t)batch * (BIG_BYTES + DENSE_FID_PART_BYTES);
      case QAL_OP_FIDELITY_REDUCE: return (size_t)batch * DENSE_FID_PART_BYTES;
      default: return 0;
    }
  }
  if (n != 64) return 0;
  switch (op) {
    case QAL_OP_ORDERED_PRODUCT: return tree_ws_bytes(batch, n_slices);
    case QAL_OP_FIDELITY: {
      const int ch = qal_default_chunk(batch, n_slices);
      const int nch = n_slices / ch;
      return (size_t)batch * nch * MAT_BYTES + tree_ws_bytes(batch, nch) + (size_t)batch * MAT_BYTES;
    }
    case QAL_OP_FIDELITY_GRAD:
    case QAL_OP_VJP:
      return 3 * (size_t)batch * n_slices * MAT_BYTES + (size_t)batch * MAT_BYTES + grad_scratch_bytes();
    default: return 0;
  }
}

int qal_build_liouvillian(int d, int batch, const qal_c128* H0, int n_ctrl, const qal_c128* Hc, int n_cops,
                          const qal_c128* C, int want_comm, qal_c128* L0, qal_c128* Lc, qal_c128* Lcomm,
                          void* stream) {
  launch_counter() = 0;
  if (d != 8 && d != 64) return QAL_ERR_UNSUPPORTED;
  if (batch < 1) return QAL_ERR_EMPTY;
  if (n_ctrl < 0 || n_ctrl > QAL_MAX_CTRL || n_cops < 0) return QAL_ERR_DIM;
  if (!H0 || !L0) return QAL_ERR_NULL;
  if (n_ctrl > 0 && (!Hc || !Lc)) return QAL_ERR_NULL;
  if (n_cops > 0 && !C) return QAL_ERR_NULL;
  if (want_comm && (n_ctrl < 1 || !Lcomm)) return n_ctrl < 1 ? QAL_ERR_DIM : QAL_ERR_NULL;
  if (d == 64) {
    if (want_comm) return QAL_ERR_UNSUPPORTED;
    return cuda_rc(launch_dense_liouvillian(batch, D2(H0), n_ctrl, D2(Hc), n_cops, D2(C), D2(L0), D2(Lc),
                                            S(stream)));
  }
  cudaError_t e = launch_liouvillian(batch, D2(H0), n_ctrl, D2(Hc), n_cops, D2(C), D2(L0), D2(Lc), S(stream));
  QAL_TRY(e);
  if (want_comm) e = launch_commutators(batch, n_ctrl, D2(L0), D2(Lc), D2(Lcomm), S(stream));
  return cuda_rc(e);
}

int qal_magnus_expm_slices(int n, int batch, int n_slices, double T, int k0, int count, int magnus_order,
                           int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0,
                           long long L0_batch_stride, const qal_c128* Lc, const qal_c128* Lcomm,
                           long long Lcomm_batch_stride, qal_c128* U_out, int chunk, qal_c128* chunk_prod,
                           int* status, void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  Common c;
  int rc = check_basis(n == 64 || n == 4096, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0,
                       L0_batch_stride, Lc, Lcomm, Lcomm_batch_stride, c, n == 4096);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!U_out && !chunk_prod) return QAL_ERR_NULL;
  if (chunk < 1 || count % chunk != 0) return QAL_ERR_DIM;
  if (n == 4096) {
    if (ctrl_mode != QAL_CTRL_PWC) return QAL_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < dense_expm_ws_bytes()) return QAL_ERR_WORKSPACE;
    if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, S(stream)) != cudaSuccess) return QAL_ERR_CUDA;
    for (int b = 0; b < batch; ++b) {
      cudaError_t e = launch_dense_expm_fold(
          D2(L0) + (size_t)b * L0_batch_stride, D2(Lc), n_ctrl, u + (size_t)b * count * n_ctrl, count, c.G.h,
          chunk_prod ? chunk : count, chunk_prod ? D2(chunk_prod) + (size_t)b * (count / chunk) * BIG : nullptr,
          U_out ? D2(U_out) + (size_t)b * count * BIG : nullptr, status ? status + b : nullptr,
          reinterpret_cast<double*>(ws), nullptr, S(stream));
      QAL_TRY(e);
    }
    return QAL_OK;
  }
  (void)ws;
  (void)ws_bytes;
  c.G.count = count;
  FwdOut O;
  O.U_nat = D2(U_out);
  O.U_img = nullptr;
  O.chunk_nat = D2(chunk_prod);
  O.chunk = chunk_prod ? chunk : 1;
  O.status = status;
  if (!chunk_prod && count % O.chunk) return QAL_ERR_DIM;
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, S(stream)) != cudaSuccess) return QAL_ERR_CUDA;
  return cuda_rc(launch_expm_fold(batch, c.B, c.G, O, S(stream)));
}

int qal_ordered_product(int n, int batch, int count, const qal_c128* U, qal_c128* out, void* ws, size_t ws_bytes,
                        void* stream) {
  launch_counter() = 0;
  if (n != 64 && n != 4096) return QAL_ERR_UNSUPPORTED;
  if (batch < 1 || count < 1) return QAL_ERR_EMPTY;
  if (!U || !out) return QAL_ERR_NULL;
  if (n == 4096) {
    const size_t needd = dense_tree_ws_bytes(batch, count);
    if (count > 1 && (!ws || ws_bytes < needd)) return QAL_ERR_WORKSPACE;
    return run_dense_tree(batch, count, D2(U), D2(out), ws, S(stream));
  }
  const size_t need = tree_ws_bytes(batch, count);
  if (need > 0 && (!ws || ws_bytes < need)) return QAL_ERR_WORKSPACE;
  return run_tree(batch, count, D2(U), D2(out), ws, S(stream));
}

int qal_ordered_scan(int n, int batch, int count, const qal_c128* U, qal_c128* prefix_excl, qal_c128* suffix_excl,
                     void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  if (n != 64) return QAL_ERR_UNSUPPORTED;
  if (batch < 1 || count < 1) return QAL_ERR_EMPTY;
  if (!U || (!prefix_excl && !suffix_excl)) return QAL_ERR_NULL;
  if (!ws || ws_bytes < 4 * (size_t)batch * count * MAT_BYTES) return QAL_ERR_WORKSPACE;
  return cuda_rc(launch_scan(batch, count, D2(U), D2(prefix_excl), D2(suffix_excl), reinterpret_cast<double2*>(ws),
                             S(stream)));
}

int qal_batched_matmul(int n, int count, const qal_c128* A, long long strideA, const qal_c128* B, long long strideB,
                       qal_c128* C, void* stream) {
  launch_counter() = 0;
  if (n != 64) return QAL_ERR_UNSUPPORTED;
  if (count < 1) return QAL_ERR_EMPTY;
  if (!A || !B || !C) return QAL_ERR_NULL;
  if ((strideA != 0 && strideA != (long long)PLANE_C) || (strideB != 0 && strideB != (long long)PLANE_C))
    return QAL_ERR_DIM;
  return cuda_rc(launch_batched_mm(count, D2(A), strideA, D2(B), strideB, D2(C), S(stream)));
}

int qal_fidelity(int d, int batch, const qal_c128* Lambda, const qal_c128* V, double* F, void* stream) {
  launch_counter() = 0;
  if (d != 8 && d != 64) return QAL_ERR_UNSUPPORTED;
  if (batch < 1) return QAL_ERR_EMPTY;
  if (!Lambda || !V || !F) return QAL_ERR_NULL;
  if (d == 64) return cuda_rc(launch_dense_fidelity(batch, D2(Lambda), D2(V), F, nullptr, S(stream)));
  return cuda_rc(launch_fidelity(batch, D2(Lambda), D2(V), F, S(stream)));
}

int qal_fidelity_ws(int d, int batch, const qal_c128* Lambda, const qal_c128* V, double* F, void* ws,
                    size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  if (d != 8 && d != 64) return QAL_ERR_UNSUPPORTED;
  if (batch < 1) return QAL_ERR_EMPTY;
  if (!Lambda || !V || !F) return QAL_ERR_NULL;
  if (d == 8) return cuda_rc(launch_fidelity(batch, D2(Lambda), D2(V), F, S(stream)));
  if (!ws || ws_bytes < qal_workspace_bytes(QAL_OP_FIDELITY_REDUCE, 4096, batch, 1, 0, 0)) return QAL_ERR_WORKSPACE;
  return cuda_rc(launch_dense_fidelity(batch, D2(Lambda), D2(V), F, reinterpret_cast<double*>(ws), S(stream)));
}

int qal_fidelity_grad(int d, int batch, int n_slices, double T, int magnus_order, int ctrl_mode, int n_ctrl,
                      const double* u, const qal_c128* L0, long long L0_batch_stride, const qal_c128* Lc,
                      const qal_c128* Lcomm, long long Lcomm_batch_stride, const qal_c128* V, double* F,
                      double* grad, qal_c128* Lambda, int* status, void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  Common c;
  int rc = check_basis(d == 8 || (d == 64 && !grad), batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0,
                       L0_batch_stride, Lc, Lcomm, Lcomm_batch_stride, c, d == 64);
  if (rc != QAL_OK) return rc;
  if (!V || !F) return QAL_ERR_NULL;
  if (d == 64) {   // forward only: one fold per pulse, then the fidelity
    const size_t needd = qal_workspace_bytes(QAL_OP_FIDELITY, 4096, batch, n_slices, n_ctrl, ctrl_mode);
    if (!ws || ws_bytes < needd) return QAL_ERR_WORKSPACE;
    double2* lam = Lambda ? D2(Lambda)
                          : reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + dense_expm_ws_bytes());
    cudaStream_t st = S(stream);
    if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
    for (int b = 0; b < batch; ++b) {
      QAL_TRY(launch_dense_expm_fold(D2(L0) + (size_t)b * L0_batch_stride, D2(Lc), n_ctrl,
                                 u + (size_t)b * n_slices * n_ctrl, n_slices, c.G.h, n_slices, lam + (size_t)b * BIG,
                                 nullptr, status ? status + b : nullptr, reinterpret_cast<double*>(ws), nullptr,
                                 st));
    }
    double* part = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + dense_expm_ws_bytes() +
                                             (size_t)batch * BIG_BYTES);
    return cuda_rc(launch_dense_fidelity(batch, lam, D2(V), F, part, st));
  }
  const size_t need = qal_workspace_bytes(grad ? QAL_OP_FIDELITY_GRAD : QAL_OP_FIDELITY, 64, batch, n_slices,
                                          n_ctrl, ctrl_mode);
  if (!ws || ws_bytes < need) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  char* w = reinterpret_cast<char*>(ws);
  if (!grad) {
    const int ch = qal_default_chunk(batch, n_slices);
    const int nch = n_slices / ch;
    double2* parts = reinterpret_cast<double2*>(w);
    w += (size_t)batch * nch * MAT_BYTES;
    double2* lam_tmp = reinterpret_cast<double2*>(w);
    w += (size_t)batch * MAT_BYTES;
    double2* lam = Lambda ? D2(Lambda) : lam_tmp;
    FwdOut O{nullptr, nullptr, parts, ch, status};
    QAL_TRY(launch_expm_fold(batch, c.B, c.G, O, st));
    rc = run_tree(batch, nch, parts, lam, w, st);
    if (rc != QAL_OK) return rc;
    return cuda_rc(launch_fidelity(batch, lam, D2(V), F, st));
  }
  // gradient path: forward (U_k images, prefix P_k) -> fidelity -> VJP with C = S_V^dag (in-kernel from V)
  double2* lam = Lambda ? D2(Lambda) : reinterpret_cast<double2*>(w + 3 * (size_t)batch * n_slices * MAT_BYTES);
  if ((rc = forward_impl(batch, c, nullptr, lam, status, ws, st)) != QAL_OK) return rc;
  QAL_TRY(launch_fidelity(batch, lam, D2(V), F, st));
  return vjp_impl(batch, c, D2(V), nullptr, 1.0 / 64.0, grad, status, ws, st);
}

int qal_propagator_forward(int d, int batch, int n_slices, double T, int k0, int count, int magnus_order,
                           int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0, long long L0_batch_stride,
                           const qal_c128* Lc, const qal_c128* Lcomm, long long Lcomm_batch_stride,
                           const qal_c128* P_init, qal_c128* Lambda, int* status, void* ws, size_t ws_bytes,
                           void* stream) {
  launch_counter() = 0;
  Common c;
  int rc = check_basis(d == 8, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0, L0_batch_stride, Lc,
                       Lcomm, Lcomm_batch_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!Lambda) return QAL_ERR_NULL;
  c.G.count = count;
  if (!ws || ws_bytes < qal_workspace_bytes(QAL_OP_VJP, 64, batch, count, n_ctrl, ctrl_mode)) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  return forward_impl(batch, c, D2(P_init), D2(Lambda), status, ws, st);
}

int qal_propagator_vjp(int d, int batch, int n_slices, double T, int k0, int count, int magnus_order, int ctrl_mode,
                       int n_ctrl, const double* u, const qal_c128* L0, long long L0_batch_stride, const qal_c128* Lc,
                       const qal_c128* Lcomm, long long Lcomm_batch_stride, const qal_c128* C, double* grad,
                       int* status, void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  Common c;
  int rc = check_basis(d == 8, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0, L0_batch_stride, Lc,
                       Lcomm, Lcomm_batch_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!C || !grad) return QAL_ERR_NULL;
  c.G.count = count;
  if (!ws || ws_bytes < qal_workspace_bytes(QAL_OP_VJP, 64, batch, count, n_ctrl, ctrl_mode)) return QAL_ERR_WORKSPACE;
  return vjp_impl(batch, c, nullptr, D2(C), 1.0, grad, status, ws, S(stream));
}

int qal_fidelity_cotangent(int d, const qal_c128* V, qal_c128* C, void* stream) {
  launch_counter() = 0;
  if (d != 8) return QAL_ERR_UNSUPPORTED;
  if (!V || !C) return QAL_ERR_NULL;
  return cuda_rc(launch_fidelity_cotangent(D2(V), D2(C), S(stream)));
}

int qal_logical_loss(int d, int batch, const qal_c128* Lambda, const qal_c128* Pproj, const qal_c128* G, double* loss,
                     qal_c128* C, void* stream) {
  launch_counter() = 0;
  if (d != 8) return QAL_ERR_UNSUPPORTED;
  if (batch < 1) return QAL_ERR_EMPTY;
  if (!Lambda || !Pproj || !G || !loss) return QAL_ERR_NULL;
  return cuda_rc(launch_logical_loss(batch, D2(Lambda), D2(Pproj), D2(G), loss, D2(C), S(stream)));
}

int qal_adam_step(int n, double* theta, const double* grad, double* m, double* v, int t, double lr, double beta1,
                  double beta2, double eps, void* stream) {
  launch_counter() = 0;
  if (n < 1) return QAL_ERR_EMPTY;
  if (t < 1) return QAL_ERR_DIM;
  if (!theta || !grad || !m || !v) return QAL_ERR_NULL;
  if (!is_fin(lr) || !is_fin(beta1) || !is_fin(beta2) || !is_fin(eps)) return QAL_ERR_NONFINITE;
  return cuda_rc(launch_adam(n, theta, grad, m, v, t, lr, beta1, beta2, eps, S(stream)));
}

int qal_sample_controls_sines(int n_ctrl, int nterm, const double* prm, double u_max, int n_slices, double T,
                              int k0, int count, double* u_out, void* stream) {
  launch_counter() = 0;
  if (n_ctrl < 1 || n_ctrl > QAL_MAX_CTRL || nterm < 1) return QAL_ERR_UNSUPPORTED;
  if (n_slices < 1 || count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!is_fin(T) || T <= 0.0 || !is_fin(u_max)) return QAL_ERR_NONFINITE;
  if (!prm || !u_out) return QAL_ERR_NULL;
  return cuda_rc(launch_sample_sines(n_ctrl, nterm, prm, u_max, T / n_slices, k0, count, u_out, S(stream)));
}

int qal_profile_begin(unsigned long long* dev_counters) {
  ProfState& P = prof();
  P.on = true;
  P.ctr = dev_counters;
  P.recs.clear();
  P.used = 0;
  P.pending = nullptr;
  return QAL_OK;
}

int qal_profile_end(double* ms, int* launches) {
  ProfState& P = prof();
  if (!ms || !launches) return QAL_ERR_NULL;
  for (int i = 0; i < NSTAGE; ++i) { ms[i] = 0.0; launches[i] = 0; }
  int rc = QAL_OK;
  for (const ProfRec& r : P.recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&t, r.e0, r.e1) != cudaSuccess) {
      rc = QAL_ERR_CUDA;
      continue;
    }
    ms[r.stage] += t;
    launches[r.stage] += 1;
  }
  P.on = false;
  P.ctr = nullptr;
  P.recs.clear();
  P.used = 0;
  return rc;
}

int qal_fp64_peak_probe(int kind, int blocks, int iters, double* flops, double* sink, void* stream) {
  launch_counter() = 0;
  if (kind != 0 && kind != 1) return QAL_ERR_UNSUPPORTED;
  if (blocks < 1 || iters < 1) return QAL_ERR_EMPTY;
  if (!flops || !sink) return QAL_ERR_NULL;
  *flops = (kind == 0) ? (double)blocks * 8.0 * iters * 8.0 * 512.0 : (double)blocks * 256.0 * iters * 8.0 * 2.0;
  return cuda_rc(launch_fp64_probe(kind, blocks, iters, sink, S(stream)));
}


int qal_block_plan_build(int n, int nmat, const qal_c128* mats, int mirror, qal_block_plan* plan) {
  launch_counter() = 0;
  if (!mats || !plan) return QAL_ERR_NULL;
  if (nmat < 1) return QAL_ERR_EMPTY;
  return build_block_plan(n, nmat, D2(mats), mirror, plan);
}

int qal_block_pack(const qal_block_plan* plan, int count, const qal_c128* nat, qal_c128* packed, int* flag,
                   void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (!nat || !packed) return QAL_ERR_NULL;
  return cuda_rc(launch_blk_pack(*plan, count, D2(nat), D2(packed), flag, S(stream)));
}

int qal_block_check(const qal_block_plan* plan, int count, const qal_c128* nat, int broadcast, int* status,
                    int nstatus, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (count < 1 || nstatus < 1) return QAL_ERR_EMPTY;
  if (!nat || !status) return QAL_ERR_NULL;
  if (!broadcast && nstatus != count) return QAL_ERR_DIM;
  return cuda_rc(launch_blk_check_status(*plan, count, D2(nat), broadcast ? 1 : 0, status, nstatus, S(stream)));
}

int qal_block_unpack(const qal_block_plan* plan, int count, const qal_c128* packed, qal_c128* nat, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (!nat || !packed) return QAL_ERR_NULL;
  return cuda_rc(launch_blk_unpack(*plan, count, D2(packed), D2(nat), S(stream)));
}

int qal_block_expm_slices(const qal_block_plan* plan, int batch, int n_slices, double T, int k0, int count,
                          int magnus_order, int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0p,
                          long long L0p_stride, const qal_c128* Lcp, const qal_c128* Lcommp,
                          long long Lcommp_stride, int chunk, qal_c128* chunk_prod, int* status, void* stream) {
  launch_counter() = 0;
  BlkCommon c;
  int rc = check_block_basis(plan, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0p, L0p_stride, Lcp,
                             Lcommp, Lcommp_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (chunk < 1 || count % chunk) return QAL_ERR_DIM;
  if (!chunk_prod) return QAL_ERR_NULL;
  c.G.count = count;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  BlkFwdOut O{nullptr, D2(chunk_prod), chunk, status, nullptr};
  return cuda_rc(launch_blk_expm_fold(*plan, batch, c.B, c.G, O, st));
}

int qal_block_ordered_product(const qal_block_plan* plan, int batch, int count, const qal_c128* U, qal_c128* out,
                              void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (batch < 1 || count < 1) return QAL_ERR_EMPTY;
  if (!U || !out) return QAL_ERR_NULL;
  const size_t need = blk_tree_ws_bytes(plan, batch, count);
  if (need && (!ws || ws_bytes < need)) return QAL_ERR_WORKSPACE;
  return run_blk_tree(plan, batch, count, D2(U), D2(out), ws, S(stream));
}

int qal_block_fidelity(const qal_block_plan* plan, int batch, const qal_c128* Lambda_packed, const qal_c128* V,
                       double* F, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (batch < 1) return QAL_ERR_EMPTY;
  if (!Lambda_packed || !V || !F) return QAL_ERR_NULL;
  return cuda_rc(launch_blk_fidelity(*plan, batch, D2(Lambda_packed), D2(V), F, S(stream)));
}

size_t qal_block_workspace_bytes(const qal_block_plan* plan, int op, int batch, int n_slices) {
  if (check_plan(plan) != QAL_OK || batch < 1 || n_slices < 1) return 0;
  const size_t mb = blk_mat_bytes(plan);
  switch (op) {
    case QAL_OP_ORDERED_PRODUCT: return blk_tree_ws_bytes(plan, batch, n_slices);
    case QAL_OP_FIDELITY: {
      const int ch = blk_default_chunk(batch, n_slices);
      const int nch = n_slices / ch;
      return (size_t)batch * nch * mb + blk_tree_ws_bytes(plan, batch, nch) + (size_t)batch * mb;
    }
    case QAL_OP_FIDELITY_GRAD:
    case QAL_OP_VJP:
      return blk_grad_ws_bytes(plan, batch, n_slices);
    default: return 0;
  }
}

int qal_block_fidelity_grad(const qal_block_plan* plan, int batch, int n_slices, double T, int magnus_order,
                            int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0p, long long L0p_stride,
                            const qal_c128* Lcp, const qal_c128* Lcommp, long long Lcommp_stride, const qal_c128* V,
                            double* F, double* grad, qal_c128* Lambda_packed, int* status, void* ws, size_t ws_bytes,
                            void* stream) {
  launch_counter() = 0;
  BlkCommon c;
  int rc = check_block_basis(plan, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0p, L0p_stride, Lcp,
                             Lcommp, Lcommp_stride, c);
  if (rc != QAL_OK) return rc;
  if (!V || !F) return QAL_ERR_NULL;
  const size_t need = qal_block_workspace_bytes(plan, grad ? QAL_OP_FIDELITY_GRAD : QAL_OP_FIDELITY, batch, n_slices);
  if (!ws || ws_bytes < need) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  char* w = reinterpret_cast<char*>(ws);
  const size_t mb = blk_mat_bytes(plan);
  if (!grad) {
    const int ch = blk_default_chunk(batch, n_slices);
    const int nch = n_slices / ch;
    double2* parts = reinterpret_cast<double2*>(w);
    w += (size_t)batch * nch * mb;
    double2* lam_tmp = reinterpret_cast<double2*>(w);
    w += (size_t)batch * mb;
    double2* lam = Lambda_packed ? D2(Lambda_packed) : lam_tmp;
    BlkFwdOut O{nullptr, parts, ch, status, nullptr};
    QAL_TRY(launch_blk_expm_fold(*plan, batch, c.B, c.G, O, st));
    if ((rc = run_blk_tree(plan, batch, nch, parts, lam, w, st)) != QAL_OK) return rc;
    return cuda_rc(launch_blk_fidelity(*plan, batch, lam, D2(V), F, st));
  }
  return blk_fidelity_grad_impl(plan, batch, c, D2(V), F, grad, D2(Lambda_packed), status, ws, st);
}

int qal_block_propagator_vjp(const qal_block_plan* plan, int batch, int n_slices, double T, int k0, int count,
                             int magnus_order, int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0p,
                             long long L0p_stride, const qal_c128* Lcp, const qal_c128* Lcommp,
                             long long Lcommp_stride, const qal_c128* Cp, double* grad, qal_c128* Lambda_packed,
                             int* status, void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  BlkCommon c;
  int rc = check_block_basis(plan, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0p, L0p_stride, Lcp,
                             Lcommp, Lcommp_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!Cp || !grad) return QAL_ERR_NULL;
  c.G.count = count;
  if (!ws || ws_bytes < qal_block_workspace_bytes(plan, QAL_OP_VJP, batch, count)) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  return blk_fidelity_grad_impl(plan, batch, c, nullptr, nullptr, grad, D2(Lambda_packed), status, ws, st, D2(Cp));
}

int qal_block_propagator_forward(const qal_block_plan* plan, int batch, int n_slices, double T, int k0, int count,
                                 int magnus_order, int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0p,
                                 long long L0p_stride, const qal_c128* Lcp, const qal_c128* Lcommp,
                                 long long Lcommp_stride, qal_c128* Lambda_packed, int* status, void* ws,
                                 size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  BlkCommon c;
  int rc = check_block_basis(plan, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0p, L0p_stride, Lcp,
                             Lcommp, Lcommp_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!Lambda_packed) return QAL_ERR_NULL;
  c.G.count = count;
  if (!ws || ws_bytes < qal_block_workspace_bytes(plan, QAL_OP_VJP, batch, count)) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int) * batch, st) != cudaSuccess) return QAL_ERR_CUDA;
  return blk_forward_impl(plan, batch, c, D2(Lambda_packed), status, ws, st, false, nullptr);
}

int qal_block_propagator_backward(const qal_block_plan* plan, int batch, int n_slices, double T, int k0, int count,
                                  int magnus_order, int ctrl_mode, int n_ctrl, const double* u, const qal_c128* L0p,
                                  long long L0p_stride, const qal_c128* Lcp, const qal_c128* Lcommp,
                                  long long Lcommp_stride, const qal_c128* Cp, double* grad, int* status, void* ws,
                                  size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  BlkCommon c;
  int rc = check_block_basis(plan, batch, n_slices, T, magnus_order, ctrl_mode, n_ctrl, u, L0p, L0p_stride, Lcp,
                             Lcommp, Lcommp_stride, c);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (k0 < 0 || (long long)k0 + count > n_slices) return QAL_ERR_DIM;
  if (!Cp || !grad) return QAL_ERR_NULL;
  c.G.count = count;
  if (!ws || ws_bytes < qal_block_workspace_bytes(plan, QAL_OP_VJP, batch, count)) return QAL_ERR_WORKSPACE;
  return blk_backward_impl(plan, batch, c, nullptr, grad, status, ws, S(stream), D2(Cp), false);
}

int qal_block_ordered_scan(const qal_block_plan* plan, int batch, int count, const qal_c128* U,
                           qal_c128* prefix_excl, qal_c128* suffix_excl, void* ws, size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (batch < 1 || count < 1) return QAL_ERR_EMPTY;
  if (!U || (!prefix_excl && !suffix_excl)) return QAL_ERR_NULL;
  if (!ws || ws_bytes < 4 * (size_t)batch * count * blk_mat_bytes(plan)) return QAL_ERR_WORKSPACE;
  return cuda_rc(launch_blk_scan(*plan, batch, count, D2(U), D2(prefix_excl), D2(suffix_excl),
                                 reinterpret_cast<double2*>(ws), S(stream)));
}

int qal_block_batched_matmul(const qal_block_plan* plan, int count, const qal_c128* A, long long strideA,
                             const qal_c128* B, long long strideB, qal_c128* C, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (count < 1) return QAL_ERR_EMPTY;
  if (!A || !B || !C) return QAL_ERR_NULL;
  if ((strideA != 0 && strideA != (long long)plan->packed) || (strideB != 0 && strideB != (long long)plan->packed))
    return QAL_ERR_DIM;
  return cuda_rc(launch_blk_batched_mm(*plan, count, D2(A), strideA, D2(B), strideB, D2(C), S(stream)));
}

int qal_block_fidelity_cotangent(const qal_block_plan* plan, const qal_c128* V, qal_c128* C, void* stream) {
  launch_counter() = 0;
  int rc = check_plan(plan);
  if (rc != QAL_OK) return rc;
  if (!V || !C) return QAL_ERR_NULL;
  return cuda_rc(launch_blk_fidelity_cotangent(*plan, D2(V), D2(C), S(stream)));
}

size_t qal_bigblock_plan_workspace_bytes(void) { return bb_plan_ws_bytes(); }

int qal_bigblock_plan_build(int nmat, const qal_c128* mats, int mirror, qal_bigblock_plan* plan, void* ws,
                            size_t ws_bytes, void* stream) {
  launch_counter() = 0;
  if (!mats || !plan) return QAL_ERR_NULL;
  if (nmat < 1) return QAL_ERR_EMPTY;
  if (!ws || ws_bytes < bb_plan_ws_bytes()) return QAL_ERR_WORKSPACE;
  return build_bigblock_plan(nmat, D2(mats), mirror, plan, ws, S(stream));
}

size_t qal_bigblock_workspace_bytes(const qal_bigblock_plan* plan) {
  if (!plan || plan->n != 4096 || plan->nb < 1) return 0;
  return bb_ws_bytes(*plan);
}

int qal_bigblock_expm_slices(const qal_bigblock_plan* plan, int n_slices, double T, int count, int n_ctrl,
                             const double* u, const qal_c128* L0, const qal_c128* Lc, int chunk,
                             qal_c128* chunk_prod, int* status, int* flag, void* ws, size_t ws_bytes,
                             void* stream) {
  launch_counter() = 0;
  if (!plan || !u || !L0 || !Lc || !chunk_prod) return QAL_ERR_NULL;
  if (plan->n != 4096 || plan->nb < 1 || plan->nb > QAL_BB_MAX_BLOCKS) return QAL_ERR_UNSUPPORTED;
  if (n_slices < 1 || count < 1) return QAL_ERR_EMPTY;
  if (count > n_slices || chunk < 1 || count % chunk) return QAL_ERR_DIM;
  if (n_ctrl < 1 || n_ctrl > QAL_MAX_CTRL) return QAL_ERR_UNSUPPORTED;
  if (!is_fin(T) || T <= 0.0) return QAL_ERR_NONFINITE;
  if (!ws || ws_bytes < bb_ws_bytes(*plan)) return QAL_ERR_WORKSPACE;
  cudaStream_t st = S(stream);
  if (status && cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess) return QAL_ERR_CUDA;
  return cuda_rc(launch_bb_expm_fold(*plan, D2(L0), D2(Lc), n_ctrl, u, count, T / n_slices, chunk, D2(chunk_prod),
                                     status, flag, reinterpret_cast<double*>(ws), st));
}
}  // extern "C"

namespace {
size_t blk_grad_ws_bytes(const qal_block_plan* p, int batch, int n_slices) {
  const size_t img = (size_t)p->packed * 16;
  return 3 * (size_t)batch * n_slices * img + (size_t)batch * img + blk_grad_scratch_bytes(*p, batch, n_slices);
}
// workspace layout of the block gradient path: U_k, P_k, X_{k+1} image sequences, Lambda, scheme codes
struct BlkGradWs {
  double *U, *P, *X;
  double2* lam_tmp;
  unsigned short* scheme;
};
BlkGradWs blk_grad_ws(const qal_block_plan* p, int batch, int count, void* ws) {
  const size_t seq = (size_t)batch * count * 2 * p->packed;   // doubles per image sequence
  BlkGradWs w;
  w.U = reinterpret_cast<double*>(ws);
  w.P = w.U + seq;
  w.X = w.P + seq;
  w.lam_tmp = reinterpret_cast<double2*>(w.X + seq);
  w.scheme = reinterpret_cast<unsigned short*>(w.lam_tmp + (size_t)batch * p->packed);
  return w;
}
// forward of the gradient path, two layouts with the same results (U_k images, prefix P_k images, (m, s)
// codes, Lambda):
//  * fused (large batches): one CTA slot per pulse folds its slices in order -- expm + prefix product per
//    slice in one kernel; 19.4 KB of images written per slice.
//  * split (small batches, e.g. the 512 pulses per GPU of configs[2] at G = 8, where one chain per pulse
//    leaves the fused kernel latency-bound in a single wave): the persistent expm kernel exponentiates every
//    slice independently (full occupancy), then the prefix chain folds the stored U_k -- concurrently with
//    the suffix chain when its seed is known (the fidelity gradient).  Costs one more read of the U_k
//    images per chain (the chains run at ~85% of the HBM bandwidth).
#ifndef QAL_BLK_SPLIT_BELOW
#define QAL_BLK_SPLIT_BELOW 8   // split forward below this many pulses per SM
#endif
bool blk_split_forward(int batch) { return batch < QAL_BLK_SPLIT_BELOW * num_sms(); }
int blk_forward_impl(const qal_block_plan* p, int batch, const BlkCommon& c, double2* Lam, int* status, void* ws,
                     cudaStream_t st, bool with_suffix, const double2* V) {
  const BlkGradWs w = blk_grad_ws(p, batch, c.G.count, ws);
  double2* lam = Lam ? Lam : w.lam_tmp;
  if (!blk_split_forward(batch)) {
    BlkFwdOut O{w.U, lam, c.G.count, status, w.P, w.scheme};
    QAL_TRY(launch_blk_expm_fold(*p, batch, c.B, c.G, O, st));
    return with_suffix ? cuda_rc(launch_blk_suffix_chain(*p, batch, c.G.count, w.U, V, nullptr, w.X, st)) : QAL_OK;
  }
  BlkFwdOut O{w.U, nullptr, 1, status, nullptr, w.scheme};
  QAL_TRY(launch_blk_expm_fold(*p, batch, c.B, c.G, O, st));
  return cuda_rc(launch_blk_chains(*p, batch, c.G.count, w.U, w.P, lam, V, nullptr, with_suffix ? w.X : nullptr, st));
}
// reverse pass on a stored forward: suffix chain (X_{k+1}, seeded by S_V^dag or Cseed) -> gradient slices
int blk_backward_impl(const qal_block_plan* p, int batch, const BlkCommon& c, const double2* V, double* grad,
                      int* status, void* ws, cudaStream_t st, const double2* Cseed, bool suffix_done) {
  const BlkGradWs w = blk_grad_ws(p, batch, c.G.count, ws);
  if (!suffix_done) QAL_TRY(launch_blk_suffix_chain(*p, batch, c.G.count, w.U, V, Cseed, w.X, st));
  QAL_TRY(launch_blk_grad_slices(*p, batch, c.B, c.G, w.P, w.X, grad, status, w.scheme, Cseed ? 1.0 : 1.0 / 64.0, st));
  return QAL_OK;
}
// forward -> fidelity -> suffix chain -> gradient slices
int blk_fidelity_grad_impl(const qal_block_plan* p, int batch, const BlkCommon& c, const double2* V, double* F,
                           double* grad, double2* Lam, int* status, void* ws, cudaStream_t st,
                           const double2* Cseed) {
  const BlkGradWs w = blk_grad_ws(p, batch, c.G.count, ws);
  double2* lam = Lam ? Lam : w.lam_tmp;
  const bool fid = Cseed == nullptr;   // the seed S_V^dag is known up front: suffix chain beside the prefix
  int rc = blk_forward_impl(p, batch, c, lam, status, ws, st, fid, V);
  if (rc != QAL_OK) return rc;
  if (F) QAL_TRY(launch_blk_fidelity(*p, batch, lam, V, F, st));
  return blk_backward_impl(p, batch, c, V, grad, status, ws, st, Cseed, fid);
}
}  // namespace
