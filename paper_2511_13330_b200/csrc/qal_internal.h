// qal_internal.h -- launcher interface between qal_api.cu and the kernel TUs.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/qal.h"

namespace qal {

constexpr int MAXJ = 8;
constexpr size_t MAT_BYTES = 64 * 64 * 16;   // one 64x64 complex128 matrix / image
constexpr size_t PLANE_C = 64 * 64;          // complex elements per matrix

// Generator basis of the Magnus slice (a3): Omega_k = sum_m alpha_m(k) B_m with
// B = {L0_b, L_1..L_J, [L0_b, L_j] (J), [L_a, L_c] (a<c)}.
struct Basis {
  const double2* L0;
  long long L0_stride;      // complex elements between pulses (0 = shared)
  const double2* Lc;        // [J][64][64]
  const double2* Lcomm;     // [.][ncomm][64][64] or nullptr
  long long Lcomm_stride;   // complex elements between pulses (0 = shared)
  int J;
  int ncomm;                // 0 when the commutator basis is not used
};

struct SliceGrid {
  double h;                 // T / n_slices
  double c4;                // sqrt(3) h^2 / 12 for order 4, 0 for order 2
  int mode;                 // QAL_CTRL_PWC / QAL_CTRL_NODES
  const double* u;          // [batch][count][nodes][J]
  int count;                // slices per pulse in this call
};

struct FwdOut {
  double2* U_nat;           // [batch][count] natural, or nullptr
  double* U_img;            // [batch][count] images (internal), or nullptr
  double2* chunk_nat;       // [batch][count/chunk] natural, or nullptr
  int chunk;
  int* status;              // [batch] or nullptr
};

// coherence-block path (qal_blocks.cu): packed generator basis and forward outputs
struct BlkBasis {
  const double2* L0;       // packed [batch|1][packed]
  long long L0_stride;     // complex elements between pulses (0 = shared)
  const double2* Lc;       // packed [J][packed]
  const double2* Lcomm;    // packed [batch|1][ncomm][packed] or nullptr
  long long Lcomm_stride;
  int J, ncomm, packed;
};
struct BlkFwdOut {
  double* U_img;       // [batch][count] packed images, or nullptr
  double2* chunk_nat;  // [batch][count/chunk] packed natural, or nullptr
  int chunk;
  int* status;
  double* P_img;       // gradient path (chunk == count): prefix images P_k = U_{k-1}..U_0, or nullptr
  unsigned short* scheme = nullptr;   // gradient path: (m, s) code per [batch][count][group], or nullptr
};
int build_block_plan(int n, int nmat, const double2* mats, int mirror, qal_block_plan* out);
cudaError_t launch_blk_expm_fold(const qal_block_plan& p, int batch, const BlkBasis& B, const SliceGrid& G,
                                 const BlkFwdOut& O, cudaStream_t st);
cudaError_t launch_blk_tree_level(const qal_block_plan& p, int batch, int cnt, const double2* in, double2* out,
                                  cudaStream_t st);
cudaError_t launch_blk_pack(const qal_block_plan& p, int count, const double2* nat, double2* packed, int* flag,
                            cudaStream_t st);
cudaError_t launch_blk_check_status(const qal_block_plan& p, int count, const double2* nat, int broadcast, int* status,
                                   int nstatus, cudaStream_t st);
cudaError_t launch_blk_unpack(const qal_block_plan& p, int count, const double2* packed, double2* nat,
                              cudaStream_t st);
cudaError_t launch_blk_suffix_chain(const qal_block_plan& p, int batch, int N, const double* U_img,
                                    const double2* V, const double2* Cseed, double* X_img, cudaStream_t st);
cudaError_t launch_blk_chains(const qal_block_plan& p, int batch, int N, const double* U_img, double* P_img,
                              double2* lam, const double2* V, const double2* Cseed, double* X_img, cudaStream_t st);
cudaError_t launch_blk_grad_slices(const qal_block_plan& p, int batch, const BlkBasis& B, const SliceGrid& G,
                                   const double* P_img, const double* X_img, double* grad, int* status,
                                   const unsigned short* scheme, double gscale, cudaStream_t st);
cudaError_t launch_blk_scan(const qal_block_plan& p, int batch, int cnt, const double2* U, double2* pre, double2* suf,
                            double2* ws, cudaStream_t st);
cudaError_t launch_blk_batched_mm(const qal_block_plan& p, int count, const double2* A, long long sa,
                                  const double2* B, long long sb, double2* Cout, cudaStream_t st);
cudaError_t launch_blk_fidelity_cotangent(const qal_block_plan& p, const double2* V, double2* Cout, cudaStream_t st);
size_t blk_grad_scratch_bytes(const qal_block_plan& p, int batch, int n_slices);
cudaError_t launch_blk_fidelity(const qal_block_plan& p, int batch, const double2* Lam, const double2* V, double* F,
                                cudaStream_t st);

// coherence blocks on the n = 4096 path (qal_bigblocks.cu)
size_t bb_plan_ws_bytes();
int build_bigblock_plan(int nmat, const double2* mats, int mirror, qal_bigblock_plan* out, void* ws, cudaStream_t st);
size_t bb_ws_bytes(const qal_bigblock_plan& p);
cudaError_t launch_bb_expm_fold(const qal_bigblock_plan& p, const double2* L0, const double2* Lc, int J,
                                const double* u, int count, double h, int chunk, double2* chunk_nat, int* status,
                                int* flag, double* ws, cudaStream_t st);

int num_sms();
int& launch_counter();
// per-(device, kernel) dynamic shared-memory opt-in (qal_api.cu)
cudaError_t ensure_smem(const void* fn, size_t bytes);

// profiling window (qal_profile_begin/end): stage ids as in qal.h
enum { ST_LIOUV = 0, ST_COMM, ST_EXPM, ST_TREE, ST_FID, ST_PREFIX, ST_SUFFIX, ST_GRAD, ST_DENSE_GEMM,
       ST_BLK_EXPM, ST_BLK_TREE, ST_BLK_PREFIX, ST_BLK_SUFFIX, ST_BLK_GRAD, ST_BLK_GEMM, ST_BLK_FOLD, NSTAGE };
unsigned long long* prof_counter(int stage);   // device counter slot or nullptr
void prof_pre(int stage, cudaStream_t st);      // record start event (no-op when off)
void prof_post(int stage, cudaStream_t st);     // record end event

cudaError_t launch_expm_fold(int batch, const Basis& B, const SliceGrid& G, const FwdOut& O, cudaStream_t st);
cudaError_t launch_tree_level(int batch, int cnt, const double2* in, double2* out, cudaStream_t st);
cudaError_t launch_fidelity(int batch, const double2* Lam, const double2* V, double* F, cudaStream_t st);
cudaError_t launch_liouvillian(int batch, const double2* H0, int J, const double2* Hc, int ncops,
                               const double2* C, double2* L0, double2* Lc, cudaStream_t st);
cudaError_t launch_commutators(int batch, int J, const double2* L0, const double2* Lc, double2* Lcomm,
                               cudaStream_t st);
// prefix P_{k+1} = U_k P_k (P_0 = I) and suffix X_k = X_{k+1} U_k (X_N = S_V^dag) over
// per-pulse image sequences; see qal_grad.cu
cudaError_t launch_prefix_chain(int batch, int N, const double* U_img, double* P_img, double2* Lam_nat,
                                const double2* P_init, cudaStream_t st);
cudaError_t launch_suffix_chain(int batch, int N, const double* U_img, const double2* V, const double2* Cseed,
                                double* X_img, cudaStream_t st);
cudaError_t launch_grad_slices(int batch, const Basis& B, const SliceGrid& G, const double* P_img,
                               const double* X_img, double* grad, int* status, double* scratch, double gscale,
                               cudaStream_t st);
cudaError_t launch_scan(int batch, int cnt, const double2* U, double2* pre, double2* suf, double2* ws,
                        cudaStream_t st);
cudaError_t launch_batched_mm(int count, const double2* A, long long sa, const double2* B, long long sb, double2* C,
                              cudaStream_t st);
cudaError_t launch_fidelity_cotangent(const double2* V, double2* C, cudaStream_t st);
// Eqs. 16-17 logical loss + cotangent, and Adam (qal_product.cu)
cudaError_t launch_logical_loss(int batch, const double2* Lam, const double2* Pproj, const double2* Gt, double* loss,
                                double2* C, cudaStream_t st);
cudaError_t launch_adam(int n, double* theta, const double* g, double* m, double* v, int t, double lr, double b1,
                        double b2, double eps, cudaStream_t st);
size_t grad_scratch_bytes();
cudaError_t launch_sample_sines(int J, int nterm, const double* prm, double umax, double h, int k0, int count,
                               double* out, cudaStream_t st);
// n = 4096 (d = 64) dense path, qal_dense.cu
size_t dense_expm_ws_bytes();
cudaError_t launch_dense_expm_fold(const double2* L0, const double2* Lc, int J, const double* u, int count,
                                   double h, int chunk, double2* chunk_nat, double2* U_nat, int* status,
                                   double* ws, unsigned long long* nprod_host, cudaStream_t st);
cudaError_t launch_dense_tree_pair(const double2* Alater, const double2* Bearlier, double2* out, double* ws,
                                   cudaStream_t st);
cudaError_t launch_dense_liouvillian(int batch, const double2* H0, int J, const double2* Hc, int ncops,
                                     const double2* C, double2* L0, double2* Lc, cudaStream_t st);
cudaError_t launch_dense_fidelity(int batch, const double2* Lam, const double2* V, double* F, double* part,
                                  cudaStream_t st);
constexpr size_t DENSE_FID_PART_BYTES = 512 * sizeof(double);   // per pulse (n = 4096 slab partials)
cudaError_t launch_fp64_probe(int kind, int blocks, int iters, double* sink, cudaStream_t st);

}  // namespace qal
