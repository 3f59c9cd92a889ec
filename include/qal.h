/*
 * qal.h -- C ABI of libqal.so, the B200 (sm_100a) hot path of the Qalibrate
 * method (arxiv 2511.13330): time-sliced Magnus superoperator propagator of the
 * Lindblad equation, gate fidelity and its gradient.
 *
 * Citation keys: "P:n" = PAPER.md line n (section / equation named beside it);
 * "A#" = a reading listed in DESIGN.md "Readings of the paper".
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Matrices are ROW-MAJOR; complex numbers are interleaved {re, im} doubles
 *    (== torch.complex128 == cuDoubleComplex).  vec(rho) is column stacking,
 *    vec(rho)[i + d*j] = rho[i][j] (A5; the convention under which Eq. 8, P:107,
 *    holds).
 *  - Every array pointer is a DEVICE pointer owned by the caller.  The library
 *    never allocates, frees or retains device memory in these calls (except
 *    the per-process function attribute setup done once per device).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All work is enqueued on it; no call synchronises the host.
 *  - Arguments are validated synchronously BEFORE any launch; a call that
 *    returns an error code has enqueued nothing and written nothing.
 *  - Numeric failures that can only be seen on the device (a non-finite slice
 *    generator) are reported per pulse in the optional `status` array
 *    (device int[batch]; 0 = ok, QAL_ERR_NONFINITE otherwise).  `status` is
 *    overwritten, not accumulated.
 *  - Determinism: identical inputs and shapes give bit-identical outputs; no
 *    reduction uses atomics and every tree has a fixed shape keyed to the
 *    slice count and chunk size only (A16).
 *  - Supported sizes: d = 8 (superoperator n = d*d = 64, the three-spin
 *    exchange-only qubit of P:59) on every entry point, and d = 64 (n = 4096, two
 *    exchange-only qubits = six spins, BASELINE configs[4]) on the forward path:
 *    build_liouvillian (want_comm = 0), magnus_expm_slices (PWC controls; degree-16
 *    Taylor with device-chosen s <= 8), ordered_product, fidelity and fidelity_grad
 *    with grad == NULL.  Other sizes return QAL_ERR_UNSUPPORTED.
 *    Controls: 1 <= n_ctrl <= QAL_MAX_CTRL.
 */
#ifndef QAL_H
#define QAL_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } qal_c128;

enum {
    QAL_OK = 0,
    QAL_ERR_NULL = -1,        /* a required pointer is NULL                          */
    QAL_ERR_DIM = -2,         /* inconsistent sizes (chunk does not divide count ...) */
    QAL_ERR_EMPTY = -3,       /* batch, slice count or product length is zero        */
    QAL_ERR_NONFINITE = -4,   /* non-finite scalar argument, or device status flag   */
    QAL_ERR_UNSUPPORTED = -5, /* d / n / n_ctrl / mode outside what is implemented   */
    QAL_ERR_WORKSPACE = -6,   /* ws NULL or ws_bytes < qal_workspace_bytes(...)       */
    QAL_ERR_CUDA = -7,        /* a CUDA launch failed (cudaGetLastError)              */
    QAL_ERR_STRUCTURE = -8    /* block path: an operator couples two blocks of the plan */
};

enum {
    QAL_CTRL_PWC = 0,   /* u[batch][count][J]: value held on the whole slice        */
    QAL_CTRL_NODES = 1  /* u[batch][count][2][J]: values at the two Gauss-Legendre nodes   */
                        /* tau_{k,1,2} = t_k + (1/2 -+ sqrt(3)/6) h of slice k (A1, A2)     */
};

enum {                   /* op codes for qal_workspace_bytes */
    QAL_OP_ORDERED_PRODUCT = 1,
    QAL_OP_FIDELITY = 2,      /* qal_fidelity_grad with grad == NULL */
    QAL_OP_FIDELITY_GRAD = 3, /* qal_fidelity_grad with grad != NULL */
    QAL_OP_EXPM_SLICES = 4,   /* qal_magnus_expm_slices (non-zero only for n = 4096) */
    QAL_OP_VJP = 5,           /* qal_propagator_forward + qal_propagator_vjp (n_slices = count) */
    QAL_OP_FIDELITY_REDUCE = 6 /* qal_fidelity_ws (n = 4096: 512 partial sums per pulse; n = 64: 0) */
};

#define QAL_MAX_CTRL 8
#define QAL_ABI_VERSION 2

int qal_abi_version(void);

/*
 * Real FP64 matrix multiplications the library spends per complex matrix product:
 * 3 (Gauss / "3M": P = Ar Br, Q = Ai Bi, R = (Ar+Ai)(Br+Bi); Re = P - Q, Im = R - P - Q)
 * when built with -DQAL_USE_3M, else 4 (the default).  Algorithmic flop accounting counts
 * 2 n^3 per real multiplication, i.e. 6 n^3 per complex product for the 3M form.
 */
int qal_real_mults_per_complex_product(void);
const char *qal_status_string(int code);
/* the CUDA runtime's message for the error behind this host thread's last QAL_ERR_CUDA */
const char *qal_last_cuda_error(void);

/*
 * Eq. 8 from Eq. 6: the Liouvillian superoperator is linear
 * in H, so L(t) = L0 + sum_j u_j(t) L_j with
 *   L0 = -i (I (x) H0 - H0^T (x) I) + sum_c [ conj(c) (x) c - 1/2 I (x) c^dag c
 *                                              - 1/2 (c^dag c)^T (x) I ]
 *   L_j = -i (I (x) H_j - H_j^T (x) I)
 * where the collapse operators c carry sqrt(rate) (A6: sigma-_i / sqrt(T1),
 * sigma_z_i sqrt(1/(2 T2))).
 *   d        Hilbert dimension (8).  n = d*d.
 *   batch    number of drift Hamiltonians H0 (per-pulse Zeeman offsets), >= 1.
 *   H0       [batch][d][d]   Hc [n_ctrl][d][d]   C [n_cops][d][d] (n_cops >= 0; C may be
 *            NULL iff n_cops == 0).
 *   want_comm  if nonzero also write the bilinear commutator basis of the
 *            4th-order Magnus generator (A2):
 *            Lcomm[b][j]            = [L0_b, L_j]          j = 0..J-1
 *            Lcomm[b][J + p(a,c)]   = [L_a, L_c]           a < c, lexicographic pairs
 *            i.e. n_comm = J + J(J-1)/2 matrices per batch entry.
 *   Outputs L0 [batch][n][n], Lc [n_ctrl][n][n], Lcomm [batch][n_comm][n][n] (or NULL
 *   when want_comm == 0).
 */
int qal_build_liouvillian(int d, int batch, const qal_c128 *H0, int n_ctrl, const qal_c128 *Hc,
                          int n_cops, const qal_c128 *C, int want_comm, qal_c128 *L0, qal_c128 *Lc,
                          qal_c128 *Lcomm, void *stream);

/*
 * Eqs. 13-15, generalised to the 4th-order Magnus method (A1, A2):
 * for every slice k of the uniform grid t_k = k h, h = T / n_slices,
 *   A_a   = L0 + sum_j u_j(tau_{k,a}) L_j                                   (a = 1, 2)
 *   Omega = (h/2)(A_1 + A_2) - (sqrt(3) h^2 / 12) [A_1, A_2]               (order 4)
 *   Omega = (h/2)(A_1 + A_2)                                               (order 2)
 *   U_k   = expm(Omega)     (Eq. 14; scaling and squaring around a Taylor
 *                            polynomial whose truncation bound is <= 2^-53, A15)
 * and the left fold of every `chunk` consecutive slices (Eq. 15, later slice on
 * the LEFT, A4): chunk_prod[b][c] = U_{k0+(c+1)chunk-1} ... U_{k0+c chunk}.
 *   n            64.
 *   n_slices, T  define the grid (h = T / n_slices).  The call processes the
 *                `count` slices k0 .. k0+count-1 (0 <= k0, k0+count <= n_slices);
 *                u points at the row of slice k0.
 *   magnus_order 2 or 4.  ctrl_mode QAL_CTRL_PWC or QAL_CTRL_NODES.
 *   u            PWC: [batch][count][J]; NODES: [batch][count][2][J] (f64).
 *   L0           [batch or 1][n][n]; L0_batch_stride = n*n or 0 (shared).
 *   Lc           [J][n][n].
 *   Lcomm        as written by qal_build_liouvillian; required iff
 *                (ctrl_mode == NODES && magnus_order == 4), else ignored;
 *                Lcomm_batch_stride = n_comm*n*n or 0.
 *   U_out        optional [batch][count][n][n]: every U_k.
 *   chunk        >= 1, must divide count.  chunk_prod optional
 *                [batch][count/chunk][n][n].  At least one of U_out / chunk_prod.
 *   status       optional device int[batch].
 *   ws, ws_bytes n = 64: unused (NULL, 0).  n = 4096: >= qal_workspace_bytes(QAL_OP_EXPM_SLICES,
 *                4096, ...) bytes (eight tiled 4096^2 matrices, ~2.1 GB); pulses run one after
 *                the other, each product filling the GPU.
 */
int qal_magnus_expm_slices(int n, int batch, int n_slices, double T, int k0, int count,
                           int magnus_order, int ctrl_mode, int n_ctrl, const double *u,
                           const qal_c128 *L0, long long L0_batch_stride, const qal_c128 *Lc,
                           const qal_c128 *Lcomm, long long Lcomm_batch_stride, qal_c128 *U_out,
                           int chunk, qal_c128 *chunk_prod, int *status, void *ws, size_t ws_bytes,
                           void *stream);

/*
 * Eq. 15 with the tree reduction of P:141: out[b] = U[b][count-1] ... U[b][0]
 * (later factor on the LEFT, A4), evaluated as a balanced binary tree whose shape
 * depends on `count` only (pairs (2i, 2i+1) -> U[2i+1] U[2i] per level; an odd
 * last element is carried up unchanged).
 *   U    [batch][count][n][n], time order.  out [batch][n][n].  count >= 1.
 *   ws   >= qal_workspace_bytes(QAL_OP_ORDERED_PRODUCT, n, batch, count, 0, 0) bytes of
 *        device memory (may be NULL when that is 0, i.e. count <= 2).
 */
int qal_ordered_product(int n, int batch, int count, const qal_c128 *U, qal_c128 *out, void *ws,
                        size_t ws_bytes, void *stream);

/*
 * Log-depth scans of Eq. 15 (P:137-141 tree reduction generalised to all prefixes / suffixes;
 * Hillis-Steele levels, later factor on the LEFT), for single long pulses whose sequential
 * chains would leave the GPU idle:
 *   prefix_excl[b][s] = U[b][s-1] ... U[b][0]          (identity at s = 0)
 *   suffix_excl[b][s] = U[b][count-1] ... U[b][s+1]    (identity at s = count-1)
 * Either output may be NULL.  U [batch][count][n][n]; ws >= 4 * batch * count * n * n * 16 bytes.
 */
int qal_ordered_scan(int n, int batch, int count, const qal_c128 *U, qal_c128 *prefix_excl,
                     qal_c128 *suffix_excl, void *ws, size_t ws_bytes, void *stream);

/* C[i] = A[i] B[i], i < count, with element strides strideA / strideB = n*n or 0 (broadcast). */
int qal_batched_matmul(int n, int count, const qal_c128 *A, long long strideA, const qal_c128 *B,
                       long long strideB, qal_c128 *C, void *stream);

/*
 * Gate (process) fidelity to a target unitary V (A8, replaces Eqs. 16-17 on
 * this path):
 *   F[b] = Re Tr(S_V^dag Lambda[b]) / d^2,  S_V = conj(V) (x) V
 * (the superoperator of rho -> V rho V^dag under column stacking).  S_V is never
 * formed: S_V[i+dj, k+dl] = conj(V[j][l]) V[i][k].  Fixed-order reduction.
 *   Lambda [batch][n][n], V [d][d], F [batch] (f64).
 * d = 64: one CTA per pulse reads the 268 MB matrix (no workspace; use qal_fidelity_ws for the
 * bandwidth-bound form).  The library holds no device state, so calls on any streams are independent.
 */
int qal_fidelity(int d, int batch, const qal_c128 *Lambda, const qal_c128 *V, double *F,
                 void *stream);

/* qal_fidelity with a caller workspace: d = 64 reduces each pulse over 512 row slabs (512 CTAs per
 * pulse, HBM bound) into ws, then sums the 512 partials in a fixed order.
 * ws >= qal_workspace_bytes(QAL_OP_FIDELITY_REDUCE, n, batch, 1, 0, 0) (0 for d = 8). */
int qal_fidelity_ws(int d, int batch, const qal_c128 *Lambda, const qal_c128 *V, double *F, void *ws,
                    size_t ws_bytes, void *stream);

/*
 * Control table of configs[3] (a1, NODES mode; A11): the smooth random controls
 *   s_j(t) = sum_m a_{jm} sin(2 pi f_{jm} t + phi_{jm}) / sqrt(sum_m a_{jm}^2 / 2)
 *   u_j(t) = clip(u_max/2 (1 + s_j(t)/2), 0, u_max)
 * sampled at the two Gauss-Legendre nodes tau_{k,1,2} = t_k + (1/2 -+ sqrt(3)/6) h of the
 * slices k0 .. k0+count-1 of the grid t_k = k h, h = T / n_slices.
 *   prm    device [n_ctrl][nterm][3] = (a, f [GHz], phi).   u_out device [count][2][n_ctrl].
 */
int qal_sample_controls_sines(int n_ctrl, int nterm, const double *prm, double u_max, int n_slices,
                              double T, int k0, int count, double *u_out, void *stream);

/*
 * The whole hot path for a batch of pulses: propagator (as above, full grid,
 * k0 = 0, count = n_slices), fidelity and, if grad != NULL, the gradient of F
 * with respect to every control value (A14; P:185 motivates the adjoint form):
 *   dF/du_{k,j} = Re Tr(G_k dU_k/du_{k,j}) / d^2,
 *   G_k = P_k S_V^dag U_{N-1} ... U_{k+1},  P_k = U_{k-1} ... U_0,
 * evaluated with ONE adjoint Frechet derivative per slice,
 *   W_k = L_exp(Omega_k, G_k)    (so that Re Tr(G_k L(Omega_k, E)) = Re Tr(W_k E)),
 * and dF/du_{k,j} = Re Tr(W_k dOmega_k/du_{k,j}) / d^2.  grad has the layout of u.
 *   F       [batch] out.  grad [batch][...] out or NULL.  Lambda optional out
 *           [batch][n][n].
 *   ws      >= qal_workspace_bytes(grad ? QAL_OP_FIDELITY_GRAD : QAL_OP_FIDELITY, n, batch,
 *           n_slices, n_ctrl, ctrl_mode) bytes.
 * Other arguments as for qal_magnus_expm_slices.
 */
int qal_fidelity_grad(int d, int batch, int n_slices, double T, int magnus_order, int ctrl_mode,
                      int n_ctrl, const double *u, const qal_c128 *L0, long long L0_batch_stride,
                      const qal_c128 *Lc, const qal_c128 *Lcomm, long long Lcomm_batch_stride,
                      const qal_c128 *V, double *F, double *grad, qal_c128 *Lambda, int *status,
                      void *ws, size_t ws_bytes, void *stream);

/*
 * The gradient path split in two, for objectives other than the fidelity and for time-sharded
 * horizons (the reverse-mode counterpart of Eq. 15; P:185 motivates avoiding autodiff).
 *
 * qal_propagator_forward: for slices k0 .. k0+count-1 of the grid (as qal_magnus_expm_slices),
 *   Lambda[b] = U_{k0+count-1} ... U_{k0} P_init[b]   (P_init NULL = identity),
 *   and stores every U_k and every prefix P_k = U_{k-1} ... U_{k0} P_init in `ws` for a following
 *   qal_propagator_vjp with the same arguments and the same ws.
 * qal_propagator_vjp: for any scalar objective with dL = Re Tr(C[b] dLambda[b]) (C = the cotangent,
 *   device [batch][n][n]), writes grad[b] = dL/du (layout of u) with one adjoint Frechet
 *   derivative per slice (as qal_fidelity_grad, which is the special case C = S_V^dag / d^2).
 * ws: >= qal_workspace_bytes(QAL_OP_VJP, n, batch, count, n_ctrl, ctrl_mode).
 */
int qal_propagator_forward(int d, int batch, int n_slices, double T, int k0, int count, int magnus_order,
                           int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0,
                           long long L0_batch_stride, const qal_c128 *Lc, const qal_c128 *Lcomm,
                           long long Lcomm_batch_stride, const qal_c128 *P_init, qal_c128 *Lambda,
                           int *status, void *ws, size_t ws_bytes, void *stream);
int qal_propagator_vjp(int d, int batch, int n_slices, double T, int k0, int count, int magnus_order,
                       int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0,
                       long long L0_batch_stride, const qal_c128 *Lc, const qal_c128 *Lcomm,
                       long long Lcomm_batch_stride, const qal_c128 *C, double *grad, int *status,
                       void *ws, size_t ws_bytes, void *stream);

/* Cotangent of the fidelity (A8): C = S_V^dag / d^2 (device [n][n]), so that dF = Re Tr(C dLambda).
 * Used to seed qal_propagator_vjp on time-sharded horizons. */
int qal_fidelity_cotangent(int d, const qal_c128 *V, qal_c128 *C, void *stream);

/*
 * Eqs. 16-17: the paper's calibration objective.  P = [vec(rho_0) vec(rho_1)] (device
 * [n][2], rho_k = |phi_k><phi_k| of the logical states of Eqs. 2-3), target G (device [2][2]):
 *   Pi = P^dag Lambda P,   loss[b] = 1/4 ||Pi - G||_F^2   (the Frobenius norm of Eq. 17 with A^dag A,
 *   DESIGN.md A22), and, if C != NULL, the cotangent C[b] = 1/2 P (Pi - G)^dag P^dag (so that
 *   d loss = Re Tr(C dLambda), the input of qal_propagator_vjp).
 */
int qal_logical_loss(int d, int batch, const qal_c128 *Lambda, const qal_c128 *Pproj, const qal_c128 *G,
                     double *loss, qal_c128 *C, void *stream);

/* Adam (ref [13]) on device arrays of n doubles, step t >= 1 (bias correction):
 *   m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;  theta <- theta - lr (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps) */
int qal_adam_step(int n, double *theta, const double *grad, double *m, double *v, int t, double lr,
                  double beta1, double beta2, double eps, void *stream);

/* Device workspace (bytes) an op needs; 0 when none.  `flags` = ctrl_mode for the
 * fidelity ops, 0 otherwise. */
size_t qal_workspace_bytes(int op, int n, int batch, int n_slices, int n_ctrl, int flags);

/* Chunk size qal_fidelity_grad uses for the forward fold of a fidelity-only call
 * (a function of n_slices and batch only; exported so callers can reproduce it). */
int qal_default_chunk(int batch, int n_slices);

/*
 * FP64 roofline probe (bench only): kind 0 = DMMA.8x8x4 loop, kind 1 = DFMA
 * loop; `blocks` CTAs of 256 threads, `iters` inner iterations.  Returns the FP64
 * flop count one launch performs in *flops (host pointer).  `sink` is a device
 * double that is written only to defeat dead-code elimination.
 */
int qal_fp64_peak_probe(int kind, int blocks, int iters, double *flops, double *sink, void *stream);

/* ===================================================================================
 * Coherence-block path (pin P-13).  Every operator of the problem
 * conserves total S_z (Eq. 6), so the superoperators of Eq. 8 and
 * everything built from them by Eqs. 13-15 are block diagonal by coherence
 * order q = m_a - m_b (d = 8: blocks 20/15/15/6/6/1/1).  Hermiticity preservation
 * (Lambda[s(R), s(C)] = conj(Lambda[R, C]), s(i + d j) = j + d i) pairs q with -q.
 * The path computes exactly the same Omega_k, U_k, Lambda, F and dF/du as the dense path,
 * restricted to the blocks (2.13% of the dense flops with the mirror and the real q = 0 block).
 *
 * A PACKED matrix is the concatenation of the plan's super-block matrices (groups g of
 * padded width width[g] = 8, 16 or 24; each row-major complex128, entries on padding
 * rows / columns are 0), `packed` complex elements in total.  Packed row row0[g] + r is
 * natural index perm[row0[g] + r] (-1 = padding).
 * =================================================================================== */
#define QAL_BLK_MAX_GROUPS 16
#define QAL_BLK_MAX_ROWS 96

typedef struct {
    int n;                              /* superoperator dimension (64)                       */
    int d;                              /* Hilbert dimension (8)                              */
    int mirror;                         /* 1: one block of every Hermitian-mirror pair stored */
    int ngroups;                        /* super-blocks                                       */
    int nrows;                          /* packed rows = sum of widths (<= QAL_BLK_MAX_ROWS)   */
    int packed;                         /* complex elements per packed matrix = sum width^2   */
    int n_components;                   /* connected components of the basis sparsity graph  */
    int width[QAL_BLK_MAX_GROUPS];      /* padded width of group g: 8, 16 or 24               */
    int used[QAL_BLK_MAX_GROUPS];       /* rows of group g that are not padding               */
    int row0[QAL_BLK_MAX_GROUPS];       /* first packed row of group g                        */
    int off[QAL_BLK_MAX_GROUPS];        /* complex offset of group g inside a packed matrix   */
    double flops[QAL_BLK_MAX_GROUPS];   /* algorithmic flops of one product of group g:
                                           2 cplx_mults sum s^3 over complex components, 2 sum
                                           s^3 over real ones (padding excluded)              */
    int perm[QAL_BLK_MAX_ROWS];         /* packed row -> natural index, -1 = padding          */
    int weight[QAL_BLK_MAX_ROWS];       /* 0 padding, 1 self-mirror component (or mirror
                                           off), 2 component whose mirror is implied         */
    int inv[64];                        /* natural index -> packed row, -1 = not stored       */
    int comp[64];                       /* natural index -> component id                      */
    /* Self-mirrored components (s(R) in the component for every R, e.g. coherence order 0) are
     * stored in the basis of vectorised Hermitian matrices, vec = T x with columns e_R (R = s(R))
     * and (e_R + e_sR)/sqrt2, i (e_R - e_sR)/sqrt2 (R < s(R)).  T is unitary and every
     * Hermiticity-preserving map is real there, so these groups run in real arithmetic
     * (1 real multiplication per product instead of 4).  Packed entries of a real group are
     * (M'[r][c], 0) with M' = T^dag M T.                                                    */
    int real[QAL_BLK_MAX_GROUPS];       /* 1: group g holds real-basis components              */
    int rtype[QAL_BLK_MAX_ROWS];        /* 0 complex row, 1 real diagonal e_R, 2 pair column a,
                                           3 pair column b (perm = the pair's smaller index)  */
    int ncode[64];                      /* natural index: 0 complex group, 1 real diagonal,
                                           2 pair representative R < s(R), 3 pair mirror      */
    int cplx_mults;                     /* real multiplications per complex block product the
                                           library executes (4, or 3 with the Gauss form)     */
    int launch_sets;                    /* launch layout of the forward, suffix-chain and
                                           gradient kernels (caller option, set after
                                           qal_block_plan_build; QAL_BLK_SETS_*): results are
                                           identical (gradient: up to the trace-sum order)     */
} qal_block_plan;

enum {
    QAL_BLK_SETS_DEFAULT = 0,  /* one launch per group, several items per CTA (role-compiled kernels) */
    QAL_BLK_SETS_FUSED = 1,    /* one launch, every group of one item per CTA                         */
    QAL_BLK_SETS_PAIRS = 2     /* one launch per group, two items per CTA                             */
};

/*
 * Structure detection (host only, no device work): the connected components of the union
 * sparsity pattern of `nmat` HOST matrices mats[nmat][n][n] (pass every generator the
 * calls will use: L0 of every pulse or a representative plus k_blk_check, L_j, commutators),
 * the Hermitian mirror pairing (QAL_ERR_STRUCTURE if it does not map components onto
 * components) and a first-fit-decreasing packing into super-blocks.  n must be 64;
 * components larger than 24 -> QAL_ERR_UNSUPPORTED.
 */
int qal_block_plan_build(int n, int nmat, const qal_c128 *mats, int mirror, qal_block_plan *plan);

/*
 * natural [count][n][n] (device) -> packed [count][plan->packed] (device).  If `flag` (device
 * int, caller-zeroed) is not NULL the call also verifies that every entry coupling two
 * different components is exactly zero and sets *flag = QAL_ERR_STRUCTURE otherwise.
 */
int qal_block_pack(const qal_block_plan *plan, int count, const qal_c128 *nat, qal_c128 *packed, int *flag,
                   void *stream);

/*
 * The device structure check of qal_block_pack reported per pulse, for a caller that runs it after the
 * block calls of a step (those reset `status` on entry): every entry of nat[e] ([count][n][n], device)
 * coupling two components of the plan must be exactly zero (A26; Eq. 8 conserves the coherence order
 * only if every operator of Eq. 6 conserves S_z).  A failing matrix e sets status[e] = QAL_ERR_STRUCTURE
 * (broadcast = 0: one matrix per pulse, nstatus == count, e.g. L0_b), or every status[0 .. nstatus)
 * (broadcast = 1: a basis matrix shared by all pulses, e.g. L_j).  Entries of passing matrices are left
 * as they are.  The F / gradient of a flagged pulse are not meaningful.
 */
int qal_block_check(const qal_block_plan *plan, int count, const qal_c128 *nat, int broadcast, int *status,
                    int nstatus, void *stream);

/* packed -> natural [count][n][n]; blocks of mirrored components are filled from their stored
 * partner by Lambda[s(R), s(C)] = conj(Lambda[R, C]); entries between components are 0. */
int qal_block_unpack(const qal_block_plan *plan, int count, const qal_c128 *packed, qal_c128 *nat, void *stream);

/*
 * qal_magnus_expm_slices on packed operands: L0p [batch|1][packed] (L0p_stride = packed or 0),
 * Lcp [J][packed], Lcommp [batch|1][ncomm][packed] (NODES + order 4 only; stride ncomm*packed
 * or 0).  Output chunk_prod [batch][count/chunk][packed] (required).  No workspace.
 * Other arguments and errors as qal_magnus_expm_slices.
 */
int qal_block_expm_slices(const qal_block_plan *plan, int batch, int n_slices, double T, int k0, int count,
                          int magnus_order, int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0p,
                          long long L0p_stride, const qal_c128 *Lcp, const qal_c128 *Lcommp,
                          long long Lcommp_stride, int chunk, qal_c128 *chunk_prod, int *status, void *stream);

/* qal_ordered_product on packed matrices: out[b] = U[b][count-1] ... U[b][0] (same tree shape).
 * ws >= qal_block_workspace_bytes(plan, QAL_OP_ORDERED_PRODUCT, batch, count). */
int qal_block_ordered_product(const qal_block_plan *plan, int batch, int count, const qal_c128 *U, qal_c128 *out,
                              void *ws, size_t ws_bytes, void *stream);

/* qal_fidelity on packed Lambda (mirrored components counted twice). */
int qal_block_fidelity(const qal_block_plan *plan, int batch, const qal_c128 *Lambda_packed, const qal_c128 *V,
                       double *F, void *stream);

/*
 * qal_fidelity_grad on packed operands (plan built with mirror = 1 or 0; the fidelity cotangent
 * S_V^dag is Hermiticity preserving, so the mirror is exact).  Lambda_packed optional out
 * [batch][packed].  ws >= qal_block_workspace_bytes(plan, grad ? QAL_OP_FIDELITY_GRAD :
 * QAL_OP_FIDELITY, batch, n_slices).
 */
int qal_block_fidelity_grad(const qal_block_plan *plan, int batch, int n_slices, double T, int magnus_order,
                            int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0p, long long L0p_stride,
                            const qal_c128 *Lcp, const qal_c128 *Lcommp, long long Lcommp_stride,
                            const qal_c128 *V, double *F, double *grad, qal_c128 *Lambda_packed, int *status,
                            void *ws, size_t ws_bytes, void *stream);

/*
 * The reverse pass of the block path for a general objective (qal_propagator_forward + _vjp on packed
 * operands): forward over slices k0 .. k0+count-1 (P_init = I), then
 * grad = dL/du for dL = Re Tr(C[b] dLambda[b]) with C packed [batch][packed] (pack it with
 * qal_block_pack, or build it with the block ops).  C must preserve Hermiticity (every cotangent of a
 * real objective of a Hermiticity-preserving Lambda does: S_V^dag, the Eq. 16-17 loss cotangent, the
 * time-sharded seeds), because the plan stores one block of each mirror pair and the q = 0 block in the
 * real basis.  Lambda_packed optional out.  ws >= qal_block_workspace_bytes(plan, QAL_OP_VJP, batch, count).
 */
int qal_block_propagator_vjp(const qal_block_plan *plan, int batch, int n_slices, double T, int k0, int count,
                             int magnus_order, int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0p,
                             long long L0p_stride, const qal_c128 *Lcp, const qal_c128 *Lcommp,
                             long long Lcommp_stride, const qal_c128 *Cp, double *grad, qal_c128 *Lambda_packed,
                             int *status, void *ws, size_t ws_bytes, void *stream);

/*
 * qal_block_propagator_vjp in two calls (the counterpart of qal_propagator_forward / _vjp): the forward
 * writes Lambda_packed [batch][packed] (required) and keeps every U_k, prefix P_k and the (m, s) choice of
 * every slice in `ws`; the backward then runs only the reverse pass (suffix chain seeded with Cp, one
 * adjoint Frechet derivative per slice) on that stored forward.  Both calls take the same arguments and
 * the same ws (>= qal_block_workspace_bytes(plan, QAL_OP_VJP, batch, count)); the cotangent may be
 * computed from Lambda in between (the time-sharded gradient of NEXT f2 does).  The forward resets
 * `status`, the backward only adds flags.
 */
int qal_block_propagator_forward(const qal_block_plan *plan, int batch, int n_slices, double T, int k0, int count,
                                 int magnus_order, int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0p,
                                 long long L0p_stride, const qal_c128 *Lcp, const qal_c128 *Lcommp,
                                 long long Lcommp_stride, qal_c128 *Lambda_packed, int *status, void *ws,
                                 size_t ws_bytes, void *stream);
int qal_block_propagator_backward(const qal_block_plan *plan, int batch, int n_slices, double T, int k0, int count,
                                  int magnus_order, int ctrl_mode, int n_ctrl, const double *u, const qal_c128 *L0p,
                                  long long L0p_stride, const qal_c128 *Lcp, const qal_c128 *Lcommp,
                                  long long Lcommp_stride, const qal_c128 *Cp, double *grad, int *status, void *ws,
                                  size_t ws_bytes, void *stream);

/* qal_ordered_scan on packed matrices (exclusive prefix / suffix products, Hillis-Steele levels).
 * ws >= 4 * batch * count * plan->packed * 16 bytes. */
int qal_block_ordered_scan(const qal_block_plan *plan, int batch, int count, const qal_c128 *U,
                           qal_c128 *prefix_excl, qal_c128 *suffix_excl, void *ws, size_t ws_bytes, void *stream);

/* qal_batched_matmul on packed matrices: C[i] = A[i] B[i], strides plan->packed or 0 (broadcast). */
int qal_block_batched_matmul(const qal_block_plan *plan, int count, const qal_c128 *A, long long strideA,
                             const qal_c128 *B, long long strideB, qal_c128 *C, void *stream);

/* qal_fidelity_cotangent in packed form: C = S_V^dag / d^2 on the stored blocks (A8). */
int qal_block_fidelity_cotangent(const qal_block_plan *plan, const qal_c128 *V, qal_c128 *C, void *stream);

size_t qal_block_workspace_bytes(const qal_block_plan *plan, int op, int batch, int n_slices);

/* ===================================================================================
 * Coherence blocks on the n = 4096 path (d = 64: configs[4] six spins, the 3-dot Hubbard model):
 * the same structure as above with blocks far wider than 24 (six spins: 924, 792, 495, 220, 66, 12, 1
 * with the mirror), each stored as a grid of 64 x 64 tile images and multiplied by a block-diagonal
 * tiled DMMA GEMM.  One pulse per call, PWC controls, like the dense n = 4096 path.
 * =================================================================================== */
#define QAL_BB_MAX_BLOCKS 48
#define QAL_BB_MAX_ROWS 8192

typedef struct {
    int n, d, mirror, nb, n_components;
    int size[QAL_BB_MAX_BLOCKS];        /* used rows of block b (components packed best-fit)  */
    int nt[QAL_BB_MAX_BLOCKS];          /* 64 x 64 tiles per dimension of block b             */
    int row0[QAL_BB_MAX_BLOCKS];        /* first packed row of block b (64-aligned)           */
    int weight[QAL_BB_MAX_BLOCKS];      /* reserved (1); mirrored blocks are filled at unpack */
    double flops[QAL_BB_MAX_BLOCKS];    /* algorithmic flops of one product of block b        */
    double flops_per_product;           /* sum over the blocks                                */
    int nrows, ntiles;                  /* packed rows (64 x sum nt), output tiles (sum nt^2) */
    long long total_doubles;            /* doubles of one tiled-block matrix                 */
    int perm[QAL_BB_MAX_ROWS];          /* packed row -> natural index, -1 = padding          */
    int inv[4096];                      /* natural index -> packed row, -1 = mirrored         */
    int comp[4096];                     /* natural index -> component                         */
    int real[QAL_BB_MAX_BLOCKS];        /* block b holds self-mirrored components in the real
                                           Hermitian basis (as qal_block_plan.real)           */
    int rtype[QAL_BB_MAX_ROWS];         /* as qal_block_plan.rtype                            */
    int ncode[4096];                    /* as qal_block_plan.ncode                            */
} qal_bigblock_plan;

/* Structure detection for n = 4096: the union non-zero pattern of the DEVICE matrices
 * mats[nmat][4096][4096] is computed on the device into the caller's workspace (a 2 MB bitmask,
 * ws_bytes >= qal_bigblock_plan_workspace_bytes()), its connected components and Hermitian mirror
 * pairing on the host (a setup call: synchronises `stream`).  The library allocates nothing.
 * QAL_ERR_UNSUPPORTED beyond 48 stored blocks. */
size_t qal_bigblock_plan_workspace_bytes(void);
int qal_bigblock_plan_build(int nmat, const qal_c128 *mats, int mirror, qal_bigblock_plan *plan, void *ws,
                            size_t ws_bytes, void *stream);

/*
 * Device workspace of qal_bigblock_expm_slices: six tiled-block matrices per slice of a batch (slices
 * are processed in batches of up to 64, as many as ~4 GB holds for the plan's tile count), the two
 * running chunk products, per-slice norm partials and plan records, and the index tables.
 */
size_t qal_bigblock_workspace_bytes(const qal_bigblock_plan *plan);

/*
 * qal_magnus_expm_slices for n = 4096 on the coherence blocks: slices 0 .. count-1 of one pulse
 * (PWC u [count][n_ctrl], L0 [4096][4096], Lc [n_ctrl][4096][4096], natural layout), chunk folds
 * written to chunk_prod [count/chunk][4096][4096] (natural, mirror-filled, zero between blocks).
 * If `flag` (device int, caller-zeroed) is given, every basis entry coupling two blocks is checked
 * (QAL_ERR_STRUCTURE).  ws >= qal_bigblock_workspace_bytes(plan).  Slices are exponentiated in
 * batches that never cross a chunk boundary; each batch's U_k are multiplied by a balanced tree (later
 * slice on the left, Eq. 15) and folded into the chunk product, so the rounding order
 * differs from a slice-by-slice fold (same product, within the BJ tolerance).
 */
int qal_bigblock_expm_slices(const qal_bigblock_plan *plan, int n_slices, double T, int count, int n_ctrl,
                             const double *u, const qal_c128 *L0, const qal_c128 *Lc, int chunk,
                             qal_c128 *chunk_prod, int *status, int *flag, void *ws, size_t ws_bytes,
                             void *stream);

/*
 * Stage profiling (bench.py's roofline and the expm-vs-product split, the Fig. 2
 * analog of P:167-171).  Between qal_profile_begin and qal_profile_end every kernel
 * the library enqueues is bracketed by CUDA events on its launch stream and, if
 * `dev_counters` (device unsigned long long[QAL_NSTAGE], zeroed by the caller) is
 * not NULL, each kernel adds the number of 64x64 complex matrix products it actually
 * executed (the (m, s) choice is per slice) to dev_counters[stage].
 * qal_profile_end synchronises the recorded events and writes, per stage, the summed
 * device milliseconds and the number of launches (host arrays of QAL_NSTAGE).
 * Not thread-safe; one profiling window per process at a time.
 */
enum { QAL_ST_LIOUV = 0, QAL_ST_COMM = 1, QAL_ST_EXPM = 2, QAL_ST_TREE = 3, QAL_ST_FID = 4,
       QAL_ST_PREFIX = 5, QAL_ST_SUFFIX = 6, QAL_ST_GRAD = 7, QAL_ST_DENSE_GEMM = 8,
       /* coherence-block path: these counters accumulate ALGORITHMIC FLOPs (8 s^3 per complex
        * product of an s x s block, padding excluded), not product counts */
       QAL_ST_BLK_EXPM = 9, QAL_ST_BLK_TREE = 10, QAL_ST_BLK_PREFIX = 11, QAL_ST_BLK_SUFFIX = 12,
       QAL_ST_BLK_GRAD = 13, QAL_ST_BLK_GEMM = 14,
       /* the fold products inside the fused block forward (k_blk_expm_fold): flops only, no
        * launches of their own (their time is inside QAL_ST_BLK_EXPM); QAL_ST_BLK_PREFIX counts
        * the separate prefix-chain kernel alone */
       QAL_ST_BLK_FOLD = 15, QAL_NSTAGE = 16 };
int qal_profile_begin(unsigned long long *dev_counters);
int qal_profile_end(double *ms, int *launches);

/* Number of kernels the last call on this host thread enqueued (launch accounting
 * for bench.py's gpu_launches); reset by every qal_* call that launches. */
int qal_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* QAL_H */
