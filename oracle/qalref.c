/*
 * qalref.c -- the ORACLE for the Qalibrate hot path (arxiv 2511.13330).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2511_13330_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or constant generator with the
 * CUDA path.
 *
 * Plain, slow, sequential complex128 C: literal Kronecker products, triple-loop
 * matrix products, a term-by-term Taylor series.  Each function cites the
 * PAPER.md line (P:n) and the DESIGN.md reading (A#) it follows.
 *
 * Layout: row-major; vec(rho) is column stacking, vec(rho)[i + d*j] = rho[i][j]
 * (A5; the only convention under which Eq. 8, holds).
 *
 * Parity status:
 *   build_liouvillian   pinned (Eq. 6 <-> Eq. 8 cross-check, P-3, P-6, P-13)
 *   lindblad_rhs        pinned (closed forms P-6 via RK4; Eq. 6 evaluated directly)
 *   expm                pinned (scipy.linalg.expm, closed forms P-11)
 *   magnus_generator    pinned (order-4 convergence vs independent ODE solver, P-7)
 *   propagate           pinned (P-1, P-2, P-3, P-4, P-5, P-12)
 *   fidelity            pinned (P-10)
 *   frechet / gradient  pinned (scipy.linalg.expm_frechet, central FD P-8)
 *   rk4                 pinned (analytic precession, order 4)
 *   vjp                 pinned (equals gradient for C = S_V^dag/d^2; central FD of Re Tr(C Lambda))
 *   logical_loss        pinned (Pi = I for Lambda = I, logical swap, FD of the loss vs cotangent)
 *   adam_step           pinned (closed forms: first step lr sign(g); constant gradient)
 *   sines_eval          pinned by the mathematics of A11 (the paper prints no values): one-term
 *                       extremes u_max/2 (1 +- 1/sqrt 2) and period, unit RMS, Cauchy-Schwarz
 *                       clipping, Gauss-Legendre nodes vs numpy leggauss (tests/test_oracle_pins.py)
 */
#include <complex.h>
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

#define QALREF_OK 0
#define QALREF_ERR_DIM (-2)
#define QALREF_ERR_ALLOC (-8)

/* ------------------------------------------------------------------ */
/* plain linear algebra                                                */
/* ------------------------------------------------------------------ */

/* C = A B (n x n), triple loop; C must not alias A or B.  Rows are independent, so
 * outside an enclosing parallel region they are split over OpenMP threads: every
 * C[i][j] is still one sequential sum over k, bit-identical to the single-thread loop. */
static void mm(int n, const cplx *A, const cplx *B, cplx *C)
{
    #pragma omp parallel for schedule(static) if (n >= 64 && !omp_in_parallel())
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            cplx s = 0;
            for (int k = 0; k < n; ++k)
                s += A[(size_t)i * n + k] * B[(size_t)k * n + j];
            C[(size_t)i * n + j] = s;
        }
}

/* K = P (x) Q with P: p x p, Q: q x q  ->  K[(a*q + c)][(b*q + e)] = P[a][b] Q[c][e] */
static void kron(int p, const cplx *P, int q, const cplx *Q, cplx *K)
{
    int n = p * q;
    for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b)
            for (int c = 0; c < q; ++c)
                for (int e = 0; e < q; ++e)
                    K[(size_t)(a * q + c) * n + (b * q + e)] = P[a * p + b] * Q[c * q + e];
}

static double norm1(int n, const cplx *A)   /* max column abs sum */
{
    double best = 0.0;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += cabs(A[(size_t)i * n + j]);
        if (s > best) best = s;
    }
    return best;
}

static void eye(int n, cplx *A)
{
    memset(A, 0, sizeof(cplx) * (size_t)n * n);
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] = 1.0;
}

/* ------------------------------------------------------------------ */
/* Eq. 8: the Liouvillian superoperator, literal Kronecker form      */
/*   L = -i (I (x) H - H^T (x) I)                                               */
/*       + sum_k [ conj(c_k) (x) c_k - 1/2 I (x) c_k^dag c_k - 1/2 (c_k^dag c_k)^T (x) I ] */
/* The L_k of Eq. 8 are the collapse operators c_k (A6: sqrt(rate) folded in).   */
/* With linearity of Eq. 8 in H: L(t) = L0 + sum_j u_j(t) L_j where L0 is built  */
/* from H0 and all c_k, and L_j from H_j alone (no dissipator).                  */
/* ------------------------------------------------------------------ */
static void liouv_hamiltonian_part(int d, const cplx *H, cplx *L, int accumulate)
{
    int n = d * d;
    cplx *Id = malloc(sizeof(cplx) * d * d);
    cplx *Ht = malloc(sizeof(cplx) * d * d);
    cplx *K1 = malloc(sizeof(cplx) * (size_t)n * n);
    cplx *K2 = malloc(sizeof(cplx) * (size_t)n * n);
    eye(d, Id);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) Ht[a * d + b] = H[b * d + a];
    kron(d, Id, d, H, K1);      /* I (x) H   */
    kron(d, Ht, d, Id, K2);     /* H^T (x) I */
    for (size_t e = 0; e < (size_t)n * n; ++e) {
        cplx term = -_Complex_I * (K1[e] - K2[e]);
        L[e] = accumulate ? L[e] + term : term;
    }
    free(Id); free(Ht); free(K1); free(K2);
}

static void liouv_dissipator_add(int d, const cplx *c, cplx *L)
{
    int n = d * d;
    cplx *Id = malloc(sizeof(cplx) * d * d);
    cplx *cc = malloc(sizeof(cplx) * d * d);     /* conj(c) */
    cplx *cd = malloc(sizeof(cplx) * d * d);     /* c^dag */
    cplx *cdc = malloc(sizeof(cplx) * d * d);    /* c^dag c */
    cplx *cdct = malloc(sizeof(cplx) * d * d);   /* (c^dag c)^T */
    cplx *K = malloc(sizeof(cplx) * (size_t)n * n);
    eye(d, Id);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            cc[a * d + b] = conj(c[a * d + b]);
            cd[a * d + b] = conj(c[b * d + a]);
        }
    mm(d, cd, c, cdc);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) cdct[a * d + b] = cdc[b * d + a];
    kron(d, cc, d, c, K);
    for (size_t e = 0; e < (size_t)n * n; ++e) L[e] += K[e];
    kron(d, Id, d, cdc, K);
    for (size_t e = 0; e < (size_t)n * n; ++e) L[e] -= 0.5 * K[e];
    kron(d, cdct, d, Id, K);
    for (size_t e = 0; e < (size_t)n * n; ++e) L[e] -= 0.5 * K[e];
    free(Id); free(cc); free(cd); free(cdc); free(cdct); free(K);
}

/* L0 [n][n] from H0 and the collapse ops; Lc [J][n][n] from the control Hamiltonians. */
int qalref_build_liouvillian(int d, const cplx *H0, int J, const cplx *Hc, int ncops,
                             const cplx *C, cplx *L0, cplx *Lc)
{
    if (d < 1 || J < 0 || ncops < 0) return QALREF_ERR_DIM;
    int n = d * d;
    liouv_hamiltonian_part(d, H0, L0, 0);
    for (int k = 0; k < ncops; ++k) liouv_dissipator_add(d, C + (size_t)k * d * d, L0);
    for (int j = 0; j < J; ++j) liouv_hamiltonian_part(d, Hc + (size_t)j * d * d, Lc + (size_t)j * n * n, 0);
    return QALREF_OK;
}

/* Eq. 6 evaluated directly in matrix form (hbar = 1, A18):
 *   drho/dt = -i [H, rho] + sum_k ( c_k rho c_k^dag - 1/2 {c_k^dag c_k, rho} )          */
int qalref_lindblad_rhs(int d, const cplx *H, int ncops, const cplx *C, const cplx *rho, cplx *out)
{
    cplx *t1 = malloc(sizeof(cplx) * d * d), *t2 = malloc(sizeof(cplx) * d * d);
    cplx *cd = malloc(sizeof(cplx) * d * d), *cdc = malloc(sizeof(cplx) * d * d);
    mm(d, H, rho, t1);
    mm(d, rho, H, t2);
    for (int e = 0; e < d * d; ++e) out[e] = -_Complex_I * (t1[e] - t2[e]);
    for (int k = 0; k < ncops; ++k) {
        const cplx *c = C + (size_t)k * d * d;
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) cd[a * d + b] = conj(c[b * d + a]);
        mm(d, c, rho, t1);
        mm(d, t1, cd, t2);                       /* c rho c^dag */
        for (int e = 0; e < d * d; ++e) out[e] += t2[e];
        mm(d, cd, c, cdc);
        mm(d, cdc, rho, t1);
        mm(d, rho, cdc, t2);
        for (int e = 0; e < d * d; ++e) out[e] -= 0.5 * (t1[e] + t2[e]);
    }
    free(t1); free(t2); free(cd); free(cdc);
    return QALREF_OK;
}

/* ------------------------------------------------------------------ */
/* Eq. 14: U = exp(Lbar).  Oracle step O4: scaling and squaring around a  */
/* term-by-term Taylor series (A3: "T exp" of one matrix is the plain exponential). */
/*   s = max(0, ceil(log2(||A||_1 / 0.5))), X = A / 2^s,                           */
/*   sum_i X^i / i! until ||term||_1 < 2^-60 ||sum||_1 (at most 40 terms),          */
/*   then square s times.                                                         */
/* ------------------------------------------------------------------ */
int qalref_expm(int n, const cplx *A, cplx *E)
{
    size_t nn = (size_t)n * n;
    cplx *X = malloc(sizeof(cplx) * nn), *term = malloc(sizeof(cplx) * nn), *tmp = malloc(sizeof(cplx) * nn);
    if (!X || !term || !tmp) { free(X); free(term); free(tmp); return QALREF_ERR_ALLOC; }
    double nrm = norm1(n, A);
    int s = 0;
    if (nrm > 0.5) s = (int)ceil(log2(nrm / 0.5));
    double scale = ldexp(1.0, -s);
    for (size_t e = 0; e < nn; ++e) X[e] = A[e] * scale;
    eye(n, E);
    eye(n, term);
    for (int i = 1; i <= 40; ++i) {
        mm(n, term, X, tmp);
        for (size_t e = 0; e < nn; ++e) term[e] = tmp[e] / (double)i;
        for (size_t e = 0; e < nn; ++e) E[e] += term[e];
        if (norm1(n, term) < ldexp(1.0, -60) * norm1(n, E)) break;
    }
    for (int r = 0; r < s; ++r) {
        mm(n, E, E, tmp);
        memcpy(E, tmp, sizeof(cplx) * nn);
    }
    free(X); free(term); free(tmp);
    return QALREF_OK;
}

/* ------------------------------------------------------------------ */
/* Controls (the coefficient matrix of the control Hamiltonians).            */
/* mode 0 (PWC):   u[k][j]        held on the whole slice                           */
/* mode 1 (NODES): u[k][a][j]     value at Gauss-Legendre node a of slice k          */
/* ------------------------------------------------------------------ */
static double ctrl(int mode, int J, const double *u, int k, int a, int j)
{
    return mode == 0 ? u[(size_t)k * J + j] : u[((size_t)k * 2 + a) * J + j];
}

/* A = L0 + sum_j v_j L_j  (Eq. 8 is linear in H) */
static void assemble(int n, int J, const cplx *L0, const cplx *Lc, const double *v, cplx *A)
{
    size_t nn = (size_t)n * n;
    for (size_t e = 0; e < nn; ++e) {
        cplx s = L0[e];
        for (int j = 0; j < J; ++j) s += v[j] * Lc[(size_t)j * nn + e];
        A[e] = s;
    }
}

/* ------------------------------------------------------------------ */
/* Oracle step O3: the slice generator.                                            */
/* order 4 (A1, A2; Blanes et al. [1], P:209 -- the 4th-order Magnus method with    */
/* two Gauss-Legendre nodes):                                                      */
/*   A_a = L(tau_a),  Omega = (h/2)(A_1 + A_2) - (sqrt(3) h^2 / 12) [A_1, A_2]      */
/*   with A_1 at the EARLIER node tau_1 = t_k + (1/2 - sqrt(3)/6) h.                */
/* order 2: Omega = (h/2)(A_1 + A_2) (Eq. 13, by 2-node quadrature).         */
/* The commutator is formed with explicit products; no shortcut for A_1 = A_2.      */
/* ------------------------------------------------------------------ */
int qalref_magnus_generator(int n, int order, double h, int J, const cplx *L0, const cplx *Lc,
                            const double *u1, const double *u2, cplx *Omega)
{
    size_t nn = (size_t)n * n;
    cplx *A1 = malloc(sizeof(cplx) * nn), *A2 = malloc(sizeof(cplx) * nn);
    cplx *P = malloc(sizeof(cplx) * nn), *Q = malloc(sizeof(cplx) * nn);
    assemble(n, J, L0, Lc, u1, A1);
    assemble(n, J, L0, Lc, u2, A2);
    for (size_t e = 0; e < nn; ++e) Omega[e] = 0.5 * h * (A1[e] + A2[e]);
    if (order == 4) {
        double c = sqrt(3.0) * h * h / 12.0;
        mm(n, A1, A2, P);
        mm(n, A2, A1, Q);
        for (size_t e = 0; e < nn; ++e) Omega[e] -= c * (P[e] - Q[e]);
    }
    free(A1); free(A2); free(P); free(Q);
    return QALREF_OK;
}

static void slice_generator(int n, int N, double T, int order, int mode, int J, const double *u,
                            const cplx *L0, const cplx *Lc, int k, cplx *Omega)
{
    double h = T / N;
    double u1[64], u2[64];
    for (int j = 0; j < J; ++j) { u1[j] = ctrl(mode, J, u, k, 0, j); u2[j] = ctrl(mode, J, u, k, 1, j); }
    qalref_magnus_generator(n, order, h, J, L0, Lc, u1, u2, Omega);
}

/* ------------------------------------------------------------------ */
/* Oracle step O5 (Eq. 15): Lambda = U_{k1-1} ... U_{k0}, later slice on */
/* the LEFT (A4), by a sequential left fold from the identity.  Optionally stores  */
/* every U_k (Ustore[k - k0]).                                                      */
/* ------------------------------------------------------------------ */
int qalref_propagate(int n, int N, double T, int order, int mode, int J, const double *u,
                     const cplx *L0, const cplx *Lc, int k0, int k1, cplx *Lambda, cplx *Ustore)
{
    if (J > 64 || k0 < 0 || k1 > N || k0 > k1) return QALREF_ERR_DIM;
    size_t nn = (size_t)n * n;
    cplx *Om = malloc(sizeof(cplx) * nn), *U = malloc(sizeof(cplx) * nn), *tmp = malloc(sizeof(cplx) * nn);
    eye(n, Lambda);
    for (int k = k0; k < k1; ++k) {
        slice_generator(n, N, T, order, mode, J, u, L0, Lc, k, Om);
        qalref_expm(n, Om, U);
        if (Ustore) memcpy(Ustore + (size_t)(k - k0) * nn, U, sizeof(cplx) * nn);
        mm(n, U, Lambda, tmp);
        memcpy(Lambda, tmp, sizeof(cplx) * nn);
    }
    free(Om); free(U); free(tmp);
    return QALREF_OK;
}

/* ------------------------------------------------------------------ */
/* Oracle step O6: gate (process) fidelity to the target V (A8):                    */
/*   F = Re Tr(S_V^dag Lambda) / d^2,  S_V = conj(V) (x) V formed explicitly         */
/*   (the superoperator of rho -> V rho V^dag under column stacking, Eq. 8's rule).   */
/* ------------------------------------------------------------------ */
double qalref_fidelity(int d, const cplx *Lambda, const cplx *V)
{
    int n = d * d;
    cplx *Vc = malloc(sizeof(cplx) * d * d);
    cplx *S = malloc(sizeof(cplx) * (size_t)n * n);
    for (int e = 0; e < d * d; ++e) Vc[e] = conj(V[e]);
    kron(d, Vc, d, V, S);
    double acc = 0.0;
    for (size_t e = 0; e < (size_t)n * n; ++e) acc += creal(conj(S[e]) * Lambda[e]);
    free(Vc); free(S);
    return acc / ((double)d * d);
}

/* ------------------------------------------------------------------ */
/* Frechet derivative of exp (the "expm Frechet derivative" of BASELINE north_star): */
/*   expm([[A, E], [0, A]]) = [[e^A, L(A,E)], [0, e^A]]  -> L = top-right block,      */
/* computed with the dense 2n x 2n exponential (oracle step O7).                     */
/* ------------------------------------------------------------------ */
int qalref_frechet(int n, const cplx *A, const cplx *E, cplx *Lout, cplx *expA)
{
    int m = 2 * n;
    cplx *Aug = calloc((size_t)m * m, sizeof(cplx)), *R = malloc(sizeof(cplx) * (size_t)m * m);
    if (!Aug || !R) { free(Aug); free(R); return QALREF_ERR_ALLOC; }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            Aug[(size_t)i * m + j] = A[(size_t)i * n + j];
            Aug[(size_t)(i + n) * m + (j + n)] = A[(size_t)i * n + j];
            Aug[(size_t)i * m + (j + n)] = E[(size_t)i * n + j];
        }
    qalref_expm(m, Aug, R);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            Lout[(size_t)i * n + j] = R[(size_t)i * m + (j + n)];
            if (expA) expA[(size_t)i * n + j] = R[(size_t)i * m + j];
        }
    free(Aug); free(R);
    return QALREF_OK;
}

/* ------------------------------------------------------------------ */
/* Oracle step O7: fidelity gradient with respect to every control value.            */
/*   F = Re Tr(S_V^dag U_{N-1} ... U_0) / d^2                                         */
/*   dF/du = Re Tr(G_k dU_k) / d^2,  G_k = P_k S_V^dag U_{N-1}...U_{k+1},             */
/*   P_k = U_{k-1} ... U_0,  dU_k = L(Omega_k, dOmega_k/du)  (per direction, dense     */
/*   2n x 2n augmented exponential -- not the adjoint form the CUDA path uses).        */
/* dOmega_k/du from the O3 formula by the product rule, explicit products:             */
/*   PWC  (u_{k,j} on both nodes): (h/2)(2 L_j) - c([L_j, A_2] + [A_1, L_j])           */
/*   NODES (u_j(tau_{k,1})):        (h/2) L_j     - c [L_j, A_2]                        */
/*   NODES (u_j(tau_{k,2})):        (h/2) L_j     - c [A_1, L_j]                        */
/* grad has the layout of u.  Returns F in *F.                                        */
/* ------------------------------------------------------------------ */
static int gradient_core(int d, int N, double T, int order, int mode, int J, const double *u,
                         const cplx *L0, const cplx *Lc, const cplx *V, const cplx *Cseed, double *F,
                         double *grad, cplx *LambdaOut);

int qalref_gradient(int d, int N, double T, int order, int mode, int J, const double *u,
                    const cplx *L0, const cplx *Lc, const cplx *V, double *F, double *grad,
                    cplx *LambdaOut)
{
    return gradient_core(d, N, T, order, mode, J, u, L0, Lc, V, NULL, F, grad, LambdaOut);
}

/* Reverse-mode product for any scalar objective with dL = Re Tr(C dLambda): the same per-direction
 * augmented exponentials as qalref_gradient, with the suffix seeded by C instead of S_V^dag / d^2. */
int qalref_vjp(int n, int N, double T, int order, int mode, int J, const double *u, const cplx *L0,
               const cplx *Lc, const cplx *C, double *grad, cplx *LambdaOut)
{
    double F = 0.0;
    int d = (int)lround(sqrt((double)n));
    return gradient_core(d, N, T, order, mode, J, u, L0, Lc, NULL, C, &F, grad, LambdaOut);
}

static int gradient_core(int d, int N, double T, int order, int mode, int J, const double *u,
                         const cplx *L0, const cplx *Lc, const cplx *V, const cplx *Cseed, double *F,
                         double *grad, cplx *LambdaOut)
{
    if (J > 64) return QALREF_ERR_DIM;
    int n = d * d;
    size_t nn = (size_t)n * n;
    double h = T / N;
    double c4 = (order == 4) ? sqrt(3.0) * h * h / 12.0 : 0.0;
    cplx *U = malloc(sizeof(cplx) * nn * N);        /* U_k */
    cplx *P = malloc(sizeof(cplx) * nn * (N + 1));  /* P_k = U_{k-1}..U_0, P_0 = I */
    cplx *X = malloc(sizeof(cplx) * nn * (N + 1));  /* X_k = S_V^dag U_{N-1}..U_k, X_N = S_V^dag */
    cplx *Om = malloc(sizeof(cplx) * nn * N);
    cplx *S = malloc(sizeof(cplx) * nn), *Vc = malloc(sizeof(cplx) * d * d);
    if (!U || !P || !X || !Om || !S || !Vc) return QALREF_ERR_ALLOC;

    eye(n, P);
    for (int k = 0; k < N; ++k) {
        slice_generator(n, N, T, order, mode, J, u, L0, Lc, k, Om + (size_t)k * nn);
        qalref_expm(n, Om + (size_t)k * nn, U + (size_t)k * nn);
        mm(n, U + (size_t)k * nn, P + (size_t)k * nn, P + (size_t)(k + 1) * nn);
    }
    if (LambdaOut) memcpy(LambdaOut, P + (size_t)N * nn, sizeof(cplx) * nn);
    double scale = 1.0;
    if (Cseed) {
        /* X_N = C */
        memcpy(X + (size_t)N * nn, Cseed, sizeof(cplx) * nn);
    } else {
        *F = qalref_fidelity(d, P + (size_t)N * nn, V);
        /* X_N = S_V^dag (explicit conjugate transpose of conj(V) (x) V), objective scaled by 1/d^2 */
        for (int e = 0; e < d * d; ++e) Vc[e] = conj(V[e]);
        kron(d, Vc, d, V, S);
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) X[(size_t)N * nn + (size_t)a * n + b] = conj(S[(size_t)b * n + a]);
        scale = 1.0 / ((double)d * d);
    }
    for (int k = N - 1; k >= 0; --k)
        mm(n, X + (size_t)(k + 1) * nn, U + (size_t)k * nn, X + (size_t)k * nn);

    int nodes = (mode == 1) ? 2 : 1;
    int ndir = N * nodes * J;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int dir = 0; dir < ndir; ++dir) {
        int k = dir / (nodes * J);
        int a = (dir / J) % nodes;
        int j = dir % J;
        cplx *A1 = malloc(sizeof(cplx) * nn), *A2 = malloc(sizeof(cplx) * nn);
        cplx *E = malloc(sizeof(cplx) * nn), *T1 = malloc(sizeof(cplx) * nn), *T2 = malloc(sizeof(cplx) * nn);
        cplx *G = malloc(sizeof(cplx) * nn), *dU = malloc(sizeof(cplx) * nn);
        double v1[64], v2[64];
        for (int q = 0; q < J; ++q) { v1[q] = ctrl(mode, J, u, k, 0, q); v2[q] = ctrl(mode, J, u, k, 1, q); }
        assemble(n, J, L0, Lc, v1, A1);
        assemble(n, J, L0, Lc, v2, A2);
        const cplx *Lj = Lc + (size_t)j * nn;
        double wgt = (mode == 0) ? h : 0.5 * h;
        for (size_t e = 0; e < nn; ++e) E[e] = wgt * Lj[e];
        if (order == 4) {
            if (mode == 0 || a == 0) {             /* [L_j, A_2] */
                mm(n, Lj, A2, T1); mm(n, A2, Lj, T2);
                for (size_t e = 0; e < nn; ++e) E[e] -= c4 * (T1[e] - T2[e]);
            }
            if (mode == 0 || a == 1) {             /* [A_1, L_j] */
                mm(n, A1, Lj, T1); mm(n, Lj, A1, T2);
                for (size_t e = 0; e < nn; ++e) E[e] -= c4 * (T1[e] - T2[e]);
            }
        }
        qalref_frechet(n, Om + (size_t)k * nn, E, dU, NULL);
        mm(n, P + (size_t)k * nn, X + (size_t)(k + 1) * nn, G);
        double acc = 0.0;
        for (int r = 0; r < n; ++r)
            for (int q = 0; q < n; ++q) acc += creal(G[(size_t)r * n + q] * dU[(size_t)q * n + r]);
        grad[dir] = acc * scale;
        free(A1); free(A2); free(E); free(T1); free(T2); free(G); free(dU);
    }
    free(U); free(P); free(X); free(Om); free(S); free(Vc);
    return QALREF_OK;
}

/* ------------------------------------------------------------------ */
/* configs[3] control function (A11):                                               */
/*   s_j(t) = sum_m a_m sin(2 pi f_m t + phi_m) / sqrt(sum_m a_m^2 / 2)               */
/*   u_j(t) = clip(u_max/2 (1 + 0.5 s_j(t)), 0, u_max)                                */
/* prm[j][m][3] = (a, f, phi).  The paper prints no values; pinned by A11's mathematics. */
/* ------------------------------------------------------------------ */
void qalref_sines_eval(int J, int nterm, const double *prm, double umax, double t, double *out)
{
    for (int j = 0; j < J; ++j) {
        double s = 0.0, a2 = 0.0;
        for (int m = 0; m < nterm; ++m) {
            const double *p = prm + ((size_t)j * nterm + m) * 3;
            s += p[0] * sin(2.0 * M_PI * p[1] * t + p[2]);
            a2 += p[0] * p[0];
        }
        s /= sqrt(a2 / 2.0);
        double v = 0.5 * umax * (1.0 + 0.5 * s);
        out[j] = v < 0.0 ? 0.0 : (v > umax ? umax : v);
    }
}

/* Sample the sinusoid controls at the two Gauss-Legendre nodes of every slice of the
 * uniform grid t_k = k T / N (A2): tau_{k,1,2} = t_k + (1/2 -+ sqrt(3)/6) h.
 * out[k][a][j] for k in [k0, k1).                                                 */
void qalref_sines_nodes(int J, int nterm, const double *prm, double umax, int N, double T,
                        int k0, int k1, double *out)
{
    double h = T / N, c = sqrt(3.0) / 6.0;
    for (int k = k0; k < k1; ++k) {
        double tk = k * h;
        qalref_sines_eval(J, nterm, prm, umax, tk + (0.5 - c) * h, out + ((size_t)(k - k0) * 2 + 0) * J);
        qalref_sines_eval(J, nterm, prm, umax, tk + (0.5 + c) * h, out + ((size_t)(k - k0) * 2 + 1) * J);
    }
}

/* ------------------------------------------------------------------ */
/* Oracle step O8 (Eqs. 9-10): fixed-step classical RK4 of                */
/*   dLambda/dt = L(t) Lambda, Lambda(0) = I,  L(t) = L0 + sum_j u_j(t) L_j,          */
/* with `sub` steps per slice of the uniform grid.  Controls:                        */
/*   cmode 0: PWC table u[k][j] (the slice's value on the whole closed slice)         */
/*   cmode 2: sinusoid function (prm, umax) evaluated at every RK stage time           */
/* ------------------------------------------------------------------ */
int qalref_rk4(int n, int N, double T, int sub, int cmode, int J, const double *u,
               const double *prm, int nterm, double umax,
               const cplx *L0, const cplx *Lc, cplx *Lambda)
{
    if (J > 64) return QALREF_ERR_DIM;
    size_t nn = (size_t)n * n;
    double h = T / N, dt = h / sub;
    cplx *Lt = malloc(sizeof(cplx) * nn), *Y = malloc(sizeof(cplx) * nn);
    cplx *k1 = malloc(sizeof(cplx) * nn), *k2 = malloc(sizeof(cplx) * nn);
    cplx *k3 = malloc(sizeof(cplx) * nn), *k4 = malloc(sizeof(cplx) * nn);
    double v[64];
    eye(n, Lambda);
    for (int k = 0; k < N; ++k) {
        for (int s = 0; s < sub; ++s) {
            double t0 = k * h + s * dt;
            double ts[3] = {t0, t0 + 0.5 * dt, t0 + dt};
            cplx *ks[4] = {k1, k2, k3, k4};
            for (int st = 0; st < 4; ++st) {
                double t = ts[(st + 1) / 2];
                if (cmode == 0) for (int j = 0; j < J; ++j) v[j] = u[(size_t)k * J + j];
                else qalref_sines_eval(J, nterm, prm, umax, t, v);
                assemble(n, J, L0, Lc, v, Lt);
                if (st == 0) memcpy(Y, Lambda, sizeof(cplx) * nn);
                else {
                    double w = (st == 3) ? 1.0 : 0.5;
                    for (size_t e = 0; e < nn; ++e) Y[e] = Lambda[e] + w * dt * ks[st - 1][e];
                }
                mm(n, Lt, Y, ks[st]);
            }
            for (size_t e = 0; e < nn; ++e)
                Lambda[e] += dt / 6.0 * (k1[e] + 2.0 * k2[e] + 2.0 * k3[e] + k4[e]);
        }
    }
    free(Lt); free(Y); free(k1); free(k2); free(k3); free(k4);
    return QALREF_OK;
}

/* cotangent of the fidelity: C = S_V^dag / d^2 with S_V = conj(V) (x) V formed explicitly */
void qalref_fidelity_cotangent(int d, const cplx *V, cplx *C)
{
    int n = d * d;
    cplx *Vc = malloc(sizeof(cplx) * d * d), *S = malloc(sizeof(cplx) * (size_t)n * n);
    for (int e = 0; e < d * d; ++e) Vc[e] = conj(V[e]);
    kron(d, Vc, d, V, S);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) C[(size_t)a * n + b] = conj(S[(size_t)b * n + a]) / ((double)d * d);
    free(Vc); free(S);
}

/* ------------------------------------------------------------------ */
/* Eqs. 16-17: Pi = P^dag Lambda P with P (n x 2) the flattened logical density       */
/* matrices; loss = (1/4) ||Pi - G||_F^2 with ||A||_F^2 = Tr(A^dag A) (A22); cotangent             */
/* C = 1/2 P (Pi - G)^dag P^dag of d loss = Re Tr(C dLambda).  Explicit products, plain loops.     */
/* ------------------------------------------------------------------ */
int qalref_logical_loss(int n, const cplx *Lambda, const cplx *P, const cplx *G, double *loss, cplx *C)
{
    cplx *LP = malloc(sizeof(cplx) * (size_t)n * 2);   /* Lambda P, n x 2 */
    cplx Pi[4], A[4];
    for (int i = 0; i < n; ++i)
        for (int b = 0; b < 2; ++b) {
            cplx s = 0;
            for (int j = 0; j < n; ++j) s += Lambda[(size_t)i * n + j] * P[(size_t)j * 2 + b];
            LP[(size_t)i * 2 + b] = s;
        }
    double l = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            cplx s = 0;
            for (int i = 0; i < n; ++i) s += conj(P[(size_t)i * 2 + a]) * LP[(size_t)i * 2 + b];
            Pi[a * 2 + b] = s;
            A[a * 2 + b] = s - G[a * 2 + b];
        }
    for (int a = 0; a < 2; ++a)              /* Tr(A^dag A) = sum_{ab} conj(A_ab) A_ab */
        for (int b = 0; b < 2; ++b) l += creal(conj(A[a * 2 + b]) * A[a * 2 + b]);
    *loss = 0.25 * l;
    if (C) {
        cplx PAd[2 * 64 * 64];               /* P A^dag (n x 2), n <= 4096 */
        if (n > 2048) { free(LP); return QALREF_ERR_DIM; }
        for (int i = 0; i < n; ++i)
            for (int b = 0; b < 2; ++b) {
                cplx s = 0;
                for (int a = 0; a < 2; ++a) s += P[(size_t)i * 2 + a] * conj(A[b * 2 + a]);
                PAd[i * 2 + b] = s;
            }
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                cplx s = 0;
                for (int b = 0; b < 2; ++b) s += PAd[i * 2 + b] * conj(P[(size_t)j * 2 + b]);
                C[(size_t)i * n + j] = 0.5 * s;
            }
    }
    free(LP);
    return QALREF_OK;
}

/* Adam (Kingma & Ba, ref [13]) with bias correction, step t >= 1 */
void qalref_adam_step(int n, double *theta, const double *g, double *m, double *v, int t, double lr, double b1,
                      double b2, double eps)
{
    for (int i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        double mh = m[i] / (1.0 - pow(b1, t)), vh = v[i] / (1.0 - pow(b2, t));
        theta[i] -= lr * mh / (sqrt(vh) + eps);
    }
}

/* plain product, exported for the ordered-product pins (P-12): C = A B */
void qalref_matmul(int n, const cplx *A, const cplx *B, cplx *C) { mm(n, A, B, C); }

/* rows r0..r1-1 of A B (n x n), plain sums -- sampled checks of the n = 4096 products */
void qalref_matmul_rows(int n, const cplx *A, const cplx *B, int r0, int r1, cplx *C)
{
    #pragma omp parallel for schedule(static)
    for (int i = r0; i < r1; ++i)
        for (int j = 0; j < n; ++j) {
            cplx s = 0;
            for (int k = 0; k < n; ++k)
                s += A[(size_t)i * n + k] * B[(size_t)k * n + j];
            C[(size_t)(i - r0) * n + j] = s;
        }
}

/* ------------------------------------------------------------------ */
/* Eq. 6 integrated directly on the density matrix (d x d), classical RK4 with  */
/* `sub` steps per slice of the uniform grid, PWC controls u[k][j] (H(t) = H0 +         */
/* sum_j u_j H_j on slice k).  O(d^3) per stage: the d = 64 (configs[4]) dissipative    */
/* check never forms a 4096 x 4096 superoperator.                                       */
/* ------------------------------------------------------------------ */
int qalref_evolve_rho(int d, const cplx *H0, int J, const cplx *Hc, int ncops, const cplx *C, int N, double T,
                      int sub, const double *u, const cplx *rho0, cplx *rho)
{
    size_t dd = (size_t)d * d;
    double h = T / N, dt = h / sub;
    cplx *H = malloc(sizeof(cplx) * dd), *Y = malloc(sizeof(cplx) * dd);
    cplx *k1 = malloc(sizeof(cplx) * dd), *k2 = malloc(sizeof(cplx) * dd);
    cplx *k3 = malloc(sizeof(cplx) * dd), *k4 = malloc(sizeof(cplx) * dd);
    memcpy(rho, rho0, sizeof(cplx) * dd);
    for (int k = 0; k < N; ++k) {
        for (size_t e = 0; e < dd; ++e) {
            cplx s = H0[e];
            for (int j = 0; j < J; ++j) s += u[(size_t)k * J + j] * Hc[(size_t)j * dd + e];
            H[e] = s;
        }
        for (int s = 0; s < sub; ++s) {
            qalref_lindblad_rhs(d, H, ncops, C, rho, k1);
            for (size_t e = 0; e < dd; ++e) Y[e] = rho[e] + 0.5 * dt * k1[e];
            qalref_lindblad_rhs(d, H, ncops, C, Y, k2);
            for (size_t e = 0; e < dd; ++e) Y[e] = rho[e] + 0.5 * dt * k2[e];
            qalref_lindblad_rhs(d, H, ncops, C, Y, k3);
            for (size_t e = 0; e < dd; ++e) Y[e] = rho[e] + dt * k3[e];
            qalref_lindblad_rhs(d, H, ncops, C, Y, k4);
            for (size_t e = 0; e < dd; ++e) rho[e] += dt / 6.0 * (k1[e] + 2.0 * k2[e] + 2.0 * k3[e] + k4[e]);
        }
    }
    free(H); free(Y); free(k1); free(k2); free(k3); free(k4);
    return QALREF_OK;
}
