/*
 * iga_lr.h — C ABI of the B200-native low-rank IgA operator library (libigalr.so).
 *
 * The hot path of arXiv:1811.06797 ("low-rank IgA"): mass and stiffness matrices held as
 * sums of Kronecker products of banded univariate B-spline matrices,
 *     M = sum_r  M_r^z (x) M_r^y (x) M_r^x                 Eq. (massFinal)
 *     K = sum_kl sum_r K_klr^z (x) K_klr^y (x) K_klr^x     Eq. (stiffnessFinal)
 * (the build calls K "S"), their univariate factors assembled by Gauss quadrature
 *     M^(d)(w)_ij     = int beta_i beta_j w                 Eq. (massMatrix1D)
 *     K^(d)_kl(q)_ij  = int delta(l,d)beta_i delta(k,d)beta_j q
 * and the implicit-Euler KKT matvec of Eq. (KKTSystem) PAPER.md:313-319 with
 *     calM = I (x) M,  calK = I (x) tau K + C (x) M        Eqs. (M_kron)/(K_kron) PAPER.md:316,326-331.
 *
 * Conventions
 *   - Directions: index 0 = x (fastest, contiguous), 1 = y, 2 = z (slowest).  The paper's
 *     (x)_{d=1..D} lists the slowest direction first.
 *   - Vectors are fp64, C-ordered [batch][nz][ny][nx] in DEVICE memory unless a function
 *     says HOST.  With IGA_DIRICHLET the extents are the interior ones (n_d - 2).
 *   - Every function returns iga_status (0 == IGA_OK).  On failure a message is stored in a
 *     thread-local buffer readable with iga_last_error().  No CPU fallback exists: a missing
 *     or failing GPU returns IGA_ECUDA.
 *   - Device work is stream-ordered on the caller's stream (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  No call synchronises the device except
 *     iga_lr_assemble_factors (it waits for its own uploads) and the *_host entry points.
 *   - Thread safety: an iga_lr_op is immutable after assembly; concurrent applies on
 *     different streams are allowed (scratch memory is stream-ordered, cudaMallocAsync).
 *     Internally the op caches, behind a mutex: the fixup tables of its launch shapes (built
 *     on first use with one small H2D copy), a side stream on which small meshes run the mass
 *     part beside the stiffness part (event fork/join on the caller's stream), and the copy
 *     streams of iga_lr_apply_host (host-buffer calls on one op run one at a time).
 */
#ifndef IGA_LR_H
#define IGA_LR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IGA_OK = 0,
    IGA_EINVAL = 1,        /* invalid argument (knots, sizes, pointers, aliasing, tau/beta) */
    IGA_ENOMEM = 2,        /* host or device allocation failed */
    IGA_ECUDA = 3,         /* CUDA runtime error (message carries cudaGetErrorString) */
    IGA_EUNSUPPORTED = 4,  /* degree / quadrature size / plan shape outside compiled range */
    IGA_ESTATE = 5         /* operation needs a part the op was not assembled with */
} iga_status;

/* Opaque assembled operator.  Owns its device memory (banded factors + plan). */
typedef struct iga_lr_op iga_lr_op;

/* One univariate spline space: degree p >= 1, n >= p+1 basis functions, open knot vector
   of n+p+1 HOST doubles (Eq. (knotVector): first/last p+1 knots 0/1,
   nondecreasing, interior multiplicity <= p).  Copied by the library. */
typedef struct {
    int32_t p;
    int32_t n;
    const double* knots;
} iga_dir;

/* Tensor-product space S^3 = S_x (x) S_y (x) S_z.  nq = Gauss points per
   nonempty knot span in every direction (0 => p+1, reading G1 of DESIGN.md). */
typedef struct {
    iga_dir dir[3];
    int32_t nq;
} iga_space;

/* A rank-R separable weight  f(x,y,z) = sum_r coef[r] * f_r^x(x) f_r^y(y) f_r^z(z)
   (the paper's W_R : B~ of Eq. (weightLowRank), and q_kl PAPER.md:202-206).
   tab[d] is a HOST array [R][nnodes_d]: f_r^d tabulated at the quadrature nodes of direction
   d in the order returned by iga_quad_nodes (the caller evaluates w_r^(d).B~^(d) there).
   coef may be NULL (all ones).  Copied by the library. */
typedef struct {
    int32_t R;
    const double* coef;
    const double* tab[3];
} iga_sep;

/* flags of iga_lr_assemble_factors */
#define IGA_DIRICHLET 0x1u   /* drop the first and last basis index in every direction
                                ("omitting the boundary nodes") */

/* flags of the apply entry points (kernel path selection; results agree to rounding) */
#define IGA_PATH_AUTO 0x0u      /* fused sm_100a kernel when the plan fits, else unfused */
#define IGA_PATH_UNFUSED 0x10u  /* one launch per mode-product stage through HBM scratch */
#define IGA_PATH_FUSED 0x20u    /* fused kernel; IGA_EUNSUPPORTED if the plan does not fit */
#define IGA_PATH_FUSED_V1 0x40u /* force the first-generation fused kernel (testing) */

/* Quadrature nodes of direction dir (0..2): nq-point Gauss-Legendre on each nonempty span,
   ascending.  nodes_out may be NULL to query *nnodes (= nonempty spans * nq). HOST memory. */
iga_status iga_quad_nodes(const iga_space* sp, int32_t dir, double* nodes_out, int64_t* nnodes);

/* Assemble the banded univariate factors on the GPU and build the evaluation plan.
     omega : mass weight (NULL => op has no mass part)                      Eq. (massFinal)
     q     : array of 9 pointers, q[k*3+l] = weight q_kl of Eq. (stiffnessMatrix)
             (k = direction differentiated on the column/test function j, l = on the row
             function i: K_ij = sum_kl int q_kl d_l beta_i d_k beta_j);
             q == NULL => no stiffness part; q[b] == NULL => zero block.
   Univariate factors are deduplicated by (direction, tabulated weight content, derivative
   pattern); Dirichlet slicing is applied to every factor.  Blocks on `stream` until the
   factors are resident.  *out receives a new op (free with iga_lr_destroy). */
iga_status iga_lr_assemble_factors(const iga_space* sp, const iga_sep* omega, const iga_sep* const* q,
                                   uint32_t flags, void* stream, iga_lr_op** out);

void iga_lr_destroy(iga_lr_op* op);

/* y_mass = alpha * M x   (if y_mass != NULL)
   y_stiff = gamma * S x  (if y_stiff != NULL)
   If y_mass == y_stiff (non-NULL) the single output receives alpha*M x + gamma*S x.
   x, y: DEVICE fp64 [batch][nz][ny][nx], 8-byte aligned, outputs must not alias x.
   flags: IGA_PATH_*.  Errors: IGA_EINVAL (batch < 1, NULL x, aliasing, misalignment),
   IGA_ESTATE (output requested for a part the op lacks). */
iga_status iga_lr_apply(const iga_lr_op* op, const double* x, double* y_mass, double* y_stiff, double alpha,
                        double gamma, int32_t batch, uint32_t flags, void* stream);

/* Two-input form used by the KKT matvec: out = alpha * M x_mass + gamma * S x_stiff
   (either input may be NULL to drop that part). Same layout rules as iga_lr_apply. */
iga_status iga_lr_apply2(const iga_lr_op* op, const double* x_mass, const double* x_stiff, double* out,
                         double alpha, double gamma, int32_t batch, uint32_t flags, void* stream);

/* KKT matvec, Eq. (KKTSystem) PAPER.md:313-319:
     out = [ tau calM, 0, calK^T ; 0, tau beta calM, -tau calM ; calK, -tau calM, 0 ] in
   with calM = I_nt (x) M, calK = I_nt (x) tau S + C (x) M, C = bidiagonal (1 on the
   diagonal, -1 below).  in/out: DEVICE fp64 [3][n_t][nz][ny][nx], blocks
   (y, u, lambda).  Needs an op with mass and stiffness (else IGA_ESTATE);
   tau > 0, beta > 0, n_t >= 1 (else IGA_EINVAL).  in and out must not alias.
   calK^T carries S^T (PAPER.md:306 writes the y-row as lambda_k (M + tau K)): when the op was
   assembled with q[k*3+l] and q[l*3+k] that differ (in R, coefficients or tables), S is not
   symmetric and the op holds a second plan for S^T (block (k,l) of S^T = weight q_kl with the
   derivative patterns of block (l,k)), so the KKT matrix stays symmetric for MINRES.
   Workspace: stream-ordered scratch from the op's pool, 5 n_t vectors ([M y, M u, M lambda,
   tau S^T lambda, tau S y]; the rows are combined per time step afterwards) on the canonical
   route, 3 n_t vectors on the generic fallback; the call does not synchronise `stream`. */
iga_status iga_kkt_apply(const iga_lr_op* op, int32_t n_t, double tau, double beta, const double* in,
                         double* out, uint32_t flags, void* stream);

/* ---------------------------------------------------------------- KKT solve (NEXT-1)
   All-at-once solve of Eq. (KKTSystem) PAPER.md:313-319 for (y, u, lambda) by MINRES (Paige &
   Saunders; the Krylov method the paper names for its reduced KKT systems),
   with iga_kkt_apply as the matvec and an optional block-diagonal preconditioner.

   Preconditioner (iga_kkt_prec_*): P = blkdiag(tau calMh, tau beta calMh, Sh), Sh the
   Pearson-Stoll-Wathen "matching" Schur-complement approximation
       Sh = (1/tau) (calKh + g calMh) calMh^{-1} (calKh + g calMh)',  g = tau / sqrt(beta),
   with M, S replaced by mbar M0, sbar S0: the unit-weight Kronecker mass / Laplace-stiffness of
   the op's spline spaces (factors of Eq. (massMatrix1D) with w = 1), scaled by the op's own
   Rayleigh quotients on the smoothest mode.  All solves run in the fast-diagonalisation basis
   of the univariate pencils (K0d, M0d); see DESIGN.md §11.  The preconditioner is tied to
   (op extents, n_t, tau, beta) and must not outlive the op's device.
     iga_kkt_prec_create : builds it (host eigen-decompositions + one op apply; synchronises).
     iga_kkt_prec_apply  : out = P^{-1} in (DEVICE [3][n_t][Nz][Ny][Nx]; in != out).
     iga_kkt_prec_info   : mbar, sbar and the univariate eigenvalues (HOST, m_x + m_y + m_z).
   MINRES (iga_kkt_minres):
     prec: NULL (P = I) or a preconditioner built for the same op, n_t, tau, beta.
     rhs : DEVICE fp64 [3][n_t][Nz][Ny][Nx] (blocks y, u, lambda; e.g. [tau M yhat; 0; 0]).
     x   : DEVICE fp64, same layout.  On entry the initial guess if flags has IGA_MINRES_X0,
           otherwise ignored (x_0 = 0); on return the last MINRES iterate.
     rtol: stop when |r_j|_{P^{-1}} <= rtol |r_0|_{P^{-1}} (|eta| of the recurrence);
     maxit: iteration cap (0 => only r_0 is formed).   flags: IGA_PATH_* | IGA_MINRES_X0.
   Workspace (7-8 vectors) is stream-ordered scratch; the call synchronises `stream` once per
   iteration (8-byte read of |eta|) and before returning.  Reductions are deterministic.
   Errors: as iga_kkt_apply, plus IGA_EINVAL for rhs == x, maxit < 0, rtol < 0, a
   preconditioner built for other arguments. */
#define IGA_MINRES_X0 0x100u
typedef struct iga_kkt_prec iga_kkt_prec;
typedef struct {
    int32_t iters;      /* MINRES iterations performed */
    int32_t converged;  /* 1 if |r| <= rtol |r_0| */
    double relres;      /* |r_iters| / |r_0| (recurrence estimate, P^{-1} norm) */
    double res0;        /* |r_0| = |rhs - A x_0|_{P^{-1}} */
} iga_minres_info;
iga_status iga_kkt_prec_create(const iga_lr_op* op, int32_t n_t, double tau, double beta, uint32_t flags,
                               void* stream, iga_kkt_prec** out);
void iga_kkt_prec_destroy(iga_kkt_prec* prec);
iga_status iga_kkt_prec_apply(const iga_kkt_prec* prec, const double* in, double* out, void* stream);
iga_status iga_kkt_prec_info(const iga_kkt_prec* prec, double* mbar, double* sbar, double* lam);
iga_status iga_kkt_minres(const iga_lr_op* op, const iga_kkt_prec* prec, int32_t n_t, double tau, double beta,
                          const double* rhs, double* x, double rtol, int32_t maxit, uint32_t flags, void* stream,
                          iga_minres_info* info);

/* ---------------------------------------------------------------- low-rank weights (NEXT-2)
   The step before the path: samples of a weight function (omega =
   |det grad G| or an entry q_kl of Q) at the Greville points of an interpolation space S~ ->
   the rank-R separable form iga_sep that iga_lr_assemble_factors consumes.
     iga_greville: Greville abscissae (t_{i+1} + ... + t_{i+p}) / p of one direction (HOST, n).
     iga_weight_lowrank:
       target : the op's space (its quadrature nodes tabulate the factors).
       tilde  : 3 iga_dir of S~ (x, y, z); degree p~ <= 15.
       samples: HOST fp64 [n~z][n~y][n~x], the weight at the Greville points (x fastest).
       eps    : relative Frobenius accuracy of the TT-SVD of the samples (Oseledets'
                truncation eps |.|_F / sqrt(D-1) per unfolding); 0 => exact up to rounding.
       max_terms: cap on R = R1 R2.
       Steps: TT-SVD (slowest direction first) -> the univariate collocation solves of
       Eq. (weightEquationSolve) PAPER.md:256-262 per factor vector -> the R1 R2 canonical
       terms of Eq. (TTranks) PAPER.md:243-246 tabulated at the target's nodes.
       Errors: IGA_EINVAL (bad spaces, non-finite samples, singular collocation).
     iga_weight_lowrank_sep: a view (valid until _free) as iga_sep (coef = 1), the TT ranks
       (R1, R2) and the relative TT truncation error of the samples. */
typedef struct iga_lowrank_weight iga_lowrank_weight;
iga_status iga_greville(const iga_dir* d, double* out);
iga_status iga_weight_lowrank(const iga_space* target, const iga_dir* tilde, const double* samples, double eps,
                              int32_t max_terms, iga_lowrank_weight** out);
iga_status iga_weight_lowrank_sep(const iga_lowrank_weight* w, iga_sep* sep, int32_t* tt_ranks, double* tt_error);
void iga_weight_lowrank_free(iga_lowrank_weight* w);

/* End-to-end variants with HOST buffers (pageable or pinned): copy in, apply, copy out,
   synchronise `stream`.  Device staging is stream-ordered scratch owned by the call.
   iga_lr_apply_host pipelines the batch vector by vector (H2D, apply, D2H on three streams
   ordered by events): with pinned buffers both copy directions overlap the kernels.  Its
   result equals per-vector iga_lr_apply calls bit for bit (and a batched call to rounding). */
iga_status iga_lr_apply_host(const iga_lr_op* op, const double* x_host, double* y_mass_host,
                             double* y_stiff_host, double alpha, double gamma, int32_t batch, uint32_t flags,
                             void* stream);
iga_status iga_kkt_apply_host(const iga_lr_op* op, int32_t n_t, double tau, double beta, const double* in_host,
                              double* out_host, uint32_t flags, void* stream);

/* ---------------------------------------------------------------- introspection */
typedef struct {
    int64_t dims[3];             /* kept DoF extents (x, y, z) */
    int32_t p[3];
    int32_t nq;
    int32_t n_factors[3];        /* distinct banded factors per direction */
    int32_t n_rounds;            /* plan rounds (shared-prefix evaluation groups) */
    int32_t n_xprod, n_yprod, n_zprod; /* mode products per vector in the plan */
    int32_t has_mass, has_stiff;
    int32_t fused_ok;            /* 1 if the first-generation fused kernel supports this plan */
    int32_t fused2_ok;           /* 1 if the TMEM-ring fused kernel (v2) supports every part */
    /* Algorithmic flops (2 * nnz of every banded mode product) of the plan that
       the IGA_PATH_AUTO route executes for one vector: the canonical / fused-v2 per-part plans
       when they exist (reading A: 3R mass + 17R stiffness mode products), else the greedy plans. */
    double plan_flops_per_vec;   /* mass + stiffness apply of one vector */
    double min_bytes_per_vec;    /* 8 * (1 input + outputs) * N */
    double plan_flops_mass;      /* ... of a mass-only apply of one vector */
    double plan_flops_stiff;     /* ... of a stiffness-only apply of one vector */
    int32_t canon_mass;          /* 1 if the auto route runs the canonical mass kernel */
    int32_t canon_stiff;         /* 1 if the auto route runs the canonical (reading-A) stiffness kernel */
    int32_t stiff_symmetric;     /* 1 if q_kl and q_lk are identical for all k != l (K = K^T) */
    int32_t f2_rounds_stiff;     /* rounds of the fused-v2 stiffness plan (0 if none) */
} iga_lr_info_t;

iga_status iga_lr_info(const iga_lr_op* op, iga_lr_info_t* info);

/* Copy factor `factor_id` of direction `dir` to HOST band storage [m_d][2p+1]:
   band[i*(2p+1) + k] = F[i][i-p+k] (0 outside the matrix).  *pattern receives a*2+b where
   a/b are the derivative orders on the row/column function; *table receives the id of the
   deduplicated weight table.  Either output pointer may be NULL. */
iga_status iga_lr_export_factor(const iga_lr_op* op, int32_t dir, int32_t factor_id, double* host_band,
                                int32_t* pattern, int32_t* table);

/* ---- NEXT-3: the Kronecker operators on tensor-train vectors ----------
   A 3D TT vector (Eq. (tt)) with ranks (R1, R2) is three DEVICE fp64 cores in
   the paper's order (slowest direction first):
       Gz [n_z][R1],  Gy [R1][n_y][R2],  Gx [R2][n_x]
   v(iz, iy, ix) = sum_{a,b} Gz[iz][a] Gy[a][iy][b] Gx[b][ix]   (extents m_d of the op).
   The op is a sum of T Kronecker terms c_t Az_t (x) Ay_t (x) Ax_t of one part
   (part 0 = mass M, 1 = stiffness K; Eqs. (massFinal)/(stiffnessFinal)).

   iga_lr_terms: the T terms of `part` (the op's deduplicated, r-major term list): n_terms,
     and if non-NULL, HOST fid[t*3 + d] = factor id in direction d (0 x, 1 y, 2 z; see
     iga_lr_export_factor) and coef[t].  IGA_ESTATE if the op lacks the part.

   iga_tt_kron_apply: w = A v for a TT vector v, exactly, as T TT terms with v's ranks
     (the rank-(T R1, T R2) TT of w is their block concatenation):
       Wz [T][n_z][R1] = c_t Az_t Gz,  Wy [T][R1][n_y][R2] = Ay_t Gy,  Wx [T][R2][n_x] = Ax_t Gx
     (mode products along the physical index; w = sum_t Wz[t] Wy[t] Wx[t]).  DEVICE in/out,
     outputs must not alias inputs.

   iga_tt_interfaces: the frame interfaces of site `site` (0 x, 1 y, 2 z) for every term:
     the projection F_{!=d}^T A F_{!=d} of Eq. (KKT_red) with the frame
     matrix of Eq. (frame) equals sum_t c_t L_t (x) A^(d)_t (x) R_t, with
       L_t [Rl][Rl] = contraction of the cores left of d (slower directions) with A_t there,
       R_t [Rr][Rr] = the same for the cores right of d (faster directions);
     Rl = 1 (site z), R1 (y), R2 (x); Rr = R1 (z), R2 (y), 1 (x).  L, R: DEVICE [T][..][..].
     The coefficient c_t is not folded in.  (Orthogonality of the frame is the caller's.)

   iga_tt_local_apply: y = (sum_t c_t L_t (x) A^(d)_t (x) R_t) x for a local core
     x, y [Rl][m_d][Rr] (the reduced-system matvec of Eq. (KKT_red)); DEVICE, no aliasing.
   Errors: IGA_EINVAL (NULL pointers, ranks < 1, site outside 0..2), IGA_ESTATE (missing part),
   IGA_ECUDA. */
iga_status iga_lr_terms(const iga_lr_op* op, int32_t part, int32_t* n_terms, int32_t* fid, double* coef);
iga_status iga_tt_kron_apply(const iga_lr_op* op, int32_t part, int32_t R1, int32_t R2, const double* gz,
                             const double* gy, const double* gx, double* wz, double* wy, double* wx, void* stream);
iga_status iga_tt_interfaces(const iga_lr_op* op, int32_t part, int32_t site, int32_t R1, int32_t R2,
                             const double* gz, const double* gy, const double* gx, double* L, double* R,
                             void* stream);
iga_status iga_tt_local_apply(const iga_lr_op* op, int32_t part, int32_t site, int32_t Rl, int32_t Rr,
                              const double* L, const double* R, const double* x, double* y, void* stream);

/* Human-readable message of the last failing call on this thread ("" if none). */
const char* iga_last_error(void);

/* Library version string. */
const char* iga_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IGA_LR_H */
