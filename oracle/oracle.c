/*
 * oracle.c — CPU ORACLE for the low-rank IgA operator apply (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant with the
 * CUDA path (paper_1811_06797_b200/); it computes the *definitions* of the paper, not
 * the Kronecker method:
 *
 *   - knot vector / Cox-de Boor recursion ............ PAPER.md:51-63 (§2, Eq. knotVector)
 *   - B-spline derivative (textbook de Boor formula) .. used by delta(k,d)
 *   - Gauss-Legendre rule (Newton on P_m) per span ..... quadrature reading G1 (p+1 nodes)
 *   - mass matrix  M_ij = int beta_i beta_j omega ..... PAPER.md:136-139 Eq. (massMatrix)
 *   - stiffness    K_ij = sum_kl int q_kl d_l beta_i d_k beta_j
 *                                                      PAPER.md:140-143 Eq. (stiffnessMatrix)
 *   - univariate Gram  int B (x) B w ................ PAPER.md:192-196 Eq. (massMatrix1D),
 *                                                      PAPER.md:217-220 (K^{(d)}_{k,l})
 *   - Dirichlet: "omitting the boundary nodes" ........ PAPER.md:293
 *
 * All integrals use the same composite rule as the method: nq-point Gauss-Legendre on every
 * nonempty knot span, tensorised in 3D.  Weights are evaluated from their closed form
 * (synth/ term rows: coef * prod_d (1 + amp_d sin(k_d pi t_d + phi_d))) at every 3D point.
 *
 * Three routes compute y = A x: CSR assembly + naive SpMV (orc_assemble_csr/orc_spmv),
 * the element-loop bilinear form (orc_apply_matfree) and the same bilinear form for a
 * chosen set of rows (orc_apply_rows).  They are cross-checked in tests (pin P12).
 *
 * fp64 throughout, compiled without -ffast-math.  OpenMP only parallelises independent
 * rows / same-colour elements; every output is summed in a fixed order (deterministic).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_TERM 10
#define ORC_MAXP 8

/* ------------------------------------------------------------------------------------ */
/* Gauss-Legendre on [-1, 1]: Newton iteration on P_m using the three-term recurrence.   */
/* ------------------------------------------------------------------------------------ */
int orc_gauss_legendre(int m, double* x, double* w) {
    if (m < 1 || m > 64) return 1;
    for (int i = 0; i < m; ++i) {
        double z = cos(M_PI * (i + 0.75) / (m + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int j = 1; j <= m; ++j) { /* P_j = ((2j-1) z P_{j-1} - (j-1) P_{j-2}) / j */
                double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
            }
            dp = m * (z * p0 - p1) / (z * z - 1.0);
            double dz = p0 / dp;
            z -= dz;
            if (fabs(dz) < 1e-17) break;
        }
        /* recompute derivative at converged z for the weight */
        double p0 = 1.0, p1 = 0.0;
        for (int j = 1; j <= m; ++j) {
            double p2 = p1;
            p1 = p0;
            p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
        }
        dp = m * (z * p0 - p1) / (z * z - 1.0);
        /* ascending order */
        x[m - 1 - i] = z;
        w[m - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* All n B-spline values and first derivatives at t by the full Cox-de Boor triangle     */
/* (PAPER.md:58-63).  0/0 := 0.  Half-open spans; t == last knot belongs to the last     */
/* nonempty span (right-endpoint convention).                                */
/* ------------------------------------------------------------------------------------ */
int orc_basis_all(const double* knots, int n, int p, double t, double* vals, double* ders) {
    int m = n + p + 1; /* number of knots */
    if (p < 0 || p > ORC_MAXP || n < p + 1) return 1;
    double* N = (double*)calloc((size_t)m, sizeof(double));
    double* Nprev = (double*)calloc((size_t)m, sizeof(double));
    if (!N || !Nprev) { free(N); free(Nprev); return 2; }
    /* degree 0 */
    int last = -1;
    for (int i = 0; i < m - 1; ++i)
        if (knots[i] < knots[i + 1]) last = i;
    for (int i = 0; i < m - 1; ++i) {
        if (knots[i] <= t && t < knots[i + 1]) N[i] = 1.0;
    }
    if (t == knots[m - 1] && last >= 0) N[last] = 1.0;
    for (int j = 1; j <= p; ++j) {
        memcpy(Nprev, N, sizeof(double) * (size_t)m);
        for (int i = 0; i + j + 1 < m; ++i) {
            double a = 0.0, b = 0.0;
            double d1 = knots[i + j] - knots[i];
            double d2 = knots[i + j + 1] - knots[i + 1];
            if (d1 != 0.0) a = (t - knots[i]) / d1 * Nprev[i];
            if (d2 != 0.0) b = (knots[i + j + 1] - t) / d2 * Nprev[i + 1];
            N[i] = a + b;
        }
        for (int i = m - j - 1; i < m; ++i) N[i] = 0.0;
    }
    for (int i = 0; i < n; ++i) vals[i] = N[i];
    if (ders) {
        /* beta'_{i,p} = p beta_{i,p-1}/(x_{i+p}-x_i) - p beta_{i+1,p-1}/(x_{i+p+1}-x_{i+1}) */
        for (int i = 0; i < n; ++i) {
            double d = 0.0;
            if (p > 0) {
                double d1 = knots[i + p] - knots[i];
                double d2 = knots[i + p + 1] - knots[i + 1];
                if (d1 != 0.0) d += p * Nprev[i] / d1;
                if (d2 != 0.0) d -= p * Nprev[i + 1] / d2;
            }
            ders[i] = d;
        }
        if (p == 0)
            for (int i = 0; i < n; ++i) ders[i] = 0.0;
    }
    free(N);
    free(Nprev);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* 1D tables: composite Gauss rule on nonempty spans + local basis values.               */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int n, p, nq, ne;   /* ne = number of nonempty spans (elements) */
    int* first;         /* [ne] index of first nonzero basis function on element */
    double* node;       /* [ne*nq] */
    double* wgt;        /* [ne*nq] Gauss weight times span length / 2 */
    double* B;          /* [ne*nq*(p+1)] values of basis first..first+p */
    double* D;          /* [ne*nq*(p+1)] first derivatives */
} orc_tab1d;

static void orc_tab_free(orc_tab1d* T) {
    free(T->first); free(T->node); free(T->wgt); free(T->B); free(T->D);
    memset(T, 0, sizeof(*T));
}

static int orc_tab_build(orc_tab1d* T, const double* knots, int n, int p, int nq) {
    memset(T, 0, sizeof(*T));
    if (p < 1 || p > ORC_MAXP || n < p + 1 || nq < 1 || nq > 64) return 1;
    int m = n + p + 1;
    for (int i = 0; i + 1 < m; ++i)
        if (knots[i] > knots[i + 1]) return 1;
    int ne = 0;
    for (int s = p; s < n; ++s)
        if (knots[s] < knots[s + 1]) ++ne;
    T->n = n; T->p = p; T->nq = nq; T->ne = ne;
    T->first = (int*)malloc(sizeof(int) * (size_t)ne);
    T->node = (double*)malloc(sizeof(double) * (size_t)ne * nq);
    T->wgt = (double*)malloc(sizeof(double) * (size_t)ne * nq);
    T->B = (double*)malloc(sizeof(double) * (size_t)ne * nq * (p + 1));
    T->D = (double*)malloc(sizeof(double) * (size_t)ne * nq * (p + 1));
    double gx[64], gw[64];
    orc_gauss_legendre(nq, gx, gw);
    double* vals = (double*)malloc(sizeof(double) * (size_t)n);
    double* ders = (double*)malloc(sizeof(double) * (size_t)n);
    int e = 0;
    for (int s = p; s < n; ++s) {
        double a = knots[s], b = knots[s + 1];
        if (!(a < b)) continue;
        T->first[e] = s - p;
        for (int q = 0; q < nq; ++q) {
            double t = 0.5 * (a + b) + 0.5 * (b - a) * gx[q];
            T->node[e * nq + q] = t;
            T->wgt[e * nq + q] = 0.5 * (b - a) * gw[q];
            orc_basis_all(knots, n, p, t, vals, ders);
            for (int l = 0; l <= p; ++l) {
                T->B[(e * nq + q) * (p + 1) + l] = vals[s - p + l];
                T->D[(e * nq + q) * (p + 1) + l] = ders[s - p + l];
            }
        }
        ++e;
    }
    free(vals);
    free(ders);
    return 0;
}


/* ------------------------------------------------------------------------------------ */
/* Univariate weighted Gram (Eq. massMatrix1D / K^{(d)}_{k,l}):                          */
/*   out[i*n+j] = int beta_i^{(a)} beta_j^{(b)} (1 + amp sin(k pi t + phi)) dt           */
/* a, b in {0,1} are derivative orders on the row (i) and column (j) function.           */
/* ------------------------------------------------------------------------------------ */
int orc_gram_1d(const double* knots, int n, int p, int nq, double amp, double k, double phi,
                int a, int b, double* out) {
    orc_tab1d T;
    if (orc_tab_build(&T, knots, n, p, nq)) return 1;
    memset(out, 0, sizeof(double) * (size_t)n * n);
    for (int e = 0; e < T.ne; ++e)
        for (int q = 0; q < nq; ++q) {
            double t = T.node[e * nq + q];
            double W = T.wgt[e * nq + q] * (1.0 + amp * sin(k * M_PI * t + phi));
            const double* Bi = (a ? T.D : T.B) + (e * nq + q) * (p + 1);
            const double* Bj = (b ? T.D : T.B) + (e * nq + q) * (p + 1);
            for (int li = 0; li <= p; ++li)
                for (int lj = 0; lj <= p; ++lj)
                    out[(size_t)(T.first[e] + li) * n + (T.first[e] + lj)] += W * Bi[li] * Bj[lj];
        }
    orc_tab_free(&T);
    return 0;
}

int orc_quad_nodes(const double* knots, int n, int p, int nq, double* nodes, int64_t* count) {
    orc_tab1d T;
    if (orc_tab_build(&T, knots, n, p, nq)) return 1;
    *count = (int64_t)T.ne * nq;
    if (nodes) memcpy(nodes, T.node, sizeof(double) * (size_t)T.ne * nq);
    orc_tab_free(&T);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* 3D problem description                                                                */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    orc_tab1d T[3];          /* x, y, z */
    int lo[3], hi[3];        /* kept DoF index range per direction (Dirichlet drops ends) */
    int m[3];                /* kept extents */
    int nt_m;
    const double* terms_m;   /* mass weight terms (nt_m may be 0 => no mass) */
    int nt_q[9];
    const double* terms_q[9];/* stiffness blocks q_kl, k*3+l, k,l over x,y,z */
    /* closed-form univariate factors tabulated at the 1D nodes:
       fm[d][r*nn_d + g] = 1 + amp sin(k pi t_g + phi) of mass term r, fq[b][d][...] likewise */
    double* fm[3];
    double* fq[9][3];
    /* optional general (non-separable) weights tabulated at every tensor quadrature point:
       w3[c][gz][gy][gx], c = 0 omega, c = 1 + k*3 + l q_kl (NULL => the separable closed form) */
    const double* w3;
} orc_prob;

static int orc_prob_build(orc_prob* P, const int* n, const int* p, const double* const* knots, int nq,
                          int nt_m, const double* terms_m, const int* nt_q, const double* terms_q,
                          int dirichlet, const double* w3) {
    memset(P, 0, sizeof(*P));
    P->w3 = w3;
    for (int d = 0; d < 3; ++d) {
        if (orc_tab_build(&P->T[d], knots[d], n[d], p[d], nq)) return 1;
        if (dirichlet) {
            if (n[d] < 3) return 1;
            P->lo[d] = 1; P->hi[d] = n[d] - 2;
        } else {
            P->lo[d] = 0; P->hi[d] = n[d] - 1;
        }
        P->m[d] = P->hi[d] - P->lo[d] + 1;
    }
    P->nt_m = nt_m;
    P->terms_m = terms_m;
    size_t off = 0;
    for (int b = 0; b < 9; ++b) {
        P->nt_q[b] = nt_q ? nt_q[b] : 0;
        P->terms_q[b] = (terms_q && P->nt_q[b]) ? terms_q + off * ORC_TERM : NULL;
        off += (size_t)P->nt_q[b];
    }
    for (int d = 0; d < 3; ++d) {
        int nn = P->T[d].ne * nq;
        if (P->nt_m) {
            P->fm[d] = (double*)malloc(sizeof(double) * (size_t)P->nt_m * nn);
            for (int r = 0; r < P->nt_m; ++r) {
                const double* T = P->terms_m + (size_t)r * ORC_TERM;
                for (int g = 0; g < nn; ++g)
                    P->fm[d][(size_t)r * nn + g] =
                        1.0 + T[1 + 3 * d] * sin(T[2 + 3 * d] * M_PI * P->T[d].node[g] + T[3 + 3 * d]);
            }
        }
        for (int b = 0; b < 9; ++b) {
            if (!P->nt_q[b]) continue;
            P->fq[b][d] = (double*)malloc(sizeof(double) * (size_t)P->nt_q[b] * nn);
            for (int r = 0; r < P->nt_q[b]; ++r) {
                const double* T = P->terms_q[b] + (size_t)r * ORC_TERM;
                for (int g = 0; g < nn; ++g)
                    P->fq[b][d][(size_t)r * nn + g] =
                        1.0 + T[1 + 3 * d] * sin(T[2 + 3 * d] * M_PI * P->T[d].node[g] + T[3 + 3 * d]);
            }
        }
    }
    return 0;
}

static void orc_prob_free(orc_prob* P) {
    for (int d = 0; d < 3; ++d) {
        orc_tab_free(&P->T[d]);
        free(P->fm[d]);
        for (int b = 0; b < 9; ++b) free(P->fq[b][d]);
    }
}

/* weights at the 3D point with 1D node indices (gx,gy,gz): omega and q[9] (q[k*3+l]),
   omega(x) = sum_r coef_r f_r^x(x) f_r^y(y) f_r^z(z)  (separable closed form) */
static void orc_point_weights(const orc_prob* P, int gx, int gy, int gz, double* om, double* q) {
    const int nx = P->T[0].ne * P->T[0].nq, ny = P->T[1].ne * P->T[1].nq, nz = P->T[2].ne * P->T[2].nq;
    if (P->w3) { /* tabulated general weights (the geometry's omega and Q at the point) */
        const size_t np = (size_t)nx * ny * nz, at = ((size_t)gz * ny + gy) * nx + gx;
        *om = P->w3[at];
        for (int b = 0; b < 9; ++b) q[b] = P->w3[(size_t)(1 + b) * np + at];
        return;
    }
    double s = 0.0;
    for (int r = 0; r < P->nt_m; ++r)
        s += P->terms_m[(size_t)r * ORC_TERM] * P->fm[0][(size_t)r * nx + gx] * P->fm[1][(size_t)r * ny + gy] *
             P->fm[2][(size_t)r * nz + gz];
    *om = s;
    for (int b = 0; b < 9; ++b) {
        double t = 0.0;
        for (int r = 0; r < P->nt_q[b]; ++r)
            t += P->terms_q[b][(size_t)r * ORC_TERM] * P->fq[b][0][(size_t)r * nx + gx] *
                 P->fq[b][1][(size_t)r * ny + gy] * P->fq[b][2][(size_t)r * nz + gz];
        q[b] = t;
    }
}

/* element index range whose support contains basis function i (per direction) */
static void orc_elems_of(const orc_tab1d* T, int i, int* e0, int* e1) {
    *e0 = T->ne; *e1 = -1;
    for (int e = 0; e < T->ne; ++e)
        if (T->first[e] <= i && i <= T->first[e] + T->p) {
            if (e < *e0) *e0 = e;
            if (e > *e1) *e1 = e;
        }
}

/* ------------------------------------------------------------------------------------ */
/* CSR pattern: row i has columns j with |i_d - j_d| <= p_d for every d (within kept set) */
/* ------------------------------------------------------------------------------------ */
static int64_t orc_row_cols(const orc_prob* P, int ix, int iy, int iz, int* lo, int* w) {
    int I[3] = {ix, iy, iz};
    int64_t c = 1;
    for (int d = 0; d < 3; ++d) {
        int a = I[d] - P->T[d].p, b = I[d] + P->T[d].p;
        if (a < P->lo[d]) a = P->lo[d];
        if (b > P->hi[d]) b = P->hi[d];
        lo[d] = a;
        w[d] = b - a + 1;
        c *= w[d];
    }
    return c;
}

int64_t orc_csr_nnz(const int* n, const int* p, int dirichlet) {
    int64_t tot = 1;
    for (int d = 0; d < 3; ++d) {
        int lo = dirichlet ? 1 : 0, hi = dirichlet ? n[d] - 2 : n[d] - 1;
        int64_t s = 0;
        for (int i = lo; i <= hi; ++i) {
            int a = i - p[d], b = i + p[d];
            if (a < lo) a = lo;
            if (b > hi) b = hi;
            s += b - a + 1;
        }
        tot *= s;
    }
    return tot;
}

/*
 * Assemble M and S (either may be NULL) as CSR over the kept DoFs, row-major
 * index ((iz*my)+iy)*mx+ix.  Each row is owned by one thread and computed as
 *   M_ij = sum_{elements E} sum_{points} W omega beta_i beta_j
 *   S_ij = sum_E sum_pts W sum_kl q_kl d_l beta_i d_k beta_j
 */
int orc_assemble_csr_rows(const int* n, const int* p, const double* kx, const double* ky, const double* kz,
                          int nq, int nt_m, const double* terms_m, const int* nt_q, const double* terms_q,
                          int dirichlet, const double* w3, int64_t r0, int64_t r1, int64_t* rowptr, int32_t* colidx,
                          double* valM, double* valS);

/* rows [r0, r1) of the kept DoFs: rowptr[0..r1-r0] local to the range, global column indices */
static int orc_assemble_rows(const orc_prob* Pp, int64_t r0, int64_t r1, int nq, int64_t* rowptr, int32_t* colidx,
                             double* valM, double* valS) {
    const orc_prob P = *Pp;
    const int mx = P.m[0], my = P.m[1];
    const int64_t nrows = r1 - r0;
    /* row pointers (sequential prefix sum) */
    rowptr[0] = 0;
    for (int64_t rr = 0; rr < nrows; ++rr) {
        const int64_t r = r0 + rr;
        int ix = (int)(r % mx) + P.lo[0], iy = (int)((r / mx) % my) + P.lo[1], iz = (int)(r / ((int64_t)mx * my)) + P.lo[2];
        int lo[3], w[3];
        rowptr[rr + 1] = rowptr[rr] + orc_row_cols(&P, ix, iy, iz, lo, w);
    }
    const int px = P.T[0].p, py = P.T[1].p, pz = P.T[2].p;
    const int nqq = nq;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t rr = 0; rr < nrows; ++rr) {
        const int64_t r = r0 + rr;
        int ix = (int)(r % mx) + P.lo[0], iy = (int)((r / mx) % my) + P.lo[1], iz = (int)(r / ((int64_t)mx * my)) + P.lo[2];
        int lo[3], w[3];
        int64_t ncol = orc_row_cols(&P, ix, iy, iz, lo, w);
        int64_t base = rowptr[rr];
        for (int64_t c = 0; c < ncol; ++c) {
            int jx = lo[0] + (int)(c % w[0]), jy = lo[1] + (int)((c / w[0]) % w[1]), jz = lo[2] + (int)(c / ((int64_t)w[0] * w[1]));
            colidx[base + c] = (int32_t)((((int64_t)(jz - P.lo[2]) * my) + (jy - P.lo[1])) * mx + (jx - P.lo[0]));
            if (valM) valM[base + c] = 0.0;
            if (valS) valS[base + c] = 0.0;
        }
        int ex0, ex1, ey0, ey1, ez0, ez1;
        orc_elems_of(&P.T[0], ix, &ex0, &ex1);
        orc_elems_of(&P.T[1], iy, &ey0, &ey1);
        orc_elems_of(&P.T[2], iz, &ez0, &ez1);
        for (int ez = ez0; ez <= ez1; ++ez)
            for (int ey = ey0; ey <= ey1; ++ey)
                for (int ex = ex0; ex <= ex1; ++ex) {
                    int fx = P.T[0].first[ex], fy = P.T[1].first[ey], fz = P.T[2].first[ez];
                    for (int qz = 0; qz < nqq; ++qz)
                        for (int qy = 0; qy < nqq; ++qy)
                            for (int qx = 0; qx < nqq; ++qx) {
                                int gx = ex * nqq + qx, gy = ey * nqq + qy, gz = ez * nqq + qz;
                                double W = P.T[0].wgt[gx] * P.T[1].wgt[gy] * P.T[2].wgt[gz];
                                double om, q[9];
                                orc_point_weights(&P, gx, gy, gz, &om, q);
                                const double* Bx = P.T[0].B + (size_t)gx * (px + 1);
                                const double* By = P.T[1].B + (size_t)gy * (py + 1);
                                const double* Bz = P.T[2].B + (size_t)gz * (pz + 1);
                                const double* Dx = P.T[0].D + (size_t)gx * (px + 1);
                                const double* Dy = P.T[1].D + (size_t)gy * (py + 1);
                                const double* Dz = P.T[2].D + (size_t)gz * (pz + 1);
                                /* row function beta_i and its gradient (x,y,z) */
                                double bi = Bx[ix - fx] * By[iy - fy] * Bz[iz - fz];
                                double gi[3] = {Dx[ix - fx] * By[iy - fy] * Bz[iz - fz],
                                                Bx[ix - fx] * Dy[iy - fy] * Bz[iz - fz],
                                                Bx[ix - fx] * By[iy - fy] * Dz[iz - fz]};
                                for (int jz = fz; jz <= fz + pz; ++jz) {
                                    if (jz < P.lo[2] || jz > P.hi[2]) continue;
                                    for (int jy = fy; jy <= fy + py; ++jy) {
                                        if (jy < P.lo[1] || jy > P.hi[1]) continue;
                                        for (int jx = fx; jx <= fx + px; ++jx) {
                                            if (jx < P.lo[0] || jx > P.hi[0]) continue;
                                            int64_t c = ((int64_t)(jz - lo[2]) * w[1] + (jy - lo[1])) * w[0] + (jx - lo[0]);
                                            double bj = Bx[jx - fx] * By[jy - fy] * Bz[jz - fz];
                                            if (valM) valM[base + c] += W * om * bi * bj;
                                            if (valS) {
                                                double gj[3] = {Dx[jx - fx] * By[jy - fy] * Bz[jz - fz],
                                                                Bx[jx - fx] * Dy[jy - fy] * Bz[jz - fz],
                                                                Bx[jx - fx] * By[jy - fy] * Dz[jz - fz]};
                                                double s = 0.0;
                                                for (int k = 0; k < 3; ++k)
                                                    for (int l = 0; l < 3; ++l) s += q[k * 3 + l] * gi[l] * gj[k];
                                                valS[base + c] += W * s;
                                            }
                                        }
                                    }
                                }
                            }
                }
    }
    return 0;
}

int orc_assemble_csr(const int* n, const int* p, const double* kx, const double* ky, const double* kz,
                     int nq, int nt_m, const double* terms_m, const int* nt_q, const double* terms_q,
                     int dirichlet, const double* w3, int64_t* rowptr, int32_t* colidx, double* valM, double* valS) {
    return orc_assemble_csr_rows(n, p, kx, ky, kz, nq, nt_m, terms_m, nt_q, terms_q, dirichlet, w3, 0, -1, rowptr,
                                 colidx, valM, valS);
}

/* the same assembly restricted to the rows [r0, r1) (r1 < 0: all rows); rowptr has r1-r0+1
   entries starting at 0.  Bench samples of full-size CSR (bench.py cpu_baseline). */
int orc_assemble_csr_rows(const int* n, const int* p, const double* kx, const double* ky, const double* kz,
                          int nq, int nt_m, const double* terms_m, const int* nt_q, const double* terms_q,
                          int dirichlet, const double* w3, int64_t r0, int64_t r1, int64_t* rowptr, int32_t* colidx,
                          double* valM, double* valS) {
    const double* knots[3] = {kx, ky, kz};
    orc_prob P;
    if (orc_prob_build(&P, n, p, knots, nq, nt_m, terms_m, nt_q, terms_q, dirichlet, w3)) {
        orc_prob_free(&P);
        return 1;
    }
    const int64_t nrows = (int64_t)P.m[0] * P.m[1] * P.m[2];
    if (r1 < 0) r1 = nrows;
    int rc = 1;
    if (r0 >= 0 && r0 <= r1 && r1 <= nrows) rc = orc_assemble_rows(&P, r0, r1, nq, rowptr, colidx, valM, valS);
    orc_prob_free(&P);
    return rc;
}

/* nnz of the rows [r0, r1) */
int64_t orc_csr_rows_nnz(const int* n, const int* p, int dirichlet, int64_t r0, int64_t r1) {
    const int lo = dirichlet ? 1 : 0;
    const int m[3] = {n[0] - 2 * lo, n[1] - 2 * lo, n[2] - 2 * lo};
    int64_t tot = 0;
    for (int64_t r = r0; r < r1; ++r) {
        const int ii[3] = {(int)(r % m[0]) + lo, (int)((r / m[0]) % m[1]) + lo, (int)(r / ((int64_t)m[0] * m[1])) + lo};
        int64_t c = 1;
        for (int d = 0; d < 3; ++d) {
            const int hi = n[d] - 1 - lo;
            int a = ii[d] - p[d], b = ii[d] + p[d];
            if (a < lo) a = lo;
            if (b > hi) b = hi;
            c *= b - a + 1;
        }
        tot += c;
    }
    return tot;
}

/* OpenMP threads of the oracle's parallel loops (bench: 1 thread vs all cores) */
#include <omp.h>
void orc_set_threads(int t) { omp_set_num_threads(t > 0 ? t : omp_get_num_procs()); }
int orc_get_threads(void) { return omp_get_max_threads(); }

/* naive CSR SpMV, y = A x; rows independent */
int orc_spmv(int64_t nrows, const int64_t* rowptr, const int32_t* colidx, const double* val, const double* x,
             double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        double s = 0.0;
        for (int64_t c = rowptr[r]; c < rowptr[r + 1]; ++c) s += val[c] * x[colidx[c]];
        y[r] = s;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Bilinear-form apply.  For one element E and one point:                                */
/*   u = sum_j x_j beta_j,  grad u = sum_j x_j grad beta_j  (direct sums over E's         */
/*   (p+1)^3 functions, no factorisation), then contribution to y_i:                     */
/*   yM_i += W omega u beta_i ;  yS_i += W sum_l d_l beta_i (sum_k q_kl d_k u)           */
/* which is sum_j M_ij x_j and sum_j K_ij x_j of Eqs. (massMatrix)/(stiffnessMatrix).    */
/* ------------------------------------------------------------------------------------ */
static inline int64_t orc_kept_index(const orc_prob* P, int jx, int jy, int jz) {
    if (jx < P->lo[0] || jx > P->hi[0] || jy < P->lo[1] || jy > P->hi[1] || jz < P->lo[2] || jz > P->hi[2])
        return -1;
    return (((int64_t)(jz - P->lo[2]) * P->m[1]) + (jy - P->lo[1])) * P->m[0] + (jx - P->lo[0]);
}

/* point values for element (ex,ey,ez), point (qx,qy,qz): u, grad u; plus weights */
static void orc_point_eval(const orc_prob* P, const double* x, int ex, int ey, int ez, int qx, int qy, int qz,
                           double* W, double* om, double* q, double* u, double* gu) {
    const int nq = P->T[0].nq;
    const int px = P->T[0].p, py = P->T[1].p, pz = P->T[2].p;
    int gx = ex * nq + qx, gy = ey * nq + qy, gz = ez * nq + qz;
    *W = P->T[0].wgt[gx] * P->T[1].wgt[gy] * P->T[2].wgt[gz];
    orc_point_weights(P, gx, gy, gz, om, q);
    const double* Bx = P->T[0].B + (size_t)gx * (px + 1);
    const double* By = P->T[1].B + (size_t)gy * (py + 1);
    const double* Bz = P->T[2].B + (size_t)gz * (pz + 1);
    const double* Dx = P->T[0].D + (size_t)gx * (px + 1);
    const double* Dy = P->T[1].D + (size_t)gy * (py + 1);
    const double* Dz = P->T[2].D + (size_t)gz * (pz + 1);
    int fx = P->T[0].first[ex], fy = P->T[1].first[ey], fz = P->T[2].first[ez];
    double su = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int lz = 0; lz <= pz; ++lz)
        for (int ly = 0; ly <= py; ++ly)
            for (int lx = 0; lx <= px; ++lx) {
                int64_t j = orc_kept_index(P, fx + lx, fy + ly, fz + lz);
                if (j < 0) continue;
                double xj = x[j];
                su += xj * Bx[lx] * By[ly] * Bz[lz];
                s0 += xj * Dx[lx] * By[ly] * Bz[lz];
                s1 += xj * Bx[lx] * Dy[ly] * Bz[lz];
                s2 += xj * Bx[lx] * By[ly] * Dz[lz];
            }
    *u = su;
    gu[0] = s0; gu[1] = s1; gu[2] = s2;
}

/* contribution of point to row function (lx,ly,lz) local in element */
static inline void orc_point_test(const orc_prob* P, int ex, int ey, int ez, int qx, int qy, int qz, int lx, int ly,
                                  int lz, double W, double om, const double* q, double u, const double* gu,
                                  double* cm, double* cs) {
    const int nq = P->T[0].nq;
    const int px = P->T[0].p, py = P->T[1].p, pz = P->T[2].p;
    int gx = ex * nq + qx, gy = ey * nq + qy, gz = ez * nq + qz;
    double bx = P->T[0].B[(size_t)gx * (px + 1) + lx], by = P->T[1].B[(size_t)gy * (py + 1) + ly],
           bz = P->T[2].B[(size_t)gz * (pz + 1) + lz];
    double dx = P->T[0].D[(size_t)gx * (px + 1) + lx], dy = P->T[1].D[(size_t)gy * (py + 1) + ly],
           dz = P->T[2].D[(size_t)gz * (pz + 1) + lz];
    double gi[3] = {dx * by * bz, bx * dy * bz, bx * by * dz};
    *cm = W * om * u * (bx * by * bz);
    double s = 0.0;
    for (int l = 0; l < 3; ++l) {
        double g = 0.0;
        for (int k = 0; k < 3; ++k) g += q[k * 3 + l] * gu[k];
        s += gi[l] * g;
    }
    *cs = W * s;
}

/* full-vector apply, elements coloured (e mod (p+1) per direction): same-colour elements
   touch disjoint rows, so each y_i is summed in a fixed order. */
int orc_apply_matfree(const int* n, const int* p, const double* kx, const double* ky, const double* kz, int nq,
                      int nt_m, const double* terms_m, const int* nt_q, const double* terms_q, int dirichlet,
                      const double* w3, const double* x, double* yM, double* yS) {
    const double* knots[3] = {kx, ky, kz};
    orc_prob P;
    if (orc_prob_build(&P, n, p, knots, nq, nt_m, terms_m, nt_q, terms_q, dirichlet, w3)) {
        orc_prob_free(&P);
        return 1;
    }
    const int64_t N = (int64_t)P.m[0] * P.m[1] * P.m[2];
    if (yM) memset(yM, 0, sizeof(double) * (size_t)N);
    if (yS) memset(yS, 0, sizeof(double) * (size_t)N);
    const int px = P.T[0].p, py = P.T[1].p, pz = P.T[2].p;
    const int nex = P.T[0].ne, ney = P.T[1].ne, nez = P.T[2].ne;
    const int npts = nq * nq * nq;
    for (int cz = 0; cz <= pz; ++cz)
        for (int cy = 0; cy <= py; ++cy)
            for (int cx = 0; cx <= px; ++cx) {
                int mx = (nex - cx + px) / (px + 1), my = (ney - cy + py) / (py + 1), mz = (nez - cz + pz) / (pz + 1);
                int64_t tot = (int64_t)mx * my * mz;
#pragma omp parallel
                {
                    double* pu = (double*)malloc(sizeof(double) * (size_t)npts * 15);
#pragma omp for schedule(dynamic, 16)
                    for (int64_t t = 0; t < tot; ++t) {
                        int ex = cx + (int)(t % mx) * (px + 1);
                        int ey = cy + (int)((t / mx) % my) * (py + 1);
                        int ez = cz + (int)(t / ((int64_t)mx * my)) * (pz + 1);
                        /* evaluate at all points of the element */
                        for (int qz = 0, k = 0; qz < nq; ++qz)
                            for (int qy = 0; qy < nq; ++qy)
                                for (int qx = 0; qx < nq; ++qx, ++k) {
                                    double* s = pu + (size_t)k * 15;
                                    orc_point_eval(&P, x, ex, ey, ez, qx, qy, qz, &s[0], &s[1], &s[2], &s[11], &s[12]);
                                }
                        int fx = P.T[0].first[ex], fy = P.T[1].first[ey], fz = P.T[2].first[ez];
                        for (int lz = 0; lz <= pz; ++lz)
                            for (int ly = 0; ly <= py; ++ly)
                                for (int lx = 0; lx <= px; ++lx) {
                                    int64_t i = orc_kept_index(&P, fx + lx, fy + ly, fz + lz);
                                    if (i < 0) continue;
                                    double am = 0.0, as = 0.0;
                                    for (int qz = 0, k = 0; qz < nq; ++qz)
                                        for (int qy = 0; qy < nq; ++qy)
                                            for (int qx = 0; qx < nq; ++qx, ++k) {
                                                double* s = pu + (size_t)k * 15;
                                                double cm, cs;
                                                orc_point_test(&P, ex, ey, ez, qx, qy, qz, lx, ly, lz, s[0], s[1], &s[2],
                                                               s[11], &s[12], &cm, &cs);
                                                am += cm;
                                                as += cs;
                                            }
                                    if (yM) yM[i] += am;
                                    if (yS) yS[i] += as;
                                }
                    }
                    free(pu);
                }
            }
    orc_prob_free(&P);
    return 0;
}

/* the same bilinear form for selected rows only (kept-DoF linear indices) */
int orc_apply_rows(const int* n, const int* p, const double* kx, const double* ky, const double* kz, int nq,
                   int nt_m, const double* terms_m, const int* nt_q, const double* terms_q, int dirichlet,
                   const double* w3, const double* x, int64_t nrows, const int64_t* rows, double* yM, double* yS) {
    const double* knots[3] = {kx, ky, kz};
    orc_prob P;
    if (orc_prob_build(&P, n, p, knots, nq, nt_m, terms_m, nt_q, terms_q, dirichlet, w3)) {
        orc_prob_free(&P);
        return 1;
    }
    const int mx = P.m[0], my = P.m[1];
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t rr = 0; rr < nrows; ++rr) {
        int64_t r = rows[rr];
        int ix = (int)(r % mx) + P.lo[0], iy = (int)((r / mx) % my) + P.lo[1], iz = (int)(r / ((int64_t)mx * my)) + P.lo[2];
        int ex0, ex1, ey0, ey1, ez0, ez1;
        orc_elems_of(&P.T[0], ix, &ex0, &ex1);
        orc_elems_of(&P.T[1], iy, &ey0, &ey1);
        orc_elems_of(&P.T[2], iz, &ez0, &ez1);
        double am = 0.0, as = 0.0;
        for (int ez = ez0; ez <= ez1; ++ez)
            for (int ey = ey0; ey <= ey1; ++ey)
                for (int ex = ex0; ex <= ex1; ++ex) {
                    int lx = ix - P.T[0].first[ex], ly = iy - P.T[1].first[ey], lz = iz - P.T[2].first[ez];
                    for (int qz = 0; qz < nq; ++qz)
                        for (int qy = 0; qy < nq; ++qy)
                            for (int qx = 0; qx < nq; ++qx) {
                                double W, om, q[9], u, gu[3], cm, cs;
                                orc_point_eval(&P, x, ex, ey, ez, qx, qy, qz, &W, &om, q, &u, gu);
                                orc_point_test(&P, ex, ey, ez, qx, qy, qz, lx, ly, lz, W, om, q, u, gu, &cm, &cs);
                                am += cm;
                                as += cs;
                            }
                }
        if (yM) yM[rr] = am;
        if (yS) yS[rr] = as;
    }
    orc_prob_free(&P);
    return 0;
}
