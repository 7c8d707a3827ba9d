// weights.cu — low-rank separable weights from samples (NEXT-2 of SURVEY §8(f)).
//
// The step before the hot path: it turns samples of a weight function (omega = |det grad G| or
// one entry q_kl of Q) into the rank-R separable form consumed by
// iga_lr_assemble_factors, following PAPER.md:177-265:
//   1. the caller samples the weight at the Greville points of the interpolation space S~
//      (iga_greville; tensor grid X = X_x (x) X_y (x) X_z);
//   2. TT-SVD of the sample tensor omega(X) with relative accuracy eps (Oseledets; truncation
//      delta = eps |omega(X)|_F / sqrt(D-1) per unfolding), TT cores omega_d(r_{d-1}, :, r_d);
//   3. Eq. (weightEquationSolve): W = sum_{r1,r2} (x)_d B~_d(X_d)^{-1}
//      vec(omega_d(r_{d-1}, :, r_d)) — one univariate collocation solve per factor vector;
//   4. Eq. (TTranks): the R = R1 R2 canonical terms of the TT format, each
//      univariate factor w_r^(d) . beta~^(d) tabulated at the target space's quadrature nodes
//      (the iga_sep tables of Eq. (weightLowRank)).
// The paper's d = 1 is the slowest direction (z here).  Host code (setup, not the apply path);
// the SVDs are one-sided Jacobi (Hestenes), relatively accurate.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "hostla.h"
#include "internal.h"

struct iga_lowrank_weight {
    int R = 0;
    int tt[2] = {0, 0};
    std::vector<double> coef;
    std::vector<double> tab[3];
    int64_t nnodes[3] = {0, 0, 0};
    double tt_error = 0.0;  // |omega(X) - TT|_F / |omega(X)|_F (from the discarded singular values)
};

namespace igalr {
namespace {

// all p+1 nonzero B-splines at t (span s with knots[s] <= t < knots[s+1], last span closed)
int basis_at(const double* kn, int n, int p, double t, double* N) {
    int s = p;
    while (s < n - 1 && !(t < kn[s + 1])) ++s;
    while (s > p && !(kn[s] <= t)) --s;
    double left[16], right[16];
    N[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = t - kn[s + 1 - j];
        right[j] = kn[s + j] - t;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double den = right[r + 1] + left[j - r];
            const double tmp = den != 0.0 ? N[r] / den : 0.0;
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
    }
    return s - p;  // first nonzero function
}

iga_status check_dir(const iga_dir& d, const char* what) {
    if (d.p < 1 || d.p > 15 || d.n < d.p + 1 || !d.knots) return set_error(IGA_EINVAL, std::string(what) + ": bad p/n/knots");
    for (int i = 0; i + 1 < d.n + d.p + 1; ++i)
        if (!(d.knots[i] <= d.knots[i + 1])) return set_error(IGA_EINVAL, std::string(what) + ": knots decrease");
    return IGA_OK;
}

// One-sided Jacobi (Hestenes) SVD of a wide matrix A (m x n, m <= n, row-major): rotate row
// pairs until all rows are mutually orthogonal; then row k = sigma_k v_k' and A = U diag(sig) V'
// with U = J' (J the accumulated row rotations).  Relative accuracy (no Gram squaring).
void jacobi_svd_wide(std::vector<double> A, int m, int n, std::vector<double>& U, std::vector<double>& sig,
                     std::vector<double>& Vt) {
    std::vector<double> J((size_t)m * m, 0.0);
    for (int i = 0; i < m; ++i) J[(size_t)i * m + i] = 1.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int i = 0; i < m - 1; ++i)
            for (int j = i + 1; j < m; ++j) {
                double al = 0.0, be = 0.0, ga = 0.0;
                const double* ri = &A[(size_t)i * n];
                const double* rj = &A[(size_t)j * n];
                for (int c = 0; c < n; ++c) {
                    al += ri[c] * ri[c];
                    be += rj[c] * rj[c];
                    ga += ri[c] * rj[c];
                }
                if (ga == 0.0 || std::fabs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
                rotated = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
                for (int c = 0; c < n; ++c) {
                    const double x = A[(size_t)i * n + c], y = A[(size_t)j * n + c];
                    A[(size_t)i * n + c] = cs * x - sn * y;
                    A[(size_t)j * n + c] = sn * x + cs * y;
                }
                for (int c = 0; c < m; ++c) {
                    const double x = J[(size_t)i * m + c], y = J[(size_t)j * m + c];
                    J[(size_t)i * m + c] = cs * x - sn * y;
                    J[(size_t)j * m + c] = sn * x + cs * y;
                }
            }
        if (!rotated) break;
    }
    sig.assign(m, 0.0);
    for (int k = 0; k < m; ++k) {
        double s2 = 0.0;
        for (int c = 0; c < n; ++c) s2 += A[(size_t)k * n + c] * A[(size_t)k * n + c];
        sig[k] = std::sqrt(s2);
    }
    std::vector<int> ord(m);
    for (int k = 0; k < m; ++k) ord[k] = k;
    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return sig[a] > sig[b]; });
    std::vector<double> s_sorted(m);
    U.assign((size_t)m * m, 0.0);
    Vt.assign((size_t)m * n, 0.0);
    for (int q = 0; q < m; ++q) {
        const int k = ord[q];
        s_sorted[q] = sig[k];
        for (int i = 0; i < m; ++i) U[(size_t)i * m + q] = J[(size_t)k * m + i];
        for (int c = 0; c < n; ++c) Vt[(size_t)q * n + c] = sig[k] > 0.0 ? A[(size_t)k * n + c] / sig[k] : 0.0;
    }
    sig = s_sorted;
}

// truncated SVD of A (m x n, row-major): A ~= U diag(sig) Vt, rank the smallest r with
// sum_{i >= r} sig_i^2 <= delta2 (at most rmax, at least 1)
void tsvd(const std::vector<double>& A, int m, int n, double delta2, int rmax, std::vector<double>& U,
          std::vector<double>& sig, std::vector<double>& Vt, double* discarded) {
    std::vector<double> Uf, Vf, sf;
    int k;
    if (m <= n) {
        jacobi_svd_wide(A, m, n, Uf, sf, Vf);  // Uf [m][m], Vf [m][n]
        k = m;
    } else {  // A' = U' S V'' (n x m, wide)  =>  A = V'' ' S U''
        std::vector<double> At((size_t)n * m);
        for (int i = 0; i < m; ++i)
            for (int c = 0; c < n; ++c) At[(size_t)c * m + i] = A[(size_t)i * n + c];
        std::vector<double> Ut, Vtt;
        jacobi_svd_wide(At, n, m, Ut, sf, Vtt);  // Ut [n][n], Vtt [n][m]
        k = n;
        Uf.assign((size_t)m * k, 0.0);
        Vf.assign((size_t)k * n, 0.0);
        for (int q = 0; q < k; ++q) {
            for (int i = 0; i < m; ++i) Uf[(size_t)i * k + q] = Vtt[(size_t)q * m + i];
            for (int c = 0; c < n; ++c) Vf[(size_t)q * n + c] = Ut[(size_t)c * k + q];
        }
    }
    // smallest r with sum_{i >= r} sig_i^2 <= delta2, the tail summed from the smallest value up
    // (no cancellation against the leading singular values)
    int r = k;
    double tail = 0.0;
    while (r > 1 && tail + sf[r - 1] * sf[r - 1] <= delta2) {
        tail += sf[r - 1] * sf[r - 1];
        --r;
    }
    while (r > rmax) {  // rank cap
        tail += sf[r - 1] * sf[r - 1];
        --r;
    }
    *discarded = tail;
    sig.assign(sf.begin(), sf.begin() + r);
    U.assign((size_t)m * r, 0.0);
    Vt.assign(Vf.begin(), Vf.begin() + (size_t)r * n);
    for (int i = 0; i < m; ++i)
        for (int q = 0; q < r; ++q) U[(size_t)i * r + q] = Uf[(size_t)i * k + q];
}

}  // namespace
}  // namespace igalr

using namespace igalr;

extern "C" iga_status iga_greville(const iga_dir* d, double* out) {
    clear_error();
    if (!d || !out) return set_error(IGA_EINVAL, "NULL argument");
    if (iga_status s = check_dir(*d, "dir")) return s;
    for (int i = 0; i < d->n; ++i) {
        double s = 0.0;
        for (int k = 1; k <= d->p; ++k) s += d->knots[i + k];
        out[i] = s / d->p;
    }
    return IGA_OK;
}

extern "C" iga_status iga_weight_lowrank(const iga_space* target, const iga_dir* tilde, const double* samples,
                                         double eps, int32_t max_terms, iga_lowrank_weight** out) {
    clear_error();
    if (!target || !tilde || !samples || !out) return set_error(IGA_EINVAL, "NULL argument");
    *out = nullptr;
    if (!(eps >= 0.0) || !std::isfinite(eps)) return set_error(IGA_EINVAL, "eps must be finite and >= 0");
    if (max_terms < 1) return set_error(IGA_EINVAL, "max_terms < 1");
    for (int d = 0; d < 3; ++d)
        if (iga_status s = check_dir(tilde[d], "tilde")) return s;
    const int nx = tilde[0].n, ny = tilde[1].n, nz = tilde[2].n;
    // collocation matrices B~_d(X_d)[i][j] = beta~_j(greville_i)
    std::vector<double> B[3];
    for (int d = 0; d < 3; ++d) {
        const iga_dir& t = tilde[d];
        std::vector<double> g(t.n);
        iga_greville(&t, g.data());
        B[d].assign((size_t)t.n * t.n, 0.0);
        double N[16];
        for (int i = 0; i < t.n; ++i) {
            const int f0 = basis_at(t.knots, t.n, t.p, g[i], N);
            for (int k = 0; k <= t.p; ++k) B[d][(size_t)i * t.n + f0 + k] = N[k];
        }
    }
    // TT-SVD, slowest direction first: unfolding [nz, ny*nx] -> R1, then [R1*ny, nx] -> R2
    const size_t tot = (size_t)nx * ny * nz;
    double fro2 = 0.0;
    for (size_t i = 0; i < tot; ++i) {
        if (!std::isfinite(samples[i])) return set_error(IGA_EINVAL, "non-finite sample");
        fro2 += samples[i] * samples[i];
    }
    const double delta2 = eps * eps * fro2 / 2.0;  // (eps |S| / sqrt(D-1))^2, D = 3
    std::vector<double> A(samples, samples + tot), U1, s1, V1, U2, s2, V2;
    double disc1 = 0.0, disc2 = 0.0;
    tsvd(A, nz, ny * nx, delta2, max_terms, U1, s1, V1, &disc1);
    const int R1 = (int)s1.size();
    std::vector<double> C((size_t)R1 * ny * nx);  // diag(s1) V1 -> [R1*ny, nx]
    for (int r = 0; r < R1; ++r)
        for (size_t c = 0; c < (size_t)ny * nx; ++c) C[(size_t)r * ny * nx + c] = s1[r] * V1[(size_t)r * ny * nx + c];
    tsvd(C, R1 * ny, nx, delta2, std::max(1, max_terms / R1), U2, s2, V2, &disc2);
    const int R2 = (int)s2.size();
    // canonical terms (r1, r2): z U1[:, r1], y U2[(r1, :), r2], x s2[r2] V2[r2, :]
    iga_lowrank_weight* W = new iga_lowrank_weight();
    W->R = R1 * R2;
    W->tt[0] = R1;
    W->tt[1] = R2;
    W->tt_error = fro2 > 0 ? std::sqrt((disc1 + disc2) / fro2) : 0.0;
    W->coef.assign(W->R, 1.0);
    std::vector<double> nodes[3];
    for (int d = 0; d < 3; ++d) {
        int64_t nn = 0;
        if (iga_status s = iga_quad_nodes(target, d, nullptr, &nn)) {
            delete W;
            return s;
        }
        nodes[d].resize(nn);
        iga_quad_nodes(target, d, nodes[d].data(), &nn);
        W->nnodes[d] = nn;
        W->tab[d].assign((size_t)W->R * nn, 0.0);
    }
    auto tabulate = [&](int d, std::vector<double> f, double* dst) -> bool {
        std::vector<double> Bc(B[d]);
        if (!hostla::lu_solve(Bc, tilde[d].n, f)) return false;  // coefficients of the factor in S~_d
        double N[16];
        for (size_t q = 0; q < nodes[d].size(); ++q) {
            const int f0 = basis_at(tilde[d].knots, tilde[d].n, tilde[d].p, nodes[d][q], N);
            double v = 0.0;
            for (int k = 0; k <= tilde[d].p; ++k) v += f[f0 + k] * N[k];
            dst[q] = v;
        }
        return true;
    };
    bool ok = true;
    for (int r1 = 0; r1 < R1 && ok; ++r1)
        for (int r2 = 0; r2 < R2 && ok; ++r2) {
            const int r = r1 * R2 + r2;
            std::vector<double> fz(nz), fy(ny), fx(nx);
            for (int i = 0; i < nz; ++i) fz[i] = U1[(size_t)i * R1 + r1];
            for (int i = 0; i < ny; ++i) fy[i] = U2[((size_t)r1 * ny + i) * R2 + r2];
            for (int i = 0; i < nx; ++i) fx[i] = s2[r2] * V2[(size_t)r2 * nx + i];
            ok = tabulate(2, fz, &W->tab[2][(size_t)r * W->nnodes[2]]) &&
                 tabulate(1, fy, &W->tab[1][(size_t)r * W->nnodes[1]]) &&
                 tabulate(0, fx, &W->tab[0][(size_t)r * W->nnodes[0]]);
        }
    if (!ok) {
        delete W;
        return set_error(IGA_EINVAL, "singular collocation matrix (Schoenberg-Whitney fails at the Greville points)");
    }
    *out = W;
    return IGA_OK;
}

extern "C" iga_status iga_weight_lowrank_sep(const iga_lowrank_weight* w, iga_sep* sep, int32_t* tt_ranks,
                                             double* tt_error) {
    clear_error();
    if (!w || !sep) return set_error(IGA_EINVAL, "NULL argument");
    sep->R = w->R;
    sep->coef = w->coef.data();
    for (int d = 0; d < 3; ++d) sep->tab[d] = w->tab[d].data();
    if (tt_ranks) {
        tt_ranks[0] = w->tt[0];
        tt_ranks[1] = w->tt[1];
    }
    if (tt_error) *tt_error = w->tt_error;
    return IGA_OK;
}

extern "C" void iga_weight_lowrank_free(iga_lowrank_weight* w) { delete w; }
