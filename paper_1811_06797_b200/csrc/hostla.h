// hostla.h — small dense host linear algebra (row-major, n up to a few hundred) shared by the
// setup code of the KKT preconditioner (prec.cu) and the low-rank weights (weights.cu).
// Setup only: never on the apply path.
#pragma once
#include <cmath>
#include <vector>

namespace igalr {
namespace hostla {

// Cholesky A = L L' (row-major, lower); false if not SPD
inline bool cholesky(std::vector<double>& a, int n) {
    for (int j = 0; j < n; ++j) {
        double d = a[j * n + j];
        for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
        if (!(d > 0.0)) return false;
        d = std::sqrt(d);
        a[j * n + j] = d;
        for (int i = j + 1; i < n; ++i) {
            double s = a[i * n + j];
            for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
            a[i * n + j] = s / d;
        }
        for (int i = 0; i < j; ++i) a[i * n + j] = 0.0;
    }
    return true;
}

// cyclic Jacobi eigen-decomposition of symmetric C (row-major, destroyed): C = Q diag(lam) Q'
inline void jacobi_eig(std::vector<double>& c, int n, std::vector<double>& q, std::vector<double>& lam) {
    q.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) q[i * n + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) (i == j ? diag : off) += c[i * n + j] * c[i * n + j];
        if (off <= 1e-32 * diag) break;
        for (int p = 0; p < n - 1; ++p)
            for (int r = p + 1; r < n; ++r) {
                const double apr = c[p * n + r];
                if (std::fabs(apr) < 1e-300) continue;
                const double theta = (c[r * n + r] - c[p * n + p]) / (2.0 * apr);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < n; ++k) {  // columns p, r
                    const double ckp = c[k * n + p], ckr = c[k * n + r];
                    c[k * n + p] = cs * ckp - sn * ckr;
                    c[k * n + r] = sn * ckp + cs * ckr;
                }
                for (int k = 0; k < n; ++k) {  // rows p, r
                    const double cpk = c[p * n + k], crk = c[r * n + k];
                    c[p * n + k] = cs * cpk - sn * crk;
                    c[r * n + k] = sn * cpk + cs * crk;
                }
                for (int k = 0; k < n; ++k) {
                    const double qkp = q[k * n + p], qkr = q[k * n + r];
                    q[k * n + p] = cs * qkp - sn * qkr;
                    q[k * n + r] = sn * qkp + cs * qkr;
                }
            }
    }
    lam.resize(n);
    for (int i = 0; i < n; ++i) lam[i] = c[i * n + i];
}

// K v = lam M v with V' M V = I:  V = L^{-T} Q,  L^{-1} K L^{-T} = Q diag(lam) Q'
inline bool gen_eig(std::vector<double> M, const std::vector<double>& K, int n, std::vector<double>& V,
             std::vector<double>& lam) {
    if (!cholesky(M, n)) return false;
    const std::vector<double>& L = M;
    std::vector<double> Y(K);  // Y = L^{-1} K  (forward substitution, column by column)
    for (int col = 0; col < n; ++col)
        for (int i = 0; i < n; ++i) {
            double s = Y[i * n + col];
            for (int k = 0; k < i; ++k) s -= L[i * n + k] * Y[k * n + col];
            Y[i * n + col] = s / L[i * n + i];
        }
    std::vector<double> C((size_t)n * n);  // C = L^{-1} Y'  (= L^{-1} K L^{-T})
    for (int col = 0; col < n; ++col)
        for (int i = 0; i < n; ++i) {
            double s = Y[col * n + i];
            for (int k = 0; k < i; ++k) s -= L[i * n + k] * C[k * n + col];
            C[i * n + col] = s / L[i * n + i];
        }
    for (int i = 0; i < n; ++i)  // symmetrise rounding
        for (int j = i + 1; j < n; ++j) C[i * n + j] = C[j * n + i] = 0.5 * (C[i * n + j] + C[j * n + i]);
    std::vector<double> Q;
    jacobi_eig(C, n, Q, lam);
    V.assign((size_t)n * n, 0.0);  // L' V = Q  (back substitution)
    for (int col = 0; col < n; ++col)
        for (int i = n - 1; i >= 0; --i) {
            double s = Q[i * n + col];
            for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * V[k * n + col];
            V[i * n + col] = s / L[i * n + i];
        }
    return true;
}

// Solve A x = b in place (LU with partial pivoting); A is destroyed.  False if singular.
inline bool lu_solve(std::vector<double>& A, int n, std::vector<double>& b) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int pr = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(A[(size_t)i * n + k]) > std::fabs(A[(size_t)pr * n + k])) pr = i;
        if (A[(size_t)pr * n + k] == 0.0) return false;
        if (pr != k) {
            for (int j = 0; j < n; ++j) std::swap(A[(size_t)k * n + j], A[(size_t)pr * n + j]);
            std::swap(b[k], b[pr]);
        }
        for (int i = k + 1; i < n; ++i) {
            const double f = A[(size_t)i * n + k] / A[(size_t)k * n + k];
            A[(size_t)i * n + k] = f;
            for (int j = k + 1; j < n; ++j) A[(size_t)i * n + j] -= f * A[(size_t)k * n + j];
            b[i] -= f * b[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= A[(size_t)i * n + j] * b[j];
        b[i] = s / A[(size_t)i * n + i];
    }
    return true;
}

}  // namespace hostla
}  // namespace igalr
