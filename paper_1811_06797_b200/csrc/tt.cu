// tt.cu — NEXT-3: the low-rank Kronecker operators on tensor-train vectors.
//
// The paper solves its KKT systems in the TT format with Block AMEn: the
// operators stay sums of Kronecker products of the univariate factors (Eqs. (M_kron)/(K_kron)
// PAPER.md:326-331), are applied to TT cores factor by factor, and are projected onto the frame
// of Eq. (frame) as F_{!=d}^T A F_{!=d} = sum_t c_t L_t (x) A_t^(d) (x) R_t
// (Eq. (KKT_red): "assembled efficiently using the multiplication of tensor
// trains factor by factor").  Three entry points (include/iga_lr.h):
//   iga_tt_kron_apply   A v for a 3D TT v: one banded mode product per core and term;
//   iga_tt_interfaces   the per-term interfaces L_t, R_t of a site;
//   iga_tt_local_apply  the reduced-system matvec y = sum_t c_t (L_t (x) A_t^(d) (x) R_t) x.
// Everything is fp64 on the caller's stream; sums run in a fixed order (deterministic).
// Sizes here are small (TT ranks ~ tens, n ~ 10^2): the kernels are plain one-thread-per-output
// loops, bounded by launch latency rather than a roofline.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"

using namespace igalr;

namespace {

constexpr int kMaxTT = 128;  // terms per call (kernel-parameter table)

struct TermTab {
    int T;
    int fid[kMaxTT];
    double coef[kMaxTT];
};

// out[t][a][i][b] = s_t * sum_k F_{f_t}[i][k] in[t?][a][i-p+k][b]  (band storage of factor f:
// band[(f*m + i)*bw + k] = F[i][i-p+k], zero outside the matrix).  in_tstride = 0 shares the input.
__global__ void k_tt_mode(const double* __restrict__ band, int m, int p, const TermTab tab, bool use_coef,
                          const double* __restrict__ in, long long in_tstride, double* __restrict__ out, int A,
                          int B) {
    const long long per = (long long)A * m * B;
    const long long total = per * tab.T;
    const int bw = 2 * p + 1;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < total;
         id += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(id / per);
        long long r = id - t * per;
        const int a = (int)(r / ((long long)m * B));
        r -= (long long)a * m * B;
        const int i = (int)(r / B), b = (int)(r - (long long)i * B);
        const double* F = band + ((size_t)tab.fid[t] * m + i) * bw;
        const double* x = in + t * in_tstride + (long long)a * m * B + b;
        double s = 0.0;
        for (int k = 0; k < bw; ++k) {
            const int j = i - p + k;
            if (j >= 0 && j < m) s = fma(F[k], x[(long long)j * B], s);
        }
        out[id] = use_coef ? tab.coef[t] * s : s;
    }
}

// out[t][p][q] = sum_k X[k*xk + p*xp] * H[t*ht + k*hk + q*hq]   (t < T, p < P, q < Q, k < K)
__global__ void k_tt_contract(const double* __restrict__ X, long long xk, long long xp, const double* __restrict__ H,
                              long long ht, long long hk, long long hq, double* __restrict__ out, int T, int P,
                              int Q, int K) {
    const long long total = (long long)T * P * Q;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < total;
         id += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(id / ((long long)P * Q));
        const int pq = (int)(id - (long long)t * P * Q);
        const int pi = pq / Q, q = pq - pi * Q;
        double s = 0.0;
        for (int k = 0; k < K; ++k) s = fma(X[k * xk + pi * xp], H[t * ht + k * hk + q * hq], s);
        out[id] = s;
    }
}

// Z[t][a'][i][b] = sum_{b'} H[t][a'][i][b'] * S[t][b][b']     ([T][A][m][B] x [T][B][B]);
// h_tstride = 0 shares one H between the terms
__global__ void k_tt_right(const double* __restrict__ H, long long h_tstride, const double* __restrict__ S,
                           double* __restrict__ Z, int T, int A, int m, int B) {
    const long long per = (long long)A * m * B;
    const long long total = per * T;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < total;
         id += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(id / per);
        const long long r = id - t * per;
        const long long row = r / B;  // (a', i)
        const int b = (int)(r - row * B);
        const double* h = H + t * h_tstride + row * B;
        const double* sr = S + ((long long)t * B + b) * B;
        double s = 0.0;
        for (int q = 0; q < B; ++q) s = fma(h[q], sr[q], s);
        Z[id] = s;
    }
}

// Z[t][b'][i][a] ... left variant: Z[t][a][i][b'] = sum_{a'} S[t][a][a'] * H[t][a'][i][b']
__global__ void k_tt_left(const double* __restrict__ S, const double* __restrict__ H, double* __restrict__ Z, int T,
                          int A, int m, int B) {
    const long long per = (long long)A * m * B;
    const long long total = per * T;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < total;
         id += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(id / per);
        const long long r = id - t * per;
        const int a = (int)(r / ((long long)m * B));
        const long long ib = r - (long long)a * m * B;
        const double* sr = S + ((long long)t * A + a) * A;
        const double* h = H + t * per + ib;
        double s = 0.0;
        for (int q = 0; q < A; ++q) s = fma(sr[q], h[(long long)q * m * B], s);
        Z[id] = s;
    }
}

// y[id] = sum_t c_t Z[t][id]  (terms summed in order)
__global__ void k_tt_sum_terms(const double* __restrict__ Z, const TermTab tab, double* __restrict__ y, long long per) {
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < per;
         id += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < tab.T; ++t) s = fma(tab.coef[t], Z[t * per + id], s);
        y[id] = s;
    }
}

// R_t = L_t = 1 for an empty side
__global__ void k_fill(double* p, long long n, double v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

iga_status term_tab(const iga_lr_op* op, int part, int dir, TermTab* tab) {
    tab->T = 0;
    for (const KTerm& t : op->kterms) {
        if (t.part != part || t.c == 0.0) continue;
        if (tab->T >= kMaxTT) return set_error(IGA_EUNSUPPORTED, "more than 128 Kronecker terms");
        tab->fid[tab->T] = t.f[dir];
        tab->coef[tab->T] = t.c;
        ++tab->T;
    }
    if (!tab->T) return set_error(IGA_ESTATE, "op has no terms of this part");
    return IGA_OK;
}

// H = A_t^(d) applied to a core [A][m_d][B] along its physical index (all terms)
cudaError_t mode(const iga_lr_op* op, int d, const TermTab& tab, bool coef, const double* in, long long in_ts,
                 double* out, int A, int B, cudaStream_t st) {
    const long long n = (long long)tab.T * A * op->m[d] * B;
    k_tt_mode<<<grid_for(n), 256, 0, st>>>(op->F[d].band, op->m[d], op->p[d], tab, coef, in, in_ts, out, A, B);
    return cudaGetLastError();
}

// Interfaces of one side.  right(d): R_t over the directions faster than d; left(d): L_t over
// the slower ones.  Cores: z [mz][R1], y [R1][my][R2], x [R2][mx].
cudaError_t right_of_y(const iga_lr_op* op, const TermTab& tx, int R2, const double* gx, double* Rx, double* tmp,
                       cudaStream_t st) {
    // R_t[b][b'] = sum_i Gx[b][i] (Ax_t Gx)[b'][i]
    cudaError_t e = mode(op, 0, tx, false, gx, 0, tmp, R2, 1, st);
    if (e) return e;
    const int mx = op->m[0];
    k_tt_contract<<<grid_for((long long)tx.T * R2 * R2), 256, 0, st>>>(gx, 1, mx, tmp, (long long)R2 * mx, 1, mx, Rx,
                                                                        tx.T, R2, R2, mx);
    return cudaGetLastError();
}
cudaError_t left_of_y(const iga_lr_op* op, const TermTab& tz, int R1, const double* gz, double* Lz, double* tmp,
                      cudaStream_t st) {
    // L_t[a][a'] = sum_i Gz[i][a] (Az_t Gz)[i][a']
    cudaError_t e = mode(op, 2, tz, false, gz, 0, tmp, 1, R1, st);
    if (e) return e;
    const int mz = op->m[2];
    k_tt_contract<<<grid_for((long long)tz.T * R1 * R1), 256, 0, st>>>(gz, R1, 1, tmp, (long long)mz * R1, R1, 1, Lz,
                                                                        tz.T, R1, R1, mz);
    return cudaGetLastError();
}

iga_status check_op(const iga_lr_op* op, int part) {
    if (!op) return set_error(IGA_EINVAL, "op is NULL");
    if (part != 0 && part != 1) return set_error(IGA_EINVAL, "part must be 0 (mass) or 1 (stiffness)");
    if (part == 0 && !op->has_mass) return set_error(IGA_ESTATE, "op has no mass part");
    if (part == 1 && !op->has_stiff) return set_error(IGA_ESTATE, "op has no stiffness part");
    return IGA_OK;
}

}  // namespace

extern "C" {

iga_status iga_lr_terms(const iga_lr_op* op, int32_t part, int32_t* n_terms, int32_t* fid, double* coef) {
    if (iga_status s = check_op(op, part)) return s;
    if (!n_terms) return set_error(IGA_EINVAL, "n_terms is NULL");
    int T = 0;
    for (const KTerm& t : op->kterms) {
        if (t.part != part || t.c == 0.0) continue;
        if (fid)
            for (int d = 0; d < 3; ++d) fid[T * 3 + d] = t.f[d];
        if (coef) coef[T] = t.c;
        ++T;
    }
    *n_terms = T;
    return IGA_OK;
}

iga_status iga_tt_kron_apply(const iga_lr_op* op, int32_t part, int32_t R1, int32_t R2, const double* gz,
                             const double* gy, const double* gx, double* wz, double* wy, double* wx, void* stream) {
    NvtxRange nvtx_("iga_tt_kron_apply");
    if (iga_status s = check_op(op, part)) return s;
    if (R1 < 1 || R2 < 1) return set_error(IGA_EINVAL, "TT ranks must be >= 1");
    if (!gz || !gy || !gx || !wz || !wy || !wx) return set_error(IGA_EINVAL, "NULL core pointer");
    cudaStream_t st = (cudaStream_t)stream;
    TermTab tx, ty, tz;
    if (iga_status s = term_tab(op, part, 0, &tx)) return s;
    term_tab(op, part, 1, &ty);
    term_tab(op, part, 2, &tz);
    cudaError_t e = mode(op, 2, tz, true, gz, 0, wz, 1, R1, st);  // c_t Az_t Gz
    if (!e) e = mode(op, 1, ty, false, gy, 0, wy, R1, R2, st);      // Ay_t Gy
    if (!e) e = mode(op, 0, tx, false, gx, 0, wx, R2, 1, st);       // Ax_t Gx
    if (e) return cuda_error(e, "iga_tt_kron_apply");
    return IGA_OK;
}

iga_status iga_tt_interfaces(const iga_lr_op* op, int32_t part, int32_t site, int32_t R1, int32_t R2,
                             const double* gz, const double* gy, const double* gx, double* L, double* R,
                             void* stream) {
    NvtxRange nvtx_("iga_tt_interfaces");
    if (iga_status s = check_op(op, part)) return s;
    if (R1 < 1 || R2 < 1) return set_error(IGA_EINVAL, "TT ranks must be >= 1");
    if (site < 0 || site > 2) return set_error(IGA_EINVAL, "site must be 0 (x), 1 (y) or 2 (z)");
    if (!gz || !gy || !gx || !L || !R) return set_error(IGA_EINVAL, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    TermTab tx, ty, tz;
    if (iga_status s = term_tab(op, part, 0, &tx)) return s;
    term_tab(op, part, 1, &ty);
    term_tab(op, part, 2, &tz);
    const int T = tx.T, mx = op->m[0], my = op->m[1], mz = op->m[2];
    // scratch: mode products of a core (largest: [T][R1][my][R2]) and one contraction stage
    const size_t big = (size_t)T * R1 * my * R2;
    const size_t small = (size_t)T * (size_t)std::max({R1 * R1, R2 * R2, R2 * mx, R1 * mz});
    double *s1 = nullptr, *s2 = nullptr, *s3 = nullptr;
    cudaError_t e = pool_alloc(op->pool, (void**)&s1, sizeof(double) * big, st);
    if (!e) e = pool_alloc(op->pool, (void**)&s2, sizeof(double) * big, st);
    if (!e) e = pool_alloc(op->pool, (void**)&s3, sizeof(double) * small, st);
    if (!e) {
        if (site == 1) {  // L over z, R over x
            e = left_of_y(op, tz, R1, gz, L, s3, st);
            if (!e) e = right_of_y(op, tx, R2, gx, R, s3, st);
        } else if (site == 2) {  // L = 1; R over (y, x): R_t[a][a'] = sum_{iy,b} Gy[a][iy][b] Z_t[a'][iy][b]
            k_fill<<<grid_for(T), 256, 0, st>>>(L, T, 1.0);
            double* Rx = s3;  // [T][R2][R2]
            double* tx_buf = nullptr;  // the x mode product [T][R2][mx]
            e = pool_alloc(op->pool, (void**)&tx_buf, sizeof(double) * (size_t)T * R2 * mx, st);
            if (!e) e = right_of_y(op, tx, R2, gx, Rx, tx_buf, st);
            if (!e) e = mode(op, 1, ty, false, gy, 0, s1, R1, R2, st);  // Hy[t][a'][iy][b']
            if (!e) {
                k_tt_right<<<grid_for((long long)big), 256, 0, st>>>(s1, (long long)R1 * my * R2, Rx, s2, T, R1, my,
                                                                     R2);  // Z[t][a'][iy][b]
                e = cudaGetLastError();
            }
            if (!e) {
                const long long K = (long long)my * R2;
                k_tt_contract<<<grid_for((long long)T * R1 * R1), 256, 0, st>>>(gy, 1, K, s2, (long long)R1 * K, 1, K,
                                                                                  R, T, R1, R1, (int)K);
                e = cudaGetLastError();
            }
            if (tx_buf) cudaFreeAsync(tx_buf, st);
        } else {  // site x: R = 1; L over (z, y): L_t[b][b'] = sum_{a,iy} Gy[a][iy][b] Z_t[a][iy][b']
            k_fill<<<grid_for(T), 256, 0, st>>>(R, T, 1.0);
            double* Lz = s3;  // [T][R1][R1]
            double* tz_buf = nullptr;
            e = pool_alloc(op->pool, (void**)&tz_buf, sizeof(double) * (size_t)T * R1 * mz, st);
            if (!e) e = left_of_y(op, tz, R1, gz, Lz, tz_buf, st);
            if (!e) e = mode(op, 1, ty, false, gy, 0, s1, R1, R2, st);  // Hy[t][a'][iy][b']
            if (!e) {
                k_tt_left<<<grid_for((long long)big), 256, 0, st>>>(Lz, s1, s2, T, R1, my, R2);  // Z[t][a][iy][b']
                e = cudaGetLastError();
            }
            if (!e) {
                const long long K = (long long)R1 * my;  // (a, iy)
                k_tt_contract<<<grid_for((long long)T * R2 * R2), 256, 0, st>>>(gy, R2, 1, s2, K * R2, R2, 1, L, T,
                                                                                  R2, R2, (int)K);
                e = cudaGetLastError();
            }
            if (tz_buf) cudaFreeAsync(tz_buf, st);
        }
    }
    if (s1) cudaFreeAsync(s1, st);
    if (s2) cudaFreeAsync(s2, st);
    if (s3) cudaFreeAsync(s3, st);
    if (e) return cuda_error(e, "iga_tt_interfaces");
    return IGA_OK;
}

iga_status iga_tt_local_apply(const iga_lr_op* op, int32_t part, int32_t site, int32_t Rl, int32_t Rr,
                              const double* L, const double* R, const double* x, double* y, void* stream) {
    NvtxRange nvtx_("iga_tt_local_apply");
    if (iga_status s = check_op(op, part)) return s;
    if (Rl < 1 || Rr < 1) return set_error(IGA_EINVAL, "ranks must be >= 1");
    if (site < 0 || site > 2) return set_error(IGA_EINVAL, "site must be 0 (x), 1 (y) or 2 (z)");
    if (!L || !R || !x || !y) return set_error(IGA_EINVAL, "NULL pointer");
    if (x == y) return set_error(IGA_EINVAL, "x and y alias");
    cudaStream_t st = (cudaStream_t)stream;
    TermTab tab;
    if (iga_status s = term_tab(op, part, site, &tab)) return s;
    const int m = op->m[site], T = tab.T;
    const size_t per = (size_t)Rl * m * Rr;
    double *a = nullptr, *b = nullptr;
    cudaError_t e = pool_alloc(op->pool, (void**)&a, sizeof(double) * per * T, st);
    if (!e) e = pool_alloc(op->pool, (void**)&b, sizeof(double) * per * T, st);
    if (!e) {
        // a[t][r'][j][s] = sum_{s'} R_t[s][s'] x[r'][j][s']   (x shared by all terms)
        k_tt_right<<<grid_for((long long)per * T), 256, 0, st>>>(x, 0, R, a, T, Rl, m, Rr);
        e = cudaGetLastError();
        // b[t] = A_t^(d) a[t] along the physical index
        if (!e) e = mode(op, site, tab, false, a, (long long)per, b, Rl, Rr, st);
        // c[t][r][i][s] = sum_{r'} L_t[r][r'] b[t][r'][i][s] (into a), then y = sum_t c_t c[t]
        if (!e) {
            k_tt_left<<<grid_for((long long)per * T), 256, 0, st>>>(L, b, a, T, Rl, m, Rr);
            e = cudaGetLastError();
        }
        if (!e) {
            k_tt_sum_terms<<<grid_for((long long)per), 256, 0, st>>>(a, tab, y, (long long)per);
            e = cudaGetLastError();
        }
    }
    if (a) cudaFreeAsync(a, st);
    if (b) cudaFreeAsync(b, st);
    if (e) return cuda_error(e, "iga_tt_local_apply");
    return IGA_OK;
}

}  // extern "C"
