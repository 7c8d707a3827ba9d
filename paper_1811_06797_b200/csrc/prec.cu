// prec.cu — block-diagonal KKT preconditioner from Kronecker-structured solves (NEXT-1).
//
// For Eq. (KKTSystem),  A = [[tau calM, 0, calK'], [0, tau beta calM, -tau calM],
// [calK, -tau calM, 0]]  with calM = I (x) M, calK = I (x) tau S + C (x) M, the
// preconditioner is  P = blkdiag(tau calMh, tau beta calMh, Sh)  with the Schur-complement
// approximation of Pearson, Stoll & Wathen ("matching"):
//     Sh = (1/tau) (calKh + g calMh) calMh^{-1} (calKh + g calMh)',   g = tau / sqrt(beta),
// where Mh = mbar M0, Sh0 = sbar S0 replace M and S by the unit-weight Kronecker operators
//     M0 = M0z (x) M0y (x) M0x,   S0 = K0z(x)M0y(x)M0x + M0z(x)K0y(x)M0x + M0z(x)M0y(x)K0x
// (univariate factors of Eq. (massMatrix1D) with w = 1 and the (1,1)-pattern stiffness factor,
// PAPER.md:192-196, 217-220), scaled by Rayleigh quotients of the op's own M and S on the
// smoothest mode.  Every solve is done in the fast-diagonalisation basis: per direction
// K0d V = M0d V Lambda_d with V' M0d V = I, so with W = Vz (x) Vy (x) Vx
//     M0^{-1} = W W',   (a M0 + b S0)^{-1} = W diag(1 / (a + b (lz + ly + lx))) W'.
// calKh + g calMh is block lower bidiagonal in time (diagonal D = (1+g) Mh + tau Sh0, subdiagonal
// -Mh), so Sh^{-1} = tau (calKh + g calMh)^{-T} calMh (calKh + g calMh)^{-1} becomes, in the
// transformed variables, a forward and a backward first-order recurrence per spatial point:
//     zc_k = (rc_k + mbar zc_{k-1}) / Delta,   vc_k = mbar (zc_k + vc_{k+1}) / Delta,   out = tau W vc
// with Delta = (1+g) mbar + tau sbar (lz + ly + lx).  One application = two batched
// three-mode dense transforms (W', W) plus the pointwise work.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "hostla.h"
#include "internal.h"

struct iga_kkt_prec {
    int m[3];
    int n_t;
    double tau, beta, g, mbar, sbar;
    double* dA[3];   // V_d  (row-major [m][m]: out index, in index)
    double* dAt[3];  // V_d'
    double* dlam[3];
    int device;
    cudaMemPool_t pool = nullptr;  // scratch of iga_kkt_prec_apply (kept mapped)
};

namespace igalr {
namespace {

int grid_of(long long n) {
    const long long nb = (n + 255) / 256;
    return (int)(nb < 148 * 32 ? nb : 148 * 32);
}

// ---- device kernels
// out[o][i][c] = sum_j A[i][j] in[o][j][c]  (a dense mode product along the middle index)
__global__ void k_mode(const double* __restrict__ A, const double* __restrict__ in, double* __restrict__ out,
                       long long outer, int n, long long inner) {
    const long long tot = outer * n * inner;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (long long)gridDim.x * blockDim.x) {
        const long long c = g % inner;
        const long long oi = g / inner;
        const int i = (int)(oi % n);
        const long long o = oi / n;
        const double* src = in + o * n * inner + c;
        const double* a = A + (size_t)i * n;
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc = fma(__ldg(a + j), src[(long long)j * inner], acc);
        out[g] = acc;
    }
}

// Slab form of the same product for n <= 64: one CTA per (o, 64-column chunk), A and the input
// slab staged in shared memory; warp w owns rows i = w, w+8, ..., each lane two columns.
constexpr int kSlabC = 64;
constexpr int kSlabRows = 8;  // rows per warp (n <= 64)
__global__ void __launch_bounds__(256) k_mode_slab(const double* __restrict__ A, const double* __restrict__ in,
                                                   double* __restrict__ out, long long outer, int n, long long inner) {
    extern __shared__ double sm[];
    double* As = sm;                      // [n][n+1]
    double* Is = sm + n * (n + 1);        // [n][kSlabC]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) As[(t / n) * (n + 1) + t % n] = A[t];
    const long long nchunk = (inner + kSlabC - 1) / kSlabC;
    for (long long blk = blockIdx.x; blk < outer * nchunk; blk += gridDim.x) {
        const long long o = blk / nchunk;
        const long long c0 = (blk - o * nchunk) * kSlabC;
        const int cw = (int)min((long long)kSlabC, inner - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < n * kSlabC; t += blockDim.x) {
            const int j = t / kSlabC, cc = t % kSlabC;
            Is[t] = cc < cw ? in[(o * n + j) * inner + c0 + cc] : 0.0;
        }
        __syncthreads();
        double acc[kSlabRows][2];
#pragma unroll
        for (int r = 0; r < kSlabRows; ++r) acc[r][0] = acc[r][1] = 0.0;
        for (int j = 0; j < n; ++j) {
            const double x0 = Is[j * kSlabC + lane], x1 = Is[j * kSlabC + lane + 32];
#pragma unroll
            for (int r = 0; r < kSlabRows; ++r) {
                const int i = warp + 8 * r;
                const double a = i < n ? As[i * (n + 1) + j] : 0.0;
                acc[r][0] = fma(a, x0, acc[r][0]);
                acc[r][1] = fma(a, x1, acc[r][1]);
            }
        }
#pragma unroll
        for (int r = 0; r < kSlabRows; ++r) {
            const int i = warp + 8 * r;
            if (i >= n) continue;
            double* dst = out + (o * n + i) * inner + c0;
            if (lane < cw) dst[lane] = acc[r][0];
            if (lane + 32 < cw) dst[lane + 32] = acc[r][1];
        }
    }
}

// Contiguous-line form (inner = 1, n <= 64): out[o][i] = sum_j A[i][j] in[o][j]; one CTA per 64
// lines, staged transposed (columns = lines) and written back through shared memory.
__global__ void __launch_bounds__(256) k_mode_lines(const double* __restrict__ A, const double* __restrict__ in,
                                                    double* __restrict__ out, long long outer, int n) {
    extern __shared__ double sm[];
    double* As = sm;                      // [n][n+1]
    double* Is = sm + n * (n + 1);        // [n][kSlabC]  (Is[j][line])
    double* Os = Is + n * kSlabC;         // [kSlabC][n+1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) As[(t / n) * (n + 1) + t % n] = A[t];
    const long long nblk = (outer + kSlabC - 1) / kSlabC;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long o0 = blk * kSlabC;
        const int cw = (int)min((long long)kSlabC, outer - o0);
        __syncthreads();
        for (int t = threadIdx.x; t < kSlabC * n; t += blockDim.x) {  // contiguous global reads
            const int ll = t / n, j = t % n;
            Is[j * kSlabC + ll] = ll < cw ? in[(o0 + ll) * n + j] : 0.0;
        }
        __syncthreads();
        double acc[kSlabRows][2];
#pragma unroll
        for (int r = 0; r < kSlabRows; ++r) acc[r][0] = acc[r][1] = 0.0;
        for (int j = 0; j < n; ++j) {
            const double x0 = Is[j * kSlabC + lane], x1 = Is[j * kSlabC + lane + 32];
#pragma unroll
            for (int r = 0; r < kSlabRows; ++r) {
                const int i = warp + 8 * r;
                const double a = i < n ? As[i * (n + 1) + j] : 0.0;
                acc[r][0] = fma(a, x0, acc[r][0]);
                acc[r][1] = fma(a, x1, acc[r][1]);
            }
        }
#pragma unroll
        for (int r = 0; r < kSlabRows; ++r) {
            const int i = warp + 8 * r;
            if (i >= n) continue;
            Os[lane * (n + 1) + i] = acc[r][0];
            Os[(lane + 32) * (n + 1) + i] = acc[r][1];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < cw * n; t += blockDim.x) {  // contiguous global writes
            const int ll = t / n, i = t % n;
            out[(o0 + ll) * n + i] = Os[ll * (n + 1) + i];
        }
    }
}

// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) form of the same dense mode product for n <= 64:
// the fast-diagonalisation transforms are dense n x n contractions, the one place on this path
// where a dense tile is not mostly padding (n = 46: 92 % of each 48 x 48 tile is useful).
// A CTA takes a 64-column tile X[j][c] (slab: columns of one o; LINES: 64 contiguous lines,
// staged transposed), out = A X as 8x8 tiles: warp w owns columns 8w..8w+7 and every 8-row
// tile, accumulating over k-steps of 4.  Fragments (PTX m8n8k4 .f64): a = A[l/4][l%4],
// b = X[l%4][l/4], d = D[l/4][2(l%4) + {0,1}] for lane l.
constexpr int kMmaC = 64;
template <bool LINES>
__global__ void __launch_bounds__(256, 3) k_mode_mma(const double* __restrict__ A, const double* __restrict__ in,
                                                  double* __restrict__ out, long long outer, int n, long long inner) {
    extern __shared__ double sm[];
    const int NM = (n + 7) & ~7, KN = (n + 3) & ~3;
    const int XP = kMmaC + 8;               // X pitch (== 8 mod 16 doubles)
    double* As = sm;                        // [NM/8][KN/4][32] fragment order
    double* Xs = As + NM * KN;              // [KN][XP], columns swizzled (xs below)
    double* Os = Xs + KN * XP;              // LINES: [kMmaC][n + 1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // X tile index with the column XOR-swizzled by (row/2)%8: the staging stores (16 consecutive
    // rows of one column for LINES, consecutive columns for slabs) and the B-fragment loads
    // (rows k..k+3 x 8 columns) each touch all 16 eight-byte banks once per wavefront
    auto xs = [&](int j, int c) { return j * XP + (c ^ ((j >> 1) & 7)); };
    // A in fragment order: As[(m * (KN/4) + k) * 32 + l] = A[8m + l/4][4k + l%4], so a warp's
    // fragment load is 32 consecutive doubles (no bank conflicts)
    const int KS = KN >> 2;
    for (int t = threadIdx.x; t < NM * KN; t += blockDim.x) {
        const int l = t & 31, mk = t >> 5;
        const int m = mk / KS, k = mk - m * KS;
        const int i = m * 8 + (l >> 2), j = k * 4 + (l & 3);
        As[t] = (i < n && j < n) ? A[i * n + j] : 0.0;
    }
    const long long nchunk = LINES ? (outer + kMmaC - 1) / kMmaC : (inner + kMmaC - 1) / kMmaC;
    const long long nblk = LINES ? nchunk : outer * nchunk;
    // tile coordinates: (o, c0, cw)
    auto tile = [&](long long blk, long long& o, long long& c0, int& cw) {
        if (LINES) {
            o = 0;
            c0 = blk * kMmaC;
            cw = (int)min((long long)kMmaC, outer - c0);
        } else {
            o = blk / nchunk;
            c0 = (blk - o * nchunk) * kMmaC;
            cw = (int)min((long long)kMmaC, inner - c0);
        }
    };
    // staging: all of a thread's loads (<= 16) are issued before its shared-memory stores
    constexpr int kPer = (64 * kMmaC) / 256;
    auto load = [&](long long blk, double* v) {
        long long o, c0;
        int cw;
        tile(blk, o, c0, cw);
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int t = threadIdx.x + q * 256;
            if (LINES) {
                const int ll = t / n, j = t - ll * n;
                v[q] = (t < kMmaC * n && ll < cw) ? __ldg(in + (c0 + ll) * n + j) : 0.0;
            } else {
                const int j = t / kMmaC, cc = t - j * kMmaC;
                v[q] = (t < n * kMmaC && cc < cw) ? __ldg(in + (o * n + j) * inner + c0 + cc) : 0.0;
            }
        }
    };
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        long long o, c0;
        int cw;
        tile(blk, o, c0, cw);
        double v[kPer];
        load(blk, v);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int t = threadIdx.x + q * 256;
            if (LINES) {
                const int ll = t / n, j = t - ll * n;
                if (t < kMmaC * n) Xs[xs(j, ll)] = v[q];
            } else {
                const int j = t / kMmaC, cc = t - j * kMmaC;
                if (t < n * kMmaC) Xs[xs(j, cc)] = v[q];
            }
        }
        for (int t = threadIdx.x; t < (KN - n) * kMmaC; t += blockDim.x)  // zero K padding rows
            Xs[xs(n + t / kMmaC, t % kMmaC)] = 0.0;
        __syncthreads();
        double acc[8][2];
#pragma unroll
        for (int m = 0; m < 8; ++m) acc[m][0] = acc[m][1] = 0.0;
        const int nm = NM >> 3;
        for (int k0 = 0; k0 < KN; k0 += 4) {
            const double b = Xs[xs(k0 + (lane & 3), warp * 8 + (lane >> 2))];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m < nm) {
                    const double a = As[(m * KS + (k0 >> 2)) * 32 + lane];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc[m][0]), "+d"(acc[m][1])
                                 : "d"(a), "d"(b));
                }
            }
        }
        const int col = warp * 8 + 2 * (lane & 3);
        if (LINES) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int i = m * 8 + (lane >> 2);
                if (m < nm && i < n) {
                    Os[col * (n + 1) + i] = acc[m][0];
                    Os[(col + 1) * (n + 1) + i] = acc[m][1];
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < cw * n; t += blockDim.x) {  // contiguous global writes
                const int ll = t / n, i = t - ll * n;
                out[(c0 + ll) * n + i] = Os[ll * (n + 1) + i];
            }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int i = m * 8 + (lane >> 2);
                if (m < nm && i < n) {
                    double* dst = out + (o * n + i) * inner + c0 + col;
                    if (col < cw) dst[0] = acc[m][0];
                    if (col + 1 < cw) dst[1] = acc[m][1];
                }
            }
        }
    }
}

// out = A x_d in along the middle index of [outer][n][inner]
void mode_product(const double* A, const double* in, double* out, long long outer, int n, long long inner,
                  cudaStream_t st) {
    const long long tot = outer * n * inner;
    if (n > 8 * kSlabRows) {
        k_mode<<<grid_of(tot), 256, 0, st>>>(A, in, out, outer, n, inner);
        return;
    }
    {
        // DMMA path (n <= 64)
        const int NM = (n + 7) & ~7, KN = (n + 3) & ~3;
        const size_t sm = sizeof(double) * ((size_t)NM * KN + (size_t)KN * (kMmaC + 8) +
                                            (inner == 1 ? (size_t)kMmaC * (n + 1) : 0));
        const long long nblk = inner == 1 ? (outer + kMmaC - 1) / kMmaC : outer * ((inner + kMmaC - 1) / kMmaC);
        const int grid = (int)std::min(nblk, 148LL * 8);
        if (inner == 1) {
            cudaFuncSetAttribute(k_mode_mma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_mode_mma<true><<<grid, 256, sm, st>>>(A, in, out, outer, n, inner);
        } else {
            cudaFuncSetAttribute(k_mode_mma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_mode_mma<false><<<grid, 256, sm, st>>>(A, in, out, outer, n, inner);
        }
        return;
    }
    if (inner == 1) {
        const size_t sm = sizeof(double) * ((size_t)n * (n + 1) + (size_t)n * kSlabC + (size_t)kSlabC * (n + 1));
        const long long nb = (outer + kSlabC - 1) / kSlabC;
        cudaFuncSetAttribute(k_mode_lines, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_mode_lines<<<(int)std::min(nb, 148LL * 8), 256, sm, st>>>(A, in, out, outer, n);
    } else {
        const size_t sm = sizeof(double) * ((size_t)n * (n + 1) + (size_t)n * kSlabC);
        const long long nb = outer * ((inner + kSlabC - 1) / kSlabC);
        cudaFuncSetAttribute(k_mode_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_mode_slab<<<(int)std::min(nb, 148LL * 8), 256, sm, st>>>(A, in, out, outer, n, inner);
    }
}

// pointwise part in the transformed basis: blocks y, u scaled; block lambda: the two recurrences
__global__ void k_prec_point(double* __restrict__ t, int n_t, int mx, int my, int mz, const double* __restrict__ lx,
                             const double* __restrict__ ly, const double* __restrict__ lz, double sy, double su,
                             double dconst, double dlam, double mbar, double tau) {
    const long long N = (long long)mx * my * mz;
    const long long blk = (long long)n_t * N;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(p % mx), iy = (int)((p / mx) % my), iz = (int)(p / ((long long)mx * my));
        const double delta = dconst + dlam * (lx[ix] + ly[iy] + lz[iz]);
        const double inv = 1.0 / delta;
        for (int k = 0; k < n_t; ++k) {
            t[(long long)k * N + p] *= sy;
            t[blk + (long long)k * N + p] *= su;
        }
        double* l = t + 2 * blk;
        double z = 0.0;
        for (int k = 0; k < n_t; ++k) {  // forward: zc_k = (rc_k + mbar zc_{k-1}) / Delta
            z = (l[(long long)k * N + p] + mbar * z) * inv;
            l[(long long)k * N + p] = z;
        }
        double v = 0.0;
        for (int k = n_t - 1; k >= 0; --k) {  // backward: vc_k = mbar (zc_k + vc_{k+1}) / Delta
            v = mbar * (l[(long long)k * N + p] + v) * inv;
            l[(long long)k * N + p] = tau * v;
        }
    }
}

// three mode products of W (trans = false) or W' (trans = true) on B vectors, without copies:
// in -> mid (x), mid -> res (y), res -> mid (z); the result lands in `mid`, `res` is scratch
void apply_W(const iga_kkt_prec* P, bool trans, long long B, const double* in, double* mid, double* res,
             cudaStream_t st) {
    const long long mx = P->m[0], my = P->m[1], mz = P->m[2];
    const double* const* A = trans ? P->dAt : P->dA;
    mode_product(A[0], in, mid, B * mz * my, (int)mx, 1, st);
    mode_product(A[1], mid, res, B * mz, (int)my, mx, st);
    mode_product(A[2], res, mid, B, (int)mz, my * mx, st);
}

}  // namespace

iga_status kkt_prec_apply(const iga_kkt_prec* P, const double* in, double* out, double* tmp, cudaStream_t st) {
    const long long N = (long long)P->m[0] * P->m[1] * P->m[2];
    const long long B = 3LL * P->n_t;
    apply_W(P, true, B, in, tmp, out, st);  // tmp = W' in   (out as scratch)
    k_prec_point<<<grid_of(N), 256, 0, st>>>(tmp, P->n_t, P->m[0], P->m[1], P->m[2], P->dlam[0], P->dlam[1],
                                             P->dlam[2], 1.0 / (P->tau * P->mbar),
                                             1.0 / (P->tau * P->beta * P->mbar), (1.0 + P->g) * P->mbar,
                                             P->tau * P->sbar, P->mbar, P->tau);
    // W tmp: tmp -> out (x), out -> tmp (y), tmp -> out (z); no copies
    {
        const long long mx = P->m[0], my = P->m[1], mz = P->m[2];
        mode_product(P->dA[0], tmp, out, B * mz * my, (int)mx, 1, st);
        mode_product(P->dA[1], out, tmp, B * mz, (int)my, mx, st);
        mode_product(P->dA[2], tmp, out, B, (int)mz, my * mx, st);
    }
    cudaError_t e = cudaGetLastError();
    if (e) return cuda_error(e, "kkt preconditioner");
    return IGA_OK;
}

bool kkt_prec_matches(const iga_kkt_prec* P, const iga_lr_op* op, int n_t, double tau, double beta) {
    return P->n_t == n_t && P->tau == tau && P->beta == beta && P->m[0] == op->m[0] && P->m[1] == op->m[1] &&
           P->m[2] == op->m[2];
}

}  // namespace igalr

using namespace igalr;

extern "C" iga_status iga_kkt_prec_create(const iga_lr_op* op, int32_t n_t, double tau, double beta, uint32_t flags,
                                          void* stream, iga_kkt_prec** out) {
    NvtxRange nvtx_("iga_kkt_prec_create");
    clear_error();
    if (!op || !out) return set_error(IGA_EINVAL, "NULL op/out");
    *out = nullptr;
    if (!op->has_mass || !op->has_stiff) return set_error(IGA_ESTATE, "KKT needs mass and stiffness");
    if (n_t < 1) return set_error(IGA_EINVAL, "n_t < 1");
    if (!(tau > 0.0) || !std::isfinite(tau)) return set_error(IGA_EINVAL, "tau must be > 0");
    if (!(beta > 0.0) || !std::isfinite(beta)) return set_error(IGA_EINVAL, "beta must be > 0");
    cudaStream_t st = (cudaStream_t)stream;
    iga_kkt_prec* P = new iga_kkt_prec();
    memset(P, 0, sizeof *P);
    if (cudaError_t e0 = make_pool(op->device, &P->pool)) {
        delete P;
        return cuda_error(e0, "cudaMemPoolCreate");
    }
    P->n_t = n_t;
    P->tau = tau;
    P->beta = beta;
    P->g = tau / std::sqrt(beta);
    cudaGetDevice(&P->device);
    std::vector<double> V[3], lam[3];
    for (int d = 0; d < 3; ++d) {
        const DirQuad& q = op->quad[d];
        const int m = op->m[d];
        P->m[d] = m;
        // unit-weight univariate mass (0,0) and stiffness (1,1) factors
        std::vector<std::vector<double>> tables(1, std::vector<double>(q.node.size(), 1.0));
        std::vector<FactorSpec> specs = {{0, 0, 0}, {0, 1, 1}};
        DirFactors F;
        iga_status s = assemble_dir(q, tables, specs, op->dirichlet, st, &F);
        if (s) {
            iga_kkt_prec_destroy(P);
            return s;
        }
        std::vector<double> band((size_t)2 * m * F.bw);
        cudaError_t e = cudaMemcpyAsync(band.data(), F.band, sizeof(double) * band.size(), cudaMemcpyDeviceToHost, st);
        if (!e) e = cudaStreamSynchronize(st);
        cudaFree(F.band);
        if (e) {
            iga_kkt_prec_destroy(P);
            return cuda_error(e, "prec factors D2H");
        }
        std::vector<double> M0((size_t)m * m, 0.0), K0((size_t)m * m, 0.0);
        const int p = F.p;
        for (int i = 0; i < m; ++i)
            for (int k = 0; k < F.bw; ++k) {
                const int j = i - p + k;
                if (j < 0 || j >= m) continue;
                M0[(size_t)i * m + j] = band[(size_t)i * F.bw + k];
                K0[(size_t)i * m + j] = band[((size_t)m + i) * F.bw + k];
            }
        if (!hostla::gen_eig(M0, K0, m, V[d], lam[d])) {
            iga_kkt_prec_destroy(P);
            return set_error(IGA_EINVAL, "unit-weight mass factor is not SPD");
        }
    }
    // scalings: Rayleigh quotients of the op's M and S on the smoothest mode v1 = W e_(i0,j0,k0)
    int i0[3];
    // (smallest POSITIVE eigenvalue: without Dirichlet the constant mode lies in the kernel of
    // K0d, where the stiffness quotient would be 0/0)
    for (int d = 0; d < 3; ++d) {
        const double lmax = *std::max_element(lam[d].begin(), lam[d].end());
        i0[d] = -1;
        for (int i = 0; i < (int)lam[d].size(); ++i)
            if (lam[d][i] > 1e-8 * lmax && (i0[d] < 0 || lam[d][i] < lam[d][i0[d]])) i0[d] = i;
        if (i0[d] < 0) i0[d] = 0;
    }
    const int mx = P->m[0], my = P->m[1], mz = P->m[2];
    const size_t N = (size_t)mx * my * mz;
    std::vector<double> v1(N), ym(N), ys(N);
    for (int z = 0; z < mz; ++z)
        for (int y = 0; y < my; ++y)
            for (int x = 0; x < mx; ++x)
                v1[((size_t)z * my + y) * mx + x] =
                    V[2][(size_t)z * mz + i0[2]] * V[1][(size_t)y * my + i0[1]] * V[0][(size_t)x * mx + i0[0]];
    double* dv = nullptr;
    cudaError_t e = pool_alloc(P->pool, (void**)&dv, sizeof(double) * 3 * N, st);
    if (!e) e = cudaMemcpyAsync(dv, v1.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st);
    iga_status s = IGA_OK;
    if (e) s = cuda_error(e, "prec scaling");
    if (!s) s = iga_lr_apply(op, dv, dv + N, dv + 2 * N, 1.0, 1.0, 1, flags, stream);
    if (!s) {
        e = cudaMemcpyAsync(ym.data(), dv + N, sizeof(double) * N, cudaMemcpyDeviceToHost, st);
        if (!e) e = cudaMemcpyAsync(ys.data(), dv + 2 * N, sizeof(double) * N, cudaMemcpyDeviceToHost, st);
        if (!e) e = cudaStreamSynchronize(st);
        if (e) s = cuda_error(e, "prec scaling");
    }
    if (dv) cudaFreeAsync(dv, st);
    if (s) {
        iga_kkt_prec_destroy(P);
        return s;
    }
    double vm = 0.0, vs = 0.0;
    for (size_t i = 0; i < N; ++i) {
        vm += v1[i] * ym[i];
        vs += v1[i] * ys[i];
    }
    P->mbar = vm;  // (v1' M0 v1 = 1)
    P->sbar = vs / (lam[0][i0[0]] + lam[1][i0[1]] + lam[2][i0[2]]);
    if (!(P->mbar > 0.0) || !(P->sbar > 0.0)) {
        iga_kkt_prec_destroy(P);
        return set_error(IGA_EINVAL, "preconditioner scalings are not positive");
    }
    for (int d = 0; d < 3; ++d) {
        const int m = P->m[d];
        std::vector<double> At((size_t)m * m);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) At[(size_t)i * m + j] = V[d][(size_t)j * m + i];
        e = cudaMalloc(&P->dA[d], sizeof(double) * m * m);
        if (!e) e = cudaMalloc(&P->dAt[d], sizeof(double) * m * m);
        if (!e) e = cudaMalloc(&P->dlam[d], sizeof(double) * m);
        if (!e) e = cudaMemcpyAsync(P->dA[d], V[d].data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st);
        if (!e) e = cudaMemcpyAsync(P->dAt[d], At.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st);
        if (!e) e = cudaMemcpyAsync(P->dlam[d], lam[d].data(), sizeof(double) * m, cudaMemcpyHostToDevice, st);
        if (!e) e = cudaStreamSynchronize(st);  // (At is a local)
        if (e) {
            iga_kkt_prec_destroy(P);
            return cuda_error(e, "prec upload");
        }
    }
    *out = P;
    return IGA_OK;
}

extern "C" void iga_kkt_prec_destroy(iga_kkt_prec* P) {
    if (!P) return;
    for (int d = 0; d < 3; ++d) {
        if (P->dA[d]) cudaFree(P->dA[d]);
        if (P->dAt[d]) cudaFree(P->dAt[d]);
        if (P->dlam[d]) cudaFree(P->dlam[d]);
    }
    if (P->pool) cudaMemPoolDestroy(P->pool);
    delete P;
}

extern "C" iga_status iga_kkt_prec_apply(const iga_kkt_prec* P, const double* in, double* out, void* stream) {
    NvtxRange nvtx_("iga_kkt_prec_apply");
    clear_error();
    if (!P || !in || !out) return set_error(IGA_EINVAL, "NULL argument");
    if (in == out) return set_error(IGA_EINVAL, "in and out alias");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t tot = (size_t)3 * P->n_t * P->m[0] * P->m[1] * P->m[2];
    double* tmp = nullptr;
    cudaError_t e = pool_alloc(P->pool, (void**)&tmp, sizeof(double) * tot, st);
    if (e) return cuda_error(e, "cudaMallocAsync(prec)");
    iga_status s = kkt_prec_apply(P, in, out, tmp, st);
    cudaFreeAsync(tmp, st);
    return s;
}

extern "C" iga_status iga_kkt_prec_info(const iga_kkt_prec* P, double* mbar, double* sbar, double* lam_out) {
    clear_error();
    if (!P) return set_error(IGA_EINVAL, "NULL prec");
    if (mbar) *mbar = P->mbar;
    if (sbar) *sbar = P->sbar;
    if (lam_out) {
        size_t off = 0;
        for (int d = 0; d < 3; ++d) {
            cudaError_t e = cudaMemcpy(lam_out + off, P->dlam[d], sizeof(double) * P->m[d], cudaMemcpyDeviceToHost);
            if (e) return cuda_error(e, "prec info");
            off += P->m[d];
        }
    }
    return IGA_OK;
}
