// kkt.cu — per-time-step combinations of the KKT matvec (Eq. (KKTSystem)).
//
// With calM = I (x) M and calK = I (x) tau S + C (x) M (C: 1 on the diagonal, -1 below,
// PAPER.md:316-318), the three block rows for step k = 1..n_t (y_0 = 0, lambda_{n_t+1} = 0) are
//   r_y[k]   = tau M y_k + (M + tau S)^T lambda_k - M lambda_{k+1} = M b_k + tau S^T lambda_k
//   r_u[k]   = tau beta M u_k - tau M lambda_k                   = tau M a_k
//   r_lam[k] = (M + tau S) y_k - M y_{k-1} - tau M u_k          = M c_k + tau S y_k
// with a_k = beta u_k - lambda_k,  b_k = tau y_k + lambda_k - lambda_{k+1},
//      c_k = y_k - y_{k-1} - tau u_k.  This kernel forms them as
// [b, tau*a, c] so that one mass apply over a batch of 3*n_t vectors writes (r_y, r_u, r_lam)
// = (M b, tau M a, M c) directly into the output blocks; the two stiffness terms accumulate.
#include "internal.h"

namespace igalr {

__global__ void k_kkt_combos(const double* __restrict__ in, double* __restrict__ abc, int n_t, long long N, double tau,
                             double beta) {
    const long long blk = (long long)n_t * N;
    const double* y = in;
    const double* u = in + blk;
    const double* l = in + 2 * blk;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < blk; g += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(g / N);
        const double yk = y[g], uk = u[g], lk = l[g];
        const double lnext = (k + 1 < n_t) ? l[g + N] : 0.0;
        const double yprev = (k >= 1) ? y[g - N] : 0.0;
        abc[g] = tau * yk + lk - lnext;             // b_k
        abc[blk + g] = tau * (beta * uk - lk);      // tau * a_k
        abc[2 * blk + g] = yk - yprev - tau * uk;   // c_k
    }
}

// Canonical route: the spatial operators are applied to the input blocks themselves (one mass launch
// over [y, u, lambda], one stiffness launch over [lambda, y]) and the time-step combinations are taken
// afterwards, so no launch read-modify-writes its output:
//   T = [M y, M u, M lambda, tau S^T lambda, tau S y]   ([5][n_t][N])
//   r_y[k]   = tau T0[k] + T2[k] - T2[k+1] + T3[k]
//   r_u[k]   = tau (beta T1[k] - T2[k])
//   r_lam[k] = T0[k] - T0[k-1] - tau T1[k] + T4[k]
// (the same three rows by linearity of M; y_0 = 0, lambda_{n_t+1} = 0)
__global__ void k_kkt_combine(const double* __restrict__ T, double* __restrict__ out, int n_t, long long N, double tau,
                              double beta) {
    const long long blk = (long long)n_t * N;
    const double *My = T, *Mu = T + blk, *Ml = T + 2 * blk, *Sl = T + 3 * blk, *Sy = T + 4 * blk;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < blk; g += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(g / N);
        const double my = My[g], mu = Mu[g], ml = Ml[g];
        const double mlnext = (k + 1 < n_t) ? Ml[g + N] : 0.0;
        const double myprev = (k >= 1) ? My[g - N] : 0.0;
        out[g] = ((tau * my + ml) - mlnext) + Sl[g];
        out[blk + g] = tau * (beta * mu - ml);
        out[2 * blk + g] = ((my - myprev) - tau * mu) + Sy[g];
    }
}

iga_status kkt_combine(const double* T, double* out, int n_t, int64_t N, double tau, double beta, cudaStream_t st) {
    const long long blk = (long long)n_t * N;
    const int th = 256;
    long long nb = (blk + th - 1) / th;
    k_kkt_combine<<<(int)(nb < 148 * 32 ? nb : 148 * 32), th, 0, st>>>(T, out, n_t, N, tau, beta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "k_kkt_combine");
    return IGA_OK;
}

iga_status kkt_combos(const double* in, double* abc, int n_t, int64_t N, double tau, double beta, cudaStream_t st) {
    const long long blk = (long long)n_t * N;
    const int th = 256;
    long long nb = (blk + th - 1) / th;
    k_kkt_combos<<<(int)(nb < 148 * 32 ? nb : 148 * 32), th, 0, st>>>(in, abc, n_t, N, tau, beta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "k_kkt_combos");
    return IGA_OK;
}

}  // namespace igalr
