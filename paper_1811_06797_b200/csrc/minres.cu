// minres.cu — all-at-once solve of the KKT system (NEXT-1 of SURVEY §8(f)).
//
// MINRES (Paige & Saunders) on the symmetric indefinite saddle-point system of Eq. (KKTSystem)
// PAPER.md:313-319, with iga_kkt_apply as the matvec.  The paper solves the (reduced) KKT
// systems of its Block AMEn sweeps "efficiently by e.g. MINRES"; here the
// same Krylov method runs on the full dense-vector system.  Unpreconditioned form of the
// Lanczos-based recurrence (Elman, Silvester & Wathen, Algorithm 2.4 with P = I):
//
//   q_0 = 0, r_0 = b - A x_0, gamma_1 = |r_0|, q_1 = r_0 / gamma_1, eta = gamma_1,
//   c_0 = c_1 = 1, s_0 = s_1 = 0, w_0 = w_1 = 0;  for j = 1, 2, ...
//     delta_j = q_j' A q_j
//     r = A q_j - delta_j q_j - gamma_j q_{j-1},   gamma_{j+1} = |r|,   q_{j+1} = r / gamma_{j+1}
//     a0 = c_j delta_j - c_{j-1} s_j gamma_j,   a1 = sqrt(a0^2 + gamma_{j+1}^2)
//     a2 = s_j delta_j + c_{j-1} c_j gamma_j,   a3 = s_{j-1} gamma_j
//     c_{j+1} = a0 / a1,   s_{j+1} = gamma_{j+1} / a1
//     w_{j+1} = (q_j - a3 w_{j-1} - a2 w_j) / a1,   x_j = x_{j-1} + c_{j+1} eta w_{j+1}
//     eta = -s_{j+1} eta                      (|eta| = |b - A x_j| in exact arithmetic)
//
// Every vector operation is a kernel of this file; the scalar recurrence runs in a one-thread
// kernel on device-resident state, so an iteration needs no host round trip except the
// convergence test (one 8-byte read of |eta|).  Dot products reduce in a fixed order over a
// fixed grid (bitwise reproducible).
#include <cmath>

#include "internal.h"

namespace igalr {
namespace {

constexpr int kDotBlocks = 148 * 4;
constexpr int kThreads = 256;

struct MinresState {
    double gamma;       // gamma_j
    double gamma_next;  // gamma_{j+1}
    double delta;       // delta_j
    double c_prev, c, s_prev, s;
    double eta;
    double a1, a2, a3;  // this iteration's rotation coefficients
    double ceta;        // c_{j+1} * eta (before the eta update)
    double inv_gamma;   // 1 / gamma_{j+1} (0 on breakdown)
    double dots[2];     // reduction results: [0] delta, [1] gamma_{j+1}^2 (or |r_0|^2)
};

// Partial dot products: grid-stride accumulation (fixed per-thread order), fixed-tree block sum.
__global__ void __launch_bounds__(kThreads) k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                         long long n, double* __restrict__ part) {
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s = fma(a[i], b[i], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(kThreads) k_dot_final(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// y = x * s (s from device memory); optional: q_prev = 0, w = w_prev = 0
__global__ void k_start(const double* __restrict__ r, double* __restrict__ q, double* __restrict__ q_prev,
                        double* __restrict__ w, double* __restrict__ w_prev, long long n, const MinresState* st) {
    const double s = st->inv_gamma;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        q[i] = r[i] * s;
        q_prev[i] = 0.0;
        w[i] = 0.0;
        w_prev[i] = 0.0;
    }
}

// r = Aq - delta q - gamma q_prev   (in place in the matvec output)
__global__ void k_lanczos(double* __restrict__ aq, const double* __restrict__ q, const double* __restrict__ q_prev,
                          long long n, const MinresState* st) {
    const double d = st->dots[0], g = st->gamma;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        aq[i] = aq[i] - d * q[i] - g * q_prev[i];
}

// b - A x0  (in place in the matvec output)
__global__ void k_residual0(double* __restrict__ ax, const double* __restrict__ b, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        ax[i] = b[i] - ax[i];
}

__global__ void k_init_state(MinresState* st) {
    const double g = sqrt(st->dots[1]);
    st->gamma = g;
    st->eta = g;
    st->c_prev = st->c = 1.0;
    st->s_prev = st->s = 0.0;
    st->inv_gamma = g > 0.0 ? 1.0 / g : 0.0;
}

// the scalar recurrence of one iteration (one thread)
__global__ void k_scalars(MinresState* st) {
    const double delta = st->dots[0];
    const double gn = sqrt(st->dots[1]);
    const double g = st->gamma;
    const double a0 = st->c * delta - st->c_prev * st->s * g;
    const double a1 = sqrt(a0 * a0 + gn * gn);
    const double a2 = st->s * delta + st->c_prev * st->c * g;
    const double a3 = st->s_prev * g;
    const double cn = a1 > 0.0 ? a0 / a1 : 1.0;
    const double sn = a1 > 0.0 ? gn / a1 : 0.0;
    st->delta = delta;
    st->gamma_next = gn;
    st->a1 = a1;
    st->a2 = a2;
    st->a3 = a3;
    st->ceta = cn * st->eta;
    st->eta = -sn * st->eta;
    st->c_prev = st->c;
    st->c = cn;
    st->s_prev = st->s;
    st->s = sn;
    st->gamma = gn;
    st->inv_gamma = gn > 0.0 ? 1.0 / gn : 0.0;
}

// w_new = (q - a3 w_prev - a2 w) / a1 (into w_prev), x += c_{j+1} eta w_new, r /= gamma_{j+1}
__global__ void k_update(const double* __restrict__ q, double* __restrict__ w_prev, const double* __restrict__ w,
                         double* __restrict__ x, double* __restrict__ r, long long n, const MinresState* st) {
    const double a1 = st->a1, a2 = st->a2, a3 = st->a3, ce = st->ceta, ig = st->inv_gamma;
    const double ia1 = a1 > 0.0 ? 1.0 / a1 : 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double wn = (q[i] - a3 * w_prev[i] - a2 * w[i]) * ia1;
        w_prev[i] = wn;
        x[i] = fma(ce, wn, x[i]);
        r[i] = r[i] * ig;
    }
}

int grid_for(long long n) {
    const long long nb = (n + kThreads - 1) / kThreads;
    return (int)(nb < 148 * 16 ? nb : 148 * 16);
}

}  // namespace
}  // namespace igalr

using namespace igalr;

extern "C" iga_status iga_kkt_minres(const iga_lr_op* op, int32_t n_t, double tau, double beta, const double* rhs,
                                     double* x, double rtol, int32_t maxit, uint32_t flags, void* stream,
                                     iga_minres_info* info) {
    clear_error();
    if (!op) return set_error(IGA_EINVAL, "op is NULL");
    if (!rhs || !x) return set_error(IGA_EINVAL, "NULL rhs/x");
    if (rhs == x) return set_error(IGA_EINVAL, "rhs and x alias");
    if (maxit < 0) return set_error(IGA_EINVAL, "maxit < 0");
    if (!(rtol >= 0.0) || !std::isfinite(rtol)) return set_error(IGA_EINVAL, "rtol must be finite and >= 0");
    if (!op->has_mass || !op->has_stiff) return set_error(IGA_ESTATE, "KKT needs mass and stiffness");
    if (n_t < 1) return set_error(IGA_EINVAL, "n_t < 1");
    if (!(tau > 0.0) || !std::isfinite(tau)) return set_error(IGA_EINVAL, "tau must be > 0");
    if (!(beta > 0.0) || !std::isfinite(beta)) return set_error(IGA_EINVAL, "beta must be > 0");
    if ((((uintptr_t)rhs) & 7) || (((uintptr_t)x) & 7)) return set_error(IGA_EINVAL, "rhs/x not 8-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 3LL * n_t * op->m[0] * op->m[1] * op->m[2];
    const uint32_t kflags = flags & ~IGA_MINRES_X0;
    // workspace: q_prev, q, r (matvec output), w_prev, w  + dot partials + state
    double* ws = nullptr;
    const size_t vec = (size_t)n;
    cudaError_t e = cudaMallocAsync(&ws, sizeof(double) * (5 * vec + kDotBlocks) + sizeof(MinresState), st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(minres)");
    double* q_prev = ws;
    double* q = ws + vec;
    double* r = ws + 2 * vec;
    double* w_prev = ws + 3 * vec;
    double* w = ws + 4 * vec;
    double* part = ws + 5 * vec;
    MinresState* S = reinterpret_cast<MinresState*>(part + kDotBlocks);
    double* pinned = nullptr;
    iga_status s = IGA_OK;
    int it = 0;
    double res0 = 0.0, res = 0.0;
    const int gb = grid_for(n);
    auto dot = [&](const double* a, const double* b, int slot) {
        k_dot_partial<<<kDotBlocks, kThreads, 0, st>>>(a, b, n, part);
        k_dot_final<<<1, kThreads, 0, st>>>(part, kDotBlocks, &S->dots[slot]);
    };
    auto read_eta = [&](double* out) -> iga_status {
        cudaError_t e2 = cudaMemcpyAsync(pinned, &S->eta, sizeof(double), cudaMemcpyDeviceToHost, st);
        if (!e2) e2 = cudaStreamSynchronize(st);
        if (e2) return cuda_error(e2, "minres |eta| read");
        *out = fabs(*pinned);
        return IGA_OK;
    };
    e = cudaMallocHost(&pinned, sizeof(double));
    if (e != cudaSuccess) {
        cudaFreeAsync(ws, st);
        return cuda_error(e, "cudaMallocHost(minres)");
    }
    // r_0 = b - A x_0 (x_0 = 0 unless IGA_MINRES_X0)
    if (flags & IGA_MINRES_X0) {
        s = iga_kkt_apply(op, n_t, tau, beta, x, r, kflags, stream);
        if (!s) k_residual0<<<gb, kThreads, 0, st>>>(r, rhs, n);
    } else {
        e = cudaMemcpyAsync(r, rhs, sizeof(double) * vec, cudaMemcpyDeviceToDevice, st);
        if (!e) e = cudaMemsetAsync(x, 0, sizeof(double) * vec, st);
        if (e) s = cuda_error(e, "minres init");
    }
    if (!s) {
        dot(r, r, 1);
        k_init_state<<<1, 1, 0, st>>>(S);
        k_start<<<gb, kThreads, 0, st>>>(r, q, q_prev, w, w_prev, n, S);
        e = cudaGetLastError();
        if (e) s = cuda_error(e, "minres start");
    }
    if (!s) s = read_eta(&res0);
    res = res0;
    while (!s && it < maxit && res > rtol * res0) {
        s = iga_kkt_apply(op, n_t, tau, beta, q, r, kflags, stream);  // r = A q_j
        if (s) break;
        dot(r, q, 0);                                                   // delta_j
        k_lanczos<<<gb, kThreads, 0, st>>>(r, q, q_prev, n, S);       // r -= delta q + gamma q_prev
        dot(r, r, 1);                                                   // gamma_{j+1}^2
        k_scalars<<<1, 1, 0, st>>>(S);
        k_update<<<gb, kThreads, 0, st>>>(q, w_prev, w, x, r, n, S);  // w_{j+1}, x_j, q_{j+1} (in r)
        e = cudaGetLastError();
        if (e) {
            s = cuda_error(e, "minres iteration");
            break;
        }
        // rotate: q_prev <- q, q <- q_{j+1}, r <- free; w_prev <- w, w <- w_{j+1}
        double* t = q_prev;
        q_prev = q;
        q = r;
        r = t;
        t = w_prev;
        w_prev = w;
        w = t;
        ++it;
        s = read_eta(&res);
    }
    cudaFreeAsync(ws, st);
    cudaStreamSynchronize(st);
    cudaFreeHost(pinned);
    if (info) {
        info->iters = it;
        info->res0 = res0;
        info->relres = res0 > 0.0 ? res / res0 : 0.0;
        info->converged = (res <= rtol * res0) ? 1 : 0;
    }
    return s;
}
