// minres.cu — all-at-once solve of the KKT system (NEXT-1 of SURVEY §8(f)).
//
// MINRES (Paige & Saunders) on the symmetric indefinite saddle-point system of Eq. (KKTSystem)
// PAPER.md:313-319, with iga_kkt_apply as the matvec.  The paper solves the (reduced) KKT
// systems of its Block AMEn sweeps "efficiently by e.g. MINRES"; here the
// same Krylov method runs on the full dense-vector system, optionally preconditioned by the
// block-diagonal preconditioner of prec.cu.  Preconditioned recurrence of Elman, Silvester &
// Wathen, Algorithm 2.4 (P = I without a preconditioner):
//
//   v_0 = 0, w_0 = w_1 = 0, v_1 = b - A x_0, z_1 = P^{-1} v_1, gamma_1 = sqrt(z_1'v_1), gamma_0 = 1,
//   eta = gamma_1, s_0 = s_1 = 0, c_0 = c_1 = 1;  for j = 1, 2, ...
//     z_j = z_j / gamma_j;   delta_j = (A z_j)' z_j
//     v_{j+1} = A z_j - (delta_j / gamma_j) v_j - (gamma_j / gamma_{j-1}) v_{j-1}
//     z_{j+1} = P^{-1} v_{j+1};   gamma_{j+1} = sqrt(z_{j+1}' v_{j+1})
//     a0 = c_j delta_j - c_{j-1} s_j gamma_j,   a1 = sqrt(a0^2 + gamma_{j+1}^2)
//     a2 = s_j delta_j + c_{j-1} c_j gamma_j,   a3 = s_{j-1} gamma_j
//     c_{j+1} = a0 / a1,   s_{j+1} = gamma_{j+1} / a1
//     w_{j+1} = (z_j - a3 w_{j-1} - a2 w_j) / a1,   x_j = x_{j-1} + c_{j+1} eta w_{j+1}
//     eta = -s_{j+1} eta              (|eta| = |b - A x_j|_{P^{-1}} in exact arithmetic)
//
// Every vector operation is a kernel of this file (or prec.cu); the scalar recurrence runs in a
// one-thread kernel on device-resident state, so an iteration needs no host round trip except
// the convergence test (one 8-byte read of |eta|).  Dot products reduce in a fixed order over a
// fixed grid (bitwise reproducible).
#include <cmath>

#include "internal.h"

namespace igalr {
namespace {

constexpr int kDotBlocks = 148 * 4;
constexpr int kThreads = 256;

struct MinresState {
    double gamma;       // gamma_j
    double gamma_prev;  // gamma_{j-1}
    double c_prev, c, s_prev, s;
    double eta;
    double a1, a2, a3;  // this iteration's rotation coefficients
    double ceta;        // c_{j+1} * eta (before the eta update)
    double inv_gamma;   // 1 / gamma_{j+1} (0 on breakdown)
    double dots[2];     // reduction results: [0] delta_j, [1] z_{j+1}'v_{j+1} (or z_1'v_1)
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

// z_1 /= gamma_1; v_0 = w_0 = w_1 = 0
__global__ void k_start(double* __restrict__ z, double* __restrict__ v_prev, double* __restrict__ w,
                        double* __restrict__ w_prev, long long n, const MinresState* st) {
    const double s = st->inv_gamma;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        z[i] = z[i] * s;
        v_prev[i] = 0.0;
        w[i] = 0.0;
        w_prev[i] = 0.0;
    }
}

// v_{j+1} = A z_j - (delta_j / gamma_j) v_j - (gamma_j / gamma_{j-1}) v_{j-1}   (in place in A z_j)
__global__ void k_lanczos(double* __restrict__ az, const double* __restrict__ v, const double* __restrict__ v_prev,
                          long long n, const MinresState* st) {
    const double d = st->dots[0] / st->gamma, g = st->gamma / st->gamma_prev;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        az[i] = az[i] - d * v[i] - g * v_prev[i];
}

// b - A x0  (in place in the matvec output)
__global__ void k_residual0(double* __restrict__ ax, const double* __restrict__ b, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        ax[i] = b[i] - ax[i];
}

__global__ void k_init_state(MinresState* st) {
    const double g = sqrt(fmax(st->dots[1], 0.0));
    st->gamma = g;
    st->gamma_prev = 1.0;
    st->eta = g;
    st->c_prev = st->c = 1.0;
    st->s_prev = st->s = 0.0;
    st->inv_gamma = g > 0.0 ? 1.0 / g : 0.0;
}

// the scalar recurrence of one iteration (one thread)
__global__ void k_scalars(MinresState* st) {
    const double delta = st->dots[0];
    const double gn = sqrt(fmax(st->dots[1], 0.0));
    const double g = st->gamma;
    const double a0 = st->c * delta - st->c_prev * st->s * g;
    const double a1 = sqrt(a0 * a0 + gn * gn);
    const double a2 = st->s * delta + st->c_prev * st->c * g;
    const double a3 = st->s_prev * g;
    const double cn = a1 > 0.0 ? a0 / a1 : 1.0;
    const double sn = a1 > 0.0 ? gn / a1 : 0.0;
    st->a1 = a1;
    st->a2 = a2;
    st->a3 = a3;
    st->ceta = cn * st->eta;
    st->eta = -sn * st->eta;
    st->c_prev = st->c;
    st->c = cn;
    st->s_prev = st->s;
    st->s = sn;
    st->gamma_prev = g;
    st->gamma = gn;
    st->inv_gamma = gn > 0.0 ? 1.0 / gn : 0.0;
}

// w_{j+1} = (z_j - a3 w_{j-1} - a2 w_j) / a1 (into w_prev), x += c_{j+1} eta w_{j+1},
// z_{j+1} /= gamma_{j+1}
__global__ void k_update(const double* __restrict__ z, double* __restrict__ w_prev, const double* __restrict__ w,
                         double* __restrict__ x, double* __restrict__ z_next, long long n, const MinresState* st) {
    const double a1 = st->a1, a2 = st->a2, a3 = st->a3, ce = st->ceta, ig = st->inv_gamma;
    const double ia1 = a1 > 0.0 ? 1.0 / a1 : 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double wn = (z[i] - a3 * w_prev[i] - a2 * w[i]) * ia1;
        w_prev[i] = wn;
        x[i] = fma(ce, wn, x[i]);
        z_next[i] = z_next[i] * ig;
    }
}

int grid_for(long long n) {
    const long long nb = (n + kThreads - 1) / kThreads;
    return (int)(nb < 148 * 16 ? nb : 148 * 16);
}

}  // namespace
}  // namespace igalr

using namespace igalr;

extern "C" iga_status iga_kkt_minres(const iga_lr_op* op, const iga_kkt_prec* prec, int32_t n_t, double tau,
                                     double beta, const double* rhs, double* x, double rtol, int32_t maxit,
                                     uint32_t flags, void* stream, iga_minres_info* info) {
    NvtxRange nvtx_("iga_kkt_minres");
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
    if (prec && (!kkt_prec_matches(prec, op, n_t, tau, beta)))
        return set_error(IGA_EINVAL, "preconditioner was built for another op / n_t / tau / beta");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 3LL * n_t * op->m[0] * op->m[1] * op->m[2];
    const uint32_t kflags = flags & ~IGA_MINRES_X0;
    // workspace: v_prev, v, az (A z_j, then v_{j+1}), z, z_next, w_prev, w, P scratch
    double* ws = nullptr;
    const size_t vec = (size_t)n;
    const int nvec = prec ? 8 : 7;
    cudaError_t e = pool_alloc(op->pool, (void**)&ws, sizeof(double) * (nvec * vec + kDotBlocks) + sizeof(MinresState), st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(minres)");
    double* v_prev = ws;
    double* v = ws + vec;
    double* az = ws + 2 * vec;
    double* z = ws + 3 * vec;
    double* z_next = ws + 4 * vec;
    double* w_prev = ws + 5 * vec;
    double* w = ws + 6 * vec;
    double* ptmp = prec ? ws + 7 * vec : nullptr;
    double* part = ws + nvec * vec;
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
    auto precond = [&](const double* in, double* out) -> iga_status {  // out = P^{-1} in
        if (prec) return kkt_prec_apply(prec, in, out, ptmp, st);
        cudaError_t e2 = cudaMemcpyAsync(out, in, sizeof(double) * vec, cudaMemcpyDeviceToDevice, st);
        return e2 ? cuda_error(e2, "minres copy") : IGA_OK;
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
    // v_1 = b - A x_0 (x_0 = 0 unless IGA_MINRES_X0)
    if (flags & IGA_MINRES_X0) {
        s = iga_kkt_apply(op, n_t, tau, beta, x, v, kflags, stream);
        if (!s) k_residual0<<<gb, kThreads, 0, st>>>(v, rhs, n);
    } else {
        e = cudaMemcpyAsync(v, rhs, sizeof(double) * vec, cudaMemcpyDeviceToDevice, st);
        if (!e) e = cudaMemsetAsync(x, 0, sizeof(double) * vec, st);
        if (e) s = cuda_error(e, "minres init");
    }
    if (!s) s = precond(v, z);  // z_1 = P^{-1} v_1
    if (!s) {
        dot(z, v, 1);
        k_init_state<<<1, 1, 0, st>>>(S);
        k_start<<<gb, kThreads, 0, st>>>(z, v_prev, w, w_prev, n, S);
        e = cudaGetLastError();
        if (e) s = cuda_error(e, "minres start");
    }
    if (!s) s = read_eta(&res0);
    res = res0;
    while (!s && it < maxit && res > rtol * res0) {
        s = iga_kkt_apply(op, n_t, tau, beta, z, az, kflags, stream);  // A z_j
        if (s) break;
        dot(az, z, 0);                                                  // delta_j
        k_lanczos<<<gb, kThreads, 0, st>>>(az, v, v_prev, n, S);     // v_{j+1}
        s = precond(az, z_next);                                        // z_{j+1} = P^{-1} v_{j+1}
        if (s) break;
        dot(z_next, az, 1);                                             // gamma_{j+1}^2
        k_scalars<<<1, 1, 0, st>>>(S);
        k_update<<<gb, kThreads, 0, st>>>(z, w_prev, w, x, z_next, n, S);
        e = cudaGetLastError();
        if (e) {
            s = cuda_error(e, "minres iteration");
            break;
        }
        // rotate: v_prev <- v, v <- v_{j+1}; z <- z_{j+1}; w_prev <- w, w <- w_{j+1}
        double* t = v_prev;
        v_prev = v;
        v = az;
        az = t;
        t = z;
        z = z_next;
        z_next = t;
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
