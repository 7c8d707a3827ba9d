// apply_unfused.cu — reference GPU path: one launch per mode-product stage through HBM.
//
// Evaluates  y_part = sum over plan rounds of  F^z (x) [ sum_pairs c F^y (x) F^x ] x
// (Eqs. (massFinal)/(stiffnessFinal)) with the shared-prefix plan:
//   stage X: t_e = F^x_e  ._x  x_slot(e)          (one thread per point, all x-entries)
//   stage Y: u_j = F^y_j  ._y  t_{px(j)}          (one thread per point, all pairs)
//   stage Z: y  += sum_g scale F^z_g ._z (sum_e c_e u_e)
// Scratch is stream-ordered (cudaMallocAsync).  Deterministic: fixed summation order, no
// atomics.  Used as the correctness baseline and as the fallback for plans the fused kernel
// does not support.
#include "internal.h"

namespace igalr {

struct Dims {
    int mx, my, mz;
    long long N;  // mx*my*mz
};

__global__ void k_stage_x(Round rd, const double* __restrict__ in0, const double* __restrict__ in1,
                          const double* __restrict__ bandx, int p, Dims d, int batch, double* __restrict__ T) {
    const long long tot = d.N * batch;
    const int bw = 2 * p + 1;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(g % d.mx);
        const long long line = g - ix;  // start of the x-line
        for (int e = 0; e < rd.nx; ++e) {
            const double* src = (rd.xslot[e] ? in1 : in0) + line;
            const double* F = bandx + ((size_t)rd.xf[e] * d.mx + ix) * bw;
            double acc = 0.0;
            for (int k = 0; k < bw; ++k) {
                const int j = ix - p + k;
                if (j >= 0 && j < d.mx) acc += F[k] * src[j];
            }
            T[(size_t)e * tot + g] = acc;
        }
    }
}

__global__ void k_stage_y(Round rd, const double* __restrict__ T, const double* __restrict__ bandy, int p, Dims d,
                          int batch, double* __restrict__ U) {
    const long long tot = d.N * batch;
    const int bw = 2 * p + 1;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (long long)gridDim.x * blockDim.x) {
        const int iy = (int)((g / d.mx) % d.my);
        const long long base = g - (long long)iy * d.mx;
        for (int j = 0; j < rd.np; ++j) {
            const double* src = T + (size_t)rd.px[j] * tot + base;
            const double* F = bandy + ((size_t)rd.pf[j] * d.my + iy) * bw;
            double acc = 0.0;
            for (int k = 0; k < bw; ++k) {
                const int jj = iy - p + k;
                if (jj >= 0 && jj < d.my) acc += F[k] * src[(long long)jj * d.mx];
            }
            U[(size_t)j * tot + g] = acc;
        }
    }
}

__global__ void k_stage_z(Round rd, const double* __restrict__ U, const double* __restrict__ bandz, int p, Dims d,
                          int batch, OutMap om, int accumulate) {
    const long long tot = d.N * batch;
    const int bw = 2 * p + 1;
    const long long plane = (long long)d.mx * d.my;
    const bool same = om.dst[0] == om.dst[1];
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (long long)gridDim.x * blockDim.x) {
        const int iz = (int)((g / plane) % d.mz);
        const long long base = g - (long long)iz * plane;
        double acc[2] = {0.0, 0.0};
        for (int gi = 0; gi < rd.ng; ++gi) {
            const double* F = bandz + ((size_t)rd.gf[gi] * d.mz + iz) * bw;
            double s = 0.0;
            for (int k = 0; k < bw; ++k) {
                const int jz = iz - p + k;
                if (jz < 0 || jz >= d.mz) continue;
                double v = 0.0;
                for (int e = 0; e < rd.ne[gi]; ++e) v += rd.ec[gi][e] * U[(size_t)rd.ep[gi][e] * tot + base + (long long)jz * plane];
                s += F[k] * v;
            }
            const int part = rd.gpart[gi];
            acc[same ? 0 : part] += om.scale[part] * s;
        }
        if (same) {
            if (om.dst[0]) om.dst[0][g] = (accumulate ? om.dst[0][g] : 0.0) + acc[0];
        } else {
            for (int part = 0; part < 2; ++part)
                if (om.dst[part]) om.dst[part][g] = (accumulate ? om.dst[part][g] : 0.0) + acc[part];
        }
    }
}

__global__ void k_zero(double* a, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) a[i] = 0.0;
}

iga_status apply_unfused(const iga_lr_op* op, const Plan& pl, const OutMap& om, int batch, cudaStream_t st) {
    Dims d{op->m[0], op->m[1], op->m[2], (long long)op->m[0] * op->m[1] * op->m[2]};
    const long long tot = d.N * batch;
    double* T = nullptr;
    double* U = nullptr;
    cudaError_t e = pool_alloc(op->pool, (void**)&T, sizeof(double) * (size_t)tot * kMaxX, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(T)");
    e = pool_alloc(op->pool, (void**)&U, sizeof(double) * (size_t)tot * kMaxPair, st);
    if (e != cudaSuccess) {
        cudaFreeAsync(T, st);
        return cuda_error(e, "cudaMallocAsync(U)");
    }
    const int th = 256;
    long long nb = (tot + th - 1) / th;
    const int blocks = (int)(nb < 148 * 64 ? nb : 148 * 64);
    bool first = true;
    // parts that never receive a group still get written (zero) when requested
    for (const Round& rd : pl.rounds) {
        k_stage_x<<<blocks, th, 0, st>>>(rd, om.src[0], om.src[1], op->F[0].band, op->p[0], d, batch, T);
        k_stage_y<<<blocks, th, 0, st>>>(rd, T, op->F[1].band, op->p[1], d, batch, U);
        k_stage_z<<<blocks, th, 0, st>>>(rd, U, op->F[2].band, op->p[2], d, batch, om, first ? 0 : 1);
        first = false;
    }
    if (first) {
        for (int part = 0; part < 2; ++part)
            if (om.dst[part]) k_zero<<<blocks, th, 0, st>>>(om.dst[part], tot);
    }
    e = cudaGetLastError();
    cudaFreeAsync(T, st);
    cudaFreeAsync(U, st);
    if (e != cudaSuccess) return cuda_error(e, "apply_unfused launch");
    return IGA_OK;
}

}  // namespace igalr
