// ubench2.cu — data paths that bypass the shared-memory pipe, for the fused apply design:
//   tmem  : tcgen05.ld/st 32x32b round trips (per-thread private storage) mixed with DFMA
//   cmem  : coefficients from __constant__ (uniform index -> ULDC/LDC) feeding DFMAs,
//           working set 1..32 KB
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench2 tools/ubench2.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__constant__ double c_coef[4096];

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// NW warps per CTA, 1 CTA per SM, 512 TMEM columns. Warp w owns lanes (w%4)*32.., columns
// [(w/4)*cols_per, ...). Each step: ld x16 (16 x b32 = 8 doubles), DF DFMAs per double, st x16.
template <int NW, int DF>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem(double* out, int iters, double a) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase;
    constexpr int cols_per = 512 / (NW / 4);
    const uint32_t my = base + ((uint32_t)((warp % 4) * 32) << 16) + (uint32_t)((warp / 4) * cols_per);
    double acc = threadIdx.x * 1e-3;
    for (int i = 0; i < iters; ++i) {
        uint32_t col = (uint32_t)((i * 16) % cols_per);
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(my + col));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
#pragma unroll
        for (int d = 0; d < DF; ++d)
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = fma(v[k], a, acc);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            r[2 * k] = __double2loint(v[k]);
            r[2 * k + 1] = __double2hiint(v[k]);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                my + col),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        acc += 1e-9;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
    if (acc == 12345.0) out[threadIdx.x] = acc;
}

template <int F>
__global__ void k_cmem(double* out, int iters, int mask) {
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
    double x = 1.0 + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double c = c_coef[(i * 8 + u) & mask];
#pragma unroll
            for (int k = 0; k < F; ++k) acc[(u * F + k) & 7] = fma(c, x, acc[(u * F + k) & 7]);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename L>
static float timeit(L launch, int reps) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

int main(int argc, char** argv) {
    int sms = 148;
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    static double h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = 1e-6 * i;
    CK(cudaMemcpyToSymbol(c_coef, h, sizeof(h)));
    const char* only = argc > 1 ? argv[1] : "";
    int reps = 10;
    if (!*only || !strcmp(only, "tmem")) {
        int it = 20000;
#define TM(NW, DF)                                                                                                  \
    {                                                                                                               \
        float ms = timeit([&] { k_tmem<NW, DF><<<sms, NW * 32>>>(out, it, 0.9999999); }, reps);                    \
        double bytes = 2.0 * 128.0 * 32 * NW * (double)it * sms; /* ld + st, 64 B... per thread 64B each way */   \
        double fl = 2.0 * 8 * DF * 32.0 * NW * (double)it * sms;                                                    \
        printf("{\"bench\":\"tmem_rt\",\"warps\":%d,\"dfma_per_double\":%d,\"ms\":%.3f,\"tmem_GBps_ld+st\":%.0f,"  \
               "\"B_per_clk_per_sm\":%.1f,\"tflops\":%.2f}\n",                                                     \
               NW, DF, ms, bytes / ms / 1e6, bytes / ms / 1e-3 / 1.965e9 / sms, fl / ms / 1e9);                    \
    }
        TM(4, 0) TM(8, 0) TM(16, 0) TM(4, 2) TM(8, 2) TM(16, 2) TM(8, 4) TM(16, 4) TM(16, 8)
    }
    if (!*only || !strcmp(only, "cmem")) {
        int it = 4000;
        int blocks = sms * 8, threads = 256;
        for (int mask : {127, 511, 1023, 2047, 4095}) {
#define CM(F)                                                                                                       \
    {                                                                                                               \
        float ms = timeit([&] { k_cmem<F><<<blocks, threads>>>(out, it, mask); }, reps);                           \
        double fl = 2.0 * 8 * F * (double)it * blocks * threads;                                                    \
        printf("{\"bench\":\"cmem\",\"ws_bytes\":%d,\"dfma_per_coef\":%d,\"tflops\":%.2f}\n", (mask + 1) * 8, F, fl / ms / 1e9); \
    }
            CM(1) CM(2) CM(4)
        }
    }
    return 0;
}
