// ubench.cu — FP64 microbenchmarks on B200 (sm_100a) that set the roofline denominator
// and the design budget of the fused apply kernel.
//   dfma      : peak DFMA rate (8 independent chains per thread)
//   dmma      : mma.sync m8n8k4 f64 rate (legacy DMMA path; tcgen05 has no f64 kind)
//   bcast F   : one LDS.128 broadcast (2 coefficients) feeding 2*F DFMAs
//   lds64 F   : one conflict-free per-lane LDS.64 feeding F DFMAs
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double a = 1e-3 * threadIdx.x, b = 2e-3;
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[2 * k]), "+d"(c[2 * k + 1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F>
__global__ void k_bcast(double* out, int iters) {
    __shared__ double2 coef[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) coef[i] = make_double2(1e-6 * i, 1.0 - 1e-7 * i);
    __syncthreads();
    double x[F];
#pragma unroll
    for (int k = 0; k < F; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double2 c = coef[(i * 8 + u) & 1023];
#pragma unroll
            for (int k = 0; k < F; ++k) { x[k] = fma(x[k], c.y, c.x); }
#pragma unroll
            for (int k = 0; k < F; ++k) { x[k] = fma(x[k], c.y, -c.x); }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < F; ++k) s += x[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F>
__global__ void k_lds64(double* out, int iters, double a) {
    // per step: one conflict-free per-lane LDS.64 (address depends on the step) feeding F
    // independent DFMAs (8 accumulators).
    extern __shared__ double buf[];
    const int n = blockDim.x * 16;
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = 1e-6 * i;
    __syncthreads();
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double v = ((volatile double*)buf)[(((i * 8 + u) & 15) * blockDim.x) + threadIdx.x];
#pragma unroll
            for (int k = 0; k < F; ++k) acc[(u * F + k) & 7] = fma(v, a, acc[(u * F + k) & 7]);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F>
__global__ void k_bc2(double* out, int iters, double a) {
    // per step: one broadcast LDS.128 (2 values) feeding 2F independent DFMAs
    __shared__ double2 coef[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) coef[i] = make_double2(1e-6 * i, 1.0 - 1e-7 * i);
    __syncthreads();
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double2 c = coef[(i * 8 + u) & 1023];
#pragma unroll
            for (int k = 0; k < F; ++k) {
                acc[(u * 2 * F + 2 * k) & 7] = fma(c.x, a, acc[(u * 2 * F + 2 * k) & 7]);
                acc[(u * 2 * F + 2 * k + 1) & 7] = fma(c.y, a, acc[(u * 2 * F + 2 * k + 1) & 7]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F>
__global__ void k_bc64(double* out, int iters, double a) {
    // per step: one broadcast LDS.64 feeding F independent DFMAs
    __shared__ double coef[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) coef[i] = 1e-6 * i;
    __syncthreads();
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double c = ((volatile double*)coef)[(i * 8 + u) & 1023];
#pragma unroll
            for (int k = 0; k < F; ++k) acc[(u * F + k) & 7] = fma(c, a, acc[(u * F + k) & 7]);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F>
__global__ void k_lds128(double* out, int iters, double a) {
    // per step: one conflict-free per-lane LDS.128 (2 values) feeding 2F DFMAs
    extern __shared__ double2 buf2[];
    const int n = blockDim.x * 16;
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf2[i] = make_double2(1e-6 * i, 2e-6 * i);
    __syncthreads();
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const volatile double2* p = &buf2[(((i * 8 + u) & 15) * blockDim.x) + threadIdx.x];
            double vx = p->x, vy = p->y;
#pragma unroll
            for (int k = 0; k < F; ++k) {
                acc[(u * 2 * F + 2 * k) & 7] = fma(vx, a, acc[(u * 2 * F + 2 * k) & 7]);
                acc[(u * 2 * F + 2 * k + 1) & 7] = fma(vy, a, acc[(u * 2 * F + 2 * k + 1) & 7]);
            }
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
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    int sms = prop.multiProcessorCount;
    printf("{\"device\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,\"regs_per_sm\":%d}\n",
           prop.name, sms, prop.l2CacheSize, prop.sharedMemPerMultiprocessor, prop.sharedMemPerBlockOptin,
           prop.regsPerMultiprocessor);
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    const char* only = argc > 1 ? argv[1] : "";
    int reps = 20;
    for (int threads : {256, 512}) {
        int blocks = sms * (2048 / threads);
        int iters = 20000;
        if (!*only || !strcmp(only, "dfma")) {
            float ms = timeit([&] { k_dfma<<<blocks, threads>>>(out, iters, 0.9999999, 1e-9); }, reps);
            double fl = 2.0 * 64 * 8 * (double)iters * blocks * threads;
            printf("{\"bench\":\"dfma\",\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", threads, ms, fl / ms / 1e9);
        }
        if (!*only || !strcmp(only, "dmma")) {
            int it2 = 5000;
            float ms = timeit([&] { k_dmma<<<blocks, threads>>>(out, it2); }, reps);
            double fl = 2.0 * 256 * 16 * (double)it2 * blocks * (threads / 32);
            printf("{\"bench\":\"dmma\",\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", threads, ms, fl / ms / 1e9);
        }
        if (!*only || !strcmp(only, "bcast")) {
            int it3 = 4000;
#define BC(F)                                                                                         \
    {                                                                                                 \
        float ms = timeit([&] { k_bcast<F><<<blocks, threads>>>(out, it3); }, reps);                  \
        double fl = 2.0 * 8 * 2 * F * (double)it3 * blocks * threads;                                 \
        printf("{\"bench\":\"bcast128\",\"F\":%d,\"dfma_per_lds\":%d,\"threads\":%d,\"tflops\":%.2f}\n", F, 2 * F, threads, fl / ms / 1e9); \
    }
            BC(1) BC(2) BC(4) BC(8)
#define BC2(F)                                                                                        \
    {                                                                                                 \
        float ms = timeit([&] { k_bc2<F><<<blocks, threads>>>(out, it3, 0.9999999); }, reps);         \
        double fl = 2.0 * 8 * 2 * F * (double)it3 * blocks * threads;                                 \
        printf("{\"bench\":\"bc2_128\",\"dfma_per_lds\":%d,\"threads\":%d,\"tflops\":%.2f}\n", 2 * F, threads, fl / ms / 1e9); \
    }
            BC2(1) BC2(2) BC2(4)
        }
        if (!*only || !strcmp(only, "lds64")) {
            int it4 = 4000;
            size_t sm = (size_t)threads * 16 * 8;
#define LD(F)                                                                                         \
    {                                                                                                 \
        CK(cudaFuncSetAttribute(k_lds64<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
        float ms = timeit([&] { k_lds64<F><<<blocks, threads, sm>>>(out, it4, 0.9999999); }, reps);   \
        double fl = 2.0 * 8 * F * (double)it4 * blocks * threads;                                     \
        printf("{\"bench\":\"lds64\",\"dfma_per_lds\":%d,\"threads\":%d,\"tflops\":%.2f}\n", F, threads, fl / ms / 1e9); \
    }
            LD(1) LD(2) LD(4) LD(8)
#define B64(F)                                                                                        \
    {                                                                                                 \
        float ms = timeit([&] { k_bc64<F><<<blocks, threads>>>(out, it4, 0.9999999); }, reps);        \
        double fl = 2.0 * 8 * F * (double)it4 * blocks * threads;                                     \
        printf("{\"bench\":\"bc64\",\"dfma_per_lds\":%d,\"threads\":%d,\"tflops\":%.2f}\n", F, threads, fl / ms / 1e9); \
    }
            B64(1) B64(2) B64(4)
            size_t sm2 = (size_t)threads * 16 * 16;
#define L128(F)                                                                                       \
    {                                                                                                 \
        CK(cudaFuncSetAttribute(k_lds128<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)); \
        float ms = timeit([&] { k_lds128<F><<<blocks, threads, sm2>>>(out, it4, 0.9999999); }, reps); \
        double fl = 2.0 * 8 * 2 * F * (double)it4 * blocks * threads;                                 \
        printf("{\"bench\":\"lds128\",\"dfma_per_lds\":%d,\"threads\":%d,\"tflops\":%.2f}\n", 2 * F, threads, fl / ms / 1e9); \
    }
            L128(1) L128(2) L128(4)
        }
    }
    return 0;
}
