// DFMA dependent-chain latency and single-warp throughput vs number of independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k_chain(double* out, int iters, double a, double b, long long* cyc) {
    double x[C];
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = threadIdx.x + k;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < C; ++k) x[k] = fma(x[k], a, b);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) s += x[k];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 8 * 1024);
    long long h;
    const int iters = 4096;
#define RUN(C, W) { k_chain<C><<<1, 32 * W>>>(out, iters, 0.999999, 1e-7, cyc); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
    printf("{\"chains\":%d,\"warps\":%d,\"cycles_per_dfma_per_warp\":%.2f}\n", C, W, (double)h / iters / C); }
    RUN(1, 1) RUN(2, 1) RUN(4, 1) RUN(8, 1) RUN(16, 1) RUN(1, 4) RUN(4, 4) RUN(8, 4) RUN(1, 8) RUN(4, 8) RUN(8, 8)
    return 0;
}
