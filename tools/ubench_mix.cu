// ubench_mix.cu — do DFMA (CUDA-core FP64) and DMMA (mma.sync m8n8k4 f64) share one pipe on B200?
// One kernel, 8 warps per CTA, 148 CTAs.  Warps [0, nd) run a DFMA stream (8 independent chains,
// 2 reused operands), warps [nd, nd+nm) run a DMMA stream (4 independent accumulators), the rest idle.
// Each role has a fixed iteration count; the elapsed time of the mixed launch against the two solo
// launches tells whether the units are separate (max) or shared (sum).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mix tools/ubench_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(256, 1) k_mix(double* out, int nd, int nm, int it_d, int it_m, double a, double b) {
    const int warp = threadIdx.x >> 5;
    double s = 0.0;
    if (warp < nd) {
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
        for (int i = 0; i < it_d; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += x[k];
    } else if (warp < nd + nm) {
        double ma = 1e-3 * threadIdx.x, mb = 2e-3;
        double c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = k;
        for (int i = 0; i < it_m; ++i) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(c[2 * k]), "+d"(c[2 * k + 1]) : "d"(ma), "d"(mb));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += c[k];
    }
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

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    const int it = 4000;
    // flops: DFMA warp: it*64 FMA per thread; DMMA warp: it*16 mma * 256 FMA per warp
    auto run = [&](int nd, int nm, int itd, int itm) {
        float ms = timeit([&] { k_mix<<<sms, 256>>>(out, nd, nm, itd, itm, 1.0000001, 1e-9); }, 5);
        CK(cudaGetLastError());
        const double fl = 2.0 * sms * (nd * 32.0 * itd * 64 + nm * (double)itm * 16 * 256);
        printf("{\"bench\":\"mix\",\"dfma_warps\":%d,\"dmma_warps\":%d,\"it_dfma\":%d,\"it_dmma\":%d,\"ms\":%.4f,\"tflops\":%.2f}\n",
               nd, nm, itd, itm, ms, fl / ms / 1e9);
    };
    const int combos[][2] = {{8, 0}, {0, 8}, {4, 0}, {0, 4}, {4, 4}, {2, 0}, {0, 6}, {2, 6}, {6, 0}, {0, 2}, {6, 2}};
    for (auto& c : combos) run(c[0], c[1], it, it);
    return 0;
}
