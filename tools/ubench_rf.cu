// Register-operand bandwidth of DFMA on sm_100a: throughput of DFMA streams whose three
// 64-bit source operands are all fresh (A), one reused (B) or two reused (C), at 1-4 warps
// per SMSP.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_rf ubench_rf.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const double* in, double* out, int iters) {
    double a[8], b[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = in[(threadIdx.x + i) & 255];
        b[i] = in[(threadIdx.x + 3 * i + 1) & 255];
        c[i] = in[(threadIdx.x + 5 * i + 2) & 255];
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) c[i] = fma(a[(i + r) & 7], b[(i + 3 * r) & 7], c[i]);
                if (MODE == 1) c[i] = fma(a[r], b[(i + 3 * r) & 7], c[i]);
                if (MODE == 2) c[i] = fma(a[r], b[r], c[i]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(int threads, int iters) {
    double *in, *out;
    cudaMalloc(&in, 256 * 8);
    cudaMemset(in, 0, 256 * 8);
    cudaMalloc(&out, 148 * threads * 8);
    k<MODE><<<148, threads>>>(in, out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<148, threads>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(in);
    cudaFree(out);
    return 2.0 * 64 * (double)iters * 148 * threads / (ms * 1e-3) / 1e12;
}

int main() {
    const char* names[3] = {"3 fresh operands", "1 reused (multiplier)", "2 reused"};
    for (int t : {128, 256, 384, 512}) {
        printf("threads %d: A(%s) %.2f  B(%s) %.2f  C(%s) %.2f TF/s\n", t, names[0], run<0>(t, 20000), names[1],
               run<1>(t, 20000), names[2], run<2>(t, 20000));
    }
    return 0;
}
