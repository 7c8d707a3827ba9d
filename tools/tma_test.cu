// Standalone checks of the mbarrier / cp.async.bulk / TMA-tensor sequence used by k_canon.
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(const double* g, double* out, const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm) {
    __shared__ __align__(128) double buf[1024];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
        if (MODE & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (MODE & 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(1024 * 8) : "memory");
        if (MODE & 2) {
            const uint64_t d = (MODE & 8) ? (uint64_t)gtm : (uint64_t)&tm;
            const int c0 = (MODE & 16) ? 0 : -3, c1 = (MODE & 16) ? 0 : -2;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su(buf)), "l"(d), "r"(su(&bar)), "r"(c0), "r"(c1) : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(buf)), "l"(g), "r"(1024 * 8), "r"(su(&bar)) : "memory");
        }
    }
    asm volatile("{\n\t.reg .pred P1;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(su(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = buf[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    double *g, *o; cudaMalloc(&g, 1 << 20); cudaMalloc(&o, 1 << 20);
    double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = i; cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm; memset(&tm, 0, sizeof tm);
    cuuint64_t dims[2] = {64, 64}, strides[1] = {64 * 8}; cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult cr = ((Enc)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)cr);
    CUtensorMap* gtm; cudaMalloc(&gtm, sizeof(CUtensorMap)); cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
#define RUN(M) { k<M><<<1, 128>>>(g, o, tm, gtm); cudaError_t e = cudaDeviceSynchronize(); double r[40]; cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost); \
    printf("mode %d: %s  out[0..3]=%g %g %g %g  out[35]=%g\n", M, cudaGetErrorString(e), r[0], r[1], r[2], r[3], r[35]); if (e) return 1; }
    RUN(0) RUN(18) RUN(26) RUN(10) RUN(2)
    return 0;
}
