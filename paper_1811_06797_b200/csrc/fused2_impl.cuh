// apply_fused2.cu — fused sm_100a apply, version 2: TMEM-resident z-ring.
//
// One part (mass OR stiffness) per launch:
//   y(z,y,x) = sum_rounds sum_g Fz_g *_z  sum_{j in g} c_j  Fy_j *_y  Fx_{e(j)} *_x  v
// (Eqs. (massFinal)/(stiffnessFinal)).
//
// CTA = 4 warps (one per TMEM lane quadrant), tile = 128 x-columns x L y-rows of one batch
// vector.  Persistent CTAs walk a contiguous range of (tile, z-plane) units; for every input
// plane z' and plan round r each thread (one x-column) sweeps the L+2P rows of its column:
//   X: t_e(y') = sum_k Fx_e[x][k] v(y', x-P+k)  (x-coefs in registers, v from the smem tile)
//   Y: sliding register window over t_e; u_j = sum_k Fy_j[y][k] t_{e(j)}(y-P+k) (y-coefs are
//      smem broadcasts), G_g = sum_j c_j u_j
//   Z: ring(y,x)[slot] += Cz[g][slot] G_g  — the ring of 2P+1 output planes per point lives in
//      TMEM (tcgen05.ld/st, 32x32b); slots are physical (plane mod 2P+1), the z-coefficients
//      are permuted per z' instead of rotating the ring.
// A plane is retired inline during the last round once its last input plane is processed.
// Planes whose inputs span two CTAs' ranges are written to per-CTA scratch and summed by
// k_fixup in CTA order (deterministic; no atomics).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include <cuda.h>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"

#ifndef IGALR_ZSMEM_P
#define IGALR_ZSMEM_P 4  // (experiment knob: smallest degree whose stiffness kernel reads z from smem)
#endif
#ifndef IGALR_YTAP
#define IGALR_YTAP 1  // 1: tap-major Y stage for p = 3 (YPitch::TAP); 0: factor-major everywhere
#endif

namespace igalr {
namespace f2 {

constexpr int TXW = 32;          // columns per warp
constexpr int NW = 4;            // warps per CTA (one per TMEM lane quadrant)
constexpr int TX = TXW * NW;     // 128 columns per tile
constexpr int kMaxRounds2 = 40;

template <int NX, int NP, int NG>
struct Round2 {
    int nx, np, ng, nyf;
    int xf[NX];        // x factor of x-entry e
    int yf[NP];        // distinct y factors of the round (nyf of them)
    int pyf[NP];       // pair -> y-factor slot
    int px[NP];        // pair -> x-entry
    int pg[NP];        // pair -> group
    int plead[NP];     // 1 if the pair is its group's lead (coef folded into the group scale)
    double pc[NP];     // pair coefficient / group scale (unused for lead pairs)
    int gf[NG];        // group z factor
    double gs[NG];     // group scale (lead pair coefficient)
};

struct Args2 {
    const double* src;
    double* dst;
    double scale;
    int accumulate;
    double* scratch;       // [nctas][NSEG][4P][L][TX] partial planes
    const double* bx;      // x-factor bands; on the unpacked GSYNC path instead the per-round x records
                           // [nrounds][ceil(mx/32)][NX][32][BW] (k_build_xtab)
    const double* by;
    const double* bz;      // z-factor bands; on the GSYNC canonical path instead the per-plane z
                           // records [mz][nrounds][NGB] (slot-permuted, group-scaled; k_build_ztab)
    const void* rounds;
    int nrounds;
    int mx, my, mz, batch;
    int tiles_x, tiles_y;
    long long units;       // tiles * mz
    int nctas;
    int txt, tyt;          // tile width / height (fixup)
};
// Batch split of a canonical launch (KKT): vectors b >= bsplit read src + b*vol + src_jump and
// write dst + b*vol + dst_jump (element offsets).  A separate kernel parameter: growing Args2 moves
// the register-tight p = 4 kernel over the spill cliff.
// vp > 1 (GSYNC path only): vector packing along x.  A launch row is vp consecutive vectors' rows
// side by side (width vp * mx); packed column c of vector group g belongs to vector g * vp + c / mx,
// local column c % mx.  Seams need no gap: a factor's band row holds zeros for columns outside the
// matrix, so the taps that cross a seam multiply by 0.  Narrow meshes then fill the 32-lane column
// groups (46 columns: 72 % of a 64-wide tile; 4 packed vectors: 184 of 192 columns).
struct KSplit {
    long long bsplit, src_jump, dst_jump;
    int vp;
};

constexpr int NSEG = 4;    // max segments per CTA (checked on the host)

__host__ __device__ inline long long unit_begin(long long k, long long units, int nctas) {
    return k * units / nctas;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp8(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// ---- mbarrier / TMA helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- TMEM helpers (32x32b shape: each thread accesses its own lane)
__device__ __forceinline__ void tm_ld16(uint32_t taddr, double* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    // the wait "modifies" the destination registers so no use can be scheduled before it
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]));
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const double* v) {
    uint32_t r[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        r[2 * k] = __double2loint(v[k]);
        r[2 * k + 1] = __double2hiint(v[k]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, double* v) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
    v[0] = __hiloint2double(r[1], r[0]);
    v[1] = __hiloint2double(r[3], r[2]);
}
__device__ __forceinline__ void tm_st4(uint32_t taddr, const double* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__double2loint(v[0])),
                 "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])));
}
__device__ __forceinline__ double tm_ld1(uint32_t taddr) {
    uint32_t lo, hi;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(lo), "+r"(hi));
    return __hiloint2double(hi, lo);
}
__device__ __forceinline__ void tm_st1(uint32_t taddr, double v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__double2loint(v)),
                 "r"(__double2hiint(v)));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ring slots per point, padded to a multiple of 8 doubles (x16 loads) or +2 (x4 tail).  TIGHT
// (canonical kernel): an odd tail below 5 doubles ends in one x2 access instead of padding, so
// p = 4 (2P+1 = 9) stores 9 doubles (18 columns) per point instead of 10
template <int BW, bool TIGHT = false>
struct RingShape {
    static constexpr int REM = BW % 8;
    static constexpr int N16 = BW / 8 + (REM >= 5 ? 1 : 0);     // number of x16 chunks (8 doubles)
    static constexpr int N4 = (REM >= 5 || REM == 0) ? 0 : (TIGHT ? REM / 2 : (REM + 1) / 2);  // x4 chunks
    static constexpr int N2 = (TIGHT && REM < 5 && (REM & 1)) ? 1 : 0;  // x2 chunk (1 double)
    static constexpr int DBL = N16 * 8 + N4 * 2 + N2;  // doubles stored per point
    static constexpr int COLS = DBL * 2;               // TMEM columns per point
};

template <int BW, bool TIGHT = false>
__device__ __forceinline__ void ring_ld(uint32_t t, double* v) {
    using RS = RingShape<BW, TIGHT>;
#pragma unroll
    for (int c = 0; c < RS::N16; ++c) tm_ld16(t + c * 16, v + c * 8);
#pragma unroll
    for (int c = 0; c < RS::N4; ++c) tm_ld4(t + RS::N16 * 16 + c * 4, v + RS::N16 * 8 + c * 2);
    if constexpr (RS::N2) v[RS::DBL - 1] = tm_ld1(t + RS::COLS - 2);
}
template <int BW, bool TIGHT = false>
__device__ __forceinline__ void ring_st(uint32_t t, const double* v) {
    using RS = RingShape<BW, TIGHT>;
#pragma unroll
    for (int c = 0; c < RS::N16; ++c) tm_st16(t + c * 16, v + c * 8);
#pragma unroll
    for (int c = 0; c < RS::N4; ++c) tm_st4(t + RS::N16 * 16 + c * 4, v + RS::N16 * 8 + c * 2);
    if constexpr (RS::N2) tm_st1(t + RS::COLS - 2, v[RS::DBL - 1]);
}

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// split TMEM ring load: issue now, wait (tied to the registers) when the values are needed
template <int BW, bool TIGHT = false>
__device__ __forceinline__ void ring_issue(uint32_t t, uint32_t* r) {
    using RS = RingShape<BW, TIGHT>;
#pragma unroll
    for (int c = 0; c < RS::N16; ++c) {
        uint32_t* q = r + c * 16;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
              "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
            : "r"(t + c * 16));
    }
#pragma unroll
    for (int c = 0; c < RS::N4; ++c) {
        uint32_t* q = r + RS::N16 * 16 + c * 4;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
                     : "r"(t + RS::N16 * 16 + c * 4));
    }
    if constexpr (RS::N2) {
        uint32_t* q = r + RS::N16 * 16 + RS::N4 * 4;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                     : "=r"(q[0]), "=r"(q[1])
                     : "r"(t + RS::COLS - 2));
    }
}
template <int BW, bool TIGHT = false>
__device__ __forceinline__ void ring_wait(uint32_t* r, double* v) {
    using RS = RingShape<BW, TIGHT>;
    static_assert(RS::DBL * 2 <= 24, "ring_wait handles up to 24 registers");
    if constexpr (RS::DBL * 2 == 16) {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                       "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                       "+r"(r[15]));
    } else if constexpr (RS::DBL * 2 == 18) {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                       "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                       "+r"(r[15]), "+r"(r[16]), "+r"(r[17]));
    } else if constexpr (RS::DBL * 2 == 20) {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                       "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                       "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]));
    } else {
#pragma unroll
        for (int k = 0; k < RS::DBL * 2; ++k) asm volatile("" : "+r"(r[k]));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
#pragma unroll
    for (int k = 0; k < RS::DBL; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
}

template <int P, int L>
struct Geo {
    static constexpr int BW = 2 * P + 1;
    static constexpr int HY = L + 2 * P;          // sweep rows (incl. y-halo)
    static constexpr int HX = TX + 2 * P;         // tile columns incl. x-halo
    static constexpr int HXP = HX + 1;            // padded row pitch
};

// scratch slot of a partial output plane zo for a segment [za, zb) (see header comment)
__host__ __device__ __forceinline__ int partial_slot(int zo, int za, int zb, int P) {
    const int rel = zo - (za - P);
    if (rel < 2 * P) return rel;                  // head band
    return 2 * P + (zo - (zb - P));               // tail band
}

template <int P, int L, int NX, int NP, int NG, int NY>
__global__ void __launch_bounds__(NW * 32, 1) k_fused2(const Args2 a) {
    using G_ = Geo<P, L>;
    constexpr int BW = G_::BW, HY = G_::HY, HXP = G_::HXP;
    using RS = RingShape<BW>;
    using RoundT = Round2<NX, NP, NG>;
    static_assert(L * RS::COLS <= 512, "ring does not fit in TMEM");

    extern __shared__ __align__(16) double sm[];
    double* vin = sm;                                   // [2][HY][HXP]
    double* xcs = vin + 2 * HY * HXP;                   // [2][NX][TX][BW]
    double* ycs = xcs + 2 * NX * TX * BW;               // [nrounds][NY][L][BW]  (by y-factor slot)
    double* zcs = ycs + (size_t)a.nrounds * NY * L * BW;  // [2][nrounds][NG][BW]
    RoundT* rs = reinterpret_cast<RoundT*>(zcs + 2 * a.nrounds * NG * BW);
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cx = warp * TXW + lane;  // tile column of this thread

    // ---- TMEM allocation (512 columns, one CTA per SM)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < a.nrounds * (int)(sizeof(RoundT) / 4); i += blockDim.x)
        reinterpret_cast<int*>(rs)[i] = reinterpret_cast<const int*>(a.rounds)[i];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(warp * 32) << 16);

    const long long plane = (long long)a.mx * a.my;
    const long long u0 = unit_begin(blockIdx.x, a.units, a.nctas);
    const long long u1 = unit_begin(blockIdx.x + 1, a.units, a.nctas);

    int seg = 0;
    for (long long u = u0; u < u1; ++seg) {
        const long long tile = u / a.mz;
        const int za = (int)(u - tile * a.mz);
        const int zb = (int)min((long long)a.mz, (long long)za + (u1 - u));
        u += zb - za;
        long long tt = tile;
        const int txi = (int)(tt % a.tiles_x); tt /= a.tiles_x;
        const int tyi = (int)(tt % a.tiles_y); tt /= a.tiles_y;
        const int b = (int)tt;
        const int x0 = txi * TX, y0 = tyi * L;
        const long long vb = (long long)b * a.mz * plane;
        const int gx = x0 + cx;

        // ---- stage y-coefficients of this tile (all rounds), clear the ring
        __syncthreads();
        for (int r = 0; r < a.nrounds; ++r) {
            const RoundT& R = rs[r];
            for (int i = threadIdx.x; i < R.nyf * L * BW; i += blockDim.x) {
                const int s = i / (L * BW), rem = i - s * L * BW;
                const int row = rem / BW, k = rem - row * BW;
                const int gy = y0 + row;
                const bool ok = gy < a.my;
                cp8(ycs + ((size_t)(r * NY + s) * L + row) * BW + k,
                    ok ? a.by + ((size_t)R.yf[s] * a.my + gy) * BW + k : a.by, ok);
            }
        }
        {
            double zero[RS::DBL];
#pragma unroll
            for (int k = 0; k < RS::DBL; ++k) zero[k] = 0.0;
            for (int i = 0; i < L; ++i) ring_st<BW>(tbase + i * RS::COLS, zero);
        }

        auto stage_plane = [&](int zp, int buf) {
            double* dstp = vin + buf * HY * HXP;
            const double* srcp = a.src + vb + (long long)zp * plane;
            for (int i = threadIdx.x; i < HY * G_::HX; i += blockDim.x) {
                const int r = i / G_::HX, c = i - r * G_::HX;
                const int gy = y0 - P + r, gxx = x0 - P + c;
                const bool ok = gy >= 0 && gy < a.my && gxx >= 0 && gxx < a.mx;
                cp8(dstp + r * HXP + c, ok ? srcp + (long long)gy * a.mx + gxx : a.src, ok);
            }
            // z-coefficients of plane zp for all rounds, permuted to physical ring slots:
            // slot j holds output plane zo with zo == j (mod BW); coefficient Fz[zo][zp - zo + P]
            double* zdst = zcs + buf * a.nrounds * NG * BW;
            for (int i = threadIdx.x; i < a.nrounds * NG * BW; i += blockDim.x) {
                const int r = i / (NG * BW), rem = i - r * NG * BW;
                const int g = rem / BW, j = rem - g * BW;
                const RoundT& R = rs[r];
                int zo = zp - P + ((j - (zp - P)) % BW + BW) % BW;  // plane in [zp-P, zp+P] with zo%BW == j
                const bool ok = g < R.ng && zo >= 0 && zo < a.mz;
                cp8(zdst + i, ok ? a.bz + ((size_t)R.gf[g] * a.mz + zo) * BW + (zp - zo + P) : a.bz, ok);
            }
        };
        auto stage_xc = [&](int r, int buf) {
            const RoundT& R = rs[r];
            double* dstp = xcs + buf * NX * TX * BW;
            for (int i = threadIdx.x; i < R.nx * TX * BW; i += blockDim.x) {
                const int e = i / (TX * BW), rem = i - e * TX * BW;
                const int c = rem / BW, k = rem - c * BW;
                const int g = x0 + c;
                const bool ok = g < a.mx;
                cp8(dstp + i, ok ? a.bx + ((size_t)R.xf[e] * a.mx + g) * BW + k : a.bx, ok);
            }
        };

        const int zlo = za, zhi = zb;
        stage_plane(zlo, 0);
        stage_xc(0, 0);
        cp_commit();
        int pbuf = 0, xbuf = 0;
        for (int zp = zlo; zp < zhi; ++zp) {
            for (int r = 0; r < a.nrounds; ++r) {
                // prefetch: next round's x-coefs (and the next plane at the start of the plane)
                const bool last_round = (r == a.nrounds - 1);
                cp_wait<0>();
                tm_wait_st();
                __syncthreads();
                if (!last_round) {
                    stage_xc(r + 1, xbuf ^ 1);
                } else if (zp + 1 < zhi) {
                    stage_xc(0, xbuf ^ 1);
                }
                if (r == 0 && zp + 1 < zhi) stage_plane(zp + 1, pbuf ^ 1);
                cp_commit();

                const RoundT& R = rs[r];
                const double* vt = vin + pbuf * HY * HXP;
                const double* xc = xcs + xbuf * NX * TX * BW;
                const double* yc = ycs + (size_t)r * NY * L * BW;
                const double* zc = zcs + pbuf * a.nrounds * NG * BW + r * NG * BW;
                double xr[NX][BW];
#pragma unroll
                for (int e = 0; e < NX; ++e)
#pragma unroll
                    for (int k = 0; k < BW; ++k) xr[e][k] = (e < R.nx) ? xc[(e * TX + cx) * BW + k] : 0.0;
                double zr[NG][BW];
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int j = 0; j < BW; ++j) zr[g][j] = (g < R.ng) ? zc[g * BW + j] * R.gs[g] : 0.0;
                // retire slot of output plane zp - P in the last round (if complete here)
                const int zret = zp - P;
                const int jret = ((zret % BW) + BW) % BW;
                bool ret_valid = false, ret_complete = false;
                if (last_round && zret >= 0 && zret < a.mz) {
                    ret_valid = true;
                    const int lo = max(0, zret - P), hi = min(a.mz - 1, zret + P);
                    ret_complete = lo >= za && hi <= zb - 1;
                }

                double w[NX][BW];  // circular window of t_e over the last BW rows
#pragma unroll
                for (int e = 0; e < NX; ++e)
#pragma unroll
                    for (int k = 0; k < BW; ++k) w[e][k] = 0.0;

#pragma unroll 1
                for (int base = 0; base < HY; base += BW) {
#pragma unroll
                    for (int q = 0; q < BW; ++q) {
                        const int step = base + q;
                        if (step < HY) {
                            // X stage for sweep row `step`
                            double v[BW];
#pragma unroll
                            for (int k = 0; k < BW; ++k) v[k] = vt[step * HXP + cx + k];
#pragma unroll
                            for (int e = 0; e < NX; ++e) {
                                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                                for (int k = 0; k < BW; k += 2) acc0 = fma(xr[e][k], v[k], acc0);
#pragma unroll
                                for (int k = 1; k < BW; k += 2) acc1 = fma(xr[e][k], v[k], acc1);
                                w[e][q] = acc0 + acc1;
                            }
                            if (step >= 2 * P) {
                                const int i = step - 2 * P;  // output row in tile
                                const uint32_t tp = tbase + i * RS::COLS;
                                double ring[RS::DBL];
                                ring_ld<BW>(tp, ring);
                                double G[NG];
#pragma unroll
                                for (int g = 0; g < NG; ++g) G[g] = 0.0;
                                const double* ycr = yc + (size_t)i * BW;
#pragma unroll
                                for (int j = 0; j < NP; ++j) {
                                    if (j < R.np) {
                                        const double* fy = ycr + (size_t)R.pyf[j] * L * BW;
                                        const int e = R.px[j];
                                        double u0 = 0.0, u1 = 0.0;
#pragma unroll
                                        for (int ee = 0; ee < NX; ++ee) {
                                            if (ee == e) {
#pragma unroll
                                                for (int k = 0; k < BW; k += 2) u0 = fma(fy[k], w[ee][(q + 1 + k) % BW], u0);
#pragma unroll
                                                for (int k = 1; k < BW; k += 2) u1 = fma(fy[k], w[ee][(q + 1 + k) % BW], u1);
                                            }
                                        }
                                        const double u = u0 + u1;
                                        const int g = R.pg[j];
#pragma unroll
                                        for (int gg = 0; gg < NG; ++gg)
                                            if (gg == g) G[gg] = R.plead[j] ? G[gg] + u : fma(R.pc[j], u, G[gg]);
                                    }
                                }
#pragma unroll
                                for (int g = 0; g < NG; ++g)
#pragma unroll
                                    for (int j = 0; j < BW; ++j) ring[j] = fma(zr[g][j], G[g], ring[j]);
                                if (ret_valid) {
                                    double val = 0.0;
#pragma unroll
                                    for (int j = 0; j < BW; ++j)
                                        if (j == jret) {
                                            val = ring[j];
                                            ring[j] = 0.0;
                                        }
                                    const int gy = y0 + i;
                                    if (gy < a.my && gx < a.mx) {
                                        if (ret_complete) {
                                            const long long o = vb + (long long)zret * plane + (long long)gy * a.mx + gx;
                                            a.dst[o] = (a.accumulate ? a.dst[o] : 0.0) + a.scale * val;
                                        } else {
                                            const int slot = partial_slot(zret, za, zb, P);
                                            a.scratch[((((size_t)blockIdx.x * NSEG + seg) * 4 * P + slot) * L + i) * TX + cx] =
                                                a.scale * val;
                                        }
                                    }
                                }
                                ring_st<BW>(tp, ring);
                            }
                        }
                    }
                }
                if (last_round) pbuf ^= 1;
                xbuf ^= 1;
            }
        }
        // ---- flush planes still in the ring: zo in [zb-P, zb+P) (partial unless zb == mz)
        tm_wait_st();
        __syncthreads();
        for (int i = 0; i < L; ++i) {
            const uint32_t tp = tbase + i * RS::COLS;
            double ring[RS::DBL];
            ring_ld<BW>(tp, ring);
            const int gy = y0 + i;
#pragma unroll
            for (int s = 0; s < 2 * P; ++s) {
                const int zo = zb - P + s;
                if (zo < 0 || zo >= a.mz || zo < za - P) continue;
                // already retired inline? planes zo <= zb-1-P were retired during the sweep
                if (zo <= zb - 1 - P) continue;
                const int j = zo % BW;
                double val = 0.0;
#pragma unroll
                for (int jj = 0; jj < BW; ++jj)
                    if (jj == j) val = ring[jj];
                if (gy < a.my && gx < a.mx) {
                    const int lo = max(0, zo - P), hi = min(a.mz - 1, zo + P);
                    const bool complete = lo >= za && hi <= zb - 1;
                    if (complete) {
                        const long long o = vb + (long long)zo * plane + (long long)gy * a.mx + gx;
                        a.dst[o] = (a.accumulate ? a.dst[o] : 0.0) + a.scale * val;
                    } else {
                        const int slot = partial_slot(zo, za, zb, P);
                        a.scratch[((((size_t)blockIdx.x * NSEG + seg) * 4 * P + slot) * L + i) * TX + cx] = a.scale * val;
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_sh));
}

// ------------------------------------------------------------------------------------
// Canonical round shapes: the plan structure is compile-time, only factor ids and the
// pair/group coefficients are runtime data.  Stiffness (reading A of G6): for
// every r the 9 blocks q_kl share v_r, giving x-entries [K,E,T,M] (patterns (1,1),(0,1),
// (1,0),(0,0)), y-factors [M,T,E,K], z-groups [M,T,E,K] and the 9 (y,x)->z pairs below.
struct ShapeStiffA {
    static constexpr int NX = 4, NY = 4, NG = 4, NPAIR = 9;
    __host__ __device__ static constexpr int px(int j) { return j == 0 ? 0 : (j <= 2 ? 1 : (j == 3 || j == 6) ? 2 : 3); }
    __host__ __device__ static constexpr int py(int j) {
        return (j == 0 || j == 2 || j == 6 || j == 8) ? 0 : (j == 1 || j == 7) ? 1 : (j == 3 || j == 5) ? 2 : 3;
    }
    __host__ __device__ static constexpr int pg(int j) {
        return (j == 0 || j == 1 || j == 3 || j == 4) ? 0 : (j == 2 || j == 5) ? 1 : (j == 6 || j == 7) ? 2 : 3;
    }
    __host__ __device__ static constexpr bool lead(int j) { return j == 0 || j == 2 || j == 6 || j == 8; }
    // tap-major Y-stage issue order: consecutive pairs share their y-coefficient or their window
    // value (M:K, M:E | T:E, T:M | M:M, M:T | E:T, E:M | K:M), so every DFMA but the first of a
    // tap can take one operand from the operand-reuse cache
    __host__ __device__ static constexpr int ord(int i) {
        return i == 0 ? 0 : i == 1 ? 2 : i == 2 ? 1 : i == 3 ? 7 : i == 4 ? 8 : i == 5 ? 6 : i == 6 ? 3 : i == 7 ? 5 : 4;
    }
};
// Mass: K consecutive rank-one terms per sweep (independent pipelines sharing the input
// loads and the ring).
template <int K>
struct ShapeMassK {
    static constexpr int NX = K, NY = K, NG = K, NPAIR = K;
    __host__ __device__ static constexpr int px(int j) { return j; }
    __host__ __device__ static constexpr int py(int j) { return j; }
    __host__ __device__ static constexpr int pg(int j) { return j; }
    __host__ __device__ static constexpr bool lead(int) { return true; }
    __host__ __device__ static constexpr int ord(int i) { return i; }
};
using ShapeMass = ShapeMassK<4>;

template <class S>
struct RoundC {
    int xf[S::NX], yf[S::NY], gf[S::NG];
    int pad;
    double pc[S::NPAIR];   // coefficient ratio of non-lead pairs
    double gs[S::NG];      // group scale (lead pair coefficient)
};

template <int P, int TXT_, int TY>
struct GeoC {
    static constexpr int BW = 2 * P + 1;
    static constexpr int BWP = (BW + 1) & ~1;     // y-coef row pitch (16-byte aligned rows)
    static constexpr int HY = TY + 2 * P;
    static constexpr int HX = TXT_ + 2 * P;
    // plane rows: smem column c holds global column x0 - P - PADL + c, so that (nx even) row
    // segments start 16-byte aligned in global and shared memory (bulk copies); even pitch
    static constexpr int PADL = P & 1;
    static constexpr int HXP = (HX + PADL + 1) & ~1;
};
// y-coefficient record of one tile row: tap-major [k][NYP] (TAP: the factors of one tap are
// adjacent, so a tap's coefficients are one or two broadcast LDS.128 and all pairs' chains advance
// together) or factor-major [NY][BWP].  TAP for p = 3 only: measured on B200, c3 -0.4 %, c4 -1.4 %;
// at p = 4 the NPAIR live accumulators push the sweep into spills (c5 +2 %).
template <int NY, int BW>
struct YPitch {
    static constexpr bool TAP = IGALR_YTAP && BW == 7;
    static constexpr int NYP = (NY + 1) & ~1;
    static constexpr int BWP = (BW + 1) & ~1;
    static constexpr int ROW = TAP ? BW * NYP : NY * BWP;  // doubles per tile row
};
template <int NG, int BW>
struct ZPitch {
    static constexpr int NGB = (NG * BW + 1) & ~1;  // z-coefficients per round, 16-byte multiple
};

// Group-synchronised rounds + bulk-copied plane rows (needs bulk copies and resident y).
template <int P, bool TMA, bool YRES>
__host__ __device__ constexpr bool gsync_path() {
    return TMA && YRES;
}

// QX of the 4 TMEM lane quadrants tile x (32 columns each); the other 4/QX stack in y.
template <class S, int P, int LW, int WPQ, int QX, bool YRES, bool TMA, bool SPLIT = false, bool PACK = false>
__global__ void __launch_bounds__(NW * WPQ * 32, 1) k_canon(const Args2 a, const KSplit ks) {
    constexpr int TX = 32 * QX;                 // tile columns (shadows the 128-wide default)
    constexpr int TY = LW * WPQ * (4 / QX);     // tile rows
    using G_ = GeoC<P, TX, TY>;
    constexpr int BW = G_::BW, BWP = G_::BWP, HY = G_::HY;
    // 9-double ring (x16 + x2 accesses) when the padded 10-double ring would not fit this LW
    constexpr bool TIGHTR = LW * RingShape<BW>::COLS * WPQ > 512;
    constexpr int HXP = G_::HXP, PADL = G_::PADL;
    constexpr int VSZ = (HY * G_::HXP + 15) & ~15;  // doubles per plane buffer (128-B aligned)
    constexpr int NX = S::NX, NY = S::NY, NG = S::NG, NPAIR = S::NPAIR;
    using RS = RingShape<BW, TIGHTR>;
    using RoundT = RoundC<S>;
    static_assert(LW * RS::COLS * WPQ <= 512, "ring does not fit in TMEM");

    extern __shared__ __align__(1024) double sm[];
    double* vin = sm;                                   // [2][VSZ]  (HY x HXP planes)
    double* xcs = vin + 2 * VSZ;                        // [2][NX][TX][BW]  (per round)
    // y-coefficients: all rounds resident per segment (YRES) or double-buffered per round
    constexpr int YSLOTS = YRES ? 0 : 2;
    const int nyslots = YRES ? a.nrounds : YSLOTS;
    using YP = YPitch<NY, BW>;
    constexpr int NYP = YP::NYP, YROW = YP::ROW;
    double* ycs = xcs + 2 * NX * TX * BW;               // [nyslots][TY][YROW]
    constexpr int NGB = ZPitch<NG, BW>::NGB;
    double* zcs = ycs + (size_t)nyslots * TY * YROW;    // [2][nrounds][NGB] (per plane)
    RoundT* rs = reinterpret_cast<RoundT*>(zcs + 2 * a.nrounds * NGB);
    __shared__ uint32_t tmem_base_sh;
    // bulk-copy completion of the x-coefficient buffers, per column group (GSYNC) or CTA-wide
    __shared__ __align__(8) uint64_t xbar[QX][2];
    __shared__ __align__(8) uint64_t pbar[2];  // GSYNC: plane rows + z record landed
    uint32_t xph = 0, pph = 0;  // mbarrier parity per buffer (bit b: buffer b; no local-memory arrays)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quad = warp & 3, sub = warp >> 2;
    // column group of this warp: the WPQ warps that share a TMEM lane quadrant (and so an SMSP:
    // warp % 4) take different column groups, so a group barrier never holds both warps of one
    // scheduler at once (the other keeps the FP64 pipe busy)
    const int cg = (quad + sub) % QX;
    const int cx = cg * TXW + lane;                          // tile column of this thread
    // GSYNC: the warps of one column group (same cg: 32 columns) are the only readers of
    // the group's x-coefficients, so rounds are separated by a group barrier (named barrier
    // 1 + grp) and only the first round of a plane (new plane buffer) by a CTA barrier.
    constexpr bool GSYNC = gsync_path<P, TMA, YRES>();
    // XREC: one bulk copy per column group and round from the per-round x records (Args2::bx) instead
    // of NX band-row copies: the producer's copy issue is a uniform-register round trip per copy
    // (c3 -1.0 %).  p = 3 only: at p = 4 the change moves the mass kernel into spills (c5 +1 %)
    constexpr bool XREC = GSYNC && !PACK && P == 3;
    // GSYNC plane staging: lane 0 of every warp issues a share of the row copies (DIST) or
    // thread 0 issues all of them
    constexpr bool DIST = !(P == 3 && QX == 4);
    const int grp = GSYNC ? cg : 0;
    constexpr int GTHREADS = GSYNC ? 32 * WPQ * (4 / QX) : NW * WPQ * 32;
    const bool gprod = GSYNC ? (warp == grp && lane == 0) : (threadIdx.x == 0);  // x-copy issuer
    const int row0 = ((quad / QX) * WPQ + sub) * LW;          // first tile output row of this warp
#ifdef IGALR_EXP_NOZ
    double exp_sink = 0.0;
#endif
#ifdef IGALR_EXP_TIMERS
    // experiment: per-warp cycle accounting of the round loop (sync, coefficient loads, sweep, retire)
    long long exp_t[5] = {0, 0, 0, 0, 0}, exp_acc[4] = {0, 0, 0, 0}, exp_bar = 0, exp_pw = 0, exp_tb = 0, exp_tw = 0,
              exp_sx = 0, exp_xw = 0, exp_sp = 0;
    const long long exp_t_start = clock64();
#define EXP_T(k)                                                        \
    do {                                                                \
        exp_t[k] = clock64();                                           \
        if ((k) > 0) exp_acc[(k) - 1] += exp_t[k] - exp_t[(k) - 1];     \
    } while (0)
#else
#define EXP_T(k) do {} while (0)
#endif
    // y-coefficient rows of the tile for one round: [TY][YROW], entry (row, factor f, tap k) at
    // k * NYP + f (YTAP) or f * BWP + k; one warp per (factor, row), lane k < BW copies one tap
    auto copy_yrows = [&](double* ydst, const RoundT& R, int y0_) {
        if (lane < BW) {
            for (int rr = warp; rr < NY * TY; rr += NW * WPQ) {
                const int f = rr / TY, row = rr - f * TY;
                const int o = YP::TAP ? lane * NYP + f : f * BWP + lane;
                cp8(ydst + (size_t)row * YROW + o, a.by + ((size_t)R.yf[f] * a.my + y0_ + row) * BW + lane, true);
            }
        }
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < a.nrounds * (int)(sizeof(RoundT) / 4); i += blockDim.x)
        reinterpret_cast<int*>(rs)[i] = reinterpret_cast<const int*>(a.rounds)[i];
    if (TMA && threadIdx.x == 0) {
        for (int g = 0; g < QX; ++g)
            for (int k = 0; k < 2; ++k) mbar_init(&xbar[g][k], 1);
        for (int k = 0; k < 2; ++k) mbar_init(&pbar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(quad * 32) << 16) + (uint32_t)(sub * (512 / WPQ));

    const long long plane = (long long)a.mx * a.my;
    const long long u0 = unit_begin(blockIdx.x, a.units, a.nctas);
    const long long u1 = unit_begin(blockIdx.x + 1, a.units, a.nctas);

    int seg = 0;
    for (long long u = u0; u < u1; ++seg) {
        const long long tile = u / a.mz;
        const int za = (int)(u - tile * a.mz);
        const int zb = (int)min((long long)a.mz, (long long)za + (u1 - u));
        u += zb - za;
        long long tt = tile;
        const int txi = (int)(tt % a.tiles_x); tt /= a.tiles_x;
        const int tyi = (int)(tt % a.tiles_y); tt /= a.tiles_y;
        const int b = (int)tt;
        const int x0 = txi * TX, y0 = tyi * TY;
        // input / output vector bases; SPLIT (KKT): vectors b >= bsplit jump (a compile-time
        // variant, so the register-tight p = 4 kernels are untouched)
        // (b is the vector group: vectors b * vp .. b * vp + vp - 1, side by side along x)
        // (PACK: a compile-time variant, so the unpacked production kernels are untouched)
        const int VPK = (GSYNC && PACK) ? ks.vp : 1;
        const int WX = VPK * a.mx;  // packed row width
        auto vsrc = [&](int v) -> long long {
            return (long long)v * a.mz * plane + (SPLIT && v >= ks.bsplit ? ks.src_jump : 0);
        };
        auto vdst = [&](int v) -> long long {
            return (long long)v * a.mz * plane + (SPLIT && v >= ks.bsplit ? ks.dst_jump : 0);
        };
        const long long vbs = vsrc(b);  // (unpacked staging paths: VPK == 1)
        const long long vbd = vdst(b);
        const int gx = x0 + cx;          // packed column of this thread
        // output column of this thread: vector, local column, validity (recomputed at plane retire)
        auto out_col = [&](bool* ok) -> double* {
            if constexpr (!PACK) {
                *ok = gx < a.mx;
                return a.dst + vbd + gx;
            }
            const int vi = min(gx / a.mx, VPK - 1);
            const int vv = b * VPK + vi;
            *ok = gx < WX && vv < a.batch;
            return a.dst + vdst(vv) + (gx - vi * a.mx);
        };

        __syncthreads();
        if constexpr (GSYNC) {
            // halo zeros: the plane bulk copies only ever write in-range rows and columns
            for (int i = threadIdx.x; i < 2 * VSZ; i += blockDim.x) vin[i] = 0.0;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
        }
        if constexpr (YRES) {
            for (int r = 0; r < a.nrounds; ++r) {
                copy_yrows(ycs + (size_t)r * TY * YROW, rs[r], y0);
            }
        }
        {
            double zero[RS::DBL];
#pragma unroll
            for (int k = 0; k < RS::DBL; ++k) zero[k] = 0.0;
            for (int i = 0; i < LW; ++i) ring_st<BW, TIGHTR>(tbase + i * RS::COLS, zero);
        }

        // GSYNC: the byte count of a plane's copies, registered by thread 0 before they are issued
        // GSYNC plane rows: the packed column range [cs, ce) of the tile (halo included) in pieces of
        // one vector each; f(vector, local column, packed column, count) for the existing vectors
        auto plane_pieces = [&](auto&& f) {
            const int cs = max(x0 - P - PADL, 0);
            const int ce = min((min(x0 + TX + P, WX) + 1) & ~1, WX);
            if constexpr (!PACK) {
                f(b, cs, cs, ce - cs);
                return;
            }
            for (int c = cs; c < ce;) {
                const int vi = c / a.mx;
                const int n = min(ce, (vi + 1) * a.mx) - c;
                if (b * VPK + vi < a.batch) f(b * VPK + vi, c - vi * a.mx, c, n);
                c += n;
            }
        };
        auto stage_plane_expect = [&](int buf) {
            if (threadIdx.x == 0) {
                const int rlo = max(0, P - y0), rhi = min(HY, a.my - y0 + P);
                int ncol = 0;
                if constexpr (!PACK) plane_pieces([&](int, int, int, int n) { ncol += n; });  // (PACK: cp.async rows)
                const uint32_t rb = (uint32_t)(ncol * sizeof(double));
                const uint32_t zbytes = (uint32_t)(a.nrounds * NGB * sizeof(double));
                mbar_expect_tx(&pbar[buf], (uint32_t)max(rhi - rlo, 0) * rb + zbytes);
            }
        };
        auto stage_plane = [&](int zp, int buf) {
            if constexpr (GSYNC && PACK) {
                // packed rows: up to ~3 pieces per row, too many bulk copies for the issuing lanes (each
                // costs a uniform-register round trip): every thread copies 16-byte chunks with
                // cp.async (completion: cp.async.wait_group before the plane's CTA barrier); the z
                // record stays one bulk copy on pbar[buf]
                const int cbase = x0 - P - PADL;
                const int rlo = max(0, P - y0), rhi = min(HY, a.my - y0 + P);
                plane_pieces([&](int v, int lx, int c, int n) {
                    const double* srcp = a.src + vsrc(v) + (long long)zp * plane + lx + (long long)(y0 - P) * a.mx;
                    double* dstp = vin + buf * VSZ + (c - cbase);
                    for (int r = rlo + warp; r < rhi; r += NW * WPQ)
                        for (int k = lane; 2 * k < n; k += 32)
                            cp16(dstp + r * HXP + 2 * k, srcp + (long long)r * a.mx + 2 * k);
                });
                cp_commit();
                if (threadIdx.x == 0) {
                    stage_plane_expect(buf);
                    const uint32_t zbytes = (uint32_t)(a.nrounds * NGB * sizeof(double));
                    bulk_g2s(zcs + buf * a.nrounds * NGB, a.bz + (size_t)zp * a.nrounds * NGB, zbytes, &pbar[buf]);
                }
                return;
            }
            if constexpr (GSYNC) {
                // the in-range part of every tile row (widened to an even, 16-byte aligned column
                // range) and the plane's z record, completing on pbar[buf].  Thread 0 registers the
                // byte count first (stage_plane_expect, before the CTA barrier); lane 0 of every
                // warp then issues its share of the row copies (one thread issuing all HY rows
                // delayed warp 0 by a few hundred instructions per plane)
                // (DIST: measured per tile shape; the p = 3, 128-wide sweep ran 1.5 % slower with
                // it, so that shape keeps one issuing thread)
                if (DIST ? lane == 0 : threadIdx.x == 0) {
                    if (!DIST) stage_plane_expect(buf);
                    const int cbase = x0 - P - PADL;
                    const int rlo = max(0, P - y0), rhi = min(HY, a.my - y0 + P);
                    plane_pieces([&](int v, int lx, int c, int n) {
                        double* dstp = vin + buf * VSZ + (c - cbase);
                        const double* srcp = a.src + vsrc(v) + (long long)zp * plane + lx;
                        for (int r = rlo + (DIST ? warp : 0); r < rhi; r += (DIST ? NW * WPQ : 1))
                            bulk_g2s(dstp + r * HXP, srcp + (long long)(y0 - P + r) * a.mx,
                                     (uint32_t)(n * sizeof(double)), &pbar[buf]);
                    });
                    if (!DIST || warp == NW * WPQ - 1) {
                        const uint32_t zbytes = (uint32_t)(a.nrounds * NGB * sizeof(double));
                        bulk_g2s(zcs + buf * a.nrounds * NGB, a.bz + (size_t)zp * a.nrounds * NGB, zbytes,
                                 &pbar[buf]);
                    }
                }
                return;
            }
            double* dstp = vin + buf * VSZ;
            const double* srcp = a.src + vbs + (long long)zp * plane;
            {
                // (tensor-map boxes would give free OOB zero fill, but starting a box at a
                // negative coordinate faults on this stack — tools/tma_test.cu — so the halo'd
                // plane tile is staged with 8-byte cp.async)
                // rows by warp, contiguous columns by lane: no per-element division
                for (int r = warp; r < HY; r += NW * WPQ) {
                    const int gy = y0 - P + r;
                    const bool rowok = gy >= 0 && gy < a.my;
                    const double* srow = srcp + (long long)gy * a.mx + (x0 - P);
                    for (int c = lane; c < G_::HX; c += 32) {
                        const int gxx = x0 - P + c;
                        const bool ok = rowok && gxx >= 0 && gxx < a.mx;
                        cp8(dstp + r * HXP + PADL + c, ok ? srow + c : a.src, ok);
                    }
                }
            }
            double* zdst = zcs + buf * a.nrounds * NGB;
            for (int i = threadIdx.x; i < a.nrounds * NG * BW; i += blockDim.x) {
                const int r = i / (NG * BW), rem = i - r * NG * BW;
                const int g = rem / BW, j = rem - g * BW;
                const RoundT& R = rs[r];
                const int zo = zp - P + ((j - (zp - P)) % BW + BW) % BW;
                const bool ok = zo >= 0 && zo < a.mz;
                cp8(zdst + r * NGB + rem, ok ? a.bz + ((size_t)R.gf[g] * a.mz + zo) * BW + (zp - zo + P) : a.bz, ok);
            }
        };
        auto stage_xc = [&](int r, int buf) {
            // each factor's band rows for the tile's columns (rows) are one contiguous block
            // (entries past mx / my read the band allocation's padding or the next factor and
            // are never used for an output)
            const RoundT& R = rs[r];
            double* dstp = xcs + buf * NX * TX * BW;
            if constexpr (GSYNC) {
                // the column group's 32 columns of every x-entry
                if (gprod) {
                    mbar_expect_tx(&xbar[grp][buf], (uint32_t)(NX * TXW * BW * sizeof(double)));
                    if constexpr (XREC) {
                        // the group's x record of round r: one copy of NX x 32 band rows, laid out
                        // [NX][32][BW] at the group's slot of the buffer (k_build_xtab)
                        const int nblk = (a.mx + TXW - 1) / TXW;
                        bulk_g2s(dstp + grp * NX * TXW * BW, a.bx + ((size_t)r * nblk + x0 / TXW + grp) * NX * TXW * BW,
                                 (uint32_t)(NX * TXW * BW * sizeof(double)), &xbar[grp][buf]);
                        return;
                    }
                    if constexpr (!PACK) {
#pragma unroll
                        for (int e = 0; e < NX; ++e)
                            bulk_g2s(dstp + e * TX * BW + grp * TXW * BW,
                                     a.bx + ((size_t)R.xf[e] * a.mx + x0 + grp * TXW) * BW,
                                     (uint32_t)(TXW * BW * sizeof(double)), &xbar[grp][buf]);
                        return;
                    }
                    // packed columns [c0, c0 + 32) in pieces of one vector each (the band rows of the
                    // local columns; columns past the packed width read the last vector's padding rows)
                    const int c0 = x0 + grp * TXW;
                    for (int c = c0; c < c0 + TXW;) {
                        const int vi = min(c / a.mx, VPK - 1);
                        const int n = (vi == VPK - 1 ? c0 + TXW : min(c0 + TXW, (vi + 1) * a.mx)) - c;
#pragma unroll
                        for (int e = 0; e < NX; ++e)
                            bulk_g2s(dstp + e * TX * BW + (c - x0) * BW,
                                     a.bx + ((size_t)R.xf[e] * a.mx + (c - vi * a.mx)) * BW,
                                     (uint32_t)(n * BW * sizeof(double)), &xbar[grp][buf]);
                        c += n;
                    }
                }
            } else if constexpr (TMA) {
                if (threadIdx.x == 0) {
                    mbar_expect_tx(&xbar[0][buf], (uint32_t)(NX * TX * BW * sizeof(double)));
#pragma unroll
                    for (int e = 0; e < NX; ++e)
                        bulk_g2s(dstp + e * TX * BW, a.bx + ((size_t)R.xf[e] * a.mx + x0) * BW,
                                 (uint32_t)(TX * BW * sizeof(double)), &xbar[0][buf]);
                }
            } else {
#pragma unroll
                for (int e = 0; e < NX; ++e) {
                    const double* src = a.bx + ((size_t)R.xf[e] * a.mx + x0) * BW;
                    for (int i = threadIdx.x; i < TX * BW; i += blockDim.x) cp8(dstp + e * TX * BW + i, src + i, true);
                }
            }
            // y rows re-pitched (16-byte aligned records) for LDS.128 broadcasts
            if (YRES) return;
            copy_yrows(ycs + (size_t)buf * TY * YROW, R, y0);
        };

        if constexpr (GSYNC && DIST && !PACK) {
            stage_plane_expect(0);
            __syncthreads();  // the expected byte count is registered before any copy completes
        }
        stage_plane(za, 0);
        stage_xc(0, 0);
        cp_commit();
        int pbuf = 0, xbuf = 0;
        // single-round plans (R <= 4 mass): every plane of the segment uses the same x-coefficients, so
        // they are staged and loaded into registers once per segment (GSYNC path)
        // (the packed 64-wide p = 3 mass kernel only, c4's: the stiffness kernels have more than one round
        // for every R > 1, and the other mass variants spill 40-200 B when the registers live that long;
        // they keep the per-round array)
        constexpr bool XONCE = GSYNC && !std::is_same<S, ShapeStiffA>::value && P == 3 && QX == 2 && PACK;
        const bool xonce = XONCE && a.nrounds == 1;
        double xr_seg[XONCE ? NX : 1][XONCE ? BW : 1];
        for (int zp = za; zp < zb; ++zp) {
            for (int r = 0; r < a.nrounds; ++r) {
                const bool last_round = (r == a.nrounds - 1);
                EXP_T(0);
                if constexpr (GSYNC) {
                    tm_wait_st();
#ifdef IGALR_EXP_TIMERS
                    exp_tw += clock64() - exp_t[0];
#endif
                    if (r == 0) {  // new plane buffer: CTA barrier, then request plane z'+1
                        cp_wait<0>();  // (resident y-coefficients at a segment start)
                        if (DIST && !PACK && zp + 1 < zb) stage_plane_expect(pbuf ^ 1);
#ifdef IGALR_EXP_TIMERS
                        exp_tb = clock64();
#endif
                        __syncthreads();
#ifdef IGALR_EXP_TIMERS
                        exp_bar += clock64() - exp_tb;
#endif
#ifdef IGALR_EXP_TIMERS
                        exp_tb = clock64();
#endif
                        if (zp + 1 < zb) stage_plane(zp + 1, pbuf ^ 1);
#ifdef IGALR_EXP_TIMERS
                        exp_sp += clock64() - exp_tb;
                        exp_tb = clock64();
#endif
                        mbar_wait(&pbar[pbuf], (pph >> pbuf) & 1);
#ifdef IGALR_EXP_TIMERS
                        exp_pw += clock64() - exp_tb;
#endif
                        pph ^= 1u << pbuf;
                    } else {
                        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(GTHREADS) : "memory");
                    }
                    // the group is past round r-1: its x buffer can take round r+1
#ifdef IGALR_EXP_TIMERS
                    exp_tb = clock64();
#endif
                    if constexpr (!XONCE) {
                        if (!last_round) stage_xc(r + 1, xbuf ^ 1);
                        else if (zp + 1 < zb) stage_xc(0, xbuf ^ 1);
                    } else if (!xonce) {
                        if (!last_round) stage_xc(r + 1, xbuf ^ 1);
                        else if (zp + 1 < zb) stage_xc(0, xbuf ^ 1);
                    }
#ifdef IGALR_EXP_TIMERS
                    exp_sx += clock64() - exp_tb;
                    exp_tb = clock64();
#endif
                    if constexpr (!XONCE) {
                        mbar_wait(&xbar[grp][xbuf], (xph >> xbuf) & 1);
                        xph ^= 1u << xbuf;
                    } else if (!xonce || zp == za) {
                        mbar_wait(&xbar[grp][xbuf], (xph >> xbuf) & 1);
                        xph ^= 1u << xbuf;
                    }
#ifdef IGALR_EXP_TIMERS
                    exp_xw += clock64() - exp_tb;
#endif
                    EXP_T(1);
                } else {
                    if constexpr (TMA) {  // x-coefficients arrive by cp.async.bulk (mbarrier)
                        mbar_wait(&xbar[0][xbuf], (xph >> xbuf) & 1);
                        xph ^= 1u << xbuf;
                    }
                    cp_wait<0>();
                    tm_wait_st();
                    __syncthreads();
                    if (!last_round) stage_xc(r + 1, xbuf ^ 1);
                    else if (zp + 1 < zb) stage_xc(0, xbuf ^ 1);
                    if (r == 0 && zp + 1 < zb) stage_plane(zp + 1, pbuf ^ 1);
                    cp_commit();
                }

                const RoundT& R = rs[r];
                const double* vt = vin + pbuf * VSZ + row0 * HXP + PADL + cx;
                const double* xc = xcs + xbuf * NX * TX * BW;
                const double* yc = ycs + (size_t)(YRES ? r : xbuf) * TY * YROW + (size_t)row0 * YROW;
                const double* zc = zcs + pbuf * a.nrounds * NGB + r * NGB;
                double xr[NX][BW];
                if constexpr (XONCE) {
                    if (!xonce || zp == za) {
#pragma unroll
                        for (int e = 0; e < NX; ++e)
#pragma unroll
                            for (int k = 0; k < BW; ++k)
                                xr_seg[e][k] = XREC ? xc[((grp * NX + e) * TXW + lane) * BW + k] : xc[(e * TX + cx) * BW + k];
                    }
#pragma unroll
                    for (int e = 0; e < NX; ++e)
#pragma unroll
                        for (int k = 0; k < BW; ++k) xr[e][k] = xr_seg[e][k];
                } else {
#pragma unroll
                    for (int e = 0; e < NX; ++e)
#pragma unroll
                        for (int k = 0; k < BW; ++k)
                            xr[e][k] = XREC ? xc[((grp * NX + e) * TXW + lane) * BW + k]  // (x-record layout)
                                            : xc[(e * TX + cx) * BW + k];
                }
                // p = 4 stiffness on the GSYNC path reads the (pre-scaled) z record from shared
                // memory in the Z stage (broadcast loads) instead of holding NG x BW doubles in
                // registers: its sweep sits at the 255-register cliff.  The freed registers take the
                // pair ratios and an early TMEM ring load (c5 stiffness 1.86 -> 1.77 ms; the mass
                // shape is faster with register-resident coefficients)
                constexpr bool ZSMEM = GSYNC && P >= IGALR_ZSMEM_P && std::is_same<S, ShapeStiffA>::value;
                double zr[ZSMEM ? 1 : NG][ZSMEM ? 1 : BW];
                if constexpr (!ZSMEM) {
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const double gsc = GSYNC ? 1.0 : R.gs[g];  // (the GSYNC z record is pre-scaled)
#pragma unroll
                        for (int j = 0; j < BW; ++j) zr[g][j] = zc[g * BW + j] * gsc;
                    }
                }
                double pc[NPAIR];
#pragma unroll
                for (int j = 0; j < NPAIR; ++j) pc[j] = R.pc[j];
                const int zret = zp - P;
                const int jret = ((zret % BW) + BW) % BW;
                bool ret_valid = false, ret_complete = false;
                if (last_round && zret >= 0 && zret < a.mz) {
                    ret_valid = true;
                    const int lo = max(0, zret - P), hi = min(a.mz - 1, zret + P);
                    ret_complete = lo >= za && hi <= zb - 1;
                }
                if (SPLIT && a.accumulate && r == max(0, a.nrounds - 2) && zret >= 0 && zret < a.mz &&
                    max(0, zret - P) >= za && min(a.mz - 1, zret + P) <= zb - 1) {
                    // the plane this step retires is read-modify-written: its rows go to L2 a round
                    // ahead (an exposed HBM read per plane otherwise).  The KKT's accumulating
                    // stiffness launch only (SPLIT): in the other kernels the extra code costs more
                    // (register allocation) than the rare accumulate saves
                    bool ok;
                    const double* prow = out_col(&ok) + (long long)zret * plane + (long long)(y0 + row0) * a.mx;
                    const int nrow = min(LW, a.my - (y0 + row0));
                    if (ok)
                        for (int i = 0; i < nrow; ++i) asm volatile("prefetch.global.L2 [%0];" ::"l"(prow + (long long)i * a.mx));
                }

                double w[NX][BW];
#pragma unroll
                for (int e = 0; e < NX; ++e)
#pragma unroll
                    for (int k = 0; k < BW; ++k) w[e][k] = 0.0;

                // X stage of sweep row `step` into window slot Q (compile-time)
                auto xstage = [&](auto Qc, int step) {
                    constexpr int Q = decltype(Qc)::value;
#ifdef IGALR_EXP_EMPTY
                    w[0][Q] = vt[step * HXP] * xr[Q % NX][Q % BW];
                    return;
#endif
                    double v[BW];
#pragma unroll
                    for (int k = 0; k < BW; ++k) v[k] = vt[step * HXP + k];
#pragma unroll
                    for (int e = 0; e < NX; ++e) {
                        double acc = xr[e][0] * v[0];
#pragma unroll
                        for (int k = 1; k < BW; ++k) acc = fma(xr[e][k], v[k], acc);
                        w[e][Q] = acc;
                    }
                };
                // Y + Z stages for output row i (window newest row in slot Q)
                auto yzstage = [&](auto Qc, int i) {
                    constexpr int Q = decltype(Qc)::value;
                    const uint32_t tp = tbase + i * RS::COLS;
                    uint32_t rr[RS::DBL * 2];
                    // TMEM load in flight during the Y stage (p=3); p=4 issues it after the Y stage:
                    // its 18 registers would push the Y stage into spills
                    constexpr bool EARLY_RING = (P <= 3) || ZSMEM;
#ifndef IGALR_EXP_NOZ
                    if constexpr (EARLY_RING) ring_issue<BW, TIGHTR>(tp, rr);
#endif
                    double G[NG];
#pragma unroll
                    for (int g = 0; g < NG; ++g) G[g] = 0.0;
                    const double* ycr = yc + (size_t)i * YROW;
#ifdef IGALR_EXP_EMPTY
                    G[0] = w[0][Q] * ycr[0];
                    if (false)
#endif
                    if constexpr (YP::TAP) {
                        // tap-major: all NPAIR chains advance together (NPAIR independent chains);
                        // the NY coefficients of tap k are NYP/2 broadcast LDS.128
                        double acc[NPAIR];
#pragma unroll
                        for (int k = 0; k < BW; ++k) {
                            double yv[NYP];
                            const double2* y2 = reinterpret_cast<const double2*>(ycr + k * NYP);
#pragma unroll
                            for (int h = 0; h < NYP / 2; ++h) {
                                const double2 t2 = y2[h];
                                yv[2 * h] = t2.x;
                                yv[2 * h + 1] = t2.y;
                            }
#pragma unroll
                            for (int ii = 0; ii < NPAIR; ++ii) {
                                const int j = S::ord(ii);
                                const double wv = w[S::px(j)][(Q + 1 + k) % BW];
                                acc[j] = k == 0 ? yv[S::py(j)] * wv : fma(yv[S::py(j)], wv, acc[j]);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < NPAIR; ++j)
                            if (S::lead(j)) G[S::pg(j)] = acc[j];
#pragma unroll
                        for (int j = 0; j < NPAIR; ++j)
                            if (!S::lead(j)) G[S::pg(j)] = fma((P <= 3 || ZSMEM) ? pc[j] : R.pc[j], acc[j], G[S::pg(j)]);
                    } else {
#pragma unroll
                    for (int f = 0; f < NY; ++f) {
                        double yv[BWP];
                        const double2* y2 = reinterpret_cast<const double2*>(ycr + (size_t)f * BWP);
#pragma unroll
                        for (int k = 0; k < BWP / 2; ++k) {  // broadcast LDS.128
                            const double2 t2 = y2[k];
                            yv[2 * k] = t2.x;
                            yv[2 * k + 1] = t2.y;
                        }
#pragma unroll
                        for (int j = 0; j < NPAIR; ++j) {
                            if (S::py(j) != f) continue;
                            const int e = S::px(j);
                            const int g = S::pg(j);
                            if (S::lead(j)) {
                                // lead pair: accumulate straight into its group value
#pragma unroll
                                for (int k = 0; k < BW; ++k) G[g] = fma(yv[k], w[e][(Q + 1 + k) % BW], G[g]);
                            } else {
                                double u = yv[0] * w[e][(Q + 1) % BW];
#pragma unroll
                                for (int k = 1; k < BW; ++k) u = fma(yv[k], w[e][(Q + 1 + k) % BW], u);
                                // (p=4: the ratio is re-read from shared memory: register pressure)
                                G[g] = fma((P <= 3 || ZSMEM) ? pc[j] : R.pc[j], u, G[g]);
                            }
                        }
                    }
                    }
                    double ring[RS::DBL];
#ifndef IGALR_EXP_NOZ
                    if constexpr (!EARLY_RING) ring_issue<BW, TIGHTR>(tp, rr);
#endif
#ifdef IGALR_EXP_NOZ
                    (void)rr; (void)ring; (void)tp;
                    exp_sink = fma(G[0] + G[1], G[NG - 1] + zr[0][Q % BW], exp_sink);
#else
                    ring_wait<BW, TIGHTR>(rr, ring);
#pragma unroll
                    for (int g = 0; g < NG; ++g)
#pragma unroll
                        for (int j = 0; j < BW; ++j)
                            ring[j] = fma(ZSMEM ? zc[g * BW + j] : zr[ZSMEM ? 0 : g][ZSMEM ? 0 : j], G[g], ring[j]);
                    ring_st<BW, TIGHTR>(tp, ring);
#endif
                };
                constexpr int HYW = LW + 2 * P;        // rows swept by this warp
                constexpr int NFULL = (HYW - BW) / BW;  // full blocks after block 0
                constexpr int REM = (HYW - BW) % BW;
                EXP_T(2);
                // block 0: the first 2P rows only fill the window
                static_for<0, BW>([&](auto Qc) {
                    constexpr int Q = decltype(Qc)::value;
                    xstage(Qc, Q);
                    if constexpr (Q >= 2 * P) yzstage(Qc, Q - 2 * P);
                });
#pragma unroll 1
                for (int blk = 1; blk <= NFULL; ++blk) {
                    static_for<0, BW>([&](auto Qc) {
                        const int step = blk * BW + decltype(Qc)::value;
                        xstage(Qc, step);
                        yzstage(Qc, step - 2 * P);
                    });
                }
                static_for<0, REM>([&](auto Qc) {
                    const int step = (NFULL + 1) * BW + decltype(Qc)::value;
                    xstage(Qc, step);
                    yzstage(Qc, step - 2 * P);
                });
                EXP_T(3);
                if (ret_valid) {
                    // plane zret is final: write it (or its partial) out and clear its slot.  The
                    // LW TMEM loads are issued in chunks of 8 with one wait per chunk (a load+wait per
                    // row serialises LW TMEM round trips)
                    tm_wait_st();
                    double rv[LW];
                    static_for<0, (LW + 7) / 8>([&](auto Cc) {
                        constexpr int c0 = decltype(Cc)::value * 8;
                        constexpr int cn = LW - c0 < 8 ? LW - c0 : 8;
                        uint32_t lo[8], hi[8];
#pragma unroll
                        for (int q = 0; q < cn; ++q)
                            asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                                         : "=r"(lo[q]), "=r"(hi[q])
                                         : "r"(tbase + (c0 + q) * RS::COLS + 2 * jret));
#pragma unroll
                        for (int q = cn; q < 8; ++q) lo[q] = hi[q] = 0u;
                        asm volatile("tcgen05.wait::ld.sync.aligned;"
                                     : "+r"(lo[0]), "+r"(hi[0]), "+r"(lo[1]), "+r"(hi[1]), "+r"(lo[2]), "+r"(hi[2]),
                                       "+r"(lo[3]), "+r"(hi[3]), "+r"(lo[4]), "+r"(hi[4]), "+r"(lo[5]), "+r"(hi[5]),
                                       "+r"(lo[6]), "+r"(hi[6]), "+r"(lo[7]), "+r"(hi[7]));
#pragma unroll
                        for (int q = 0; q < cn; ++q) rv[c0 + q] = __hiloint2double(hi[q], lo[q]);
                    });
#pragma unroll
                    for (int i = 0; i < LW; ++i) tm_st1(tbase + i * RS::COLS + 2 * jret, 0.0);
                    // (measured per shape: the p = 4 mass kernel is 2.7 % faster with per-row branches)
                    constexpr bool SPLITSTORE = !(P >= 4 && !std::is_same<S, ShapeStiffA>::value);
                    if constexpr (SPLITSTORE) {
                        // stores: the plane-uniform cases (complete / partial, accumulate) are split
                        // outside the row loop, so each row is one predicated store (no per-row branches)
                        const int nrow = min(LW, a.my - (y0 + row0));  // rows of this warp inside the mesh
                        bool colok;
                        double* dcol = out_col(&colok);
                        if (ret_complete) {
                            double* drow = dcol + (long long)zret * plane + (long long)(y0 + row0) * a.mx;
                            if (a.accumulate) {
#pragma unroll
                                for (int i = 0; i < LW; ++i)
                                    if (colok && i < nrow) drow[(long long)i * a.mx] += a.scale * rv[i];
                            } else {
#pragma unroll
                                for (int i = 0; i < LW; ++i)
                                    if (colok && i < nrow) drow[(long long)i * a.mx] = a.scale * rv[i];
                            }
                        } else {
                            const int slot = partial_slot(zret, za, zb, P);
                            double* srow = a.scratch + ((((size_t)blockIdx.x * NSEG + seg) * 4 * P + slot) * TY + row0) * TX + cx;
#pragma unroll
                            for (int i = 0; i < LW; ++i)
                                if (colok && i < nrow) srow[(size_t)i * TX] = a.scale * rv[i];
                        }
                    } else {
                        bool colok;
                        double* dcol = out_col(&colok);
#pragma unroll
                        for (int i = 0; i < LW; ++i) {
                            const double val = rv[i];
                            const int gy = y0 + row0 + i;
                            if (gy < a.my && colok) {
                                if (ret_complete) {
                                    double* o = dcol + (long long)zret * plane + (long long)gy * a.mx;
                                    *o = (a.accumulate ? *o : 0.0) + a.scale * val;
                                } else {
                                    const int slot = partial_slot(zret, za, zb, P);
                                    a.scratch[((((size_t)blockIdx.x * NSEG + seg) * 4 * P + slot) * TY + row0 + i) * TX + cx] =
                                        a.scale * val;
                                }
                            }
                        }
                    }
                }
                EXP_T(4);
                if (last_round) pbuf ^= 1;
                xbuf ^= 1;
            }
        }
        tm_wait_st();
        __syncthreads();
        bool fcolok;
        double* fdcol = out_col(&fcolok);
        for (int i = 0; i < LW; ++i) {
            const uint32_t tp = tbase + i * RS::COLS;
            double ring[RS::DBL];
            ring_ld<BW, TIGHTR>(tp, ring);
            const int gy = y0 + row0 + i;
#pragma unroll
            for (int s = 0; s < 2 * P; ++s) {
                const int zo = zb - P + s;
                if (zo < 0 || zo >= a.mz) continue;
                const int j = zo % BW;
                double val = 0.0;
#pragma unroll
                for (int jj = 0; jj < BW; ++jj)
                    if (jj == j) val = ring[jj];
                if (gy < a.my && fcolok) {
                    const int lo = max(0, zo - P), hi = min(a.mz - 1, zo + P);
                    const bool complete = lo >= za && hi <= zb - 1;
                    if (complete) {
                        double* o = fdcol + (long long)zo * plane + (long long)gy * a.mx;
                        *o = (a.accumulate ? *o : 0.0) + a.scale * val;
                    } else {
                        const int slot = partial_slot(zo, za, zb, P);
                        a.scratch[((((size_t)blockIdx.x * NSEG + seg) * 4 * P + slot) * TY + row0 + i) * TX + cx] =
                            a.scale * val;
                    }
                }
            }
        }
    }
#ifdef IGALR_EXP_NOZ
    if (a.accumulate == 12345) a.dst[threadIdx.x] = exp_sink;
#endif
#ifdef IGALR_EXP_TIMERS
    if (lane == 0 && (blockIdx.x % 37) == 0)
        printf("EXPT cta %d warp %d total %lld sync %lld load %lld sweep %lld retire %lld bar %lld pwait %lld tmw %lld "
               "splane %lld sxc %lld xwait %lld\n",
               blockIdx.x, warp, clock64() - exp_t_start, exp_acc[0], exp_acc[1], exp_acc[2], exp_acc[3], exp_bar, exp_pw,
               exp_tw, exp_sp, exp_sx, exp_xw);
#endif
#undef EXP_T
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_sh));
}

template <class S, int P, int LW, int WPQ, int QX, bool YRES>
size_t smem_bytes_canon(int nrounds) {
    constexpr int TXT = 32 * QX, TYT = LW * WPQ * (4 / QX);
    using G_ = GeoC<P, TXT, TYT>;  // (padded pitch; the TMA variant uses the dense pitch, <= this)
    const size_t ys = YRES ? (size_t)nrounds : 2;
    const size_t vsz = (G_::HY * G_::HXP + 15) & ~(size_t)15;
    return sizeof(double) * (2 * vsz + 2 * S::NX * TXT * G_::BW + ys * TYT * YPitch<S::NY, G_::BW>::ROW +
                             2 * (size_t)nrounds * ZPitch<S::NG, G_::BW>::NGB) +
           sizeof(RoundC<S>) * nrounds + 64;
}

// Sum partial planes.  Only planes within P of a CTA-range boundary inside a tile can have
// inputs in several CTA ranges; one CTA per (boundary, plane offset) finds the contributing
// CTA segments once (thread 0) and all threads add their scratch entries in increasing CTA
// order (deterministic).
static __global__ void k_fixup(const Args2 a, int P, int L) {
    __shared__ int s_valid, s_n, s_b, s_zo, s_txi, s_tyi;
    __shared__ long long s_off[8];
    const int kb = 1 + blockIdx.x / (2 * P);
    const int s = blockIdx.x % (2 * P);
    if (threadIdx.x == 0) {
        s_valid = 0;
        s_n = 0;
        const long long ub = unit_begin(kb, a.units, a.nctas);
        const long long tile = ub / a.mz;
        const int zbnd = (int)(ub - tile * a.mz);
        const int zo = zbnd - P + s;
        if (zbnd != 0 && zo >= 0 && zo < a.mz) {
            long long tt = tile;
            s_txi = (int)(tt % a.tiles_x); tt /= a.tiles_x;
            s_tyi = (int)(tt % a.tiles_y); tt /= a.tiles_y;
            s_b = (int)tt;
            s_zo = zo;
            const int lo = max(0, zo - P), hi = min(a.mz - 1, zo + P);
            const long long ulo = tile * a.mz + lo, uhi = tile * a.mz + hi;
            long long k0 = kb - 1, k1 = kb;
            while (k0 > 0 && unit_begin(k0, a.units, a.nctas) > ulo) --k0;
            while (k1 + 1 < a.nctas && unit_begin(k1 + 1, a.units, a.nctas) <= uhi) ++k1;
            for (long long k = k0; k <= k1 && s_n < 8; ++k) {
                const long long cu0 = unit_begin(k, a.units, a.nctas), cu1 = unit_begin(k + 1, a.units, a.nctas);
                int seg = 0;
                for (long long u = cu0; u < cu1; ++seg) {
                    const long long t2 = u / a.mz;
                    const int sa = (int)(u - t2 * a.mz);
                    const int sb = (int)min((long long)a.mz, (long long)sa + (cu1 - u));
                    if (t2 == tile) {
                        const int slot = partial_slot(zo, sa, sb, P);
                        s_off[s_n++] = (((long long)k * NSEG + seg) * 4 * P + slot) * (long long)a.tyt * a.txt;
                        break;
                    }
                    u += sb - sa;
                }
            }
            s_valid = 1;
        }
    }
    __syncthreads();
    if (!s_valid) return;
    const long long plane = (long long)a.mx * a.my;
    const long long obase = (long long)s_b * a.mz * plane + (long long)s_zo * plane;
    for (int p = threadIdx.x; p < a.tyt * a.txt; p += blockDim.x) {
        const int i = p / a.txt, cx = p - i * a.txt;
        const int gx = s_txi * a.txt + cx, gy = s_tyi * a.tyt + i;
        if (gx >= a.mx || gy >= a.my) continue;
        double sum = 0.0;
        for (int c = 0; c < s_n; ++c) sum += a.scratch[s_off[c] + p];
        const long long o = obase + (long long)gy * a.mx + gx;
        a.dst[o] = (a.accumulate ? a.dst[o] : 0.0) + sum;
    }
}

// Fixup of the canonical kernels, driven by a host-built table (fixup_table): one CTA per partial
// output plane of a tile, summing its contributors' scratch planes in CTA order (deterministic;
// no atomics, no on-device contributor search).  Each thread sums 4 consecutive points per step,
// with all partial loads of a thread issued before its stores.
struct FixEnt {
    int b, zo, txi, tyi;
    int n, pad;
    long long off[2 * 4 + 1];  // scratch offsets of the contributors (<= 2P+1), CTA order
};
static __global__ void __launch_bounds__(256) k_fixup_tab(const Args2 a, const FixEnt* __restrict__ tab, const KSplit ks) {
    const FixEnt& E = tab[blockIdx.x];
    const int TY = a.tyt, TX = a.txt;
    const long long plane = (long long)a.mx * a.my;
    const int WX = ks.vp * a.mx;  // packed row width (E.b is the vector group)
    // element offset of packed column gx in row gy of plane E.zo, or -1 outside the vectors
    auto out_off = [&](int gx, int gy) -> long long {
        const int vi = min(gx / a.mx, ks.vp - 1);
        const int vv = E.b * ks.vp + vi;
        if (gx >= WX || vv >= a.batch) return -1;
        return (long long)vv * a.mz * plane + (vv >= ks.bsplit ? ks.dst_jump : 0) + (long long)E.zo * plane +
               (long long)gy * a.mx + (gx - vi * a.mx);
    };
    const int n = E.n;
    const int nq = TY * TX / 4;
    for (int q0 = threadIdx.x; q0 < nq; q0 += 4 * blockDim.x) {
        double4 acc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[t] = make_double4(0.0, 0.0, 0.0, 0.0);
        for (int c = 0; c < n; ++c) {
            const double2* src = reinterpret_cast<const double2*>(a.scratch + E.off[c]);
            double2 v[4][2];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int q = q0 + t * blockDim.x;
                if (q < nq) {
                    v[t][0] = __ldcg(src + 2 * q);
                    v[t][1] = __ldcg(src + 2 * q + 1);
                } else {
                    v[t][0] = v[t][1] = make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                acc[t].x += v[t][0].x;
                acc[t].y += v[t][0].y;
                acc[t].z += v[t][1].x;
                acc[t].w += v[t][1].y;
            }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int q = q0 + t * blockDim.x;
            if (q >= nq) continue;
            const int p = 4 * q;
            const int i = p / TX, cx = p - i * TX;
            const int gy = E.tyi * TY + i;
            if (gy >= a.my) continue;
            const int gx0 = E.txi * TX + cx;
            const long long o0 = out_off(gx0, gy);
            const int lx0 = gx0 - min(gx0 / a.mx, ks.vp - 1) * a.mx;
            // whole aligned quad inside one vector: one 32-byte access
            if (o0 >= 0 && lx0 + 3 < a.mx && ((uintptr_t)(a.dst + o0) & 31) == 0) {
                double4* d4 = reinterpret_cast<double4*>(a.dst + o0);
                double4 r = acc[t];
                if (a.accumulate) {
                    const double4 old = *d4;
                    r.x += old.x;
                    r.y += old.y;
                    r.z += old.z;
                    r.w += old.w;
                }
                *d4 = r;
                continue;
            }
            const double vv[4] = {acc[t].x, acc[t].y, acc[t].z, acc[t].w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const long long o = out_off(gx0 + w, gy);
                if (o < 0) continue;
                a.dst[o] = (a.accumulate ? a.dst[o] : 0.0) + vv[w];
            }
        }
    }
}

// Variant for launches with few table entries and many contributors per entry (small meshes: one CTA per
// (tile, plane) unit, up to 2P+1 contributors): FIXSPLIT blocks per entry, one quad of points per thread
// and pass, the loads of all contributors of a quad issued together (one memory round trip instead of
// 2P+1).  Same summation order as k_fixup_tab (c2: 12.3 -> about 7 us).
constexpr int FIXSPLIT = 4;
constexpr int FIXMAX = 2 * 4 + 1;  // contributors per entry (FixEnt::off)
static __global__ void __launch_bounds__(256) k_fixup_tab_wide(const Args2 a, const FixEnt* __restrict__ tab, const KSplit ks) {
    const FixEnt& E = tab[blockIdx.x / FIXSPLIT];
    const int TY = a.tyt, TX = a.txt;
    const long long plane = (long long)a.mx * a.my;
    const int WX = ks.vp * a.mx;  // packed row width (E.b is the vector group)
    // element offset of packed column gx in row gy of plane E.zo, or -1 outside the vectors
    auto out_off = [&](int gx, int gy) -> long long {
        const int vi = min(gx / a.mx, ks.vp - 1);
        const int vv = E.b * ks.vp + vi;
        if (gx >= WX || vv >= a.batch) return -1;
        return (long long)vv * a.mz * plane + (vv >= ks.bsplit ? ks.dst_jump : 0) + (long long)E.zo * plane +
               (long long)gy * a.mx + (gx - vi * a.mx);
    };
    const int n = E.n;
    const int nq = TY * TX / 4;
    for (int q = (blockIdx.x % FIXSPLIT) * blockDim.x + threadIdx.x; q < nq; q += FIXSPLIT * blockDim.x) {
        double2 v[FIXMAX][2];
#pragma unroll
        for (int c = 0; c < FIXMAX; ++c) {
            if (c < n) {
                const double2* src = reinterpret_cast<const double2*>(a.scratch + E.off[c]);
                v[c][0] = __ldcg(src + 2 * q);
                v[c][1] = __ldcg(src + 2 * q + 1);
            }
        }
        double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
        for (int c = 0; c < FIXMAX; ++c) {  // (contributors in CTA order: deterministic)
            if (c < n) {
                acc.x += v[c][0].x;
                acc.y += v[c][0].y;
                acc.z += v[c][1].x;
                acc.w += v[c][1].y;
            }
        }
        {
            const int p = 4 * q;
            const int i = p / TX, cx = p - i * TX;
            const int gy = E.tyi * TY + i;
            if (gy >= a.my) continue;
            const int gx0 = E.txi * TX + cx;
            const long long o0 = out_off(gx0, gy);
            const int lx0 = gx0 - min(gx0 / a.mx, ks.vp - 1) * a.mx;
            // whole aligned quad inside one vector: one 32-byte access
            if (o0 >= 0 && lx0 + 3 < a.mx && ((uintptr_t)(a.dst + o0) & 31) == 0) {
                double4* d4 = reinterpret_cast<double4*>(a.dst + o0);
                double4 r = acc;
                if (a.accumulate) {
                    const double4 old = *d4;
                    r.x += old.x;
                    r.y += old.y;
                    r.z += old.z;
                    r.w += old.w;
                }
                *d4 = r;
                continue;
            }
            const double vv[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const long long o = out_off(gx0 + w, gy);
                if (o < 0) continue;
                a.dst[o] = (a.accumulate ? a.dst[o] : 0.0) + vv[w];
            }
        }
    }
}

template <int P, int L, int NX, int NP, int NG, int NY>
size_t smem_bytes(int nrounds) {
    using G_ = Geo<P, L>;
    constexpr int BW = G_::BW;
    return sizeof(double) * (2 * G_::HY * G_::HXP + 2 * NX * TX * BW + (size_t)nrounds * NY * L * BW +
                             2 * (size_t)nrounds * NG * BW) +
           sizeof(Round2<NX, NP, NG>) * nrounds + 64;
}

}  // namespace f2

// ---------------------------------------------------------------------------------- host
namespace {

template <int NX, int NP, int NG, int NY>
bool build_rounds2(const Plan& pl, std::vector<f2::Round2<NX, NP, NG>>* out) {
    out->clear();
    for (const Round& R : pl.rounds) {
        // split pairs that feed several groups into one pair per group
        f2::Round2<NX, NP, NG> F;
        memset(&F, 0, sizeof F);
        if (R.nx > NX || R.ng > NG) return false;
        F.nx = R.nx;
        F.ng = R.ng;
        for (int e = 0; e < R.nx; ++e) F.xf[e] = R.xf[e];
        for (int g = 0; g < R.ng; ++g) F.gf[g] = R.gf[g];
        int np = 0;
        bool lead_done[kMaxG] = {false, false, false, false, false};
        for (int g = 0; g < R.ng; ++g) {
            for (int e = 0; e < R.ne[g]; ++e) {
                if (np >= NP) return false;
                const int j = R.ep[g][e];
                const int yfac = R.pf[j];
                int s = -1;
                for (int t = 0; t < F.nyf; ++t)
                    if (F.yf[t] == yfac) s = t;
                if (s < 0) {
                    if (F.nyf >= NY) return false;
                    s = F.nyf++;
                    F.yf[s] = yfac;
                }
                F.pyf[np] = s;
                F.px[np] = R.px[j];
                F.pg[np] = g;
                const double c = R.ec[g][e];
                if (!lead_done[g] && c != 0.0) {
                    F.plead[np] = 1;
                    F.pc[np] = 1.0;
                    F.gs[g] = c;
                    lead_done[g] = true;
                } else {
                    F.plead[np] = 0;
                    F.pc[np] = lead_done[g] ? c / F.gs[g] : 0.0;
                }
                ++np;
            }
            if (!lead_done[g]) F.gs[g] = 0.0;
        }
        F.np = np;
        out->push_back(F);
    }
    return !out->empty() && (int)out->size() <= f2::kMaxRounds2;
}

// shape of the fused-v2 round tables per part
constexpr int kSX = 4, kSP = 9, kSG = 4, kSY = 4;  // stiffness part
constexpr int kMX = 1, kMP = 1, kMG = 1, kMY = 1;  // mass part

template <int P>
constexpr int rows_per_thread() {
    return P == 3 ? 32 : (P == 4 ? 24 : (P == 2 ? 32 : 16));
}

template <int P, int L, int NX, int NP, int NG, int NY>
cudaError_t launch2(const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale, int accumulate,
                    int batch, cudaStream_t st) {
    using namespace f2;
    Args2 a;
    memset(&a, 0, sizeof a);
    a.src = src;
    a.dst = dst;
    a.scale = scale;
    a.accumulate = accumulate;
    a.bx = op->F[0].band;
    a.by = op->F[1].band;
    a.bz = op->F[2].band;
    a.rounds = pl.d_f2;
    a.nrounds = (int)pl.f2_nrounds;
    a.mx = op->m[0];
    a.my = op->m[1];
    a.mz = op->m[2];
    a.batch = batch;
    a.tiles_x = (a.mx + TX - 1) / TX;
    a.tiles_y = (a.my + L - 1) / L;
    a.txt = TX;
    a.tyt = L;
    a.units = (long long)a.tiles_x * a.tiles_y * batch * a.mz;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent CTAs (one per SM); keep segments >= 2P+2 planes and <= 3 mz units per CTA
    long long nct = sms;
    const long long minlen = 2 * P + 2;
    if (a.units / nct < minlen) nct = a.units / minlen;
    if (nct < 1) nct = 1;
    while ((a.units + nct - 1) / nct > 3LL * a.mz) nct += sms;
    a.nctas = (int)nct;
    const size_t sm = smem_bytes<P, L, NX, NP, NG, NY>(a.nrounds);
    auto kern = k_fused2<P, L, NX, NP, NG, NY>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
    const size_t scratch_elems = (size_t)a.nctas * NSEG * 4 * P * L * TX;
    e = pool_alloc(op->pool, (void**)&a.scratch, sizeof(double) * scratch_elems, st);
    if (e) return e;
    kern<<<a.nctas, NW * 32, sm, st>>>(a);
    e = cudaGetLastError();
    if (!e) {
        if (a.nctas > 1) k_fixup<<<(a.nctas - 1) * 2 * P, 256, 0, st>>>(a, P, L);
        e = cudaGetLastError();
    }
    cudaFreeAsync(a.scratch, st);
    return e;
}

template <int P>
cudaError_t launch_part(const iga_lr_op* op, const Plan& pl, int part, const double* src, double* dst, double scale,
                        int accumulate, int batch, cudaStream_t st) {
    constexpr int L = rows_per_thread<P>();
    if (part == 0) return launch2<P, L, kMX, kMP, kMG, kMY>(op, pl, src, dst, scale, accumulate, batch, st);
    return launch2<P, L, kSX, kSP, kSG, kSY>(op, pl, src, dst, scale, accumulate, batch, st);
}


// ---- canonical-shape host side
template <class S>
bool build_canon(const iga_lr_op* op, const Plan& pl, std::vector<f2::RoundC<S>>* out);

template <int K>
bool build_canon_mass(const Plan& pl, std::vector<f2::RoundC<f2::ShapeMassK<K>>>* out) {
    out->clear();
    std::vector<const Round*> terms;
    for (const Round& R : pl.rounds) {
        if (R.nx != 1 || R.np != 1 || R.ng != 1 || R.ne[0] != 1) return false;
        terms.push_back(&R);
    }
    if (terms.empty()) return false;
    for (size_t i = 0; i < terms.size(); i += K) {
        f2::RoundC<f2::ShapeMassK<K>> C;
        memset(&C, 0, sizeof C);
        for (int k = 0; k < K; ++k) {
            const bool real = i + k < terms.size();
            const Round& R = *terms[real ? i + k : 0];
            C.xf[k] = R.xf[0];
            C.yf[k] = R.pf[0];
            C.gf[k] = R.gf[0];
            C.gs[k] = real ? R.ec[0][0] : 0.0;  // padding term contributes exactly zero
            C.pc[k] = 1.0;
        }
        out->push_back(C);
    }
    return out->size() <= (size_t)f2::kMaxRounds2;
}

template <>
bool build_canon<f2::ShapeMassK<4>>(const iga_lr_op* op, const Plan& pl, std::vector<f2::RoundC<f2::ShapeMassK<4>>>* out) {
    (void)op;
    return build_canon_mass<4>(pl, out);
}
template <>
bool build_canon<f2::ShapeMassK<3>>(const iga_lr_op* op, const Plan& pl, std::vector<f2::RoundC<f2::ShapeMassK<3>>>* out) {
    (void)op;
    return build_canon_mass<3>(pl, out);
}

template <>
bool build_canon<f2::ShapeStiffA>(const iga_lr_op* op, const Plan& pl, std::vector<f2::RoundC<f2::ShapeStiffA>>* out) {
    using S = f2::ShapeStiffA;
    out->clear();
    // pattern (a*2+b) -> canonical slot; x: [K,E,T,M], y and z: [M,T,E,K]
    auto xslot = [](int pat) { return pat == 3 ? 0 : pat == 1 ? 1 : pat == 2 ? 2 : 3; };
    auto yslot = [](int pat) { return pat == 0 ? 0 : pat == 2 ? 1 : pat == 1 ? 2 : 3; };
    for (const Round& R : pl.rounds) {
        f2::RoundC<S> C;
        memset(&C, 0, sizeof C);
        int xs[4] = {-1, -1, -1, -1}, ys[4] = {-1, -1, -1, -1}, gsl[4] = {-1, -1, -1, -1};
        for (int e = 0; e < R.nx; ++e) {
            const int s = xslot(op->F[0].pattern[R.xf[e]]);
            if (xs[s] >= 0) return false;
            xs[s] = R.xf[e];
        }
        for (int g = 0; g < R.ng; ++g) {
            const int s = yslot(op->F[2].pattern[R.gf[g]]);
            if (gsl[s] >= 0) return false;
            gsl[s] = R.gf[g];
        }
        double cj[S::NPAIR];
        bool seen[S::NPAIR] = {};
        for (int g = 0; g < R.ng; ++g) {
            const int gs_ = yslot(op->F[2].pattern[R.gf[g]]);
            for (int e = 0; e < R.ne[g]; ++e) {
                const int j = R.ep[g][e];
                const int xsl = xslot(op->F[0].pattern[R.xf[R.px[j]]]);
                const int ysl = yslot(op->F[1].pattern[R.pf[j]]);
                if (ys[ysl] >= 0 && ys[ysl] != R.pf[j]) return false;
                ys[ysl] = R.pf[j];
                int cj_idx = -1;
                for (int k = 0; k < S::NPAIR; ++k)
                    if (S::px(k) == xsl && S::py(k) == ysl && S::pg(k) == gs_) cj_idx = k;
                if (cj_idx < 0 || seen[cj_idx]) return false;
                seen[cj_idx] = true;
                cj[cj_idx] = R.ec[g][e];
            }
        }
        for (int k = 0; k < S::NPAIR; ++k)
            if (!seen[k]) return false;
        for (int s = 0; s < 4; ++s)
            if (xs[s] < 0 || ys[s] < 0 || gsl[s] < 0) return false;
        for (int s = 0; s < 4; ++s) {
            C.xf[s] = xs[s];
            C.yf[s] = ys[s];
            C.gf[s] = gsl[s];
        }
        for (int k = 0; k < S::NPAIR; ++k)
            if (S::lead(k)) {
                if (cj[k] == 0.0) return false;
                C.gs[S::pg(k)] = cj[k];
                C.pc[k] = 1.0;
            }
        for (int k = 0; k < S::NPAIR; ++k)
            if (!S::lead(k)) C.pc[k] = cj[k] / C.gs[S::pg(k)];
        out->push_back(C);
    }
    return !out->empty() && out->size() <= (size_t)f2::kMaxRounds2;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static EncodeFn tensor_map_encode() {
    static EncodeFn fn = []() -> EncodeFn {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

template <int P>
struct CanonCfg {
    static constexpr int LW = P == 3 ? 16 : 12;  // rows per warp (TMEM: LW * ring cols <= 256)
    static constexpr int WPQ = 2;                // warps per TMEM lane quadrant
};

// Tile shape: QX quadrants across x and LW rows per warp.  Candidates: the degree's default LW
// with QX in {4, 2, 1}, plus (p = 3) LW = 12 with QX = 2 for meshes whose extent 32 LW tiles
// badly (e.g. 46 interior rows: 48-row tiles instead of 64).  Cost = padded area x the X stage's
// y-halo recompute (the X stage is ~1/5 of a point's FP64 work).  Ties -> the first candidate.
struct TileChoice {
    int qx, lw, vp;  // vp: vectors packed along x (GSYNC path; KSplit::vp)
};
// columns of a tile row holding packed vector data / columns covered, for vp vectors of width mx
static double pack_util(int mx, int tx, int vp) {
    const long long w = (long long)vp * mx;
    return (double)w / (double)((w + tx - 1) / tx * tx);
}
static TileChoice pick_tile(int mx, int my, int P, int batch = 1, int qx_override = 0, int vp_override = 0) {
    const int LW0 = P == 3 ? CanonCfg<3>::LW : CanonCfg<4>::LW;
    // p = 3 also weighs 48-row tiles (LW 12, QX 2); p = 4 weighs LW 13 (26-row tiles, 234 of a
    // warp's 256 TMEM columns with the 9-double ring): 256 rows tile as 10 x 26 instead of 11 x 24
    TileChoice cand[4] = {{4, LW0, 1}, {2, LW0, 1}, {1, LW0, 1}, {P == 3 ? 2 : 4, P == 3 ? 12 : 13, 1}};
    const int ncand = 4;
    TileChoice best = cand[0];
    double bc = 1e30;
    for (int i = 0; i < ncand; ++i) {
        const int tx = 32 * cand[i].qx, ty = cand[i].lw * 2 * (4 / cand[i].qx);
        // vectors per packed row: the smallest count with the best column utilisation (a batch of
        // narrow vectors fills the tile columns; one vector per row when the mesh is wide enough)
        int vp = 1;
        double ux = pack_util(mx, tx, 1);
        for (int v = 2; v <= std::min(batch, 32) && (long long)(v - 1) * mx < 4LL * tx; ++v)
            if (pack_util(mx, tx, v) > ux + 0.02) {
                ux = pack_util(mx, tx, v);
                vp = v;
            }
        if (vp_override > 0) {
            vp = std::min(vp_override, std::max(batch, 1));
            ux = pack_util(mx, tx, vp);
        }
        // (a packed tile row costs more staging copies and a wider fixup mapping: only worth it
        // when the columns are used clearly better)
        if (vp > 1 && vp_override <= 0) ux /= 1.03;
        const double waste = 1.0 / ux * (double)((my + ty - 1) / ty * ty) / my;
        const double halo = (double)(cand[i].lw + 2 * P) / cand[i].lw;
        const double cost = waste * (0.8 + 0.2 * halo);
        if (cost < bc - 1e-9) {
            bc = cost;
            best = cand[i];
            best.vp = vp;
        }
    }
    if (qx_override == 1 || qx_override == 2 || qx_override == 4) {  // (test knob)
        best = {qx_override, LW0, 1};
        if (vp_override > 0) best.vp = std::min(vp_override, std::max(batch, 1));
    }
    return best;
}

// minimum planes per persistent CTA range (see launch_canon_t)
static long long canon_minlen(const iga_lr_op* op, long long units, int P, int sms) {
    if (op->knobs.minlen > 0) return op->knobs.minlen;  // (test knob)
    return units >= (long long)sms * (2 * P + 2) ? 2 * P + 2 : 1;
}

// Partial output planes of a canonical launch and their contributors, in CTA order (the same
// enumeration the kernel's retire/flush code uses: CTA k, segment seg over tile t and input planes
// [za, zb) writes every zo in [za-P, zb+P) of the mesh, to scratch slot partial_slot(zo, za, zb, P)
// unless all of zo's input planes [zo-P, zo+P] lie in [za, zb)).  Built once per launch shape and
// cached in the op (device copy); deterministic.
static cudaError_t fixup_table(const iga_lr_op* op, const f2::Args2& a, int P, int vp, const f2::FixEnt** tab, int* n,
                               cudaStream_t st) {
    const long long key[10] = {P, a.tyt, a.txt, a.tiles_x, a.tiles_y, a.batch, a.mx, a.my, a.nctas, vp};
    std::lock_guard<std::mutex> lock(op->fix_mu);
    for (const auto& c : op->fix_cache)
        if (std::equal(key, key + 10, c.key)) {
            *tab = static_cast<const f2::FixEnt*>(c.d_tab);
            *n = c.n;
            // the upload may have been queued on another stream: order this launch after it
            return c.ready ? cudaStreamWaitEvent(st, c.ready, 0) : cudaSuccess;
        }
    std::map<std::pair<long long, int>, f2::FixEnt> ents;
    const long long TYX = (long long)a.tyt * a.txt;
    for (int k = 0; k < a.nctas; ++k) {
        const long long c0 = f2::unit_begin(k, a.units, a.nctas), c1 = f2::unit_begin(k + 1, a.units, a.nctas);
        int seg = 0;
        for (long long u = c0; u < c1; ++seg) {
            const long long tile = u / a.mz;
            const int za = (int)(u - tile * a.mz);
            const int zb = (int)std::min((long long)a.mz, (long long)za + (c1 - u));
            for (int zo = std::max(0, za - P); zo < std::min(a.mz, zb + P); ++zo) {
                const int lo = std::max(0, zo - P), hi = std::min(a.mz - 1, zo + P);
                if (lo >= za && hi <= zb - 1) continue;  // complete: written to the output directly
                f2::FixEnt& E = ents[{tile, zo}];
                if (E.n == 0) {
                    long long tt = tile;
                    E.txi = (int)(tt % a.tiles_x); tt /= a.tiles_x;
                    E.tyi = (int)(tt % a.tiles_y); tt /= a.tiles_y;
                    E.b = (int)tt;
                    E.zo = zo;
                }
                if (E.n >= 2 * 4 + 1) return cudaErrorInvalidConfiguration;
                E.off[E.n++] = (((long long)k * f2::NSEG + seg) * 4 * P + f2::partial_slot(zo, za, zb, P)) * TYX;
            }
            u += zb - za;
        }
    }
    std::vector<f2::FixEnt> v;
    v.reserve(ents.size());
    for (auto& kv : ents) v.push_back(kv.second);
    iga_lr_op::FixCache c;
    std::copy(key, key + 10, c.key);
    c.n = (int)v.size();
    c.d_tab = nullptr;
    c.ready = nullptr;
    if (!v.empty()) {
        cudaError_t e = cudaMalloc(&c.d_tab, v.size() * sizeof(f2::FixEnt));
        // (pageable source: the copy is staged before the call returns, then runs in stream order;
        // the event orders users on other streams after it)
        if (!e) e = cudaMemcpyAsync(c.d_tab, v.data(), v.size() * sizeof(f2::FixEnt), cudaMemcpyHostToDevice, st);
        if (!e) e = cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming);
        if (!e) e = cudaEventRecord(c.ready, st);
        if (e) {
            if (c.d_tab) cudaFree(c.d_tab);
            if (c.ready) cudaEventDestroy(c.ready);
            return e;
        }
    }
    op->fix_cache.push_back(c);
    *tab = static_cast<const f2::FixEnt*>(c.d_tab);
    *n = c.n;
    return cudaSuccess;
}

template <class S, int P, int QX, bool YRES, bool TMA, int LW = CanonCfg<P>::LW, bool SPLIT = false, bool PACK = false>
cudaError_t launch_canon_t(const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                           int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    using namespace f2;
    constexpr int WPQ = CanonCfg<P>::WPQ;
    constexpr int TXT = 32 * QX, TYT = LW * WPQ * (4 / QX);
    Args2 a;
    memset(&a, 0, sizeof a);
    a.src = src;
    a.dst = dst;
    a.scale = scale;
    a.accumulate = accumulate;
    a.bx = op->F[0].band;
    a.by = op->F[1].band;
    a.bz = op->F[2].band;
    a.rounds = pl.d_canon;
    if (gsync_path<P, TMA, YRES>()) a.bz = pl.d_ztab;  // GSYNC path: per-plane z records
    if (gsync_path<P, TMA, YRES>() && !PACK && P == 3) a.bx = pl.d_xtab;  // ... and per-round x records (XREC)
    a.nrounds = pl.canon_nrounds;
    a.mx = op->m[0];
    a.my = op->m[1];
    a.mz = op->m[2];
    a.batch = batch;
    // vector packing along x: the GSYNC path only (bulk-copied rows, one piece per vector)
    const int vp = PACK ? std::max(1, std::min(sp.vp, batch)) : 1;
    const int groups = (batch + vp - 1) / vp;
    a.tiles_x = (vp * a.mx + TXT - 1) / TXT;
    a.tiles_y = (a.my + TYT - 1) / TYT;
    a.txt = TXT;
    a.tyt = TYT;
    a.units = (long long)a.tiles_x * a.tiles_y * groups * a.mz;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long nct = sms;
    // CTA ranges of >= 2P+2 planes keep the fixup volume (2P partial planes per range boundary)
    // small; a mesh with fewer units than that takes one CTA per unit instead (every plane then has
    // up to 2P+1 contributors, which the table-driven fixup sums): parallelism wins there (c2).
    const long long minlen = canon_minlen(op, a.units, P, sms);
    if (a.units / nct < minlen) nct = a.units / minlen;
    if (nct < 1) nct = 1;
    while ((a.units + nct - 1) / nct > 3LL * a.mz) nct += sms;
    // a launch whose tiles nearly fill the GPU takes one whole tile per CTA instead: no range boundary
    // inside a tile, so no partial planes, no scratch traffic and no fixup launch (c4 mass: 144 tiles on
    // 148 SMs).  Measured on 48^3 meshes (B200): the boundaries cost a mass launch 7-8 % and a stiffness
    // launch 2-3 %, so whole tiles win from 92 % (mass) and 97 % (stiffness) SM fill.
    const long long ntiles = a.units / a.mz;
    const int fill = std::is_same<S, f2::ShapeStiffA>::value ? 97 : 92;
    if (op->knobs.minlen == 0 && ntiles <= sms && ntiles * 100 >= (long long)sms * fill) nct = ntiles;
    a.nctas = (int)nct;
    const size_t sm = smem_bytes_canon<S, P, LW, WPQ, QX, YRES>(a.nrounds);
    auto kern = k_canon<S, P, LW, WPQ, QX, YRES, TMA, SPLIT, PACK>;
    f2::KSplit ks;
    ks.bsplit = sp.bsplit;
    ks.src_jump = sp.src_jump;
    ks.dst_jump = sp.dst_jump;
    ks.vp = vp;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
    const size_t scratch_elems = (size_t)a.nctas * NSEG * 4 * P * TYT * TXT;
    e = pool_alloc(op->pool, (void**)&a.scratch, sizeof(double) * scratch_elems, st);
    if (e) return e;
    int nfix = 0;
    const f2::FixEnt* tab = nullptr;
    if (a.nctas > 1) {
        e = fixup_table(op, a, P, vp, &tab, &nfix, st);
        if (e) {
            cudaFreeAsync(a.scratch, st);
            return e;
        }
    }
    kern<<<a.nctas, NW * WPQ * 32, sm, st>>>(a, ks);
    e = cudaGetLastError();
    if (!e && nfix > 0) {
        // few entries (fewer than two per SM): the wide variant (its blocks would only add scheduling
        // overhead to a launch that already fills the GPU: c3 +15 us)
        if (nfix < 2 * sms) f2::k_fixup_tab_wide<<<nfix * f2::FIXSPLIT, 256, 0, st>>>(a, tab, ks);
        else f2::k_fixup_tab<<<nfix, 256, 0, st>>>(a, tab, ks);
        e = cudaGetLastError();
    }
    cudaFreeAsync(a.scratch, st);
    return e;
}

// GSYNC launch; vector packing (sp.vp > 1) has its own kernel variant, for p = 3 (p = 4 sits at the
// register cliff)
template <class S, int P, int QX, int LW, bool SPLIT>
cudaError_t launch_gsync(const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                         int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    if constexpr (P == 3) {
        if (sp.vp > 1 && batch > 1)
            return launch_canon_t<S, P, QX, true, true, LW, SPLIT, true>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    return launch_canon_t<S, P, QX, true, true, LW, SPLIT>(op, pl, src, dst, scale, accumulate, batch, st, sp);
}

template <class S, int P, int QX, int LW = CanonCfg<P>::LW>
bool yres_fits(int nrounds) {
    return f2::smem_bytes_canon<S, P, LW, 2, QX, true>(nrounds) <= 227 * 1024;
}

template <class S>
size_t canon_smem(int p, int nrounds) {
    // per-round y staging bounds the requirement of every tile shape
    size_t m = 0;
    if (p == 3) {
        m = std::max(m, f2::smem_bytes_canon<S, 3, CanonCfg<3>::LW, 2, 4, false>(nrounds));
        m = std::max(m, f2::smem_bytes_canon<S, 3, CanonCfg<3>::LW, 2, 2, false>(nrounds));
        m = std::max(m, f2::smem_bytes_canon<S, 3, CanonCfg<3>::LW, 2, 1, false>(nrounds));
    } else {
        m = std::max(m, f2::smem_bytes_canon<S, 4, CanonCfg<4>::LW, 2, 4, false>(nrounds));
        m = std::max(m, f2::smem_bytes_canon<S, 4, CanonCfg<4>::LW, 2, 2, false>(nrounds));
        m = std::max(m, f2::smem_bytes_canon<S, 4, CanonCfg<4>::LW, 2, 1, false>(nrounds));
    }
    return m;
}

template <class S, int P, int QX, int LW = CanonCfg<P>::LW>
cudaError_t launch_canon_q(const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                           int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    const bool force_off = op->knobs.no_yres != 0;
    // TMA needs 16-byte row strides (even nx), 16-byte aligned input and the driver entry point
    // bulk copies need 16-byte aligned coefficient rows: (factor * nx + x0) * BW even <=> nx even
    // the GSYNC path (TMA && YRES) also bulk-copies plane rows: 16-byte aligned input
    const bool tma = !op->knobs.no_tma && (op->m[0] % 2 == 0) && ((uintptr_t)src % 16 == 0) && pl.d_ztab;
    const bool yres = !force_off && yres_fits<S, P, QX, LW>(pl.canon_nrounds);
#ifdef IGALR_EXP_FAST  // (experiment builds: the GSYNC variants only, fast compiles)
    if (!(tma && yres)) return cudaErrorNotSupported;
    if (sp.bsplit) {
        if constexpr (P == 3 && std::is_same<S, f2::ShapeStiffA>::value)
            return launch_gsync<S, P, QX, LW, true>(op, pl, src, dst, scale, accumulate, batch, st, sp);
        return cudaErrorNotSupported;
    }
    return launch_gsync<S, P, QX, LW, false>(op, pl, src, dst, scale, accumulate, batch, st, sp);
#else
    if (sp.bsplit) {
        // batch split (KKT stiffness): p = 3 stiffness on the GSYNC path only; otherwise the
        // caller falls back to one launch per segment
        if constexpr (P == 3 && std::is_same<S, f2::ShapeStiffA>::value) {
            if (tma && yres) return launch_gsync<S, P, QX, LW, true>(op, pl, src, dst, scale, accumulate, batch, st, sp);
        }
        return cudaErrorNotSupported;
    }
    if constexpr (LW != CanonCfg<P>::LW) {
        // alternative row count: instantiated for the GSYNC path only
        if (tma && yres) return launch_gsync<S, P, QX, LW, false>(op, pl, src, dst, scale, accumulate, batch, st, sp);
        return launch_canon_q<S, P, QX>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    if (tma) {
        if (yres) return launch_gsync<S, P, QX, CanonCfg<P>::LW, false>(op, pl, src, dst, scale, accumulate, batch, st, sp);
        return launch_canon_t<S, P, QX, false, true>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    if (yres) return launch_canon_t<S, P, QX, true, false>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    return launch_canon_t<S, P, QX, false, false>(op, pl, src, dst, scale, accumulate, batch, st, sp);
#endif
}

}  // namespace

// Per-degree instantiations live in canon_p3.cu / canon_p4.cu (parallel compilation).
cudaError_t canon_launch_p3(int part, const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                            int accumulate, int batch, cudaStream_t st, const CanonSplit& sp);
cudaError_t canon_launch_p4(int part, const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                            int accumulate, int batch, cudaStream_t st, const CanonSplit& sp);

#if defined(IGALR_CANON_P) && IGALR_CANON_P != 99  // (99: experiment TUs instantiate kernels themselves)
template <class S, int P>
cudaError_t launch_canon_tile(const TileChoice& tc, const iga_lr_op* op, const Plan& pl, const double* src, double* dst,
                              double scale, int accumulate, int batch, cudaStream_t st, const CanonSplit& sp);
template <class S, int P>
cudaError_t launch_canon_deg(const iga_lr_op* op, const Plan& pl, const double* src, double* dst, double scale,
                             int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    const TileChoice tc = pick_tile(op->m[0], op->m[1], P, batch, op->knobs.qx, op->knobs.vpack);
    CanonSplit spv = sp;
    spv.vp = tc.vp;
    return launch_canon_tile<S, P>(tc, op, pl, src, dst, scale, accumulate, batch, st, spv);
}
template <class S, int P>
cudaError_t launch_canon_tile(const TileChoice& tc, const iga_lr_op* op, const Plan& pl, const double* src, double* dst,
                              double scale, int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    if constexpr (P == 3) {
        if (tc.lw == 12) return launch_canon_q<S, P, 2, 12>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    if constexpr (P == 4) {
        if (tc.lw == 13) return launch_canon_q<S, P, 4, 13>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    if (tc.qx == 4) return launch_canon_q<S, P, 4>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    if (tc.qx == 2) return launch_canon_q<S, P, 2>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    return launch_canon_q<S, P, 1>(op, pl, src, dst, scale, accumulate, batch, st, sp);
}
#define IGALR_CAT2(a, b) a##b
#define IGALR_CAT(a, b) IGALR_CAT2(a, b)
cudaError_t IGALR_CAT(canon_launch_p, IGALR_CANON_P)(int part, const iga_lr_op* op, const Plan& pl, const double* src,
                                                     double* dst, double scale, int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    if (part == 0) {
        if (pl.canon_mk == 3)
            return launch_canon_deg<f2::ShapeMassK<3>, IGALR_CANON_P>(op, pl, src, dst, scale, accumulate, batch, st, sp);
        return launch_canon_deg<f2::ShapeMassK<4>, IGALR_CANON_P>(op, pl, src, dst, scale, accumulate, batch, st, sp);
    }
    return launch_canon_deg<f2::ShapeStiffA, IGALR_CANON_P>(op, pl, src, dst, scale, accumulate, batch, st, sp);
}
#endif

#ifndef IGALR_CANON_P
namespace {

// Per-plane z-coefficient records of the GSYNC canonical kernel (one bulk copy per plane):
//   ztab[z'][r][g*BW + j] = gs_r[g] * Fz_{gf_r[g]}[zo][z' - zo + P],  zo = the output plane held in
// ring slot j while input plane z' is processed (zo = z' - P + ((j - (z' - P)) mod BW)), 0 if zo is
// outside the mesh; entries j >= NG*BW (record padding to 16 bytes) are 0.
__global__ void k_build_ztab(const double* __restrict__ bz, const int* __restrict__ gf, const double* __restrict__ gs,
                             int nrounds, int ng, int ngb, int mz, int P, double* __restrict__ ztab) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)mz * nrounds * ngb) return;
    const int BW = 2 * P + 1;
    const int q = (int)(i % ngb);
    const int r = (int)((i / ngb) % nrounds);
    const int zp = (int)(i / ((long long)ngb * nrounds));
    double v = 0.0;
    if (q < ng * BW) {
        const int g = q / BW, j = q % BW;
        const int zo = zp - P + ((j - (zp - P)) % BW + BW) % BW;
        if (zo >= 0 && zo < mz) v = gs[r * ng + g] * bz[((size_t)gf[r * ng + g] * mz + zo) * BW + (zp - zo + P)];
    }
    ztab[i] = v;
}

// Per-round x records of the unpacked GSYNC canonical kernel (one bulk copy per column group and
// round): xtab[r][b][e][c][k] = Fx_{xf_r[e]}[32 b + c][k] (band entry k of row 32 b + c), 0 past mx.
__global__ void k_build_xtab(const double* __restrict__ bx, const int* __restrict__ xf, int nrounds, int nx, int mx,
                             int BW, double* __restrict__ xtab) {
    const int nblk = (mx + 31) / 32;
    const long long n = (long long)nrounds * nblk * nx * 32 * BW;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k = (int)(i % BW);
    const int c = (int)((i / BW) % 32);
    const int e = (int)((i / (32LL * BW)) % nx);
    const int b = (int)((i / (32LL * BW * nx)) % nblk);
    const int r = (int)(i / (32LL * BW * nx * nblk));
    const int col = b * 32 + c;
    xtab[i] = col < mx ? bx[((size_t)xf[r * nx + e] * mx + col) * BW + k] : 0.0;
}

template <class S>
iga_status prepare_canon_t(const iga_lr_op* op, Plan* pl, cudaStream_t st) {
    std::vector<f2::RoundC<S>> v;
    if (!build_canon<S>(op, *pl, &v)) return IGA_EUNSUPPORTED;
    const int n = (int)v.size();
    if (canon_smem<S>(op->p[0], n) > 227 * 1024) return IGA_EUNSUPPORTED;
    cudaError_t e = cudaMalloc(&pl->d_canon, sizeof(v[0]) * n);
    if (e) return cuda_error(e, "cudaMalloc(canon rounds)");
    e = cudaMemcpyAsync(pl->d_canon, v.data(), sizeof(v[0]) * n, cudaMemcpyHostToDevice, st);
    if (e) return cuda_error(e, "canon rounds H2D");
    // per-plane z records (GSYNC path)
    const int P = op->p[2], BW = 2 * P + 1, mz = op->m[2];
    const int ngb = (S::NG * BW + 1) & ~1;
    std::vector<int> gf(n * S::NG);
    std::vector<double> gs(n * S::NG);
    for (int r = 0; r < n; ++r)
        for (int g = 0; g < S::NG; ++g) {
            gf[r * S::NG + g] = v[r].gf[g];
            gs[r * S::NG + g] = v[r].gs[g];
        }
    int* d_gf = nullptr;
    double* d_gs = nullptr;
    int* d_xf = nullptr;
    std::vector<int> xf(n * S::NX);
    for (int r = 0; r < n; ++r)
        for (int x = 0; x < S::NX; ++x) xf[r * S::NX + x] = v[r].xf[x];
    const int BWx = 2 * op->p[0] + 1, mx = op->m[0];
    const size_t nxt = (size_t)n * ((mx + 31) / 32) * S::NX * 32 * BWx;
    const size_t nz = (size_t)mz * n * ngb;
    e = cudaMalloc(&pl->d_ztab, sizeof(double) * nz);
    if (!e) e = cudaMalloc(&pl->d_xtab, sizeof(double) * nxt);
    if (!e) e = pool_alloc(op->pool, (void**)&d_xf, sizeof(int) * xf.size(), st);
    if (!e) e = cudaMemcpyAsync(d_xf, xf.data(), sizeof(int) * xf.size(), cudaMemcpyHostToDevice, st);
    if (!e) {
        k_build_xtab<<<(unsigned)((nxt + 255) / 256), 256, 0, st>>>(op->F[0].band, d_xf, n, S::NX, mx, BWx, pl->d_xtab);
        e = cudaGetLastError();
    }
    if (!e) e = pool_alloc(op->pool, (void**)&d_gf, sizeof(int) * gf.size(), st);
    if (!e) e = pool_alloc(op->pool, (void**)&d_gs, sizeof(double) * gs.size(), st);
    if (!e) e = cudaMemcpyAsync(d_gf, gf.data(), sizeof(int) * gf.size(), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemcpyAsync(d_gs, gs.data(), sizeof(double) * gs.size(), cudaMemcpyHostToDevice, st);
    if (!e) {
        k_build_ztab<<<(unsigned)((nz + 255) / 256), 256, 0, st>>>(op->F[2].band, d_gf, d_gs, n, S::NG, ngb, mz, P,
                                                                  pl->d_ztab);
        e = cudaGetLastError();
    }
    // stream-ordered temporaries (cudaFree would synchronise the device); the host tables die
    // here, so wait for this stream
    if (d_gf) cudaFreeAsync(d_gf, st);
    if (d_gs) cudaFreeAsync(d_gs, st);
    if (d_xf) cudaFreeAsync(d_xf, st);
    if (!e) e = cudaStreamSynchronize(st);
    if (e) return cuda_error(e, "canon z records");
    pl->canon_nrounds = n;
    pl->canon_ok = true;
    return IGA_OK;
}

}  // namespace

iga_status prepare_canon(const iga_lr_op* op, Plan* pl, int part, cudaStream_t st) {
    if (!fused2_supported(op)) return IGA_EUNSUPPORTED;
    if (part == 0) {
        // mass terms per sweep: 4, or 3 when that avoids zero-padding terms (e.g. R = 6)
        const int R = (int)pl->rounds.size();
        pl->canon_mk = (R % 4 != 0 && R % 3 == 0) ? 3 : 4;
        return pl->canon_mk == 3 ? prepare_canon_t<f2::ShapeMassK<3>>(op, pl, st)
                                 : prepare_canon_t<f2::ShapeMassK<4>>(op, pl, st);
    }
    return prepare_canon_t<f2::ShapeStiffA>(op, pl, st);
}

iga_status apply_canon_part(const iga_lr_op* op, const Plan& pl, int part, const double* src, double* dst, double scale,
                            int accumulate, int batch, cudaStream_t st, const CanonSplit& sp) {
    cudaError_t e = op->p[0] == 3 ? canon_launch_p3(part, op, pl, src, dst, scale, accumulate, batch, st, sp)
                                  : canon_launch_p4(part, op, pl, src, dst, scale, accumulate, batch, st, sp);
    if (e == cudaErrorNotSupported && sp.bsplit) return IGA_EUNSUPPORTED;  // (no error state)
    if (e) return cuda_error(e, "k_canon");
    return IGA_OK;
}

namespace {
}  // namespace

bool fused2_supported(const iga_lr_op* op) {
    if (op->p[0] != op->p[1] || op->p[0] != op->p[2]) return false;
    return op->p[0] == 3 || op->p[0] == 4;
}

bool canon_small_grid(const iga_lr_op* op, int batch) {
    // both parts' persistent grids fit the GPU side by side: launch them concurrently
    if (!fused2_supported(op)) return false;
    const int P = op->p[0];
    const TileChoice tc = pick_tile(op->m[0], op->m[1], P, batch, op->knobs.qx, op->knobs.vpack);
    const long long tx = 32 * tc.qx, ty = (long long)tc.lw * 2 * (4 / tc.qx);
    const long long vp = op->m[0] % 2 == 0 ? tc.vp : 1;  // (packing needs the bulk-copy path: even nx)
    const long long units =
        (vp * op->m[0] + tx - 1) / tx * ((op->m[1] + ty - 1) / ty) * ((batch + vp - 1) / vp) * op->m[2];
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 2 * units <= sms;
}

void canon_tile_choice(const iga_lr_op* op, int batch, int* qx, int* lw, int* vp) {
    const TileChoice tc = pick_tile(op->m[0], op->m[1], op->p[0], batch, op->knobs.qx, op->knobs.vpack);
    *qx = tc.qx;
    *lw = tc.lw;
    *vp = op->p[0] == 3 && op->m[0] % 2 == 0 ? std::min(tc.vp, std::max(batch, 1)) : 1;  // (launch_gsync)
}

bool fused2_preferred(const iga_lr_op* op, int batch) {
    // every mesh size: small meshes take one CTA per (tile, plane) unit (canon_small_grid)
    (void)op;
    (void)batch;
    return true;
}

iga_status prepare_fused2(const iga_lr_op* op, Plan* pl, int part, cudaStream_t st) {
    if (!fused2_supported(op)) return IGA_EUNSUPPORTED;
    size_t bytes = 0;
    std::vector<char> blob;
    if (part == 0) {
        std::vector<f2::Round2<kMX, kMP, kMG>> v;
        if (!build_rounds2<kMX, kMP, kMG, kMY>(*pl, &v)) return IGA_EUNSUPPORTED;
        bytes = sizeof(v[0]) * v.size();
        blob.assign((const char*)v.data(), (const char*)v.data() + bytes);
        pl->f2_nrounds = (int)v.size();
    } else {
        std::vector<f2::Round2<kSX, kSP, kSG>> v;
        if (!build_rounds2<kSX, kSP, kSG, kSY>(*pl, &v)) return IGA_EUNSUPPORTED;
        bytes = sizeof(v[0]) * v.size();
        blob.assign((const char*)v.data(), (const char*)v.data() + bytes);
        pl->f2_nrounds = (int)v.size();
    }
    // shared memory budget
    size_t sm = 0;
    if (op->p[0] == 3)
        sm = part ? f2::smem_bytes<3, rows_per_thread<3>(), kSX, kSP, kSG, kSY>(pl->f2_nrounds)
                  : f2::smem_bytes<3, rows_per_thread<3>(), kMX, kMP, kMG, kMY>(pl->f2_nrounds);
    else
        sm = part ? f2::smem_bytes<4, rows_per_thread<4>(), kSX, kSP, kSG, kSY>(pl->f2_nrounds)
                  : f2::smem_bytes<4, rows_per_thread<4>(), kMX, kMP, kMG, kMY>(pl->f2_nrounds);
    if (sm > 227 * 1024) return IGA_EUNSUPPORTED;
    cudaError_t e = cudaMalloc(&pl->d_f2, bytes);
    if (e) return cuda_error(e, "cudaMalloc(f2 rounds)");
    e = cudaMemcpyAsync(pl->d_f2, blob.data(), bytes, cudaMemcpyHostToDevice, st);
    if (!e) e = cudaStreamSynchronize(st);  // (blob is a local)
    if (e) return cuda_error(e, "f2 rounds H2D");
    pl->f2_ok = true;
    return IGA_OK;
}

iga_status apply_fused2_part(const iga_lr_op* op, const Plan& pl, int part, const double* src, double* dst, double scale,
                             int accumulate, int batch, cudaStream_t st) {
    cudaError_t e = cudaErrorInvalidValue;
    if (op->p[0] == 3) e = launch_part<3>(op, pl, part, src, dst, scale, accumulate, batch, st);
    else if (op->p[0] == 4) e = launch_part<4>(op, pl, part, src, dst, scale, accumulate, batch, st);
    if (e) return cuda_error(e, "k_fused2");
    return IGA_OK;
}

#endif  // !IGALR_CANON_P

}  // namespace igalr
