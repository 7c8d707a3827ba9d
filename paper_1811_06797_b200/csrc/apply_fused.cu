// apply_fused.cu — fused sm_100a apply: all three banded mode products, the pair/group sums
// and the sum over plan rounds (r) in ONE pass over HBM (x read once, outputs written once).
//
//   y_part(z,y,x) = sum_rounds sum_g F^z_g[z][.] *_z  sum_{(j,c) in g} c  F^y_j[y][.] *_y  F^x_{e(j)}[x][.] *_x  v
//   (Eqs. (massFinal)/(stiffnessFinal); plan of DESIGN.md §5.2)
//
// CTA = 32 x-columns x TY rows of one batch vector and one z-chunk; it streams the input planes
// z' of the chunk (+-p halo) through shared memory (cp.async double buffer) and keeps, per
// thread, a register ring of 2 parts x (2p+1) output planes x PR rows.  Per plane and round:
//   stage X  (all warps): t_e(y', x) = sum_k Fx_e[x][k] v(y', x-p+k) for the TY+2p rows -> smem T
//   stage YZ (all threads; thread = column x, PR consecutive rows): u_j = Fy_j *_y t_{e(j)} from a
//            register window over T, G_g += c u_j, then ring[part][s] += Fz_g[z'-p+s][2p-s] G_g.
// A plane z'-p is complete after input plane z' and is written out (coalesced along x).
// Deterministic: every output is summed in a fixed order; no atomics.
#include <cstdint>
#include <cstring>
#include <vector>

#include "internal.h"

namespace igalr {

namespace {

constexpr int TX = 32;       // tile width (one warp of columns)
constexpr int NWARPS = 8;    // threads = 256
constexpr int PR = 2;        // rows per thread in stage YZ
constexpr int TY = NWARPS * PR;  // tile height = 16
constexpr int kMaxRoundsFused = 48;

// Pair-centric view of a round (built on the host from Round).
struct FRound {
    int nx, np, ng;
    int xf[kMaxX], xslot[kMaxX];
    int pf[kMaxPair], px[kMaxPair];
    int npg[kMaxPair];                 // groups fed by pair j
    int pgg[kMaxPair][kMaxG];
    double pgc[kMaxPair][kMaxG];
    int gf[kMaxG], gpart[kMaxG];
};

struct FusedArgs {
    const double* src[2];
    double* dst[2];
    double scale[2];
    const double* bx;
    const double* by;
    const double* bz;
    const FRound* rounds;
    int nrounds;
    int mx, my, mz;
    int tiles_x, tiles_y, batch, zchunks, zlen;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int P, int NSLOT, bool TWOPART>
__global__ void __launch_bounds__(NWARPS * 32, 1) k_fused(const FusedArgs a) {
    constexpr int BW = 2 * P + 1;
    constexpr int HY = TY + 2 * P;   // rows incl. halo
    constexpr int HX = TX + 2 * P;   // cols incl. halo
    constexpr int NPART = TWOPART ? 2 : 1;

    extern __shared__ double smem[];
    double* vin = smem;                               // [2 buf][NSLOT][HY][HX]
    double* T = vin + 2 * NSLOT * HY * HX;            // [kMaxX][HY][TX]
    FRound* rs = reinterpret_cast<FRound*>(T + kMaxX * HY * TX);

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

    int bid = blockIdx.x;
    const int tx = bid % a.tiles_x; bid /= a.tiles_x;
    const int ty = bid % a.tiles_y; bid /= a.tiles_y;
    const int zc = bid % a.zchunks; bid /= a.zchunks;
    const int b = bid;
    const int x0 = tx * TX, y0 = ty * TY;
    const int zc0 = zc * a.zlen;
    const int zc1 = min(a.mz, zc0 + a.zlen);
    const int zlo = max(0, zc0 - P), zhi = min(a.mz, zc1 + P);
    const long long plane = (long long)a.mx * a.my;
    const long long vbase = (long long)b * a.mz * plane;

    for (int i = threadIdx.x; i < a.nrounds * (int)(sizeof(FRound) / 4); i += blockDim.x)
        reinterpret_cast<int*>(rs)[i] = reinterpret_cast<const int*>(a.rounds)[i];

    auto load_plane = [&](int zp, int buf) {
        for (int s = 0; s < NSLOT; ++s) {
            double* dstp = vin + (buf * NSLOT + s) * HY * HX;
            const double* srcp = a.src[s] + vbase + (long long)zp * plane;
            for (int i = threadIdx.x; i < HY * HX; i += blockDim.x) {
                const int r = i / HX, c = i - r * HX;
                const int gy = y0 - P + r, gx = x0 - P + c;
                const bool ok = gy >= 0 && gy < a.my && gx >= 0 && gx < a.mx;
                cp_async8(dstp + i, ok ? srcp + (long long)gy * a.mx + gx : a.src[s], ok);
            }
        }
        cp_async_commit();
    };

    // ring[part][slot][row]: slot s <-> output plane z' - P + s
    double ring[NPART][BW][PR];
#pragma unroll
    for (int q = 0; q < NPART; ++q)
#pragma unroll
        for (int s = 0; s < BW; ++s)
#pragma unroll
            for (int i = 0; i < PR; ++i) ring[q][s][i] = 0.0;

    const int col = lane;              // stage YZ column
    const int gx = x0 + col;
    const int ry0 = warp * PR;         // first tile row of this thread in stage YZ

    auto retire = [&](int zo) {
        if (zo >= zc0 && zo < zc1 && gx < a.mx) {
#pragma unroll
            for (int i = 0; i < PR; ++i) {
                const int gy = y0 + ry0 + i;
                if (gy < a.my) {
                    const long long o = vbase + (long long)zo * plane + (long long)gy * a.mx + gx;
                    if (TWOPART) {
                        if (a.dst[0] == a.dst[1]) {
                            a.dst[0][o] = a.scale[0] * ring[0][0][i] + a.scale[1] * ring[NPART - 1][0][i];
                        } else {
                            if (a.dst[0]) a.dst[0][o] = a.scale[0] * ring[0][0][i];
                            if (a.dst[1]) a.dst[1][o] = a.scale[1] * ring[NPART - 1][0][i];
                        }
                    } else {
                        a.dst[0][o] = a.scale[0] * ring[0][0][i];
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NPART; ++q) {
#pragma unroll
            for (int s = 0; s < BW - 1; ++s)
#pragma unroll
                for (int i = 0; i < PR; ++i) ring[q][s][i] = ring[q][s + 1][i];
#pragma unroll
            for (int i = 0; i < PR; ++i) ring[q][BW - 1][i] = 0.0;
        }
    };

    if (zlo < zhi) load_plane(zlo, 0);
    int buf = 0;
    for (int zp = zlo; zp < zhi; ++zp) {
        cp_async_wait_all();
        __syncthreads();  // plane zp resident in vin[buf]; previous T readers done
        if (zp + 1 < zhi) load_plane(zp + 1, buf ^ 1);

        for (int r = 0; r < a.nrounds; ++r) {
            const FRound& R = rs[r];
            // ---------------- stage X: rows warp, warp+8, ... of the HY halo rows, lane = column
            {
                const int c = lane;
                const int gxc = x0 + c;
                for (int e = 0; e < R.nx; ++e) {
                    double f[BW];
                    const double* Fx = a.bx + ((size_t)R.xf[e] * a.mx + min(gxc, a.mx - 1)) * BW;
#pragma unroll
                    for (int k = 0; k < BW; ++k) f[k] = __ldg(Fx + k);
                    const double* vb = vin + (buf * NSLOT + (NSLOT > 1 ? R.xslot[e] : 0)) * HY * HX;
                    for (int row = warp; row < HY; row += NWARPS) {
                        double acc = 0.0;
#pragma unroll
                        for (int k = 0; k < BW; ++k) acc = fma(f[k], vb[row * HX + c + k], acc);
                        T[(e * HY + row) * TX + c] = acc;
                    }
                }
            }
            __syncthreads();
            // ---------------- stage Y + Z
            double G[kMaxG][PR];
#pragma unroll
            for (int g = 0; g < kMaxG; ++g)
#pragma unroll
                for (int i = 0; i < PR; ++i) G[g][i] = 0.0;
            for (int e = 0; e < R.nx; ++e) {
                double w[PR + 2 * P];
#pragma unroll
                for (int k = 0; k < PR + 2 * P; ++k) w[k] = T[(e * HY + ry0 + k) * TX + col];
                for (int j = 0; j < R.np; ++j) {
                    if (R.px[j] != e) continue;
                    double u[PR];
#pragma unroll
                    for (int i = 0; i < PR; ++i) {
                        const int gy = min(y0 + ry0 + i, a.my - 1);
                        const double* Fy = a.by + ((size_t)R.pf[j] * a.my + gy) * BW;
                        double acc = 0.0;
#pragma unroll
                        for (int k = 0; k < BW; ++k) acc = fma(__ldg(Fy + k), w[i + k], acc);
                        u[i] = acc;
                    }
                    for (int q = 0; q < R.npg[j]; ++q) {
                        const int g = R.pgg[j][q];
                        const double c = R.pgc[j][q];
#pragma unroll
                        for (int gg = 0; gg < kMaxG; ++gg)
                            if (gg == g)
#pragma unroll
                                for (int i = 0; i < PR; ++i) G[gg][i] = fma(c, u[i], G[gg][i]);
                    }
                }
            }
            // z-scatter into the ring
#pragma unroll
            for (int g = 0; g < kMaxG; ++g) {
                if (g >= R.ng) break;
                const int part = TWOPART ? R.gpart[g] : 0;
                const double* Fz = a.bz + (size_t)R.gf[g] * a.mz * BW;
#pragma unroll
                for (int s = 0; s < BW; ++s) {
                    const int zo = zp - P + s;
                    const double cz = (zo >= 0 && zo < a.mz) ? __ldg(Fz + (size_t)zo * BW + (2 * P - s)) : 0.0;
#pragma unroll
                    for (int i = 0; i < PR; ++i) {
                        if (TWOPART && part) ring[NPART - 1][s][i] = fma(cz, G[g][i], ring[NPART - 1][s][i]);
                        else ring[0][s][i] = fma(cz, G[g][i], ring[0][s][i]);
                    }
                }
            }
            __syncthreads();  // T is rewritten by the next round
        }
        retire(zp - P);
        buf ^= 1;
    }
    // flush the planes still in the ring (last chunk of the z range)
    for (int zo = zhi - P; zo < zhi; ++zo) retire(zo);
}

template <int P, int NSLOT, bool TWOPART>
size_t smem_bytes() {
    constexpr int HY = TY + 2 * P, HX = TX + 2 * P;
    return sizeof(double) * (2 * NSLOT * HY * HX + kMaxX * HY * TX);
}

template <int P, int NSLOT, bool TWOPART>
cudaError_t launch(const FusedArgs& a0, int nrounds, cudaStream_t st) {
    FusedArgs a = a0;
    const size_t sm = smem_bytes<P, NSLOT, TWOPART>() + sizeof(FRound) * nrounds;
    auto kern = k_fused<P, NSLOT, TWOPART>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NWARPS * 32, sm);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long base = (long long)a.tiles_x * a.tiles_y * a.batch;
    const long long slots = (long long)sms * (occ > 0 ? occ : 1);
    int zch = 1;
    while (base * zch < slots && a.mz / (zch + 1) >= 4 * P + 8) ++zch;
    a.zchunks = zch;
    a.zlen = (a.mz + zch - 1) / zch;
    a.zchunks = (a.mz + a.zlen - 1) / a.zlen;
    const long long blocks = base * a.zchunks;
    k_fused<P, NSLOT, TWOPART><<<(unsigned)blocks, NWARPS * 32, sm, st>>>(a);
    return cudaGetLastError();
}

template <int P>
cudaError_t dispatch(const FusedArgs& a, int nrounds, int nslot, bool twopart, cudaStream_t st) {
    if (nslot == 2) return twopart ? launch<P, 2, true>(a, nrounds, st) : launch<P, 2, false>(a, nrounds, st);
    return twopart ? launch<P, 1, true>(a, nrounds, st) : launch<P, 1, false>(a, nrounds, st);
}

}  // namespace

bool fused_supported(const iga_lr_op* op, const Plan& pl) {
    if (op->p[0] != op->p[1] || op->p[0] != op->p[2]) return false;
    if (op->p[0] < 1 || op->p[0] > 5) return false;
    if (pl.rounds.empty() || (int)pl.rounds.size() > kMaxRoundsFused) return false;
    return true;
}

iga_status prepare_fused(const iga_lr_op* op, Plan* pl, cudaStream_t st) {
    (void)op;
    std::vector<FRound> fr(pl->rounds.size());
    int nslot = 1;
    int parts_seen[2] = {0, 0};
    for (size_t r = 0; r < pl->rounds.size(); ++r) {
        const Round& R = pl->rounds[r];
        FRound& F = fr[r];
        memset(&F, 0, sizeof F);
        F.nx = R.nx;
        F.np = R.np;
        F.ng = R.ng;
        for (int e = 0; e < R.nx; ++e) {
            F.xf[e] = R.xf[e];
            F.xslot[e] = R.xslot[e];
            if (R.xslot[e]) nslot = 2;
        }
        for (int j = 0; j < R.np; ++j) {
            F.pf[j] = R.pf[j];
            F.px[j] = R.px[j];
        }
        for (int g = 0; g < R.ng; ++g) {
            F.gf[g] = R.gf[g];
            F.gpart[g] = R.gpart[g];
            parts_seen[R.gpart[g]] = 1;
            for (int e = 0; e < R.ne[g]; ++e) {
                const int j = R.ep[g][e];
                F.pgg[j][F.npg[j]] = g;
                F.pgc[j][F.npg[j]] = R.ec[g][e];
                F.npg[j]++;
            }
        }
    }
    pl->fused_nslot = nslot;
    pl->fused_parts = parts_seen[0] + parts_seen[1];
    pl->fused_part = parts_seen[1] && !parts_seen[0] ? 1 : 0;
    cudaError_t e = cudaMalloc(&pl->d_fused, sizeof(FRound) * fr.size());
    if (e) return cuda_error(e, "cudaMalloc(fused rounds)");
    // (pageable source: staged before the call returns; assembly synchronises `st` at its end)
    e = cudaMemcpyAsync(pl->d_fused, fr.data(), sizeof(FRound) * fr.size(), cudaMemcpyHostToDevice, st);
    if (e) return cuda_error(e, "fused rounds H2D");
    return IGA_OK;
}

void release_fused(Plan* pl) {
    if (pl->d_fused) cudaFree(pl->d_fused);
    pl->d_fused = nullptr;
}

iga_status apply_fused(const iga_lr_op* op, const Plan& pl, const OutMap& om, int batch, cudaStream_t st) {
    const bool twopart = pl.fused_parts == 2;
    const int nslot = pl.fused_nslot;
    FusedArgs a;
    memset(&a, 0, sizeof a);
    a.src[0] = om.src[0];
    a.src[1] = om.src[1] ? om.src[1] : om.src[0];
    if (twopart) {
        a.dst[0] = om.dst[0];
        a.dst[1] = om.dst[1];
        a.scale[0] = om.scale[0];
        a.scale[1] = om.scale[1];
    } else {
        const int part = pl.fused_part;
        a.dst[0] = om.dst[part] ? om.dst[part] : om.dst[1 - part];
        a.dst[1] = a.dst[0];
        a.scale[0] = a.scale[1] = om.scale[part];
    }
    a.bx = op->F[0].band;
    a.by = op->F[1].band;
    a.bz = op->F[2].band;
    a.rounds = reinterpret_cast<const FRound*>(pl.d_fused);
    a.nrounds = (int)pl.rounds.size();
    a.mx = op->m[0];
    a.my = op->m[1];
    a.mz = op->m[2];
    a.tiles_x = (a.mx + TX - 1) / TX;
    a.tiles_y = (a.my + TY - 1) / TY;
    a.batch = batch;
    cudaError_t e;
    switch (op->p[0]) {
        case 1: e = dispatch<1>(a, a.nrounds, nslot, twopart, st); break;
        case 2: e = dispatch<2>(a, a.nrounds, nslot, twopart, st); break;
        case 3: e = dispatch<3>(a, a.nrounds, nslot, twopart, st); break;
        case 4: e = dispatch<4>(a, a.nrounds, nslot, twopart, st); break;
        case 5: e = dispatch<5>(a, a.nrounds, nslot, twopart, st); break;
        default: e = cudaErrorInvalidValue;
    }
    if (e) return cuda_error(e, "k_fused launch");
    return IGA_OK;
}

}  // namespace igalr
