// internal.h — shared declarations of libigalr (host planning + CUDA kernels).
// Not part of the ABI (see include/iga_lr.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <nvtx3/nvToolsExt.h>  // header-only; a no-op stub unless a profiler injects itself

#include <mutex>
#include <string>
#include <vector>

#include "iga_lr.h"

namespace igalr {

// NVTX range over one C-ABI call (timeline annotation for nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


constexpr int kMaxP = 6;        // compiled degree range 1..kMaxP
constexpr int kMaxNq = 16;      // Gauss points per span
constexpr int kMaxBW = 2 * kMaxP + 1;

// Plan round limits (shared-prefix evaluation).
constexpr int kMaxX = 5;   // x-entries (factor, input slot) per round
constexpr int kMaxPair = 10;  // (y factor, x-entry) pairs per round
constexpr int kMaxG = 5;   // z groups (z factor, output part) per round
constexpr int kMaxE = 4;   // (pair, coef) entries per group

// One round of the evaluation plan.  Everything a kernel needs is POD, passed by value.
struct Round {
    int nx;
    int xf[kMaxX];      // factor id in direction x
    int xslot[kMaxX];   // input slot: 0 = mass input, 1 = stiffness input
    int np;
    int pf[kMaxPair];   // factor id in direction y
    int px[kMaxPair];   // x-entry index
    int ng;
    int gf[kMaxG];      // factor id in direction z
    int gpart[kMaxG];   // 0 = mass part, 1 = stiffness part
    int ne[kMaxG];
    int ep[kMaxG][kMaxE];     // pair index
    double ec[kMaxG][kMaxE];  // coefficient
};

struct DirFactors {
    int m = 0;        // kept extent (n or n-2)
    int p = 0;
    int bw = 0;       // 2p+1
    int nf = 0;       // number of distinct factors
    double* band = nullptr;  // device [nf][m][bw], band[f][i][k] = F[i][i-p+k]
    std::vector<int> pattern;  // a*2+b per factor
    std::vector<int> table;    // dedup weight-table id per factor
};

// Univariate quadrature of one direction (A1): spans, Gauss nodes and weights.
struct DirQuad {
    int n, p, nq, ne;
    std::vector<double> knots;
    std::vector<int> span;       // [ne] knot-span index s of each nonempty span (first fn = s-p)
    std::vector<double> node;    // [ne*nq]
    std::vector<double> wgt;     // [ne*nq] Gauss weight * span length / 2
};

// Per-call output routing for kernels: groups of part g go to dst[g] with scale[g].
struct OutMap {
    double* dst[2];   // output pointers for part 0 (mass) and 1 (stiffness); may alias
    double scale[2];
    const double* src[2];  // input pointer for slot 0 (mass) and slot 1 (stiffness)
};

}  // namespace igalr

namespace igalr {
// An evaluation plan: rounds + its algorithmic cost.  The op keeps one per request kind.
struct Plan {
    std::vector<Round> rounds;
    int n_x = 0, n_y = 0, n_z = 0;  // mode products per vector
    double flops = 0;               // algorithmic flops per vector (2 * nnz per mode product)
    bool fused_ok = false;
    void* d_fused = nullptr;        // device copy of the fused kernel's round tables
    int fused_nslot = 1;            // input slots used by the plan
    int fused_parts = 1;            // 1 or 2 output parts
    int fused_part = 0;             // the part when fused_parts == 1
    void* d_f2 = nullptr;           // fused-v2 round tables (single-part plans only)
    int f2_nrounds = 0;
    bool f2_ok = false;
    void* d_canon = nullptr;        // canonical-shape round tables (apply_fused2.cu)
    double* d_ztab = nullptr;       // per-plane z records of the canonical kernel (GSYNC path)
    double* d_xtab = nullptr;       // per-round x records [round][32-column block][NX][32][BW] (GSYNC)
    int canon_nrounds = 0;
    bool canon_ok = false;
    int canon_mk = 4;               // mass terms per sweep of the canonical mass shape
};
// (the *T plans apply K^T = the stiffness with q_kl -> q_lk; built only when Q is not symmetric)
enum PlanKind {
    kPlanBoth = 0,
    kPlanBothSplit = 1,
    kPlanMass = 2,
    kPlanStiff = 3,
    kPlanF2Mass = 4,
    kPlanF2Stiff = 5,
    kPlanStiffT = 6,
    kPlanBothSplitT = 7,
    kPlanF2StiffT = 8,
    kNumPlans = 9
};
}  // namespace igalr

namespace igalr {
// One Kronecker term c * F^z (x) F^y (x) F^x of a part (factor ids per direction x, y, z).
struct KTerm {
    int part;
    int f[3];
    double c;
};
}  // namespace igalr

struct iga_lr_op {
    int n[3], p[3], m[3], nq;
    bool dirichlet;
    bool has_mass, has_stiff;
    // q_kl and q_lk carry identical weights for every k != l, so K = K^T (the KKT's calK^T block
    // reuses the K plans); otherwise the *T plans hold K^T (Eq. (KKTSystem))
    bool stiff_sym = true;
    // kernel-selection overrides for tests and experiments (iga_lr_test_knobs, include/
    // iga_lr_testing.h); all zero => the product's own choices
    struct Knobs {
        int force_generic = 0;  // 1: fused-v2 parts run k_fused2 even when a canonical plan exists
        int qx = 0;             // 1/2/4: canonical tile width in 32-column quadrants
        int minlen = 0;         // > 0: persistent-CTA range length in planes
        int no_yres = 0;        // 1: per-round y-coefficient staging
        int no_tma = 0;         // 1: no bulk-copy staging
        int vpack = 0;          // > 0: vectors packed along x per canonical tile row (1: no packing)
    } knobs;
    igalr::DirFactors F[3];
    igalr::DirQuad quad[3];   // (kept for derived operators: the KKT preconditioner)
    igalr::Plan plan[igalr::kNumPlans];
    double min_bytes = 0;
    int device = 0;
    std::vector<igalr::KTerm> kterms;  // merged term list, r-major (NEXT-3 TT functions)
    // fixup tables of the canonical kernels, per launch shape (built on first use; fused2_impl.cuh)
    struct FixCache {
        long long key[10];  // launch shape (fixup_table)
        void* d_tab;
        int n;
        cudaEvent_t ready;  // recorded after the table's upload; every user waits on it
    };
    mutable std::mutex fix_mu;
    mutable std::vector<FixCache> fix_cache;
    // side stream for running the mass part beside the stiffness part on small grids (lazily
    // created under fix_mu; abi.cu run_f2)
    mutable cudaStream_t side = nullptr;
    // host-buffer pipeline (iga_lr_apply_host): copy streams and events, created on first use
    mutable std::mutex host_mu;
    mutable cudaStream_t host_sh = nullptr, host_sd = nullptr;
    mutable std::vector<cudaEvent_t> host_ev;
    // op-owned stream-ordered memory pool for all scratch (release threshold: never), so that
    // scratch stays mapped between applies without touching the device's default pool
    cudaMemPool_t pool = nullptr;
};

namespace igalr {

// ---- stream-ordered scratch from an owned pool (abi.cu make_pool)
cudaError_t make_pool(int device, cudaMemPool_t* pool);
inline cudaError_t pool_alloc(cudaMemPool_t pool, void** p, size_t bytes, cudaStream_t st) {
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}

// ---- error plumbing (abi.cu)
iga_status set_error(iga_status s, const std::string& msg);
iga_status cuda_error(cudaError_t e, const char* where);
void clear_error();

// ---- factor assembly (factors.cu)
struct FactorSpec {
    int table;    // weight table id (rows of `tables`)
    int a, b;     // derivative order on row / column function
};
iga_status assemble_dir(const DirQuad& q, const std::vector<std::vector<double>>& tables,
                        const std::vector<FactorSpec>& specs, bool dirichlet, cudaStream_t st,
                        DirFactors* out);

// ---- apply kernels
iga_status apply_unfused(const iga_lr_op* op, const Plan& pl, const OutMap& om, int batch, cudaStream_t st);
iga_status apply_fused(const iga_lr_op* op, const Plan& pl, const OutMap& om, int batch, cudaStream_t st);
bool fused_supported(const iga_lr_op* op, const Plan& pl);
iga_status prepare_fused(const iga_lr_op* op, Plan* pl, cudaStream_t st);
void release_fused(Plan* pl);
bool fused2_supported(const iga_lr_op* op);
bool fused2_preferred(const iga_lr_op* op, int batch);
bool canon_small_grid(const iga_lr_op* op, int batch);
// canonical tile of a launch over `batch` vectors: 32*qx columns, 2*lw*(4/qx) rows, vp vectors
// packed along x (the packed variant exists for p = 3 on the bulk-copy path)
void canon_tile_choice(const iga_lr_op* op, int batch, int* qx, int* lw, int* vp);
iga_status prepare_fused2(const iga_lr_op* op, Plan* pl, int part, cudaStream_t st);
iga_status prepare_canon(const iga_lr_op* op, Plan* pl, int part, cudaStream_t st);
// Batch split of a canonical launch (KKT): vectors b >= bsplit are read at src + b*vol + src_jump
// and written at dst + b*vol + dst_jump (element offsets).  The default is the plain batch.
struct CanonSplit {
    long long bsplit = 0, src_jump = 0, dst_jump = 0;
    int vp = 1;  // vectors packed along x (set by the tile choice; the GSYNC path only)
};
iga_status apply_canon_part(const iga_lr_op* op, const Plan& pl, int part, const double* src, double* dst, double scale,
                            int accumulate, int batch, cudaStream_t st, const CanonSplit& sp = CanonSplit());
iga_status apply_fused2_part(const iga_lr_op* op, const Plan& pl, int part, const double* src, double* dst, double scale,
                             int accumulate, int batch, cudaStream_t st);
iga_status kkt_prec_apply(const iga_kkt_prec* P, const double* in, double* out, double* tmp, cudaStream_t st);
bool kkt_prec_matches(const iga_kkt_prec* P, const iga_lr_op* op, int n_t, double tau, double beta);
iga_status kkt_combos(const double* in, double* abc, int n_t, int64_t N, double tau, double beta,
                      cudaStream_t st);
iga_status kkt_combine(const double* T, double* out, int n_t, int64_t N, double tau, double beta, cudaStream_t st);

}  // namespace igalr
