// factors.cu — setup kernels: univariate Gauss-quadrature assembly of the banded factors.
//
//   F[i][j] = sum_{spans s containing i,j} sum_q  W_q  f(x_q)  beta_i^(a)(x_q)  beta_j^(b)(x_q)
//
// Eq. (massMatrix1D) PAPER.md:192-196 (a=b=0) and K^{(d)}_{k,l} PAPER.md:217-220 with
// delta(l,d) on the row and delta(k,d) on the column function (a = [l==d], b = [k==d]).
// Two kernels: basis values/derivatives at every node (local Cox-de Boor on the node's span),
// then one thread per band entry.  Band storage [factor][row][2p+1], entry k <-> column
// j = i - p + k, zero outside the (Dirichlet-sliced) matrix.
#include <cstdio>
#include <cstring>

#include "internal.h"

namespace igalr {

// p+1 nonzero B-splines and first derivatives at t on knot span s (knots[s] <= t < knots[s+1]).
// Triangular Cox-de Boor with left/right differences; derivatives from the degree p-1 values.
__global__ void k_basis_at_nodes(const double* __restrict__ knots, const int* __restrict__ span,
                                 const double* __restrict__ node, int ne, int nq, int p,
                                 double* __restrict__ Bv, double* __restrict__ Bd) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ne * nq) return;
    const int e = g / nq;
    const int s = span[e];
    const double t = node[g];
    double N[kMaxP + 1], left[kMaxP + 1], right[kMaxP + 1], Np1[kMaxP + 1];
    N[0] = 1.0;
    Np1[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = t - knots[s + 1 - j];
        right[j] = knots[s + j] - t;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double den = right[r + 1] + left[j - r];
            const double tmp = N[r] / den;
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
        if (j == p - 1)
            for (int r = 0; r <= j; ++r) Np1[r] = N[r];
    }
    if (p == 1) { Np1[0] = 1.0; }
    for (int l = 0; l <= p; ++l) {
        double d = 0.0;
        if (l >= 1) {
            const double den = knots[s + l] - knots[s - p + l];
            if (den != 0.0) d += p * Np1[l - 1] / den;
        }
        if (l <= p - 1) {
            const double den = knots[s + l + 1] - knots[s - p + l + 1];
            if (den != 0.0) d -= p * Np1[l] / den;
        }
        Bv[(size_t)g * (p + 1) + l] = N[l];
        Bd[(size_t)g * (p + 1) + l] = d;
    }
}

struct SpecDev {
    int table, a, b;
};

__global__ void k_band_entries(const SpecDev* __restrict__ specs, int nf, const double* __restrict__ tables,
                               const double* __restrict__ wgt, const double* __restrict__ Bv,
                               const double* __restrict__ Bd, const int* __restrict__ elem_of_span, int n,
                               int p, int nq, int nnodes, int m, int off, double* __restrict__ band) {
    const int bw = 2 * p + 1;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (long long)nf * m * bw) return;
    const int k = (int)(tid % bw);
    const int io = (int)((tid / bw) % m);
    const int f = (int)(tid / ((long long)bw * m));
    const int i = io + off;
    const int j = i - p + k;
    const int jo = j - off;
    double acc = 0.0;
    if (jo >= 0 && jo < m) {
        const SpecDev sp = specs[f];
        const double* tab = tables + (size_t)sp.table * nnodes;
        const double* Ba = sp.a ? Bd : Bv;
        const double* Bb = sp.b ? Bd : Bv;
        const int lo = max(max(i, j), p);
        const int hi = min(min(i, j) + p, n - 1);
        for (int s = lo; s <= hi; ++s) {
            const int e = elem_of_span[s];
            if (e < 0) continue;
            const int li = i - (s - p), lj = j - (s - p);
            for (int q = 0; q < nq; ++q) {
                const int g = e * nq + q;
                acc += wgt[g] * tab[g] * Ba[(size_t)g * (p + 1) + li] * Bb[(size_t)g * (p + 1) + lj];
            }
        }
    }
    band[tid] = acc;
}

#define CKR(x)                                              \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) return cuda_error(e_, #x);   \
    } while (0)

iga_status assemble_dir(const DirQuad& q, const std::vector<std::vector<double>>& tables,
                        const std::vector<FactorSpec>& specs, bool dirichlet, cudaStream_t st, DirFactors* out) {
    const int nnodes = q.ne * q.nq;
    const int p = q.p, n = q.n;
    const int m = dirichlet ? n - 2 : n;
    const int bw = 2 * p + 1;
    const int nf = (int)specs.size();
    out->m = m;
    out->p = p;
    out->bw = bw;
    out->nf = nf;
    out->pattern.clear();
    out->table.clear();
    for (auto& s : specs) {
        out->pattern.push_back(s.a * 2 + s.b);
        out->table.push_back(s.table);
    }
    if (nf == 0) return IGA_OK;

    std::vector<int> eos(n, -1);
    for (int e = 0; e < q.ne; ++e) eos[q.span[e]] = e;
    std::vector<double> tabs((size_t)tables.size() * nnodes);
    for (size_t t = 0; t < tables.size(); ++t) memcpy(&tabs[t * nnodes], tables[t].data(), sizeof(double) * nnodes);
    std::vector<SpecDev> sd(nf);
    for (int f = 0; f < nf; ++f) sd[f] = {specs[f].table, specs[f].a, specs[f].b};

    double *d_knots = nullptr, *d_node = nullptr, *d_wgt = nullptr, *d_tabs = nullptr, *d_Bv = nullptr, *d_Bd = nullptr;
    int *d_span = nullptr, *d_eos = nullptr;
    SpecDev* d_spec = nullptr;
    iga_status rc = IGA_OK;
    auto fail = [&](cudaError_t e, const char* w) {
        rc = cuda_error(e, w);
        return rc;
    };
    cudaError_t e;
#define TRY(x)                                   \
    if ((e = (x)) != cudaSuccess) {              \
        fail(e, #x);                             \
        goto cleanup;                            \
    }
    TRY(cudaMalloc(&d_knots, sizeof(double) * q.knots.size()));
    TRY(cudaMalloc(&d_node, sizeof(double) * nnodes));
    TRY(cudaMalloc(&d_wgt, sizeof(double) * nnodes));
    TRY(cudaMalloc(&d_tabs, sizeof(double) * (tabs.size() ? tabs.size() : 1)));
    TRY(cudaMalloc(&d_Bv, sizeof(double) * (size_t)nnodes * (p + 1)));
    TRY(cudaMalloc(&d_Bd, sizeof(double) * (size_t)nnodes * (p + 1)));
    TRY(cudaMalloc(&d_span, sizeof(int) * q.ne));
    TRY(cudaMalloc(&d_eos, sizeof(int) * n));
    TRY(cudaMalloc(&d_spec, sizeof(SpecDev) * nf));
    // tail padding: fused kernels stage whole 128-column tiles of a factor's band rows
    TRY(cudaMalloc(&out->band, sizeof(double) * ((size_t)nf * m * bw + 256 * bw)));
    TRY(cudaMemsetAsync(out->band, 0, sizeof(double) * ((size_t)nf * m * bw + 256 * bw), st));
    TRY(cudaMemcpyAsync(d_knots, q.knots.data(), sizeof(double) * q.knots.size(), cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(d_node, q.node.data(), sizeof(double) * nnodes, cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(d_wgt, q.wgt.data(), sizeof(double) * nnodes, cudaMemcpyHostToDevice, st));
    if (tabs.size()) TRY(cudaMemcpyAsync(d_tabs, tabs.data(), sizeof(double) * tabs.size(), cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(d_span, q.span.data(), sizeof(int) * q.ne, cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(d_eos, eos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(d_spec, sd.data(), sizeof(SpecDev) * nf, cudaMemcpyHostToDevice, st));
    {
        const int th = 128;
        k_basis_at_nodes<<<(nnodes + th - 1) / th, th, 0, st>>>(d_knots, d_span, d_node, q.ne, q.nq, p, d_Bv, d_Bd);
        TRY(cudaGetLastError());
        const long long tot = (long long)nf * m * bw;
        k_band_entries<<<(unsigned)((tot + th - 1) / th), th, 0, st>>>(d_spec, nf, d_tabs, d_wgt, d_Bv, d_Bd, d_eos,
                                                                         n, p, q.nq, nnodes, m, dirichlet ? 1 : 0,
                                                                         out->band);
        TRY(cudaGetLastError());
        TRY(cudaStreamSynchronize(st));
    }
cleanup:
#undef TRY
    cudaFree(d_knots);
    cudaFree(d_node);
    cudaFree(d_wgt);
    cudaFree(d_tabs);
    cudaFree(d_Bv);
    cudaFree(d_Bd);
    cudaFree(d_span);
    cudaFree(d_eos);
    cudaFree(d_spec);
    if (rc != IGA_OK && out->band) {
        cudaFree(out->band);
        out->band = nullptr;
    }
    return rc;
}

}  // namespace igalr
