// abi.cu — C ABI of libigalr (include/iga_lr.h): validation, Gauss rule, factor
// deduplication, the shared-prefix evaluation plan, and dispatch of the CUDA kernels.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "internal.h"
#include "iga_lr_testing.h"

namespace igalr {

static thread_local std::string g_err;

iga_status set_error(iga_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

iga_status cuda_error(cudaError_t e, const char* where) {
    g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return IGA_ECUDA;
}

void clear_error() { g_err.clear(); }

// ------------------------------------------------------------------------------------
// Gauss-Legendre nodes/weights on [-1,1] (Newton on the Legendre recurrence, reading G1/G2).
static void gauss_legendre(int m, double* x, double* w) {
    for (int k = 0; k < (m + 1) / 2; ++k) {
        double t = std::cos(M_PI * (4.0 * k + 3.0) / (4.0 * m + 2.0));  // k-th largest root guess
        double P = 0.0, dP = 1.0;
        for (int it = 0; it < 64; ++it) {
            double pm1 = 1.0, pc = t;  // P_0, P_1
            for (int j = 2; j <= m; ++j) {
                double pn = ((2 * j - 1) * t * pc - (j - 1) * pm1) / j;
                pm1 = pc;
                pc = pn;
            }
            if (m == 1) { pc = t; pm1 = 1.0; }
            P = pc;
            dP = m * (pm1 - t * pc) / (1.0 - t * t);
            double dt = P / dP;
            t -= dt;
            if (std::fabs(dt) <= 1e-16 * std::fabs(t) + 1e-300) break;
        }
        double pm1 = 1.0, pc = t;
        for (int j = 2; j <= m; ++j) {
            double pn = ((2 * j - 1) * t * pc - (j - 1) * pm1) / j;
            pm1 = pc;
            pc = pn;
        }
        if (m == 1) { pc = t; pm1 = 1.0; }
        dP = m * (pm1 - t * pc) / (1.0 - t * t);
        const double wk = 2.0 / ((1.0 - t * t) * dP * dP);
        x[m - 1 - k] = t;
        w[m - 1 - k] = wk;
        x[k] = -t;
        w[k] = wk;
    }
    if (m % 2 == 1) x[m / 2] = 0.0;
}

static iga_status validate_dir(const iga_dir& d, int idx) {
    char buf[256];
    if (d.p < 1 || d.p > kMaxP) {
        snprintf(buf, sizeof buf, "dir %d: degree p=%d outside supported 1..%d", idx, d.p, kMaxP);
        return set_error(d.p < 1 ? IGA_EINVAL : IGA_EUNSUPPORTED, buf);
    }
    if (d.n < d.p + 1) {
        snprintf(buf, sizeof buf, "dir %d: n=%d < p+1=%d", idx, d.n, d.p + 1);
        return set_error(IGA_EINVAL, buf);
    }
    if (!d.knots) {
        snprintf(buf, sizeof buf, "dir %d: knots is NULL", idx);
        return set_error(IGA_EINVAL, buf);
    }
    const int L = d.n + d.p + 1;
    for (int i = 0; i < L; ++i) {
        double v = d.knots[i];
        if (!std::isfinite(v) || v < 0.0 || v > 1.0) {
            snprintf(buf, sizeof buf, "dir %d: knot %d = %g outside [0,1]", idx, i, v);
            return set_error(IGA_EINVAL, buf);
        }
        if (i > 0 && v < d.knots[i - 1]) {
            snprintf(buf, sizeof buf, "dir %d: knots decrease at %d", idx, i);
            return set_error(IGA_EINVAL, buf);
        }
    }
    for (int i = 0; i <= d.p; ++i)
        if (d.knots[i] != 0.0 || d.knots[L - 1 - i] != 1.0) {
            snprintf(buf, sizeof buf, "dir %d: knot vector is not open (first/last p+1 knots must be 0/1)", idx);
            return set_error(IGA_EINVAL, buf);
        }
    // interior multiplicity <= p (Eq. (knotVector))
    int run = 1;
    for (int i = d.p + 1; i < d.n; ++i) {
        run = (d.knots[i] == d.knots[i - 1] && i - 1 > d.p) ? run + 1 : 1;
        if (d.knots[i] > 0.0 && d.knots[i] < 1.0 && run > d.p) {
            snprintf(buf, sizeof buf, "dir %d: interior knot %g has multiplicity > p", idx, d.knots[i]);
            return set_error(IGA_EINVAL, buf);
        }
    }
    return IGA_OK;
}

static iga_status validate_space(const iga_space* sp) {
    if (!sp) return set_error(IGA_EINVAL, "space is NULL");
    for (int d = 0; d < 3; ++d) {
        iga_status s = validate_dir(sp->dir[d], d);
        if (s) return s;
    }
    if (sp->nq < 0 || sp->nq > kMaxNq) return set_error(IGA_EUNSUPPORTED, "nq outside 0..16");
    return IGA_OK;
}

static int nq_of(const iga_space* sp, int d) { return sp->nq ? sp->nq : sp->dir[d].p + 1; }

static DirQuad build_quad(const iga_dir& d, int nq) {
    DirQuad q;
    q.n = d.n;
    q.p = d.p;
    q.nq = nq;
    q.knots.assign(d.knots, d.knots + d.n + d.p + 1);
    double gx[kMaxNq], gw[kMaxNq];
    gauss_legendre(nq, gx, gw);
    for (int s = d.p; s < d.n; ++s) {
        const double a = q.knots[s], b = q.knots[s + 1];
        if (!(a < b)) continue;
        q.span.push_back(s);
        const double h = b - a;
        for (int k = 0; k < nq; ++k) {
            q.node.push_back(a + 0.5 * h * (gx[k] + 1.0));
            q.wgt.push_back(0.5 * h * gw[k]);
        }
    }
    q.ne = (int)q.span.size();
    return q;
}

// nnz of the kept banded 1D matrix (all band positions inside the matrix)
static double nnz1(int m, int p) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += std::min(i + p, m - 1) - std::max(i - p, 0) + 1;
    return s;
}

struct Term {
    int part;      // 0 mass, 1 stiffness
    int f[3];      // factor ids x, y, z
    double c;
};

// Greedy packing of terms (in r-major order) into rounds of bounded shape.
struct Limits {
    int x = kMaxX, p = kMaxPair, g = kMaxG, e = kMaxE, t = 1 << 20;  // t: total (pair,group) entries
};

static void build_plan(const iga_lr_op* op, const std::vector<Term>& terms_in, bool split_slots, Plan* pl, cudaStream_t st,
                       Limits lim = Limits(), bool fused_v1 = true) {
    // merge identical terms (same part, factors, and slot semantics)
    std::vector<Term> terms;
    for (const Term& t : terms_in) {
        bool merged = false;
        for (Term& u : terms)
            if (u.part == t.part && u.f[0] == t.f[0] && u.f[1] == t.f[1] && u.f[2] == t.f[2]) {
                u.c += t.c;
                merged = true;
                break;
            }
        if (!merged) terms.push_back(t);
    }
    pl->rounds.clear();
    Round cur;
    memset(&cur, 0, sizeof cur);
    auto flush = [&]() {
        if (cur.ng) pl->rounds.push_back(cur);
        memset(&cur, 0, sizeof cur);
    };
    for (const Term& t : terms) {
        if (t.c == 0.0) continue;
        const int slot = split_slots ? t.part : 0;
        for (int attempt = 0; attempt < 2; ++attempt) {
            int xe = -1, pe = -1, ge = -1;
            for (int i = 0; i < cur.nx; ++i)
                if (cur.xf[i] == t.f[0] && cur.xslot[i] == slot) xe = i;
            int need_x = xe < 0;
            if (!need_x)
                for (int j = 0; j < cur.np; ++j)
                    if (cur.pf[j] == t.f[1] && cur.px[j] == xe) pe = j;
            int need_p = pe < 0;
            for (int g = 0; g < cur.ng; ++g)
                if (cur.gf[g] == t.f[2] && cur.gpart[g] == t.part) ge = g;
            int need_g = ge < 0;
            int need_e = 1;
            if (ge >= 0 && pe >= 0)
                for (int e = 0; e < cur.ne[ge]; ++e)
                    if (cur.ep[ge][e] == pe) need_e = 0;
            int tot_e = 0;
            for (int g = 0; g < cur.ng; ++g) tot_e += cur.ne[g];
            bool fits = cur.nx + need_x <= lim.x && cur.np + need_p <= lim.p && cur.ng + need_g <= lim.g &&
                        (need_g || cur.ne[ge] + need_e <= lim.e) && tot_e + need_e <= lim.t;
            if (!fits) {
                flush();
                continue;
            }
            if (need_x) {
                xe = cur.nx++;
                cur.xf[xe] = t.f[0];
                cur.xslot[xe] = slot;
            }
            if (need_p) {
                pe = cur.np++;
                cur.pf[pe] = t.f[1];
                cur.px[pe] = xe;
            }
            if (need_g) {
                ge = cur.ng++;
                cur.gf[ge] = t.f[2];
                cur.gpart[ge] = t.part;
                cur.ne[ge] = 0;
            }
            int ee = -1;
            for (int e = 0; e < cur.ne[ge]; ++e)
                if (cur.ep[ge][e] == pe) ee = e;
            if (ee < 0) {
                ee = cur.ne[ge]++;
                cur.ep[ge][ee] = pe;
                cur.ec[ge][ee] = 0.0;
            }
            cur.ec[ge][ee] += t.c;
            break;
        }
    }
    flush();
    pl->n_x = pl->n_y = pl->n_z = 0;
    for (const Round& r : pl->rounds) {
        pl->n_x += r.nx;
        pl->n_y += r.np;
        pl->n_z += r.ng;
    }
    const double N = (double)op->m[0] * op->m[1] * op->m[2];
    pl->flops = 2.0 * (pl->n_x * nnz1(op->m[0], op->p[0]) * (N / op->m[0]) +
                       pl->n_y * nnz1(op->m[1], op->p[1]) * (N / op->m[1]) +
                       pl->n_z * nnz1(op->m[2], op->p[2]) * (N / op->m[2]));
    pl->fused_ok = fused_v1 && fused_supported(op, *pl);
    if (pl->fused_ok && prepare_fused(op, pl, st) != IGA_OK) pl->fused_ok = false;
}

// Stream-ordered scratch must not return memory to the OS between applies (a release
// threshold of 0 makes every apply re-map ~100 MB: ms of host time), so each op owns a pool
// with an infinite threshold instead of changing the device's default pool for the process.
cudaError_t make_pool(int device, cudaMemPool_t* pool) {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof props);
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaError_t e = cudaMemPoolCreate(pool, &props);
    if (e) {
        *pool = nullptr;
        return e;
    }
    uint64_t thr = ~0ULL;
    return cudaMemPoolSetAttribute(*pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

static iga_status check_sep(const iga_sep* s, const int* nn, const char* what) {
    char buf[200];
    if (s->R < 1) {
        snprintf(buf, sizeof buf, "%s: R=%d < 1", what, s->R);
        return set_error(IGA_EINVAL, buf);
    }
    for (int d = 0; d < 3; ++d) {
        if (!s->tab[d]) {
            snprintf(buf, sizeof buf, "%s: tab[%d] is NULL", what, d);
            return set_error(IGA_EINVAL, buf);
        }
        for (long long i = 0; i < (long long)s->R * nn[d]; ++i)
            if (!std::isfinite(s->tab[d][i])) {
                snprintf(buf, sizeof buf, "%s: non-finite table value (dir %d)", what, d);
                return set_error(IGA_EINVAL, buf);
            }
    }
    if (s->coef)
        for (int r = 0; r < s->R; ++r)
            if (!std::isfinite(s->coef[r])) {
                snprintf(buf, sizeof buf, "%s: non-finite coef", what);
                return set_error(IGA_EINVAL, buf);
            }
    return IGA_OK;
}

}  // namespace igalr

using namespace igalr;

extern "C" {

const char* iga_last_error(void) { return g_err.c_str(); }

const char* iga_version(void) { return "igalr 0.1 (sm_100a)"; }

iga_status iga_quad_nodes(const iga_space* sp, int32_t dir, double* nodes_out, int64_t* nnodes) {
    g_err.clear();
    if (iga_status s = validate_space(sp)) return s;
    if (dir < 0 || dir > 2) return set_error(IGA_EINVAL, "dir must be 0..2");
    if (!nnodes) return set_error(IGA_EINVAL, "nnodes is NULL");
    DirQuad q = build_quad(sp->dir[dir], nq_of(sp, dir));
    *nnodes = (int64_t)q.node.size();
    if (nodes_out) memcpy(nodes_out, q.node.data(), sizeof(double) * q.node.size());
    return IGA_OK;
}

iga_status iga_lr_assemble_factors(const iga_space* sp, const iga_sep* omega, const iga_sep* const* q, uint32_t flags,
                                   void* stream, iga_lr_op** out) {
    NvtxRange nvtx_("iga_lr_assemble_factors");
    g_err.clear();
    if (!out) return set_error(IGA_EINVAL, "out is NULL");
    *out = nullptr;
    if (iga_status s = validate_space(sp)) return s;
    if (flags & ~IGA_DIRICHLET) return set_error(IGA_EINVAL, "unknown flags");
    const bool dir = (flags & IGA_DIRICHLET) != 0;
    for (int d = 0; d < 3; ++d)
        if (dir && sp->dir[d].n < 3) return set_error(IGA_EINVAL, "Dirichlet elimination needs n >= 3");
    bool any_q = false;
    if (q)
        for (int b = 0; b < 9; ++b) any_q |= q[b] != nullptr;
    if (!omega && !any_q) return set_error(IGA_EINVAL, "neither mass nor stiffness weight given");
    cudaStream_t st = (cudaStream_t)stream;

    DirQuad quad[3];
    int nn[3];
    for (int d = 0; d < 3; ++d) {
        quad[d] = build_quad(sp->dir[d], nq_of(sp, d));
        nn[d] = (int)quad[d].node.size();
    }
    if (omega)
        if (iga_status s = check_sep(omega, nn, "omega")) return s;
    if (q)
        for (int b = 0; b < 9; ++b)
            if (q[b]) {
                char w[16];
                snprintf(w, sizeof w, "q[%d]", b);
                if (iga_status s = check_sep(q[b], nn, w)) return s;
            }

    // Deduplicate weight tables and (table, pattern) factors per direction.
    std::vector<std::vector<double>> tables[3];
    std::vector<FactorSpec> specs[3];
    auto table_id = [&](int d, const double* t) {
        for (size_t i = 0; i < tables[d].size(); ++i)
            if (memcmp(tables[d][i].data(), t, sizeof(double) * nn[d]) == 0) return (int)i;
        tables[d].emplace_back(t, t + nn[d]);
        return (int)tables[d].size() - 1;
    };
    auto factor_id = [&](int d, int tab, int a, int b) {
        for (size_t i = 0; i < specs[d].size(); ++i)
            if (specs[d][i].table == tab && specs[d][i].a == a && specs[d][i].b == b) return (int)i;
        specs[d].push_back({tab, a, b});
        return (int)specs[d].size() - 1;
    };
    // Q is symmetric when every off-diagonal pair (q_kl, q_lk) carries the same weight (same
    // R, coefficients and tables); then K = K^T.  Otherwise the KKT matvec needs K^T
    // separately: block (k,l) of K^T is q_kl with the derivative patterns of block (l,k).
    auto same_sep = [&](const iga_sep* a, const iga_sep* b) {
        if (a == b) return true;
        if (!a || !b || a->R != b->R) return false;
        for (int r = 0; r < a->R; ++r)
            if ((a->coef ? a->coef[r] : 1.0) != (b->coef ? b->coef[r] : 1.0)) return false;
        for (int d = 0; d < 3; ++d)
            if (a->tab[d] != b->tab[d] && memcmp(a->tab[d], b->tab[d], sizeof(double) * (size_t)a->R * nn[d]) != 0)
                return false;
        return true;
    };
    bool qsym = true;
    if (q)
        for (int k = 0; k < 3; ++k)
            for (int l = k + 1; l < 3; ++l) qsym = qsym && same_sep(q[k * 3 + l], q[l * 3 + k]);
    // Terms in r-major order: mass r, then stiffness blocks (k,l) for the same r.
    std::vector<Term> terms, termsT;
    int maxR = omega ? omega->R : 0;
    if (q)
        for (int b = 0; b < 9; ++b)
            if (q[b]) maxR = std::max(maxR, (int)q[b]->R);
    for (int r = 0; r < maxR; ++r) {
        if (omega && r < omega->R) {
            Term t;
            t.part = 0;
            t.c = omega->coef ? omega->coef[r] : 1.0;
            for (int d = 0; d < 3; ++d) t.f[d] = factor_id(d, table_id(d, omega->tab[d] + (size_t)r * nn[d]), 0, 0);
            terms.push_back(t);
        }
        if (q)
            for (int b = 0; b < 9; ++b) {
                if (!q[b] || r >= q[b]->R) continue;
                const int k = b / 3, l = b % 3;  // K_ij = sum_kl q_kl d_l beta_i d_k beta_j
                Term t;
                t.part = 1;
                t.c = q[b]->coef ? q[b]->coef[r] : 1.0;
                for (int d = 0; d < 3; ++d)
                    t.f[d] = factor_id(d, table_id(d, q[b]->tab[d] + (size_t)r * nn[d]), l == d ? 1 : 0, k == d ? 1 : 0);
                terms.push_back(t);
                if (!qsym) {  // K^T: (K_kl^(d))^T = pattern (delta(k,d), delta(l,d)) with weight q_kl
                    for (int d = 0; d < 3; ++d)
                        t.f[d] = factor_id(d, table_id(d, q[b]->tab[d] + (size_t)r * nn[d]), k == d ? 1 : 0, l == d ? 1 : 0);
                    termsT.push_back(t);
                }
            }
    }

    iga_lr_op* op = new (std::nothrow) iga_lr_op();
    if (!op) return set_error(IGA_ENOMEM, "host allocation failed");
    cudaGetDevice(&op->device);
    if (cudaError_t e = make_pool(op->device, &op->pool)) {
        delete op;
        return cuda_error(e, "cudaMemPoolCreate");
    }
    op->nq = sp->nq ? sp->nq : 0;
    op->dirichlet = dir;
    op->has_mass = omega != nullptr;
    op->has_stiff = any_q;
    op->stiff_sym = qsym;
    for (int d = 0; d < 3; ++d) {
        op->n[d] = sp->dir[d].n;
        op->p[d] = sp->dir[d].p;
        op->m[d] = dir ? op->n[d] - 2 : op->n[d];
    }
    for (int d = 0; d < 3; ++d) {
        op->quad[d] = quad[d];
        iga_status s = assemble_dir(quad[d], tables[d], specs[d], dir, st, &op->F[d]);
        if (s) {
            iga_lr_destroy(op);
            return s;
        }
    }
    std::vector<Term> tm, ts;
    for (auto& t : terms) (t.part == 0 ? tm : ts).push_back(t);
    // merged term list for the TT functions (NEXT-3): identical (part, factors) terms summed
    for (const Term& t : terms) {
        bool merged = false;
        for (KTerm& u : op->kterms)
            if (u.part == t.part && u.f[0] == t.f[0] && u.f[1] == t.f[1] && u.f[2] == t.f[2]) {
                u.c += t.c;
                merged = true;
                break;
            }
        if (!merged) op->kterms.push_back({t.part, {t.f[0], t.f[1], t.f[2]}, t.c});
    }
    build_plan(op, terms, false, &op->plan[kPlanBoth], st);
    build_plan(op, terms, true, &op->plan[kPlanBothSplit], st);
    build_plan(op, tm, false, &op->plan[kPlanMass], st);
    build_plan(op, ts, false, &op->plan[kPlanStiff], st);
    if (!qsym) {
        std::vector<Term> tmT(tm);
        tmT.insert(tmT.end(), termsT.begin(), termsT.end());
        build_plan(op, termsT, false, &op->plan[kPlanStiffT], st);
        build_plan(op, tmT, true, &op->plan[kPlanBothSplitT], st);
    }
    if (fused2_supported(op)) {
        Limits lm;
        lm.x = lm.p = lm.g = lm.e = lm.t = 1;
        Limits ls;
        ls.x = 4;
        ls.p = 9;
        ls.g = 4;
        ls.e = 9;
        ls.t = 9;
        if (op->has_mass) {
            build_plan(op, tm, false, &op->plan[kPlanF2Mass], st, lm, false);
            if (prepare_fused2(op, &op->plan[kPlanF2Mass], 0, st) != IGA_OK) op->plan[kPlanF2Mass].f2_ok = false;
            prepare_canon(op, &op->plan[kPlanF2Mass], 0, st);
        }
        if (op->has_stiff) {
            build_plan(op, ts, false, &op->plan[kPlanF2Stiff], st, ls, false);
            if (prepare_fused2(op, &op->plan[kPlanF2Stiff], 1, st) != IGA_OK) op->plan[kPlanF2Stiff].f2_ok = false;
            prepare_canon(op, &op->plan[kPlanF2Stiff], 1, st);
            if (!qsym) {
                build_plan(op, termsT, false, &op->plan[kPlanF2StiffT], st, ls, false);
                if (prepare_fused2(op, &op->plan[kPlanF2StiffT], 1, st) != IGA_OK) op->plan[kPlanF2StiffT].f2_ok = false;
                prepare_canon(op, &op->plan[kPlanF2StiffT], 1, st);
            }
        }
        g_err.clear();
    }
    const double N = (double)op->m[0] * op->m[1] * op->m[2];
    op->min_bytes = 8.0 * N * (1 + (op->has_mass ? 1 : 0) + (op->has_stiff ? 1 : 0));
    // the plan uploads and z-record kernels are stream-ordered on `stream`: the op is usable
    // once they land (the call blocks on this stream only, never on the device)
    if (cudaError_t e = cudaStreamSynchronize(st)) {
        iga_lr_destroy(op);
        return cuda_error(e, "assembly");
    }
    *out = op;
    return IGA_OK;
}

void iga_lr_destroy(iga_lr_op* op) {
    if (!op) return;
    for (int d = 0; d < 3; ++d)
        if (op->F[d].band) cudaFree(op->F[d].band);
    for (int k = 0; k < kNumPlans; ++k) {
        release_fused(&op->plan[k]);
        if (op->plan[k].d_f2) cudaFree(op->plan[k].d_f2);
        if (op->plan[k].d_canon) cudaFree(op->plan[k].d_canon);
        if (op->plan[k].d_ztab) cudaFree(op->plan[k].d_ztab);
        if (op->plan[k].d_xtab) cudaFree(op->plan[k].d_xtab);
    }
    if (op->side) cudaStreamDestroy(op->side);
    if (op->host_sh) cudaStreamDestroy(op->host_sh);
    if (op->host_sd) cudaStreamDestroy(op->host_sd);
    for (cudaEvent_t x : op->host_ev) cudaEventDestroy(x);
    for (auto& c : op->fix_cache) {
        if (c.d_tab) cudaFree(c.d_tab);
        if (c.ready) cudaEventDestroy(c.ready);
    }
    if (op->pool) cudaMemPoolDestroy(op->pool);
    delete op;
}

static iga_status check_ptr(const void* p, const char* what) {
    if (((uintptr_t)p) & 7) return set_error(IGA_EINVAL, std::string(what) + " is not 8-byte aligned");
    return IGA_OK;
}

static iga_status run_plan(const iga_lr_op* op, PlanKind kind, const OutMap& om, int batch, uint32_t flags,
                           cudaStream_t st) {
    const Plan& pl = op->plan[kind];
    const uint32_t path = flags & (IGA_PATH_UNFUSED | IGA_PATH_FUSED | 0x40u);
    if ((path == IGA_PATH_FUSED || path == 0x40u) && !pl.fused_ok)
        return set_error(IGA_EUNSUPPORTED, "fused kernel does not support this plan/degree");
    if (path != IGA_PATH_UNFUSED && pl.fused_ok) return apply_fused(op, pl, om, batch, st);
    return apply_unfused(op, pl, om, batch, st);
}

// Fused-v2 routing: one launch per part (mass, stiffness); returns IGA_EUNSUPPORTED (no
// side effects) when a needed part has no fused-v2 plan.
static iga_status run_f2(const iga_lr_op* op, const double* xm, const double* xs, double* dm, double* ds, double alpha,
                         double gamma, int batch, cudaStream_t st, bool transposed = false) {
    const bool need_m = xm && dm, need_s = xs && ds;
    const PlanKind sk = transposed ? kPlanF2StiffT : kPlanF2Stiff;
    // a part runs on the canonical kernel when its plan has the canonical shape, else on the
    // generic k_fused2 (whose resident round tables bound R); neither => EUNSUPPORTED
    auto v2 = [&](const Plan& pl) { return pl.canon_ok || pl.f2_ok; };
    if (need_m && !v2(op->plan[kPlanF2Mass])) return IGA_EUNSUPPORTED;
    if (need_s && !v2(op->plan[sk])) return IGA_EUNSUPPORTED;
    iga_status s = IGA_OK;
    const bool generic = op->knobs.force_generic != 0;  // (test knob)
    auto part_run = [&](int part, const double* x, double* d, double sc, int acc, cudaStream_t ps) {
        const Plan& pl = op->plan[part ? sk : kPlanF2Mass];
        if (pl.canon_ok && !(generic && pl.f2_ok)) return apply_canon_part(op, pl, part, x, d, sc, acc, batch, ps);
        return apply_fused2_part(op, pl, part, x, d, sc, acc, batch, ps);
    };
    if (need_m && need_s && dm != ds && canon_small_grid(op, batch)) {
        // small meshes: neither persistent grid fills the GPU, so the mass part runs on a side
        // stream beside the stiffness part (fork/join with events; outputs do not alias)
        cudaStream_t side = nullptr;
        {
            std::lock_guard<std::mutex> lock(op->fix_mu);
            if (!op->side && cudaStreamCreateWithFlags(&op->side, cudaStreamNonBlocking) != cudaSuccess)
                op->side = nullptr;
            side = op->side;
        }
        cudaEvent_t ef = nullptr, ej = nullptr;
        if (side && cudaEventCreateWithFlags(&ef, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ej, cudaEventDisableTiming) == cudaSuccess) {
            cudaError_t e = cudaEventRecord(ef, st);
            if (!e) e = cudaStreamWaitEvent(side, ef, 0);
            if (e) return cuda_error(e, "fork");
            s = part_run(0, xm, dm, alpha, 0, side);
            const cudaError_t e2 = cudaEventRecord(ej, side);
            if (!s) s = part_run(1, xs, ds, gamma, 0, st);
            const cudaError_t e3 = cudaStreamWaitEvent(st, ej, 0);  // join (also on error)
            cudaEventDestroy(ef);
            cudaEventDestroy(ej);
            if (!s && (e2 || e3)) return cuda_error(e2 ? e2 : e3, "join");
            return s;
        }
        if (ef) cudaEventDestroy(ef);
        if (ej) cudaEventDestroy(ej);
    }
    if (need_m) s = part_run(0, xm, dm, alpha, 0, st);
    if (!s && need_s) s = part_run(1, xs, ds, gamma, (need_m && dm == ds) ? 1 : 0, st);
    return s;
}

static bool want_f2(const iga_lr_op* op, int batch, uint32_t flags) {
    const uint32_t path = flags & (IGA_PATH_UNFUSED | IGA_PATH_FUSED | 0x40u);
    if (path == IGA_PATH_FUSED) return true;
    return path == IGA_PATH_AUTO && fused2_preferred(op, batch);
}

// out = alpha M x_mass + gamma A x_stiff with A = K, or A = K^T when `transposed` (the KKT's
// calK^T block; the caller checks that the op holds the K^T plans)
static iga_status apply2_impl(const iga_lr_op* op, const double* x_mass, const double* x_stiff, double* out,
                              double alpha, double gamma, int32_t batch, uint32_t flags, void* stream,
                              bool transposed) {
    if (!op) return set_error(IGA_EINVAL, "op is NULL");
    if (!out) return set_error(IGA_EINVAL, "out is NULL");
    if (batch < 1) return set_error(IGA_EINVAL, "batch < 1");
    if (!x_mass && !x_stiff) return set_error(IGA_EINVAL, "both inputs NULL");
    if (x_mass && !op->has_mass) return set_error(IGA_ESTATE, "op has no mass part");
    if (x_stiff && !op->has_stiff) return set_error(IGA_ESTATE, "op has no stiffness part");
    if (out == x_mass || out == x_stiff) return set_error(IGA_EINVAL, "output aliases an input");
    for (const void* p : {(const void*)x_mass, (const void*)x_stiff, (const void*)out})
        if (iga_status s = check_ptr(p, "pointer")) return s;
    if (flags & ~(IGA_PATH_UNFUSED | IGA_PATH_FUSED | 0x40u)) return set_error(IGA_EINVAL, "unknown flags");
    if (want_f2(op, batch, flags)) {
        iga_status s = run_f2(op, x_mass, x_stiff, x_mass ? out : nullptr, x_stiff ? out : nullptr, alpha, gamma, batch,
                              (cudaStream_t)stream, transposed);
        if (s != IGA_EUNSUPPORTED) return s;
        g_err.clear();
    }
    OutMap om;
    om.src[0] = x_mass;
    om.src[1] = x_stiff;
    om.dst[0] = x_mass ? out : nullptr;
    om.dst[1] = x_stiff ? out : nullptr;
    om.scale[0] = alpha;
    om.scale[1] = gamma;
    PlanKind kind = (x_mass && x_stiff) ? (x_mass == x_stiff ? kPlanBoth : kPlanBothSplit) : (x_mass ? kPlanMass : kPlanStiff);
    if (transposed && x_stiff) kind = x_mass ? kPlanBothSplitT : kPlanStiffT;
    if (kind == kPlanMass || kind == kPlanStiff) {
        om.dst[0] = om.dst[1] = out;
        om.src[0] = om.src[1] = x_mass ? x_mass : x_stiff;
    }
    if (kind == kPlanBoth) om.dst[0] = om.dst[1] = out;
    if (kind == kPlanStiffT) {
        om.dst[0] = om.dst[1] = out;
        om.src[0] = om.src[1] = x_stiff;
    }
    return run_plan(op, kind, om, batch, flags, (cudaStream_t)stream);
}

iga_status iga_lr_apply2(const iga_lr_op* op, const double* x_mass, const double* x_stiff, double* out, double alpha,
                         double gamma, int32_t batch, uint32_t flags, void* stream) {
    NvtxRange nvtx_("iga_lr_apply2");
    g_err.clear();
    return apply2_impl(op, x_mass, x_stiff, out, alpha, gamma, batch, flags, stream, false);
}

iga_status iga_lr_apply(const iga_lr_op* op, const double* x, double* y_mass, double* y_stiff, double alpha,
                        double gamma, int32_t batch, uint32_t flags, void* stream) {
    NvtxRange nvtx_("iga_lr_apply");
    g_err.clear();
    if (!op) return set_error(IGA_EINVAL, "op is NULL");
    if (!x) return set_error(IGA_EINVAL, "x is NULL");
    if (batch < 1) return set_error(IGA_EINVAL, "batch < 1");
    if (!y_mass && !y_stiff) return set_error(IGA_EINVAL, "no output requested");
    if (y_mass && !op->has_mass) return set_error(IGA_ESTATE, "op has no mass part");
    if (y_stiff && !op->has_stiff) return set_error(IGA_ESTATE, "op has no stiffness part");
    if ((const double*)y_mass == x || (const double*)y_stiff == x) return set_error(IGA_EINVAL, "output aliases x");
    for (const void* p : {(const void*)x, (const void*)y_mass, (const void*)y_stiff})
        if (iga_status s = check_ptr(p, "pointer")) return s;
    if (flags & ~(IGA_PATH_UNFUSED | IGA_PATH_FUSED | 0x40u)) return set_error(IGA_EINVAL, "unknown flags");
    if (want_f2(op, batch, flags)) {
        iga_status s = run_f2(op, y_mass ? x : nullptr, y_stiff ? x : nullptr, y_mass, y_stiff, alpha, gamma, batch,
                              (cudaStream_t)stream);
        if (s != IGA_EUNSUPPORTED) return s;
        g_err.clear();
    }
    OutMap om;
    om.src[0] = om.src[1] = x;
    om.dst[0] = y_mass;
    om.dst[1] = y_stiff;
    om.scale[0] = alpha;
    om.scale[1] = gamma;
    PlanKind kind = (y_mass && y_stiff) ? kPlanBoth : (y_mass ? kPlanMass : kPlanStiff);
    if (kind != kPlanBoth) om.dst[0] = om.dst[1] = (y_mass ? y_mass : y_stiff);
    return run_plan(op, kind, om, batch, flags, (cudaStream_t)stream);
}

iga_status iga_kkt_apply(const iga_lr_op* op, int32_t n_t, double tau, double beta, const double* in, double* out,
                         uint32_t flags, void* stream) {
    NvtxRange nvtx_("iga_kkt_apply");
    g_err.clear();
    if (!op) return set_error(IGA_EINVAL, "op is NULL");
    if (!op->has_mass || !op->has_stiff) return set_error(IGA_ESTATE, "KKT needs mass and stiffness");
    if (n_t < 1) return set_error(IGA_EINVAL, "n_t < 1");
    if (!(tau > 0.0) || !std::isfinite(tau)) return set_error(IGA_EINVAL, "tau must be > 0");
    if (!(beta > 0.0) || !std::isfinite(beta)) return set_error(IGA_EINVAL, "beta must be > 0");
    if (!in || !out) return set_error(IGA_EINVAL, "NULL in/out");
    if (in == out) return set_error(IGA_EINVAL, "in and out alias");
    if (check_ptr(in, "in") || check_ptr(out, "out")) return IGA_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = (int64_t)op->m[0] * op->m[1] * op->m[2];
    const size_t blk = (size_t)n_t * N;
    const bool sym = op->stiff_sym;
    const bool canon = want_f2(op, 3 * n_t, flags) && op->plan[kPlanF2Mass].canon_ok && op->plan[kPlanF2Stiff].canon_ok &&
                       (sym || op->plan[kPlanF2StiffT].canon_ok) && !op->knobs.force_generic;
    if (canon) {
        // Canonical route (kkt.cu, k_kkt_combine): T = [M y, M u, M lambda, tau S^T lambda, tau S y], then
        // the per-step combinations.  One mass launch over the 3 n_t input vectors and one stiffness
        // launch over 2 n_t vectors ([lambda, y]: a batch split, vectors n_t.. read y at `in`), neither
        // accumulating: no launch reads its own output back.
        double* T = nullptr;
        cudaError_t e = pool_alloc(op->pool, (void**)&T, sizeof(double) * 5 * blk, st);
        if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(kkt)");
        iga_status s = apply_canon_part(op, op->plan[kPlanF2Mass], 0, in, T, 1.0, 0, 3 * n_t, st);
        if (!s && !sym) {
            // K != K^T: the lambda block takes the K^T plans
            s = apply_canon_part(op, op->plan[kPlanF2StiffT], 1, in + 2 * blk, T + 3 * blk, tau, 0, n_t, st);
            if (!s) s = apply_canon_part(op, op->plan[kPlanF2Stiff], 1, in, T + 4 * blk, tau, 0, n_t, st);
        } else if (!s) {
            CanonSplit sp;
            sp.bsplit = n_t;
            sp.src_jump = -3 * (long long)blk;  // in + 2 blk + b N - 3 blk = in + (b - n_t) N
            sp.dst_jump = 0;                    // T + 3 blk + b N = T + 4 blk + (b - n_t) N
            s = apply_canon_part(op, op->plan[kPlanF2Stiff], 1, in + 2 * blk, T + 3 * blk, tau, 0, 2 * n_t, st, sp);
            if (s == IGA_EUNSUPPORTED) {  // no split variant for this shape: one launch per segment
                s = apply_canon_part(op, op->plan[kPlanF2Stiff], 1, in + 2 * blk, T + 3 * blk, tau, 0, n_t, st);
                if (!s) s = apply_canon_part(op, op->plan[kPlanF2Stiff], 1, in, T + 4 * blk, tau, 0, n_t, st);
            }
        }
        if (!s) s = kkt_combine(T, out, n_t, N, tau, beta, st);
        cudaFreeAsync(T, st);
        return s;
    }
    double* abc = nullptr;  // a, b, c combos [3][n_t][N]
    cudaError_t e = pool_alloc(op->pool, (void**)&abc, sizeof(double) * 3 * blk, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(kkt)");
    iga_status s = kkt_combos(in, abc, n_t, N, tau, beta, st);  // abc = [b, tau a, c]
    if (!s) {
        // r_y = M b + tau S^T lambda ; r_u = tau M a ; r_lambda = M c + tau S y
        s = apply2_impl(op, abc, in + 2 * blk, out, 1.0, tau, n_t, flags, stream, !sym);
        if (!s) s = iga_lr_apply2(op, abc + blk, nullptr, out + blk, 1.0, 0.0, n_t, flags, stream);
        if (!s) s = iga_lr_apply2(op, abc + 2 * blk, in, out + 2 * blk, 1.0, tau, n_t, flags, stream);
    }
    cudaFreeAsync(abc, st);
    return s;
}

static iga_status host_roundtrip(const iga_lr_op* op, size_t in_elems, size_t out_elems, int nout, const double* in_h,
                                 double** out_h, cudaStream_t st, double** d_in, double** d_out) {
    cudaError_t e = pool_alloc(op->pool, (void**)d_in, sizeof(double) * in_elems, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(host in)");
    e = pool_alloc(op->pool, (void**)d_out, sizeof(double) * out_elems * nout, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(host out)");
    e = cudaMemcpyAsync(*d_in, in_h, sizeof(double) * in_elems, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_error(e, "H2D");
    (void)out_h;
    return IGA_OK;
}

// Host-buffer apply.  The batch is pipelined vector by vector over three streams: H2D copies
// (own stream), applies (the caller's stream) and D2H copies (own stream), ordered by events, so
// with pinned host buffers the PCIe transfers in both directions overlap each other and the
// kernels.  Device buffers are stream-ordered scratch on the caller's stream.
iga_status iga_lr_apply_host(const iga_lr_op* op, const double* x_host, double* y_mass_host, double* y_stiff_host,
                             double alpha, double gamma, int32_t batch, uint32_t flags, void* stream) {
    NvtxRange nvtx_("iga_lr_apply_host");
    g_err.clear();
    if (!op || !x_host || batch < 1 || (!y_mass_host && !y_stiff_host)) return set_error(IGA_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)op->m[0] * op->m[1] * op->m[2];
    const size_t tot = N * batch;
    // one host pipeline per op at a time: its copy streams and events are cached in the op
    std::lock_guard<std::mutex> pipe_lock(op->host_mu);
    double *d_in = nullptr, *d_out = nullptr;
    const bool same = y_mass_host && y_mass_host == y_stiff_host;
    int nout = same ? 1 : (y_mass_host ? 1 : 0) + (y_stiff_host ? 1 : 0);
    cudaError_t e = pool_alloc(op->pool, (void**)&d_in, sizeof(double) * tot, st);
    if (!e) e = pool_alloc(op->pool, (void**)&d_out, sizeof(double) * tot * nout, st);
    if (e) {
        if (d_in) cudaFreeAsync(d_in, st);
        return cuda_error(e, "cudaMallocAsync(host apply)");
    }
    double* dm = y_mass_host ? d_out : nullptr;
    double* ds = y_stiff_host ? (same ? d_out : d_out + (y_mass_host ? tot : 0)) : nullptr;
    const int nchunk = batch;
    // copy streams (H2D, D2H) and 3 events per chunk + 2, created once per op
    if (!op->host_sh) e = cudaStreamCreateWithFlags(&op->host_sh, cudaStreamNonBlocking);
    if (!e && !op->host_sd) e = cudaStreamCreateWithFlags(&op->host_sd, cudaStreamNonBlocking);
    const size_t nev = 3 * (size_t)nchunk + 2;
    while (!e && op->host_ev.size() < nev) {
        cudaEvent_t x = nullptr;
        e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        if (!e) op->host_ev.push_back(x);
    }
    cudaStream_t sh = op->host_sh, sd = op->host_sd;
    const std::vector<cudaEvent_t>& ev = op->host_ev;
    iga_status s = IGA_OK;
    if (!e) e = cudaEventRecord(ev[0], st);  // buffers allocated
    if (!e) e = cudaStreamWaitEvent(sh, ev[0], 0);
    if (!e) e = cudaStreamWaitEvent(sd, ev[0], 0);
    // per vector: H2D (sh) -> mass part (st) -> D2H of y_M (sd) overlapping the stiffness part
    // (st) -> D2H of y_S (sd); the D2H stream is the bottleneck (PCIe), so the first y_M leaves
    // while the first stiffness part still runs
    const bool split = y_mass_host && y_stiff_host && !same;
    for (int c = 0; c < nchunk && !e && !s; ++c) {
        const size_t off = (size_t)c * N;
        cudaEvent_t ein = ev[2 + 3 * c], em = ev[3 + 3 * c], eout = ev[4 + 3 * c];
        e = cudaMemcpyAsync(d_in + off, x_host + off, sizeof(double) * N, cudaMemcpyHostToDevice, sh);
        if (!e) e = cudaEventRecord(ein, sh);
        if (!e) e = cudaStreamWaitEvent(st, ein, 0);
        if (e) break;
        if (split) {
            s = iga_lr_apply(op, d_in + off, dm + off, nullptr, alpha, gamma, 1, flags, stream);
            if (s) break;
            e = cudaEventRecord(em, st);
            if (!e) e = cudaStreamWaitEvent(sd, em, 0);
            if (!e) e = cudaMemcpyAsync(y_mass_host + off, dm + off, sizeof(double) * N, cudaMemcpyDeviceToHost, sd);
            if (e) break;
            s = iga_lr_apply(op, d_in + off, nullptr, ds + off, alpha, gamma, 1, flags, stream);
            if (s) break;
            e = cudaEventRecord(eout, st);
            if (!e) e = cudaStreamWaitEvent(sd, eout, 0);
            if (!e) e = cudaMemcpyAsync(y_stiff_host + off, ds + off, sizeof(double) * N, cudaMemcpyDeviceToHost, sd);
            continue;
        }
        s = iga_lr_apply(op, d_in + off, dm ? dm + off : nullptr, ds ? ds + off : nullptr, alpha, gamma, 1, flags,
                         stream);
        if (s) break;
        e = cudaEventRecord(eout, st);
        if (!e) e = cudaStreamWaitEvent(sd, eout, 0);
        if (!e && y_mass_host)
            e = cudaMemcpyAsync(y_mass_host + off, dm + off, sizeof(double) * N, cudaMemcpyDeviceToHost, sd);
        if (!e && y_stiff_host && !same)
            e = cudaMemcpyAsync(y_stiff_host + off, ds + off, sizeof(double) * N, cudaMemcpyDeviceToHost, sd);
    }
    // the caller's stream waits for the last D2H before the buffers are released
    cudaError_t e3 = ev.size() > 1 ? cudaEventRecord(ev[1], sd) : cudaErrorInvalidValue;
    if (!e3) e3 = cudaStreamWaitEvent(st, ev[1], 0);
    cudaFreeAsync(d_in, st);
    cudaFreeAsync(d_out, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (s) return s;
    if (e) return cuda_error(e, "host apply pipeline");
    if (e3) return cuda_error(e3, "host apply pipeline");
    if (e2) return cuda_error(e2, "stream sync");
    return IGA_OK;
}

iga_status iga_kkt_apply_host(const iga_lr_op* op, int32_t n_t, double tau, double beta, const double* in_host,
                              double* out_host, uint32_t flags, void* stream) {
    NvtxRange nvtx_("iga_kkt_apply_host");
    g_err.clear();
    if (!op || !in_host || !out_host || n_t < 1) return set_error(IGA_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t tot = (size_t)op->m[0] * op->m[1] * op->m[2] * n_t * 3;
    double *d_in = nullptr, *d_out = nullptr;
    iga_status s = host_roundtrip(op, tot, tot, 1, in_host, nullptr, st, &d_in, &d_out);
    if (!s) s = iga_kkt_apply(op, n_t, tau, beta, d_in, d_out, flags, stream);
    cudaError_t e = cudaSuccess;
    if (!s) e = cudaMemcpyAsync(out_host, d_out, sizeof(double) * tot, cudaMemcpyDeviceToHost, st);
    if (d_in) cudaFreeAsync(d_in, st);
    if (d_out) cudaFreeAsync(d_out, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (s) return s;
    if (e) return cuda_error(e, "D2H");
    if (e2) return cuda_error(e2, "stream sync");
    return IGA_OK;
}

iga_status iga_lr_info(const iga_lr_op* op, iga_lr_info_t* info) {
    g_err.clear();
    if (!op || !info) return set_error(IGA_EINVAL, "NULL argument");
    memset(info, 0, sizeof *info);
    const Plan& pl = op->plan[op->has_mass && op->has_stiff ? kPlanBoth : (op->has_mass ? kPlanMass : kPlanStiff)];
    for (int d = 0; d < 3; ++d) {
        info->dims[d] = op->m[d];
        info->p[d] = op->p[d];
        info->n_factors[d] = op->F[d].nf;
    }
    info->nq = op->nq ? op->nq : op->p[0] + 1;
    info->n_rounds = (int32_t)pl.rounds.size();
    info->n_xprod = pl.n_x;
    info->n_yprod = pl.n_y;
    info->n_zprod = pl.n_z;
    info->has_mass = op->has_mass;
    info->has_stiff = op->has_stiff;
    info->fused_ok = pl.fused_ok;
    auto v2 = [&](const Plan& p) { return p.canon_ok || p.f2_ok; };
    info->fused2_ok = (!op->has_mass || v2(op->plan[kPlanF2Mass])) && (!op->has_stiff || v2(op->plan[kPlanF2Stiff]));
    info->min_bytes_per_vec = op->min_bytes;
    // flops of the plans the auto route executes (fused-v2 per-part plans when they exist)
    const Plan& f2m = op->plan[kPlanF2Mass];
    const Plan& f2s = op->plan[kPlanF2Stiff];
    const bool f2 = info->fused2_ok && fused2_preferred(op, 1);
    info->plan_flops_mass = op->has_mass ? (f2 ? f2m.flops : op->plan[kPlanMass].flops) : 0.0;
    info->plan_flops_stiff = op->has_stiff ? (f2 ? f2s.flops : op->plan[kPlanStiff].flops) : 0.0;
    info->plan_flops_per_vec = f2 ? info->plan_flops_mass + info->plan_flops_stiff : pl.flops;
    info->canon_mass = op->has_mass && f2 && f2m.canon_ok;
    info->canon_stiff = op->has_stiff && f2 && f2s.canon_ok;
    info->stiff_symmetric = op->stiff_sym;
    info->f2_rounds_stiff = op->has_stiff && v2(f2s) ? (int32_t)f2s.rounds.size() : 0;
    return IGA_OK;
}

iga_status iga_lr_test_knobs(iga_lr_op* op, const iga_test_knobs* k) {
    g_err.clear();
    if (!op || !k) return set_error(IGA_EINVAL, "NULL argument");
    if (k->qx != 0 && k->qx != 1 && k->qx != 2 && k->qx != 4) return set_error(IGA_EINVAL, "qx must be 0, 1, 2 or 4");
    if (k->minlen < 0) return set_error(IGA_EINVAL, "minlen < 0");
    if (k->vpack < 0) return set_error(IGA_EINVAL, "vpack < 0");
    op->knobs.force_generic = k->force_generic != 0;
    op->knobs.qx = k->qx;
    op->knobs.minlen = k->minlen;
    op->knobs.no_yres = k->no_yres != 0;
    op->knobs.no_tma = k->no_tma != 0;
    op->knobs.vpack = k->vpack;
    return IGA_OK;
}

iga_status iga_lr_test_tile(const iga_lr_op* op, int32_t batch, int32_t* qx, int32_t* lw, int32_t* vp) {
    g_err.clear();
    if (!op || !qx || !lw || !vp) return set_error(IGA_EINVAL, "NULL argument");
    if (batch < 1) return set_error(IGA_EINVAL, "batch < 1");
    if (!fused2_supported(op)) return set_error(IGA_EUNSUPPORTED, "no canonical kernel for this degree");
    int q = 0, l = 0, v = 0;
    canon_tile_choice(op, batch, &q, &l, &v);
    *qx = q;
    *lw = l;
    *vp = v;
    return IGA_OK;
}

iga_status iga_lr_export_factor(const iga_lr_op* op, int32_t dir, int32_t factor_id, double* host_band,
                                int32_t* pattern, int32_t* table) {
    g_err.clear();
    if (!op || dir < 0 || dir > 2) return set_error(IGA_EINVAL, "bad op/dir");
    const DirFactors& F = op->F[dir];
    if (factor_id < 0 || factor_id >= F.nf) return set_error(IGA_EINVAL, "factor_id out of range");
    if (pattern) *pattern = F.pattern[factor_id];
    if (table) *table = F.table[factor_id];
    if (host_band) {
        cudaError_t e = cudaMemcpy(host_band, F.band + (size_t)factor_id * F.m * F.bw, sizeof(double) * F.m * F.bw,
                                   cudaMemcpyDeviceToHost);
        if (e) return cuda_error(e, "export D2H");
    }
    return IGA_OK;
}

}  // extern "C"
