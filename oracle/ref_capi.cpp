// ref_capi.cpp -- C entry points over the REFERENCE's own code (TEST INFRASTRUCTURE).
//
// oracle/_ref/libmprec_ref.so = the unmodified reference sources
// (/root/reference/proj/src/*.cpp, compiled from where they lie by
// oracle/Makefile) + the Eigen-subset shim (oracle/eigen_shim) + this file.
// The functions below have the signatures of include/mprec_gpu.h with the
// prefix `ref_`, so tests drive the reference through the same Python wrapper
// (paper_1912_04385_b200.api.Api) as the oracle (`orc_`) and the GPU library
// (`mprec_gpu_`).  Everything here is marshalling between plain arrays and the
// reference's types; every computation is a call into the reference's public
// API (left_scale, build_preconditioner, StagePreconditioner::apply,
// AMGHierarchy::setup, rs_coarsen, ILU0Factor, gmres, residual_check,
// solve_system, condense, back_substitute).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../include/mprec_gpu.h"
#include "mprec/amg.hpp"
#include "mprec/block_matrix.hpp"
#include "mprec/condense.hpp"
#include "mprec/errors.hpp"
#include "mprec/gmres.hpp"
#include "mprec/harness.hpp"
#include "mprec/ilu0.hpp"
#include "mprec/scaling.hpp"
#include "mprec/stages.hpp"

using namespace mprec;

namespace {
thread_local std::string g_err;
thread_local int g_payload = -1;

template <class F>
int guard(F&& f) {
    g_payload = -1;
    try {
        f();
        return MPREC_OK;
    } catch (const SingularBlockError& e) {
        g_err = e.what();
        g_payload = e.cell_id;
        return MPREC_SINGULAR_BLOCK;
    } catch (const ZeroPivotError& e) {
        g_err = e.what();
        g_payload = e.row_id;
        return MPREC_ZERO_PIVOT;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return MPREC_DIMENSION;
    } catch (const IndexError& e) {
        g_err = e.what();
        return MPREC_INDEX;
    } catch (const SetupError& e) {
        g_err = e.what();
        return MPREC_SETUP;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return MPREC_CONFIG;
    } catch (const IoError& e) {
        g_err = e.what();
        return MPREC_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MPREC_INTERNAL;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

const char* kMethodNames[] = {"ilu0", "cpr-amg", "cpr-direct", "cptr3-amg", "cptr-direct", "cptr3-direct"};

MethodSpec method_spec(int m) {
    if (m < 0 || m > 5) throw ConfigError("unknown method id " + std::to_string(m));
    return parse_method(kMethodNames[m]);
}

AMGParams to_params(const mprec_amg_params* p) {
    AMGParams q;
    if (p) {
        q.strength_threshold = p->strength_threshold;
        q.max_coarse_size = p->max_coarse_size;
        q.max_levels = p->max_levels;
    }
    return q;
}

ScalingOptions to_options(const mprec_scaling_options* o) {
    ScalingOptions s;
    if (o) {
        s.diag_mode = o->diag_mode == MPREC_DIAG_SCALAR ? DiagMode::Scalar : DiagMode::Block;
        s.second_scaling_from_original = o->second_scaling_from_original != 0;
    }
    return s;
}

// Uniform BSR (column-major nb x nb blocks) -> BlockMatrix::assemble.
BlockMatrix to_block(const mprec_bsr* a) {
    if (!a || a->n_cells < 1 || a->nb < 1) throw DimensionError("bad block matrix shape");
    const int nc = a->n_cells, nb = a->nb;
    std::vector<BlockEntry> e;
    e.reserve(size_t(a->row_ptr[nc]));
    for (int c = 0; c < nc; ++c)
        for (int k = a->row_ptr[c]; k < a->row_ptr[c + 1]; ++k) {
            Eigen::MatrixXd b(nb, nb);
            std::memcpy(b.data(), a->values + size_t(k) * nb * nb, sizeof(double) * nb * nb);
            e.push_back({c, a->col_idx[k], std::move(b)});
        }
    // nb = 1 (scalar systems): one "s" unknown per cell would need P and T; a
    // P-only layout keeps the cell size at 1.
    FieldLayout lay = nb >= 2 ? FieldLayout::uniform(nc, nb - 2) : FieldLayout::uniform(nc, 0, true, false);
    return BlockMatrix::assemble(e, std::move(lay));
}

ScalarMatrix to_scalar(const mprec_csr* a) {
    std::vector<Triplet> t;
    for (int i = 0; i < a->n_rows; ++i)
        for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) t.push_back({i, a->col_idx[k], a->values[k]});
    return ScalarMatrix::from_triplets(a->n_rows, a->n_rows, std::move(t));
}

// BSR entries -> scalar triplets -> ScalarMatrix::from_triplets, without
// BlockMatrix::assemble (which would insert a missing diagonal block).
ScalarMatrix bsr_to_scalar(const mprec_bsr* a) {
    const int nb = a->nb;
    std::vector<Triplet> t;
    t.reserve(size_t(a->row_ptr[a->n_cells]) * nb * nb);
    for (int c = 0; c < a->n_cells; ++c)
        for (int k = a->row_ptr[c]; k < a->row_ptr[c + 1]; ++k)
            for (int col = 0; col < nb; ++col)
                for (int r = 0; r < nb; ++r)
                    t.push_back({c * nb + r, a->col_idx[k] * nb + col, a->values[size_t(k) * nb * nb + size_t(col) * nb + r]});
    return ScalarMatrix::from_triplets(a->n_cells * nb, a->n_cells * nb, std::move(t));
}

// Flat CSR on a block pattern -> column-major BSR block values.
void flat_to_bsr(int n_cells, int nb, const std::vector<int>& rp, const std::vector<int>& ci,
                 const ScalarMatrix& flat, double* out) {
    for (int c = 0; c < n_cells; ++c)
        for (int r = 0; r < nb; ++r) {
            int q = flat.row_ptr()[c * nb + r];
            for (int k = rp[c]; k < rp[c + 1]; ++k)
                for (int col = 0; col < nb; ++col, ++q) {
                    if (flat.col_idx()[q] != ci[k] * nb + col)
                        throw SetupError("flattened pattern does not match the block pattern");
                    out[size_t(k) * nb * nb + size_t(col) * nb + r] = flat.values()[q];
                }
        }
}

Vector vec(const double* p, int n) {
    Vector v(n);
    std::memcpy(v.data(), p, sizeof(double) * n);
    return v;
}
void put(const Vector& v, double* out) { std::memcpy(out, v.data(), sizeof(double) * v.size()); }

void fill_result(mprec_solve_result* out, const SolveResult& r, int attempts, int total, double setup_s,
                 double solve_s, double* history, int cap) {
    std::memset(out, 0, sizeof(*out));
    out->iterations = r.iterations;
    out->converged = r.converged;
    out->breakdown = r.breakdown;
    out->attempts = attempts;
    out->total_iterations = total;
    out->final_true_residual = r.final_true_residual;
    out->setup_s = setup_s;
    out->solve_s = solve_s;
    int nh = int(r.residual_history.size());
    if (history && cap < nh) nh = cap;
    if (history)
        for (int i = 0; i < nh; ++i) history[i] = r.residual_history[i];
    out->history_len = history ? nh : int(r.residual_history.size());
}
}  // namespace

struct ref_amg {
    AMGHierarchy h;
    double theta = 0.25;
};
struct ref_ilu {
    int n_cells = 0, nb = 0;
    std::vector<int> rp, ci;
    ILU0Factor f;
};
struct ref_system {
    BlockMatrix a;
    Vector b;
    std::unique_ptr<ScaledSystem> sc;
    std::unique_ptr<StagePreconditioner> prec;
    MethodSpec spec;
    AMGParams params;
    std::vector<std::unique_ptr<ref_amg>> stage_views;
    double setup_s = 0.0;
};
struct ref_condensed {
    ReducedSystem r;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_error_payload(void) { return g_payload; }

int ref_create(const mprec_bsr* a, ref_system** out) {
    return guard([&] {
        auto h = std::make_unique<ref_system>();
        h->a = to_block(a);
        *out = h.release();
    });
}

int ref_setup_opts(ref_system* h, int method, const mprec_amg_params* amg, const mprec_scaling_options* so,
                   const double* b) {
    return guard([&] {
        h->prec.reset();
        h->sc.reset();
        h->stage_views.clear();
        h->spec = method_spec(method);
        h->params = to_params(amg);
        h->b = vec(b, h->a.dim());
        const double t0 = now_s();
        h->sc = std::make_unique<ScaledSystem>(left_scale(h->a, h->b, h->spec.method, to_options(so)));
        h->prec = std::make_unique<StagePreconditioner>(build_preconditioner(*h->sc, h->spec, h->params));
        h->setup_s = now_s() - t0;
    });
}

int ref_setup(ref_system* h, int method, const mprec_amg_params* amg, const double* b) {
    return ref_setup_opts(h, method, amg, nullptr, b);
}

int ref_apply(ref_system* h, const double* r, double* z) {
    return guard([&] {
        if (!h->prec) throw SetupError("setup not done");
        put(h->prec->apply(vec(r, h->a.dim())), z);
    });
}

int ref_apply_stage(ref_system* h, int stage, const double* r, double* z) {
    return guard([&] {
        if (!h->prec) throw SetupError("setup not done");
        if (stage < 0 || stage >= h->prec->n_stages()) throw IndexError("stage out of range");
        put(h->prec->apply_stage(stage, vec(r, h->a.dim())), z);
    });
}

int ref_spmv(ref_system* h, int which, const double* x, double* y) {
    return guard([&] {
        const Vector xv = vec(x, h->a.dim());
        if (which == 0) {
            put(h->a.apply(xv), y);
        } else {
            if (!h->prec) throw SetupError("setup not done");
            put(h->prec->a_bar().apply(xv), y);
        }
    });
}

// solve_system's attempt loop (harness.cpp:198-218) on the handle's own
// preconditioner (which may carry non-default AMG / scaling options);
// ref_solve_system below is the reference's solve_system itself.
int ref_solve(ref_system* h, double tol, int max_iter, double* x, mprec_solve_result* out, double* history,
              int history_cap) {
    return guard([&] {
        if (!h->prec) throw SetupError("setup not done");
        const double t0 = now_s();
        GmresOptions opts;
        opts.tol = tol;
        opts.max_iter = max_iter;
        const BlockMatrix& a = h->a;
        const LinearOperator orig{a.dim(), [&a](const Vector& v) { return a.apply(v); }};
        SolveResult res;
        int attempts = 0, total = 0, it[3] = {0, 0, 0}, cv[3] = {0, 0, 0};
        double at[3] = {0, 0, 0}, ar[3] = {0, 0, 0};
        for (int attempt = 0; attempt < 3; ++attempt) {
            ++attempts;
            at[attempt] = opts.tol;
            res = gmres(LinearOperator::from(h->prec->a_bar()), h->sc->b_bar, h->prec->as_operator(), opts);
            total += res.iterations;
            res.final_true_residual = residual_check(orig, h->b, res.x);
            it[attempt] = res.iterations;
            cv[attempt] = res.converged;
            ar[attempt] = res.final_true_residual;
            if (!res.converged || res.final_true_residual <= tol) break;
            opts.tol *= 0.5 * tol / res.final_true_residual;
        }
        if (res.converged && res.final_true_residual > tol) res.converged = false;
        put(res.x, x);
        fill_result(out, res, attempts, total, h->setup_s, now_s() - t0, history, history_cap);
        for (int q = 0; q < 3; ++q) {
            out->attempt_iterations[q] = it[q];
            out->attempt_converged[q] = cv[q];
            out->attempt_tol[q] = at[q];
            out->attempt_true_residual[q] = ar[q];
        }
    });
}

int ref_solve_system(const mprec_bsr* a, const double* b, int method, double tol, int max_iter, double* x,
                     mprec_solve_result* out) {
    return guard([&] {
        const BlockMatrix m = to_block(a);
        const double t0 = now_s();
        const SolveOutcome o = solve_system(m, vec(b, m.dim()), method_spec(method), tol, max_iter);
        put(o.result.x, x);
        fill_result(out, o.result, -1, -1, o.setup_time_s, now_s() - t0 - o.setup_time_s, nullptr, 0);
    });
}

int ref_scaling_record(ref_system* h, char* buf, int cap) {
    return guard([&] {
        if (!h->sc) throw SetupError("setup not done");
        std::string s;
        for (const std::string& r : h->sc->scaling_record) s += (s.empty() ? "" : ", ") + r;
        if (cap > 0) {
            std::strncpy(buf, s.c_str(), size_t(cap) - 1);
            buf[cap - 1] = 0;
        }
    });
}

int ref_get_scaled(ref_system* h, double* abar, double* bbar) {
    return guard([&] {
        if (!h->sc) throw SetupError("setup not done");
        const BlockMatrix& m = h->sc->a_bar;
        if (abar)
            for (int k = 0; k < m.n_blocks(); ++k)
                std::memcpy(abar + size_t(k) * m.block(k).size(), m.block(k).data(),
                            sizeof(double) * m.block(k).size());
        if (bbar) put(h->sc->b_bar, bbar);
    });
}

// The stage's ILU0Factor is private to Stage; ILU0Factor::factor on the same
// a_bar() is deterministic, so refactoring it gives the same factors.
int ref_get_ilu(ref_system* h, double* lu) {
    return guard([&] {
        if (!h->prec) throw SetupError("setup not done");
        const BlockMatrix& m = h->sc->a_bar;
        flat_to_bsr(m.n_cells(), m.dim() / m.n_cells(), m.row_ptr(), m.col_idx(),
                    ILU0Factor::factor(h->prec->a_bar()).factors(), lu);
    });
}

int ref_n_stages(ref_system* h, int* n) {
    return guard([&] { *n = h->prec ? h->prec->n_stages() : 0; });
}

// The stage's AMGHierarchy is private to Stage; AMGHierarchy::setup on the
// same sub-system (stages.cpp:93-97, 125-127) is deterministic.
int ref_stage_amg(ref_system* h, int stage, ref_amg** out) {
    return guard([&] {
        if (!h->prec) throw SetupError("setup not done");
        if (h->spec.sub != SubSolver::Amg || stage < 0 || stage >= h->prec->n_stages() - 1)
            throw IndexError("not an AMG stage");
        const ScalarMatrix& m = h->spec.method == Method::Cptr3 && stage == 0 ? h->sc->c_tt : h->sc->b_pp;
        auto v = std::make_unique<ref_amg>();
        v->h = AMGHierarchy::setup(m, h->params);
        v->theta = h->params.strength_threshold;
        *out = v.get();
        h->stage_views.push_back(std::move(v));
    });
}

void ref_destroy(ref_system* h) { delete h; }

int ref_get_shape(ref_system* h, int* n_cells, int* nb, int* nnzb) {
    return guard([&] {
        if (n_cells) *n_cells = h->a.n_cells();
        if (nb) *nb = h->a.dim() / h->a.n_cells();
        if (nnzb) *nnzb = h->a.n_blocks();
    });
}

// ---- sub-solvers ----------------------------------------------------------

int ref_amg_create(const mprec_csr* a, const mprec_amg_params* p, ref_amg** out) {
    return guard([&] {
        auto v = std::make_unique<ref_amg>();
        const AMGParams q = to_params(p);
        v->h = AMGHierarchy::setup(to_scalar(a), q);
        v->theta = q.strength_threshold;
        *out = v.release();
    });
}

int ref_amg_apply(ref_amg* h, const double* r, double* x) {
    return guard([&] { put(h->h.apply(vec(r, h->h.dim())), x); });
}

int ref_amg_n_levels(ref_amg* h, int* n) {
    return guard([&] { *n = h->h.n_levels(); });
}

int ref_amg_level_info(ref_amg* h, int level, int* n, int* nnz_a, int* nnz_p) {
    return guard([&] {
        if (level < 0 || level >= h->h.n_levels()) throw IndexError("level out of range");
        const auto& L = h->h.level(level);
        *n = L.a.rows();
        *nnz_a = L.a.nnz();
        *nnz_p = level == 0 ? 0 : L.p.nnz();
    });
}

int ref_amg_get_csr(ref_amg* h, int level, int which, int* rp, int* ci, double* v) {
    return guard([&] {
        if (level < 0 || level >= h->h.n_levels()) throw IndexError("level out of range");
        const auto& L = h->h.level(level);
        const ScalarMatrix& m = which == 0 ? L.a : (which == 1 ? L.p : L.r);
        if (rp) std::memcpy(rp, m.row_ptr().data(), m.row_ptr().size() * sizeof(int));
        if (ci) std::memcpy(ci, m.col_idx().data(), m.col_idx().size() * sizeof(int));
        if (v) std::memcpy(v, m.values().data(), m.values().size() * sizeof(double));
    });
}

// AMGHierarchy keeps no C/F marks; rs_coarsen (amg.cpp:47-186) on the level's
// operator is the splitting setup() used.
int ref_amg_get_cf(ref_amg* h, int level, signed char* cf) {
    return guard([&] {
        if (level < 0 || level + 1 >= h->h.n_levels()) throw IndexError("level has no coarsening");
        const CoarseningResult cr = rs_coarsen(h->h.level(level).a, h->theta);
        for (size_t i = 0; i < cr.is_coarse.size(); ++i) cf[i] = cr.is_coarse[i];
    });
}

void ref_amg_destroy(ref_amg* h) { delete h; }

int ref_ilu_create(const mprec_bsr* a, ref_ilu** out) {
    return guard([&] {
        auto v = std::make_unique<ref_ilu>();
        v->n_cells = a->n_cells;
        v->nb = a->nb;
        v->rp.assign(a->row_ptr, a->row_ptr + a->n_cells + 1);
        v->ci.assign(a->col_idx, a->col_idx + a->row_ptr[a->n_cells]);
        v->f = ILU0Factor::factor(bsr_to_scalar(a));
        *out = v.release();
    });
}

int ref_ilu_apply(ref_ilu* h, const double* r, double* y) {
    return guard([&] { put(h->f.apply(vec(r, h->f.dim())), y); });
}

int ref_ilu_get(ref_ilu* h, double* lu) {
    return guard([&] { flat_to_bsr(h->n_cells, h->nb, h->rp, h->ci, h->f.factors(), lu); });
}

void ref_ilu_destroy(ref_ilu* h) { delete h; }

int ref_gmres(const mprec_bsr* a, const double* b, int prec_kind, void* prec, double tol, int max_iter, double* x,
              mprec_solve_result* out, double* history, int history_cap) {
    return guard([&] {
        const ScalarMatrix m = bsr_to_scalar(a);
        const int n = m.rows();
        LinearOperator mop;
        if (prec_kind == 0)
            mop = LinearOperator::identity(n);
        else if (prec_kind == 1)
            mop = {n, [prec](const Vector& v) { return static_cast<ref_amg*>(prec)->h.apply(v); }};
        else if (prec_kind == 2)
            mop = {n, [prec](const Vector& v) { return static_cast<ref_ilu*>(prec)->f.apply(v); }};
        else
            throw ConfigError("unknown preconditioner kind");
        GmresOptions o;
        o.tol = tol;
        o.max_iter = max_iter;
        const double t0 = now_s();
        const SolveResult r = gmres(LinearOperator::from(m), vec(b, n), mop, o);
        put(r.x, x);
        fill_result(out, r, 1, r.iterations, 0.0, now_s() - t0, history, history_cap);
    });
}

// ---- static condensation (condense.cpp:206-258) --------------------------

int ref_condense(const mprec_global_jacobian* j, ref_condensed** out) {
    return guard([&] {
        const int nc = j->n_cells, np = j->np;
        GlobalJacobian g;
        const mprec_bsr j11{nc, np, j->row_ptr, j->col_idx, j->j11};
        g.j11 = to_block(&j11);
        for (int c = 0; c < nc; ++c) {
            const int s0 = j->sec_off[c], ns = j->sec_off[c + 1] - s0;
            Eigen::MatrixXd j22(ns, ns), j21(ns, np);
            Eigen::VectorXd r2(ns);
            size_t o22 = 0;
            for (int q = 0; q < c; ++q) o22 += size_t(j->sec_off[q + 1] - j->sec_off[q]) * (j->sec_off[q + 1] - j->sec_off[q]);
            if (ns) {
                std::memcpy(j22.data(), j->j22 + o22, sizeof(double) * ns * ns);
                std::memcpy(j21.data(), j->j21 + size_t(s0) * np, sizeof(double) * ns * np);
                std::memcpy(r2.data(), j->r2 + s0, sizeof(double) * ns);
            }
            g.j22.push_back(std::move(j22));
            g.j21.push_back(std::move(j21));
            g.r2.push_back(std::move(r2));
        }
        size_t o12 = 0;
        for (int e = 0; e < j->n_j12; ++e) {
            const int c = j->j12_col[e];
            const int ns = j->sec_off[c + 1] - j->sec_off[c];
            Eigen::MatrixXd blk(np, ns);
            if (ns) std::memcpy(blk.data(), j->j12 + o12, sizeof(double) * np * ns);
            o12 += size_t(np) * ns;
            g.j12.push_back({j->j12_row[e], c, std::move(blk)});
        }
        g.r1 = vec(j->r1, nc * np);
        auto h = std::make_unique<ref_condensed>();
        h->r = condense(g);
        *out = h.release();
    });
}

int ref_condensed_shape(ref_condensed* h, int* n_cells, int* np, int* nnzb, int* n_secondary) {
    return guard([&] {
        const BlockMatrix& a = h->r.a;
        int n2 = 0;
        for (const auto& m : h->r.j21) n2 += int(m.rows());
        if (n_cells) *n_cells = a.n_cells();
        if (np) *np = a.dim() / a.n_cells();
        if (nnzb) *nnzb = a.n_blocks();
        if (n_secondary) *n_secondary = n2;
    });
}

int ref_condensed_get(ref_condensed* h, int* rp, int* ci, double* vals, double* b) {
    return guard([&] {
        const BlockMatrix& a = h->r.a;
        if (rp) std::memcpy(rp, a.row_ptr().data(), sizeof(int) * a.row_ptr().size());
        if (ci) std::memcpy(ci, a.col_idx().data(), sizeof(int) * a.col_idx().size());
        if (vals)
            for (int k = 0; k < a.n_blocks(); ++k)
                std::memcpy(vals + size_t(k) * a.block(k).size(), a.block(k).data(),
                            sizeof(double) * a.block(k).size());
        if (b) put(h->r.b, b);
    });
}

int ref_back_substitute(ref_condensed* h, const double* d1, double* d2) {
    return guard([&] {
        const Vector y = back_substitute(h->r, vec(d1, h->r.a.dim()));
        if (y.size()) put(y, d2);
    });
}

void ref_condensed_destroy(ref_condensed* h) { delete h; }

}  // extern "C"
