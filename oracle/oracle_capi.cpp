// oracle_capi.cpp -- C entry points of the CPU oracle (TEST INFRASTRUCTURE).
// Same signatures as include/mprec_gpu.h with the prefix `orc_`, so the parity
// tests drive both sides through one wrapper (tests/_native.py).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>

#include "../include/mprec_gpu.h"
#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;
thread_local int g_payload = -1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return MPREC_OK;
    } catch (const Error& e) {
        g_err = e.what();
        g_payload = e.payload;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_payload = -1;
        return MPREC_INTERNAL;
    }
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

Csr to_csr(const mprec_csr* a) {
    Csr m;
    m.rows = m.cols = a->n_rows;
    m.rp.assign(a->row_ptr, a->row_ptr + a->n_rows + 1);
    const int nnz = a->row_ptr[a->n_rows];
    m.ci.assign(a->col_idx, a->col_idx + nnz);
    m.v.assign(a->values, a->values + nnz);
    return m;
}

Bsr to_bsr(const mprec_bsr* a, int missing_diag_code = DIMENSION) {
    return Bsr::create(a->n_cells, a->nb, a->row_ptr, a->col_idx, a->values, missing_diag_code);
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

struct orc_system {
    Bsr a;
    Vec b;
    Vec b_ingested;
    ScaledSystem sc;
    StagePreconditioner prec;
    bool ready = false;
    double setup_s = 0.0;
};
struct orc_amg {
    AMGHierarchy h;
};
struct orc_condensed {
    ReducedSystem r;
};
struct orc_ilu {
    Ilu0Block f;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_error_payload(void) { return g_payload; }

int orc_create(const mprec_bsr* a, orc_system** out) {
    return guard([&] {
        auto* h = new orc_system;
        try {
            h->a = to_bsr(a);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int orc_setup_opts(orc_system* h, int method, const mprec_amg_params* amg, const mprec_scaling_options* so,
                   const double* b) {
    return guard([&] {
        if (!b) {
            if (int64_t(h->b_ingested.size()) != int64_t(h->a.dim())) throw Error(DIMENSION, "no rhs");
            b = h->b_ingested.data();
        }
        if (method < 0 || method > 5) throw Error(CONFIG, "unknown method id " + std::to_string(method));
        ScalingOptions o;
        if (so) {
            o.scalar_diag = so->diag_mode == MPREC_DIAG_SCALAR;
            o.second_scaling_from_original = so->second_scaling_from_original != 0;
        }
        h->ready = false;
        h->b.assign(b, b + h->a.dim());
        const double t0 = now_s();
        h->sc = left_scale(h->a, h->b, Method(method), o);
        h->prec = build_preconditioner(h->sc, to_params(amg));
        h->setup_s = now_s() - t0;
        h->ready = true;
    });
}

int orc_setup(orc_system* h, int method, const mprec_amg_params* amg, const double* b) {
    return orc_setup_opts(h, method, amg, nullptr, b);
}

int orc_scaling_record(orc_system* h, char* buf, int cap) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        std::string s;
        for (const std::string& r : h->sc.scaling_record) s += (s.empty() ? "" : ", ") + r;
        if (cap > 0) {
            std::strncpy(buf, s.c_str(), size_t(cap) - 1);
            buf[cap - 1] = 0;
        }
    });
}

int orc_apply(orc_system* h, const double* r, double* z) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        const Vec y = h->prec.apply(Vec(r, r + h->a.dim()));
        std::memcpy(z, y.data(), y.size() * sizeof(double));
    });
}

int orc_apply_stage(orc_system* h, int stage, const double* r, double* z) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        if (stage < 0 || stage >= int(h->prec.stages.size())) throw Error(INDEX, "stage out of range");
        const Vec y = h->prec.apply_stage(stage, Vec(r, r + h->a.dim()));
        std::memcpy(z, y.data(), y.size() * sizeof(double));
    });
}

int orc_spmv(orc_system* h, int which, const double* x, double* y) {
    return guard([&] {
        const Vec xv(x, x + h->a.dim());
        Vec r;
        if (which == 0)
            r = h->a.apply_block(xv);
        else {
            if (!h->ready) throw Error(SETUP, "setup not done");
            r = h->sc.a_bar.apply_flat(xv);
        }
        std::memcpy(y, r.data(), r.size() * sizeof(double));
    });
}

int orc_solve(orc_system* h, double tol, int max_iter, double* x, mprec_solve_result* out, double* history,
              int history_cap) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        const double t0 = now_s();
        GmresOptions opts;
        opts.tol = tol;
        opts.max_iter = max_iter;
        const Op orig = [h](const Vec& v) { return h->a.apply_block(v); };
        const Op abar = [h](const Vec& v) { return h->sc.a_bar.apply_flat(v); };
        const Op mop = [h](const Vec& v) { return h->prec.apply(v); };
        SolveResult res;
        int attempts = 0, total = 0;
        std::memset(out, 0, sizeof(*out));
        for (int attempt = 0; attempt < 3; ++attempt) {
            ++attempts;
            out->attempt_tol[attempt] = opts.tol;
            res = gmres(h->a.dim(), abar, h->sc.b_bar, mop, opts);
            total += res.iterations;
            res.final_true_residual = residual_check(orig, h->b, res.x);
            out->attempt_iterations[attempt] = res.iterations;
            out->attempt_converged[attempt] = res.converged;
            out->attempt_true_residual[attempt] = res.final_true_residual;
            if (!res.converged || res.final_true_residual <= tol) break;
            opts.tol *= 0.5 * tol / res.final_true_residual;
        }
        if (res.converged && res.final_true_residual > tol) res.converged = false;
        std::memcpy(x, res.x.data(), res.x.size() * sizeof(double));
        out->iterations = res.iterations;
        out->converged = res.converged;
        out->breakdown = res.breakdown;
        out->attempts = attempts;
        out->total_iterations = total;
        out->final_true_residual = res.final_true_residual;
        out->setup_s = h->setup_s;
        out->solve_s = now_s() - t0;
        int nh = int(res.residual_history.size());
        if (history && history_cap < nh) nh = history_cap;
        if (history)
            for (int i = 0; i < nh; ++i) history[i] = res.residual_history[i];
        out->history_len = history ? nh : int(res.residual_history.size());
    });
}

int orc_get_scaled(orc_system* h, double* abar, double* bbar) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        if (abar) std::memcpy(abar, h->sc.a_bar.val.data(), h->sc.a_bar.val.size() * sizeof(double));
        if (bbar) std::memcpy(bbar, h->sc.b_bar.data(), h->sc.b_bar.size() * sizeof(double));
    });
}

int orc_get_ilu(orc_system* h, double* lu) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        std::memcpy(lu, h->prec.ilu.lu.val.data(), h->prec.ilu.lu.val.size() * sizeof(double));
    });
}

int orc_n_stages(orc_system* h, int* n) {
    return guard([&] { *n = h->ready ? int(h->prec.stages.size()) : 0; });
}

int orc_stage_amg(orc_system* h, int stage, orc_amg** amg) {
    return guard([&] {
        if (!h->ready) throw Error(SETUP, "setup not done");
        if (stage < 0 || stage >= int(h->prec.stages.size()) || h->prec.stages[stage].kind != Stage::AMG)
            throw Error(INDEX, "not an AMG stage");  // -direct stages have no hierarchy
        // non-owning view: the oracle AMG object lives in the preconditioner
        *amg = reinterpret_cast<orc_amg*>(h->prec.stages[stage].amg.get());
    });
}

void orc_destroy(orc_system* h) { delete h; }

// read_matrix_market / read_layout / read_vector (matrix_io.cpp:40-121) +
// BlockMatrix::from_scalar (block_matrix.cpp:71-94) + ingest_external checks
// (harness.cpp:153-168); uniform layouts only (as the C ABI).
int orc_ingest(const char* mtx, const char* layout, const char* rhs, orc_system** out) {
    // C stdio, not iostreams: the oracle is loaded into Python processes whose
    // numpy may have brought another libstdc++ (iostream locale clash).
    return guard([&] {
        auto io = [](const std::string& m) { return Error(9, m); };
        struct F {
            FILE* f;
            explicit F(const char* p) : f(std::fopen(p, "r")) {}
            ~F() {
                if (f) std::fclose(f);
            }
        };
        F lf(layout);
        if (!lf.f) throw io(std::string("cannot open '") + layout + "' for reading");
        int nu = 0, nc = 0;
        if (std::fscanf(lf.f, "%d %d", &nu, &nc) != 2) throw io(std::string(layout) + ": bad layout header");
        std::vector<int> cell(nu);
        std::vector<char> tag(nu);
        for (int g = 0; g < nu; ++g) {
            char t[8];
            if (std::fscanf(lf.f, "%d %7s", &cell[g], t) != 2) throw io(std::string(layout) + ": truncated layout");
            tag[g] = t[0];
        }
        int nb = -1, g = 0;
        for (int c = 0; c < nc; ++c) {
            const int g0 = g;
            while (g < nu && cell[g] == c && tag[g] == 's') ++g;
            if (!(g < nu && cell[g] == c && tag[g] == 'P')) throw io("cell " + std::to_string(c) + " has no pressure unknown");
            ++g;
            if (!(g < nu && cell[g] == c && tag[g] == 'T'))
                throw io("cell " + std::to_string(c) + " has no temperature unknown");
            ++g;
            if (nb < 0) nb = g - g0;
            if (g - g0 != nb) throw Error(DIMENSION, "non-uniform layout");
        }
        if (g != nu || nc < 1) throw io(std::string(layout) + ": header cell count disagrees with tag list");
        const int n = nc * nb;
        F mf(mtx);
        if (!mf.f) throw io(std::string("cannot open '") + mtx + "' for reading");
        char line[4096];
        if (!std::fgets(line, sizeof line, mf.f)) throw io(std::string(mtx) + ": empty file");
        char w[5][64] = {};
        if (std::sscanf(line, "%63s %63s %63s %63s %63s", w[0], w[1], w[2], w[3], w[4]) != 5 ||
            std::strcmp(w[0], "%%MatrixMarket") || std::strcmp(w[1], "matrix") || std::strcmp(w[2], "coordinate") ||
            std::strcmp(w[3], "real") || std::strcmp(w[4], "general"))
            throw io(std::string(mtx) + ": expected 'matrix coordinate real general' header");
        do {
            if (!std::fgets(line, sizeof line, mf.f)) throw io(std::string(mtx) + ": bad size line");
        } while (line[0] == '%' || line[0] == '\n');
        int rows = 0, cols = 0, nnz = 0;
        if (std::sscanf(line, "%d %d %d", &rows, &cols, &nnz) != 3) throw io(std::string(mtx) + ": bad size line");
        if (rows != cols) throw io(std::string(mtx) + ": block matrix must be square");
        if (rows != n) throw Error(DIMENSION, "scalar matrix does not match layout dimension");
        std::vector<Triplet> t(nnz);
        for (int k = 0; k < nnz; ++k) {
            if (std::fscanf(mf.f, "%d %d %lf", &t[k].row, &t[k].col, &t[k].value) != 3)
                throw io(std::string(mtx) + ": truncated entry list");
            --t[k].row;
            --t[k].col;
        }
        const Csr a = Csr::from_triplets(n, n, std::move(t));
        std::map<std::pair<int, int>, Vec> blocks;
        for (int c = 0; c < nc; ++c) blocks[{c, c}] = Vec(size_t(nb) * nb, 0.0);
        for (int i = 0; i < n; ++i)
            for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                auto& blk = blocks[{i / nb, a.ci[k] / nb}];
                if (blk.empty()) blk.assign(size_t(nb) * nb, 0.0);
                blk[size_t(a.ci[k] % nb) * nb + i % nb] = a.v[k];
            }
        std::vector<int> rp(nc + 1, 0), ci;
        Vec vals;
        for (auto& kv : blocks) {
            ci.push_back(kv.first.second);
            vals.insert(vals.end(), kv.second.begin(), kv.second.end());
            rp[kv.first.first + 1]++;
        }
        for (int c = 0; c < nc; ++c) rp[c + 1] += rp[c];
        F rf(rhs);
        if (!rf.f) throw io(std::string("cannot open '") + rhs + "' for reading");
        Vec b;
        double x;
        while (std::fscanf(rf.f, "%lf", &x) == 1) b.push_back(x);
        if (int(b.size()) != n)
            throw io("rhs dimension " + std::to_string(b.size()) + " does not match matrix dimension " + std::to_string(n));
        auto* h = new orc_system;
        h->a = Bsr::create(nc, nb, rp.data(), ci.data(), vals.data());
        h->b_ingested = std::move(b);
        *out = h;
    });
}

int orc_condense(const mprec_global_jacobian* j, orc_condensed** out) {
    return guard([&] {
        if (!j || !out) throw Error(DIMENSION, "null argument");
        GlobalJacobian g;
        g.nc = j->n_cells;
        g.np = j->np;
        const int nc = g.nc, np = g.np;
        const int nnzb = j->row_ptr[nc];
        g.rp.assign(j->row_ptr, j->row_ptr + nc + 1);
        g.ci.assign(j->col_idx, j->col_idx + nnzb);
        g.j11.assign(j->j11, j->j11 + size_t(nnzb) * np * np);
        g.sec_off.assign(j->sec_off, j->sec_off + nc + 1);
        size_t o22 = 0;
        for (int c = 0; c < nc; ++c) {
            const int s0 = g.sec_off[c], ns = g.sec_off[c + 1] - s0;
            g.j22.emplace_back(j->j22 + o22, j->j22 + o22 + size_t(ns) * ns);
            o22 += size_t(ns) * ns;
            g.j21.emplace_back(j->j21 + size_t(s0) * np, j->j21 + size_t(s0 + ns) * np);
            g.r2.emplace_back(j->r2 + s0, j->r2 + s0 + ns);
        }
        size_t o12 = 0;
        for (int e = 0; e < j->n_j12; ++e) {
            const int c = j->j12_col[e];
            const size_t len = size_t(np) * (g.sec_off[c + 1] - g.sec_off[c]);
            g.e_row.push_back(j->j12_row[e]);
            g.e_col.push_back(c);
            g.e_blk.emplace_back(j->j12 + o12, j->j12 + o12 + len);
            o12 += len;
        }
        g.r1.assign(j->r1, j->r1 + size_t(nc) * np);
        auto h = std::make_unique<orc_condensed>();
        h->r = condense(g);
        *out = h.release();
    });
}

int orc_condensed_shape(orc_condensed* h, int* n_cells, int* np, int* nnzb, int* n_secondary) {
    return guard([&] {
        if (n_cells) *n_cells = h->r.nc;
        if (np) *np = h->r.np;
        if (nnzb) *nnzb = h->r.rp[h->r.nc];
        if (n_secondary) *n_secondary = h->r.sec_off[h->r.nc];
    });
}

int orc_condensed_get(orc_condensed* h, int* rp, int* ci, double* vals, double* b) {
    return guard([&] {
        if (rp) std::memcpy(rp, h->r.rp.data(), sizeof(int) * h->r.rp.size());
        if (ci) std::memcpy(ci, h->r.ci.data(), sizeof(int) * h->r.ci.size());
        if (vals) std::memcpy(vals, h->r.a.data(), sizeof(double) * h->r.a.size());
        if (b) std::memcpy(b, h->r.b.data(), sizeof(double) * h->r.b.size());
    });
}

int orc_condensed_system(orc_condensed* h, orc_system** out) {
    return guard([&] {
        const mprec_bsr a{h->r.nc, h->r.np, h->r.rp.data(), h->r.ci.data(), h->r.a.data()};
        auto s = std::make_unique<orc_system>();
        s->a = to_bsr(&a);
        s->b_ingested = h->r.b;
        *out = s.release();
    });
}

int orc_back_substitute(orc_condensed* h, const double* d1, double* d2) {
    return guard([&] {
        const Vec x(d1, d1 + size_t(h->r.nc) * h->r.np);
        const Vec y = back_substitute(h->r, x);
        if (!y.empty()) std::memcpy(d2, y.data(), sizeof(double) * y.size());
    });
}

void orc_condensed_destroy(orc_condensed* h) { delete h; }

int orc_get_shape(orc_system* h, int* n_cells, int* nb, int* nnzb) {
    return guard([&] {
        if (n_cells) *n_cells = h->a.nc;
        if (nb) *nb = h->a.nb;
        if (nnzb) *nnzb = h->a.rp[h->a.nc];
    });
}

int orc_get_matrix(orc_system* h, int* rp, int* ci, double* vals, double* b) {
    return guard([&] {
        if (rp) std::memcpy(rp, h->a.rp.data(), sizeof(int) * h->a.rp.size());
        if (ci) std::memcpy(ci, h->a.ci.data(), sizeof(int) * h->a.ci.size());
        if (vals) std::memcpy(vals, h->a.val.data(), sizeof(double) * h->a.val.size());
        if (b) {
            const Vec& src = h->b_ingested.empty() ? h->b : h->b_ingested;
            if (int64_t(src.size()) != int64_t(h->a.dim())) throw Error(DIMENSION, "the handle holds no rhs");
            std::memcpy(b, src.data(), sizeof(double) * src.size());
        }
    });
}

// ---- sub-solvers ----------------------------------------------------------

int orc_amg_create(const mprec_csr* a, const mprec_amg_params* p, orc_amg** out) {
    return guard([&] {
        auto* h = new AMGHierarchy(AMGHierarchy::setup(to_csr(a), to_params(p)));
        *out = reinterpret_cast<orc_amg*>(h);
    });
}

int orc_amg_apply(orc_amg* hh, const double* r, double* x) {
    return guard([&] {
        auto* h = reinterpret_cast<AMGHierarchy*>(hh);
        const int n = h->levels.front().a.rows;
        const Vec y = h->apply(Vec(r, r + n));
        std::memcpy(x, y.data(), y.size() * sizeof(double));
    });
}

int orc_amg_n_levels(orc_amg* hh, int* n) {
    return guard([&] { *n = reinterpret_cast<AMGHierarchy*>(hh)->n_levels(); });
}

int orc_amg_level_info(orc_amg* hh, int level, int* n, int* nnz_a, int* nnz_p) {
    return guard([&] {
        auto* h = reinterpret_cast<AMGHierarchy*>(hh);
        if (level < 0 || level >= h->n_levels()) throw Error(INDEX, "level out of range");
        const auto& L = h->levels[level];
        *n = L.a.rows;
        *nnz_a = L.a.nnz();
        *nnz_p = level == 0 ? 0 : L.p.nnz();
    });
}

int orc_amg_get_csr(orc_amg* hh, int level, int which, int* rp, int* ci, double* v) {
    return guard([&] {
        auto* h = reinterpret_cast<AMGHierarchy*>(hh);
        if (level < 0 || level >= h->n_levels()) throw Error(INDEX, "level out of range");
        const auto& L = h->levels[level];
        const Csr& m = which == 0 ? L.a : (which == 1 ? L.p : L.r);
        if (rp) std::memcpy(rp, m.rp.data(), m.rp.size() * sizeof(int));
        if (ci) std::memcpy(ci, m.ci.data(), m.ci.size() * sizeof(int));
        if (v) std::memcpy(v, m.v.data(), m.v.size() * sizeof(double));
    });
}

int orc_amg_get_cf(orc_amg* hh, int level, signed char* cf) {
    return guard([&] {
        auto* h = reinterpret_cast<AMGHierarchy*>(hh);
        if (level < 0 || level + 1 >= h->n_levels()) throw Error(INDEX, "level has no coarsening");
        const auto& m = h->levels[level].cf;
        for (size_t i = 0; i < m.size(); ++i) cf[i] = m[i];
    });
}

static void levels_out(const std::vector<int>& l, int* levels, int* n_levels) {
    int nl = 0;
    for (int v : l) nl = std::max(nl, v + 1);
    if (levels) std::memcpy(levels, l.data(), l.size() * sizeof(int));
    if (n_levels) *n_levels = nl;
}

int orc_amg_get_levelsets(orc_amg* hh, int level, int dir, int* levels, int* n_levels) {
    return guard([&] {
        auto* h = reinterpret_cast<AMGHierarchy*>(hh);
        if (level < 0 || level + 1 >= h->n_levels()) throw Error(INDEX, "level is not smoothed");
        if (dir != 1 && dir != -1) throw Error(INDEX, "dir must be +1 or -1");
        const Csr& a = h->levels[level].a;
        levels_out(dir > 0 ? level_sets_lower(a) : level_sets_upper(a), levels, n_levels);
    });
}

int orc_get_levelsets(orc_system* h, int dir, int* levels, int* n_levels) {
    return guard([&] {
        if (dir != 1 && dir != -1) throw Error(INDEX, "dir must be +1 or -1");
        Csr p;  // the block pattern as a cell-level CSR
        p.rows = p.cols = h->a.nc;
        p.rp = h->a.rp;
        p.ci = h->a.ci;
        p.v.assign(p.ci.size(), 1.0);
        levels_out(dir > 0 ? level_sets_lower(p) : level_sets_upper(p), levels, n_levels);
    });
}

void orc_amg_destroy(orc_amg* hh) { delete reinterpret_cast<AMGHierarchy*>(hh); }

int orc_ilu_create(const mprec_bsr* a, orc_ilu** out) {
    return guard([&] {
        auto* h = new orc_ilu;
        try {
            h->f = Ilu0Block::factor(to_bsr(a, SETUP));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int orc_ilu_apply(orc_ilu* h, const double* r, double* y) {
    return guard([&] {
        const Vec o = h->f.apply(Vec(r, r + h->f.lu.dim()));
        std::memcpy(y, o.data(), o.size() * sizeof(double));
    });
}

int orc_ilu_get(orc_ilu* h, double* lu) {
    return guard([&] { std::memcpy(lu, h->f.lu.val.data(), h->f.lu.val.size() * sizeof(double)); });
}

void orc_ilu_destroy(orc_ilu* h) { delete h; }

int orc_gmres(const mprec_bsr* a, const double* b, int prec_kind, void* prec, double tol, int max_iter,
              double* x, mprec_solve_result* out, double* history, int history_cap) {
    return guard([&] {
        const Bsr m = to_bsr(a);
        const int n = m.dim();
        const Op aop = [&m](const Vec& v) { return m.apply_flat(v); };
        Op mop;
        if (prec_kind == 0)
            mop = [](const Vec& v) { return v; };
        else if (prec_kind == 1)
            mop = [prec](const Vec& v) { return reinterpret_cast<AMGHierarchy*>(prec)->apply(v); };
        else if (prec_kind == 2)
            mop = [prec](const Vec& v) { return reinterpret_cast<orc_ilu*>(prec)->f.apply(v); };
        else
            throw Error(CONFIG, "unknown preconditioner kind");
        GmresOptions o;
        o.tol = tol;
        o.max_iter = max_iter;
        const double t0 = now_s();
        const SolveResult res = gmres(n, aop, Vec(b, b + n), mop, o);
        std::memset(out, 0, sizeof(*out));
        std::memcpy(x, res.x.data(), res.x.size() * sizeof(double));
        out->iterations = res.iterations;
        out->converged = res.converged;
        out->breakdown = res.breakdown;
        out->attempts = 1;
        out->total_iterations = res.iterations;
        out->final_true_residual = res.final_true_residual;
        out->setup_s = 0.0;
        out->solve_s = now_s() - t0;
        int nh = int(res.residual_history.size());
        if (history && history_cap < nh) nh = history_cap;
        if (history)
            for (int i = 0; i < nh; ++i) history[i] = res.residual_history[i];
        out->history_len = history ? nh : int(res.residual_history.size());
    });
}

// Reference-literal scalar route for validating the block restatement:
// flatten (block_matrix.cpp:116-128) + ILU0Factor on the scalar CSR.
int orc_ilu_scalar_factor(const mprec_bsr* a, double* lu_flat_values) {
    return guard([&] {
        const Bsr m = to_bsr(a);
        const Ilu0Scalar f = Ilu0Scalar::factor(m.to_scalar());
        std::memcpy(lu_flat_values, f.lu.v.data(), f.lu.v.size() * sizeof(double));
    });
}
int orc_ilu_scalar_apply(const mprec_bsr* a, const double* r, double* y) {
    return guard([&] {
        const Bsr m = to_bsr(a);
        const Ilu0Scalar f = Ilu0Scalar::factor(m.to_scalar());
        const Vec o = f.apply(Vec(r, r + m.dim()));
        std::memcpy(y, o.data(), o.size() * sizeof(double));
    });
}
int orc_spmv_scalar(const mprec_bsr* a, const double* x, double* y) {
    return guard([&] {
        const Bsr m = to_bsr(a);
        const Vec o = m.to_scalar().apply(Vec(x, x + m.dim()));
        std::memcpy(y, o.data(), o.size() * sizeof(double));
    });
}
int orc_level_sets(const mprec_csr* a, int* levels) {
    return guard([&] {
        const auto l = level_sets_lower(to_csr(a));
        std::memcpy(levels, l.data(), l.size() * sizeof(int));
    });
}

}  // extern "C"
