// capi.cu -- the C ABI of include/mprec_gpu.h: system handles, the staged
// right preconditioner (StagePreconditioner::apply, stages.cpp:36-59), the
// GMRES host loop over device vectors (gmres.cpp:8-106) and solve_system's
// tolerance-tightening retries (harness.cpp:190-219).
//
// Everything numeric runs in the sm_100a kernels of this library; the host
// only keeps the (max_iter+1) x max_iter Hessenberg matrix and the Givens
// rotations, exactly as the reference does, reading one Hessenberg column
// (k+2 doubles) back per iteration.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <functional>
#include <thread>

#include <cuda_profiler_api.h>

#include "condense.cuh"
#include "mprec.cuh"

using namespace mg;

namespace {
// Library load: ask for eager module loading unless the host chose otherwise.  With
// CUDA's default lazy loading every kernel is loaded at its first launch, and a
// load issued while another setup thread's multi-second kernel runs waits for it
// (+7 s on the first config-5 setup of a process).  Only effective when this
// runs before the CUDA context exists (a host linked against the library; a
// host that initialised CUDA first keeps its own setting).
struct EagerModules {
    EagerModules() { setenv("CUDA_MODULE_LOADING", "EAGER", 0); }
} g_eager_modules;

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
    } catch (const std::bad_alloc& e) {
        g_err = "host allocation failed";
        g_payload = -1;
        return MPREC_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_payload = -1;
        return MPREC_INTERNAL;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Validates a canonical BSR (block_matrix.cpp:32-69 invariants) and uploads the pattern.
void load_pattern(Ctx& c, Pattern& p, int nc, int nb, const int* rp, const int* ci,
                  int missing_diag_code = MPREC_DIMENSION) {
    if (nc < 1) throw Error(MPREC_DIMENSION, "layout needs at least one cell");
    if (nb < 1) throw Error(MPREC_DIMENSION, "block size must be >= 1");
    if (!rp || !ci) throw Error(MPREC_DIMENSION, "null pattern");
    if (rp[0] != 0) throw Error(MPREC_INDEX, "row_ptr[0] must be 0");
    p.nc = nc;
    p.nnzb = rp[nc];
    p.h_rp.assign(rp, rp + nc + 1);
    p.h_ci.assign(ci, ci + p.nnzb);
    p.h_dpos.assign(nc, -1);
    for (int r = 0; r < nc; ++r) {
        if (rp[r + 1] < rp[r]) throw Error(MPREC_INDEX, "row_ptr not monotone");
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= nc) throw Error(MPREC_INDEX, "block column out of range");
            if (k > rp[r] && ci[k] <= ci[k - 1]) throw Error(MPREC_INDEX, "block columns not sorted");
            if (ci[k] == r) p.h_dpos[r] = k;
        }
        if (p.h_dpos[r] < 0) {
            if (missing_diag_code == MPREC_SETUP) throw Error(MPREC_SETUP, "ILU(0): structurally absent diagonal");
            throw Error(MPREC_DIMENSION, "diagonal block missing in cell " + std::to_string(r), r);
        }
    }
    p.rp.upload(p.h_rp.data(), p.h_rp.size(), c.s);
    p.ci.upload(p.h_ci.data(), std::max<size_t>(p.h_ci.size(), 1), c.s);
    p.dpos.upload(p.h_dpos.data(), p.h_dpos.size(), c.s);
}

BsrView view_of(const Pattern& p, int nb, double* val) {
    BsrView v;
    v.nc = p.nc;
    v.nb = nb;
    v.nnzb = p.nnzb;
    v.rp = p.rp.p;
    v.ci = p.ci.p;
    v.dpos = p.dpos.p;
    v.val = val;
    return v;
}

using DevOp = std::function<void(const double* x, double* y)>;

struct GmresOut {
    int iterations = 0;
    bool converged = false, breakdown = false;
    std::vector<double> history;
    double final_true_residual = 0.0;
};

// Krylov basis allocated lazily in chunks of kBasisChunk vectors (at
// c5 one vector is 256 MB), stored tile-major for the Gram passes (gram.cu).
struct Basis {
    int64_t n = 0;
    std::vector<DBuf<double>> blocks;
    double* chunk(int c) {
        while (int(blocks.size()) <= c) blocks.emplace_back(size_t(basis_chunk_doubles(n)));
        return blocks[c].p;
    }
};

struct Krylov {
    Basis V;
    DBuf<double> w, t, vk, hcol;
    DBuf<double> ydev;
    DBuf<double*> ct;             // chunk pointer table
    DBuf<double> gt, pbuf, part;  // transposed Gram lower part, coefficients, pass-A partials
};

// MPREC_GRAM_FUSED=0: the unfused two-sweep orthogonalisation (A/B experiments)
static bool gram_fused() {
    static const bool on = [] {
        const char* e = getenv("MPREC_GRAM_FUSED");
        return !(e && e[0] == '0');
    }();
    return on;
}

// gmres.cpp:8-106 over device vectors.  b, x: device; n unknowns.
GmresOut gmres_dev(Ctx& c, Krylov& kr, int64_t n, const DevOp& A, const DevOp& M, const double* b, double tol,
                   int max_iter, double* x) {
    if (tol <= 0.0) throw Error(MPREC_DIMENSION, "gmres: tolerance must be positive");
    GmresOut out;
    double* sc = c.scal.p;  // [0] bnorm [1] pre_norm [2] wn [3] norm after reorth
    // work vectors first: the caller's true-residual check uses kr.t even when
    // b = 0 returns early (gmres.cpp:17-21)
    kr.w.ensure(n);
    kr.t.ensure(n);
    nrm2(c, b, n, sc + 0);
    double bnorm = 0.0;
    MG_CUDA(cudaMemcpyAsync(&bnorm, sc + 0, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (bnorm == 0.0) {
        fill(c, x, 0.0, n);
        out.converged = true;
        out.history.push_back(0.0);
        return out;
    }
    const int max_it = int(std::min<int64_t>(max_iter, n));
    kr.V.n = n;
    kr.hcol.ensure(max_it + 2);
    kr.vk.ensure(n);
    kr.ct.ensure(max_it / kBasisChunk + 2);
    kr.gt.ensure(size_t(max_it + 1) * (max_it + 1));
    kr.pbuf.ensure(max_it + 2);
    kr.part.ensure(size_t(gram_part_size(c, max_it)));
    int* gate = c.err.p + 8;
    gram_set_ptr(c, kr.ct.p, 0, kr.V.chunk(0));
    basis_put(c, kr.V.chunk(0), 0, b, bnorm, n);
    const double* const* ct = kr.ct.p;
    const int ld = max_it + 1;
    std::vector<double> h(size_t(ld) * std::max(max_it, 1), 0.0), cs(max_it), sn(max_it), g(max_it + 1, 0.0);
    auto H = [&](int i, int j) -> double& { return h[size_t(j) * ld + i]; };
    g[0] = bnorm;
    out.history.push_back(1.0);
    std::vector<double> col(max_it + 4);
    int k = 0;
    for (; k < max_it; ++k) {
        double* vk = kr.vk.p;
        basis_get(c, vk, kr.V.chunk(k / kBasisChunk), k % kBasisChunk, n);
        M(vk, kr.t.p);
        A(kr.t.p, kr.w.p);
        double* w = kr.w.p;
        double* hc = kr.hcol.p;
        // MGS (gmres.cpp:39-42) in Gram form (gram.cu): V^T w and the basis' new
        // Gram row in one pass, (I + L) h = V^T w, w -= V h in a second pass
        // one re-orthogonalisation pass when ||w|| < 0.7 pre_norm (gmres.cpp:44-50), gated on
        // device; its pass A is fused into the first sweep's pass B (gram_orthogonalise)
        // the fused pass holds <= 512 basis vectors per row in registers; below 24
        // vectors its per-sub-tile synchronisation and 32-wide butterfly cost more
        // than the separate pass A' (ncu: 0.95 ms vs 0.26 ms at k = 1)
        if (gram_fused() && k + 1 <= 512 && k >= 24) {
            gram_orthogonalise(c, ct, k, w, n, kr.gt.p, ld, kr.pbuf.p, hc, sc + 1, sc + 2, sc + 3, kr.part.p, gate);
        } else {
            gram_sweep(c, ct, k, w, n, kr.gt.p, ld, kr.pbuf.p, hc, false, k > 0, sc + 1, sc + 2, kr.part.p, nullptr);
            set_reorth_gate(c, sc + 2, sc + 1, gate);
            gram_sweep(c, ct, k, w, n, kr.gt.p, ld, kr.pbuf.p, hc, true, false, nullptr, sc + 3, kr.part.p, gate);
        }
        // read back the Hessenberg column
        MG_CUDA(cudaMemcpyAsync(col.data(), hc, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, c.s));
        double tail[3];
        int gh = 0;
        MG_CUDA(cudaMemcpyAsync(tail, sc + 1, sizeof(double) * 3, cudaMemcpyDeviceToHost, c.s));
        MG_CUDA(cudaMemcpyAsync(&gh, gate, sizeof(int), cudaMemcpyDeviceToHost, c.s));
        MG_CUDA(cudaStreamSynchronize(c.s));
        c.resolve_gate(gh != 0);  // charge the re-orthogonalisation's bytes only when it ran
        if (!c.pending.empty() && c.pending.size() > 2048) c.harvest();
        for (int i = 0; i <= k; ++i) H(i, k) = col[i];
        H(k + 1, k) = gh ? tail[2] : tail[1];
        const double subdiag = H(k + 1, k);
        for (int i = 0; i < k; ++i) {
            const double tt = cs[i] * H(i, k) + sn[i] * H(i + 1, k);
            H(i + 1, k) = -sn[i] * H(i, k) + cs[i] * H(i + 1, k);
            H(i, k) = tt;
        }
        const double denom = std::hypot(H(k, k), H(k + 1, k));
        if (denom == 0.0) {
            out.breakdown = true;
            ++k;
            break;
        }
        cs[k] = H(k, k) / denom;
        sn[k] = H(k + 1, k) / denom;
        H(k, k) = denom;
        H(k + 1, k) = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
        const double rel = std::abs(g[k + 1]) / bnorm;
        out.history.push_back(rel);
        if (rel <= tol) {
            ++k;
            break;
        }
        if (subdiag == 0.0) {
            out.breakdown = true;
            ++k;
            break;
        }
        if ((k + 1) % kBasisChunk == 0)
            gram_set_ptr(c, kr.ct.p, (k + 1) / kBasisChunk, kr.V.chunk((k + 1) / kBasisChunk));
        basis_put(c, kr.V.chunk((k + 1) / kBasisChunk), (k + 1) % kBasisChunk, w, subdiag, n);
    }
    out.iterations = k;
    if (k > 0) {
        std::vector<double> y(k, 0.0);
        for (int i = k - 1; i >= 0; --i) {
            double acc = g[i];
            for (int j = i + 1; j < k; ++j) acc -= H(i, j) * y[j];
            y[i] = acc / H(i, i);
        }
        kr.ydev.ensure(k);
        kr.ydev.upload(y.data(), k, c.s);
        basis_combine(c, ct, k, kr.ydev.p, kr.w.p, n);
        M(kr.w.p, x);
        c.sync();  // the host vectors above must outlive the async uploads
    } else {
        fill(c, x, 0.0, n);
    }
    A(x, kr.t.p);
    sub(c, kr.t.p, b, kr.t.p, n);
    nrm2(c, kr.t.p, n, sc + 0);
    double rn = 0.0;
    MG_CUDA(cudaMemcpyAsync(&rn, sc + 0, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    out.final_true_residual = rn / bnorm;
    out.converged = out.history.back() <= tol || out.final_true_residual <= tol;
    return out;
}

void fill_result(mprec_solve_result* r, const GmresOut& g, int attempts, double setup_s, double solve_s,
                 double* history, int cap, int total_iterations = -1) {
    if (!r) return;
    for (int q = 0; q < 3; ++q) {
        r->attempt_iterations[q] = q == 0 ? g.iterations : 0;
        r->attempt_converged[q] = q == 0 ? g.converged : 0;
        r->attempt_tol[q] = 0.0;
        r->attempt_true_residual[q] = q == 0 ? g.final_true_residual : 0.0;
    }
    r->total_iterations = total_iterations < 0 ? g.iterations : total_iterations;
    r->iterations = g.iterations;
    r->converged = g.converged;
    r->breakdown = g.breakdown;
    r->attempts = attempts;
    r->final_true_residual = g.final_true_residual;
    r->setup_s = setup_s;
    r->solve_s = solve_s;
    int nh = int(g.history.size());
    if (history && cap < nh) nh = cap;
    if (history)
        for (int i = 0; i < nh; ++i) history[i] = g.history[i];
    r->history_len = history ? nh : int(g.history.size());
}

}  // namespace

static bool is_cptr3_method(int m) { return m == MPREC_METHOD_CPTR3_AMG || m == MPREC_METHOD_CPTR3_DIRECT; }

// ScaledSystem::scaling_record (scaling.cpp:84, 102, 116, 144) joined as in
// solve_system (harness.cpp:197-201)
static std::string scaling_record_of(int m) {
    switch (m) {
        case MPREC_METHOD_CPR_AMG:
        case MPREC_METHOD_CPR_DIRECT: return "D_Ph*D_hh^-1";
        case MPREC_METHOD_CPTR_DIRECT: return "D_es*D_ss^-1";
        case MPREC_METHOD_CPTR3_AMG:
        case MPREC_METHOD_CPTR3_DIRECT: return "[D_Ps;D_Ts]*D_ss^-1, D_Tp*D_PP^-1";
        default: return "";
    }
}

namespace mg {
void ingest(Ctx& c, const char* mtx, const char* layout, const char* rhs, Pattern& pat, DBuf<double>& val, int* n_cells,
            int* nb_out, std::vector<double>& b);
void write_system(const char* mtx, const char* layout, const char* rhs, int nc, int nb, const std::vector<int>& rp,
                  const std::vector<int>& ci, const std::vector<double>& val, const double* b);
void ilu_timeline(Ctx& c, Ilu& ilu, const double* r, double* y, long long* ts_dev, int blocks);
void gs_bench(Ctx& c, Amg& amg, int l, int reps, double* ms_f, double* ms_b, int* nl_f, int* nl_b);
void gs_ls_experiment(Ctx& c, Amg& amg, int l, int K, int reps, double* out);
}

// ============================================================ AMG handle ==
struct mprec_gpu_amg {
    Ctx* ctx = nullptr;
    std::unique_ptr<Ctx> own_ctx;
    Amg* amg = nullptr;
    std::unique_ptr<Amg> own_amg;
    DCsr a0;
    DBuf<double> r, x;
};

// ============================================================ ILU handle ==
struct mprec_gpu_ilu {
    Ctx ctx;
    Pattern pat;
    Ilu ilu;
    DBuf<double> vals, r, y;
};

// ====================================================== condensed handle ==
struct mprec_gpu_condensed {
    Ctx ctx;
    Condensed cd;
};

// ========================================================= system handle ==
struct mprec_gpu_system {
    Ctx ctx;
    Pattern pat;
    int nb = 0;
    int64_t n = 0;
    DBuf<double> a_val, abar_val, lu_val, b, bbar, fP, fT;
    std::unique_ptr<Amg> amgT, amgP, amgE;  // amgE: CPTR's dense B_ee solve
    DCsr b_ee;
    DBuf<double> gE, xE;
    Ilu ilu;
    int method = -1;
    bool ready = false;
    double setup_s = 0.0;
    // work vectors of the stage preconditioner
    DBuf<double> gT, xT, gP, vP, z, u, w, x, r, y;
    Krylov kr;
    std::vector<std::unique_ptr<mprec_gpu_amg>> views;
    std::vector<double> b_host;  // rhs kept by mprec_gpu_ingest / the last setup
    std::string scaling_record;

    BsrView A() { return view_of(pat, nb, a_val.p); }
    BsrView Abar() { return view_of(pat, nb, abar_val.p); }
    int P() const { return nb - 2; }
    int T() const { return nb - 1; }

    static bool is_cpr(int m) { return m == MPREC_METHOD_CPR_AMG || m == MPREC_METHOD_CPR_DIRECT; }
    static bool is_cptr3(int m) { return m == MPREC_METHOD_CPTR3_AMG || m == MPREC_METHOD_CPTR3_DIRECT; }
    int n_stages() const { return method == MPREC_METHOD_ILU0 ? 1 : (is_cptr3(method) ? 3 : 2); }

    // StagePreconditioner::apply (stages.cpp:36-59), device pointers
    void prec_apply(const double* rin, double* yout) {
        Ctx& c = ctx;
        const int nc = pat.nc;
        if (method == MPREC_METHOD_ILU0) {
            ilu.apply(c, rin, yout);
        } else if (method == MPREC_METHOD_CPTR_DIRECT) {
            // x = M1 r (B_ee scope); z = r - A x; y = x + M2 z
            gather_pt(c, gE.p, rin, nc, nb);
            amgE->apply(c, gE.p, xE.p);
            scatter_pt(c, x.p, xE.p, nc, nb);
            bsr_spmv(c, Abar(), x.p, z.p, rin, MPREC_K_SPMV);
            ilu.apply(c, z.p, w.p);
            add2(c, yout, x.p, w.p, n);  // y = x + M2 z (stages.cpp:48)
        } else if (is_cpr(method)) {
            gather_stride(c, gP.p, rin, nc, nb, P());
            amgP->apply(c, gP.p, vP.p);
            bsr_col_update(c, Abar(), P(), vP.p, rin, z.p, nullptr, 0);
            ilu.apply(c, z.p, w.p);
            stage_combine(c, yout, w.p, nullptr, 0, vP.p, P(), nc, nb);
        } else {
            gather_stride(c, gT.p, rin, nc, nb, T());
            amgT->apply(c, gT.p, xT.p);
            bsr_col_update(c, Abar(), T(), xT.p, rin, z.p, gP.p, P());
            amgP->apply(c, gP.p, vP.p);
            bsr_col_update(c, Abar(), P(), vP.p, z.p, u.p, nullptr, 0);
            ilu.apply(c, u.p, w.p);
            stage_combine(c, yout, w.p, xT.p, T(), vP.p, P(), nc, nb);
        }
    }

    // Stage::apply (stages.cpp:25-34) for stage i, full vectors
    void stage_apply(int i, const double* rin, double* yout) {
        Ctx& c = ctx;
        const int nc = pat.nc;
        const int nst = n_stages();
        if (i < 0 || i >= nst) throw Error(MPREC_INDEX, "stage out of range");
        if (i == nst - 1) {
            ilu.apply(c, rin, yout);
            return;
        }
        if (method == MPREC_METHOD_CPTR_DIRECT) {
            gather_pt(c, gE.p, rin, nc, nb);
            amgE->apply(c, gE.p, xE.p);
            scatter_pt(c, yout, xE.p, nc, nb);
            return;
        }
        Amg* a = nullptr;
        int f = 0;
        if (is_cpr(method)) {
            a = amgP.get();
            f = P();
        } else if (i == 0) {
            a = amgT.get();
            f = T();
        } else {
            a = amgP.get();
            f = P();
        }
        gather_stride(c, gT.p, rin, nc, nb, f);
        a->apply(c, gT.p, xT.p);
        fill(c, w.p, 0.0, n);
        stage_combine(c, yout, w.p, xT.p, f, nullptr, 0, nc, nb);
    }

    int total_iterations = 0;
    int att_it[3] = {0, 0, 0}, att_cv[3] = {0, 0, 0};
    double att_tol[3] = {0, 0, 0}, att_res[3] = {0, 0, 0};
    void log_attempts(mprec_solve_result* r) const {
        if (!r) return;
        for (int q = 0; q < 3; ++q) {
            r->attempt_iterations[q] = att_it[q];
            r->attempt_converged[q] = att_cv[q];
            r->attempt_tol[q] = att_tol[q];
            r->attempt_true_residual[q] = att_res[q];
        }
    }
    GmresOut solve_attempts(double tol, int max_iter, double* xdev, int* attempts) {
        Ctx& c = ctx;
        // MPREC_PROFILE_SOLVE=1: bracket the solve for `ncu --profile-from-start off`
        static const bool prof = [] {
            const char* e = getenv("MPREC_PROFILE_SOLVE");
            return e && e[0] == '1';
        }();
        struct ProfRange {
            bool on;
            explicit ProfRange(bool o) : on(o) {
                if (on) cudaProfilerStart();
            }
            ~ProfRange() {
                if (on) cudaProfilerStop();
            }
        } pr(prof);
        const DevOp Aop = [this](const double* xx, double* yy) { bsr_spmv(ctx, Abar(), xx, yy, nullptr, MPREC_K_SPMV); };
        const DevOp Mop = [this](const double* xx, double* yy) { prec_apply(xx, yy); };
        double bn = 0.0;
        nrm2(c, b.p, n, c.scal.p + 8);
        MG_CUDA(cudaMemcpyAsync(&bn, c.scal.p + 8, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        double opt_tol = tol;
        GmresOut res;
        *attempts = 0;
        total_iterations = 0;
        for (int q = 0; q < 3; ++q) {
            att_it[q] = att_cv[q] = 0;
            att_tol[q] = att_res[q] = 0.0;
        }
        for (int attempt = 0; attempt < 3; ++attempt) {
            ++*attempts;
            att_tol[attempt] = opt_tol;
            res = gmres_dev(c, kr, n, Aop, Mop, bbar.p, opt_tol, max_iter, xdev);
            total_iterations += res.iterations;
            att_it[attempt] = res.iterations;
            att_cv[attempt] = res.converged;
            // residual_check on the ORIGINAL system (gmres.cpp:108-112)
            bsr_spmv(c, A(), xdev, kr.t.p, bn == 0.0 ? nullptr : b.p, MPREC_K_SPMV);
            nrm2(c, kr.t.p, n, c.scal.p + 9);
            double rn = 0.0;
            MG_CUDA(cudaMemcpyAsync(&rn, c.scal.p + 9, sizeof(double), cudaMemcpyDeviceToHost, c.s));
            c.sync();
            res.final_true_residual = bn == 0.0 ? rn : rn / bn;
            att_res[attempt] = res.final_true_residual;
            if (!res.converged || res.final_true_residual <= tol) break;
            opt_tol *= 0.5 * tol / res.final_true_residual;
        }
        if (res.converged && res.final_true_residual > tol) res.converged = false;
        last_history = res.history;
        return res;
    }
    std::vector<double> last_history;  // residual history of the last solve's last attempt
};

extern "C" {

const char* mprec_gpu_last_error(void) { return g_err.c_str(); }
int mprec_gpu_error_payload(void) { return g_payload; }

int mprec_gpu_device_info(int* sm, int* major, int* minor, int64_t* mem) {
    return guard([&] {
        int dev = 0, cnt = 0;
        MG_CUDA(cudaGetDeviceCount(&cnt));
        if (cnt < 1) throw Error(MPREC_CUDA, "no CUDA device");
        MG_CUDA(cudaGetDevice(&dev));
        cudaDeviceProp p;
        MG_CUDA(cudaGetDeviceProperties(&p, dev));
        if (sm) *sm = p.multiProcessorCount;
        if (major) *major = p.major;
        if (minor) *minor = p.minor;
        if (mem) *mem = int64_t(p.totalGlobalMem);
    });
}

int mprec_gpu_create(const mprec_bsr* a, mprec_gpu_system** out) {
    return guard([&] {
        if (!a || !out) throw Error(MPREC_DIMENSION, "null argument");
        auto h = std::make_unique<mprec_gpu_system>();
        load_pattern(h->ctx, h->pat, a->n_cells, a->nb, a->row_ptr, a->col_idx);
        h->nb = a->nb;
        h->n = int64_t(a->n_cells) * a->nb;
        h->a_val.upload(a->values, std::max<size_t>(size_t(h->pat.nnzb) * a->nb * a->nb, 1), h->ctx.s);
        h->ctx.sync();
        *out = h.release();
    });
}

int mprec_gpu_setup(mprec_gpu_system* h, int method, const mprec_amg_params* amg, const double* b) {
    return mprec_gpu_setup_opts(h, method, amg, nullptr, b);
}

int mprec_gpu_setup_opts(mprec_gpu_system* h, int method, const mprec_amg_params* amg,
                         const mprec_scaling_options* opts, const double* b) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (method < MPREC_METHOD_ILU0 || method > MPREC_METHOD_CPTR3_DIRECT)
            throw Error(MPREC_CONFIG, "unknown method id " + std::to_string(method));
        if (method != MPREC_METHOD_ILU0 && h->nb < 2)
            throw Error(MPREC_DIMENSION, "CPR/CPTR3 need P and T unknowns (nb >= 2)");
        Ctx& c = h->ctx;
        h->ready = false;
        const double t0 = now_s();
        const int64_t n = h->n;
        const size_t nv = size_t(h->pat.nnzb) * h->nb * h->nb;
        if (!b) {
            if (int64_t(h->b_host.size()) != n) throw Error(MPREC_DIMENSION, "no rhs: pass b or ingest one");
            b = h->b_host.data();
        } else {
            h->b_host.assign(b, b + n);
        }
        auto tr_pre = std::make_unique<Trace>(&c, "setup: rhs upload, operator copy");
        h->b.upload(b, n, c.s);
        h->bbar.ensure(n);
        copy(c, h->bbar.p, h->b.p, n);
        h->abar_val.ensure(nv);
        MG_CUDA(cudaMemcpyAsync(h->abar_val.p, h->a_val.p, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.s));
        tr_pre.reset();
        // left_scale (scaling.cpp:149-158)
        {
            Trace tr(&c, "left_scale");
            const int scalar_diag = opts && opts->diag_mode == MPREC_DIAG_SCALAR;
            if (opts && opts->diag_mode != MPREC_DIAG_BLOCK && opts->diag_mode != MPREC_DIAG_SCALAR)
                throw Error(MPREC_CONFIG, "unknown diag mode " + std::to_string(opts->diag_mode));
            const bool from_orig = opts && opts->second_scaling_from_original;
            left_scale(c, h->Abar(), h->bbar.p, method, scalar_diag, from_orig ? h->a_val.p : nullptr);
            h->scaling_record = scaling_record_of(method);
        }
        // build_preconditioner (stages.cpp:129-138)
        AmgParams prm;
        if (amg) {
            prm.theta = amg->strength_threshold;
            prm.max_coarse = amg->max_coarse_size;
            prm.max_levels = amg->max_levels;
        }
        const int nc = h->pat.nc;
        // views handed out by mprec_gpu_stage_amg go stale (not freed: a caller may
        // still hold them; every AMG entry point rejects a stale view)
        for (auto& v : h->views) v->amg = nullptr;
        h->amgT.reset();
        h->amgP.reset();
        h->amgE.reset();
        // -direct: the stage sub-system is factored densely (a single-level hierarchy
        // whose coarsest solve is the whole sub-system, DenseFactor in make_scoped)
        const bool direct = method == MPREC_METHOD_CPR_DIRECT || method == MPREC_METHOD_CPTR_DIRECT ||
                            method == MPREC_METHOD_CPTR3_DIRECT;
        if (direct) {
            prm.max_coarse = 0x7fffffff;
            prm.max_levels = 1;
        }
        if (method == MPREC_METHOD_CPTR_DIRECT) {
            DCsr& e = h->b_ee;
            e.n = e.m = 2 * nc;
            e.nnz = 4 * h->pat.nnzb;
            e.rp.alloc(2 * nc + 1);
            e.ci.alloc(e.nnz);
            e.v.alloc(e.nnz);
            extract_pt(c, h->Abar(), e.rp.p, e.ci.p, e.v.p);
            h->amgE = std::make_unique<Amg>();
            CsrView ev = e.view();
            ev.diag = nullptr;
            h->amgE->setup(c, ev, prm);
            h->gE.ensure(2 * nc);
            h->xE.ensure(2 * nc);
        }
        // The two stage hierarchies are independent (stages.cpp:129-138) and their
        // setup is dominated by the sequential, single-warp RS first pass: build
        // C_TT's on a second stream from a worker thread while B_PP's runs here.
        const bool want_T = is_cptr3_method(method);
        const bool want_P = method == MPREC_METHOD_CPR_AMG || method == MPREC_METHOD_CPR_DIRECT || want_T;
        CsrView aT{}, aP{};
        if (want_T) {
            h->fT.ensure(h->pat.nnzb);
            extract_field(c, h->Abar(), h->T(), h->fT.p);
            aT = CsrView{nc, nc, h->pat.nnzb, h->pat.rp.p, h->pat.ci.p, h->fT.p, h->pat.dpos.p};
            h->amgT = std::make_unique<Amg>();
        }
        if (want_P) {
            h->fP.ensure(h->pat.nnzb);
            extract_field(c, h->Abar(), h->P(), h->fP.p);
            aP = CsrView{nc, nc, h->pat.nnzb, h->pat.rp.p, h->pat.ci.p, h->fP.p, h->pat.dpos.p};
            h->amgP = std::make_unique<Amg>();
        }
        // ILU(0) of Ā (factors, packed diagonal inverses, solve streams): independent
        // of the hierarchies, so with two of them it runs on a third thread / stream
        // meanwhile (its buffers are allocated here, before any concurrency)
        bool ilu_done = false;
        auto do_ilu = [&](Ctx& cx) {
            MG_CUDA(cudaMemcpyAsync(h->lu_val.p, h->abar_val.p, nv * sizeof(double), cudaMemcpyDeviceToDevice, cx.s));
            h->ilu.lu = view_of(h->pat, h->nb, h->lu_val.p);
            h->ilu.pat = &h->pat;
            Trace tr(&cx, "ILU(0) factor");
            h->ilu.factor(cx);
            ilu_done = true;
        };
        h->lu_val.ensure(nv);
        if (h->nb == 8) h->ilu.dinv.ensure((size_t)nc * 64);
        if (want_T && want_P) {
            {
                Trace tr(&c, "setup: block-pattern sweep schedules");
                h->pat.ensure_sched(c);  // shared, read-only from here on
                c.sync();
            }
            // keep freed blocks in the stream-ordered pool while the two hierarchies are
            // built: with the default release threshold (0) every stream
            // synchronisation returns them to the driver and the next
            // cudaMallocAsync maps fresh memory, which waits for the other
            // thread's multi-second first-pass kernel; trimmed again afterwards
            struct PoolKeep {
                cudaMemPool_t pool = nullptr;
                PoolKeep() {
                    int dev = 0;
                    cudaGetDevice(&dev);
                    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) pool = nullptr;
                    unsigned long long thr = ~0ull;
                    if (pool) cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                }
                ~PoolKeep() {
                    unsigned long long thr = 0;
                    const double tt = now_s();
                    struct Rep {
                        double t;
                        ~Rep() {
                            if (trace_on()) fprintf(stderr, "[mprec] setup: pool trim %34.3f ms\n", (now_s() - t) * 1e3);
                        }
                    } rep{tt};
                    if (pool) {
                        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                        cudaMemPoolTrimTo(pool, 0);
                    }
                }
            } pool_keep;
            Ctx c2;
            std::exception_ptr err_T;
            std::thread th([&] {
                try {
                    StreamAllocScope alloc_on(c2.s);  // no device-wide syncs from allocations
                    Trace tr(&c2, "AMG(C_TT) setup total");
                    h->amgT->setup(c2, aT, prm, &h->pat);
                    c2.sync();
                } catch (...) {
                    err_T = std::current_exception();
                }
            });
            Ctx c3;
            std::exception_ptr err_I;
            std::thread thi([&] {
                try {
                    StreamAllocScope alloc_on(c3.s);
                    do_ilu(c3);
                    c3.sync();
                } catch (...) {
                    err_I = std::current_exception();
                }
            });
            std::exception_ptr err_P;
            try {
                StreamAllocScope alloc_on(c.s);
                Trace tr(&c, "AMG(B_PP) setup total");
                h->amgP->setup(c, aP, prm, &h->pat);
                c.sync();
            } catch (...) {
                err_P = std::current_exception();
            }
            th.join();
            thi.join();
            // the reference builds C_TT first (stages.cpp:129-138): its error wins
            if (err_T) std::rethrow_exception(err_T);
            if (err_P) std::rethrow_exception(err_P);
            if (err_I) std::rethrow_exception(err_I);  // (build_cptr3 factors after the hierarchies)
        } else if (want_T) {
            Trace tr(&c, "AMG(C_TT) setup total");
            h->amgT->setup(c, aT, prm, &h->pat);
        } else if (want_P) {
            Trace tr(&c, "AMG(B_PP) setup total");
            h->amgP->setup(c, aP, prm, &h->pat);
        }
        if (!ilu_done) do_ilu(c);
        if (trace_on()) fprintf(stderr, "[mprec] setup: %.3f s after the hierarchies and ILU\n", now_s() - t0);
        for (DBuf<double>* v : {&h->gT, &h->xT, &h->gP, &h->vP}) v->ensure(nc);
        for (DBuf<double>* v : {&h->z, &h->u, &h->w, &h->x, &h->r, &h->y}) v->ensure(n);
        c.sync();
        h->method = method;
        h->ready = true;
        h->setup_s = now_s() - t0;
        if (trace_on()) fprintf(stderr, "[mprec] setup: %.3f s total\n", h->setup_s);
    });
}

int mprec_gpu_ingest(const char* mtx, const char* layout, const char* rhs, mprec_gpu_system** out) {
    return guard([&] {
        if (!mtx || !layout || !rhs || !out) throw Error(MPREC_DIMENSION, "null argument");
        auto h = std::make_unique<mprec_gpu_system>();
        int nc = 0, nb = 0;
        ingest(h->ctx, mtx, layout, rhs, h->pat, h->a_val, &nc, &nb, h->b_host);
        h->nb = nb;
        h->n = int64_t(nc) * nb;
        *out = h.release();
    });
}

int mprec_gpu_condense(const mprec_global_jacobian* j, mprec_gpu_condensed** out) {
    return guard([&] {
        if (!j || !out) throw Error(MPREC_DIMENSION, "null argument");
        auto h = std::make_unique<mprec_gpu_condensed>();
        condense(h->ctx, *j, h->cd);
        *out = h.release();
    });
}

int mprec_gpu_condensed_shape(mprec_gpu_condensed* h, int* n_cells, int* np, int* nnzb, int* n_secondary) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (n_cells) *n_cells = h->cd.nc;
        if (np) *np = h->cd.np;
        if (nnzb) *nnzb = h->cd.pat.nnzb;
        if (n_secondary) *n_secondary = h->cd.n2;
    });
}

int mprec_gpu_condensed_get(mprec_gpu_condensed* h, int* rp, int* ci, double* vals, double* b) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        const Condensed& d = h->cd;
        if (rp) std::memcpy(rp, d.pat.h_rp.data(), sizeof(int) * d.pat.h_rp.size());
        if (ci) std::memcpy(ci, d.pat.h_ci.data(), sizeof(int) * d.pat.h_ci.size());
        if (vals) d.a_val.download(vals, size_t(d.pat.nnzb) * d.np * d.np, h->ctx.s);
        if (b) d.b.download(b, size_t(d.nc) * d.np, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_condensed_system(mprec_gpu_condensed* h, mprec_gpu_system** out) {
    return guard([&] {
        if (!h || !out) throw Error(MPREC_DIMENSION, "null argument");
        const Condensed& d = h->cd;
        if (d.np < 2) throw Error(MPREC_DIMENSION, "the reduced system needs P and T per cell");
        auto s = std::make_unique<mprec_gpu_system>();
        Pattern& p = s->pat;
        p.nc = d.pat.nc;
        p.nnzb = d.pat.nnzb;
        p.h_rp = d.pat.h_rp;
        p.h_ci = d.pat.h_ci;
        p.h_dpos = d.pat.h_dpos;
        p.rp.upload(p.h_rp.data(), p.h_rp.size(), s->ctx.s);
        p.ci.upload(p.h_ci.data(), p.h_ci.size(), s->ctx.s);
        p.dpos.upload(p.h_dpos.data(), p.h_dpos.size(), s->ctx.s);
        const size_t nv = size_t(d.pat.nnzb) * d.np * d.np;
        s->a_val.alloc(nv);
        h->ctx.sync();
        MG_CUDA(cudaMemcpyAsync(s->a_val.p, d.a_val.p, nv * sizeof(double), cudaMemcpyDeviceToDevice, s->ctx.s));
        s->nb = d.np;
        s->n = int64_t(d.nc) * d.np;
        s->b_host = d.b.to_host(h->ctx.s, size_t(s->n));
        s->ctx.sync();
        *out = s.release();
    });
}

int mprec_gpu_back_substitute(mprec_gpu_condensed* h, const double* d1, double* d2) {
    return guard([&] {
        if (!h || !d1 || (!d2 && h->cd.n2 > 0)) throw Error(MPREC_DIMENSION, "null argument");
        const Condensed& d = h->cd;
        DBuf<double> x1(size_t(d.nc) * d.np), x2(size_t(std::max(d.n2, 1)));
        x1.upload(d1, size_t(d.nc) * d.np, h->ctx.s);
        back_substitute(h->ctx, d, x1.p, x2.p);
        x2.download(d2, size_t(d.n2), h->ctx.s);
        h->ctx.sync();
    });
}

void mprec_gpu_condensed_destroy(mprec_gpu_condensed* h) { delete h; }

int mprec_gpu_get_shape(mprec_gpu_system* h, int* n_cells, int* nb, int* nnzb) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (n_cells) *n_cells = h->pat.nc;
        if (nb) *nb = h->nb;
        if (nnzb) *nnzb = h->pat.nnzb;
    });
}

int mprec_gpu_get_matrix(mprec_gpu_system* h, int* rp, int* ci, double* vals, double* b) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (rp) std::memcpy(rp, h->pat.h_rp.data(), sizeof(int) * h->pat.h_rp.size());
        if (ci) std::memcpy(ci, h->pat.h_ci.data(), sizeof(int) * h->pat.h_ci.size());
        if (vals) h->a_val.download(vals, size_t(h->pat.nnzb) * h->nb * h->nb, h->ctx.s);
        if (b) {
            if (int64_t(h->b_host.size()) != h->n) throw Error(MPREC_DIMENSION, "the handle holds no rhs");
            std::memcpy(b, h->b_host.data(), sizeof(double) * h->n);
        }
        h->ctx.sync();
    });
}

int mprec_gpu_write_system(mprec_gpu_system* h, const char* mtx, const char* layout, const char* rhs) {
    return guard([&] {
        if (!h || !mtx || !layout) throw Error(MPREC_DIMENSION, "null argument");
        const std::vector<double> v = h->a_val.to_host(h->ctx.s, size_t(h->pat.nnzb) * h->nb * h->nb);
        write_system(mtx, layout, rhs, h->pat.nc, h->nb, h->pat.h_rp, h->pat.h_ci, v,
                     int64_t(h->b_host.size()) == h->n ? h->b_host.data() : nullptr);
    });
}

int mprec_gpu_apply(mprec_gpu_system* h, const double* r, double* z) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        h->r.upload(r, h->n, h->ctx.s);
        h->prec_apply(h->r.p, h->y.p);
        h->y.download(z, h->n, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_apply_stage(mprec_gpu_system* h, int stage, const double* r, double* z) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        h->r.upload(r, h->n, h->ctx.s);
        h->stage_apply(stage, h->r.p, h->y.p);
        h->y.download(z, h->n, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_spmv(mprec_gpu_system* h, int which, const double* x, double* y) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (which != 0 && !h->ready) throw Error(MPREC_SETUP, "setup not done");
        h->r.ensure(h->n);
        h->y.ensure(h->n);
        h->r.upload(x, h->n, h->ctx.s);
        bsr_spmv(h->ctx, which == 0 ? h->A() : h->Abar(), h->r.p, h->y.p, nullptr, MPREC_K_SPMV);
        h->y.download(y, h->n, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_solve_dev(mprec_gpu_system* h, double tol, int max_iter, double* x_dev, mprec_solve_result* out) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        const double t0 = now_s();
        int attempts = 0;
        double* xd = x_dev ? x_dev : h->x.p;
        const GmresOut g = h->solve_attempts(tol, max_iter, xd, &attempts);
        h->ctx.sync();
        fill_result(out, g, attempts, h->setup_s, now_s() - t0, nullptr, 0, h->total_iterations);
        h->log_attempts(out);
    });
}

int mprec_gpu_last_history(mprec_gpu_system* h, double* history, int history_cap, int* len) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        const int m = int(h->last_history.size());
        if (len) *len = m;
        if (history)
            for (int i = 0; i < std::min(m, history_cap); ++i) history[i] = h->last_history[i];
    });
}

int mprec_gpu_solve(mprec_gpu_system* h, double tol, int max_iter, double* x, mprec_solve_result* out,
                    double* history, int history_cap) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        const double t0 = now_s();
        int attempts = 0;
        const GmresOut g = h->solve_attempts(tol, max_iter, h->x.p, &attempts);
        h->x.download(x, h->n, h->ctx.s);
        h->ctx.sync();
        fill_result(out, g, attempts, h->setup_s, now_s() - t0, history, history_cap, h->total_iterations);
        h->log_attempts(out);
    });
}

int mprec_gpu_solve_system(const mprec_bsr* a, const double* b, int method, double tol, int max_iter, double* x,
                           mprec_solve_result* out) {
    mprec_gpu_system* h = nullptr;
    const double t0 = now_s();
    int st = mprec_gpu_create(a, &h);
    const double t1 = now_s();
    if (st == MPREC_OK) st = mprec_gpu_setup(h, method, nullptr, b);
    const double t2 = now_s();
    if (st == MPREC_OK) st = mprec_gpu_solve(h, tol, max_iter, x, out, nullptr, 0);
    const double t3 = now_s();
    if (h) {
        std::string keep = g_err;
        int kp = g_payload;
        mprec_gpu_destroy(h);
        g_err = keep;
        g_payload = kp;
    }
    if (trace_on())
        fprintf(stderr, "[mprec] solve_system: create (validate + H2D) %.3f s, setup %.3f s, solve %.3f s, destroy %.3f s\n",
                t1 - t0, t2 - t1, t3 - t2, now_s() - t3);
    return st;
}

int mprec_gpu_scaling_record(mprec_gpu_system* h, char* buf, int cap) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        if (!buf || cap < 1) throw Error(MPREC_DIMENSION, "empty buffer");
        std::strncpy(buf, h->scaling_record.c_str(), size_t(cap) - 1);
        buf[cap - 1] = 0;
    });
}

int mprec_gpu_get_scaled(mprec_gpu_system* h, double* abar, double* bbar) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        if (abar) h->abar_val.download(abar, size_t(h->pat.nnzb) * h->nb * h->nb, h->ctx.s);
        if (bbar) h->bbar.download(bbar, h->n, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_get_ilu(mprec_gpu_system* h, double* lu) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        h->lu_val.download(lu, size_t(h->pat.nnzb) * h->nb * h->nb, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_n_stages(mprec_gpu_system* h, int* n) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        *n = !h->ready ? 0 : h->n_stages();
    });
}

int mprec_gpu_stage_amg(mprec_gpu_system* h, int stage, mprec_gpu_amg** out) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        Amg* a = nullptr;  // -direct stages have no hierarchy (as in the oracle)
        if (h->method == MPREC_METHOD_CPR_AMG && stage == 0) a = h->amgP.get();
        if (h->method == MPREC_METHOD_CPTR3_AMG && stage == 0) a = h->amgT.get();
        if (h->method == MPREC_METHOD_CPTR3_AMG && stage == 1) a = h->amgP.get();
        if (!a) throw Error(MPREC_INDEX, "not an AMG stage");
        for (auto& v : h->views)  // one live view per stage hierarchy
            if (v->amg == a) {
                *out = v.get();
                return;
            }
        auto v = std::make_unique<mprec_gpu_amg>();
        v->ctx = &h->ctx;
        v->amg = a;
        *out = v.get();
        h->views.push_back(std::move(v));
    });
}

void mprec_gpu_destroy(mprec_gpu_system* h) {
    if (!h) return;
    try {
        h->ctx.sync();
    } catch (...) {
    }
    delete h;
}

// ------------------------------------------------------------------ AMG ---
int mprec_gpu_amg_create(const mprec_csr* a, const mprec_amg_params* p, mprec_gpu_amg** out) {
    return guard([&] {
        if (!a || !out) throw Error(MPREC_DIMENSION, "null argument");
        const int n = a->n_rows;
        if (n < 0) throw Error(MPREC_DIMENSION, "negative matrix dimension");
        const int nnz = a->row_ptr[n];
        for (int i = 0; i < n; ++i)
            for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
                if (a->col_idx[k] < 0 || a->col_idx[k] >= n) throw Error(MPREC_INDEX, "column out of range");
                if (k > a->row_ptr[i] && a->col_idx[k] <= a->col_idx[k - 1])
                    throw Error(MPREC_INDEX, "CSR not canonical (columns must be strictly increasing)");
            }
        auto h = std::make_unique<mprec_gpu_amg>();
        h->own_ctx = std::make_unique<Ctx>();
        h->ctx = h->own_ctx.get();
        Ctx& c = *h->ctx;
        h->a0.n = h->a0.m = n;
        h->a0.nnz = nnz;
        h->a0.rp.upload(a->row_ptr, n + 1, c.s);
        h->a0.ci.upload(a->col_idx, std::max(nnz, 1), c.s);
        h->a0.v.upload(a->values, std::max(nnz, 1), c.s);
        AmgParams prm;
        if (p) {
            prm.theta = p->strength_threshold;
            prm.max_coarse = p->max_coarse_size;
            prm.max_levels = p->max_levels;
        }
        h->own_amg = std::make_unique<Amg>();
        h->amg = h->own_amg.get();
        CsrView v = h->a0.view();
        v.diag = nullptr;
        h->amg->setup(c, v, prm);
        c.sync();
        *out = h.release();
    });
}

int mprec_gpu_amg_apply(mprec_gpu_amg* h, const double* r, double* x) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        Ctx& c = *h->ctx;
        const int n = h->amg->lv[0]->n;
        h->r.upload(r, std::max(n, 1), c.s);
        h->x.ensure(std::max(n, 1));
        h->amg->apply(c, h->r.p, h->x.p);
        h->x.download(x, n, c.s);
        c.sync();
    });
}

int mprec_gpu_amg_n_levels(mprec_gpu_amg* h, int* n) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        *n = h->amg->n_levels();
    });
}

int mprec_gpu_amg_level_info(mprec_gpu_amg* h, int l, int* n, int* nnz_a, int* nnz_p) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        if (l < 0 || l >= h->amg->n_levels()) throw Error(MPREC_INDEX, "level out of range");
        const AmgLevel& L = *h->amg->lv[l];
        *n = L.n;
        *nnz_a = L.a.nnz;
        *nnz_p = l == 0 ? 0 : L.p.nnz;
    });
}

int mprec_gpu_amg_get_csr(mprec_gpu_amg* h, int l, int which, int* rp, int* ci, double* v) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        if (l < 0 || l >= h->amg->n_levels()) throw Error(MPREC_INDEX, "level out of range");
        if (which != 0 && l == 0) throw Error(MPREC_INDEX, "level 0 has no P/R");
        Ctx& c = *h->ctx;
        const AmgLevel& L = *h->amg->lv[l];
        CsrView m = which == 0 ? L.a : (which == 1 ? L.p.view() : L.r.view());
        if (rp) MG_CUDA(cudaMemcpyAsync(rp, m.rp, sizeof(int) * (m.n + 1), cudaMemcpyDeviceToHost, c.s));
        if (ci && m.nnz) MG_CUDA(cudaMemcpyAsync(ci, m.ci, sizeof(int) * m.nnz, cudaMemcpyDeviceToHost, c.s));
        if (v && m.nnz) MG_CUDA(cudaMemcpyAsync(v, m.v, sizeof(double) * m.nnz, cudaMemcpyDeviceToHost, c.s));
        c.sync();
    });
}

static void levels_out(Ctx& c, const int* dev_levels, int n, int nlev, int* levels, int* n_levels) {
    if (levels && n > 0) MG_CUDA(cudaMemcpyAsync(levels, dev_levels, sizeof(int) * n, cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (n_levels) *n_levels = nlev;
}

int mprec_gpu_amg_get_levelsets(mprec_gpu_amg* h, int l, int dir, int* levels, int* n_levels) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        if (l < 0 || l + 1 >= h->amg->n_levels()) throw Error(MPREC_INDEX, "level is not smoothed");
        if (dir != 1 && dir != -1) throw Error(MPREC_INDEX, "dir must be +1 or -1");
        const AmgLevel& L = *h->amg->lv[l];
        const int* lev = dir > 0 ? L.glev_f : L.glev_b;
        if (!lev) throw Error(MPREC_SETUP, "no sweep schedule on this level");
        // level 0 may borrow the block pattern's schedule (same DAG, shared)
        const Sched& own = dir > 0 ? L.own_fwd : L.own_bwd;
        int nlev = own.nlev;
        if (lev != own.level.p) {
            std::vector<int> hl(L.n);
            MG_CUDA(cudaMemcpyAsync(hl.data(), lev, sizeof(int) * L.n, cudaMemcpyDeviceToHost, h->ctx->s));
            h->ctx->sync();
            nlev = 0;
            for (int v : hl) nlev = std::max(nlev, v + 1);
        }
        levels_out(*h->ctx, lev, L.n, nlev, levels, n_levels);
    });
}

int mprec_gpu_get_levelsets(mprec_gpu_system* h, int dir, int* levels, int* n_levels) {
    return guard([&] {
        if (!h) throw Error(MPREC_DIMENSION, "null handle");
        if (dir != 1 && dir != -1) throw Error(MPREC_INDEX, "dir must be +1 or -1");
        h->pat.ensure_sched(h->ctx);
        const Sched& s = dir > 0 ? h->pat.fwd : h->pat.bwd;
        levels_out(h->ctx, s.level.p, h->pat.nc, s.nlev, levels, n_levels);
    });
}

int mprec_gpu_amg_get_cf(mprec_gpu_amg* h, int l, signed char* cf) {
    return guard([&] {
        if (!h || !h->amg) throw Error(MPREC_SETUP, "stale AMG view: its system was set up again");
        if (l < 0 || l + 1 >= h->amg->n_levels()) throw Error(MPREC_INDEX, "level has no coarsening");
        Ctx& c = *h->ctx;
        const AmgLevel& L = *h->amg->lv[l];
        std::vector<signed char> m = L.cf.to_host(c.s, L.n);
        for (int i = 0; i < L.n; ++i) cf[i] = m[i] == 1 ? 1 : 0;
    });
}

void mprec_gpu_amg_destroy(mprec_gpu_amg* h) {
    if (!h || !h->own_amg) return;  // views are owned by their system
    delete h;
}

// ------------------------------------------------------------------ ILU ---
int mprec_gpu_ilu_create(const mprec_bsr* a, mprec_gpu_ilu** out) {
    return guard([&] {
        if (!a || !out) throw Error(MPREC_DIMENSION, "null argument");
        auto h = std::make_unique<mprec_gpu_ilu>();
        load_pattern(h->ctx, h->pat, a->n_cells, a->nb, a->row_ptr, a->col_idx, MPREC_SETUP);
        const size_t nv = std::max<size_t>(size_t(h->pat.nnzb) * a->nb * a->nb, 1);
        h->vals.upload(a->values, nv, h->ctx.s);
        h->ilu.lu = view_of(h->pat, a->nb, h->vals.p);
        h->ilu.pat = &h->pat;
        h->ilu.factor(h->ctx);
        h->ctx.sync();
        *out = h.release();
    });
}

int mprec_gpu_ilu_apply(mprec_gpu_ilu* h, const double* r, double* y) {
    return guard([&] {
        const int64_t n = int64_t(h->pat.nc) * h->ilu.lu.nb;
        h->r.upload(r, n, h->ctx.s);
        h->y.ensure(n);
        h->ilu.apply(h->ctx, h->r.p, h->y.p);
        h->y.download(y, n, h->ctx.s);
        h->ctx.sync();
    });
}

int mprec_gpu_ilu_get(mprec_gpu_ilu* h, double* lu) {
    return guard([&] {
        h->vals.download(lu, size_t(h->pat.nnzb) * h->ilu.lu.nb * h->ilu.lu.nb, h->ctx.s);
        h->ctx.sync();
    });
}

void mprec_gpu_ilu_destroy(mprec_gpu_ilu* h) { delete h; }

// ---------------------------------------------------------------- GMRES ---
int mprec_gpu_gmres(const mprec_bsr* a, const double* b, int prec_kind, void* prec, double tol, int max_iter,
                    double* x, mprec_solve_result* out, double* history, int history_cap) {
    return guard([&] {
        if (!a) throw Error(MPREC_DIMENSION, "null argument");
        std::unique_ptr<Ctx> own;
        Ctx* c = nullptr;
        if (prec_kind == 1)
            c = static_cast<mprec_gpu_amg*>(prec)->ctx;
        else if (prec_kind == 2)
            c = &static_cast<mprec_gpu_ilu*>(prec)->ctx;
        else if (prec_kind == 0) {
            own = std::make_unique<Ctx>();
            c = own.get();
        } else
            throw Error(MPREC_CONFIG, "unknown preconditioner kind");
        Pattern pat;
        load_pattern(*c, pat, a->n_cells, a->nb, a->row_ptr, a->col_idx);
        const int64_t n = int64_t(a->n_cells) * a->nb;
        DBuf<double> vals, bd, xd, tmp;
        vals.upload(a->values, std::max<size_t>(size_t(pat.nnzb) * a->nb * a->nb, 1), c->s);
        bd.upload(b, n, c->s);
        xd.ensure(n);
        tmp.ensure(n);
        const BsrView av = view_of(pat, a->nb, vals.p);
        const DevOp Aop = [&](const double* xx, double* yy) { bsr_spmv(*c, av, xx, yy, nullptr, MPREC_K_SPMV); };
        DevOp Mop;
        if (prec_kind == 0)
            Mop = [&](const double* xx, double* yy) { copy(*c, yy, xx, n); };
        else if (prec_kind == 1) {
            auto* ah = static_cast<mprec_gpu_amg*>(prec);
            if (ah->amg->lv[0]->n != n) throw Error(MPREC_DIMENSION, "preconditioner dimension mismatch");
            Mop = [&, ah](const double* xx, double* yy) { ah->amg->apply(*c, xx, yy); };
        } else {
            auto* ih = static_cast<mprec_gpu_ilu*>(prec);
            if (int64_t(ih->ilu.lu.nc) * ih->ilu.lu.nb != n)
                throw Error(MPREC_DIMENSION, "preconditioner dimension mismatch");
            Mop = [&, ih](const double* xx, double* yy) { ih->ilu.apply(*c, xx, yy); };
        }
        const double t0 = now_s();
        Krylov kr;
        const GmresOut g = gmres_dev(*c, kr, n, Aop, Mop, bd.p, tol, max_iter, xd.p);
        xd.download(x, n, c->s);
        c->sync();
        fill_result(out, g, 1, 0.0, now_s() - t0, history, history_cap);
    });
}

// ----------------------------------------------------------- measurement ---
int mprec_gpu_profile(mprec_gpu_system* h, int enable) {
    return guard([&] {
        h->ctx.harvest();
        h->ctx.profile = enable != 0;
    });
}

// Diagnostics (not in the public header): timeline of one forward ILU sweep.
int mprec_gpu_debug_ilu_timeline(mprec_gpu_system* h, int blocks, long long* ts, int* order, int* nlev) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        DBuf<long long> t(2 * h->pat.nc);
        fill(h->ctx, h->r.p, 1.0, h->n);
        const double t0 = now_s();
        ilu_timeline(h->ctx, h->ilu, h->r.p, h->y.p, t.p, blocks);
        fprintf(stderr, "ilu fwd sweep wall %.3f ms\n", 1e3 * (now_s() - t0));
        t.download(ts, 2 * h->pat.nc, h->ctx.s);
        h->pat.fwd.order.download(order, h->pat.nc, h->ctx.s);
        *nlev = h->pat.fwd.nlev;
        h->ctx.sync();
    });
}

// Diagnostics: sweep timing on one AMG level (stage as in mprec_gpu_stage_amg).
int mprec_gpu_debug_gs(mprec_gpu_system* h, int stage, int level, int reps, double* ms_f, double* ms_b, int* nl_f,
                       int* nl_b) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        Amg* a = (h->method == MPREC_METHOD_CPTR3_AMG && stage == 0) ? h->amgT.get() : h->amgP.get();
        if (!a || level < 0 || level + 1 >= a->n_levels()) throw Error(MPREC_INDEX, "level out of range");
        gs_bench(h->ctx, *a, level, reps, ms_f, ms_b, nl_f, nl_b);
        if (level == 0 && *nl_f >= 0) {
            *nl_f = h->pat.fwd.nlev;
            *nl_b = h->pat.bwd.nlev;
        }
    });
}

// Diagnostics: level-synchronous sweep programs with K groups on one level vs the current kernel.
int mprec_gpu_debug_gs_ls(mprec_gpu_system* h, int stage, int level, int K, int reps, double* out10) {
    return guard([&] {
        if (!h || !h->ready) throw Error(MPREC_SETUP, "setup not done");
        Amg* a = (h->method == MPREC_METHOD_CPTR3_AMG && stage == 0) ? h->amgT.get() : h->amgP.get();
        if (!a || level < 0 || level + 1 >= a->n_levels()) throw Error(MPREC_INDEX, "level out of range");
        gs_ls_experiment(h->ctx, *a, level, K, reps, out10);
    });
}

int mprec_gpu_stream(mprec_gpu_system* h, void** stream) {
    return guard([&] { *stream = (void*)h->ctx.s; });
}

int mprec_gpu_kernel_stats(mprec_gpu_system* h, int kc, double* ms, int64_t* launches, double* bytes) {
    return guard([&] {
        if (kc < 0 || kc >= MPREC_K_COUNT) throw Error(MPREC_INDEX, "kernel class out of range");
        h->ctx.harvest();
        if (ms) *ms = h->ctx.stat[kc].ms;
        if (launches) *launches = h->ctx.stat[kc].launches;
        if (bytes) *bytes = h->ctx.stat[kc].bytes;
    });
}

int mprec_gpu_reset_stats(mprec_gpu_system* h) {
    return guard([&] { h->ctx.reset_stats(); });
}

int mprec_gpu_launch_count(mprec_gpu_system* h, int64_t* launches) {
    return guard([&] { *launches = h->ctx.launches; });
}

}  // extern "C"
