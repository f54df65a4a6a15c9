// C++ drop-in check: the facade (include/mprec_gpu.hpp) used the way the
// reference's own doctest suites use mprec:: (proj/tests/test_krylov.cpp,
// test_subprec.cpp, test_stages.cpp, acceptance.cpp).  Prints one line per
// case; exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../../include/mprec_gpu.hpp"
#include "../../paper_1912_04385_b200/csrc/gen/mprec_gen.h"

using namespace mprec::gpu;

#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            std::exit(1);                                                    \
        }                                                                    \
    } while (0)

static ScalarMatrix laplacian_1d(int n) {
    ScalarMatrix m;
    m.n = n;
    m.row_ptr.push_back(0);
    for (int i = 0; i < n; ++i) {
        if (i > 0) m.col_idx.push_back(i - 1), m.values.push_back(-1.0);
        m.col_idx.push_back(i), m.values.push_back(2.0);
        if (i + 1 < n) m.col_idx.push_back(i + 1), m.values.push_back(-1.0);
        m.row_ptr.push_back(int(m.col_idx.size()));
    }
    return m;
}

static Vector random_vec(int n, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    Vector v(n);
    for (auto& x : v) x = u(rng);
    return v;
}

int main() {
    // test_krylov.cpp:46-53 -- identity converges in one iteration
    {
        ScalarMatrix id;
        id.n = 20;
        for (int i = 0; i <= 20; ++i) id.row_ptr.push_back(i);
        for (int i = 0; i < 20; ++i) id.col_idx.push_back(i), id.values.push_back(1.0);
        const Vector b = random_vec(20, 1);
        const SolveResult r = gmres(id.as_block(), b);
        CHECK(r.converged && r.iterations == 1);
        std::printf("ok identity gmres: %d iteration\n", r.iterations);
    }
    // test_subprec.cpp:157-168 -- coarsening halves a 1-d chain
    {
        AMGParams p;
        p.max_coarse_size = 32;
        const AMGHierarchy h = AMGHierarchy::setup(laplacian_1d(64), p);
        CHECK(h.n_levels() == 2);
        int n = 0, na = 0, np = 0;
        check(mprec_gpu_amg_level_info(h.handle(), 1, &n, &na, &np));
        CHECK(n == 32 && np > 0);
        std::printf("ok 1-d chain coarsens to %d C points\n", n);
    }
    // test_subprec.cpp:124-134 -- typed errors with payloads
    {
        ScalarMatrix z;
        z.n = 2;
        z.row_ptr = {0, 2, 4};
        z.col_idx = {0, 1, 0, 1};
        z.values = {1.0, 1.0, 2.0, 2.0};
        bool thrown = false;
        try {
            ILU0Factor::factor(z);
        } catch (const ZeroPivotError& e) {
            thrown = e.row_id == 1;
        }
        CHECK(thrown);
        ScalarMatrix nd;
        nd.n = 2;
        nd.row_ptr = {0, 1, 3};
        nd.col_idx = {1, 0, 1};
        nd.values = {1.0, 1.0, 1.0};
        thrown = false;
        try {
            ILU0Factor::factor(nd);
        } catch (const SetupError&) {
            thrown = true;
        }
        CHECK(thrown);
        thrown = false;
        try {
            parse_method("cptr-amg");
        } catch (const ConfigError&) {
            thrown = true;
        }
        CHECK(thrown);
        std::printf("ok ZeroPivotError{row 1}, SetupError, ConfigError\n");
    }
    // harness solve_system on a BASELINE-generator system (both methods)
    {
        mprec_gen_spec s{16, 12, 4, 1.0, 1.0, 1, 9};
        BlockMatrix a;
        a.n_cells = s.nx * s.ny;
        a.nb = s.nb;
        const int64_t nnzb = mprec_gen_nnzb(s.nx, s.ny);
        a.row_ptr.resize(a.n_cells + 1);
        a.col_idx.resize(nnzb);
        a.values.resize(size_t(nnzb) * s.nb * s.nb);
        Vector xs(a.dim()), b(a.dim());
        mprec_gen_pattern(s.nx, s.ny, a.row_ptr.data(), a.col_idx.data());
        mprec_gen_fill(&s, a.row_ptr.data(), a.col_idx.data(), a.values.data(), xs.data(), b.data(), 1);
        for (const char* name : {"cpr-amg", "cptr3-amg"}) {
            const SolveOutcome o = solve_system(a, b, parse_method(name));
            double err = 0, nx = 0;
            for (int i = 0; i < a.dim(); ++i) err += (o.result.x[i] - xs[i]) * (o.result.x[i] - xs[i]), nx += xs[i] * xs[i];
            CHECK(o.result.converged && o.result.final_true_residual <= 1e-8 && std::sqrt(err / nx) < 1e-6);
            std::printf("ok solve_system %s: %d iterations, true residual %.2e\n", name, o.result.iterations,
                        o.result.final_true_residual);
        }
    }
    // MethodSpec{Method, SubSolver} incl. the -direct sub-solvers, ScalingOptions,
    // scaling_record (scaling.hpp:13-30, harness.hpp:79-83)
    {
        mprec_gen_spec s{12, 10, 4, 1.0, 1.0, 1, 7};
        BlockMatrix a;
        a.n_cells = s.nx * s.ny;
        a.nb = s.nb;
        const int64_t nnzb = mprec_gen_nnzb(s.nx, s.ny);
        a.row_ptr.resize(a.n_cells + 1);
        a.col_idx.resize(nnzb);
        a.values.resize(size_t(nnzb) * s.nb * s.nb);
        Vector xs(a.dim()), b(a.dim());
        mprec_gen_pattern(s.nx, s.ny, a.row_ptr.data(), a.col_idx.data());
        mprec_gen_fill(&s, a.row_ptr.data(), a.col_idx.data(), a.values.data(), xs.data(), b.data(), 1);
        for (const char* name : {"ilu0", "cpr-direct", "cpr-amg", "cptr-direct", "cptr3-direct", "cptr3-amg"}) {
            const MethodSpec spec = parse_method(name);
            CHECK(method_name(spec) == name);
            const SolveOutcome o = solve_system(a, b, spec);
            CHECK(o.result.converged && o.result.final_true_residual <= 1e-8);
            std::printf("ok %s: %d iterations, scaling record '%s'\n", name, o.result.iterations,
                        o.scaling_record.c_str());
        }
        CHECK(solve_system(a, b, parse_method("cptr3-amg")).scaling_record == "[D_Ps;D_Ts]*D_ss^-1, D_Tp*D_PP^-1");
        CHECK(solve_system(a, b, parse_method("cpr-amg")).scaling_record == "D_Ph*D_hh^-1");
        ScalingOptions so;
        so.diag_mode = DiagMode::Scalar;
        so.second_scaling_from_original = true;
        const StagePreconditioner p = StagePreconditioner::build(a, b, {Method::Cptr3, SubSolver::Amg}, {}, so);
        const SolveResult r = p.solve();
        CHECK(r.converged && p.n_stages() == 3 && p.spec().sub == SubSolver::Amg);
        std::printf("ok ScalingOptions{Scalar, from original}: %d iterations\n", r.iterations);
    }
    // BlockMatrix::assemble semantics: duplicates summed, zero diagonal inserted
    {
        const BlockMatrix m = BlockMatrix::assemble(2, 1, {{{0, 1}, {1.0}}, {{0, 1}, {2.0}}, {{1, 1}, {5.0}}});
        CHECK(m.row_ptr == std::vector<int>({0, 2, 3}) && m.values[1] == 3.0 && m.values[0] == 0.0);
        std::printf("ok assemble\n");
    }
    std::printf("all facade checks passed\n");
    return 0;
}
