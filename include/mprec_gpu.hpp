// mprec_gpu.hpp -- C++ host facade over the C ABI (include/mprec_gpu.h) that
// mirrors the reference's solve-path interface (proj/include/mprec/*.hpp):
// same names, argument meaning, defaults and exception classes, with
// std::vector<double> in place of Eigen::VectorXd (Eigen is not a dependency
// of the B200 library).  Header-only; link against libmprec_gpu.so.
//
//   reference                                   facade
//   ---------                                   ------
//   BlockMatrix::assemble (block_matrix.hpp:56)  BlockMatrix::assemble
//   MethodSpec / parse_method (scaling.hpp:13-22) MethodSpec / parse_method / method_name
//   ScalingOptions (scaling.hpp:22-30)          ScalingOptions
//   left_scale + build_preconditioner           StagePreconditioner::build
//     (scaling.hpp:65, stages.hpp:85)
//   StagePreconditioner::apply (stages.hpp:47)  StagePreconditioner::apply
//   solve_system (harness.hpp:87)               solve_system
//   AMGHierarchy::setup/apply (amg.hpp:30-34)   AMGHierarchy
//   ILU0Factor::factor/apply (ilu0.hpp:13-16)   ILU0Factor
//   gmres (gmres.hpp:41)                        gmres (matrix operator)
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mprec_gpu.h"

namespace mprec {
namespace gpu {

using Vector = std::vector<double>;

// ---- errors.hpp:9-59 --------------------------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct DimensionError : Error {
    using Error::Error;
};
struct IndexError : Error {
    using Error::Error;
};
struct SingularBlockError : Error {
    SingularBlockError(const std::string& m, int cell) : Error(m), cell_id(cell) {}
    int cell_id;
};
struct ZeroPivotError : Error {
    ZeroPivotError(const std::string& m, int row) : Error(m), row_id(row) {}
    int row_id;
};
struct SetupError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int st) {
    if (st == MPREC_OK) return;
    const std::string m = mprec_gpu_last_error();
    const int p = mprec_gpu_error_payload();
    switch (st) {
        case MPREC_DIMENSION: throw DimensionError(m);
        case MPREC_INDEX: throw IndexError(m);
        case MPREC_SINGULAR_BLOCK: throw SingularBlockError(m, p);
        case MPREC_ZERO_PIVOT: throw ZeroPivotError(m, p);
        case MPREC_SETUP: throw SetupError(m);
        case MPREC_CONFIG: throw ConfigError(m);
        case MPREC_CUDA: throw DeviceError(m);
        default: throw Error(m);
    }
}

// ---- scaling.hpp:10-30 --------------------------------------------------------
enum class Method { Ilu0, Cpr, Cptr, Cptr3 };
enum class SubSolver { Direct, Amg };

struct MethodSpec {  // scaling.hpp:13-16
    Method method = Method::Ilu0;
    SubSolver sub = SubSolver::Direct;
};

// parse_method (scaling.cpp:5-15)
inline MethodSpec parse_method(const std::string& name) {
    if (name == "ilu0") return {Method::Ilu0, SubSolver::Direct};
    if (name == "cpr-direct") return {Method::Cpr, SubSolver::Direct};
    if (name == "cpr-amg") return {Method::Cpr, SubSolver::Amg};
    if (name == "cptr-direct") return {Method::Cptr, SubSolver::Direct};
    if (name == "cptr-amg") throw ConfigError("cptr supports only the -direct sub-solver");
    if (name == "cptr3-direct") return {Method::Cptr3, SubSolver::Direct};
    if (name == "cptr3-amg") return {Method::Cptr3, SubSolver::Amg};
    throw ConfigError("unknown method '" + name + "'");
}

// method_name (scaling.cpp:17-25)
inline std::string method_name(const MethodSpec& s) {
    switch (s.method) {
        case Method::Ilu0: return "ilu0";
        case Method::Cpr: return s.sub == SubSolver::Amg ? "cpr-amg" : "cpr-direct";
        case Method::Cptr: return "cptr-direct";
        case Method::Cptr3: return s.sub == SubSolver::Amg ? "cptr3-amg" : "cptr3-direct";
    }
    return "?";
}

// MethodSpec -> the C ABI's mprec_method id
inline int method_id(const MethodSpec& s) {
    switch (s.method) {
        case Method::Ilu0: return MPREC_METHOD_ILU0;
        case Method::Cpr: return s.sub == SubSolver::Amg ? MPREC_METHOD_CPR_AMG : MPREC_METHOD_CPR_DIRECT;
        case Method::Cptr:
            if (s.sub == SubSolver::Amg) throw ConfigError("cptr supports only the -direct sub-solver");
            return MPREC_METHOD_CPTR_DIRECT;
        case Method::Cptr3: return s.sub == SubSolver::Amg ? MPREC_METHOD_CPTR3_AMG : MPREC_METHOD_CPTR3_DIRECT;
    }
    throw ConfigError("unreachable method");
}

enum class DiagMode { Block, Scalar };  // block_matrix.hpp:46

struct ScalingOptions {  // scaling.hpp:22-30
    DiagMode diag_mode = DiagMode::Block;
    bool second_scaling_from_original = false;
    mprec_scaling_options c() const {
        return {diag_mode == DiagMode::Scalar ? MPREC_DIAG_SCALAR : MPREC_DIAG_BLOCK,
                second_scaling_from_original ? 1 : 0};
    }
};

struct AMGParams {  // amg.hpp:12-16
    double strength_threshold = 0.25;
    int max_coarse_size = 1000;
    int max_levels = 25;
    mprec_amg_params c() const { return {strength_threshold, max_coarse_size, max_levels}; }
};

struct GmresOptions {  // gmres.hpp:23-26
    double tol = 1e-8;
    int max_iter = 500;
};

struct SolveResult {  // gmres.hpp:28-36
    Vector x;
    int iterations = 0;
    bool converged = false;
    bool breakdown = false;
    std::vector<double> residual_history;
    double final_true_residual = 0.0;
    double wall_time_s = 0.0;
};

struct SolveOutcome {  // harness.hpp:79-83
    SolveResult result;
    double setup_time_s = 0.0;
    std::string scaling_record;  // applied D factors, ", "-joined (harness.cpp:197-201)
};

// ---- uniform-layout BlockMatrix (block_matrix.hpp:50-101) --------------------
// Blocks are nb x nb, COLUMN-MAJOR (Eigen's default), intra-cell order (s..., P, T).
struct BlockMatrix {
    int n_cells = 0, nb = 0;
    std::vector<int> row_ptr, col_idx;
    std::vector<double> values;

    int dim() const { return n_cells * nb; }
    mprec_bsr c() const { return {n_cells, nb, row_ptr.data(), col_idx.data(), values.data()}; }

    // BlockMatrix::assemble (block_matrix.cpp:32-69): duplicates summed, the
    // diagonal block always present.  blocks: ((row, col), column-major nb*nb).
    static BlockMatrix assemble(int n_cells, int nb,
                                const std::vector<std::pair<std::pair<int, int>, Vector>>& entries) {
        std::map<std::pair<int, int>, Vector> merged;
        for (const auto& e : entries) {
            if (e.first.first < 0 || e.first.first >= n_cells || e.first.second < 0 || e.first.second >= n_cells)
                throw IndexError("block entry cell index out of range");
            if (int(e.second.size()) != nb * nb) throw DimensionError("block dimensions inconsistent with layout");
            auto it = merged.find(e.first);
            if (it == merged.end())
                merged.emplace(e.first, e.second);
            else
                for (int k = 0; k < nb * nb; ++k) it->second[k] += e.second[k];
        }
        for (int c = 0; c < n_cells; ++c)
            if (!merged.count({c, c})) merged.emplace(std::make_pair(c, c), Vector(size_t(nb) * nb, 0.0));
        BlockMatrix m;
        m.n_cells = n_cells;
        m.nb = nb;
        m.row_ptr.assign(n_cells + 1, 0);
        for (const auto& kv : merged) {
            m.col_idx.push_back(kv.first.second);
            m.values.insert(m.values.end(), kv.second.begin(), kv.second.end());
            m.row_ptr[kv.first.first + 1]++;
        }
        for (int c = 0; c < n_cells; ++c) m.row_ptr[c + 1] += m.row_ptr[c];
        return m;
    }
};

// left_scale + build_preconditioner on the device; apply == StagePreconditioner::apply.
class StagePreconditioner {
   public:
    // left_scale(a, b, spec.method, so) + build_preconditioner(scaled, spec, p)
    static StagePreconditioner build(const BlockMatrix& a, const Vector& b, const MethodSpec& spec,
                                     const AMGParams& p = {}, const ScalingOptions& so = {}) {
        StagePreconditioner s;
        const int mid = method_id(spec);
        mprec_gpu_system* h = nullptr;
        const mprec_bsr ca = a.c();
        check(mprec_gpu_create(&ca, &h));
        s.h_.reset(h, mprec_gpu_destroy);
        if (int(b.size()) != a.dim()) throw DimensionError("rhs length mismatch");
        const mprec_amg_params cp = p.c();
        const mprec_scaling_options co = so.c();
        check(mprec_gpu_setup_opts(h, mid, &cp, &co, b.data()));
        s.n_ = a.dim();
        s.spec_ = spec;
        return s;
    }
    MethodSpec spec() const { return spec_; }
    // ScaledSystem::scaling_record, ", "-joined
    std::string scaling_record() const {
        char buf[256];
        check(mprec_gpu_scaling_record(h_.get(), buf, int(sizeof buf)));
        return buf;
    }
    int n_stages() const {
        int n = 0;
        check(mprec_gpu_n_stages(h_.get(), &n));
        return n;
    }
    Vector apply(const Vector& r) const {
        if (int(r.size()) != n_) throw DimensionError("apply length mismatch");
        Vector z(n_);
        check(mprec_gpu_apply(h_.get(), r.data(), z.data()));
        return z;
    }
    Vector apply_stage(int i, const Vector& r) const {
        Vector z(n_);
        check(mprec_gpu_apply_stage(h_.get(), i, r.data(), z.data()));
        return z;
    }
    // solve_system's GMRES part (harness.cpp:198-218) on this system
    SolveResult solve(double tol = 1e-8, int max_iter = 500) const {
        SolveResult r;
        r.x.assign(n_, 0.0);
        mprec_solve_result o{};
        std::vector<double> hist(size_t(std::min(max_iter, n_)) + 2);
        check(mprec_gpu_solve(h_.get(), tol, max_iter, r.x.data(), &o, hist.data(), int(hist.size())));
        r.iterations = o.iterations;
        r.converged = o.converged != 0;
        r.breakdown = o.breakdown != 0;
        r.residual_history.assign(hist.begin(), hist.begin() + o.history_len);
        r.final_true_residual = o.final_true_residual;
        r.wall_time_s = o.solve_s;
        setup_s_ = o.setup_s;
        return r;
    }
    double setup_time_s() const { return setup_s_; }

   private:
    std::shared_ptr<mprec_gpu_system> h_;
    int n_ = 0;
    MethodSpec spec_;
    mutable double setup_s_ = 0.0;
};

// solve_system (harness.hpp:87-88, harness.cpp:190-219)
inline SolveOutcome solve_system(const BlockMatrix& a, const Vector& b, const MethodSpec& method, double tol = 1e-8,
                                 int max_iter = 500) {
    const StagePreconditioner p = StagePreconditioner::build(a, b, method);
    SolveOutcome out;
    out.result = p.solve(tol, max_iter);
    out.setup_time_s = p.setup_time_s();
    out.scaling_record = p.scaling_record();
    return out;
}

// ---- sub-solvers ---------------------------------------------------------------
struct ScalarMatrix {  // canonical CSR (scalar_matrix.hpp:20-62)
    int n = 0;
    std::vector<int> row_ptr, col_idx;
    std::vector<double> values;
    mprec_csr c() const { return {n, row_ptr.data(), col_idx.data(), values.data()}; }
    BlockMatrix as_block() const { return BlockMatrix{n, 1, row_ptr, col_idx, values}; }
};

class AMGHierarchy {  // amg.hpp:21-49
   public:
    static AMGHierarchy setup(const ScalarMatrix& a, const AMGParams& p = {}) {
        AMGHierarchy h;
        mprec_gpu_amg* g = nullptr;
        const mprec_csr ca = a.c();
        const mprec_amg_params cp = p.c();
        check(mprec_gpu_amg_create(&ca, &cp, &g));
        h.h_.reset(g, mprec_gpu_amg_destroy);
        h.n_ = a.n;
        return h;
    }
    Vector apply(const Vector& r) const {
        Vector x(n_);
        check(mprec_gpu_amg_apply(h_.get(), r.data(), x.data()));
        return x;
    }
    int n_levels() const {
        int n = 0;
        check(mprec_gpu_amg_n_levels(h_.get(), &n));
        return n;
    }
    mprec_gpu_amg* handle() const { return h_.get(); }

   private:
    std::shared_ptr<mprec_gpu_amg> h_;
    int n_ = 0;
};

class ILU0Factor {  // ilu0.hpp:9-24
   public:
    static ILU0Factor factor(const BlockMatrix& a) {
        ILU0Factor f;
        mprec_gpu_ilu* g = nullptr;
        const mprec_bsr ca = a.c();
        check(mprec_gpu_ilu_create(&ca, &g));
        f.h_.reset(g, mprec_gpu_ilu_destroy);
        f.n_ = a.dim();
        return f;
    }
    static ILU0Factor factor(const ScalarMatrix& a) { return factor(a.as_block()); }
    Vector apply(const Vector& r) const {
        Vector y(n_);
        check(mprec_gpu_ilu_apply(h_.get(), r.data(), y.data()));
        return y;
    }
    mprec_gpu_ilu* handle() const { return h_.get(); }

   private:
    std::shared_ptr<mprec_gpu_ilu> h_;
    int n_ = 0;
};

// gmres (gmres.hpp:41-42) with a matrix operator and an optional device preconditioner
inline SolveResult gmres(const BlockMatrix& a, const Vector& b, const AMGHierarchy* amg = nullptr,
                         const ILU0Factor* ilu = nullptr, const GmresOptions& o = {}) {
    SolveResult r;
    r.x.assign(a.dim(), 0.0);
    mprec_solve_result out{};
    std::vector<double> hist(size_t(std::min(o.max_iter, a.dim())) + 2);
    const mprec_bsr ca = a.c();
    const int kind = amg ? 1 : (ilu ? 2 : 0);
    void* p = amg ? static_cast<void*>(amg->handle()) : (ilu ? static_cast<void*>(ilu->handle()) : nullptr);
    check(mprec_gpu_gmres(&ca, b.data(), kind, p, o.tol, o.max_iter, r.x.data(), &out, hist.data(),
                          int(hist.size())));
    r.iterations = out.iterations;
    r.converged = out.converged != 0;
    r.breakdown = out.breakdown != 0;
    r.residual_history.assign(hist.begin(), hist.begin() + out.history_len);
    r.final_true_residual = out.final_true_residual;
    r.wall_time_s = out.solve_s;
    return r;
}

}  // namespace gpu
}  // namespace mprec
