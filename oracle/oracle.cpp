// oracle.cpp -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
// See oracle.hpp.  Build with -ffp-contract=off: every a*b+c below is a rounded
// multiply followed by a rounded add, as the reference's scalar loops are.
#include "oracle.hpp"

#include <map>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <queue>

namespace oracle {

// ===================================================================== Csr ==

// scalar_matrix.cpp:8-35 (stable sort keeps duplicate summation deterministic)
Csr Csr::from_triplets(int rows, int cols, std::vector<Triplet> t) {
    if (rows < 0 || cols < 0) throw Error(DIMENSION, "negative matrix dimension");
    for (const auto& e : t)
        if (e.row < 0 || e.row >= rows || e.col < 0 || e.col >= cols)
            throw Error(INDEX, "triplet index out of range");
    std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    Csr m;
    m.rows = rows;
    m.cols = cols;
    m.rp.assign(rows + 1, 0);
    m.ci.reserve(t.size());
    m.v.reserve(t.size());
    size_t i = 0;
    for (int r = 0; r < rows; ++r) {
        while (i < t.size() && t[i].row == r) {
            const int c = t[i].col;
            double v = 0.0;
            while (i < t.size() && t[i].row == r && t[i].col == c) {
                v += t[i].value;
                ++i;
            }
            m.ci.push_back(c);
            m.v.push_back(v);
        }
        m.rp[r + 1] = int(m.ci.size());
    }
    return m;
}

double Csr::coeff(int i, int j) const {
    auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
    auto it = std::lower_bound(b, e, j);
    if (it != e && *it == j) return v[it - ci.begin()];
    return 0.0;
}

double* Csr::find(int i, int j) {
    auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
    auto it = std::lower_bound(b, e, j);
    if (it != e && *it == j) return &v[it - ci.begin()];
    return nullptr;
}

// scalar_matrix.cpp:79-88
Vec Csr::apply(const Vec& x) const {
    if (int(x.size()) != cols) throw Error(DIMENSION, "spmv length mismatch");
    Vec y(rows, 0.0);
    for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) acc += v[k] * x[ci[k]];
        y[i] = acc;
    }
    return y;
}

// scalar_matrix.cpp:98-105
Csr Csr::transpose() const {
    std::vector<Triplet> t;
    t.reserve(ci.size());
    for (int i = 0; i < rows; ++i)
        for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({ci[k], i, v[k]});
    return from_triplets(cols, rows, std::move(t));
}

// scalar_matrix.cpp:120-151 (Gustavson, dense accumulator, symbolic zeros kept)
Csr Csr::multiply(const Csr& a, const Csr& b) {
    if (a.cols != b.rows) throw Error(DIMENSION, "sparse multiply dimension mismatch");
    Csr c;
    c.rows = a.rows;
    c.cols = b.cols;
    c.rp.assign(a.rows + 1, 0);
    std::vector<double> work(b.cols, 0.0);
    std::vector<char> mark(b.cols, 0);
    std::vector<int> touched;
    touched.reserve(64);
    for (int i = 0; i < a.rows; ++i) {
        touched.clear();
        for (int ka = a.rp[i]; ka < a.rp[i + 1]; ++ka) {
            const int j = a.ci[ka];
            const double av = a.v[ka];
            for (int kb = b.rp[j]; kb < b.rp[j + 1]; ++kb) {
                const int col = b.ci[kb];
                if (!mark[col]) {
                    mark[col] = 1;
                    touched.push_back(col);
                }
                work[col] += av * b.v[kb];
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int col : touched) {
            mark[col] = 0;
            c.ci.push_back(col);
            c.v.push_back(work[col]);
            work[col] = 0.0;
        }
        c.rp[i + 1] = int(c.ci.size());
    }
    return c;
}

// ===================================================================== Bsr ==

Bsr Bsr::create(int n_cells, int nb, const int* rp, const int* ci, const double* val, int missing_diag_code) {
    if (n_cells < 1) throw Error(DIMENSION, "layout needs at least one cell");
    if (nb < 1) throw Error(DIMENSION, "block size must be >= 1");
    if (rp[0] != 0) throw Error(INDEX, "row_ptr[0] must be 0");
    Bsr m;
    m.nc = n_cells;
    m.nb = nb;
    m.rp.assign(rp, rp + n_cells + 1);
    const int nnzb = rp[n_cells];
    m.ci.assign(ci, ci + nnzb);
    m.val.assign(val, val + int64_t(nnzb) * nb * nb);
    m.dpos.assign(n_cells, -1);
    for (int c = 0; c < n_cells; ++c) {
        if (rp[c + 1] < rp[c]) throw Error(INDEX, "row_ptr not monotone");
        for (int k = rp[c]; k < rp[c + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= n_cells) throw Error(INDEX, "block column out of range");
            if (k > rp[c] && ci[k] <= ci[k - 1]) throw Error(INDEX, "block columns not sorted");
            if (ci[k] == c) m.dpos[c] = k;
        }
        if (m.dpos[c] < 0) {
            if (missing_diag_code == SETUP) throw Error(SETUP, "ILU(0): structurally absent diagonal");
            throw Error(DIMENSION, "diagonal block missing in cell " + std::to_string(c), c);
        }
    }
    return m;
}

int Bsr::find_block(int row, int col) const {
    auto b = ci.begin() + rp[row], e = ci.begin() + rp[row + 1];
    auto it = std::lower_bound(b, e, col);
    if (it != e && *it == col) return int(it - ci.begin());
    return -1;
}

// block_matrix.cpp:103-114.
Vec Bsr::apply_block(const Vec& x) const {
    if (int64_t(x.size()) != int64_t(dim())) throw Error(DIMENSION, "spmv length mismatch");
    // yc += B_k * x_k: the block product is summed over the block's columns
    // from the first term into a temporary, then added (the product convention
    // of the Eigen call sites, oracle/eigen_shim/shim.hpp).
    Vec y(size_t(dim()), 0.0);
    for (int c = 0; c < nc; ++c) {
        double* yc = &y[size_t(c) * nb];
        for (int k = rp[c]; k < rp[c + 1]; ++k) {
            const double* xs = &x[size_t(ci[k]) * nb];
            for (int r = 0; r < nb; ++r) {
                double acc = at(k, r, 0) * xs[0];
                for (int col = 1; col < nb; ++col) acc += at(k, r, col) * xs[col];
                yc[r] += acc;
            }
        }
    }
    return y;
}

// ScalarMatrix::apply on the flattening: per scalar row, columns ascending.
Vec Bsr::apply_flat(const Vec& x) const {
    if (int64_t(x.size()) != int64_t(dim())) throw Error(DIMENSION, "spmv length mismatch");
    Vec y(size_t(dim()), 0.0);
    for (int c = 0; c < nc; ++c)
        for (int r = 0; r < nb; ++r) {
            double acc = 0.0;
            for (int k = rp[c]; k < rp[c + 1]; ++k) {
                const double* xs = &x[size_t(ci[k]) * nb];
                for (int col = 0; col < nb; ++col) acc += at(k, r, col) * xs[col];
            }
            y[size_t(c) * nb + r] = acc;
        }
    return y;
}

// block_matrix.cpp:116-128 (the triplets are already in canonical order)
Csr Bsr::to_scalar() const {
    Csr m;
    m.rows = m.cols = dim();
    m.rp.assign(dim() + 1, 0);
    const int64_t nnz = int64_t(rp[nc]) * nb * nb;
    m.ci.reserve(nnz);
    m.v.reserve(nnz);
    for (int c = 0; c < nc; ++c)
        for (int r = 0; r < nb; ++r) {
            for (int k = rp[c]; k < rp[c + 1]; ++k)
                for (int col = 0; col < nb; ++col) {
                    m.ci.push_back(ci[k] * nb + col);
                    m.v.push_back(at(k, r, col));
                }
            m.rp[c * nb + r + 1] = int(m.ci.size());
        }
    return m;
}

// block_matrix.cpp:142-170 for a single-field selection (P or T): all stored
// entries kept, pattern = block pattern.
Csr Bsr::extract_field(int local) const {
    Csr m;
    m.rows = m.cols = nc;
    m.rp.assign(rp.begin(), rp.end());
    m.ci.assign(ci.begin(), ci.end());
    m.v.resize(ci.size());
    for (int k = 0; k < rp[nc]; ++k) m.v[k] = at(k, local, local);
    return m;
}

// extract_submatrix({P,T},{P,T}) (block_matrix.cpp:142-170): rows/cols in cell
// order then (P, T); every stored entry kept.
static Csr extract_pt(const Bsr& a) {
    const int P = a.nb - 2, T = a.nb - 1;
    Csr m;
    m.rows = m.cols = 2 * a.nc;
    m.rp.assign(2 * a.nc + 1, 0);
    for (int c = 0; c < a.nc; ++c)
        for (int r = 0; r < 2; ++r) {
            const int fr = r == 0 ? P : T;
            for (int k = a.rp[c]; k < a.rp[c + 1]; ++k)
                for (int q = 0; q < 2; ++q) {
                    m.ci.push_back(2 * a.ci[k] + q);
                    m.v.push_back(a.at(k, fr, q == 0 ? P : T));
                }
            m.rp[2 * c + r + 1] = int(m.ci.size());
        }
    return m;
}

// ================================================================ DenseLU ==
// Eigen::PartialPivLU unblocked path (partial_lu_impl::unblocked_lu).
void DenseLU::factor(const double* a, int n_) {
    n = n_;
    lu.assign(a, a + size_t(n) * n);
    perm.resize(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    auto A = [&](int i, int j) -> double& { return lu[size_t(j) * n + i]; };
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(A(k, k));
        for (int i = k + 1; i < n; ++i)
            if (std::abs(A(i, k)) > best) {
                best = std::abs(A(i, k));
                p = i;
            }
        if (best != 0.0) {
            if (p != k) {
                for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
                std::swap(perm[k], perm[p]);
            }
            const double d = A(k, k);
            for (int i = k + 1; i < n; ++i) A(i, k) = A(i, k) / d;
        }
        for (int j = k + 1; j < n; ++j) {
            const double ukj = A(k, j);
            for (int i = k + 1; i < n; ++i) A(i, j) = A(i, j) - A(i, k) * ukj;
        }
    }
}

bool DenseLU::pivots_ok(double tol, int* bad) const {
    for (int i = 0; i < n; ++i)
        if (std::abs(lu[size_t(i) * n + i]) <= tol) {
            if (bad) *bad = i;
            return false;
        }
    return true;
}

void DenseLU::solve_inplace(double* x) const {
    std::vector<double> t(n);
    for (int i = 0; i < n; ++i) t[i] = x[perm[i]];
    for (int j = 0; j < n; ++j) {
        const double xj = t[j];
        for (int i = j + 1; i < n; ++i) t[i] = t[i] - lu[size_t(j) * n + i] * xj;
    }
    for (int j = n - 1; j >= 0; --j) {
        t[j] = t[j] / lu[size_t(j) * n + j];
        const double xj = t[j];
        for (int i = 0; i < j; ++i) t[i] = t[i] - lu[size_t(j) * n + i] * xj;
    }
    for (int i = 0; i < n; ++i) x[i] = t[i];
}

Vec DenseLU::inverse() const {
    Vec inv(size_t(n) * n, 0.0);
    for (int j = 0; j < n; ++j) {
        double* col = &inv[size_t(j) * n];
        col[j] = 1.0;
        solve_inplace(col);
    }
    return inv;
}

// dense_factor.cpp:7-19
DenseFactor DenseFactor::factor(const Csr& a) {
    if (a.rows != a.cols) throw Error(DIMENSION, "dense factor needs a square matrix");
    const int n = a.rows;
    Vec d(size_t(n) * n, 0.0);
    double scale = 0.0;
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) d[size_t(a.ci[k]) * n + i] = a.v[k];
    for (double x : d) scale = std::max(scale, std::abs(x));
    DenseFactor f;
    f.lu.factor(d.data(), n);
    int bad = -1;
    if (n > 0 && !f.lu.pivots_ok(1e-14 * scale, &bad))
        throw Error(SINGULAR_BLOCK, "singular dense-factor pivot block in cell " + std::to_string(bad), bad);
    return f;
}

Vec DenseFactor::solve(const Vec& r) const {
    if (int(r.size()) != lu.n) throw Error(DIMENSION, "dense solve length mismatch");
    Vec x = r;
    lu.solve_inplace(x.data());
    return x;
}

// ================================================================== ILU(0) ==

// ilu0.cpp:7-39, line for line
Ilu0Scalar Ilu0Scalar::factor(const Csr& a) {
    if (a.rows != a.cols) throw Error(DIMENSION, "ILU(0) needs a square matrix");
    const int n = a.rows;
    Ilu0Scalar f;
    f.lu = a;
    f.diag.assign(n, -1);
    const auto& rp = f.lu.rp;
    const auto& ci = f.lu.ci;
    auto& v = f.lu.v;
    for (int i = 0; i < n; ++i)
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) f.diag[i] = k;
    for (int i = 0; i < n; ++i)
        if (f.diag[i] < 0) throw Error(SETUP, "ILU(0): structurally absent diagonal");
    for (int i = 1; i < n; ++i) {
        for (int kk = rp[i]; kk < rp[i + 1] && ci[kk] < i; ++kk) {
            const int k = ci[kk];
            const double piv = v[f.diag[k]];
            if (piv == 0.0) throw Error(ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(k), k);
            const double factor = v[kk] / piv;
            v[kk] = factor;
            for (int kj = f.diag[k] + 1; kj < rp[k + 1]; ++kj) {
                const int j = ci[kj];
                if (double* p = f.lu.find(i, j)) *p -= factor * v[kj];
            }
        }
        if (v[f.diag[i]] == 0.0) throw Error(ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(i), i);
    }
    return f;
}

// ilu0.cpp:41-59
Vec Ilu0Scalar::apply(const Vec& r) const {
    const int n = lu.rows;
    if (int(r.size()) != n) throw Error(DIMENSION, "ILU(0) apply length mismatch");
    Vec y = r;
    for (int i = 0; i < n; ++i) {
        double acc = y[i];
        for (int k = lu.rp[i]; k < lu.rp[i + 1] && lu.ci[k] < i; ++k) acc -= lu.v[k] * y[lu.ci[k]];
        y[i] = acc;
    }
    for (int i = n - 1; i >= 0; --i) {
        double acc = y[i];
        for (int k = diag[i] + 1; k < lu.rp[i + 1]; ++k) acc -= lu.v[k] * y[lu.ci[k]];
        y[i] = acc / lu.v[diag[i]];
    }
    return y;
}

// The scalar IKJ elimination of ilu0.cpp:23-37 executed on the block pattern.
// Scalar row i = (I, r).  Its k-sequence is: every column of the lower blocks
// (I,K), K ascending, in-block column ascending; then the diagonal-block
// columns r' < r.  Rows of one block row only interact through the diagonal
// block, so the lower-block phase may be run for all r together; every entry
// still sees exactly the reference's update sequence (k ascending).
Ilu0Block Ilu0Block::factor(const Bsr& a) {
    Ilu0Block f;
    f.lu = a;
    Bsr& m = f.lu;
    const int nb = m.nb;
    for (int I = 0; I < m.nc; ++I) {
        for (int k = m.rp[I]; k < m.rp[I + 1] && m.ci[k] < I; ++k) {
            const int K = m.ci[k];
            const int dK = m.dpos[K];
            for (int rk = 0; rk < nb; ++rk) {
                const double piv = m.at(dK, rk, rk);
                const int krow = K * nb + rk;
                if (piv == 0.0)
                    throw Error(ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(krow), krow);
                for (int r = 0; r < nb; ++r) {
                    const double fac = m.at(k, r, rk) / piv;
                    m.at(k, r, rk) = fac;
                    for (int c = rk + 1; c < nb; ++c) m.at(k, r, c) -= fac * m.at(dK, rk, c);
                    for (int kj = dK + 1; kj < m.rp[K + 1]; ++kj) {
                        const int kI = m.find_block(I, m.ci[kj]);
                        if (kI < 0) continue;
                        for (int c = 0; c < nb; ++c) m.at(kI, r, c) -= fac * m.at(kj, rk, c);
                    }
                }
            }
        }
        const int d = m.dpos[I];
        for (int r = 0; r < nb; ++r) {
            for (int rp_ = 0; rp_ < r; ++rp_) {
                const double piv = m.at(d, rp_, rp_);
                const int krow = I * nb + rp_;
                if (piv == 0.0)
                    throw Error(ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(krow), krow);
                const double fac = m.at(d, r, rp_) / piv;
                m.at(d, r, rp_) = fac;
                for (int c = rp_ + 1; c < nb; ++c) m.at(d, r, c) -= fac * m.at(d, rp_, c);
                for (int kb = d + 1; kb < m.rp[I + 1]; ++kb)
                    for (int c = 0; c < nb; ++c) m.at(kb, r, c) -= fac * m.at(kb, rp_, c);
            }
            const int i = I * nb + r;
            if (i >= 1 && m.at(d, r, r) == 0.0)
                throw Error(ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(i), i);
        }
    }
    return f;
}

Vec Ilu0Block::apply(const Vec& rhs) const {
    const Bsr& m = lu;
    const int nb = m.nb;
    if (int64_t(rhs.size()) != int64_t(m.dim())) throw Error(DIMENSION, "ILU(0) apply length mismatch");
    Vec y = rhs;
    for (int I = 0; I < m.nc; ++I) {
        const int d = m.dpos[I];
        for (int r = 0; r < nb; ++r) {
            double acc = y[size_t(I) * nb + r];
            for (int k = m.rp[I]; k < d; ++k) {
                const double* ys = &y[size_t(m.ci[k]) * nb];
                for (int c = 0; c < nb; ++c) acc -= m.at(k, r, c) * ys[c];
            }
            for (int c = 0; c < r; ++c) acc -= m.at(d, r, c) * y[size_t(I) * nb + c];
            y[size_t(I) * nb + r] = acc;
        }
    }
    for (int I = m.nc - 1; I >= 0; --I) {
        const int d = m.dpos[I];
        for (int r = nb - 1; r >= 0; --r) {
            double acc = y[size_t(I) * nb + r];
            for (int c = r + 1; c < nb; ++c) acc -= m.at(d, r, c) * y[size_t(I) * nb + c];
            for (int k = d + 1; k < m.rp[I + 1]; ++k) {
                const double* ys = &y[size_t(m.ci[k]) * nb];
                for (int c = 0; c < nb; ++c) acc -= m.at(k, r, c) * ys[c];
            }
            y[size_t(I) * nb + r] = acc / m.at(d, r, r);
        }
    }
    return y;
}

// ===================================================================== AMG ==
namespace {

enum class Mark : char { Undecided, Coarse, Fine };

// amg.cpp:14-22
std::vector<int> diag_positions(const Csr& a) {
    std::vector<int> d(a.rows, -1);
    for (int i = 0; i < a.rows; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) d[i] = k;
    for (int i = 0; i < a.rows; ++i)
        if (d[i] < 0) throw Error(SETUP, "AMG: structurally absent diagonal");
    return d;
}

// amg.cpp:25-43
void sym_gauss_seidel(const Csr& a, const std::vector<int>& diag, Vec& x, const Vec& b) {
    const int n = a.rows;
    for (int i = 0; i < n; ++i) {
        double acc = b[i];
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] != i) acc -= a.v[k] * x[a.ci[k]];
        x[i] = acc / a.v[diag[i]];
    }
    for (int i = n - 1; i >= 0; --i) {
        double acc = b[i];
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] != i) acc -= a.v[k] * x[a.ci[k]];
        x[i] = acc / a.v[diag[i]];
    }
}

}  // namespace

// amg.cpp:47-186
CoarseningResult rs_coarsen(const Csr& a, double theta) {
    const int n = a.rows;
    const auto& rp = a.rp;
    const auto& ci = a.ci;
    const auto& av = a.v;

    std::vector<std::vector<int>> strong(n), strong_t(n);
    for (int i = 0; i < n; ++i) {
        double m = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] != i) m = std::max(m, -av[k]);
        if (m <= 0.0) continue;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (j != i && -av[k] >= theta * m) {
                strong[i].push_back(j);
                strong_t[j].push_back(i);
            }
        }
    }

    std::vector<Mark> mark(n, Mark::Undecided);
    std::vector<int> lambda(n);
    using Entry = std::pair<int, int>;
    std::priority_queue<Entry> heap;
    int n_undecided = 0;
    for (int i = 0; i < n; ++i) {
        lambda[i] = int(strong_t[i].size());
        if (strong[i].empty() && strong_t[i].empty()) {
            mark[i] = Mark::Fine;
        } else {
            heap.emplace(lambda[i], -i);
            ++n_undecided;
        }
    }
    while (n_undecided > 0) {
        int i = -1;
        while (!heap.empty()) {
            auto [lam, neg] = heap.top();
            heap.pop();
            const int cand = -neg;
            if (mark[cand] == Mark::Undecided && lam == lambda[cand]) {
                i = cand;
                break;
            }
        }
        if (i < 0) break;
        mark[i] = Mark::Coarse;
        --n_undecided;
        for (int j : strong_t[i]) {
            if (mark[j] != Mark::Undecided) continue;
            mark[j] = Mark::Fine;
            --n_undecided;
            for (int k : strong[j])
                if (mark[k] == Mark::Undecided) {
                    ++lambda[k];
                    heap.emplace(lambda[k], -k);
                }
        }
    }

    std::vector<char> in_ci(n, 0);
    for (int i = 0; i < n; ++i) {
        if (mark[i] != Mark::Fine || strong[i].empty()) continue;
        for (int j : strong[i])
            if (mark[j] == Mark::Coarse) in_ci[j] = 1;
        for (int j : strong[i]) {
            if (mark[j] != Mark::Fine) continue;
            bool shared = false;
            for (int k : strong[j])
                if (in_ci[k]) {
                    shared = true;
                    break;
                }
            if (!shared) {
                mark[j] = Mark::Coarse;
                in_ci[j] = 1;
            }
        }
        for (int j : strong[i]) in_ci[j] = 0;
        in_ci[i] = 0;
    }
    for (int i = 0; i < n; ++i) {
        if (mark[i] != Mark::Fine || strong[i].empty()) continue;
        bool has_c = false;
        for (int j : strong[i])
            if (mark[j] == Mark::Coarse) has_c = true;
        if (!has_c) mark[i] = Mark::Coarse;
    }

    std::vector<int> coarse_id(n, -1);
    int nc = 0;
    for (int i = 0; i < n; ++i)
        if (mark[i] == Mark::Coarse) coarse_id[i] = nc++;

    std::vector<Triplet> pt;
    for (int i = 0; i < n; ++i) {
        if (mark[i] == Mark::Coarse) {
            pt.push_back({i, coarse_id[i], 1.0});
            continue;
        }
        if (strong[i].empty()) continue;
        double sum_neg_all = 0.0, sum_pos_all = 0.0, sum_neg_c = 0.0, sum_pos_c = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (j == i) continue;
            (av[k] < 0.0 ? sum_neg_all : sum_pos_all) += av[k];
            if (coarse_id[j] >= 0 && std::find(strong[i].begin(), strong[i].end(), j) != strong[i].end())
                (av[k] < 0.0 ? sum_neg_c : sum_pos_c) += av[k];
        }
        double aii = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) aii = av[k];
        if (sum_pos_c == 0.0) aii += sum_pos_all;
        const double alpha = sum_neg_c != 0.0 ? sum_neg_all / sum_neg_c : 0.0;
        const double beta = sum_pos_c != 0.0 ? sum_pos_all / sum_pos_c : 0.0;
        for (int j : strong[i]) {
            if (coarse_id[j] < 0) continue;
            const double aij = a.coeff(i, j);
            const double w = aij < 0.0 ? -alpha * aij / aii : -beta * aij / aii;
            if (w != 0.0) pt.push_back({i, coarse_id[j], w});
        }
    }

    CoarseningResult res;
    res.is_coarse.assign(n, 0);
    for (int i = 0; i < n; ++i) res.is_coarse[i] = coarse_id[i] >= 0 ? 1 : 0;
    res.p = Csr::from_triplets(n, nc, std::move(pt));
    return res;
}

// amg.cpp:188-214
AMGHierarchy AMGHierarchy::setup(const Csr& a, const AMGParams& params) {
    if (a.rows != a.cols) throw Error(DIMENSION, "AMG needs a square matrix");
    AMGHierarchy h;
    h.params = params;
    Level finest;
    finest.a = a;
    finest.diag_pos = diag_positions(a);
    h.levels.push_back(std::move(finest));
    while (h.levels.back().a.rows > params.max_coarse_size && int(h.levels.size()) < params.max_levels) {
        const Csr& af = h.levels.back().a;
        CoarseningResult cr = rs_coarsen(af, params.strength_threshold);
        const int nc = cr.p.cols;
        if (nc == 0) break;
        if (nc > int(0.95 * af.rows))
            throw Error(SETUP, "AMG coarsening stagnated at size " + std::to_string(af.rows));
        h.levels.back().cf = cr.is_coarse;
        Level lvl;
        lvl.p = std::move(cr.p);
        lvl.r = lvl.p.transpose();
        lvl.a = Csr::multiply(lvl.r, Csr::multiply(af, lvl.p));
        lvl.diag_pos = diag_positions(lvl.a);
        h.levels.push_back(std::move(lvl));
    }
    h.coarse = DenseFactor::factor(h.levels.back().a);
    return h;
}

// amg.cpp:216-231
void AMGHierarchy::cycle(int l, const Vec& r, Vec& x) const {
    const Level& lvl = levels[l];
    if (l == n_levels() - 1) {
        x = coarse.solve(r);
        return;
    }
    std::fill(x.begin(), x.end(), 0.0);
    sym_gauss_seidel(lvl.a, lvl.diag_pos, x, r);
    const Vec ax = lvl.a.apply(x);
    Vec resid(r.size());
    for (size_t i = 0; i < r.size(); ++i) resid[i] = r[i] - ax[i];
    const Level& next = levels[l + 1];
    const Vec rc = next.r.apply(resid);
    Vec ec(rc.size(), 0.0);
    cycle(l + 1, rc, ec);
    const Vec pe = next.p.apply(ec);
    for (size_t i = 0; i < x.size(); ++i) x[i] = x[i] + pe[i];
    sym_gauss_seidel(lvl.a, lvl.diag_pos, x, r);
}

// amg.cpp:233-238
Vec AMGHierarchy::apply(const Vec& r) const {
    if (int(r.size()) != levels.front().a.rows) throw Error(DIMENSION, "AMG apply length mismatch");
    Vec x(r.size(), 0.0);
    cycle(0, r, x);
    return x;
}

// ================================================================= scaling ==
namespace {

// inverted_copy of one square block (block_matrix.cpp:10-30); column-major.
bool invert_block(const Vec& b, int m, Vec& inv) {
    double scale = 0.0;
    for (double x : b) scale = std::max(scale, std::abs(x));
    const double tol = 1e-12 * scale;
    DenseLU lu;
    lu.factor(b.data(), m);
    if (!lu.pivots_ok(tol, nullptr)) return false;
    inv = lu.inverse();
    return true;
}

// W = L * R for small column-major matrices, k-sum sequential from the first term
// (Eigen lazy product restated).
Vec small_mul(const Vec& l, int rows, int inner, const Vec& r, int cols) {
    Vec w(size_t(rows) * cols, 0.0);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            double acc = l[size_t(0) * rows + i] * r[size_t(j) * inner + 0];
            for (int k = 1; k < inner; ++k) acc += l[size_t(k) * rows + i] * r[size_t(j) * inner + k];
            w[size_t(j) * rows + i] = acc;
        }
    return w;
}

// BlockMatrix::row_combine (block_matrix.cpp:201-221) + scale_rhs (scaling.cpp:49-61)
// for one cell: rows tl -= W * rows sl, W column-major (|tl| x |sl|).
void combine_cell(Bsr& a, Vec& b, int c, const std::vector<int>& tl, const std::vector<int>& sl,
                  const Vec& w) {
    const int nb = a.nb, nt = int(tl.size()), ns = int(sl.size());
    if (nt == 0 || ns == 0) return;
    std::vector<double> upd(nt);
    for (int k = a.rp[c]; k < a.rp[c + 1]; ++k)
        for (int col = 0; col < nb; ++col) {
            for (int i = 0; i < nt; ++i) {
                double acc = w[size_t(0) * nt + i] * a.at(k, sl[0], col);
                for (int s = 1; s < ns; ++s) acc += w[size_t(s) * nt + i] * a.at(k, sl[s], col);
                upd[i] = acc;
            }
            for (int i = 0; i < nt; ++i) a.at(k, tl[i], col) -= upd[i];
        }
    const size_t off = size_t(c) * nb;
    for (int i = 0; i < nt; ++i) {
        double acc = w[size_t(0) * nt + i] * b[off + sl[0]];
        for (int s = 1; s < ns; ++s) acc += w[size_t(s) * nt + i] * b[off + sl[s]];
        upd[i] = acc;
    }
    for (int i = 0; i < nt; ++i) b[off + tl[i]] -= upd[i];
}

// scaling_factors (scaling.cpp:31-46) for target fields tl, source fields sl,
// evaluated on `a`: D_ts is the full cell block, D_ss the block or (scalar_diag,
// DiagMode::Scalar, block_matrix.cpp:186-193) its diagonal.  Throws
// SingularBlock(cell, what) at the first cell (ascending) whose D_ss fails the
// pivot check.
std::vector<Vec> scaling_factors(const Bsr& a, const std::vector<int>& tl, const std::vector<int>& sl,
                                 const char* what, bool scalar_diag) {
    const int nt = int(tl.size()), ns = int(sl.size());
    std::vector<Vec> w(a.nc);
    if (ns == 0) {
        for (auto& x : w) x.clear();
        return w;
    }
    std::vector<Vec> inv(a.nc);
    for (int c = 0; c < a.nc; ++c) {
        const int d = a.dpos[c];
        Vec dss(size_t(ns) * ns);
        for (int j = 0; j < ns; ++j)
            for (int i = 0; i < ns; ++i) dss[size_t(j) * ns + i] = (scalar_diag && i != j) ? 0.0 : a.at(d, sl[i], sl[j]);
        if (!invert_block(dss, ns, inv[c]))
            throw Error(SINGULAR_BLOCK, std::string("singular ") + what + " block in cell " + std::to_string(c), c);
    }
    for (int c = 0; c < a.nc; ++c) {
        const int d = a.dpos[c];
        Vec dts(size_t(nt) * ns);
        for (int j = 0; j < ns; ++j)
            for (int i = 0; i < nt; ++i) dts[size_t(j) * nt + i] = a.at(d, tl[i], sl[j]);
        w[c] = small_mul(dts, nt, ns, inv[c], ns);
    }
    return w;
}

}  // namespace

// scaling.cpp:73-88 (CPR) / :107-147 (CPTR3) / :149-158 (dispatch)
ScaledSystem left_scale(const Bsr& a, const Vec& b, Method m, const ScalingOptions& o) {
    if (int64_t(b.size()) != int64_t(a.dim())) throw Error(DIMENSION, "rhs length mismatch");
    if (a.nb < 2 && m != Method::Ilu0) throw Error(DIMENSION, "CPR/CPTR3 need P and T unknowns (nb >= 2)");
    ScaledSystem s;
    s.method = m;
    s.a_bar = a;
    s.b_bar = b;
    const int nb = a.nb, ns = nb - 2, P = nb - 2, T = nb - 1;
    if (m == Method::Ilu0) return s;
    std::vector<int> S;
    for (int k = 0; k < ns; ++k) S.push_back(k);
    if (m == Method::CptrDirect) {  // scaling.cpp:90-105
        const auto w = scaling_factors(a, {P, T}, S, "D_ss", o.scalar_diag);
        for (int c = 0; c < a.nc; ++c) combine_cell(s.a_bar, s.b_bar, c, {P, T}, S, w[c]);
        s.scaling_record.push_back("D_es*D_ss^-1");
        s.b_ee = extract_pt(s.a_bar);
        return s;
    }
    if (m == Method::Cpr || m == Method::CprDirect) {
        std::vector<int> h = S;
        h.push_back(T);
        const auto w = scaling_factors(a, {P}, h, "D_hh", o.scalar_diag);
        for (int c = 0; c < a.nc; ++c) combine_cell(s.a_bar, s.b_bar, c, {P}, h, w[c]);
        s.scaling_record.push_back("D_Ph*D_hh^-1");
        s.b_pp = s.a_bar.extract_field(P);
        return s;
    }
    if (m == Method::Cptr3 || m == Method::Cptr3Direct) {
        const auto w1 = scaling_factors(a, {P, T}, S, "D_ss", o.scalar_diag);
        for (int c = 0; c < a.nc; ++c) combine_cell(s.a_bar, s.b_bar, c, {P, T}, S, w1[c]);
        s.scaling_record.push_back("[D_Ps;D_Ts]*D_ss^-1");
        // second scaling: D_Tp (once-scaled) * D_PP^-1, D_PP of the once-scaled
        // matrix or, with second_scaling_from_original, of A (scaling.cpp:126)
        const Bsr& pp_source = o.second_scaling_from_original ? a : s.a_bar;
        std::vector<Vec> w2(a.nc);
        for (int c = 0; c < a.nc; ++c) {
            const int d = s.a_bar.dpos[c];
            Vec inv;
            if (!invert_block(Vec{pp_source.at(pp_source.dpos[c], P, P)}, 1, inv))
                throw Error(SINGULAR_BLOCK, "singular D_PP block in cell " + std::to_string(c), c);
            w2[c] = Vec{s.a_bar.at(d, T, P) * inv[0]};
        }
        for (int c = 0; c < a.nc; ++c) combine_cell(s.a_bar, s.b_bar, c, {T}, {P}, w2[c]);
        s.scaling_record.push_back("D_Tp*D_PP^-1");
        s.b_pp = s.a_bar.extract_field(P);
        s.c_tt = s.a_bar.extract_field(T);
        return s;
    }
    throw Error(CONFIG, "unsupported method");
}

// ================================================================== stages ==

// stages.cpp:25-34
Vec Stage::apply(const Vec& r, const Ilu0Block& ilu) const {
    if (kind == ILU) return ilu.apply(r);
    Vec y(r.size(), 0.0);
    if (scope.empty()) return y;
    Vec sub(scope.size());
    for (size_t i = 0; i < scope.size(); ++i) sub[i] = r[scope[i]];
    const Vec sol = kind == AMG ? amg->apply(sub) : direct->solve(sub);
    for (size_t i = 0; i < scope.size(); ++i) y[scope[i]] = sol[i];
    return y;
}

Vec StagePreconditioner::apply_stage(int i, const Vec& r) const { return stages[i].apply(r, ilu); }

// stages.cpp:36-59
Vec StagePreconditioner::apply(const Vec& r) const {
    const size_t n = r.size();
    if (stages.size() == 1) return stages[0].apply(r, ilu);
    if (stages.size() == 2) {
        const Vec x = stages[0].apply(r, ilu);
        const Vec ax = a_bar->apply_flat(x);
        Vec z(n);
        for (size_t i = 0; i < n; ++i) z[i] = r[i] - ax[i];
        const Vec w = stages[1].apply(z, ilu);
        Vec y(n);
        for (size_t i = 0; i < n; ++i) y[i] = x[i] + w[i];
        return y;
    }
    if (stages.size() == 3) {
        const Vec x = stages[0].apply(r, ilu);
        const Vec ax = a_bar->apply_flat(x);
        Vec z(n);
        for (size_t i = 0; i < n; ++i) z[i] = r[i] - ax[i];
        const Vec v = stages[1].apply(z, ilu);
        const Vec av = a_bar->apply_flat(v);
        Vec u(n);
        for (size_t i = 0; i < n; ++i) u[i] = z[i] - av[i];
        const Vec w = stages[2].apply(u, ilu);
        Vec y(n);
        for (size_t i = 0; i < n; ++i) y[i] = (x[i] + v[i]) + w[i];
        return y;
    }
    throw Error(SETUP, "unsupported stage count");
}

namespace {
std::vector<int> field_scope(int nc, int nb, int local) {
    std::vector<int> s(nc);
    for (int c = 0; c < nc; ++c) s[c] = c * nb + local;
    return s;
}
}  // namespace

// stages.cpp:63-138 (AMG sub-solvers; ILU(0) on the flattened scaled matrix)
StagePreconditioner build_preconditioner(const ScaledSystem& sc, const AMGParams& p) {
    StagePreconditioner pc;
    pc.method = sc.method;
    pc.a_bar = &sc.a_bar;
    const int nc = sc.a_bar.nc, nb = sc.a_bar.nb;
    const bool direct = sc.method == Method::CprDirect || sc.method == Method::CptrDirect ||
                        sc.method == Method::Cptr3Direct;
    // make_scoped (stages.cpp:67-76)
    auto scoped = [&](const Csr& sub, std::vector<int> scope) {
        Stage s;
        s.scope = std::move(scope);
        if (direct) {
            s.kind = Stage::DIRECT;
            s.direct = std::make_shared<DenseFactor>(DenseFactor::factor(sub));
        } else {
            s.kind = Stage::AMG;
            s.amg = std::make_shared<AMGHierarchy>(AMGHierarchy::setup(sub, p));
        }
        return s;
    };
    if (sc.method == Method::Cpr || sc.method == Method::CprDirect) {
        pc.stages.push_back(scoped(sc.b_pp, field_scope(nc, nb, nb - 2)));
    } else if (sc.method == Method::Cptr3 || sc.method == Method::Cptr3Direct) {
        pc.stages.push_back(scoped(sc.c_tt, field_scope(nc, nb, nb - 1)));
        pc.stages.push_back(scoped(sc.b_pp, field_scope(nc, nb, nb - 2)));
    } else if (sc.method == Method::CptrDirect) {
        std::vector<int> e;
        for (int c = 0; c < nc; ++c) {
            e.push_back(c * nb + nb - 2);
            e.push_back(c * nb + nb - 1);
        }
        pc.stages.push_back(scoped(sc.b_ee, e));
    }
    pc.ilu = Ilu0Block::factor(sc.a_bar);
    Stage ilu;
    ilu.kind = Stage::ILU;
    pc.stages.push_back(ilu);
    return pc;
}

// =================================================================== GMRES ==

double vdot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
double vnorm(const Vec& x) { return std::sqrt(vdot(x, x)); }

// gmres.cpp:8-106
SolveResult gmres(int n, const Op& a, const Vec& b, const Op& m, const GmresOptions& opts) {
    if (int(b.size()) != n) throw Error(DIMENSION, "gmres: rhs length mismatch");
    if (opts.tol <= 0.0) throw Error(DIMENSION, "gmres: tolerance must be positive");
    const auto t0 = std::chrono::steady_clock::now();
    SolveResult res;
    res.x.assign(n, 0.0);
    const double bnorm = vnorm(b);
    if (bnorm == 0.0) {
        res.converged = true;
        res.residual_history.push_back(0.0);
        return res;
    }
    const int max_iter = std::min(opts.max_iter, n);
    std::vector<Vec> v;
    v.reserve(max_iter + 1);
    {
        Vec v0(n);
        for (int i = 0; i < n; ++i) v0[i] = b[i] / bnorm;
        v.push_back(std::move(v0));
    }
    const int ld = max_iter + 1;
    std::vector<double> h(size_t(ld) * std::max(max_iter, 1), 0.0);
    auto H = [&](int i, int j) -> double& { return h[size_t(j) * ld + i]; };
    std::vector<double> cs(max_iter), sn(max_iter), g(max_iter + 1, 0.0);
    g[0] = bnorm;
    res.residual_history.push_back(1.0);

    int k = 0;
    for (; k < max_iter; ++k) {
        Vec w = a(m(v[k]));
        const double pre_norm = vnorm(w);
        for (int i = 0; i <= k; ++i) {
            H(i, k) = vdot(v[i], w);
            const double hik = H(i, k);
            for (int j = 0; j < n; ++j) w[j] -= hik * v[i][j];
        }
        if (vnorm(w) < 0.7 * pre_norm) {
            for (int i = 0; i <= k; ++i) {
                const double c = vdot(v[i], w);
                H(i, k) += c;
                for (int j = 0; j < n; ++j) w[j] -= c * v[i][j];
            }
        }
        H(k + 1, k) = vnorm(w);
        const double subdiag = H(k + 1, k);
        for (int i = 0; i < k; ++i) {
            const double t = cs[i] * H(i, k) + sn[i] * H(i + 1, k);
            H(i + 1, k) = -sn[i] * H(i, k) + cs[i] * H(i + 1, k);
            H(i, k) = t;
        }
        const double denom = std::hypot(H(k, k), H(k + 1, k));
        if (denom == 0.0) {
            res.breakdown = true;
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
        res.residual_history.push_back(rel);
        if (rel <= opts.tol) {
            ++k;
            break;
        }
        if (subdiag == 0.0) {
            res.breakdown = true;
            ++k;
            break;
        }
        Vec vn(n);
        for (int j = 0; j < n; ++j) vn[j] = w[j] / subdiag;
        v.push_back(std::move(vn));
    }
    res.iterations = k;
    if (k > 0) {
        Vec y(k, 0.0);
        for (int i = k - 1; i >= 0; --i) {
            double acc = g[i];
            for (int j = i + 1; j < k; ++j) acc -= H(i, j) * y[j];
            y[i] = acc / H(i, i);
        }
        Vec z(n, 0.0);
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < n; ++j) z[j] += y[i] * v[i][j];
        res.x = m(z);
    }
    const Vec ax = a(res.x);
    Vec d(n);
    for (int j = 0; j < n; ++j) d[j] = b[j] - ax[j];
    res.final_true_residual = vnorm(d) / bnorm;
    res.converged = res.residual_history.back() <= opts.tol || res.final_true_residual <= opts.tol;
    res.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

// gmres.cpp:108-112
double residual_check(const Op& a, const Vec& b, const Vec& x) {
    const double bnorm = vnorm(b);
    const Vec ax = a(x);
    if (bnorm == 0.0) return vnorm(ax);
    Vec d(b.size());
    for (size_t j = 0; j < b.size(); ++j) d[j] = b[j] - ax[j];
    return vnorm(d) / bnorm;
}

// harness.cpp:190-219
SolveOutcome solve_system(const Bsr& a, const Vec& b, Method m, double tol, int max_iter) {
    SolveOutcome out;
    const auto t0 = std::chrono::steady_clock::now();
    const ScaledSystem scaled = left_scale(a, b, m);
    const StagePreconditioner prec = build_preconditioner(scaled);
    out.setup_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    GmresOptions opts;
    opts.tol = tol;
    opts.max_iter = max_iter;
    const Op orig = [&a](const Vec& v) { return a.apply_block(v); };
    const Op abar = [&scaled](const Vec& v) { return scaled.a_bar.apply_flat(v); };
    const Op mop = [&prec](const Vec& v) { return prec.apply(v); };
    for (int attempt = 0; attempt < 3; ++attempt) {
        out.result = gmres(a.dim(), abar, scaled.b_bar, mop, opts);
        out.result.final_true_residual = residual_check(orig, b, out.result.x);
        if (!out.result.converged || out.result.final_true_residual <= tol) break;
        opts.tol *= 0.5 * tol / out.result.final_true_residual;
    }
    if (out.result.converged && out.result.final_true_residual > tol) out.result.converged = false;
    return out;
}

// Backward sweep (amg.cpp:37-42, ilu0.cpp:52-57): row i waits for stored k > i.
std::vector<int> level_sets_upper(const Csr& a) {
    std::vector<int> lev(a.rows, 0);
    for (int i = a.rows - 1; i >= 0; --i) {
        int l = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] > i) l = std::max(l, lev[a.ci[k]] + 1);
        lev[i] = l;
    }
    return lev;
}

std::vector<int> level_sets_lower(const Csr& a) {
    std::vector<int> lev(a.rows, 0);
    for (int i = 0; i < a.rows; ++i) {
        int l = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) l = std::max(l, lev[a.ci[k]] + 1);
        lev[i] = l;
    }
    return lev;
}

// ======================================================= condensation ==
// condense.cpp:206-241.  Per cell: PartialPivLU of J22 (DenseLU, Eigen's
// unblocked order) with the 1e-14 relative pivot test; entries = J11 blocks,
// then -J12_e (J22_c^-1 J21_c) in J12 list order, merged like
// BlockMatrix::assemble (std::map on (row, col), duplicates summed in entry
// order); b = -r1 + J12_e (J22_c^-1 r2_c).  Small products sum k ascending
// from the first term.
ReducedSystem condense(const GlobalJacobian& j) {
    const int nc = j.nc, np = j.np;
    ReducedSystem red;
    red.nc = nc;
    red.np = np;
    red.sec_off = j.sec_off;
    red.j21 = j.j21;
    red.r2 = j.r2;
    red.lu.resize(nc);
    for (int c = 0; c < nc; ++c) {
        const int ns = j.sec_off[c + 1] - j.sec_off[c];
        if (ns == 0) continue;
        red.lu[c].factor(j.j22[c].data(), ns);
        double scale = 0.0;
        for (double v : j.j22[c]) scale = std::max(scale, std::abs(v));
        if (!red.lu[c].pivots_ok(1e-14 * (scale > 0.0 ? scale : 1.0), nullptr))
            throw Error(SINGULAR_BLOCK, "singular secondary block", c);
    }
    const size_t bs = size_t(np) * np;
    std::map<std::pair<int, int>, Vec> merged;
    auto add = [&](int r, int c, const double* blk) {
        auto key = std::make_pair(r, c);
        auto it = merged.find(key);
        if (it == merged.end()) {
            merged.emplace(key, Vec(blk, blk + bs));
        } else {
            for (size_t e = 0; e < bs; ++e) it->second[e] = it->second[e] + blk[e];
        }
    };
    for (int r = 0; r < nc; ++r)
        for (int k = j.rp[r]; k < j.rp[r + 1]; ++k) add(r, j.ci[k], &j.j11[size_t(k) * bs]);
    red.b.resize(size_t(nc) * np);
    for (size_t e = 0; e < red.b.size(); ++e) red.b[e] = -j.r1[e];
    for (size_t e = 0; e < j.e_row.size(); ++e) {
        const int r = j.e_row[e], c = j.e_col[e];
        const int ns = j.sec_off[c + 1] - j.sec_off[c];
        if (ns == 0) continue;
        // X = J22^-1 [J21 | r2]  (ns x (np+1))
        Vec x(size_t(ns) * (np + 1));
        for (int q = 0; q <= np; ++q) {
            double* col = &x[size_t(q) * ns];
            for (int i = 0; i < ns; ++i) col[i] = q < np ? j.j21[c][size_t(q) * ns + i] : j.r2[c][i];
            red.lu[c].solve_inplace(col);
        }
        const Vec& a = j.e_blk[e];  // np x ns
        Vec corr(bs);
        for (int q = 0; q <= np; ++q)
            for (int i = 0; i < np; ++i) {
                double acc = a[i] * x[size_t(q) * ns];
                for (int k = 1; k < ns; ++k) acc = acc + a[size_t(k) * np + i] * x[size_t(q) * ns + k];
                if (q < np)
                    corr[size_t(q) * np + i] = -acc;
                else
                    red.b[size_t(r) * np + i] = red.b[size_t(r) * np + i] + acc;
            }
        add(r, c, corr.data());
    }
    // BlockMatrix::assemble: diagonal blocks always present
    for (int c = 0; c < nc; ++c)
        if (merged.find({c, c}) == merged.end()) merged.emplace(std::make_pair(c, c), Vec(bs, 0.0));
    red.rp.assign(nc + 1, 0);
    for (const auto& [key, blk] : merged) {
        red.ci.push_back(key.second);
        red.a.insert(red.a.end(), blk.begin(), blk.end());
        red.rp[key.first + 1]++;
    }
    for (int r = 0; r < nc; ++r) red.rp[r + 1] += red.rp[r];
    return red;
}

// condense.cpp:243-258: d2_c = J22_c^-1 (-r2_c - J21_c d1_c)
Vec back_substitute(const ReducedSystem& r, const Vec& d1) {
    if (int64_t(d1.size()) != int64_t(r.nc) * r.np) throw Error(DIMENSION, "primary update dimension mismatch");
    Vec d2(size_t(r.sec_off[r.nc]));
    for (int c = 0; c < r.nc; ++c) {
        const int s0 = r.sec_off[c], ns = r.sec_off[c + 1] - s0;
        if (ns == 0) continue;
        Vec t(ns);
        for (int i = 0; i < ns; ++i) {
            double acc = r.j21[c][i] * d1[size_t(c) * r.np];
            for (int k = 1; k < r.np; ++k) acc = acc + r.j21[c][size_t(k) * ns + i] * d1[size_t(c) * r.np + k];
            t[i] = -r.r2[c][i] - acc;
        }
        r.lu[c].solve_inplace(t.data());
        for (int i = 0; i < ns; ++i) d2[s0 + i] = t[i];
    }
    return d2;
}

}  // namespace oracle
