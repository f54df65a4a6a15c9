// shim.hpp -- the Eigen3 subset the reference's solve path uses (TEST INFRASTRUCTURE).
//
// The reference (`proj/`) needs Eigen3 >= 3.3 (proj/CMakeLists.txt:8), which is
// not in this image.  oracle/_ref compiles the reference's own, unmodified
// sources against this header so the oracle restatement can be checked against
// the reference's control flow (oracle/Makefile, target `ref`).  It is NOT
// Eigen: it implements the types and members the reference calls with eager
// evaluation and ONE fixed arithmetic convention, the one oracle/oracle.cpp
// states for the Eigen call sites:
//   * a matrix product C = A*B is evaluated per entry as a sum over k
//     ascending, starting from the first term (acc = a_i0 b_0j; acc += ...),
//     into a temporary; `x += A*B` / `x -= A*B` then add / subtract that
//     temporary (Eigen's lazy coefficient-based product);
//   * dot / squaredNorm / sum: sequential from 0.0 in index order; norm =
//     sqrt(squaredNorm); maxCoeff / minCoeff: first extreme in storage order;
//   * PartialPivLU: the unblocked right-looking LU with first-maximum row
//     pivoting (Eigen's partial_lu_impl::unblocked_lu), column-oriented
//     forward / backward substitution, inverse() = solve(I);
//   * element-wise ops and scalar ops one rounding each, no FMA contraction
//     (compile with -ffp-contract=off).
// Eigen's real SIMD kernels round differently at the last-bit level; parity at
// that level is unpinned, which is why one convention is fixed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum { ColMajor = 0, RowMajor = 1, AutoAlign = 0 };
enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };

class View;
template <class Scalar, int R, int C, int O = 0, int MR = R, int MC = C>
class Matrix;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Matrix2d = Matrix<double, 2, 2>;
using Vector2d = Matrix<double, 2, 1>;

// Strided 2-D region: entry (i, j) lives at p[i * rs + j * cs].
struct Region {
    double* p = nullptr;
    Index r = 0, c = 0, rs = 1, cs = 0;
    double& at(Index i, Index j) const { return p[i * rs + j * cs]; }
    double& lin(Index k) const { return c == 1 ? at(k, 0) : (r == 1 ? at(0, k) : at(k % r, k / r)); }
};

class RowwiseSum;

// Read-only operations shared by matrices and views (CRTP).
template <class D>
class Ops {
public:
    Region rg() const { return static_cast<const D&>(*this).region(); }
    Index rows() const { return rg().r; }
    Index cols() const { return rg().c; }
    Index size() const { return rg().r * rg().c; }
    double operator()(Index i, Index j) const { return rg().at(i, j); }
    double operator()(Index k) const { return rg().lin(k); }
    double operator[](Index k) const { return rg().lin(k); }
    double coeff(Index i, Index j) const { return rg().at(i, j); }
    double coeff(Index k) const { return rg().lin(k); }

    View block(Index i, Index j, Index r, Index c) const;
    View row(Index i) const;
    View col(Index j) const;
    View segment(Index i, Index n) const;
    View head(Index n) const;
    View tail(Index n) const;
    View diagonal() const;
    View topLeftCorner(Index r, Index c) const;
    View topRows(Index n) const;
    View leftCols(Index n) const;
    View array() const;
    View matrix() const;
    RowwiseSum rowwise() const;

    MatrixXd eval() const;
    MatrixXd transpose() const;
    MatrixXd cwiseAbs() const;
    MatrixXd inverse() const;

    double maxCoeff() const {
        const Region g = rg();
        double m = g.lin(0);
        for (Index k = 1; k < size(); ++k)
            if (g.lin(k) > m) m = g.lin(k);
        return m;
    }
    double minCoeff() const {
        const Region g = rg();
        double m = g.lin(0);
        for (Index k = 1; k < size(); ++k)
            if (g.lin(k) < m) m = g.lin(k);
        return m;
    }
    double sum() const {
        const Region g = rg();
        double s = 0.0;
        for (Index j = 0; j < g.c; ++j)
            for (Index i = 0; i < g.r; ++i) s += g.at(i, j);
        return s;
    }
    double squaredNorm() const {
        const Region g = rg();
        double s = 0.0;
        for (Index j = 0; j < g.c; ++j)
            for (Index i = 0; i < g.r; ++i) s += g.at(i, j) * g.at(i, j);
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    template <class E>
    double dot(const Ops<E>& o) const {
        const Region a = rg(), b = o.rg();
        if (a.r * a.c != b.r * b.c) throw std::logic_error("eigen shim: dot size mismatch");
        double s = 0.0;
        for (Index k = 0; k < a.r * a.c; ++k) s += a.lin(k) * b.lin(k);
        return s;
    }
    double determinant() const;
    bool isZero(double prec = 1e-12) const {
        const Region g = rg();
        for (Index k = 0; k < size(); ++k)
            if (std::abs(g.lin(k)) > prec) return false;
        return true;
    }
    bool allFinite() const {
        const Region g = rg();
        for (Index k = 0; k < size(); ++k)
            if (!std::isfinite(g.lin(k))) return false;
        return true;
    }
};

// Element-wise writes through a region (views and matrices).
template <class E>
void assign_region(const Region& dst, const Ops<E>& src) {
    const Region s = src.rg();
    if (s.r != dst.r || s.c != dst.c) throw std::logic_error("eigen shim: assignment size mismatch");
    // copy through a temporary: source and destination may alias
    std::vector<double> t(size_t(s.r * s.c));
    for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) t[size_t(j * s.r + i)] = s.at(i, j);
    for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) dst.at(i, j) = t[size_t(j * s.r + i)];
}

template <class E, class F>
void update_region(const Region& dst, const Ops<E>& src, F f) {
    const Region s = src.rg();
    if (s.r != dst.r || s.c != dst.c) throw std::logic_error("eigen shim: update size mismatch");
    std::vector<double> t(size_t(s.r * s.c));
    for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) t[size_t(j * s.r + i)] = s.at(i, j);
    for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) dst.at(i, j) = f(dst.at(i, j), t[size_t(j * s.r + i)]);
}

// Non-owning writable view (block, row, segment, diagonal, array()).
class View : public Ops<View> {
public:
    Region g;
    explicit View(Region r) : g(r) {}
    View(const View&) = default;
    Region region() const { return g; }

    double& operator()(Index i, Index j) const { return g.at(i, j); }
    double& operator()(Index k) const { return g.lin(k); }
    double& operator[](Index k) const { return g.lin(k); }
    double& coeffRef(Index i, Index j) const { return g.at(i, j); }
    double& coeffRef(Index k) const { return g.lin(k); }

    View& operator=(const View& o) {
        assign_region(g, o);
        return *this;
    }
    template <class E>
    View& operator=(const Ops<E>& o) {
        assign_region(g, o);
        return *this;
    }
    template <class E>
    View& operator+=(const Ops<E>& o) {
        update_region(g, o, [](double a, double b) { return a + b; });
        return *this;
    }
    template <class E>
    View& operator-=(const Ops<E>& o) {
        update_region(g, o, [](double a, double b) { return a - b; });
        return *this;
    }
    View& operator*=(double s) {
        for (Index k = 0; k < size(); ++k) g.lin(k) *= s;
        return *this;
    }
    View& operator/=(double s) {
        for (Index k = 0; k < size(); ++k) g.lin(k) /= s;
        return *this;
    }
    View& operator+=(double s) {  // array() += scalar
        for (Index k = 0; k < size(); ++k) g.lin(k) += s;
        return *this;
    }
    void setZero() {
        for (Index k = 0; k < size(); ++k) g.lin(k) = 0.0;
    }
    void setConstant(double v) {
        for (Index k = 0; k < size(); ++k) g.lin(k) = v;
    }
    void fill(double v) { setConstant(v); }
};

template <class D>
View Ops<D>::block(Index i, Index j, Index r, Index c) const {
    const Region g = rg();
    if (i < 0 || j < 0 || r < 0 || c < 0 || i + r > g.r || j + c > g.c)
        throw std::logic_error("eigen shim: block out of range");
    return View(Region{g.p + i * g.rs + j * g.cs, r, c, g.rs, g.cs});
}
template <class D>
View Ops<D>::row(Index i) const {
    return block(i, 0, 1, rg().c);
}
template <class D>
View Ops<D>::col(Index j) const {
    return block(0, j, rg().r, 1);
}
template <class D>
View Ops<D>::segment(Index i, Index n) const {
    const Region g = rg();
    return g.c == 1 ? block(i, 0, n, 1) : block(0, i, 1, n);
}
template <class D>
View Ops<D>::head(Index n) const {
    return segment(0, n);
}
template <class D>
View Ops<D>::tail(Index n) const {
    return segment(size() - n, n);
}
template <class D>
View Ops<D>::diagonal() const {
    const Region g = rg();
    return View(Region{g.p, std::min(g.r, g.c), 1, g.rs + g.cs, 0});
}
template <class D>
View Ops<D>::topLeftCorner(Index r, Index c) const {
    return block(0, 0, r, c);
}
template <class D>
View Ops<D>::topRows(Index n) const {
    return block(0, 0, n, rg().c);
}
template <class D>
View Ops<D>::leftCols(Index n) const {
    return block(0, 0, rg().r, n);
}
template <class D>
View Ops<D>::array() const {
    return View(rg());
}
template <class D>
View Ops<D>::matrix() const {
    return View(rg());
}

// Dense owning matrix, column-major (Eigen's default storage order).
template <class Scalar, int R, int C, int O, int MR, int MC>
class Matrix : public Ops<Matrix<Scalar, R, C, O, MR, MC>> {
    static_assert(std::is_same_v<Scalar, double>, "eigen shim: double only");

public:
    static constexpr bool kVector = (R == 1 || C == 1);
    Index r_ = (R > 0 ? R : 0), c_ = (C > 0 ? C : 0);
    std::vector<double> d_ = std::vector<double>(size_t(r_ * c_), 0.0);

    Matrix() = default;
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix& o) {
        r_ = o.r_;
        c_ = o.c_;
        d_ = o.d_;
        return *this;
    }
    Matrix& operator=(Matrix&& o) noexcept {
        r_ = o.r_;
        c_ = o.c_;
        d_ = std::move(o.d_);
        return *this;
    }
    template <class I, std::enable_if_t<std::is_integral_v<I>, int> = 0>
    explicit Matrix(I n) {
        static_assert(kVector, "eigen shim: single-size constructor needs a vector type");
        if (C == 1) resize(Index(n), 1);
        else resize(1, Index(n));
    }
    template <class I, class J, std::enable_if_t<std::is_integral_v<I> && std::is_integral_v<J>, int> = 0>
    Matrix(I r, J c) {
        resize(Index(r), Index(c));
    }
    Matrix(double x, double y) {  // fixed-size 2-vector constructor
        static_assert(kVector, "eigen shim: (x, y) constructor needs a vector type");
        if (C == 1) resize(2, 1);
        else resize(1, 2);
        d_[0] = x;
        d_[1] = y;
    }
    template <class E>
    Matrix(const Ops<E>& o) {
        const Region s = o.rg();
        resize(s.r, s.c);
        for (Index j = 0; j < s.c; ++j)
            for (Index i = 0; i < s.r; ++i) d_[size_t(j * s.r + i)] = s.at(i, j);
    }
    template <class E>
    Matrix& operator=(const Ops<E>& o) {
        Matrix t(o);
        *this = std::move(t);
        return *this;
    }

    Region region() const { return Region{const_cast<double*>(d_.data()), r_, c_, 1, r_}; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }

    void resize(Index r, Index c) {
        if (r < 0 || c < 0) throw std::logic_error("eigen shim: negative size");
        r_ = r;
        c_ = c;
        d_.assign(size_t(r * c), 0.0);
    }
    void resize(Index n) {
        static_assert(kVector, "eigen shim: resize(n) needs a vector type");
        if (C == 1) resize(n, 1);
        else resize(1, n);
    }
    void conservativeResize(Index n) {
        static_assert(kVector, "eigen shim: conservativeResize(n) needs a vector type");
        std::vector<double> old = std::move(d_);
        resize(n);
        for (Index k = 0; k < std::min<Index>(n, Index(old.size())); ++k) d_[size_t(k)] = old[size_t(k)];
    }

    double& operator()(Index i, Index j) { return d_[size_t(j * r_ + i)]; }
    double operator()(Index i, Index j) const { return d_[size_t(j * r_ + i)]; }
    double& operator()(Index k) { return d_[size_t(k)]; }
    double operator()(Index k) const { return d_[size_t(k)]; }
    double& operator[](Index k) { return d_[size_t(k)]; }
    double operator[](Index k) const { return d_[size_t(k)]; }
    double& coeffRef(Index i, Index j) { return (*this)(i, j); }
    double& coeffRef(Index k) { return d_[size_t(k)]; }

    template <class E>
    Matrix& operator+=(const Ops<E>& o) {
        update_region(region(), o, [](double a, double b) { return a + b; });
        return *this;
    }
    template <class E>
    Matrix& operator-=(const Ops<E>& o) {
        update_region(region(), o, [](double a, double b) { return a - b; });
        return *this;
    }
    Matrix& operator*=(double s) {
        for (double& v : d_) v *= s;
        return *this;
    }
    Matrix& operator/=(double s) {
        for (double& v : d_) v /= s;
        return *this;
    }
    void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }
    void setZero(Index n) {
        resize(n);
        setZero();
    }
    void setZero(Index r, Index c) { resize(r, c); }
    void setConstant(double v) { std::fill(d_.begin(), d_.end(), v); }
    void setOnes() { setConstant(1.0); }
    void fill(double v) { setConstant(v); }

    static Matrix Zero() { return Matrix(); }
    template <class I, std::enable_if_t<std::is_integral_v<I>, int> = 0>
    static Matrix Zero(I n) {
        return Matrix(n);
    }
    template <class I, class J>
    static Matrix Zero(I r, J c) {
        return Matrix(Index(r), Index(c));
    }
    template <class I>
    static Matrix Ones(I n) {
        Matrix m(n);
        m.setOnes();
        return m;
    }
    template <class I, class J>
    static Matrix Ones(I r, J c) {
        Matrix m(static_cast<Index>(r), static_cast<Index>(c));
        m.setOnes();
        return m;
    }
    template <class I, class J>
    static Matrix Constant(I r, J c, double v) {
        Matrix m(static_cast<Index>(r), static_cast<Index>(c));
        m.setConstant(v);
        return m;
    }
    template <class I>
    static Matrix Constant(I n, double v) {
        Matrix m(n);
        m.setConstant(v);
        return m;
    }
    template <class I, class J>
    static Matrix Identity(I r, J c) {
        Matrix m(static_cast<Index>(r), static_cast<Index>(c));
        for (Index i = 0; i < std::min<Index>(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    template <class I>
    static Matrix Identity(I n) {
        return Identity(n, n);
    }
    static Matrix Identity() { return Identity(R, C); }
    // Generator called once per entry in storage order (Eigen's linear traversal).
    template <class I, class F>
    static Matrix NullaryExpr(I n, F f) {
        Matrix m(n);
        for (Index k = 0; k < Index(n); ++k) m.d_[size_t(k)] = f(k);
        return m;
    }
};

template <class D>
MatrixXd Ops<D>::eval() const {
    return MatrixXd(*this);
}
template <class D>
MatrixXd Ops<D>::transpose() const {
    const Region g = rg();
    MatrixXd t(g.c, g.r);
    for (Index j = 0; j < g.c; ++j)
        for (Index i = 0; i < g.r; ++i) t(j, i) = g.at(i, j);
    return t;
}
template <class D>
MatrixXd Ops<D>::cwiseAbs() const {
    MatrixXd t(*this);
    for (double& v : t.d_) v = std::abs(v);
    return t;
}

// rowwise().sum() / rowwise().maxCoeff(): per-row reductions in column order.
class RowwiseSum {
public:
    Region g;
    MatrixXd sum() const {
        MatrixXd s(g.r, 1);
        for (Index i = 0; i < g.r; ++i) {
            double acc = 0.0;
            for (Index j = 0; j < g.c; ++j) acc += g.at(i, j);
            s(i, 0) = acc;
        }
        return s;
    }
    MatrixXd maxCoeff() const {
        MatrixXd s(g.r, 1);
        for (Index i = 0; i < g.r; ++i) {
            double m = g.at(i, 0);
            for (Index j = 1; j < g.c; ++j)
                if (g.at(i, j) > m) m = g.at(i, j);
            s(i, 0) = m;
        }
        return s;
    }
};
template <class D>
RowwiseSum Ops<D>::rowwise() const {
    return RowwiseSum{rg()};
}

// ---- arithmetic (eager) -------------------------------------------------------
template <class A, class B>
MatrixXd operator+(const Ops<A>& a, const Ops<B>& b) {
    MatrixXd t(a);
    t += b;
    return t;
}
template <class A, class B>
MatrixXd operator-(const Ops<A>& a, const Ops<B>& b) {
    MatrixXd t(a);
    t -= b;
    return t;
}
template <class A>
MatrixXd operator-(const Ops<A>& a) {
    MatrixXd t(a);
    for (double& v : t.d_) v = -v;
    return t;
}
template <class A, class S, std::enable_if_t<std::is_arithmetic_v<S>, int> = 0>
MatrixXd operator*(const Ops<A>& a, S s) {
    MatrixXd t(a);
    for (double& v : t.d_) v = v * double(s);
    return t;
}
template <class A, class S, std::enable_if_t<std::is_arithmetic_v<S>, int> = 0>
MatrixXd operator*(S s, const Ops<A>& a) {
    MatrixXd t(a);
    for (double& v : t.d_) v = double(s) * v;
    return t;
}
template <class A, class S, std::enable_if_t<std::is_arithmetic_v<S>, int> = 0>
MatrixXd operator/(const Ops<A>& a, S s) {
    MatrixXd t(a);
    for (double& v : t.d_) v = v / double(s);
    return t;
}
// Product: per entry, k ascending from the first term, into a temporary.
template <class A, class B>
MatrixXd operator*(const Ops<A>& a, const Ops<B>& b) {
    const Region l = a.rg(), r = b.rg();
    if (l.c != r.r) throw std::logic_error("eigen shim: product size mismatch");
    MatrixXd t(l.r, r.c);
    if (l.c == 0) return t;
    for (Index j = 0; j < r.c; ++j)
        for (Index i = 0; i < l.r; ++i) {
            double acc = l.at(i, 0) * r.at(0, j);
            for (Index k = 1; k < l.c; ++k) acc += l.at(i, k) * r.at(k, j);
            t(i, j) = acc;
        }
    return t;
}

template <class D>
std::ostream& operator<<(std::ostream& os, const Ops<D>& m) {
    const Region g = m.rg();
    for (Index i = 0; i < g.r; ++i) {
        for (Index j = 0; j < g.c; ++j) os << (j ? " " : "") << g.at(i, j);
        if (i + 1 < g.r) os << "\n";
    }
    return os;
}

// ---- PartialPivLU ------------------------------------------------------------
class PermutationIndices {
public:
    std::vector<int> v;
    Index size() const { return Index(v.size()); }
    int operator[](Index i) const { return v[size_t(i)]; }
    int operator()(Index i) const { return v[size_t(i)]; }
};
class PermutationMatrix {
public:
    PermutationIndices idx;
    const PermutationIndices& indices() const { return idx; }
};

template <class MatrixType>
class PartialPivLU {
public:
    PartialPivLU() = default;
    template <class E>
    explicit PartialPivLU(const Ops<E>& a) {
        compute(a);
    }
    template <class E>
    PartialPivLU& compute(const Ops<E>& a) {
        lu_ = MatrixXd(a);
        const Index n = lu_.rows();
        if (lu_.cols() != n) throw std::logic_error("eigen shim: PartialPivLU needs a square matrix");
        row_of_.resize(size_t(n));
        for (Index i = 0; i < n; ++i) row_of_[size_t(i)] = int(i);
        for (Index k = 0; k < n; ++k) {
            Index p = k;
            double best = std::abs(lu_(k, k));
            for (Index i = k + 1; i < n; ++i)
                if (std::abs(lu_(i, k)) > best) {
                    best = std::abs(lu_(i, k));
                    p = i;
                }
            if (best != 0.0) {
                if (p != k) {
                    for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
                    std::swap(row_of_[size_t(k)], row_of_[size_t(p)]);
                }
                const double d = lu_(k, k);
                for (Index i = k + 1; i < n; ++i) lu_(i, k) = lu_(i, k) / d;
            }
            for (Index j = k + 1; j < n; ++j) {
                const double ukj = lu_(k, j);
                for (Index i = k + 1; i < n; ++i) lu_(i, j) = lu_(i, j) - lu_(i, k) * ukj;
            }
        }
        // P A = L U with P x placing x[i] at position indices[i] (Eigen's convention)
        perm_.idx.v.assign(size_t(n), 0);
        for (Index k = 0; k < n; ++k) perm_.idx.v[size_t(row_of_[size_t(k)])] = int(k);
        return *this;
    }
    const MatrixXd& matrixLU() const { return lu_; }
    const PermutationMatrix& permutationP() const { return perm_; }
    Index rows() const { return lu_.rows(); }
    Index cols() const { return lu_.cols(); }

    template <class E>
    MatrixXd solve(const Ops<E>& b) const {
        const Index n = lu_.rows();
        const Region g = b.rg();
        if (g.r != n) throw std::logic_error("eigen shim: solve size mismatch");
        MatrixXd x(n, g.c);
        std::vector<double> t(static_cast<size_t>(n));
        for (Index q = 0; q < g.c; ++q) {
            for (Index i = 0; i < n; ++i) t[size_t(i)] = g.at(row_of_[size_t(i)], q);
            for (Index j = 0; j < n; ++j) {
                const double xj = t[size_t(j)];
                for (Index i = j + 1; i < n; ++i) t[size_t(i)] = t[size_t(i)] - lu_(i, j) * xj;
            }
            for (Index j = n - 1; j >= 0; --j) {
                t[size_t(j)] = t[size_t(j)] / lu_(j, j);
                const double xj = t[size_t(j)];
                for (Index i = 0; i < j; ++i) t[size_t(i)] = t[size_t(i)] - lu_(i, j) * xj;
            }
            for (Index i = 0; i < n; ++i) x(i, q) = t[size_t(i)];
        }
        return x;
    }
    MatrixXd inverse() const { return solve(MatrixXd::Identity(lu_.rows(), lu_.rows())); }
    double determinant() const {
        double d = 1.0;
        for (Index i = 0; i < lu_.rows(); ++i) d *= lu_(i, i);
        Index swaps = 0;
        std::vector<int> seen(row_of_);
        for (Index i = 0; i < Index(seen.size()); ++i)
            while (seen[size_t(i)] != int(i)) {
                std::swap(seen[size_t(i)], seen[size_t(seen[size_t(i)])]);
                ++swaps;
            }
        return swaps % 2 ? -d : d;
    }

private:
    MatrixXd lu_;
    std::vector<int> row_of_;  // row_of_[k] = original row placed at position k
    PermutationMatrix perm_;
};

// 2x2 closed forms (Eigen's compute_inverse_size2 / determinant of a 2x2);
// larger sizes go through the LU.
template <class D>
double Ops<D>::determinant() const {
    const Region g = rg();
    if (g.r != g.c) throw std::logic_error("eigen shim: determinant of a non-square matrix");
    if (g.r == 0) return 1.0;
    if (g.r == 1) return g.at(0, 0);
    if (g.r == 2) return g.at(0, 0) * g.at(1, 1) - g.at(1, 0) * g.at(0, 1);
    return PartialPivLU<MatrixXd>(*this).determinant();
}
template <class D>
MatrixXd Ops<D>::inverse() const {
    const Region g = rg();
    if (g.r != g.c) throw std::logic_error("eigen shim: inverse of a non-square matrix");
    if (g.r == 2) {
        const double invdet = 1.0 / determinant();
        MatrixXd m(2, 2);
        m(0, 0) = g.at(1, 1) * invdet;
        m(1, 0) = -g.at(1, 0) * invdet;
        m(0, 1) = -g.at(0, 1) * invdet;
        m(1, 1) = g.at(0, 0) * invdet;
        return m;
    }
    return PartialPivLU<MatrixXd>(*this).inverse();
}

}  // namespace Eigen
