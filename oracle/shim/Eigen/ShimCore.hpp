// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Minimal Eigen-subset shim so that the reference headers
// (/root/reference/proj/include/cpdd/*.hpp) and the reference's own GTest
// suites compile UNMODIFIED in this container, where Eigen 3 is absent
// (SURVEY.md section 8(c), Appendix D lists the API surface covered here).
//
// Everything is evaluated eagerly (no expression templates).  Reductions
// (sum / dot / squaredNorm / norm) follow the summation order of real Eigen
// 3.4 compiled for x86-64 with its default SSE2 packets of two doubles
// (Eigen/src/Core/Redux.h: LinearVectorizedTraversal), so the shim reproduces
// the reference's floating-point results as closely as a re-implementation
// can.  Only the SparseLU backend differs (see SparseLU.hpp).
#ifndef ORACLE_EIGEN_SHIM_CORE_HPP
#define ORACLE_EIGEN_SHIM_CORE_HPP

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int Infinity = -1;

enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

namespace internal {

// Sum of n contiguous values in the order of Eigen's vectorised redux for a
// dynamic-size, 16-byte aligned vector with packet size 2 (Redux.h,
// redux_impl<..., LinearVectorizedTraversal, NoUnrolling>).
template <class F>
inline double redux_dynamic(Index n, F&& coeff) {
    if (n <= 0) return 0.0;
    const Index ps = 2;
    const Index aligned2 = (n / (2 * ps)) * (2 * ps);
    const Index aligned = (n / ps) * ps;
    if (aligned == 0) {
        double res = coeff(0);
        for (Index i = 1; i < n; ++i) res = res + coeff(i);
        return res;
    }
    double p0a = coeff(0), p0b = coeff(1);
    if (aligned > ps) {
        double p1a = coeff(2), p1b = coeff(3);
        for (Index i = 2 * ps; i < aligned2; i += 2 * ps) {
            p0a = p0a + coeff(i);
            p0b = p0b + coeff(i + 1);
            p1a = p1a + coeff(i + 2);
            p1b = p1b + coeff(i + 3);
        }
        p0a = p0a + p1a;
        p0b = p0b + p1b;
        if (aligned > aligned2) {
            p0a = p0a + coeff(aligned2);
            p0b = p0b + coeff(aligned2 + 1);
        }
    }
    double res = p0a + p0b;
    for (Index i = aligned; i < n; ++i) res = res + coeff(i);
    return res;
}

// Fixed sizes 1..4 (CompleteUnrolling + LinearVectorizedTraversal, Packet2d).
template <class F>
inline double redux_fixed(int n, F&& coeff) {
    switch (n) {
        case 1: return coeff(0);
        case 2: return coeff(0) + coeff(1);
        case 3: return (coeff(0) + coeff(1)) + coeff(2);
        case 4: return (coeff(0) + coeff(2)) + (coeff(1) + coeff(3));
        default: return redux_dynamic(n, coeff);
    }
}

template <int R, int C>
struct Storage {
    static constexpr bool fixed = (R != Dynamic && C != Dynamic);
};

}  // namespace internal

template <typename Scalar, int Rows, int Cols, int Options = 0, int MaxRows = Rows,
          int MaxCols = Cols>
class Matrix;

template <typename Derived>
class Map;

template <typename Scalar_, int Rows, int Cols, int Options, int MaxRows, int MaxCols>
class Matrix {
public:
    using Scalar = Scalar_;
    using RealScalar = Scalar_;
    static constexpr bool kFixed = internal::Storage<Rows, Cols>::fixed;
    static constexpr int RowsAtCompileTime = Rows;
    static constexpr int ColsAtCompileTime = Cols;
    static constexpr int SizeAtCompileTime = kFixed ? Rows * Cols : Dynamic;
    using Store = std::conditional_t<kFixed, std::array<Scalar, (kFixed ? Rows * Cols : 1)>,
                                     std::vector<Scalar>>;

    Matrix() {
        if constexpr (kFixed) d_.fill(Scalar(0));
        rows_ = Rows == Dynamic ? 0 : Rows;
        cols_ = Cols == Dynamic ? 0 : Cols;
    }
    // dynamic vector of size n, or a fixed 2-vector's (x, y) when both are doubles
    template <typename T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    explicit Matrix(T n) {
        static_assert(!kFixed, "size constructor on fixed-size matrix");
        if constexpr (Cols == 1) {
            rows_ = static_cast<Index>(n);
            cols_ = 1;
        } else if constexpr (Rows == 1) {
            rows_ = 1;
            cols_ = static_cast<Index>(n);
        }
        d_.assign(static_cast<std::size_t>(n), Scalar(0));
    }
    template <typename T, typename U,
              std::enable_if_t<std::is_integral_v<T> && std::is_integral_v<U>, int> = 0>
    Matrix(T r, U c) {
        if constexpr (kFixed) {
            // Eigen treats Matrix<double,2,1>(int,int) as coefficients.
            static_assert(Rows * Cols == 2, "two-scalar constructor needs a 2-vector");
            d_[0] = Scalar(r);
            d_[1] = Scalar(c);
            rows_ = Rows;
            cols_ = Cols;
        } else {
            rows_ = static_cast<Index>(r);
            cols_ = static_cast<Index>(c);
            d_.assign(static_cast<std::size_t>(rows_ * cols_), Scalar(0));
        }
    }
    template <typename T, typename U,
              std::enable_if_t<!(std::is_integral_v<T> && std::is_integral_v<U>), int> = 0>
    Matrix(T x, U y) {
        static_assert(kFixed && Rows * Cols == 2, "two-scalar constructor needs a 2-vector");
        d_[0] = Scalar(x);
        d_[1] = Scalar(y);
        rows_ = Rows;
        cols_ = Cols;
    }
    Matrix(Scalar x, Scalar y, Scalar z) {
        static_assert(kFixed && Rows * Cols == 3, "three-scalar constructor needs a 3-vector");
        d_[0] = x;
        d_[1] = y;
        d_[2] = z;
        rows_ = Rows;
        cols_ = Cols;
    }
    Matrix(Scalar x, Scalar y, Scalar z, Scalar w) {
        static_assert(kFixed && Rows * Cols == 4, "four-scalar constructor needs a 4-vector");
        d_[0] = x;
        d_[1] = y;
        d_[2] = z;
        d_[3] = w;
        rows_ = Rows;
        cols_ = Cols;
    }
    template <typename D>
    Matrix(const Map<D>& m);

    // ------------------------------------------------------------ shape
    Index rows() const { return kFixed ? Rows : rows_; }
    Index cols() const { return kFixed ? Cols : cols_; }
    Index size() const { return rows() * cols(); }
    void resize(Index n) {
        static_assert(!kFixed, "resize on fixed-size matrix");
        if constexpr (Cols == 1) {
            rows_ = n;
            cols_ = 1;
        } else {
            rows_ = 1;
            cols_ = n;
        }
        d_.resize(static_cast<std::size_t>(n));
    }
    void resize(Index r, Index c) {
        static_assert(!kFixed, "resize on fixed-size matrix");
        rows_ = r;
        cols_ = c;
        d_.resize(static_cast<std::size_t>(r * c));
    }
    Scalar* data() { return d_.data(); }
    const Scalar* data() const { return d_.data(); }

    // ------------------------------------------------------------ access
    Scalar& operator[](Index i) { return d_[static_cast<std::size_t>(i)]; }
    const Scalar& operator[](Index i) const { return d_[static_cast<std::size_t>(i)]; }
    Scalar& operator()(Index i) { return d_[static_cast<std::size_t>(i)]; }
    const Scalar& operator()(Index i) const { return d_[static_cast<std::size_t>(i)]; }
    Scalar& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * rows())]; }
    const Scalar& operator()(Index i, Index j) const {
        return d_[static_cast<std::size_t>(i + j * rows())];
    }
    Scalar coeff(Index i) const { return d_[static_cast<std::size_t>(i)]; }
    Scalar& x() { return d_[0]; }
    Scalar& y() { return d_[1]; }
    Scalar& z() { return d_[2]; }
    Scalar x() const { return d_[0]; }
    Scalar y() const { return d_[1]; }
    Scalar z() const { return d_[2]; }

    // ------------------------------------------------------------ factories
    static Matrix Zero() {
        static_assert(kFixed, "Zero() needs a fixed size");
        Matrix m;
        return m;
    }
    static Matrix Zero(Index n) {
        Matrix m(n);
        return m;
    }
    static Matrix Zero(Index r, Index c) {
        Matrix m(r, c);
        return m;
    }
    static Matrix Ones() {
        Matrix m;
        for (auto& v : m.d_) v = Scalar(1);
        return m;
    }
    static Matrix Ones(Index n) {
        Matrix m(n);
        for (auto& v : m.d_) v = Scalar(1);
        return m;
    }
    static Matrix Constant(Index n, Scalar c) {
        Matrix m(n);
        for (auto& v : m.d_) v = c;
        return m;
    }
    static Matrix Unit(int k) {
        Matrix m;
        m.d_[k] = Scalar(1);
        return m;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }
    void setZero() { std::fill(d_.begin(), d_.end(), Scalar(0)); }
    void setOnes() { std::fill(d_.begin(), d_.end(), Scalar(1)); }

    // ------------------------------------------------------------ comma init
    struct CommaInit {
        Matrix* m;
        Index k;
        CommaInit& operator,(Scalar v) {
            (*m)[k++] = v;
            return *this;
        }
    };
    CommaInit operator<<(Scalar v) {
        d_[0] = v;
        return CommaInit{this, 1};
    }

    // ------------------------------------------------------------ arithmetic
    Matrix operator-() const {
        Matrix r = *this;
        for (auto& v : r.d_) v = -v;
        return r;
    }
    Matrix& operator+=(const Matrix& o) {
        check_same(o);
        for (std::size_t i = 0; i < d_.size(); ++i) d_[i] = d_[i] + o.d_[i];
        return *this;
    }
    Matrix& operator-=(const Matrix& o) {
        check_same(o);
        for (std::size_t i = 0; i < d_.size(); ++i) d_[i] = d_[i] - o.d_[i];
        return *this;
    }
    Matrix& operator*=(Scalar s) {
        for (auto& v : d_) v = v * s;
        return *this;
    }
    Matrix& operator/=(Scalar s) {
        for (auto& v : d_) v = v / s;
        return *this;
    }
    friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
    friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
    friend Matrix operator*(Matrix a, Scalar s) { return a *= s; }
    friend Matrix operator*(Scalar s, Matrix a) {
        for (auto& v : a.d_) v = s * v;
        return a;
    }
    friend Matrix operator/(Matrix a, Scalar s) { return a /= s; }

    bool operator==(const Matrix& o) const {
        return rows() == o.rows() && cols() == o.cols() &&
               std::equal(d_.begin(), d_.end(), o.d_.begin());
    }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

    // ------------------------------------------------------------ reductions
    template <class F>
    Scalar redux(F&& f) const {
        if constexpr (kFixed)
            return internal::redux_fixed(Rows * Cols, f);
        else
            return internal::redux_dynamic(size(), f);
    }
    Scalar sum() const {
        return redux([&](Index i) { return d_[static_cast<std::size_t>(i)]; });
    }
    Scalar squaredNorm() const {
        return redux([&](Index i) {
            const Scalar v = d_[static_cast<std::size_t>(i)];
            return v * v;
        });
    }
    Scalar norm() const { return std::sqrt(squaredNorm()); }
    Scalar dot(const Matrix& o) const {
        check_same(o);
        return redux([&](Index i) {
            return d_[static_cast<std::size_t>(i)] * o.d_[static_cast<std::size_t>(i)];
        });
    }
    Matrix normalized() const {
        const Scalar z = squaredNorm();
        if (z > Scalar(0)) return *this / std::sqrt(z);
        return *this;
    }
    void normalize() { *this = normalized(); }
    Matrix cross(const Matrix& b) const {
        static_assert(kFixed && Rows * Cols == 3, "cross needs 3-vectors");
        const Matrix& a = *this;
        return Matrix(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                      a[0] * b[1] - a[1] * b[0]);
    }
    Matrix cwiseMin(const Matrix& o) const {
        Matrix r = *this;
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = std::min(d_[i], o.d_[i]);
        return r;
    }
    Matrix cwiseMax(const Matrix& o) const {
        Matrix r = *this;
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = std::max(d_[i], o.d_[i]);
        return r;
    }
    Matrix cwiseAbs() const {
        Matrix r = *this;
        for (auto& v : r.d_) v = std::abs(v);
        return r;
    }
    Matrix cwiseProduct(const Matrix& o) const {
        Matrix r = *this;
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] * o.d_[i];
        return r;
    }
    Scalar maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
    Scalar minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
    bool isZero(Scalar prec = Scalar(1e-12)) const {
        for (auto v : d_)
            if (std::abs(v) > prec) return false;
        return true;
    }
    bool allFinite() const {
        for (auto v : d_)
            if (!std::isfinite(v)) return false;
        return true;
    }
    template <int P>
    Scalar lpNorm() const {
        if constexpr (P == Infinity) {
            Scalar m = 0;
            for (auto v : d_) m = std::max(m, std::abs(v));
            return m;
        } else if constexpr (P == 1) {
            return redux([&](Index i) { return std::abs(d_[static_cast<std::size_t>(i)]); });
        } else {
            static_assert(P == 2, "lpNorm<1|2|Infinity> only");
            return norm();
        }
    }
    Matrix head(Index n) const {
        Matrix r(n);
        for (Index i = 0; i < n; ++i) r[i] = d_[static_cast<std::size_t>(i)];
        return r;
    }
    Matrix tail(Index n) const {
        Matrix r(n);
        const Index off = size() - n;
        for (Index i = 0; i < n; ++i) r[i] = d_[static_cast<std::size_t>(off + i)];
        return r;
    }
    Matrix segment(Index s, Index n) const {
        Matrix r(n);
        for (Index i = 0; i < n; ++i) r[i] = d_[static_cast<std::size_t>(s + i)];
        return r;
    }

private:
    Store d_{};
    Index rows_ = 0, cols_ = 0;

    void check_same(const Matrix& o) const {
        if (rows() != o.rows() || cols() != o.cols())
            throw std::logic_error("Eigen shim: size mismatch in binary operation");
    }

    template <typename, int, int, int, int, int>
    friend class Matrix;
};

using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;

// Dense matrix-vector and matrix-matrix products (test-only helpers in the
// reference suites; plain row-by-column accumulation).
inline VectorXd operator*(const MatrixXd& A, const VectorXd& x) {
    if (A.cols() != x.size()) throw std::logic_error("Eigen shim: product size mismatch");
    VectorXd y = VectorXd::Zero(A.rows());
    for (Index j = 0; j < A.cols(); ++j) {
        const double xj = x[j];
        for (Index i = 0; i < A.rows(); ++i) y[i] += A(i, j) * xj;
    }
    return y;
}
inline MatrixXd operator*(const MatrixXd& A, const MatrixXd& B) {
    if (A.cols() != B.rows()) throw std::logic_error("Eigen shim: product size mismatch");
    MatrixXd C = MatrixXd::Zero(A.rows(), B.cols());
    for (Index j = 0; j < B.cols(); ++j)
        for (Index k = 0; k < A.cols(); ++k) {
            const double b = B(k, j);
            for (Index i = 0; i < A.rows(); ++i) C(i, j) += A(i, k) * b;
        }
    return C;
}

/** Map<VectorXd>(ptr, n): read view that converts to an owning vector. */
template <typename Derived>
class Map {
public:
    using Scalar = typename Derived::Scalar;
    Map(const Scalar* p, Index n) : p_(p), n_(n) {}
    Index size() const { return n_; }
    const Scalar* data() const { return p_; }

private:
    const Scalar* p_;
    Index n_;
};

template <typename S, int R, int C, int O, int MR, int MC>
template <typename D>
Matrix<S, R, C, O, MR, MC>::Matrix(const Map<D>& m) : Matrix(m.size()) {
    for (Index i = 0; i < m.size(); ++i) d_[static_cast<std::size_t>(i)] = m.data()[i];
}

/** Dense LU with complete pivoting (test oracle in the reference suites). */
template <typename MatrixType>
class FullPivLU {
public:
    explicit FullPivLU(const MatrixType& A) : lu_(A), n_(A.rows()) {
        if (A.rows() != A.cols()) throw std::logic_error("FullPivLU shim: square only");
        rp_.resize(n_);
        cp_.resize(n_);
        for (Index i = 0; i < n_; ++i) rp_[i] = cp_[i] = i;
        for (Index k = 0; k < n_; ++k) {
            Index bi = k, bj = k;
            double best = -1;
            for (Index j = k; j < n_; ++j)
                for (Index i = k; i < n_; ++i)
                    if (std::abs(lu_(i, j)) > best) {
                        best = std::abs(lu_(i, j));
                        bi = i;
                        bj = j;
                    }
            if (best == 0.0) {
                rank_ = k;
                return;
            }
            if (bi != k) {
                for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(bi, j));
                std::swap(rp_[k], rp_[bi]);
            }
            if (bj != k) {
                for (Index i = 0; i < n_; ++i) std::swap(lu_(i, k), lu_(i, bj));
                std::swap(cp_[k], cp_[bj]);
            }
            const double piv = lu_(k, k);
            for (Index i = k + 1; i < n_; ++i) lu_(i, k) /= piv;
            for (Index j = k + 1; j < n_; ++j) {
                const double u = lu_(k, j);
                if (u == 0.0) continue;
                for (Index i = k + 1; i < n_; ++i) lu_(i, j) -= lu_(i, k) * u;
            }
        }
        rank_ = n_;
    }
    VectorXd solve(const VectorXd& b) const {
        VectorXd y(n_);
        for (Index i = 0; i < n_; ++i) y[i] = b[rp_[i]];
        for (Index i = 0; i < rank_; ++i)
            for (Index k = 0; k < i; ++k) y[i] -= lu_(i, k) * y[k];
        VectorXd z = VectorXd::Zero(n_);
        for (Index i = rank_ - 1; i >= 0; --i) {
            double s = y[i];
            for (Index k = i + 1; k < rank_; ++k) s -= lu_(i, k) * z[k];
            z[i] = s / lu_(i, i);
        }
        VectorXd x = VectorXd::Zero(n_);
        for (Index i = 0; i < n_; ++i) x[cp_[i]] = z[i];
        return x;
    }
    Index rank() const { return rank_; }

private:
    MatrixType lu_;
    Index n_;
    std::vector<Index> rp_, cp_;
    Index rank_ = 0;
};

}  // namespace Eigen

#endif  // ORACLE_EIGEN_SHIM_CORE_HPP
