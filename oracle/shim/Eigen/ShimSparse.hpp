// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Sparse part of the Eigen-subset shim: SparseMatrix / Triplet and a
// SparseLU stand-in honouring the contract of the reference's DirectSolver
// (proj/include/cpdd/direct.hpp:36-68): factor once, info()==Success unless
// singular, each solve with a small relative residual.
//
// Real Eigen's SparseLU (supernodal, COLAMD column ordering, partial
// pivoting) is not available here.  This stand-in restates the published
// alternative the survey identified for these matrices (SURVEY.md section 7,
// hard part 2): reverse Cuthill-McKee symmetric ordering, then a profile
// (skyline / envelope) LU without pivoting, with a banded
// partial-pivoting LU as the fallback whenever a pivot is tiny relative to
// its row or non-finite.
#ifndef ORACLE_EIGEN_SHIM_SPARSE_HPP
#define ORACLE_EIGEN_SHIM_SPARSE_HPP

#include "ShimCore.hpp"

#include <deque>
#include <numeric>

namespace Eigen {

template <typename Scalar>
class Triplet {
public:
    Triplet(Index r, Index c, Scalar v) : r_(r), c_(c), v_(v) {}
    Index row() const { return r_; }
    Index col() const { return c_; }
    Scalar value() const { return v_; }

private:
    Index r_, c_;
    Scalar v_;
};

/** Compressed-row sparse matrix (duplicates summed in triplet order). */
template <typename Scalar_, int Options = 0, typename StorageIndex = int>
class SparseMatrix {
public:
    using Scalar = Scalar_;
    SparseMatrix() = default;
    SparseMatrix(Index r, Index c) : rows_(r), cols_(c), ptr_(static_cast<std::size_t>(r) + 1, 0) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index nonZeros() const { return static_cast<Index>(col_.size()); }

    template <typename It>
    void setFromTriplets(It begin, It end) {
        std::vector<std::vector<std::pair<int, Scalar>>> rows(static_cast<std::size_t>(rows_));
        for (It it = begin; it != end; ++it) {
            if (it->row() < 0 || it->row() >= rows_ || it->col() < 0 || it->col() >= cols_)
                throw std::logic_error("SparseMatrix shim: triplet out of range");
            rows[static_cast<std::size_t>(it->row())].emplace_back(static_cast<int>(it->col()),
                                                                   it->value());
        }
        ptr_.assign(static_cast<std::size_t>(rows_) + 1, 0);
        col_.clear();
        val_.clear();
        for (Index i = 0; i < rows_; ++i) {
            auto& r = rows[static_cast<std::size_t>(i)];
            std::stable_sort(r.begin(), r.end(),
                             [](const auto& a, const auto& b) { return a.first < b.first; });
            for (std::size_t k = 0; k < r.size(); ++k) {
                if (k > 0 && r[k - 1].first == r[k].first)
                    val_.back() += r[k].second;
                else {
                    col_.push_back(r[k].first);
                    val_.push_back(r[k].second);
                }
            }
            ptr_[static_cast<std::size_t>(i) + 1] = static_cast<Index>(col_.size());
        }
    }
    void makeCompressed() {}

    const std::vector<Index>& row_ptr() const { return ptr_; }
    const std::vector<int>& col_index() const { return col_; }
    const std::vector<Scalar>& values() const { return val_; }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<Index> ptr_;
    std::vector<int> col_;
    std::vector<Scalar> val_;
};

template <typename StorageIndex>
struct COLAMDOrdering {};

namespace internal {

/** Reverse Cuthill-McKee on the symmetric pattern adj (sorted neighbour
 *  lists).  Each component starts from a pseudo-peripheral node found by
 *  repeated BFS from the lowest-degree unvisited node; neighbours are
 *  visited by increasing (degree, index).  Returns perm[new] = old. */
inline std::vector<int> rcm_order(const std::vector<std::vector<int>>& adj) {
    const int n = static_cast<int>(adj.size());
    std::vector<int> order;
    order.reserve(static_cast<std::size_t>(n));
    std::vector<char> done(static_cast<std::size_t>(n), 0);
    std::vector<int> level(static_cast<std::size_t>(n), -1);
    auto deg = [&](int v) { return static_cast<int>(adj[static_cast<std::size_t>(v)].size()); };
    auto bfs_last_level = [&](int s, int& ecc) {
        // returns a min-degree node of the last BFS level within s's component
        std::vector<int> q{s};
        std::vector<int> touched{s};
        level[static_cast<std::size_t>(s)] = 0;
        std::size_t h = 0;
        int last = 0;
        while (h < q.size()) {
            int v = q[h++];
            last = level[static_cast<std::size_t>(v)];
            for (int w : adj[static_cast<std::size_t>(v)])
                if (!done[static_cast<std::size_t>(w)] && level[static_cast<std::size_t>(w)] < 0) {
                    level[static_cast<std::size_t>(w)] = level[static_cast<std::size_t>(v)] + 1;
                    q.push_back(w);
                    touched.push_back(w);
                }
        }
        int best = -1;
        for (int v : q)
            if (level[static_cast<std::size_t>(v)] == last &&
                (best < 0 || deg(v) < deg(best) || (deg(v) == deg(best) && v < best)))
                best = v;
        for (int v : touched) level[static_cast<std::size_t>(v)] = -1;
        ecc = last;
        return best;
    };
    for (;;) {
        int s = -1;
        for (int v = 0; v < n; ++v)
            if (!done[static_cast<std::size_t>(v)] && (s < 0 || deg(v) < deg(s))) s = v;
        if (s < 0) break;
        int ecc = 0;
        int cand = bfs_last_level(s, ecc);
        for (int it = 0; it < 8; ++it) {
            int ecc2 = 0;
            int next = bfs_last_level(cand, ecc2);
            if (ecc2 <= ecc) break;
            ecc = ecc2;
            s = cand;
            cand = next;
        }
        s = cand;
        std::size_t start = order.size();
        order.push_back(s);
        done[static_cast<std::size_t>(s)] = 1;
        for (std::size_t h = start; h < order.size(); ++h) {
            int v = order[h];
            std::vector<int> nb;
            for (int w : adj[static_cast<std::size_t>(v)])
                if (!done[static_cast<std::size_t>(w)]) nb.push_back(w);
            std::sort(nb.begin(), nb.end(), [&](int a, int b) {
                return deg(a) != deg(b) ? deg(a) < deg(b) : a < b;
            });
            for (int w : nb) {
                done[static_cast<std::size_t>(w)] = 1;
                order.push_back(w);
            }
        }
    }
    std::reverse(order.begin(), order.end());
    return order;
}

}  // namespace internal

template <typename MatrixType, typename OrderingType = COLAMDOrdering<int>>
class SparseLU {
public:
    SparseLU() = default;

    void analyzePattern(const MatrixType& A) {
        n_ = A.rows();
        if (A.rows() != A.cols()) throw std::logic_error("SparseLU shim: square only");
        std::vector<std::vector<int>> adj(static_cast<std::size_t>(n_));
        const auto& ptr = A.row_ptr();
        const auto& col = A.col_index();
        for (Index i = 0; i < n_; ++i)
            for (Index k = ptr[static_cast<std::size_t>(i)]; k < ptr[static_cast<std::size_t>(i) + 1]; ++k) {
                int j = col[static_cast<std::size_t>(k)];
                if (j == i) continue;
                adj[static_cast<std::size_t>(i)].push_back(j);
                adj[static_cast<std::size_t>(j)].push_back(static_cast<int>(i));
            }
        for (auto& a : adj) {
            std::sort(a.begin(), a.end());
            a.erase(std::unique(a.begin(), a.end()), a.end());
        }
        perm_ = internal::rcm_order(adj);
        inv_.assign(static_cast<std::size_t>(n_), 0);
        for (Index k = 0; k < n_; ++k) inv_[static_cast<std::size_t>(perm_[static_cast<std::size_t>(k)])] = static_cast<int>(k);
        // envelope: first[i] = min permuted index among row/col neighbours <= i
        first_.assign(static_cast<std::size_t>(n_), 0);
        for (Index i = 0; i < n_; ++i) {
            int pi = inv_[static_cast<std::size_t>(i)];
            int f = pi;
            for (int j : adj[static_cast<std::size_t>(i)]) f = std::min(f, inv_[static_cast<std::size_t>(j)]);
            first_[static_cast<std::size_t>(pi)] = f;
        }
        off_.assign(static_cast<std::size_t>(n_) + 1, 0);
        for (Index i = 0; i < n_; ++i)
            off_[static_cast<std::size_t>(i) + 1] = off_[static_cast<std::size_t>(i)] + (i - first_[static_cast<std::size_t>(i)]);
        analyzed_ = true;
    }

    void factorize(const MatrixType& A) {
        if (!analyzed_) analyzePattern(A);
        info_ = Success;
        banded_ = false;
        const std::size_t tot = static_cast<std::size_t>(off_[static_cast<std::size_t>(n_)]);
        L_.assign(tot, 0.0);
        U_.assign(tot, 0.0);
        D_.assign(static_cast<std::size_t>(n_), 0.0);
        std::vector<double> rowmax(static_cast<std::size_t>(n_), 0.0);
        const auto& ptr = A.row_ptr();
        const auto& col = A.col_index();
        const auto& val = A.values();
        for (Index i = 0; i < n_; ++i)
            for (Index k = ptr[static_cast<std::size_t>(i)]; k < ptr[static_cast<std::size_t>(i) + 1]; ++k) {
                const int pi = inv_[static_cast<std::size_t>(i)];
                const int pj = inv_[static_cast<std::size_t>(col[static_cast<std::size_t>(k)])];
                const double v = val[static_cast<std::size_t>(k)];
                rowmax[static_cast<std::size_t>(pi)] = std::max(rowmax[static_cast<std::size_t>(pi)], std::abs(v));
                if (pi == pj)
                    D_[static_cast<std::size_t>(pi)] += v;
                else if (pj < pi)
                    L_[static_cast<std::size_t>(off_[static_cast<std::size_t>(pi)] + (pj - first_[static_cast<std::size_t>(pi)]))] += v;
                else
                    U_[static_cast<std::size_t>(off_[static_cast<std::size_t>(pj)] + (pi - first_[static_cast<std::size_t>(pj)]))] += v;
            }
        // profile Crout: row i of L and column i of U by bordering
        bool ok = true;
        for (Index i = 0; i < n_ && ok; ++i) {
            const int fi = first_[static_cast<std::size_t>(i)];
            double* Li = L_.data() + off_[static_cast<std::size_t>(i)];
            double* Ui = U_.data() + off_[static_cast<std::size_t>(i)];
            for (Index j = fi; j < i; ++j) {
                const int fj = first_[static_cast<std::size_t>(j)];
                const int lo = std::max(fi, fj);
                const double* Lj = L_.data() + off_[static_cast<std::size_t>(j)];
                const double* Uj = U_.data() + off_[static_cast<std::size_t>(j)];
                double sl = Li[j - fi], su = Ui[j - fi];
                for (int k = lo; k < j; ++k) {
                    sl -= Li[k - fi] * Uj[k - fj];
                    su -= Lj[k - fj] * Ui[k - fi];
                }
                Li[j - fi] = sl / D_[static_cast<std::size_t>(j)];
                Ui[j - fi] = su;
            }
            double d = D_[static_cast<std::size_t>(i)];
            for (Index k = fi; k < i; ++k) d -= Li[k - fi] * Ui[k - fi];
            D_[static_cast<std::size_t>(i)] = d;
            if (!std::isfinite(d) || std::abs(d) <= 1e-10 * rowmax[static_cast<std::size_t>(i)]) ok = false;
        }
        if (!ok) factorize_banded(A);
    }

    ComputationInfo info() const { return info_; }

    VectorXd solve(const VectorXd& b) const {
        VectorXd y(n_);
        for (Index k = 0; k < n_; ++k) y[k] = b[perm_[static_cast<std::size_t>(k)]];
        if (banded_) {
            solve_banded(y);
        } else {
            for (Index i = 0; i < n_; ++i) {
                const int fi = first_[static_cast<std::size_t>(i)];
                const double* Li = L_.data() + off_[static_cast<std::size_t>(i)];
                double s = y[i];
                for (Index k = fi; k < i; ++k) s -= Li[k - fi] * y[k];
                y[i] = s;
            }
            for (Index i = n_ - 1; i >= 0; --i) {
                const int fi = first_[static_cast<std::size_t>(i)];
                const double* Ui = U_.data() + off_[static_cast<std::size_t>(i)];
                const double xi = y[i] / D_[static_cast<std::size_t>(i)];
                y[i] = xi;
                for (Index k = fi; k < i; ++k) y[k] -= Ui[k - fi] * xi;
            }
        }
        VectorXd x(n_);
        for (Index k = 0; k < n_; ++k) x[perm_[static_cast<std::size_t>(k)]] = y[k];
        return x;
    }

    bool used_pivoting_fallback() const { return banded_; }
    Index envelope_entries() const { return off_.empty() ? 0 : 2 * off_.back() + n_; }

private:
    Index n_ = 0;
    bool analyzed_ = false, banded_ = false;
    ComputationInfo info_ = InvalidInput;
    std::vector<int> perm_, inv_, first_;
    std::vector<Index> off_;
    std::vector<double> L_, U_, D_;
    // banded partial-pivoting fallback (LAPACK dgbtrf layout)
    Index kl_ = 0, ku_ = 0, ldab_ = 0;
    std::vector<double> ab_;
    std::vector<int> ipiv_;

    double& AB(Index i, Index j) { return ab_[static_cast<std::size_t>((kl_ + ku_ + i - j) + j * ldab_)]; }
    double ABc(Index i, Index j) const { return ab_[static_cast<std::size_t>((kl_ + ku_ + i - j) + j * ldab_)]; }

    void factorize_banded(const MatrixType& A) {
        banded_ = true;
        L_.clear(); U_.clear(); D_.clear();
        const auto& ptr = A.row_ptr();
        const auto& col = A.col_index();
        const auto& val = A.values();
        kl_ = ku_ = 0;
        for (Index i = 0; i < n_; ++i)
            for (Index k = ptr[static_cast<std::size_t>(i)]; k < ptr[static_cast<std::size_t>(i) + 1]; ++k) {
                Index pi = inv_[static_cast<std::size_t>(i)], pj = inv_[static_cast<std::size_t>(col[static_cast<std::size_t>(k)])];
                kl_ = std::max(kl_, pi - pj);
                ku_ = std::max(ku_, pj - pi);
            }
        ldab_ = 2 * kl_ + ku_ + 1;
        ab_.assign(static_cast<std::size_t>(ldab_ * n_), 0.0);
        for (Index i = 0; i < n_; ++i)
            for (Index k = ptr[static_cast<std::size_t>(i)]; k < ptr[static_cast<std::size_t>(i) + 1]; ++k)
                AB(inv_[static_cast<std::size_t>(i)], inv_[static_cast<std::size_t>(col[static_cast<std::size_t>(k)])]) += val[static_cast<std::size_t>(k)];
        ipiv_.assign(static_cast<std::size_t>(n_), 0);
        const Index kv = kl_ + ku_;
        for (Index j = 0; j < n_; ++j) {
            const Index iend = std::min(n_ - 1, j + kl_);
            Index p = j;
            double best = std::abs(AB(j, j));
            for (Index i = j + 1; i <= iend; ++i)
                if (std::abs(AB(i, j)) > best) {
                    best = std::abs(AB(i, j));
                    p = i;
                }
            ipiv_[static_cast<std::size_t>(j)] = static_cast<int>(p);
            if (best == 0.0 || !std::isfinite(best)) {
                info_ = NumericalIssue;
                return;
            }
            const Index jend = std::min(n_ - 1, j + kv);
            if (p != j)
                for (Index c = j; c <= jend; ++c) std::swap(AB(j, c), AB(p, c));
            const double piv = AB(j, j);
            for (Index i = j + 1; i <= iend; ++i) AB(i, j) /= piv;
            for (Index c = j + 1; c <= jend; ++c) {
                const double u = AB(j, c);
                if (u == 0.0) continue;
                for (Index i = j + 1; i <= iend; ++i) AB(i, c) -= AB(i, j) * u;
            }
        }
    }

    void solve_banded(VectorXd& y) const {
        const Index kv = kl_ + ku_;
        for (Index j = 0; j < n_; ++j) {
            const Index p = ipiv_[static_cast<std::size_t>(j)];
            if (p != j) std::swap(y[j], y[p]);
            const Index iend = std::min(n_ - 1, j + kl_);
            for (Index i = j + 1; i <= iend; ++i) y[i] -= ABc(i, j) * y[j];
        }
        for (Index j = n_ - 1; j >= 0; --j) {
            y[j] /= ABc(j, j);
            const Index ibeg = std::max<Index>(0, j - kv);
            for (Index i = ibeg; i < j; ++i) y[i] -= ABc(i, j) * y[j];
        }
    }
};

}  // namespace Eigen

#endif  // ORACLE_EIGEN_SHIM_SPARSE_HPP
