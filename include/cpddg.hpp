// cpddg.hpp -- header-only drop-in adapter for callers of the reference
// library ("cpdd", proj/include/cpdd/).  Include it AFTER the reference
// headers; it adds device-backed twins of the reference's hot-path types and
// overloads of its solver entry points, with the same names, argument
// meaning, value semantics and exceptions:
//
//   reference                                    drop-in
//   -------------------------------------------  ---------------------------------------------
//   SparseOperator A = assemble_helmholtz(g,E,c)  DeviceHelmholtz A(g, c)
//     A.apply(x)           (sparse.hpp:65-75)       A.apply(x)
//   std::vector<LocalOperator> via assemble_local DeviceSchwarz M(locals, n)   (factor = false is
//     (transmission.hpp:73-138), SchwarzPreconditioner (solve.hpp:64-86)      enough: factors on device)
//     M.apply(r)                                    M.apply(r)
//   gmres_solve(A, b, &M, tol, it, restart)       gmres_solve(A, b, &M, tol, it, restart)
//   stationary_solve(A, b, M, tol, it)            stationary_solve(A, b, M, tol, it)
//
// Status codes of the C ABI are rethrown as the reference's ConfigError /
// DivergenceError / IoError / InternalError (core.hpp:73-95), so run_solve's
// error handling and the CLI exit codes are unchanged.  Vectors cross to the
// device once per call (H2D of the input, D2H of the output).
#pragma once

#include "cpddg.h"

#include <cuda_runtime_api.h>

#include <memory>
#include <string>
#include <vector>

namespace cpdd {

namespace cpddg_detail {

inline void check(int rc) {
    if (rc == CPDDG_OK) return;
    char buf[2048];
    cpddg_last_error(buf, sizeof buf);
    const std::string msg(buf);
    switch (rc) {
        case CPDDG_ERR_CONFIG: throw ConfigError(msg);
        case CPDDG_ERR_DIVERGENCE: throw DivergenceError(msg);
        case CPDDG_ERR_IO: throw IoError(msg);
        default: throw InternalError(msg);
    }
}

inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw InternalError(std::string("CUDA: ") + cudaGetErrorString(e));
}

/** Owning device vector. */
struct DVec {
    double* p = nullptr;
    int n = 0;
    explicit DVec(int n_) : n(n_) { cuda(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(double) * (n > 0 ? n : 1))); }
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    ~DVec() {
        if (p) cudaFree(p);
    }
    void upload(const Eigen::VectorXd& v) {
        cuda(cudaMemcpy(p, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    Eigen::VectorXd download() const {
        Eigen::VectorXd v(n);
        cuda(cudaMemcpy(v.data(), p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        return v;
    }
};

}  // namespace cpddg_detail

/** Device twin of the assembled Helmholtz SparseOperator (matrix-free). */
class DeviceHelmholtz {
public:
    template <int D>
    DeviceHelmholtz(const BandGrid<D>& g, double c) : n_(g.n_active()) {
        const int nb = g.n_active() + g.n_ghost();
        std::vector<int32_t> ix(static_cast<std::size_t>(nb) * D);
        std::vector<double> cp(static_cast<std::size_t>(nb) * D);
        for (int k = 0; k < nb; ++k) {
            const BandNode<D>& node = g.node(k);
            for (int a = 0; a < D; ++a) {
                ix[static_cast<std::size_t>(k) * D + a] = node.ix[a];
                cp[static_cast<std::size_t>(k) * D + a] = node.cp.cp[a];
            }
        }
        cpddg_band_desc d{D, g.p, g.n_active(), g.n_ghost(), g.h, c, ix.data(), cp.data()};
        cpddg_op* h = nullptr;
        cpddg_detail::check(cpddg_op_create(&d, &h));
        op_.reset(h);
    }
    int rows() const { return n_; }
    int cols() const { return n_; }
    cpddg_op* handle() const { return op_.get(); }

    /** y = A x (SparseOperator::apply, sparse.hpp:65-75). */
    Eigen::VectorXd apply(const Eigen::VectorXd& x) const {
        if (x.size() != n_) throw InternalError("sparse apply: size mismatch");
        cpddg_detail::DVec dx(n_), dy(n_);
        dx.upload(x);
        cpddg_detail::check(cpddg_op_apply(op_.get(), dx.p, dy.p, nullptr));
        return dy.download();
    }

private:
    struct Del {
        void operator()(cpddg_op* p) const { cpddg_op_destroy(p); }
    };
    std::unique_ptr<cpddg_op, Del> op_;
    int n_ = 0;
};

/** Device twin of SchwarzPreconditioner over the reference's LocalOperators
 *  (only their index maps and matrices are read; the LU happens on device). */
class DeviceSchwarz {
public:
    DeviceSchwarz(const std::vector<LocalOperator>& locals, int n_global) : n_(n_global) {
        std::vector<cpddg_local_desc> d(locals.size());
        std::vector<std::vector<int32_t>> sl(locals.size()), sg(locals.size());
        for (std::size_t j = 0; j < locals.size(); ++j) {
            const LocalOperator& L = locals[j];
            for (const auto& [loc, glob] : L.scatter) {
                sl[j].push_back(loc);
                sg[j].push_back(glob);
            }
            d[j] = cpddg_local_desc{L.n_overlap, L.n_bc, L.overlap.data(), static_cast<int>(sl[j].size()),
                                    sl[j].data(), sg[j].data(), L.A.row_ptr().data(), L.A.col_index().data(),
                                    L.A.values().data()};
        }
        cpddg_pc_options opt{0, 1};  // probe every local factor, like the Python path (api.py)
        cpddg_pc* h = nullptr;
        cpddg_detail::check(cpddg_pc_create(n_global, static_cast<int>(d.size()), d.data(), &opt, &h));
        pc_.reset(h);
    }
    int n_global() const { return n_; }
    cpddg_pc* handle() const { return pc_.get(); }

    /** z = sum_j Rt_j^T A_j^-1 R_j r (SchwarzPreconditioner::apply, solve.hpp:69-77). */
    Eigen::VectorXd apply(const Eigen::VectorXd& r) const {
        cpddg_detail::DVec dr(n_), dz(n_);
        dr.upload(r);
        cpddg_detail::check(cpddg_pc_apply(pc_.get(), dr.p, dz.p, nullptr));
        return dz.download();
    }

private:
    struct Del {
        void operator()(cpddg_pc* p) const { cpddg_pc_destroy(p); }
    };
    std::unique_ptr<cpddg_pc, Del> pc_;
    int n_ = 0;
};

namespace cpddg_detail {

template <class Fn>
SolveResult run(Fn&& fn, int n, const Eigen::VectorXd& b, double rel_tol, int max_iter, int restart) {
    DVec db(n), du(n);
    db.upload(b);
    std::vector<double> res(static_cast<std::size_t>(max_iter) + 2);
    cpddg_log log{};
    log.residuals = res.data();
    log.capacity = static_cast<int>(res.size());
    cpddg_solve_params prm{rel_tol, max_iter, restart, 0};
    check(fn(db.p, du.p, &prm, &log));
    SolveResult out;
    out.u = du.download();
    out.log.residuals.assign(res.begin(), res.begin() + std::min(log.n_residuals, log.capacity));
    out.log.iterations = log.iterations;
    out.log.converged = log.converged != 0;
    out.log.final_true_residual = log.final_true_residual;
    out.log.timings.solve = log.seconds;
    return out;
}

}  // namespace cpddg_detail

/** gmres_solve (solve.hpp:128-214) on the device path. */
inline SolveResult gmres_solve(const DeviceHelmholtz& A, const Eigen::VectorXd& b, const DeviceSchwarz* M,
                               double rel_tol, int max_iter, int restart = 0) {
    if (b.size() != A.rows()) throw InternalError("sparse apply: size mismatch");
    return cpddg_detail::run(
        [&](const double* db, double* du, const cpddg_solve_params* prm, cpddg_log* log) {
            return cpddg_gmres(A.handle(), M ? M->handle() : nullptr, db, du, prm, log, nullptr);
        },
        A.rows(), b, rel_tol, max_iter, restart);
}

/** stationary_solve (solve.hpp:95-123) on the device path. */
inline SolveResult stationary_solve(const DeviceHelmholtz& A, const Eigen::VectorXd& b, const DeviceSchwarz& M,
                                    double rel_tol, int max_iter) {
    if (b.size() != A.rows()) throw InternalError("sparse apply: size mismatch");
    return cpddg_detail::run(
        [&](const double* db, double* du, const cpddg_solve_params* prm, cpddg_log* log) {
            return cpddg_stationary(A.handle(), M.handle(), db, du, prm, log, nullptr);
        },
        A.rows(), b, rel_tol, max_iter, 0);
}

}  // namespace cpdd
