// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// C API over the UNMODIFIED reference pipeline (/root/reference/proj/include,
// compiled against oracle/shim).  It replaces the CLI front end
// proj/tools/cpm.cpp (CLI11 is absent) with a handle-based interface so
// tests/ can read every intermediate of the reference setup (band, E, A,
// aligned partition, subdomain sets, local matrices) and bench.py's
// reference arm can time the reference solve.  Steps mirror run_solve
// (proj/include/cpdd/pipeline.hpp:183-241) one call each.
#include "cpdd/cpdd.hpp"

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <unistd.h>
#include <variant>

namespace {

using namespace cpdd;

void set_err(char* err, int n, const std::string& msg) {
    if (err && n > 0) std::snprintf(err, static_cast<std::size_t>(n), "%s", msg.c_str());
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

template <int D>
struct Impl {
    RunConfig cfg;
    std::unique_ptr<BuiltProblem<D>> P;
    std::vector<int> part;
    int align_moves = 0;
    std::vector<Subdomain<D>> subs;
    std::unique_ptr<SchwarzPreconditioner> M;
    std::vector<LocalOperator> locals_view;  // unfactored copies for export when requested
    double t_mesh_decomp = 0, t_locals = 0;
};

struct Handle {
    int dim = 0;
    std::variant<std::monostate, Impl<2>, Impl<3>> impl;
    std::unique_ptr<ThreadPool> pool;
    std::string last_error;
};

template <class F>
int guard(Handle* h, F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        if (h) h->last_error = std::string("ConfigError: ") + e.what();
        return 2;
    } catch (const DivergenceError& e) {
        if (h) h->last_error = std::string("DivergenceError: ") + e.what();
        return 3;
    } catch (const IoError& e) {
        if (h) h->last_error = std::string("IoError: ") + e.what();
        return 4;
    } catch (const InternalError& e) {
        if (h) h->last_error = std::string("InternalError: ") + e.what();
        return 1;
    } catch (const std::exception& e) {
        if (h) h->last_error = std::string("exception: ") + e.what();
        return 1;
    }
}

template <class F>
int visit(Handle* h, F&& f) {
    return guard(h, [&] {
        if (h->dim == 2)
            f(std::get<Impl<2>>(h->impl));
        else
            f(std::get<Impl<3>>(h->impl));
    });
}

RunConfig parse_ini(const char* text) {
    RunConfig cfg;
    std::istringstream in(text ? text : "");
    std::string line;
    while (std::getline(in, line)) {
        std::string t = detail::trim(line);
        if (t.empty() || t[0] == '#' || t[0] == ';') continue;
        if (t.front() == '[' && t.back() == ']') continue;
        auto eq = t.find('=');
        if (eq == std::string::npos) throw ConfigError("expected 'key = value', got '" + t + "'");
        apply_setting(cfg, detail::trim(t.substr(0, eq)), detail::trim(t.substr(eq + 1)));
    }
    validate(cfg);
    return cfg;
}

template <class T>
struct DimOf;
template <int D>
struct DimOf<Impl<D>> {
    static constexpr int value = D;
};

template <int D>
const SparseOperator& pick(const Impl<D>& I, int which) {
    return which == 0 ? I.P->E : I.P->A;
}

}  // namespace

extern "C" {

/** Parse an INI text (keys of proj/include/cpdd/config.hpp:104-180), build the
 *  problem (build_problem, pipeline.hpp:155-168). */
void* cref_create(const char* ini, int workers, char* err, int errlen) {
    auto* h = new Handle;
    int rc = guard(h, [&] {
        RunConfig cfg = parse_ini(ini);
        h->dim = dimension_of(cfg);
        h->pool = std::make_unique<ThreadPool>(workers > 0 ? workers : cfg.workers);
        if (h->dim == 2) {
            Impl<2> I;
            I.cfg = cfg;
            I.P = std::make_unique<BuiltProblem<2>>(build_problem<2>(cfg));
            h->impl = std::move(I);
        } else {
            Impl<3> I;
            I.cfg = cfg;
            I.P = std::make_unique<BuiltProblem<3>>(build_problem<3>(cfg));
            h->impl = std::move(I);
        }
    });
    if (rc != 0) {
        set_err(err, errlen, h->last_error);
        delete h;
        return nullptr;
    }
    return h;
}

void cref_destroy(void* hv) { delete static_cast<Handle*>(hv); }

int cref_last_error(void* hv, char* buf, int n) {
    set_err(buf, n, static_cast<Handle*>(hv)->last_error);
    return 0;
}

int cref_sizes(void* hv, int* dim, int* na, int* ng, int* p, double* h) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        *dim = H->dim;
        *na = I.P->grid.n_active();
        *ng = I.P->grid.n_ghost();
        *p = I.P->grid.p;
        *h = I.P->grid.h;
    });
}

double cref_phase(void* hv, int which) {
    auto* H = static_cast<Handle*>(hv);
    double v = -1;
    visit(H, [&](auto& I) {
        const PhaseTimings& t = I.P->timings;
        v = which == 0 ? t.mesh : which == 1 ? t.global_matrix : which == 2 ? t.local_operators : t.solve;
    });
    return v;
}

/** Band nodes in band-code order (actives then ghosts): lattice index, x, cp,
 *  normal, dist (band.hpp:29-34, 36-60). */
int cref_band(void* hv, int* ix, double* x, double* cp, double* nrm, double* dist) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const auto& g = I.P->grid;
        constexpr int D = DimOf<std::decay_t<decltype(I)>>::value;
        const int nb = g.n_active() + g.n_ghost();
        for (int k = 0; k < nb; ++k) {
            const auto& n = g.node(k);
            for (int a = 0; a < D; ++a) {
                ix[k * D + a] = n.ix[a];
                x[k * D + a] = n.x[a];
                cp[k * D + a] = n.cp.cp[a];
                nrm[k * D + a] = n.cp.normal[a];
            }
            dist[k] = n.cp.dist;
        }
    });
}

long long cref_nnz(void* hv, int which) {
    auto* H = static_cast<Handle*>(hv);
    long long v = -1;
    visit(H, [&](auto& I) { v = pick(I, which).nonzeros(); });
    return v;
}

/** CSR of E (which=0, operators.hpp:30-51) or A (which=1, operators.hpp:96-112). */
int cref_csr(void* hv, int which, long long* ptr, int* col, double* val) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const SparseOperator& S = pick(I, which);
        for (std::size_t k = 0; k < S.row_ptr().size(); ++k) ptr[k] = S.row_ptr()[k];
        std::memcpy(col, S.col_index().data(), S.col_index().size() * sizeof(int));
        std::memcpy(val, S.values().data(), S.values().size() * sizeof(double));
    });
}

int cref_rhs(void* hv, double* b) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        std::memcpy(b, I.P->b.data(), sizeof(double) * static_cast<std::size_t>(I.P->b.size()));
    });
}

/** y = A x through SparseOperator::apply (sparse.hpp:65-75). */
int cref_apply_A(void* hv, const double* x, double* y) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const int n = I.P->A.cols();
        Eigen::VectorXd xv = Eigen::Map<Eigen::VectorXd>(x, n);
        Eigen::VectorXd yv = I.P->A.apply(xv);
        std::memcpy(y, yv.data(), sizeof(double) * static_cast<std::size_t>(n));
    });
}

/** Decompose (pipeline.hpp:186-216): load the partition through the
 *  reference's load_partition (file written from `part_in`, or cfg
 *  partition_in if part_in is NULL), align_interfaces, build_subdomains, and
 *  assemble (+factor) the locals on the thread pool.  part_out receives the
 *  aligned labels. */
int cref_decompose(void* hv, const int* part_in, int* part_out, int* moves, int factor) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        double t0 = now_s();
        if (std::getenv("CREF_DEBUG")) std::fprintf(stderr, "enter\n");
        auto& P = *I.P;
        const SolverConfig& sc = I.cfg.solver;
        NodeGraph graph = build_graph(P.grid);
        (void)graph;
        std::string path = I.cfg.partition_in;
        std::string tmp;
        if (part_in) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "/tmp/cref_part_%d_%p.txt", static_cast<int>(getpid()),
                          static_cast<void*>(H));
            tmp = buf;
            std::ofstream out(tmp);
            for (int i = 0; i < P.grid.n_active(); ++i) out << part_in[i] << "\n";
            path = tmp;
        }
        if (path.empty())
            I.part = partition_graph(graph, sc.n_subdomains, sc.seed);
        else {
            I.part = load_partition(path, P.grid.n_active());
            const int np = *std::max_element(I.part.begin(), I.part.end()) + 1;
            if (np != sc.n_subdomains)
                throw ConfigError("partition file defines " + std::to_string(np) +
                                  " parts but n_subdomains = " + std::to_string(sc.n_subdomains));
        }
        if (!tmp.empty()) std::remove(tmp.c_str());
        if (std::getenv("CREF_DEBUG")) std::fprintf(stderr, "loaded\n");
        I.align_moves = align_interfaces(P.grid, I.part, P.grid.p);
        if (std::getenv("CREF_DEBUG")) std::fprintf(stderr, "aligned\n");
        I.subs = build_subdomains(P.grid, P.surface, I.part, P.E, sc.n_overlap, sc.robin());
        double t1 = now_s();
        if (std::getenv("CREF_DEBUG")) std::fprintf(stderr, "subdomains\n");
        TransmissionSpec spec;
        spec.kind = sc.robin() ? TransmissionSpec::Kind::robin : TransmissionSpec::Kind::dirichlet;
        spec.alpha = sc.alpha;
        spec.alpha_cross = sc.effective_alpha_cross();
        std::vector<LocalOperator> locals(I.subs.size());
        auto build_one = [&](int j) { locals[j] = assemble_local(P.grid, P.A, I.subs[j], spec, factor != 0); };
        H->pool->run_batch(static_cast<int>(I.subs.size()), build_one);
        double t2 = now_s();
        I.M = std::make_unique<SchwarzPreconditioner>(std::move(locals), P.grid.n_active(), H->pool.get());
        I.t_mesh_decomp = t1 - t0;
        I.t_locals = t2 - t1;
        if (part_out) std::memcpy(part_out, I.part.data(), sizeof(int) * I.part.size());
        if (moves) *moves = I.align_moves;
    });
}

double cref_decompose_time(void* hv, int which) {
    auto* H = static_cast<Handle*>(hv);
    double v = -1;
    visit(H, [&](auto& I) { v = which == 0 ? I.t_mesh_decomp : I.t_locals; });
    return v;
}

int cref_n_sub(void* hv) {
    auto* H = static_cast<Handle*>(hv);
    int n = -1;
    visit(H, [&](auto& I) { n = static_cast<int>(I.subs.size()); });
    return n;
}

/** counts[0..7] = |disjoint|, |overlap|, |final_layer|, |ghosts|, |bc|,
 *  fallback_count, n_lambda, n_cross_flagged. */
int cref_sub_counts(void* hv, int j, int* counts) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const auto& S = I.subs.at(static_cast<std::size_t>(j));
        counts[0] = static_cast<int>(S.disjoint.size());
        counts[1] = static_cast<int>(S.overlap.size());
        counts[2] = static_cast<int>(S.final_layer.size());
        counts[3] = static_cast<int>(S.ghosts.size());
        counts[4] = static_cast<int>(S.bc.size());
        counts[5] = S.fallback_count;
        counts[6] = S.n_lambda;
        int nc = 0;
        for (const auto& b : S.bc) nc += b.cross_flagged ? 1 : 0;
        counts[7] = nc;
    });
}

/** Index sets of subdomain j (subdomain.hpp:47-56) and its boundary nodes
 *  (subdomain.hpp:30-44).  bc_int is |bc| x (D + 4): ix..., global_active,
 *  is_ghost_type, cross_flagged, fallback.  bc_real is |bc| x (4D + 1):
 *  x, cp, cp_local, conormal, dq. */
int cref_sub_sets(void* hv, int j, int* disjoint, int* overlap, int* final_layer, int* ghosts,
                  int* bc_int, double* bc_real) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const auto& S = I.subs.at(static_cast<std::size_t>(j));
        constexpr int D = DimOf<std::decay_t<decltype(I)>>::value;
        std::copy(S.disjoint.begin(), S.disjoint.end(), disjoint);
        std::copy(S.overlap.begin(), S.overlap.end(), overlap);
        std::copy(S.final_layer.begin(), S.final_layer.end(), final_layer);
        std::copy(S.ghosts.begin(), S.ghosts.end(), ghosts);
        for (std::size_t b = 0; b < S.bc.size(); ++b) {
            const auto& n = S.bc[b];
            int* qi = bc_int + b * (D + 4);
            for (int a = 0; a < D; ++a) qi[a] = n.ix[a];
            qi[D] = n.global_active;
            qi[D + 1] = n.is_ghost_type;
            qi[D + 2] = n.cross_flagged;
            qi[D + 3] = n.fallback;
            double* qr = bc_real + b * (4 * D + 1);
            for (int a = 0; a < D; ++a) {
                qr[a] = n.x[a];
                qr[D + a] = n.cp[a];
                qr[2 * D + a] = n.cp_local[a];
                qr[3 * D + a] = n.conormal[a];
            }
            qr[4 * D] = n.dq;
        }
    });
}

/** Local operator j (transmission.hpp:47-70): sizes[0..3] = n_overlap, n_bc,
 *  nnz, |scatter|. */
int cref_local_sizes(void* hv, int j, long long* sizes) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const LocalOperator& L = I.M->locals().at(static_cast<std::size_t>(j));
        sizes[0] = L.n_overlap;
        sizes[1] = L.n_bc;
        sizes[2] = L.A.nonzeros();
        sizes[3] = static_cast<long long>(L.scatter.size());
    });
}

int cref_local(void* hv, int j, long long* ptr, int* col, double* val, int* sc_local,
               int* sc_global) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const LocalOperator& L = I.M->locals().at(static_cast<std::size_t>(j));
        for (std::size_t k = 0; k < L.A.row_ptr().size(); ++k) ptr[k] = L.A.row_ptr()[k];
        std::memcpy(col, L.A.col_index().data(), L.A.col_index().size() * sizeof(int));
        std::memcpy(val, L.A.values().data(), L.A.values().size() * sizeof(double));
        for (std::size_t k = 0; k < L.scatter.size(); ++k) {
            sc_local[k] = L.scatter[k].first;
            sc_global[k] = L.scatter[k].second;
        }
    });
}

/** z = M r through SchwarzPreconditioner::apply (solve.hpp:64-86). */
int cref_pc_apply(void* hv, const double* r, double* z) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const int n = I.P->grid.n_active();
        Eigen::VectorXd rv = Eigen::Map<Eigen::VectorXd>(r, n);
        Eigen::VectorXd zv = I.M->apply(rv);
        std::memcpy(z, zv.data(), sizeof(double) * static_cast<std::size_t>(n));
    });
}

/** Solve A u = b with the configured mode (gmres_solve / stationary_solve,
 *  solve.hpp:95-214) and the decomposed preconditioner.  b == NULL uses the
 *  problem's rhs.  Returns the residual history (up to cap entries),
 *  iterations, converged flag, final true residual and solve seconds. */
int cref_solve(void* hv, const double* b, double* u, double* residuals, int cap, int* n_res,
               int* iters, int* converged, double* final_true, double* seconds) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const int n = I.P->grid.n_active();
        Eigen::VectorXd bv = b ? Eigen::VectorXd(Eigen::Map<Eigen::VectorXd>(b, n)) : I.P->b;
        const SolverConfig& sc = I.cfg.solver;
        double t0 = now_s();
        SolveResult res =
            sc.mode == SolverConfig::Mode::gmres
                ? gmres_solve(I.P->A, bv, I.M.get(), sc.rel_tol, effective_max_iter(sc), sc.gmres_restart)
                : stationary_solve(I.P->A, bv, *I.M, sc.rel_tol, effective_max_iter(sc));
        *seconds = now_s() - t0;
        if (u) std::memcpy(u, res.u.data(), sizeof(double) * static_cast<std::size_t>(n));
        *n_res = static_cast<int>(res.log.residuals.size());
        for (int k = 0; k < std::min(cap, *n_res); ++k) residuals[k] = res.log.residuals[static_cast<std::size_t>(k)];
        *iters = res.log.iterations;
        *converged = res.log.converged;
        *final_true = res.log.final_true_residual;
    });
}

/** The reference's own run_solve (pipeline.hpp:183-241) end to end, with its
 *  PhaseTimings: t[0..3] = mesh, global_matrix, local_operators, solve. */
int cref_run_solve(void* hv, double* u, int* iters, int* converged, double* final_rel, double* t) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        constexpr int D = DimOf<std::decay_t<decltype(I)>>::value;
        SolveOutputs<D> out = run_solve<D>(I.cfg, *I.P, H->pool.get());
        const int n = I.P->grid.n_active();
        if (u) std::memcpy(u, out.u.data(), sizeof(double) * static_cast<std::size_t>(n));
        *iters = out.log.iterations;
        *converged = out.log.converged;
        *final_rel = out.final_relative_residual;
        t[0] = out.log.timings.mesh;
        t[1] = out.log.timings.global_matrix;
        t[2] = out.log.timings.local_operators;
        t[3] = out.log.timings.solve;
    });
}

/** Install subdomain systems given as the reference's own LocalOperator fields
 *  (transmission.hpp:47-70: n_overlap, n_bc, overlap, scatter, A) and factor
 *  each with the reference's DirectSolver (direct.hpp:41-52) on the thread
 *  pool, then build the SchwarzPreconditioner (solve.hpp:64-86).  Used by the
 *  CPU baseline at sizes where the reference's serial build_subdomains is too
 *  slow to run inside a benchmark (its outputs are bit-identical to the
 *  device path's setup; tests/test_setup_parity.py). */
int cref_set_locals(void* hv, int n_sub, const int* n_overlap, const int* n_bc, const int* const* overlap,
                    const int* n_scatter, const int* const* sc_local, const int* const* sc_global,
                    const long long* const* row_ptr, const int* const* col, const double* const* val) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        double t0 = now_s();
        std::vector<LocalOperator> locals(static_cast<std::size_t>(n_sub));
        auto build_one = [&](int j) {
            LocalOperator& L = locals[static_cast<std::size_t>(j)];
            L.id = j;
            L.n_overlap = n_overlap[j];
            L.n_bc = n_bc[j];
            L.overlap.assign(overlap[j], overlap[j] + n_overlap[j]);
            for (int k = 0; k < n_scatter[j]; ++k) L.scatter.emplace_back(sc_local[j][k], sc_global[j][k]);
            const int n = L.n_local();
            L.A = SparseOperator(n, n);
            std::vector<std::pair<int, double>> row;
            for (int r = 0; r < n; ++r) {
                for (long long k = row_ptr[j][r]; k < row_ptr[j][r + 1]; ++k) row.emplace_back(col[j][k], val[j][k]);
                L.A.append_row(row);
            }
            L.lu.factor(L.A, "subdomain " + std::to_string(j));
        };
        H->pool->run_batch(n_sub, build_one);
        I.M = std::make_unique<SchwarzPreconditioner>(std::move(locals), I.P->grid.n_active(), H->pool.get());
        I.t_locals = now_s() - t0;
    });
}

/** gmres_solve / stationary_solve with an explicit iteration cap and
 *  tolerance (a bounded sample of the configured solve). */
int cref_solve_capped(void* hv, const double* b, int max_iter, double rel_tol, int* iters, double* seconds,
                      double* last_residual) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const int n = I.P->grid.n_active();
        Eigen::VectorXd bv = Eigen::VectorXd(Eigen::Map<Eigen::VectorXd>(b, n));
        const SolverConfig& sc = I.cfg.solver;
        double t0 = now_s();
        SolveResult res = sc.mode == SolverConfig::Mode::gmres
                              ? gmres_solve(I.P->A, bv, I.M.get(), rel_tol, max_iter, sc.gmres_restart)
                              : stationary_solve(I.P->A, bv, *I.M, rel_tol, max_iter);
        *seconds = now_s() - t0;
        *iters = res.log.iterations;
        *last_residual = res.log.residuals.back();
    });
}

/** The reference's own writers (io.hpp:82-115) on the problem's band, a given
 *  solution / residual history and phase times (byte-format oracle). */
int cref_write_outputs(void* hv, const char* dir, const double* u, const double* residuals, int n_res,
                       const double* t4, int gmres_mode) {
    auto* H = static_cast<Handle*>(hv);
    return visit(H, [&](auto& I) {
        const int n = I.P->grid.n_active();
        Eigen::VectorXd uv = Eigen::VectorXd(Eigen::Map<Eigen::VectorXd>(u, n));
        write_solution(std::string(dir) + "/solution.csv", I.P->grid, uv);
        IterationLog log;
        log.residuals.assign(residuals, residuals + n_res);
        write_iterations(std::string(dir) + "/iterations.csv", log);
        PhaseTimings t;
        t.mesh = t4[0];
        t.global_matrix = t4[1];
        t.local_operators = t4[2];
        t.solve = t4[3];
        write_timings(std::string(dir) + "/timings.csv", t, gmres_mode != 0);
    });
}

}  // extern "C"
