// C ABI: host setup (include/cpddg.h, "Host setup" section).
#include "setup.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstring>

namespace cpddg {

namespace {
thread_local std::string g_last_error;
thread_local int g_last_code = CPDDG_OK;
}  // namespace

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    g_last_code = code;
    return code;
}

namespace {

template <int D>
void create_impl(const cpddg_problem_desc& d, cpddg_setup* s) {
    auto* I = new SetupImpl<D>();
    s->impl = std::unique_ptr<void, void (*)(void*)>(I, [](void* p) { delete static_cast<SetupImpl<D>*>(p); });
    Surface<D>& S = I->surface;
    if constexpr (D == 2) {
        if (d.surface != CPDDG_CIRCLE) throw ConfigError("surface is not available in 2D");
        if (d.radius <= 0) throw ConfigError("circle radius must be positive");
        S.kind = SurfaceKind::circle;
        S.radius = d.radius;
    } else {
        switch (d.surface) {
            case CPDDG_SPHERE:
                if (d.radius <= 0) throw ConfigError("sphere radius must be positive");
                S.kind = SurfaceKind::sphere;
                S.radius = d.radius;
                break;
            case CPDDG_TORUS:
                if (!(d.minor_radius > 0 && d.minor_radius < d.major_radius))
                    throw ConfigError("torus radii must satisfy 0 < minor_r < major_R");
                S.kind = SurfaceKind::torus;
                S.major_R = d.major_radius;
                S.minor_r = d.minor_radius;
                break;
            case CPDDG_TRIMESH:
                if (!d.obj_path) throw ConfigError("surface obj requires the obj key");
                S.kind = SurfaceKind::trimesh;
                S.mesh = std::make_shared<const TriMesh>(TriMesh::load_obj(d.obj_path));
                break;
            default: throw ConfigError("surface is not available in 3D");
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    if (d.device_setup)
        I->band = build_band_device<D>(S, d.h, d.p, d.tube_radius, &I->dev);
    else
        I->band = build_band_tube<D>(S, d.h, d.p, d.tube_radius, d.workers);
    const auto t1 = std::chrono::steady_clock::now();
    I->E = build_extension<D>(I->band, d.workers);
    const auto t2 = std::chrono::steady_clock::now();
    I->A = assemble_helmholtz<D>(I->band, I->E, d.c, d.workers);
    const auto t3 = std::chrono::steady_clock::now();
    I->t_band = std::chrono::duration<double>(t1 - t0).count();
    I->t_E = std::chrono::duration<double>(t2 - t1).count();
    I->t_A = std::chrono::duration<double>(t3 - t2).count();
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] setup: band %.3f s, E %.3f s, A %.3f s\n",
                     std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
                     std::chrono::duration<double>(t3 - t2).count());
}

template <int D>
void decompose_impl(cpddg_setup* s, const int32_t* part, int n_part, int n_overlap, int method, double alpha,
                    double alpha_cross, int32_t* part_out, int* moves) {
    SetupImpl<D>& I = impl_of<D>(s);
    if (!part) throw ConfigError("a partition is required (partition_graph is not part of this path)");
    if (n_part != I.band.n_active)
        throw ConfigError("partition file has " + std::to_string(n_part) + " entries but the mesh has " +
                          std::to_string(I.band.n_active) + " active nodes");
    if (n_overlap < 1) throw ConfigError("n_overlap must be at least 1");
    const bool robin = method == CPDDG_ORAS;
    if (robin) {
        if (alpha <= 0) throw ConfigError("alpha must be positive for the Robin method");
        if (alpha_cross == 0) throw ConfigError("alpha_cross must be positive for the Robin method");
        if (alpha_cross >= 0 && alpha_cross < alpha) throw ConfigError("alpha_cross must be at least alpha");
    }
    I.part.assign(part, part + I.band.n_active);
    validate_partition(I.part, I.band.n_active);
    I.robin = robin;
    bool done = false;
    if (s->device_setup && I.dev) {
        // device sets; past their index limits (> 1023 subdomains, |lattice index| >= 2^17) the
        // host restatement below produces the identical result
        const std::vector<int> part0 = I.part;
        try {
            I.moves = decompose_device<D>(*I.dev, I.band, I.part, n_overlap, robin, I.subs, &I.t_align, &I.t_sets);
            done = true;
        } catch (const DeviceSetLimit&) {
            I.part = part0;
        }
    }
    if (!done) {
        const auto t0 = std::chrono::steady_clock::now();
        I.moves = align_interfaces<D>(I.band, I.part, I.band.p);
        const auto t1 = std::chrono::steady_clock::now();
        I.subs = build_subdomains<D>(I.band, I.surface, I.part, I.E, n_overlap, robin, s->workers);
        I.t_align = std::chrono::duration<double>(t1 - t0).count();
        I.t_sets = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    }
    const auto tl = std::chrono::steady_clock::now();
    TransmissionSpec spec;
    spec.robin = robin;
    spec.alpha = alpha;
    spec.alpha_cross = alpha_cross < 0 ? alpha : alpha_cross;
    I.locals = assemble_locals<D>(I.band, I.A, I.subs, spec, s->workers);
    I.t_local = std::chrono::duration<double>(std::chrono::steady_clock::now() - tl).count();
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] decompose: align %.3f s, sets %.3f s, local systems %.3f s\n", I.t_align,
                     I.t_sets, I.t_local);
    if (part_out) std::copy(I.part.begin(), I.part.end(), part_out);
    if (moves) *moves = I.moves;
}

template <class F>
void dispatch(const cpddg_setup* s, F&& f) {
    if (!s) throw InternalError("null setup handle");
    if (s->dim == 2)
        f(impl_of<2>(s));
    else
        f(impl_of<3>(s));
}

template <class T>
struct DimOf;
template <int D>
struct DimOf<SetupImpl<D>> {
    static constexpr int value = D;
};

}  // namespace
}  // namespace cpddg

using namespace cpddg;

extern "C" {

int cpddg_last_error(char* buf, size_t len) {
    if (buf && len > 0) {
        std::strncpy(buf, g_last_error.c_str(), len - 1);
        buf[len - 1] = '\0';
    }
    return g_last_code;
}

const char* cpddg_version(void) { return "cpddg 0.1 (sm_100a, FP64)"; }

int cpddg_setup_create(const cpddg_problem_desc* desc, cpddg_setup** out) {
    return guarded([&] {
        if (!desc || !out) throw InternalError("null argument");
        if (!(desc->h > 0)) throw ConfigError("grid spacing h must be positive");
        if (desc->p < 1 || desc->p > 7) throw ConfigError("interpolation degree p must be in 1..7");
        if (desc->c <= 0) throw ConfigError("c must be positive");
        auto s = std::make_unique<cpddg_setup>();
        s->dim = desc->dim;
        s->workers = desc->workers;
        s->device_setup = desc->device_setup;
        s->c = desc->c;
        if (desc->dim == 2)
            create_impl<2>(*desc, s.get());
        else if (desc->dim == 3)
            create_impl<3>(*desc, s.get());
        else
            throw ConfigError("dimension must be 2 or 3");
        *out = s.release();
    });
}

int cpddg_setup_timings(const cpddg_setup* s, double* t) {
    return guarded([&] {
        if (!t) throw InternalError("null argument");
        dispatch(s, [&](auto& I) {
            const double v[6] = {I.t_band, I.t_E, I.t_A, I.t_align, I.t_sets, I.t_local};
            std::copy(v, v + 6, t);
        });
    });
}

int cpddg_setup_destroy(cpddg_setup* s) {
    delete s;
    return CPDDG_OK;
}

int cpddg_setup_sizes(const cpddg_setup* s, int* n_active, int* n_ghost, int64_t* nnz_E, int64_t* nnz_A) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            if (n_active) *n_active = I.band.n_active;
            if (n_ghost) *n_ghost = I.band.n_ghost;
            if (nnz_E) *nnz_E = I.E.nnz();
            if (nnz_A) *nnz_A = I.A.nnz();
        });
    });
}

int cpddg_setup_band(const cpddg_setup* s, int32_t* ix, double* cp, double* normal, double* dist) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            constexpr int D = DimOf<std::decay_t<decltype(I)>>::value;
            const auto& g = I.band;
            for (int k = 0; k < g.n_band(); ++k) {
                for (int a = 0; a < D; ++a) {
                    if (ix) ix[k * D + a] = g.ix[static_cast<std::size_t>(k)][a];
                    if (cp) cp[k * D + a] = g.cp[static_cast<std::size_t>(k)][a];
                    if (normal) normal[k * D + a] = g.normal[static_cast<std::size_t>(k)][a];
                }
                if (dist) dist[k] = g.dist[static_cast<std::size_t>(k)];
            }
        });
    });
}

int cpddg_setup_csr(const cpddg_setup* s, int which, int64_t* row_ptr, int32_t* col, double* val) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            const Csr& M = which == 0 ? I.E : I.A;
            std::copy(M.ptr.begin(), M.ptr.end(), row_ptr);
            std::copy(M.col.begin(), M.col.end(), col);
            std::copy(M.val.begin(), M.val.end(), val);
        });
    });
}

int cpddg_setup_decompose(cpddg_setup* s, const int32_t* part, int n_part, int n_overlap, int method, double alpha,
                          double alpha_cross, int32_t* part_out, int* moves) {
    return guarded([&] {
        if (!s) throw InternalError("null setup handle");
        if (s->dim == 2)
            decompose_impl<2>(s, part, n_part, n_overlap, method, alpha, alpha_cross, part_out, moves);
        else
            decompose_impl<3>(s, part, n_part, n_overlap, method, alpha, alpha_cross, part_out, moves);
    });
}

int cpddg_setup_n_subdomains(const cpddg_setup* s) {
    int n = -1;
    guarded([&] { dispatch(s, [&](auto& I) { n = static_cast<int>(I.subs.size()); }); });
    return n;
}

int cpddg_setup_subdomain_counts(const cpddg_setup* s, int j, int32_t* counts) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            const auto& S = I.subs.at(static_cast<std::size_t>(j));
            counts[0] = static_cast<int32_t>(S.disjoint.size());
            counts[1] = static_cast<int32_t>(S.overlap.size());
            counts[2] = static_cast<int32_t>(S.final_layer.size());
            counts[3] = static_cast<int32_t>(S.ghosts.size());
            counts[4] = static_cast<int32_t>(S.bc.size());
            counts[5] = S.fallback_count;
            counts[6] = S.n_lambda;
            int nc = 0;
            for (const auto& b : S.bc) nc += b.cross_flagged ? 1 : 0;
            counts[7] = nc;
        });
    });
}

int cpddg_setup_subdomain_sets(const cpddg_setup* s, int j, int32_t* disjoint, int32_t* overlap,
                               int32_t* final_layer, int32_t* ghosts, int32_t* bc_int, double* bc_real) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            constexpr int D = DimOf<std::decay_t<decltype(I)>>::value;
            const auto& S = I.subs.at(static_cast<std::size_t>(j));
            std::copy(S.disjoint.begin(), S.disjoint.end(), disjoint);
            std::copy(S.overlap.begin(), S.overlap.end(), overlap);
            std::copy(S.final_layer.begin(), S.final_layer.end(), final_layer);
            std::copy(S.ghosts.begin(), S.ghosts.end(), ghosts);
            for (std::size_t b = 0; b < S.bc.size(); ++b) {
                const auto& n = S.bc[b];
                int32_t* qi = bc_int + b * (D + 4);
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
    });
}

int cpddg_setup_local_sizes(const cpddg_setup* s, int j, int64_t* sizes) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            const LocalSystem& L = I.locals.at(static_cast<std::size_t>(j));
            sizes[0] = L.n_overlap;
            sizes[1] = L.n_bc;
            sizes[2] = L.A.nnz();
            sizes[3] = static_cast<int64_t>(L.scatter_local.size());
        });
    });
}

int cpddg_setup_local(const cpddg_setup* s, int j, int64_t* row_ptr, int32_t* col, double* val,
                      int32_t* scatter_local, int32_t* scatter_global) {
    return guarded([&] {
        dispatch(s, [&](auto& I) {
            const LocalSystem& L = I.locals.at(static_cast<std::size_t>(j));
            std::copy(L.A.ptr.begin(), L.A.ptr.end(), row_ptr);
            std::copy(L.A.col.begin(), L.A.col.end(), col);
            std::copy(L.A.val.begin(), L.A.val.end(), val);
            std::copy(L.scatter_local.begin(), L.scatter_local.end(), scatter_local);
            std::copy(L.scatter_global.begin(), L.scatter_global.end(), scatter_global);
        });
    });
}

}  // extern "C"
