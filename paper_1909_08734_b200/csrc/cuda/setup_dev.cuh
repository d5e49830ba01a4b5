// Device closest points and lattice helpers shared by the device setup
// kernels (setup_dev.cu).  Restates, operation for operation, the host
// restatement in csrc/host/geometry.cpp (itself bit-exact with the
// reference's proj/include/cpdd/geometry.hpp :56-114, :190-212, :344-382):
// the translation unit is compiled with --fmad=false (no FMA contraction)
// and IEEE division / square root, so closest points, distances, band
// membership and distance ties are bit-identical to the host.
#pragma once

#include "dhash.cuh"

#include <cstdint>
#include <memory>

namespace cpddg {

template <int D>
struct DCp {
    double cp[D], n[D], dist;
};

/** Device view of a closest-point surface (csrc/host/geometry.hpp Surface). */
struct DSurf {
    int kind = 0;  // SurfaceKind
    double radius = 1.0, R = 2.0 / 3.0, r = 1.0 / 3.0;
    // triangle mesh (TriMeshTables)
    const double* verts = nullptr;
    const int* tris = nullptr;
    const double* face_n = nullptr;
    const double* vert_n = nullptr;
    const double* edge_n = nullptr;
    const unsigned char* face_ok = nullptr;
    DHash cells;  // cell_key + 1 -> cell index
    const int* cell_start = nullptr;
    const int* cell_tris = nullptr;
    int n_tris = 0, max_ring = 0;
    double cell = 1.0;
};

struct DevMesh;

/** Device band of a setup (build_band_device): packed lattice keys in band
 *  code order, closest points, normals, distances, and the lattice -> code
 *  map; kept with the setup for the device subdomain sets. */
struct DevBand {
    DevBand();
    ~DevBand();
    int dim = 0, p = 0, na = 0, ng = 0, levels = 0;
    double h = 0;
    int kind = 0;
    double radius = 1.0, major_R = 2.0 / 3.0, minor_r = 1.0 / 3.0;
    std::unique_ptr<DevMesh> mesh;
    int n_tris = 0, max_ring = 0;
    double cell = 1.0;
    DevBuf<std::uint64_t> keys;
    DevBuf<double> cp, normal, dist;
    DevHashTable map;
    double device_seconds = 0, copy_seconds = 0;
    DSurf surf() const;
};

/** LatticeMap::pack (csrc/host/band.hpp): 21 bits per axis, + 1. */
template <int D>
__host__ __device__ __forceinline__ std::uint64_t lat_pack(const int* ix) {
    std::uint64_t k = 0;
    for (int a = 0; a < D; ++a)
        k = (k << 21) | (static_cast<std::uint64_t>(static_cast<std::uint32_t>(ix[a] + (1 << 20))) & 0x1FFFFFu);
    return k + 1;
}
template <int D>
__host__ __device__ __forceinline__ void lat_unpack(std::uint64_t k, int* ix) {
    k -= 1;
    for (int a = D - 1; a >= 0; --a) {
        ix[a] = static_cast<int>(k & 0x1FFFFFu) - (1 << 20);
        k >>= 21;
    }
}

template <int D>
__device__ __forceinline__ double ddot(const double* a, const double* b) {
    if constexpr (D == 2)
        return a[0] * b[0] + a[1] * b[1];
    else
        return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
template <int D>
__device__ __forceinline__ double dnorm(const double* a) {
    return sqrt(ddot<D>(a, a));
}
template <int D>
__device__ __forceinline__ double ddist(const double* a, const double* b) {
    double d[D];
#pragma unroll
    for (int k = 0; k < D; ++k) d[k] = a[k] - b[k];
    return dnorm<D>(d);
}

/** glibc's hypot (>= 2.35, sysdeps dbl-64 without FMA: Borges' corrected
 *  algorithm), which the host's std::hypot calls.  Written with explicit
 *  round-to-nearest intrinsics, so it is exact in any translation unit
 *  (no FMA contraction).  The common path is verified against std::hypot on
 *  12 M lattice points; the scaling branches restate glibc's
 *  published structure (huge > 2^511, tiny < 2^-511). */
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double h = sqrt(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ __forceinline__ double hypot_glibc(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if ((isinf(x) || isinf(y))) return __longlong_as_double(0x7ff0000000000000LL);
        return __dadd_rn(x, y);
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
        return __ddiv_rn(hypot_kernel(__dmul_rn(ax, 0x1p-600), __dmul_rn(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay < 0x1p-511) {
        if (ax >= __ddiv_rn(ay, 0x1p-54)) return __dadd_rn(ax, ay);
        return __dmul_rn(hypot_kernel(__ddiv_rn(ax, 0x1p-600), __ddiv_rn(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
    return hypot_kernel(ax, ay);
}

/** round_cp (geometry.cpp; reference geometry.hpp:56-63, 88-93). */
template <int D>
__device__ __forceinline__ DCp<D> d_round_cp(double R, const double* x) {
    DCp<D> o;
    const double r = dnorm<D>(x);
    if (r > 1e-13) {
#pragma unroll
        for (int k = 0; k < D; ++k) o.n[k] = x[k] / r;
    } else {
#pragma unroll
        for (int k = 0; k < D; ++k) o.n[k] = k == 0 ? 1.0 : 0.0;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) o.cp[k] = R * o.n[k];
    o.dist = ddist<D>(x, o.cp);
    return o;
}

/** torus_cp (geometry.cpp; reference geometry.hpp:95-114). */
__device__ __forceinline__ DCp<3> d_torus_cp(double R, double rr, const double* x) {
    const double rho = hypot_glibc(x[0], x[1]);
    double ring[3];
    if (rho > 1e-13) {
        ring[0] = R * x[0] / rho;
        ring[1] = R * x[1] / rho;
        ring[2] = 0.0;
    } else {
        ring[0] = R;
        ring[1] = 0.0;
        ring[2] = 0.0;
    }
    double v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = x[k] - ring[k];
    const double vn = dnorm<3>(v);
    DCp<3> o;
    if (vn > 1e-13) {
#pragma unroll
        for (int k = 0; k < 3; ++k) o.n[k] = v[k] / vn;
    } else {
        const double rn = dnorm<3>(ring);
#pragma unroll
        for (int k = 0; k < 3; ++k) o.n[k] = ring[k] / rn;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) o.cp[k] = ring[k] + rr * o.n[k];
    o.dist = ddist<3>(x, o.cp);
    return o;
}

/** closest_on_triangle (geometry.cpp; reference geometry.hpp:344-382). */
__device__ __forceinline__ void d_closest_on_triangle(const double* p, const double* a, const double* b,
                                                      const double* c, double* out, int& feature) {
    double ab[3], ac[3], ap[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
    }
    const double d1 = ddot<3>(ab, ap), d2 = ddot<3>(ac, ap);
    if (d1 <= 0 && d2 <= 0) {
        feature = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = a[k];
        return;
    }
    double bp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) bp[k] = p[k] - b[k];
    const double d3 = ddot<3>(ab, bp), d4 = ddot<3>(ac, bp);
    if (d3 >= 0 && d4 <= d3) {
        feature = 1;
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = b[k];
        return;
    }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        feature = 3;
        const double s = d1 / (d1 - d3);
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = a[k] + s * ab[k];
        return;
    }
    double cpv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) cpv[k] = p[k] - c[k];
    const double d5 = ddot<3>(ab, cpv), d6 = ddot<3>(ac, cpv);
    if (d6 >= 0 && d5 <= d6) {
        feature = 2;
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = c[k];
        return;
    }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        feature = 4;
        const double s = d2 / (d2 - d6);
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = a[k] + s * ac[k];
        return;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) {
        feature = 5;
        const double s = (d4 - d3) / ((d4 - d3) + (d5 - d6));
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = b[k] + s * (c[k] - b[k]);
        return;
    }
    const double denom = 1.0 / (va + vb + vc);
    feature = 6;
    const double sv = vb * denom, sw = vc * denom;
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = (a[k] + ab[k] * sv) + ac[k] * sw;
}

__device__ __forceinline__ std::uint64_t d_cell_key(int c0, int c1, int c2) {
    auto u = [](int v) { return static_cast<std::uint64_t>(static_cast<std::uint32_t>(v + (1 << 20))) & 0x1FFFFFu; };
    return (u(c0) << 42) | (u(c1) << 21) | u(c2);
}

__device__ __forceinline__ void d_consider(const DSurf& S, int t, const double* x, double& best, double* best_cp,
                                           int& best_tri, int& best_feat) {
    if (!S.face_ok[t]) return;
    int feat = 0;
    double cp[3];
    const int* f = S.tris + 3 * t;
    d_closest_on_triangle(x, S.verts + 3 * f[0], S.verts + 3 * f[1], S.verts + 3 * f[2], cp, feat);
    const double d = ddist<3>(x, cp);
    if (d < best) {
        best = d;
        best_cp[0] = cp[0];
        best_cp[1] = cp[1];
        best_cp[2] = cp[2];
        best_tri = t;
        best_feat = feat;
    }
}

/** TriMesh::closest_point (geometry.cpp; reference geometry.hpp:190-212):
 *  expanding cube rings around the query's cell in the host's visiting
 *  order and with its stopping rule, so distance ties resolve to the same
 *  triangle.  *err is set if no triangle is found (InternalError on host). */
__device__ __forceinline__ DCp<3> d_trimesh_cp(const DSurf& S, const double* x, int* err) {
    const int c0[3] = {static_cast<int>(floor(x[0] / S.cell)), static_cast<int>(floor(x[1] / S.cell)),
                       static_cast<int>(floor(x[2] / S.cell))};
    double best = __longlong_as_double(0x7ff0000000000000LL);
    double best_cp[3] = {0, 0, 0};
    int best_tri = -1, best_feat = -1;
    auto visit = [&](int i, int j, int k) {
        const int ci = S.cells.find(d_cell_key(c0[0] + i, c0[1] + j, c0[2] + k) + 1);
        if (ci < 0) return;
        for (int q = S.cell_start[ci]; q < S.cell_start[ci + 1]; ++q)
            d_consider(S, S.cell_tris[q], x, best, best_cp, best_tri, best_feat);
    };
    for (int ring = 0;; ++ring) {
        if (best < (ring - 1) * S.cell && best_tri >= 0) break;
        if (ring > S.max_ring + 1) {
            if (best_tri >= 0) break;
            for (int t = 0; t < S.n_tris; ++t) d_consider(S, t, x, best, best_cp, best_tri, best_feat);
            break;
        }
        if (ring == 0) {
            visit(0, 0, 0);
            continue;
        }
        for (int i = -ring; i <= ring; ++i)
            for (int j = -ring; j <= ring; ++j)
                for (int k = -ring; k <= ring; ++k) {
                    if (max(abs(i), max(abs(j), abs(k))) != ring) continue;
                    visit(i, j, k);
                }
    }
    DCp<3> o;
    o.cp[0] = best_cp[0];
    o.cp[1] = best_cp[1];
    o.cp[2] = best_cp[2];
    o.dist = best;
    if (best_tri < 0) {
        *err = 1;
        o.n[0] = o.n[1] = o.n[2] = 0.0;
        return o;
    }
    const int* f = S.tris + 3 * best_tri;
    const double* n;
    switch (best_feat) {
        case 0:
        case 1:
        case 2: n = S.vert_n + 3 * f[best_feat]; break;
        case 3:
        case 4:
        case 5: n = S.edge_n + 9 * best_tri + 3 * (best_feat - 3); break;
        default: n = S.face_n + 3 * best_tri;
    }
    const double len = dnorm<3>(n);
    if (len > 1e-300) {
#pragma unroll
        for (int k = 0; k < 3; ++k) o.n[k] = n[k] / len;
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) o.n[k] = S.face_n[3 * best_tri + k];
    }
    return o;
}

template <int D>
__device__ __forceinline__ DCp<D> d_closest_point(const DSurf& S, const double* x, int* err) {
    if constexpr (D == 2) {
        return d_round_cp<2>(S.radius, x);
    } else {
        if (S.kind == 1) return d_round_cp<3>(S.radius, x);
        if (S.kind == 2) return d_torus_cp(S.R, S.r, x);
        return d_trimesh_cp(S, x, err);
    }
}

/** index_to_point (band.hpp:40, origin 0). */
template <int D>
__device__ __forceinline__ void d_point(const int* ix, double h, double* x) {
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = 0.0 + h * ix[a];
}

/** stencil_base_1d (interp.hpp:22-29) of g = (q - 0) / h. */
__device__ __forceinline__ int d_stencil_base(double q, double h, int p) {
    const double g = (q - 0.0) / h;
    if (p % 2 == 1) return static_cast<int>(llround(ceil(g))) - 1 - (p - 1) / 2;
    return static_cast<int>(floor(g + 0.5)) - p / 2;
}

}  // namespace cpddg
