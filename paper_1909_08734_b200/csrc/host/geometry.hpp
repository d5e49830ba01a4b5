// Host setup: fixed-dimension vector arithmetic and closest-point queries.
//
// Restates proj/include/cpdd/geometry.hpp (CpResult :25-30, circle :56-63,
// sphere :88-93, torus :95-114, TriMesh :120-409) on plain arrays.  Every
// reduction follows one canonical order, the one the reference's Eigen
// build uses for 2- and 3-vectors ((a0*b0 + a1*b1) + a2*b2, see
// oracle/shim/Eigen/ShimCore.hpp), so closest points, distances and hence
// band membership are bit-identical to the reference.  Compiled with
// -ffp-contract=off: no FMA contraction anywhere in setup code.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace cpddg {

// ---------------------------------------------------------------- errors
// Mirrors the reference hierarchy (proj/include/cpdd/core.hpp:73-95); the
// C ABI maps each to the status codes of include/cpddg.h.
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DivergenceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InternalError : std::logic_error {
    using std::logic_error::logic_error;
};

template <int D>
using Vec = std::array<double, D>;
template <int D>
using Ix = std::array<int, D>;

template <int D>
inline double dot(const Vec<D>& a, const Vec<D>& b) {
    if constexpr (D == 2)
        return a[0] * b[0] + a[1] * b[1];
    else
        return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
template <int D>
inline double norm(const Vec<D>& a) {
    return std::sqrt(dot<D>(a, a));
}
template <int D>
inline Vec<D> sub(const Vec<D>& a, const Vec<D>& b) {
    Vec<D> r;
    for (int k = 0; k < D; ++k) r[k] = a[k] - b[k];
    return r;
}
template <int D>
inline Vec<D> add(const Vec<D>& a, const Vec<D>& b) {
    Vec<D> r;
    for (int k = 0; k < D; ++k) r[k] = a[k] + b[k];
    return r;
}
template <int D>
inline Vec<D> scale(double s, const Vec<D>& a) {
    Vec<D> r;
    for (int k = 0; k < D; ++k) r[k] = s * a[k];
    return r;
}
template <int D>
inline Vec<D> divide(const Vec<D>& a, double s) {
    Vec<D> r;
    for (int k = 0; k < D; ++k) r[k] = a[k] / s;
    return r;
}
inline Vec<3> cross(const Vec<3>& a, const Vec<3>& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}

/** Lattice node position: origin + h * ix with origin 0 (band.hpp:40). */
template <int D>
inline Vec<D> index_to_point(const Ix<D>& ix, double h) {
    Vec<D> x;
    for (int a = 0; a < D; ++a) x[a] = 0.0 + h * ix[a];
    return x;
}

/** core.hpp:60-62. */
inline int round_half_up(double g) { return static_cast<int>(std::floor(g + 0.5)); }

/** core.hpp:64-69 (origin 0: (x - 0)/h). */
template <int D>
inline Ix<D> nearest_node(const Vec<D>& x, double h) {
    Ix<D> ix;
    for (int a = 0; a < D; ++a) ix[a] = round_half_up((x[a] - 0.0) / h);
    return ix;
}

template <int D>
struct CpResult {
    Vec<D> cp;
    Vec<D> normal;
    double dist;
};

enum class SurfaceKind : int { circle = 0, sphere = 1, torus = 2, trimesh = 3 };

class TriMesh;

/** Closest-point function of one surface (geometry.hpp:427-519). */
template <int D>
struct Surface {
    SurfaceKind kind = SurfaceKind::circle;
    double radius = 1.0;              // circle, sphere
    double major_R = 2.0 / 3.0;       // torus
    double minor_r = 1.0 / 3.0;
    std::shared_ptr<const TriMesh> mesh;

    CpResult<D> closest_point(const Vec<D>& x) const;
    Vec<D> sample_point() const;
    double curvature_bound() const;  // < 0: unknown (triangle meshes)
};

/** Flattened TriMesh tables for the device closest-point query
 *  (setup_dev.cu): per triangle its vertices, face normal, validity and the
 *  three edge pseudo-normals (edges ab, ac, bc = features 3, 4, 5); the
 *  spatial hash as cell keys (sorted) with CSR triangle lists in the hash's
 *  insertion order. */
struct TriMeshTables {
    std::vector<double> verts, vert_n;   // 3 per vertex
    std::vector<int> tris;               // 3 per triangle
    std::vector<double> face_n;          // 3 per triangle
    std::vector<double> edge_n;          // 9 per triangle
    std::vector<unsigned char> face_ok;  // 1 per triangle
    std::vector<std::uint64_t> cell_keys;
    std::vector<int> cell_start, cell_tris;
    double cell = 1.0;
    int max_ring = 0;
};

/** Triangulated surface (geometry.hpp:120-409): uniform spatial hash, angle-
 *  weighted vertex/edge pseudo-normals, nearest triangle by expanding rings. */
class TriMesh {
public:
    TriMesh(std::vector<Vec<3>> verts, std::vector<std::array<int, 3>> tris);
    static TriMesh load_obj(const std::string& path);
    CpResult<3> closest_point(const Vec<3>& x) const;
    const std::vector<Vec<3>>& vertices() const { return verts_; }
    const std::vector<std::array<int, 3>>& triangles() const { return tris_; }
    int degenerate_count() const { return n_degenerate_; }
    TriMeshTables tables() const;

private:
    std::vector<Vec<3>> verts_;
    std::vector<std::array<int, 3>> tris_;
    std::vector<Vec<3>> face_n_, vert_n_;
    std::vector<char> face_ok_;
    std::unordered_map<std::uint64_t, Vec<3>> edge_n_;
    std::unordered_map<std::uint64_t, std::vector<int>> cells_;
    double cell_ = 1.0;
    int max_ring_ = 0;
    int n_degenerate_ = 0, n_valid_ = 0;

    void build_normals();
    void build_hash();
    Ix<3> cell_of(const Vec<3>& x) const;
    void consider(int t, const Vec<3>& x, double& best, Vec<3>& best_cp, int& best_tri,
                  int& best_feat) const;
    Vec<3> feature_normal(int tri, int feat) const;
};

}  // namespace cpddg
