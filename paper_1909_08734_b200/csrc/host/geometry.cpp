// Closest-point queries (restates proj/include/cpdd/geometry.hpp; see
// geometry.hpp here for the bit-exactness rules).
#include "geometry.hpp"

#include <algorithm>
#include <fstream>
#include <limits>
#include <sstream>

namespace cpddg {

namespace {

// geometry.hpp:56-63 / :88-93: r = |x|, n = x/r (azimuth 0 at the centre),
// cp = R n, dist = |x - cp| (not |r - R|: different rounding).
template <int D>
CpResult<D> round_cp(double R, const Vec<D>& x) {
    const double r = norm<D>(x);
    Vec<D> n{};
    if (r > 1e-13) {
        n = divide<D>(x, r);
    } else {
        n[0] = 1.0;
    }
    const Vec<D> cp = scale<D>(R, n);
    return {cp, n, norm<D>(sub<D>(x, cp))};
}

// geometry.hpp:95-114.
CpResult<3> torus_cp(double R, double rr, const Vec<3>& x) {
    const double rho = std::hypot(x[0], x[1]);
    Vec<3> ring;
    if (rho > 1e-13)
        ring = {R * x[0] / rho, R * x[1] / rho, 0.0};
    else
        ring = {R, 0.0, 0.0};
    const Vec<3> v = sub<3>(x, ring);
    const double vn = norm<3>(v);
    Vec<3> n = vn > 1e-13 ? divide<3>(v, vn) : divide<3>(ring, norm<3>(ring));
    const Vec<3> cp = add<3>(ring, scale<3>(rr, n));
    return {cp, n, norm<3>(sub<3>(x, cp))};
}

Vec<3> normalized(const Vec<3>& v) {
    const double z = dot<3>(v, v);
    return z > 0 ? divide<3>(v, std::sqrt(z)) : v;
}

std::uint64_t edge_key(int a, int b) {
    if (a > b) std::swap(a, b);
    return (static_cast<std::uint64_t>(a) << 32) | static_cast<std::uint32_t>(b);
}

std::uint64_t cell_key(const Ix<3>& c) {
    auto u = [](int v) { return static_cast<std::uint64_t>(static_cast<std::uint32_t>(v + (1 << 20))) & 0x1FFFFFu; };
    return (u(c[0]) << 42) | (u(c[1]) << 21) | u(c[2]);
}

// Closest point on one triangle with the active feature
// (0/1/2 vertex, 3/4/5 edge ab/ac/bc, 6 interior): geometry.hpp:344-382.
Vec<3> closest_on_triangle(const Vec<3>& p, const Vec<3>& a, const Vec<3>& b, const Vec<3>& c,
                           int& feature) {
    const Vec<3> ab = sub<3>(b, a), ac = sub<3>(c, a), ap = sub<3>(p, a);
    const double d1 = dot<3>(ab, ap), d2 = dot<3>(ac, ap);
    if (d1 <= 0 && d2 <= 0) {
        feature = 0;
        return a;
    }
    const Vec<3> bp = sub<3>(p, b);
    const double d3 = dot<3>(ab, bp), d4 = dot<3>(ac, bp);
    if (d3 >= 0 && d4 <= d3) {
        feature = 1;
        return b;
    }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        feature = 3;
        return add<3>(a, scale<3>(d1 / (d1 - d3), ab));
    }
    const Vec<3> cp = sub<3>(p, c);
    const double d5 = dot<3>(ab, cp), d6 = dot<3>(ac, cp);
    if (d6 >= 0 && d5 <= d6) {
        feature = 2;
        return c;
    }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        feature = 4;
        return add<3>(a, scale<3>(d2 / (d2 - d6), ac));
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) {
        feature = 5;
        return add<3>(b, scale<3>((d4 - d3) / ((d4 - d3) + (d5 - d6)), sub<3>(c, b)));
    }
    const double denom = 1.0 / (va + vb + vc);
    feature = 6;
    const double sv = vb * denom, sw = vc * denom;
    Vec<3> r;
    for (int k = 0; k < 3; ++k) r[k] = (a[k] + ab[k] * sv) + ac[k] * sw;
    return r;
}

}  // namespace

// ------------------------------------------------------------------ Surface

template <>
CpResult<2> Surface<2>::closest_point(const Vec<2>& x) const {
    if (kind != SurfaceKind::circle) throw ConfigError("surface is not available in 2D");
    return round_cp<2>(radius, x);
}

template <>
CpResult<3> Surface<3>::closest_point(const Vec<3>& x) const {
    switch (kind) {
        case SurfaceKind::sphere: return round_cp<3>(radius, x);
        case SurfaceKind::torus: return torus_cp(major_R, minor_r, x);
        case SurfaceKind::trimesh: return mesh->closest_point(x);
        default: throw ConfigError("surface is not available in 3D");
    }
}

template <>
Vec<2> Surface<2>::sample_point() const {
    return {radius, 0.0};
}

template <>
Vec<3> Surface<3>::sample_point() const {
    switch (kind) {
        case SurfaceKind::sphere: return {radius, 0.0, 0.0};
        case SurfaceKind::torus: return {major_R + minor_r, 0.0, 0.0};
        case SurfaceKind::trimesh: return mesh->vertices().at(mesh->triangles()[0][0]);
        default: throw ConfigError("surface is not available in 3D");
    }
}

template <int D>
double Surface<D>::curvature_bound() const {
    switch (kind) {
        case SurfaceKind::circle:
        case SurfaceKind::sphere: return 1.0 / radius;
        case SurfaceKind::torus: return std::max(1.0 / minor_r, 1.0 / (major_R - minor_r));
        default: return -1.0;
    }
}
template double Surface<2>::curvature_bound() const;
template double Surface<3>::curvature_bound() const;

// ------------------------------------------------------------------ TriMesh

TriMesh::TriMesh(std::vector<Vec<3>> verts, std::vector<std::array<int, 3>> tris)
    : verts_(std::move(verts)), tris_(std::move(tris)) {
    if (tris_.empty()) throw ConfigError("triangle mesh has no triangles");
    for (const auto& t : tris_)
        for (int k = 0; k < 3; ++k)
            if (t[k] < 0 || t[k] >= static_cast<int>(verts_.size()))
                throw ConfigError("triangle index out of range");
    build_normals();
    build_hash();
    if (n_valid_ == 0) throw ConfigError("all triangles are degenerate");
}

TriMesh TriMesh::load_obj(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open OBJ file: " + path);
    std::vector<Vec<3>> vs;
    std::vector<std::array<int, 3>> fs;
    std::string line;
    while (std::getline(in, line)) {
        std::istringstream ls(line);
        std::string tag;
        if (!(ls >> tag)) continue;
        if (tag == "v") {
            Vec<3> v;
            if (!(ls >> v[0] >> v[1] >> v[2]))
                throw IoError("malformed vertex line in " + path + ": " + line);
            vs.push_back(v);
        } else if (tag == "f") {
            std::array<int, 3> f{};
            int k = 0;
            std::string tok;
            while (ls >> tok) {
                if (k >= 3) throw IoError("non-triangular face in " + path + ": " + line);
                const int idx = std::atoi(tok.c_str());
                if (idx <= 0 || idx > static_cast<int>(vs.size()))
                    throw IoError("face index out of range in " + path + ": " + line);
                f[k++] = idx - 1;
            }
            if (k != 3) throw IoError("non-triangular face in " + path + ": " + line);
            fs.push_back(f);
        }
    }
    if (fs.empty()) throw IoError("OBJ file has no triangular faces: " + path);
    return TriMesh(std::move(vs), std::move(fs));
}

void TriMesh::build_normals() {
    face_n_.assign(tris_.size(), Vec<3>{0, 0, 0});
    face_ok_.assign(tris_.size(), 0);
    vert_n_.assign(verts_.size(), Vec<3>{0, 0, 0});
    edge_n_.clear();
    n_degenerate_ = n_valid_ = 0;
    for (std::size_t t = 0; t < tris_.size(); ++t) {
        const auto& f = tris_[t];
        const Vec<3>&a = verts_[f[0]], &b = verts_[f[1]], &c = verts_[f[2]];
        Vec<3> n = cross(sub<3>(b, a), sub<3>(c, a));
        const double len = norm<3>(n);
        if (len < 1e-300) {
            ++n_degenerate_;
            continue;
        }
        ++n_valid_;
        n = divide<3>(n, len);
        face_n_[t] = n;
        face_ok_[t] = !(std::abs(n[0]) <= 1e-12 && std::abs(n[1]) <= 1e-12 && std::abs(n[2]) <= 1e-12);
        for (int k = 0; k < 3; ++k) {
            const Vec<3> e1 = normalized(sub<3>(verts_[f[(k + 1) % 3]], verts_[f[k]]));
            const Vec<3> e2 = normalized(sub<3>(verts_[f[(k + 2) % 3]], verts_[f[k]]));
            const double ang = std::acos(std::clamp(dot<3>(e1, e2), -1.0, 1.0));
            vert_n_[f[k]] = add<3>(vert_n_[f[k]], scale<3>(ang, n));
        }
        for (int k = 0; k < 3; ++k) {
            Vec<3>& e = edge_n_[edge_key(f[k], f[(k + 1) % 3])];
            e = add<3>(e, n);
        }
    }
}

Ix<3> TriMesh::cell_of(const Vec<3>& x) const {
    return {static_cast<int>(std::floor(x[0] / cell_)), static_cast<int>(std::floor(x[1] / cell_)),
            static_cast<int>(std::floor(x[2] / cell_))};
}

void TriMesh::build_hash() {
    cells_.clear();
    cell_ = 0.0;
    auto bbox = [&](std::size_t t, Vec<3>& lo, Vec<3>& hi) {
        const auto& f = tris_[t];
        lo = hi = verts_[f[0]];
        for (int k = 1; k < 3; ++k)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], verts_[f[k]][a]);
                hi[a] = std::max(hi[a], verts_[f[k]][a]);
            }
    };
    for (std::size_t t = 0; t < tris_.size(); ++t) {
        if (!face_ok_[t]) continue;
        Vec<3> lo, hi;
        bbox(t, lo, hi);
        cell_ = std::max(cell_, std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]}));
    }
    if (cell_ <= 0) cell_ = 1.0;
    Ix<3> clo{0, 0, 0}, chi{0, 0, 0};
    bool first = true;
    for (std::size_t t = 0; t < tris_.size(); ++t) {
        if (!face_ok_[t]) continue;
        Vec<3> lo, hi;
        bbox(t, lo, hi);
        const Ix<3> a = cell_of(lo), b = cell_of(hi);
        for (int i = a[0]; i <= b[0]; ++i)
            for (int j = a[1]; j <= b[1]; ++j)
                for (int k = a[2]; k <= b[2]; ++k)
                    cells_[cell_key({i, j, k})].push_back(static_cast<int>(t));
        if (first) {
            clo = a;
            chi = b;
            first = false;
        } else {
            for (int d = 0; d < 3; ++d) {
                clo[d] = std::min(clo[d], a[d]);
                chi[d] = std::max(chi[d], b[d]);
            }
        }
    }
    max_ring_ = 0;
    for (int d = 0; d < 3; ++d) max_ring_ = std::max(max_ring_, chi[d] - clo[d] + 2);
}

void TriMesh::consider(int t, const Vec<3>& x, double& best, Vec<3>& best_cp, int& best_tri,
                       int& best_feat) const {
    if (!face_ok_[t]) return;
    int feat = 0;
    const auto& f = tris_[t];
    const Vec<3> cp = closest_on_triangle(x, verts_[f[0]], verts_[f[1]], verts_[f[2]], feat);
    const double d = norm<3>(sub<3>(x, cp));
    if (d < best) {
        best = d;
        best_cp = cp;
        best_tri = t;
        best_feat = feat;
    }
}

Vec<3> TriMesh::feature_normal(int tri, int feat) const {
    if (tri < 0) throw InternalError("closest-point query found no triangle");
    const auto& f = tris_[tri];
    Vec<3> n;
    switch (feat) {
        case 0:
        case 1:
        case 2: n = vert_n_[f[feat]]; break;
        case 3: n = edge_n_.at(edge_key(f[0], f[1])); break;
        case 4: n = edge_n_.at(edge_key(f[0], f[2])); break;
        case 5: n = edge_n_.at(edge_key(f[1], f[2])); break;
        default: n = face_n_[tri];
    }
    const double len = norm<3>(n);
    return len > 1e-300 ? divide<3>(n, len) : face_n_[tri];
}

TriMeshTables TriMesh::tables() const {
    TriMeshTables T;
    for (const auto& v : verts_) T.verts.insert(T.verts.end(), v.begin(), v.end());
    for (const auto& v : vert_n_) T.vert_n.insert(T.vert_n.end(), v.begin(), v.end());
    for (std::size_t t = 0; t < tris_.size(); ++t) {
        const auto& f = tris_[t];
        T.tris.insert(T.tris.end(), f.begin(), f.end());
        T.face_n.insert(T.face_n.end(), face_n_[t].begin(), face_n_[t].end());
        T.face_ok.push_back(static_cast<unsigned char>(face_ok_[t]));
        const std::uint64_t ek[3] = {edge_key(f[0], f[1]), edge_key(f[0], f[2]), edge_key(f[1], f[2])};
        for (std::uint64_t k : ek) {
            auto it = edge_n_.find(k);
            const Vec<3> e = it == edge_n_.end() ? Vec<3>{0, 0, 0} : it->second;
            T.edge_n.insert(T.edge_n.end(), e.begin(), e.end());
        }
    }
    std::vector<std::uint64_t> keys;
    keys.reserve(cells_.size());
    for (const auto& kv : cells_) keys.push_back(kv.first);
    std::sort(keys.begin(), keys.end());
    T.cell_start.push_back(0);
    for (std::uint64_t k : keys) {
        const auto& l = cells_.at(k);
        T.cell_tris.insert(T.cell_tris.end(), l.begin(), l.end());
        T.cell_start.push_back(static_cast<int>(T.cell_tris.size()));
    }
    T.cell_keys = std::move(keys);
    T.cell = cell_;
    T.max_ring = max_ring_;
    return T;
}

// geometry.hpp:190-212: expanding cube rings around the query's cell, with
// the same visiting order (i, j, k nested, shell cells only) and the same
// stopping rule, so ties resolve to the same triangle.
CpResult<3> TriMesh::closest_point(const Vec<3>& x) const {
    const Ix<3> c0 = cell_of(x);
    double best = std::numeric_limits<double>::infinity();
    Vec<3> best_cp{0, 0, 0};
    int best_tri = -1, best_feat = -1;
    auto visit_cell = [&](const Ix<3>& c) {
        auto it = cells_.find(cell_key(c));
        if (it == cells_.end()) return;
        for (int t : it->second) consider(t, x, best, best_cp, best_tri, best_feat);
    };
    for (int ring = 0;; ++ring) {
        if (best < (ring - 1) * cell_ && best_tri >= 0) break;
        if (ring > max_ring_ + 1) {
            if (best_tri >= 0) break;
            for (int t = 0; t < static_cast<int>(tris_.size()); ++t)
                consider(t, x, best, best_cp, best_tri, best_feat);
            break;
        }
        if (ring == 0) {
            visit_cell(c0);
            continue;
        }
        for (int i = -ring; i <= ring; ++i)
            for (int j = -ring; j <= ring; ++j)
                for (int k = -ring; k <= ring; ++k) {
                    if (std::max({std::abs(i), std::abs(j), std::abs(k)}) != ring) continue;
                    visit_cell({c0[0] + i, c0[1] + j, c0[2] + k});
                }
    }
    return {best_cp, feature_normal(best_tri, best_feat), best};
}

}  // namespace cpddg
