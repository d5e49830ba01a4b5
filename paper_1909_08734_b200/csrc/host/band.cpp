// Band construction (restates proj/include/cpdd/band.hpp:78-182 and
// proj/include/cpdd/interp.hpp:35-91; see band.hpp here).
#include "band.hpp"
#include "decomp.hpp"

#include <algorithm>
#include <deque>
#include <numeric>
#include <string>

namespace cpddg {

// ---------------------------------------------------------------- LatticeMap

void LatticeMap::reserve(std::size_t n) {
    std::size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap <= keys_.size()) return;
    std::vector<std::uint64_t> ok = std::move(keys_);
    std::vector<std::int64_t> ov = std::move(vals_);
    keys_.assign(cap, 0);
    vals_.assign(cap, -1);
    mask_ = cap - 1;
    n_ = 0;
    for (std::size_t i = 0; i < ok.size(); ++i)
        if (ok[i]) insert(ok[i], ov[i]);
}

void LatticeMap::clear() {
    std::fill(keys_.begin(), keys_.end(), 0);
    std::fill(vals_.begin(), vals_.end(), -1);
    n_ = 0;
}

void LatticeMap::grow() { reserve(keys_.empty() ? 16 : keys_.size()); }

bool LatticeMap::insert(std::uint64_t key, std::int64_t val) {
    if (2 * (n_ + 1) > keys_.size()) grow();
    std::size_t i = mix(key) & mask_;
    while (keys_[i]) {
        if (keys_[i] == key) return false;
        i = (i + 1) & mask_;
    }
    keys_[i] = key;
    vals_[i] = val;
    ++n_;
    return true;
}

void LatticeMap::set(std::uint64_t key, std::int64_t val) {
    if (2 * (n_ + 1) > keys_.size()) grow();
    std::size_t i = mix(key) & mask_;
    while (keys_[i]) {
        if (keys_[i] == key) {
            vals_[i] = val;
            return;
        }
        i = (i + 1) & mask_;
    }
    keys_[i] = key;
    vals_[i] = val;
    ++n_;
}

std::int64_t LatticeMap::find(std::uint64_t key) const {
    if (keys_.empty()) return -1;
    std::size_t i = mix(key) & mask_;
    while (keys_[i]) {
        if (keys_[i] == key) return vals_[i];
        i = (i + 1) & mask_;
    }
    return -1;
}

// ------------------------------------------------------------------ stencils

void interp_weights_1d(int p, double t, double* w) {
    if (t < -1e-9 || t > p + 1e-9)
        throw InternalError("interp_weights_1d: offset " + std::to_string(t) +
                            " outside stencil range [0," + std::to_string(p) + "]");
    for (int j = 0; j <= p; ++j)
        if (std::abs(t - j) < 1e-12) {
            for (int k = 0; k <= p; ++k) w[k] = (k == j) ? 1.0 : 0.0;
            return;
        }
    double sum = 0.0, b = 1.0;
    for (int j = 0; j <= p; ++j) {
        w[j] = b / (t - j);
        sum += w[j];
        b *= -static_cast<double>(p - j) / (j + 1);
    }
    for (int j = 0; j <= p; ++j) w[j] /= sum;
}

template <int D>
Stencil1D<D> stencil_of(const Vec<D>& q, double h, int p) {
    if (p < 1 || p > 7) throw ConfigError("interpolation degree must be in [1,7]");
    Stencil1D<D> s;
    for (int a = 0; a < D; ++a) {
        const double g = (q[a] - 0.0) / h;  // true division, never a reciprocal multiply
        s.base[a] = stencil_base_1d(g, p);
        interp_weights_1d(p, g - s.base[a], s.w[a]);
    }
    return s;
}
template Stencil1D<2> stencil_of<2>(const Vec<2>&, double, int);
template Stencil1D<3> stencil_of<3>(const Vec<3>&, double, int);

// ---------------------------------------------------------------------- band

namespace {

template <int D>
struct Node {
    Ix<D> ix;
    CpResult<D> cp;
};

template <int D>
void close_stencils(const Surface<D>& surface, double h, int p, std::vector<Node<D>>& act, LatticeMap& amap,
                    int workers) {
    // closure under CP stencils (band.hpp:124-142): the final set is the
    // least closed superset, independent of visiting order, so it is built in
    // rounds -- check the newest nodes' stencils in parallel, add what is
    // missing (their CPs in parallel), repeat until nothing is added.
    const int pp = p + 1;
    int count = 1;
    for (int a = 0; a < D; ++a) count *= pp;
    std::size_t begin = 0;
    while (begin < act.size()) {
        const std::size_t end = act.size();
        const int n = static_cast<int>(end - begin);
        const int chunk = 4096;
        const int nch = (n + chunk - 1) / chunk;
        std::vector<std::vector<Ix<D>>> missing(static_cast<std::size_t>(nch));
        parallel_for(nch, workers, [&](int c, int) {
            const std::size_t e = std::min(end, begin + static_cast<std::size_t>(c + 1) * chunk);
            for (std::size_t w = begin + static_cast<std::size_t>(c) * chunk; w < e; ++w) {
                const Stencil1D<D> s = stencil_of<D>(act[w].cp.cp, h, p);
                for (int k = 0; k < count; ++k) {
                    Ix<D> q;
                    int rem = k;
                    for (int a = 0; a < D; ++a) {
                        q[a] = s.base[a] + rem % pp;
                        rem /= pp;
                    }
                    if (amap.find(LatticeMap::pack(q.data(), D)) < 0) missing[static_cast<std::size_t>(c)].push_back(q);
                }
            }
        });
        std::vector<Ix<D>> add;
        for (auto& m : missing)
            for (const auto& q : m)
                if (amap.insert(LatticeMap::pack(q.data(), D), static_cast<std::int64_t>(end + add.size())))
                    add.push_back(q);
        std::vector<CpResult<D>> cps(add.size());
        parallel_for(static_cast<int>(add.size()), workers, [&](int k, int) {
            cps[static_cast<std::size_t>(k)] = surface.closest_point(index_to_point<D>(add[static_cast<std::size_t>(k)], h));
        });
        for (std::size_t k = 0; k < add.size(); ++k) act.push_back({add[k], cps[k]});
        begin = end;
    }
}

}  // namespace

template <int D>
Band<D> build_band_tube(const Surface<D>& surface, double h, int p, double tube_radius, int workers) {
    if (h <= 0) throw ConfigError("grid spacing h must be positive");
    if (p < 1) throw ConfigError("interpolation degree must be at least 1");
    Band<D> g;
    g.h = h;
    g.p = p;
    g.tube_radius = tube_radius > 0 ? tube_radius : stencil_reach<D>(h, p);

    // flood fill from the node nearest a surface sample (band.hpp:158-176),
    // level-synchronous: the closest points of a whole BFS level are computed
    // in parallel, then the level is expanded serially.  The accepted set is
    // the connected component of {dist <= radius} containing the seed, as in
    // the reference's queue order (finalize sorts, so order is immaterial).
    std::vector<Node<D>> act;
    LatticeMap amap, seen;
    const Ix<D> seed = nearest_node<D>(surface.sample_point(), h);
    seen.insert(LatticeMap::pack(seed.data(), D), 0);
    std::vector<Ix<D>> level{seed}, next;
    std::vector<CpResult<D>> cps;
    Ix<D> nbr[2 * D];
    while (!level.empty()) {
        cps.resize(level.size());
        const int nl = static_cast<int>(level.size());
        const int chunk = 2048;
        parallel_for((nl + chunk - 1) / chunk, workers, [&](int c, int) {
            const int e = std::min(nl, (c + 1) * chunk);
            for (int q = c * chunk; q < e; ++q)
                cps[static_cast<std::size_t>(q)] = surface.closest_point(index_to_point<D>(level[static_cast<std::size_t>(q)], h));
        });
        next.clear();
        for (int q = 0; q < nl; ++q) {
            if (cps[static_cast<std::size_t>(q)].dist > g.tube_radius) continue;
            const Ix<D>& ix = level[static_cast<std::size_t>(q)];
            amap.insert(LatticeMap::pack(ix.data(), D), static_cast<std::int64_t>(act.size()));
            act.push_back({ix, cps[static_cast<std::size_t>(q)]});
            neighbors_of<D>(ix, nbr);
            for (int k = 0; k < 2 * D; ++k)
                if (seen.insert(LatticeMap::pack(nbr[k].data(), D), 0)) next.push_back(nbr[k]);
        }
        level.swap(next);
    }
    if (act.empty()) throw ConfigError("band is empty: grid spacing too large for the surface");
    close_stencils<D>(surface, h, p, act, amap, workers);

    // finalize (band.hpp:78-118): lexicographic actives, then ghosts
    std::sort(act.begin(), act.end(), [](const Node<D>& a, const Node<D>& b) { return a.ix < b.ix; });
    std::vector<Ix<D>> gh;
    {
        LatticeMap gseen;
        for (const auto& n : act) {
            neighbors_of<D>(n.ix, nbr);
            for (int k = 0; k < 2 * D; ++k) {
                const std::uint64_t key = LatticeMap::pack(nbr[k].data(), D);
                if (amap.find(key) >= 0) continue;
                if (gseen.insert(key, 0)) gh.push_back(nbr[k]);
            }
        }
    }
    std::sort(gh.begin(), gh.end());
    g.n_active = static_cast<int>(act.size());
    g.n_ghost = static_cast<int>(gh.size());
    const std::size_t nb = act.size() + gh.size();
    g.ix.resize(nb);
    g.cp.resize(nb);
    g.normal.resize(nb);
    g.dist.resize(nb);
    for (std::size_t k = 0; k < act.size(); ++k) {
        g.ix[k] = act[k].ix;
        g.cp[k] = act[k].cp.cp;
        g.normal[k] = act[k].cp.normal;
        g.dist[k] = act[k].cp.dist;
    }
    {
        const int ng = static_cast<int>(gh.size());
        const int chunk = 2048;
        parallel_for((ng + chunk - 1) / chunk, workers, [&](int cc, int) {
            const int e = std::min(ng, (cc + 1) * chunk);
            for (int k = cc * chunk; k < e; ++k) {
                const std::size_t c = act.size() + static_cast<std::size_t>(k);
                const CpResult<D> r = surface.closest_point(index_to_point<D>(gh[static_cast<std::size_t>(k)], h));
                g.ix[c] = gh[static_cast<std::size_t>(k)];
                g.cp[c] = r.cp;
                g.normal[c] = r.normal;
                g.dist[c] = r.dist;
            }
        });
    }
    g.map.reserve(nb);
    for (std::size_t k = 0; k < nb; ++k)
        g.map.insert(LatticeMap::pack(g.ix[k].data(), D), static_cast<std::int64_t>(k));
    const double kappa = surface.curvature_bound();
    if (kappa > 0) {
        const double ghost_reach = g.tube_radius + std::sqrt(double(D)) * h;
        if (ghost_reach >= 1.0 / kappa) g.tube_radius_warning = true;
    }
    return g;
}

template Band<2> build_band_tube<2>(const Surface<2>&, double, int, double, int);
template Band<3> build_band_tube<3>(const Surface<3>&, double, int, double, int);

}  // namespace cpddg
