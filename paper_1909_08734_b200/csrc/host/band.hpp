// Host setup: interpolation stencils and the computational band.
//
// Restates proj/include/cpdd/interp.hpp (stencil_base_1d :22-29,
// interp_weights_1d :35-54, interp_stencil :59-91, stencil_reach :95-98) and
// proj/include/cpdd/band.hpp (build_band_tube :150-182, close_stencils
// :124-142, finalize_band :78-118).  The band is kept as structure-of-arrays
// (lattice index, closest point, normal, distance per band code) with an
// open-addressing lattice map instead of std::unordered_map; ordering is the
// reference's: actives lexicographic by lattice index, then ghosts
// lexicographic, code = ordinal (ghosts offset by N_A).
#pragma once

#include "geometry.hpp"

#include <cstdint>
#include <vector>

namespace cpddg {

/** Open-addressing hash map from a packed lattice index to an int64 code. */
class LatticeMap {
public:
    static std::uint64_t pack(const int* ix, int dim) {
        std::uint64_t k = 0;
        for (int a = 0; a < dim; ++a)
            k = (k << 21) | (static_cast<std::uint64_t>(static_cast<std::uint32_t>(ix[a] + (1 << 20))) & 0x1FFFFFu);
        return k + 1;  // 0 marks an empty slot
    }
    void reserve(std::size_t n);
    void clear();
    /** Insert key -> val; returns false (and keeps the old value) if present. */
    bool insert(std::uint64_t key, std::int64_t val);
    std::int64_t find(std::uint64_t key) const;  // -1 if absent
    void set(std::uint64_t key, std::int64_t val);
    std::size_t size() const { return n_; }

private:
    std::vector<std::uint64_t> keys_;
    std::vector<std::int64_t> vals_;
    std::size_t mask_ = 0, n_ = 0;
    static std::size_t mix(std::uint64_t k) {
        k ^= k >> 33;
        k *= 0xff51afd7ed558ccdULL;
        k ^= k >> 33;
        k *= 0xc4ceb9fe1a85ec53ULL;
        k ^= k >> 33;
        return static_cast<std::size_t>(k);
    }
    void grow();
};

/** stencil_base_1d (interp.hpp:22-29). */
inline int stencil_base_1d(double g, int p) {
    if (p % 2 == 1) return static_cast<int>(std::lround(std::ceil(g))) - 1 - (p - 1) / 2;
    return round_half_up(g) - p / 2;
}

/** Barycentric weights on nodes 0..p at t (interp.hpp:35-54). */
void interp_weights_1d(int p, double t, double* w);

/** Per-axis stencil of q: base lattice coordinate and 1-D weights.  The
 *  tensor weight of node offset (o_0, .., o_{D-1}) is
 *  ((1 * w[0][o_0]) * w[1][o_1]) * w[2][o_2] (interp.hpp:77-83). */
template <int D>
struct Stencil1D {
    int base[D];
    double w[D][8];
};

template <int D>
Stencil1D<D> stencil_of(const Vec<D>& q, double h, int p);

/** stencil_reach (interp.hpp:95-98). */
template <int D>
inline double stencil_reach(double h, int p) {
    return 0.5 * (p + 1) * std::sqrt(static_cast<double>(D)) * h;
}

template <int D>
struct Band {
    double h = 0;
    int p = 0;
    double tube_radius = 0;
    bool tube_radius_warning = false;
    int n_active = 0, n_ghost = 0;
    std::vector<Ix<D>> ix;         // per band code
    std::vector<Vec<D>> cp, normal;
    std::vector<double> dist;
    LatticeMap map;

    int n_band() const { return n_active + n_ghost; }
    std::int64_t lookup(const Ix<D>& q) const { return map.find(LatticeMap::pack(q.data(), D)); }
    bool is_active(std::int64_t code) const { return code >= 0 && code < n_active; }
    Vec<D> x(std::int64_t code) const { return index_to_point<D>(ix[static_cast<std::size_t>(code)], h); }
};

/** Axis neighbours in the reference order: axis 0 -, axis 0 +, axis 1 -, ...
 *  (band.hpp:64-73). */
template <int D>
inline void neighbors_of(const Ix<D>& ix, Ix<D>* out) {
    for (int a = 0; a < D; ++a) {
        Ix<D> m = ix, q = ix;
        m[a] -= 1;
        q[a] += 1;
        out[2 * a] = m;
        out[2 * a + 1] = q;
    }
}

/** Tube band (band.hpp:150-182).  tube_radius <= 0 selects the reference
 *  radius stencil_reach = (p+1)/2 sqrt(d) h; a positive value overrides it
 *  (BASELINE.json states sqrt(13) h / sqrt(17) h). */
template <int D>
Band<D> build_band_tube(const Surface<D>& surface, double h, int p, double tube_radius = 0.0, int workers = 0);

}  // namespace cpddg
