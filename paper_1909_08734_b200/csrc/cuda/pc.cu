// Device restricted additive Schwarz preconditioner (RAS / ORAS).
//
// Replaces, per subdomain j, the reference's LocalOperator +
// DirectSolver (transmission.hpp:47-138, direct.hpp:36-68: Eigen SparseLU
// with COLAMD) and SchwarzPreconditioner::apply (solve.hpp:64-86):
//
//   z = sum_j Rt_j^T A_j^-1 [R_j r ; 0]
//
// Setup (cpddg_pc_create):
//   host   per subdomain, on a thread pool: reverse Cuthill-McKee ordering of
//          pattern(A_j + A_j^T), its symmetric envelope (profile) f_i, and
//          the scatter of A_j into envelope storage.  Dirichlet (RAS)
//          closures -- BC rows that are unit rows with a zero right-hand
//          side (transmission.hpp:117-134, :59-63) -- are eliminated first:
//          z_b = 0 exactly, so only the overlap block A_oo is factored.
//   device k_factor: one CTA per subdomain, right-looking blocked LU without
//          pivoting inside the envelope (fill stays inside the profile):
//          32-wide panels (dense diagonal block in shared memory, row-wise
//          triangular solves for the L and U panels) and a 64x64-tiled
//          trailing update of the envelope with both triangles per tile.
//          Zero / non-finite pivots raise DivergenceError exactly where the
//          reference's SparseLU reports a singular factorisation.
// Apply (cpddg_pc_apply): k_solve, one CTA per subdomain (largest first):
//   gather R_j r into shared memory, blocked forward substitution (32-row
//   panels: warp-per-row coalesced dot over the row's envelope, then a
//   one-warp shuffle triangle), blocked backward substitution by columns
//   (one-warp triangle, then thread-per-row axpy over 32 contiguous U
//   columns), and the restricted scatter Rt_j^T of the owned rows.
// Storage: L row i and U column i (transposed) are contiguous runs over
// [f_i, i); per-row tables are concatenated over subdomains.
#include "../host/ordering.hpp"
#include "../host/setup.hpp"
#include "common.cuh"
#include "op.cuh"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <cmath>
#include <mutex>
#include <numeric>

namespace cpddg {

namespace {

/** Streaming loads of factor data: ld.global.nc with L1::no_allocate (the
 *  data is used once; keeps L1 for the index tables).  Measured on B200
 *  (scripts/micro/ld_variants.cu): one SM streams 162 GB/s this way but only
 *  58 GB/s with ld.global.cs (__ldcs), which capped the doubly-loaded SMs. */
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

constexpr int NB = 32;    // factor panel width
constexpr int TILE = 64;  // trailing-update tile


struct HostSub {
    int n = 0;
    bool reduced = false;
    bool pivoted = false;      // factored on the host with partial pivoting (band LU): P A = L U
    std::vector<int> rowperm;  // pivoted: factor-order row i of P A is row rowperm[i] of A
    std::vector<double> preL, preU, prediag;  // pivoted: the factors in envelope storage
    std::int64_t ne = 0, neU = 0;  // envelope entries of L (rows) and U (columns)
    std::vector<int> inv;      // local (old) index -> factor order
    std::vector<double> probe; // b = A_sys x_probe in factor order
    std::vector<int> first, firstU, rlast, urlast, gidx, sidx;
    std::vector<std::int64_t> roff, roffU;

};

/** Sparse-row LU with partial pivoting (the explicit form P A = L U of
 *  LAPACK getrf) of an n x n system in factor order with lower bandwidth bl.
 *  Every row keeps its own window [lo, lo + v.size()) of columns: lo never
 *  decreases (elimination at step k only fills columns > k), the right end
 *  grows with the fill, and a row swap is a swap of row identities, so the
 *  L part travels with its row.  Pivot candidates at step k lie in positions
 *  [k, k + bl] (a row only moves down by a swap at a step within bl of it).
 *  Throws DivergenceError on an exactly zero pivot column: the reference's
 *  SparseLU reports such a system singular (direct.hpp:47-50).  This is the
 *  fallback for local systems whose no-pivot device factorisation fails
 *  (DirectSolver pivots, direct.hpp:41-52); it costs ~n bl (bl + bu) flops
 *  on one host thread. */
struct PivLU {
    struct Row {
        int lo = 0;
        std::vector<double> v;
        double get(int c) const { return c >= lo && c < lo + static_cast<int>(v.size()) ? v[static_cast<std::size_t>(c - lo)] : 0.0; }
        int hi() const { return lo + static_cast<int>(v.size()); }
    };
    int n = 0, bl = 0;
    std::vector<Row> rows;   // by identity (the original factor-order row)
    std::vector<int> pos;    // position -> row identity (= P)
};

void piv_lu(PivLU& F, const std::string& what) {
    const int n = F.n, bl = F.bl;
    F.pos.resize(static_cast<std::size_t>(n));
    std::iota(F.pos.begin(), F.pos.end(), 0);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(k)])].get(k));
        for (int q = k + 1; q <= std::min(n - 1, k + bl); ++q) {
            const double a = std::abs(F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(q)])].get(k));
            if (a > best) {
                best = a;
                p = q;
            }
        }
        if (!(best > 0.0) || !std::isfinite(best)) throw DivergenceError("singular factorization of " + what);
        std::swap(F.pos[static_cast<std::size_t>(k)], F.pos[static_cast<std::size_t>(p)]);
        const PivLU::Row& P = F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(k)])];
        const double piv = P.get(k);
        const int phi = P.hi();
        for (int q = k + 1; q <= std::min(n - 1, k + bl); ++q) {
            PivLU::Row& R = F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(q)])];
            const double a = R.get(k);
            if (a == 0.0) continue;
            const double l = a / piv;
            if (R.hi() < phi) R.v.resize(static_cast<std::size_t>(phi - R.lo), 0.0);
            R.v[static_cast<std::size_t>(k - R.lo)] = l;
            for (int c = k + 1; c < phi; ++c) R.v[static_cast<std::size_t>(c - R.lo)] -= l * P.v[static_cast<std::size_t>(c - P.lo)];
        }
    }
}

HostSub analyse(const cpddg_local_desc& d, int n_global, bool pivot = false, int j_sub = -1) {
    const int nl = d.n_overlap + d.n_bc;
    if (d.n_overlap < 0 || d.n_bc < 0 || nl <= 0) throw InternalError("empty local system");
    const std::int64_t* rp = d.row_ptr;
    for (int r = 0; r < nl; ++r)
        if (rp[r + 1] < rp[r]) throw InternalError("local CSR row pointer is not monotone");
    for (std::int64_t k = 0; k < rp[nl]; ++k)
        if (d.col[k] < 0 || d.col[k] >= nl) throw InternalError("local CSR column out of range");
    // Dirichlet closure: every BC row is the unit row e_b (transmission.hpp:117-118)
    bool reducible = true;
    for (int r = d.n_overlap; r < nl && reducible; ++r)
        reducible = rp[r + 1] - rp[r] == 1 && d.col[rp[r]] == r && d.val[rp[r]] == 1.0;
    HostSub S;
    S.reduced = reducible && d.n_bc > 0;
    const int n = reducible ? d.n_overlap : nl;
    S.n = n;
    // pattern(A + A^T) without the diagonal, CSR.  Rows with increasing columns
    // (what append_row of sparse.hpp:35-46 produces): the transpose by a
    // counting pass is sorted too, and each row is the merge of the two sorted
    // lists (a third of the time of sorting the concatenation); any other
    // input: count, fill, sort + unique per row.
    bool sorted_rows = true;
    for (int r = 0; r < n && sorted_rows; ++r)
        for (std::int64_t k = rp[r] + 1; k < rp[r + 1]; ++k)
            if (d.col[k] < d.col[k - 1]) {
                sorted_rows = false;
                break;
            }
    Graph gr;
    if (sorted_rows) {
        std::vector<int> tc(static_cast<std::size_t>(n) + 1, 0);
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k)
                if (const int c = d.col[k]; c < n && c != r) ++tc[static_cast<std::size_t>(c) + 1];
        for (int v = 0; v < n; ++v) tc[static_cast<std::size_t>(v) + 1] += tc[static_cast<std::size_t>(v)];
        std::vector<int> tr(static_cast<std::size_t>(tc[static_cast<std::size_t>(n)])), fill(tc.begin(), tc.end() - 1);
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k)
                if (const int c = d.col[k]; c < n && c != r) tr[static_cast<std::size_t>(fill[static_cast<std::size_t>(c)]++)] = r;
        gr.xadj.assign(static_cast<std::size_t>(n) + 1, 0);
        gr.adj.reserve(2 * tr.size());
        for (int v = 0; v < n; ++v) {
            const int* a = d.col + rp[v];
            const int* ae = d.col + rp[v + 1];
            const int* b = tr.data() + tc[static_cast<std::size_t>(v)];
            const int* be = tr.data() + tc[static_cast<std::size_t>(v) + 1];
            int last = -1;
            while (a != ae || b != be) {
                const int x = (b == be || (a != ae && *a <= *b)) ? *a++ : *b++;
                if (x < n && x != v && x != last) {
                    gr.adj.push_back(x);
                    last = x;
                }
            }
            gr.xadj[static_cast<std::size_t>(v) + 1] = static_cast<int>(gr.adj.size());
        }
    } else {
        std::vector<int> cnt(static_cast<std::size_t>(n) + 1, 0);
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int c = d.col[k];
                if (c >= n || c == r) continue;
                ++cnt[static_cast<std::size_t>(r) + 1];
                ++cnt[static_cast<std::size_t>(c) + 1];
            }
        for (int v = 0; v < n; ++v) cnt[static_cast<std::size_t>(v) + 1] += cnt[static_cast<std::size_t>(v)];
        std::vector<int> raw(static_cast<std::size_t>(cnt[static_cast<std::size_t>(n)])), fill(cnt.begin(), cnt.end() - 1);
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int c = d.col[k];
                if (c >= n || c == r) continue;
                raw[static_cast<std::size_t>(fill[static_cast<std::size_t>(r)]++)] = c;
                raw[static_cast<std::size_t>(fill[static_cast<std::size_t>(c)]++)] = r;
            }
        gr.xadj.assign(static_cast<std::size_t>(n) + 1, 0);
        gr.adj.reserve(raw.size());
        for (int v = 0; v < n; ++v) {
            int* b = raw.data() + cnt[static_cast<std::size_t>(v)];
            int* e = raw.data() + cnt[static_cast<std::size_t>(v) + 1];
            std::sort(b, e);
            e = std::unique(b, e);
            gr.adj.insert(gr.adj.end(), b, e);
            gr.xadj[static_cast<std::size_t>(v) + 1] = static_cast<int>(gr.adj.size());
        }
    }
    // Ordering: reverse Cuthill-McKee, or (default) Sloan's profile ordering when
    // it stores fewer envelope entries without pushing the longest row / column
    // into a larger y window of k_solve_win (CPDDG_ORDER=rcm|sloan).
    std::vector<int> perm = rcm(gr);
    std::vector<int> inv(static_cast<std::size_t>(n));
    struct Profile {
        std::int64_t entries = 0;
        int reach = 0;
    };
    auto profile_of = [&](const std::vector<int>& pm) {
        for (int k = 0; k < n; ++k) inv[static_cast<std::size_t>(pm[static_cast<std::size_t>(k)])] = k;
        std::vector<int> fl(static_cast<std::size_t>(n)), fu(static_cast<std::size_t>(n));
        std::iota(fl.begin(), fl.end(), 0);
        std::iota(fu.begin(), fu.end(), 0);
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int c = d.col[k];
                if (c >= n || c == r) continue;
                const int pi = inv[static_cast<std::size_t>(r)], pj = inv[static_cast<std::size_t>(c)];
                if (pj < pi)
                    fl[static_cast<std::size_t>(pi)] = std::min(fl[static_cast<std::size_t>(pi)], pj);
                else
                    fu[static_cast<std::size_t>(pj)] = std::min(fu[static_cast<std::size_t>(pj)], pi);
            }
        Profile P;
        for (int i = 0; i < n; ++i) {
            P.entries += (i - fl[static_cast<std::size_t>(i)]) + (i - fu[static_cast<std::size_t>(i)]);
            P.reach = std::max({P.reach, i - fl[static_cast<std::size_t>(i)], i - fu[static_cast<std::size_t>(i)]});
        }
        return P;
    };
    static const bool use_sloan = [] {
        const char* e = std::getenv("CPDDG_ORDER");
        return !(e && std::string(e) == "rcm");
    }();
    if (use_sloan && n > 64) {
        auto window = [](int reach) {  // k_solve_win's window class (win_geometry, RB = 16)
            int W = 2048;
            while (W < reach + 96) W *= 2;
            return W;
        };
        const Profile base = profile_of(perm);
        Profile best = base;
        for (int w1 : {8, 32}) {
            std::vector<int> cand = sloan(gr, w1, 1);
            const Profile P = profile_of(cand);
            if (P.entries < best.entries && window(P.reach) <= window(base.reach)) {
                best = P;
                perm = std::move(cand);
                break;
            }
        }
    }
    for (int k = 0; k < n; ++k) inv[static_cast<std::size_t>(perm[static_cast<std::size_t>(k)])] = k;
    PivLU F;
    if (pivot) {
        // host LU with partial pivoting in factor order; the envelopes below
        // then come from the factors' own nonzeros
        int bl = 0;
        F.n = n;
        F.rows.resize(static_cast<std::size_t>(n));
        std::vector<int> hi(static_cast<std::size_t>(n), 0);
        for (int i = 0; i < n; ++i) {
            F.rows[static_cast<std::size_t>(i)].lo = i;
            hi[static_cast<std::size_t>(i)] = i + 1;
        }
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int c = d.col[k];
                if (c >= n) continue;
                const int pi = inv[static_cast<std::size_t>(r)], pj = inv[static_cast<std::size_t>(c)];
                bl = std::max(bl, pi - pj);
                F.rows[static_cast<std::size_t>(pi)].lo = std::min(F.rows[static_cast<std::size_t>(pi)].lo, pj);
                hi[static_cast<std::size_t>(pi)] = std::max(hi[static_cast<std::size_t>(pi)], pj + 1);
            }
        for (int i = 0; i < n; ++i) {
            PivLU::Row& R = F.rows[static_cast<std::size_t>(i)];
            R.v.assign(static_cast<std::size_t>(hi[static_cast<std::size_t>(i)] - R.lo), 0.0);
        }
        for (int r = 0; r < n; ++r)
            for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int c = d.col[k];
                if (c >= n) continue;
                PivLU::Row& R = F.rows[static_cast<std::size_t>(inv[static_cast<std::size_t>(r)])];
                R.v[static_cast<std::size_t>(inv[static_cast<std::size_t>(c)] - R.lo)] += d.val[k];
            }
        F.bl = bl;
        piv_lu(F, "subdomain " + std::to_string(j_sub));
        S.pivoted = true;
        S.rowperm = F.pos;
    }
    // envelopes of the actual (nonsymmetric) pattern in factor order: L row i
    // starts at fL_i (first nonzero left of the diagonal), U column c at fU_c
    // (first nonzero above it).  LU without pivoting keeps its fill inside
    // both: l_ij = 0 for j < fL_i and u_ic = 0 for i < fU_c by induction on
    // the elimination, so L is stored by rows over [fL_i, i) and U by
    // columns over [fU_c, c).  (CPDDG_ENVELOPE=sym: the symmetric profile
    // min(fL, fU) for both, the previous layout.)
    S.first.resize(static_cast<std::size_t>(n));
    S.firstU.resize(static_cast<std::size_t>(n));
    std::iota(S.first.begin(), S.first.end(), 0);
    std::iota(S.firstU.begin(), S.firstU.end(), 0);
    for (int r = 0; r < n; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = d.col[k];
            if (c >= n || c == r) continue;
            const int pi = inv[static_cast<std::size_t>(r)], pj = inv[static_cast<std::size_t>(c)];
            if (pj < pi)
                S.first[static_cast<std::size_t>(pi)] = std::min(S.first[static_cast<std::size_t>(pi)], pj);
            else
                S.firstU[static_cast<std::size_t>(pj)] = std::min(S.firstU[static_cast<std::size_t>(pj)], pi);
        }
    if (pivot) {  // the factors' own envelopes (fill included)
        std::iota(S.first.begin(), S.first.end(), 0);
        std::iota(S.firstU.begin(), S.firstU.end(), 0);
        for (int i = 0; i < n; ++i) {
            const PivLU::Row& R = F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(i)])];
            for (int c = R.lo; c < R.hi(); ++c) {
                if (c == i || R.v[static_cast<std::size_t>(c - R.lo)] == 0.0) continue;
                if (c < i)
                    S.first[static_cast<std::size_t>(i)] = std::min(S.first[static_cast<std::size_t>(i)], c);
                else
                    S.firstU[static_cast<std::size_t>(c)] = std::min(S.firstU[static_cast<std::size_t>(c)], i);
            }
        }
    }
    static const bool sym_env = [] {
        const char* e = std::getenv("CPDDG_ENVELOPE");
        return e && std::string(e) == "sym";
    }();
    if (sym_env)
        for (int i = 0; i < n; ++i)
            S.first[static_cast<std::size_t>(i)] = S.firstU[static_cast<std::size_t>(i)] =
                std::min(S.first[static_cast<std::size_t>(i)], S.firstU[static_cast<std::size_t>(i)]);
    // 16-byte alignment for vector loads: every row (of L) / column (of U)
    // starts at an even column and has even length, so column pairs
    // (2m, 2m+1) are double2-aligned.  The extra slots are structural zeros
    // that the no-pivot factorisation never fills (they lie outside the
    // envelope), so they cost at most two stored zeros per row.
    for (int i = 0; i < n; ++i) {
        S.first[static_cast<std::size_t>(i)] &= ~1;
        S.firstU[static_cast<std::size_t>(i)] &= ~1;
    }
    auto offsets = [&](const std::vector<int>& f, std::vector<std::int64_t>& ro) {
        ro.assign(static_cast<std::size_t>(n) + 1, 0);
        for (int i = 0; i < n; ++i)
            ro[static_cast<std::size_t>(i) + 1] = ro[static_cast<std::size_t>(i)] + ((i + (i & 1)) - f[static_cast<std::size_t>(i)]);
        const std::int64_t total = ro.back();
        ro.pop_back();
        return total;
    };
    S.ne = offsets(S.first, S.roff);
    S.neU = offsets(S.firstU, S.roffU);
    // rlast_i: largest row whose L row or U column starts at or before i (the
    // factorisation's panel reach); urlast_i: U columns only (reversed U rows)
    auto reach = [&](std::initializer_list<const std::vector<int>*> fs) {
        std::vector<int> maxrow(static_cast<std::size_t>(n), -1), out(static_cast<std::size_t>(n));
        for (const auto* f : fs)
            for (int i = 0; i < n; ++i)
                maxrow[static_cast<std::size_t>((*f)[static_cast<std::size_t>(i)])] =
                    std::max(maxrow[static_cast<std::size_t>((*f)[static_cast<std::size_t>(i)])], i);
        int run = -1;
        for (int i = 0; i < n; ++i) {
            run = std::max(run, maxrow[static_cast<std::size_t>(i)]);
            out[static_cast<std::size_t>(i)] = std::max(run, i);
        }
        return out;
    };
    if (pivot) {  // the factors in envelope storage (k_factor skips this subdomain)
        S.preL.assign(static_cast<std::size_t>(S.ne), 0.0);
        S.preU.assign(static_cast<std::size_t>(S.neU), 0.0);
        S.prediag.assign(static_cast<std::size_t>(n), 0.0);
        for (int i = 0; i < n; ++i) {
            const PivLU::Row& R = F.rows[static_cast<std::size_t>(F.pos[static_cast<std::size_t>(i)])];
            S.prediag[static_cast<std::size_t>(i)] = R.get(i);
            for (int c = std::max(R.lo, S.first[static_cast<std::size_t>(i)]); c < std::min(i, R.hi()); ++c)
                S.preL[static_cast<std::size_t>(S.roff[static_cast<std::size_t>(i)] + c - S.first[static_cast<std::size_t>(i)])] =
                    R.v[static_cast<std::size_t>(c - R.lo)];
            for (int c = std::max(i + 1, R.lo); c < R.hi(); ++c) {
                const double u = R.v[static_cast<std::size_t>(c - R.lo)];
                if (u != 0.0)
                    S.preU[static_cast<std::size_t>(S.roffU[static_cast<std::size_t>(c)] + i - S.firstU[static_cast<std::size_t>(c)])] = u;
            }
        }
        F.rows.clear();
        F.rows.shrink_to_fit();
    }
    S.rlast = reach({&S.first, &S.firstU});
    S.urlast = reach({&S.firstU});
    // factor probe: b = A_sys x with x_i = 1 + (i mod 7) / 8 in factor order
    S.probe.assign(static_cast<std::size_t>(n), 0.0);
    for (int r = 0; r < n; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = d.col[k];
            if (c >= n) continue;
            const int pc_ = inv[static_cast<std::size_t>(c)];
            S.probe[static_cast<std::size_t>(inv[static_cast<std::size_t>(r)])] += d.val[k] * (1.0 + (pc_ % 7) / 8.0);
        }
    S.inv = inv;
    S.gidx.assign(static_cast<std::size_t>(n), -1);
    S.sidx.assign(static_cast<std::size_t>(n), -1);
    for (int o = 0; o < std::min(n, d.n_overlap); ++o) {
        const int g = d.overlap[o];
        if (g < 0 || g >= n_global) throw InternalError("overlap index out of range");
        S.gidx[static_cast<std::size_t>(inv[static_cast<std::size_t>(o)])] = g;
    }
    if (pivot) {  // L U z = P b: row i gathers the right-hand side of row rowperm[i]
        std::vector<int> g2(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) g2[static_cast<std::size_t>(i)] = S.gidx[static_cast<std::size_t>(S.rowperm[static_cast<std::size_t>(i)])];
        S.gidx = std::move(g2);
    }
    for (int k = 0; k < d.n_scatter; ++k) {
        const int lo = d.scatter_local[k], g = d.scatter_global[k];
        if (lo < 0 || lo >= n || g < 0 || g >= n_global) throw InternalError("scatter index out of range");
        S.sidx[static_cast<std::size_t>(inv[static_cast<std::size_t>(lo)])] = g;
    }
    return S;
}

/** The entries of A_j as (destination, value) pairs: destination = slot in
 *  the concatenated L (tag 0), U (tag 1) or diagonal (tag 2) storage, tag in
 *  the top two bits.  Built on the host per subdomain (16 bytes per entry)
 *  and scattered on the device into the zeroed envelopes (k_scatter_pairs):
 *  the envelopes themselves (~40 MB per headline subdomain, mostly fill)
 *  never cross the host link. */
constexpr int kTagShift = 62;
std::int64_t scatter_pairs(const cpddg_local_desc& d, const HostSub& S, std::int64_t eb, std::int64_t ebu,
                           std::int64_t v0, std::int64_t* dst, double* val) {
    const int n = S.n;
    const std::int64_t* rp = d.row_ptr;
    std::int64_t m = 0;
    for (int r = 0; r < n; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = d.col[k];
            if (c >= n) continue;  // eliminated Dirichlet closure column (z_b = 0)
            const int pi = S.inv[static_cast<std::size_t>(r)], pj = S.inv[static_cast<std::size_t>(c)];
            std::int64_t to;
            if (pi == pj)
                to = (2LL << kTagShift) | (v0 + pi);
            else if (pj < pi)
                to = eb + S.roff[static_cast<std::size_t>(pi)] + (pj - S.first[static_cast<std::size_t>(pi)]);
            else
                to = (1LL << kTagShift) | (ebu + S.roffU[static_cast<std::size_t>(pj)] + (pi - S.firstU[static_cast<std::size_t>(pj)]));
            dst[m] = to;
            val[m] = d.val[k];
            ++m;
        }
    return m;
}

__global__ void k_scatter_pairs(std::int64_t m, const std::int64_t* __restrict__ dst, const double* __restrict__ val,
                                double* L, double* U, double* diag) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < m;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t t = dst[e];
        const int tag = static_cast<int>(static_cast<unsigned long long>(t) >> kTagShift);
        const std::int64_t i = t & ((1LL << kTagShift) - 1);
        double* base = tag == 0 ? L : tag == 1 ? U : diag;
        atomicAdd(base + i, val[e]);  // duplicate (r, c) entries of the CSR are summed
    }
}

struct SubPtrs {
    int n;
    const int* first;          // L rows
    const std::int64_t* roff;
    const int* firstU;         // U columns
    const std::int64_t* roffU;
    const int* rlast;
    double* diag;
    double* L;
    double* U;
};

__device__ __forceinline__ SubPtrs sub_ptrs(int j, const int* n_rows, const std::int64_t* vbase,
                                            const std::int64_t* ebase, const std::int64_t* ebaseU,
                                            const int* first, const std::int64_t* roff, const int* firstU,
                                            const std::int64_t* roffU, const int* rlast, double* diag,
                                            double* L, double* U) {
    const std::int64_t vb = vbase[j];
    return {n_rows[j], first + vb, roff + vb, firstU + vb, roffU + vb, rlast + vb, diag + vb, L + ebase[j],
            U + ebaseU[j]};
}

// ------------------------------------------------------------ factorisation

constexpr int kFactorThreads = 256;
constexpr int kTS = TILE + 1;  // padded tile row stride (doubles) -- tiles are [NB][TILE+1]

__global__ void __launch_bounds__(kFactorThreads, 2) k_factor(const int* __restrict__ order,
                                                           const int* __restrict__ n_rows,
                                                           const std::int64_t* __restrict__ vbase,
                                                           const std::int64_t* __restrict__ ebase,
                                                           const std::int64_t* __restrict__ ebaseU,
                                                           const int* __restrict__ first_all,
                                                           const std::int64_t* __restrict__ roff_all,
                                                           const int* __restrict__ firstU_all,
                                                           const std::int64_t* __restrict__ roffU_all,
                                                           const int* __restrict__ rlast_all,
                                                           double* diag_all, double* L_all, double* U_all,
                                                           double* dinv_all, int* status,
                                                           const int* __restrict__ prefactored) {
    const int j = order[blockIdx.x];
    const SubPtrs S = sub_ptrs(j, n_rows, vbase, ebase, ebaseU, first_all, roff_all, firstU_all, roffU_all,
                               rlast_all, diag_all, L_all, U_all);
    const bool pre = prefactored[j] != 0;  // factored on the host with pivoting: pivots only
    extern __shared__ double sm[];
    double* A11 = sm;                            // [NB][NB+1]
    double* Xi = A11 + NB * (NB + 1);            // [NB][TILE+1]: X rows of tile i, transposed (p-major)
    double* Yi = Xi + NB * kTS;
    double* Xj = Yi + NB * kTS;
    double* Yj = Xj + NB * kTS;
    const int tid = threadIdx.x;
    const int n = S.n;
    __shared__ int skip_tile;

    for (int k0 = 0; k0 < (pre ? 0 : n); k0 += NB) {
        const int kb = min(NB, n - k0), k1 = k0 + kb;
        const int R = S.rlast[k1 - 1];  // last row touching the panel columns
        // (1) diagonal block into shared memory
        for (int e = tid; e < NB * NB; e += blockDim.x) {
            const int r = e / NB, c = e % NB;
            double v = 0.0;
            if (r < kb && c < kb) {
                const int gr = k0 + r, gc = k0 + c;
                if (r == c)
                    v = S.diag[gr];
                else if (r > c) {
                    const int f = S.first[gr];
                    if (gc >= f) v = S.L[S.roff[gr] + gc - f];
                } else {
                    const int f = S.firstU[gc];
                    if (gr >= f) v = S.U[S.roffU[gc] + gr - f];
                }
            }
            A11[r * (NB + 1) + c] = v;
        }
        __syncthreads();
        // (2) unblocked LU of the diagonal block
        for (int p = 0; p < kb; ++p) {
            const double piv = A11[p * (NB + 1) + p];
            for (int r = p + 1 + tid; r < kb; r += blockDim.x) A11[r * (NB + 1) + p] /= piv;
            __syncthreads();
            for (int e = tid; e < (kb - p - 1) * (kb - p - 1); e += blockDim.x) {
                const int r = p + 1 + e / (kb - p - 1), c = p + 1 + e % (kb - p - 1);
                A11[r * (NB + 1) + c] -= A11[r * (NB + 1) + p] * A11[p * (NB + 1) + c];
            }
            __syncthreads();
        }
        for (int e = tid; e < kb * kb; e += blockDim.x) {
            const int r = e / kb, c = e % kb;
            const int gr = k0 + r, gc = k0 + c;
            const double v = A11[r * (NB + 1) + c];
            if (r == c)
                S.diag[gr] = v;
            else if (r > c) {
                const int f = S.first[gr];
                if (gc >= f) S.L[S.roff[gr] + gc - f] = v;
            } else {
                const int f = S.firstU[gc];
                if (gr >= f) S.U[S.roffU[gc] + gr - f] = v;
            }
        }
        // (3)+(4) panels: rows i in [k1, R]
        for (int i = k1 + tid; i <= R; i += blockDim.x) {
            const int f = S.first[i], fu = S.firstU[i];
            if (f >= k1 && fu >= k1) continue;  // no entries in the panel columns
            const std::int64_t ro = S.roff[i] - f, rou = S.roffU[i] - fu;
            double x[NB], u[NB];
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                const int gc = k0 + p;
                x[p] = p < kb && gc >= f ? S.L[ro + gc] : 0.0;
                u[p] = p < kb && gc >= fu ? S.U[rou + gc] : 0.0;
            }
            // L21: x U11 = a  (forward over columns)
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                if (p < kb) {
                    double s = x[p];
#pragma unroll
                    for (int q = 0; q < p; ++q) s -= x[q] * A11[q * (NB + 1) + p];
                    x[p] = s / A11[p * (NB + 1) + p];
                }
            }
            // U12^T: L11 u = a  (unit lower)
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                if (p < kb) {
                    double s = u[p];
#pragma unroll
                    for (int q = 0; q < p; ++q) s -= A11[p * (NB + 1) + q] * u[q];
                    u[p] = s;
                }
            }
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                const int gc = k0 + p;
                if (p < kb && gc >= f) S.L[ro + gc] = x[p];
                if (p < kb && gc >= fu) S.U[rou + gc] = u[p];
            }
        }
        __syncthreads();
        // (5) trailing update of rows/cols [k1, R]: lower tiles (bi >= bj) get
        //     L[i][c] -= X_i . Y_c  and  Ut[i][c] -= Y_i . X_c  (c < i), diag -= X_i . Y_i
        const int m = R - k1 + 1;
        if (m > 0) {
            const int nt = (m + TILE - 1) / TILE;
            for (int t = 0; t < nt * (nt + 1) / 2; ++t) {
                // t -> (bi, bj), bj <= bi
                int bi = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
                while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
                while (bi * (bi + 1) / 2 > t) --bi;
                const int bj = t - bi * (bi + 1) / 2;
                const int i0 = k1 + bi * TILE, j0 = k1 + bj * TILE;
                // skip tiles whose rows or columns carry no panel entries (X, Y = 0)
                __syncthreads();
                if (tid < 32) {
                    int mi = INT_MAX, mj = INT_MAX;
                    for (int q = tid; q < TILE; q += 32) {
                        if (i0 + q <= R) mi = min(mi, min(S.first[i0 + q], S.firstU[i0 + q]));
                        if (j0 + q <= R) mj = min(mj, min(S.first[j0 + q], S.firstU[j0 + q]));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        mi = min(mi, __shfl_xor_sync(0xffffffffu, mi, o));
                        mj = min(mj, __shfl_xor_sync(0xffffffffu, mj, o));
                    }
                    if (tid == 0) skip_tile = !(mi < k1 && mj < k1);
                }
                __syncthreads();
                if (skip_tile) continue;
                for (int e = tid; e < NB * TILE; e += blockDim.x) {
                    const int r = e / NB, p = e % NB;
                    const int gi = i0 + r, gj = j0 + r, gc = k0 + p;
                    double xi = 0, yi = 0, xj = 0, yj = 0;
                    if (p < kb) {
                        if (gi <= R) {
                            const int f = S.first[gi], fu = S.firstU[gi];
                            if (gc >= f) xi = S.L[S.roff[gi] + gc - f];
                            if (gc >= fu) yi = S.U[S.roffU[gi] + gc - fu];
                        }
                        if (gj <= R) {
                            const int f = S.first[gj], fu = S.firstU[gj];
                            if (gc >= f) xj = S.L[S.roff[gj] + gc - f];
                            if (gc >= fu) yj = S.U[S.roffU[gj] + gc - fu];
                        }
                    }
                    Xi[p * kTS + r] = xi;
                    Yi[p * kTS + r] = yi;
                    Xj[p * kTS + r] = xj;
                    Yj[p * kTS + r] = yj;
                }
                __syncthreads();
                // FP64 tensor cores: warp w owns the 8-row band w of the tile and all
                // eight 8-column blocks; mma.m8n8k4 over the panel width
                // (k chunks of 4; rows p >= kb of the staged panels are zero).
                const int warp = tid >> 5, lane = tid & 31;
                const int lr = lane >> 2, lk = lane & 3;
                double cL[8][2], cU[8][2];
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) cL[cb][0] = cL[cb][1] = cU[cb][0] = cU[cb][1] = 0.0;
                for (int kc = 0; kc < kb; kc += 4) {
                    const int p = kc + lk;
                    const double ax = Xi[p * kTS + warp * 8 + lr];  // A(row, k) = X_i
                    const double ay = Yi[p * kTS + warp * 8 + lr];  // A(row, k) = Y_i
#pragma unroll
                    for (int cb = 0; cb < 8; ++cb) {
                        const double by = Yj[p * kTS + cb * 8 + lr];  // B(k, col) = Y_j^T
                        const double bx = Xj[p * kTS + cb * 8 + lr];  // B(k, col) = X_j^T
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                     : "+d"(cL[cb][0]), "+d"(cL[cb][1])
                                     : "d"(ax), "d"(by));
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                     : "+d"(cU[cb][0]), "+d"(cU[cb][1])
                                     : "d"(ay), "d"(bx));
                    }
                }
                {
                    const int gi = i0 + warp * 8 + lr;
                    if (gi <= R) {
                        const int f = S.first[gi], fu = S.firstU[gi];
                        const std::int64_t ro = S.roff[gi] - f, rou = S.roffU[gi] - fu;
#pragma unroll
                        for (int cb = 0; cb < 8; ++cb)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int gc = j0 + cb * 8 + 2 * lk + e;
                                if (gc > R) continue;
                                if (gc < gi) {
                                    if (gc >= f) S.L[ro + gc] -= cL[cb][e];
                                    if (gc >= fu) S.U[rou + gc] -= cU[cb][e];
                                } else if (gc == gi) {
                                    S.diag[gi] -= cL[cb][e];
                                }
                            }
                    }
                }
            }
        }
        __syncthreads();
    }
    // pivot check: a zero or non-finite pivot is a singular factorisation
    int bad = 0;
    double* dinv = dinv_all + vbase[j];
    for (int i = tid; i < n; i += blockDim.x) {
        const double d = S.diag[i];
        if (!(fabs(d) > 0.0) || !isfinite(d)) bad = 1;
        dinv[i] = 1.0 / d;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) status[j] = bad;
}

/** k_factor with a software-pipelined trailing update (the default; the
 *  round-1 kernel above stays as CPDDG_FACTOR=v1).  One CTA of 512 threads
 *  per SM and subdomain.  Per panel, the 64-row blocks of the trailing
 *  window that carry panel entries are listed once (no per-tile skip test),
 *  and the active tiles (bi >= bj) are walked with their four panel slices
 *  (X_i, Y_i, X_j, Y_j: 64 rows x 32 panel columns, row-major, 36-double
 *  stride) staged by 16-byte cp.async with zero fill outside the envelopes
 *  into one of two shared buffers while the previous tile runs on the FP64
 *  tensor cores; the tile's old L / U values are loaded before its MMAs and
 *  written after.  16 warps: warp w owns rows 8 (w % 8) .. + 8 and columns
 *  32 (w / 8) .. + 32 of the tile.  Same fragments and k order as k_factor:
 *  the factors are bitwise identical. */
constexpr int kF2Threads = 512;
constexpr int kF2Stride = 36;                      // doubles per staged row (2-way conflict-free fragments)
constexpr int kF2Arr = TILE * kF2Stride;           // one staged array
constexpr int kF2Buf = 4 * kF2Arr;                 // X_i, Y_i, X_j, Y_j
constexpr int kF2MaxBlk = 256;                     // trailing-window blocks (reach <= 16384 rows; else k_factor)
__global__ void __launch_bounds__(kF2Threads, 1) k_factor2(const int* __restrict__ order,
                                                          const int* __restrict__ n_rows,
                                                          const std::int64_t* __restrict__ vbase,
                                                          const std::int64_t* __restrict__ ebase,
                                                          const std::int64_t* __restrict__ ebaseU,
                                                          const int* __restrict__ first_all,
                                                          const std::int64_t* __restrict__ roff_all,
                                                          const int* __restrict__ firstU_all,
                                                          const std::int64_t* __restrict__ roffU_all,
                                                          const int* __restrict__ rlast_all,
                                                          double* diag_all, double* L_all, double* U_all,
                                                          double* dinv_all, int* status,
                                                          const int* __restrict__ prefactored) {
    const int j = order[blockIdx.x];
    const SubPtrs S = sub_ptrs(j, n_rows, vbase, ebase, ebaseU, first_all, roff_all, firstU_all, roffU_all,
                               rlast_all, diag_all, L_all, U_all);
    const bool pre = prefactored[j] != 0;
    extern __shared__ __align__(16) double sm[];
    double* A11 = sm;                     // [NB][NB+1]
    double* bufs = A11 + NB * (NB + 1);   // [2][4][TILE][kF2Stride]  (NB*(NB+1) is even: 16-byte aligned)
    __shared__ int act[kF2MaxBlk];        // active 64-row blocks of the trailing window
    __shared__ unsigned char actf[kF2MaxBlk];
    __shared__ int n_act;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n = S.n;
    const unsigned bufs_s = static_cast<unsigned>(__cvta_generic_to_shared(bufs));

    for (int k0 = 0; k0 < (pre ? 0 : n); k0 += NB) {
        const int kb = min(NB, n - k0), k1 = k0 + kb;
        const int R = S.rlast[k1 - 1];
        // (1) diagonal block into shared memory
        for (int e = tid; e < NB * NB; e += blockDim.x) {
            const int r = e / NB, c = e % NB;
            double v = 0.0;
            if (r < kb && c < kb) {
                const int gr = k0 + r, gc = k0 + c;
                if (r == c)
                    v = S.diag[gr];
                else if (r > c) {
                    const int f = S.first[gr];
                    if (gc >= f) v = S.L[S.roff[gr] + gc - f];
                } else {
                    const int f = S.firstU[gc];
                    if (gr >= f) v = S.U[S.roffU[gc] + gr - f];
                }
            }
            A11[r * (NB + 1) + c] = v;
        }
        __syncthreads();
        // (2) unblocked LU of the diagonal block
        for (int p = 0; p < kb; ++p) {
            const double piv = A11[p * (NB + 1) + p];
            for (int r = p + 1 + tid; r < kb; r += blockDim.x) A11[r * (NB + 1) + p] /= piv;
            __syncthreads();
            for (int e = tid; e < (kb - p - 1) * (kb - p - 1); e += blockDim.x) {
                const int r = p + 1 + e / (kb - p - 1), c = p + 1 + e % (kb - p - 1);
                A11[r * (NB + 1) + c] -= A11[r * (NB + 1) + p] * A11[p * (NB + 1) + c];
            }
            __syncthreads();
        }
        for (int e = tid; e < kb * kb; e += blockDim.x) {
            const int r = e / kb, c = e % kb;
            const int gr = k0 + r, gc = k0 + c;
            const double v = A11[r * (NB + 1) + c];
            if (r == c)
                S.diag[gr] = v;
            else if (r > c) {
                const int f = S.first[gr];
                if (gc >= f) S.L[S.roff[gr] + gc - f] = v;
            } else {
                const int f = S.firstU[gc];
                if (gr >= f) S.U[S.roffU[gc] + gr - f] = v;
            }
        }
        // (3)+(4) panels: rows i in [k1, R]
        for (int i = k1 + tid; i <= R; i += blockDim.x) {
            const int f = S.first[i], fu = S.firstU[i];
            if (f >= k1 && fu >= k1) continue;
            const std::int64_t ro = S.roff[i] - f, rou = S.roffU[i] - fu;
            double x[NB], u[NB];
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                const int gc = k0 + p;
                x[p] = p < kb && gc >= f ? S.L[ro + gc] : 0.0;
                u[p] = p < kb && gc >= fu ? S.U[rou + gc] : 0.0;
            }
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                if (p < kb) {
                    double s = x[p];
#pragma unroll
                    for (int q = 0; q < p; ++q) s -= x[q] * A11[q * (NB + 1) + p];
                    x[p] = s / A11[p * (NB + 1) + p];
                }
            }
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                if (p < kb) {
                    double s = u[p];
#pragma unroll
                    for (int q = 0; q < p; ++q) s -= A11[p * (NB + 1) + q] * u[q];
                    u[p] = s;
                }
            }
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                const int gc = k0 + p;
                if (p < kb && gc >= f) S.L[ro + gc] = x[p];
                if (p < kb && gc >= fu) S.U[rou + gc] = u[p];
            }
        }
        // (5) trailing update of rows/cols [k1, R]
        const int m = R - k1 + 1;
        const int nblk = m > 0 ? (m + TILE - 1) / TILE : 0;
        // active blocks: some row carries an L or U entry in the panel columns
        for (int b = warp; b < nblk; b += kF2Threads / 32) {
            bool a = false;
            for (int q = lane; q < TILE; q += 32) {
                const int r = k1 + b * TILE + q;
                if (r <= R && min(S.first[r], S.firstU[r]) < k1) a = true;
            }
            a = __any_sync(0xffffffffu, a);
            if (lane == 0) actf[b] = a;
        }
        __syncthreads();  // panels written, block flags set
        if (warp == 0) {  // compaction in block order
            int cnt = 0;
            for (int b0 = 0; b0 < nblk; b0 += 32) {
                const bool a = b0 + lane < nblk && actf[b0 + lane];
                const unsigned bal = __ballot_sync(0xffffffffu, a);
                if (a) act[cnt + __popc(bal & ((1u << lane) - 1u))] = b0 + lane;
                cnt += __popc(bal);
            }
            if (lane == 0) n_act = cnt;
        }
        __syncthreads();
        const int na = n_act;
        const int ntiles = na * (na + 1) / 2;
        // staging: thread -> (array, row) = (tid >> 7, (tid >> 1) & 63), 8 column pairs (tid & 1) * 8 ..
        const int sarr = tid >> 7, srow = (tid >> 1) & 63, spp0 = (tid & 1) * 8;
        auto tile_of = [&](int t, int& bi, int& bj) {
            int b = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while ((b + 1) * (b + 2) / 2 <= t) ++b;
            while (b * (b + 1) / 2 > t) --b;
            bi = act[b];
            bj = act[t - b * (b + 1) / 2];
        };
        auto stage = [&](int t, int buf) {
            int bi, bj;
            tile_of(t, bi, bj);
            const int g = k1 + (sarr < 2 ? bi : bj) * TILE + srow;  // X_i, Y_i, X_j, Y_j
            const bool isY = sarr & 1;
            const unsigned dst = bufs_s + static_cast<unsigned>(((buf * 4 + sarr) * kF2Arr + srow * kF2Stride + 2 * spp0) * 8);
            int f = INT_MAX;
            const double* src = S.L;
            if (g <= R) {
                f = isY ? S.firstU[g] : S.first[g];
                src = (isY ? S.U + S.roffU[g] : S.L + S.roff[g]) - f;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int p = 2 * (spp0 + q), gc = k0 + p;
                const int bytes = (gc >= f && p < kb) ? (p + 1 < kb ? 16 : 8) : 0;
                const double* sp = bytes ? src + gc : S.L;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + 16 * q), "l"(sp), "r"(bytes)
                             : "memory");
            }
        };
        const int rb = warp & 7, ch = warp >> 3;
        const int lr = lane >> 2, lk = lane & 3;
        if (ntiles > 0) stage(0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        for (int t = 0; t < ntiles; ++t) {
            if (t + 1 < ntiles) stage(t + 1, (t + 1) & 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            int bi, bj;
            tile_of(t, bi, bj);
            const int i0 = k1 + bi * TILE, j0 = k1 + bj * TILE;
            // old values of this warp's 8 x 32 block (issued before the MMAs)
            const int gi = i0 + rb * 8 + lr;
            int f = 0, fu = 0;
            std::int64_t ro = 0, rou = 0;
            if (gi <= R) {
                f = S.first[gi];
                fu = S.firstU[gi];
                ro = S.roff[gi] - f;
                rou = S.roffU[gi] - fu;
            }
            double oL[4][2], oU[4][2];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int gc = j0 + ch * 32 + cb * 8 + 2 * lk + e;
                    const bool in = gi <= R && gc <= R && gc < gi;
                    oL[cb][e] = in && gc >= f ? S.L[ro + gc] : 0.0;
                    oU[cb][e] = in && gc >= fu ? S.U[rou + gc] : 0.0;
                }
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            const double* B = bufs + (t & 1) * kF2Buf;
            const double* Xi = B;
            const double* Yi = B + kF2Arr;
            const double* Xj = B + 2 * kF2Arr;
            const double* Yj = B + 3 * kF2Arr;
            double cL[4][2], cU[4][2];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) cL[cb][0] = cL[cb][1] = cU[cb][0] = cU[cb][1] = 0.0;
            for (int kc = 0; kc < kb; kc += 4) {
                const int p = kc + lk;
                const double ax = Xi[(rb * 8 + lr) * kF2Stride + p];
                const double ay = Yi[(rb * 8 + lr) * kF2Stride + p];
#pragma unroll
                for (int cb = 0; cb < 4; ++cb) {
                    const int col = ch * 32 + cb * 8 + lr;
                    const double by = Yj[col * kF2Stride + p];
                    const double bx = Xj[col * kF2Stride + p];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(cL[cb][0]), "+d"(cL[cb][1])
                                 : "d"(ax), "d"(by));
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(cU[cb][0]), "+d"(cU[cb][1])
                                 : "d"(ay), "d"(bx));
                }
            }
            if (gi <= R) {
#pragma unroll
                for (int cb = 0; cb < 4; ++cb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int gc = j0 + ch * 32 + cb * 8 + 2 * lk + e;
                        if (gc > R) continue;
                        if (gc < gi) {
                            if (gc >= f) S.L[ro + gc] = oL[cb][e] - cL[cb][e];
                            if (gc >= fu) S.U[rou + gc] = oU[cb][e] - cU[cb][e];
                        } else if (gc == gi) {
                            S.diag[gi] -= cL[cb][e];
                        }
                    }
            }
            __syncthreads();  // this buffer is restaged two tiles on
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    int bad = 0;
    double* dinv = dinv_all + vbase[j];
    for (int i = tid; i < n; i += blockDim.x) {
        const double d = S.diag[i];
        if (!(fabs(d) > 0.0) || !isfinite(d)) bad = 1;
        dinv[i] = 1.0 / d;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) status[j] = bad;
}

// ---------------------------------------------------------------- solve

/** Block shape of the pipelined triangular solves: NW warps per CTA (warp 0
 *  solves triangles, NW-1 stream panel rows), RPW rows per panel warp, so a
 *  block has RB = RPW (NW-1) rows (even: 16-byte vector loads never straddle
 *  the partial/stash boundary).  Chosen per launch from the subdomain count:
 *  one CTA per subdomain and every CTA resident in a single wave. */
template <int NW, int RPW, int MINB>
struct SolveShape {
    static constexpr int kWarps = NW, kThreads = 32 * NW, kRows = RPW, kMinBlocks = MINB;
    static constexpr int RB = RPW * (NW - 1);
    static constexpr int TS = 2 * RB + 1;  // padded stash row (previous block + own triangle)
    static_assert(RB % 2 == 0 && RB <= 32, "block rows must be even and fit one warp");
};
using ShapeBig = SolveShape<31, 1, 1>;    // n_sub <= #SMs: 992 threads, one CTA per SM
using ShapeMid = SolveShape<16, 2, 2>;    // n_sub <= 2 #SMs: 512 threads, two per SM
using ShapeSmall = SolveShape<8, 2, 4>;   // more subdomains: 256 threads, up to four per SM
using ShapeRec = SolveShape<15, 1, 2>;    // record solve, n_sub > #SMs: one row per panel warp, 2 per SM
using ShapeRec8 = SolveShape<9, 1, 2>;    // record solve with the streamed path's RB = 8 (its fallback)
constexpr int RB = ShapeMid::RB;  // the column-layout backward (upper_solve_cols) uses ShapeMid
constexpr int TS = ShapeMid::TS;
constexpr int kSolveThreads = ShapeMid::kThreads;

/** Block record layout: RB rows of [W | T^-1 | 0], row stride 2 RB + 1 (the
 *  stash's padded stride, so a record copies linearly into it); RB even
 *  keeps records 16-byte aligned. */
__host__ __device__ constexpr int rec_stride(int rb) { return 2 * rb + 1; }
__host__ __device__ constexpr int rec_size(int rb) { return rb * (2 * rb + 1); }
// distance between records: 128-byte aligned (whole lines for the bulk copies)
__host__ __device__ constexpr int rec_pitch(int rb) { return (rec_size(rb) + 15) / 16 * 16; }

// development timing trace (CPDDG_SOLVE_DEBUG & 16): per block of CTA 0,
// [k][0] step start, [k][1] warp 0 done, [k][2 + w] panel warp w done
__device__ long long g_trace[1024][20];

/** Prefetch [p, p + bytes) into L2 with the bulk-copy engine
 *  (cp.async.bulk.prefetch.L2; p and bytes 16-byte aligned). */
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
    const char* c = static_cast<const char*>(p);
    while (bytes > 0) {
        const unsigned b = static_cast<unsigned>(bytes < 65536 ? bytes : 65536);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(b) : "memory");
        c += b;
        bytes -= b;
    }
}

/** L2 prefetch of the contiguous storage of rows [b, e) (L) or columns
 *  [b, e) (U): row i occupies [ro_i, ro_i + (i + (i & 1)) - f_i). */
__device__ __noinline__ void prefetch_rows(const double* V, const int* f, const std::int64_t* ro, int b, int e) {
    if (b >= e) return;
    const std::int64_t lo = ro[b];
    const int l = e - 1;
    const std::int64_t hi = ro[l] + (l + (l & 1)) - f[l];
    if (hi > lo) prefetch_l2(V + lo, (hi - lo) * 8);
}

/** L2 prefetch of the far parts of rows [b, e) in the record layout: row i
 *  occupies [ro_i, ro_i + lim_i - f_i), lim_i = max(f_i, (i / rb - 1) rb). */
__device__ __noinline__ void prefetch_rows_far(const double* V, const int* f, const std::int64_t* ro, int b, int e,
                                               int rb) {
    if (b >= e) return;
    const std::int64_t lo = ro[b];
    const int l = e - 1;
    const std::int64_t hi = ro[l] + max(0, (l / rb - 1) * rb - f[l]);
    if (hi > lo) prefetch_l2(V + lo, (hi - lo) * 8);
}

/** Pipelined blocked lower-triangular solve y <- T^{-1} y in shared memory,
 *  T unit lower (d == nullptr) or lower with diagonal d.  Row i of T holds
 *  columns [f_i, i) contiguously at V + ro[i].  Blocks of RB rows: while warp
 *  0 solves the RB x RB triangle of block k, warps 1..15 stream block k+1's
 *  rows (two rows each, 8 loads in flight per lane, streaming cache hints)
 *  into a partial dot over the already-final columns and stash the entries
 *  that fall in blocks k and k+1; one barrier per block. */
template <class SH>
__device__ __forceinline__ void lower_solve(int n, const int* __restrict__ f, const std::int64_t* __restrict__ ro,
                                            const double* __restrict__ V, const double* __restrict__ d,
                                            double* y, double (*part)[SH::RB + 2], double (*tri)[SH::RB][SH::TS],
                                            int dbg = 0) {
    constexpr int RB = SH::RB;
    constexpr int kRowsPerWarp = SH::kRows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + RB - 1) / RB;
    auto panel = [&](int b0, int buf) {
        const int lim = b0 - RB;  // columns < lim are final
        const bool trp = (dbg & 16) && blockIdx.x == 0 && warp == 1 && lane == 0 && b0 / RB - 1 < 1024 && b0 >= RB;
        if (trp) g_trace[b0 / RB - 1][17] = clock64();
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            const int rr = kRowsPerWarp * (warp - 1) + q;
            const int i = b0 + rr;
            double s = 0.0;
            if (i < n) {
                const int fi = __ldg(f + i);
                const double* Li = V + (__ldg(ro + i) - fi);
                // stash loads first: they share the round trip of the partial loads
                const int col0 = lim + lane, col1 = lim + lane + 32;
                const double t0 = (lane < 2 * RB && col0 >= fi && col0 < i) ? ld_stream(Li + col0) : 0.0;
                const double t1 = (lane + 32 < 2 * RB && col1 >= fi && col1 < i) ? ld_stream(Li + col1) : 0.0;
                double s1 = 0.0, s2 = 0.0, s3 = 0.0;
                const double2* Li2 = reinterpret_cast<const double2*>(Li + fi);  // fi even, row 16B-aligned
                const double2* y2 = reinterpret_cast<const double2*>(y);
                for (int base = fi; base < lim; base += 512) {
                    double2 a[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int c = base + 2 * lane + 64 * u;
                        a[u] = c < lim ? ld_stream(Li2 + ((c - fi) >> 1)) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const int c = base + 2 * lane + 64 * u;
                        if (c < lim) {
                            const double2 yy = y2[c >> 1];
                            s = fma(a[u].x, yy.x, s);
                            s1 = fma(a[u].y, yy.y, s1);
                        }
                        if (c + 64 < lim) {
                            const double2 yy = y2[(c + 64) >> 1];
                            s2 = fma(a[u + 1].x, yy.x, s2);
                            s3 = fma(a[u + 1].y, yy.y, s3);
                        }
                    }
                }
                s = (s + s1) + (s2 + s3);
                if (trp && q == 0) g_trace[b0 / RB - 1][18] = clock64();
                if (lane < 2 * RB) tri[buf][rr][lane] = t0;
                if (lane + 32 < 2 * RB) tri[buf][rr][lane + 32] = t1;
            } else {
                for (int cc = lane; cc < 2 * RB; cc += 32) tri[buf][rr][cc] = 0.0;
            }
            s = warp_sum(s);
            if (trp && q == 0) g_trace[b0 / RB - 1][19] = clock64();
            if (lane == 0) part[buf][rr] = s;
        }
    };
    // rows of a block are contiguous in V: stream them into L2 two blocks ahead
    auto prefetch_block = [&](int k) {
        if (k < nblk) prefetch_rows(V, f, ro, k * RB, min(n, k * RB + RB));
    };
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2 + (dbg >> 8); ++q) prefetch_block(q);
    }
    if (warp > 0) panel(0, 0);
    __syncthreads();
    for (int k = 0; k < nblk; ++k) {
        const int cur = k & 1;
        const int r0 = k * RB;
        const bool tr = (dbg & 16) && blockIdx.x == 0 && k < 1024;
        if (tr && threadIdx.x == 0) g_trace[k][0] = clock64();
        if (threadIdx.x == 0 && !(dbg & 4)) prefetch_block(k + 2 + (dbg >> 8));
        if (warp == 0 && !(dbg & 1)) {
            const int i = r0 + lane;
            const bool live = lane < RB && i < n;
            // this lane's reciprocal pivot, loaded before the chain (a load
            // inside the substitution loop would sit on its critical path)
            const double dl = (d && live) ? __ldg(d + i) : 1.0;
            double s = 0.0;
            if (live) {
                s = y[i] - part[cur][lane];
                if (r0 >= RB) {
#pragma unroll 6
                    for (int c = 0; c < RB; ++c) s = fma(-tri[cur][lane][c], y[r0 - RB + c], s);
                }
            }
            const int rb = min(RB, n - r0);
            for (int c = 0; c < rb; ++c) {
                if (d && lane == c) s *= dl;  // d: reciprocal pivots
                const double xc = __shfl_sync(0xffffffffu, s, c);
                if (lane > c && live) s = fma(-tri[cur][lane][RB + c], xc, s);
            }
            if (live) y[i] = s;
            if (tr && lane == 0) g_trace[k][1] = clock64();
        } else if (warp > 0 && k + 1 < nblk && !(dbg & 2)) {
            panel((k + 1) * RB, cur ^ 1);
            if (tr && lane == 0 && warp < 18) g_trace[k][1 + warp] = clock64();
        }
        __syncthreads();
    }
}

/** Record lower solve y <- T^-1 y (T unit lower, or lower with its pivots
 *  folded into the records) on the far parts of T's rows: row i keeps
 *  columns [f_i, (i / RB - 1) RB) at V + ro_i, the rest of the row is in the
 *  block records [W | T_kk^-1] (k_block_records).  Step k: warp 0 forms
 *  x_k = T_kk^-1 (y_k - part_k) - W_k x_{k-1} (no dependent chain); panel
 *  warp w owns rows RPW (w-1) .. of every block and computes block k+1's
 *  far-part dots.  The far part of a row does not depend on x, so the first
 *  512 columns of each warp's first row of block k+2 are loaded at the end
 *  of step k and held in registers across the barrier: a step waits on one
 *  load round trip (the warp's other rows), not two.  Row tables (f, ro) go
 *  through a shared ring three blocks ahead, records by cp.async a step
 *  ahead; one barrier per block. */
template <class SH>
__device__ __forceinline__ void lower_solve_rec(int n, const int* __restrict__ f, const std::int64_t* __restrict__ ro,
                                                const double* __restrict__ V, const double* __restrict__ rec,
                                                double* y, double (*part)[SH::RB + 2], double (*tri)[SH::RB][SH::TS],
                                                int (*tf)[SH::RB], long long (*tro)[SH::RB], int dbg) {
    constexpr int RB = SH::RB, RPW = SH::kRows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ptid = threadIdx.x - 32;
    const int nblk = (n + RB - 1) / RB;
    const int rr0 = RPW * (warp - 1);  // this panel warp's first row in a block
    const double2* y2 = reinterpret_cast<const double2*>(y);
    // table loads are issued at a step's start and stored at its end (a store
    // right after the load would stall the loading warp for a round trip)
    auto table_load = [&](int B, int& fv, long long& rv) {
        fv = 0;
        rv = 0;
        if (B < nblk && ptid >= 0 && ptid < RB && B * RB + ptid < n) {
            fv = __ldg(f + B * RB + ptid);
            rv = __ldg(ro + B * RB + ptid);
        }
    };
    auto table_store = [&](int B, int fv, long long rv) {
        if (B < nblk && ptid >= 0 && ptid < RB) {
            tf[B & 3][ptid] = fv;
            tro[B & 3][ptid] = rv;
        }
    };
    auto load_table = [&](int B) {
        int fv;
        long long rv;
        table_load(B, fv, rv);
        table_store(B, fv, rv);
    };
    auto load_rec = [&](int B, int buf) {
        const double* src = rec + static_cast<std::int64_t>(B) * rec_pitch(RB);
        const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(&tri[buf][0][0]));
        for (int e = 2 * ptid; e < rec_size(RB); e += 2 * (blockDim.x - 32))
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + 8 * e), "l"(src + e) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double2 pre[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pre[u] = make_double2(0.0, 0.0);
    // first 512 columns of row rr0 of block B (far part [f, (B - 1) RB))
    auto issue_pre = [&](int B) {
        const int i = B * RB + rr0, lim = (B - 1) * RB;
        const bool ok = B < nblk && i < n;
        const int fi = ok ? tf[B & 3][rr0] : 0;
        const double2* L2 = reinterpret_cast<const double2*>(V + (ok ? tro[B & 3][rr0] : 0));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int c = fi + 2 * lane + 64 * u;
            pre[u] = (ok && c < lim) ? ld_stream(L2 + lane + 32 * u) : make_double2(0.0, 0.0);
        }
    };
    // dot of y with the columns [c, lim) of a row held as a[] (c = fi + 2 lane + 64 u + base)
    auto dot8 = [&](const double2* a, int cb, int lim, double& s0, double& s1, double& s2, double& s3) {
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            const int c = cb + 2 * lane + 64 * u;
            if (c < lim) {
                const double2 yy = y2[c >> 1];
                s0 = fma(a[u].x, yy.x, s0);
                s1 = fma(a[u].y, yy.y, s1);
            }
            if (c + 64 < lim) {
                const double2 yy = y2[(c + 64) >> 1];
                s2 = fma(a[u + 1].x, yy.x, s2);
                s3 = fma(a[u + 1].y, yy.y, s3);
            }
        }
    };
    // the rest of a row from column cb on, loaded in this step
    auto stream_row = [&](const double2* L2, int fi, int cb, int lim, double& s0, double& s1, double& s2,
                          double& s3) {
        for (int base = cb; base < lim; base += 512) {
            double2 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = base + 2 * lane + 64 * u;
                a[u] = c < lim ? ld_stream(L2 + ((c - fi) >> 1)) : make_double2(0.0, 0.0);
            }
            dot8(a, base, lim, s0, s1, s2, s3);
        }
    };
    auto panel = [&](int B, int buf, bool tr) {
        const bool tw = tr && lane == 0 && warp == 1;
        const int b0 = B * RB, lim = b0 - RB;
        if (!(dbg & 2)) load_rec(B, buf);  // dbg & 2: no records (timing experiments)
        double sr[RPW];
        {
            const int fi = tf[B & 3][rr0];
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            dot8(pre, fi, lim, s0, s1, s2, s3);
            if (fi + 512 < lim)
                stream_row(reinterpret_cast<const double2*>(V + tro[B & 3][rr0]), fi, fi + 512, lim, s0, s1, s2, s3);
            sr[0] = (s0 + s1) + (s2 + s3);
        }
        if (tw) g_trace[B - 1][2] = clock64();
#pragma unroll
        for (int q = 1; q < RPW; ++q) {
            const int fi = tf[B & 3][rr0 + q];
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            stream_row(reinterpret_cast<const double2*>(V + tro[B & 3][rr0 + q]), fi, fi, lim, s0, s1, s2, s3);
            sr[q] = (s0 + s1) + (s2 + s3);
        }
        if (tw) g_trace[B - 1][3] = clock64();
        issue_pre(B + 1);  // in flight across the barrier
        if (tw) g_trace[B - 1][4] = clock64();
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const double s = warp_sum(sr[q]);
            if (lane == 0) part[buf][rr0 + q] = s;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (tw) g_trace[B - 1][5] = clock64();
        if (tr && lane == 0) g_trace[B - 1][6 + warp] = clock64();
    };
    // L2 bulk prefetch of block B's far rows (tables from the shared ring) and record
    auto prefetch_block = [&](int B) {
        if (B < nblk) {
            const int l = min(RB, n - B * RB) - 1;
            const long long lo = tro[B & 3][0];
            const long long hi = tro[B & 3][l] + max(0, (B - 1) * RB - tf[B & 3][l]);
            if (hi > lo) prefetch_l2(V + lo, (hi - lo) * 8);
            prefetch_l2(rec + static_cast<std::int64_t>(B) * rec_pitch(RB), 8LL * rec_size(RB));
        }
    };
    load_table(0);
    load_table(1);
    load_table(2);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = 0; q < 2; ++q) prefetch_block(q);
    if (warp > 0) panel(0, 0, false);  // block 0: empty far parts, record 0, pre for block 1
    __syncthreads();
    for (int k = 0; k < nblk; ++k) {
        const int cur = k & 1;
        const int r0 = k * RB;
        const bool tr = (dbg & 16) && blockIdx.x == (dbg >> 16) && k < 1024;
        if (tr && threadIdx.x == 0) g_trace[k][0] = clock64();
        // L2 bulk prefetch two blocks ahead (tables of block k + 2 are in the
        // ring since step k - 1); dbg & 4: off
        if (!(dbg & 4) && threadIdx.x == 0) prefetch_block(k + 2);
        if (warp == 0 && !(dbg & 1)) {  // dbg & 1: warp 0 idle (timing experiments)
            const int i = r0 + lane;
            const bool live = lane < RB && i < n;
            const double t = live ? y[i] - part[cur][lane] : 0.0;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            const double* trow = tri[cur][lane < RB ? lane : 0];
#pragma unroll
            for (int c = 0; c < RB; c += 2) {
                const double t0 = __shfl_sync(0xffffffffu, t, c);
                const double t1 = __shfl_sync(0xffffffffu, t, c + 1);
                a2 = fma(trow[RB + c], t0, a2);
                a3 = fma(trow[RB + c + 1], t1, a3);
            }
            if (r0 >= RB) {
#pragma unroll
                for (int c = 0; c < RB; c += 2) {
                    a0 = fma(trow[c], y[r0 - RB + c], a0);
                    a1 = fma(trow[c + 1], y[r0 - RB + c + 1], a1);
                }
            }
            if (live) y[i] = (a2 + a3) - (a0 + a1);
            if (tr && lane == 0) g_trace[k][1] = clock64();
        } else if (warp > 0) {
            int fv;
            long long rv;
            table_load(k + 3, fv, rv);
            if (k + 1 < nblk) panel(k + 1, cur ^ 1, tr);
            table_store(k + 3, fv, rv);
        }
        __syncthreads();
    }
}

/** Re-lay U (column profile storage from the factorisation) as reversed
 *  rows for a row-oriented backward pass: reversed row i' = n-1-i holds
 *  U(i, j), j in (i, rlast_i], at reversed column j' = n-1-j over
 *  [uf_i', i') (uf even, lengths even: 16-byte aligned like L).  Entries of
 *  the row range outside the column profile are stored zeros. */
__global__ void __launch_bounds__(256) k_reverse_u(const int* __restrict__ order, const int* __restrict__ n_rows,
                                                   const std::int64_t* __restrict__ vbase,
                                                   const std::int64_t* __restrict__ ebase,
                                                   const std::int64_t* __restrict__ ubase,
                                                   const int* __restrict__ first_all,
                                                   const std::int64_t* __restrict__ roff_all,
                                                   const int* __restrict__ ufirst_all,
                                                   const std::int64_t* __restrict__ uroff_all,
                                                   const double* __restrict__ dinv_all,
                                                   const double* __restrict__ Ucol_all, double* __restrict__ Urev_all,
                                                   double* __restrict__ drev_all) {
    const int j = order[blockIdx.x];
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    const int* first = first_all + vb;
    const std::int64_t* roff = roff_all + vb;
    const int* ufirst = ufirst_all + vb;
    const std::int64_t* uroff = uroff_all + vb;
    const double* Ucol = Ucol_all + ebase[j];
    double* Urev = Urev_all + ubase[j];
    for (int ip = threadIdx.x; ip < n; ip += blockDim.x) {
        const int i = n - 1 - ip;
        drev_all[vb + ip] = dinv_all[vb + i];
        const int fpr = ufirst[ip];
        double* out = Urev + uroff[ip] - fpr;
        const int end = ip + (ip & 1);
        for (int jp = fpr; jp < end; ++jp) {
            double v = 0.0;
            if (jp < ip) {
                const int c = n - 1 - jp;
                const int fc = first[c];
                if (c > i && i >= fc) v = Ucol[roff[c] + i - fc];
            }
            out[jp] = v;
        }
    }
}

/** Block records of the blocked lower solve (T unit lower, or lower with
 *  reciprocal pivots d), for blocks of RB rows.  Block k (rows r0 = k RB ..)
 *  satisfies T_kk x_k = s_k - T_k,k-1 x_{k-1}, s_k = y_k - (row dots over
 *  the columns before block k-1), so with the block's triangle inverted
 *
 *      x_k = T_kk^-1 s_k - W_k x_{k-1},   W_k = T_kk^-1 T_k,k-1,
 *
 *  a dense RB x 2RB matrix-vector product instead of RB dependent
 *  substitution steps.  Record k = [W_k | T_kk^-1] row-major (RB x 2RB,
 *  zero-padded past the last row; W_0 = 0).  One warp per block: lane e
 *  solves T_kk x = e_e (the reference substitution order, column by column)
 *  into X[.][e]; then W = X P with P the block's previous-block columns. */
template <int RB>
__global__ void __launch_bounds__(64) k_block_records(const int* __restrict__ n_rows,
                                                       const std::int64_t* __restrict__ vbase,
                                                       const std::int64_t* __restrict__ ebase,
                                                       const int* __restrict__ f_all,
                                                       const std::int64_t* __restrict__ ro_all,
                                                       const double* __restrict__ V_all,
                                                       const double* __restrict__ d_all,
                                                       const std::int64_t* __restrict__ rbase,
                                                       double* __restrict__ rec_all) {
    __shared__ double X[2][RB][33], P[2][RB][33];
    const int j = blockIdx.x;
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    const int* f = f_all + vb;
    const std::int64_t* ro = ro_all + vb;
    const double* V = V_all + ebase[j];
    const double* d = d_all ? d_all + vb : nullptr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + RB - 1) / RB;
    for (int k = blockIdx.y * 2 + warp; k < nblk; k += 2 * gridDim.y) {
        const int r0 = k * RB, rb = min(RB, n - r0);
        double* rec = rec_all + rbase[j] + static_cast<std::int64_t>(k) * rec_pitch(RB);
        for (int i = 0; i < RB; ++i) {
            double s = 0.0;
            if (i < rb) {
                const int gi = r0 + i;
                const double* Ti = V + ro[gi] - f[gi];
                s = lane == i ? 1.0 : 0.0;
                for (int c = max(0, f[gi] - r0); c < i; ++c) s = fma(-Ti[r0 + c], X[warp][c][lane], s);
                if (d) s *= d[gi];
                // previous-block columns of this row
                const int pc = r0 - RB + lane;
                P[warp][i][lane] = (k > 0 && lane < RB && pc >= f[gi]) ? Ti[pc] : 0.0;
            } else {
                P[warp][i][lane] = 0.0;
            }
            X[warp][i][lane] = s;
            __syncwarp();
        }
        for (int i = 0; i < RB; ++i) {
            if (lane < RB) {
                double w = 0.0;
                for (int m = 0; m <= i && m < rb; ++m) w = fma(X[warp][i][m], P[warp][m][lane], w);
                rec[i * rec_stride(RB) + lane] = w;
                rec[i * rec_stride(RB) + RB + lane] = X[warp][i][lane];
                if (lane == 0) rec[i * rec_stride(RB) + 2 * RB] = 0.0;
            }
        }
        __syncwarp();
    }
}

/** Block records of the column-oriented backward solve U x = y (blocks of
 *  RB rows from the last): block K satisfies U_KK x_K = y_K - U_K,K+1 x_{K+1}
 *  - (updates of blocks > K + 1), so record K = [W_K | U_KK^-1] with
 *  W_K = U_KK^-1 U_K,K+1 (zero for the last block).  U column c holds rows
 *  [f_c, c) at V + ro_c; d = reciprocal pivots.  One warp per block: lane e
 *  solves U_KK x = e_e by backward substitution into X[.][e]. */
template <int RB>
__global__ void __launch_bounds__(64) k_block_records_upper(const int* __restrict__ n_rows,
                                                            const std::int64_t* __restrict__ vbase,
                                                            const std::int64_t* __restrict__ ebase,
                                                            const int* __restrict__ f_all,
                                                            const std::int64_t* __restrict__ ro_all,
                                                            const double* __restrict__ V_all,
                                                            const double* __restrict__ d_all,
                                                            const std::int64_t* __restrict__ rbase,
                                                            double* __restrict__ rec_all) {
    __shared__ double X[2][RB][33], P[2][RB][33];
    const int j = blockIdx.x;
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    const int* f = f_all + vb;
    const std::int64_t* ro = ro_all + vb;
    const double* V = V_all + ebase[j];
    const double* d = d_all + vb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + RB - 1) / RB;
    auto U = [&](int r, int c) { return r >= f[c] ? V[ro[c] + r - f[c]] : 0.0; };
    for (int k = blockIdx.y * 2 + warp; k < nblk; k += 2 * gridDim.y) {
        const int r0 = k * RB, rb = min(RB, n - r0);
        double* rec = rec_all + rbase[j] + static_cast<std::int64_t>(k) * rec_pitch(RB);
        for (int i = RB - 1; i >= 0; --i) {
            double s = 0.0;
            if (i < rb) {
                const int gi = r0 + i;
                s = lane == i ? 1.0 : 0.0;
                for (int c = rb - 1; c > i; --c) s = fma(-U(gi, r0 + c), X[warp][c][lane], s);
                s *= d[gi];
                const int nc = r0 + RB + lane;  // next block's columns
                P[warp][i][lane] = (lane < RB && nc < n) ? U(gi, nc) : 0.0;
            } else {
                P[warp][i][lane] = 0.0;
            }
            X[warp][i][lane] = s;
            __syncwarp();
        }
        for (int i = 0; i < RB; ++i) {
            if (lane < RB) {
                double w = 0.0;
                for (int m = i; m < rb; ++m) w = fma(X[warp][i][m], P[warp][m][lane], w);
                rec[i * rec_stride(RB) + lane] = w;
                rec[i * rec_stride(RB) + RB + lane] = X[warp][i][lane];
                if (lane == 0) rec[i * rec_stride(RB) + 2 * RB] = 0.0;
            }
        }
        __syncwarp();
    }
}

/** Far part of each row for the record solve: row i keeps columns
 *  [f_i, lim_i), lim_i = max(f_i, (i / RB - 1) RB) -- everything left of the
 *  previous block (the rest is in the block records).  lim_i and f_i are
 *  even, so rows stay 16-byte aligned.  One warp per row. */
template <int RB>
__global__ void __launch_bounds__(256) k_compact_rows(const int* __restrict__ n_rows,
                                                      const std::int64_t* __restrict__ vbase,
                                                      const std::int64_t* __restrict__ ebase,
                                                      const int* __restrict__ f_all,
                                                      const std::int64_t* __restrict__ ro_all,
                                                      const double* __restrict__ V_all,
                                                      const std::int64_t* __restrict__ cbase,
                                                      const std::int64_t* __restrict__ roc_all,
                                                      double* __restrict__ Vc_all) {
    const int j = blockIdx.x;
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = warp; i < n; i += 8) {
        const int fi = f_all[vb + i];
        const int lim = max(fi, (i / RB - 1) * RB);
        const double* src = V_all + ebase[j] + ro_all[vb + i] - fi;
        double* dst = Vc_all + cbase[j] + roc_all[vb + i] - fi;
        for (int c = fi + lane; c < lim; c += 32) dst[c] = src[c];
    }
}

/** Pipelined blocked backward substitution U x = y with U stored by columns
 *  (column c holds rows [f_c, c) contiguously at V + ro[c]; reciprocal
 *  pivots d).  Blocks of RB columns from the last.  Step K: warp 0 applies
 *  block K+1's columns to block K's rows and solves block K's triangle, both
 *  from a shared-memory stash; warps 1..15 apply block K+1's columns to every
 *  row above block K (thread per row pair, coalesced 16-byte loads down the
 *  columns), load the stash for block K-1 and the column tables (f, ro) of
 *  block K-2.  Every load of a step is independent of the step's other loads
 *  (tables come from shared memory, loaded a step ahead), so a step costs
 *  the round trips of its update batches only; one barrier per block.
 *  Streams each stored entry of U exactly once.  cf, cro: [4][RB] ring of
 *  column tables indexed by block % 4. */
__device__ __forceinline__ void upper_solve_cols(int n, const int* __restrict__ f,
                                                 const std::int64_t* __restrict__ ro,
                                                 const double* __restrict__ V, const double* __restrict__ d,
                                                 double* y, double (*tri)[RB][TS], int (*cf)[RB],
                                                 long long (*cro)[RB], int pf) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + RB - 1) / RB;
    const int ptid = threadIdx.x - 32, pthreads = blockDim.x - 32;
    constexpr int kStash = (RB * 2 * RB + 479) / 480;  // stash entries per panel thread
    // column table of block K into ring slot K % 4 (panel threads < RB)
    auto table_load = [&](int K, int& tf, long long& tro) {
        const int col = K * RB + ptid;
        tf = n;
        tro = 0;
        if (K >= 0 && ptid < RB && col < n) {
            tf = __ldg(f + col);
            tro = __ldg(ro + col);
        }
    };
    auto table_store = [&](int K, int tf, long long tro) {
        if (K >= 0 && ptid < RB) {
            cf[K & 3][ptid] = tf;
            cro[K & 3][ptid] = tro;
        }
    };
    // stash for block K: tri[buf][i][c] = U(c0+i, c0+c), c in [0, 2RB): block
    // K's columns then block K+1's; tables of blocks K, K+1 in shared memory
    auto stash_load = [&](int K, double* v) {
        const int c0 = K * RB;
#pragma unroll
        for (int q = 0; q < kStash; ++q) {
            const int e = ptid + q * pthreads;
            v[q] = 0.0;
            if (e < RB * 2 * RB) {
                const int il = e / (2 * RB), cl = e % (2 * RB);
                const int i = c0 + il, col = c0 + cl;
                if (col < n && i < col) {
                    const int slot = (cl < RB ? K : K + 1) & 3, cc = cl < RB ? cl : cl - RB;
                    const int fc = cf[slot][cc];
                    if (i >= fc) v[q] = ld_stream(V + cro[slot][cc] + (i - fc));
                }
            }
        }
    };
    auto stash_store = [&](const double* v, int buf) {
#pragma unroll
        for (int q = 0; q < kStash; ++q) {
            const int e = ptid + q * pthreads;
            if (e < RB * 2 * RB) tri[buf][e / (2 * RB)][e % (2 * RB)] = v[q];
        }
    };
    auto prefetch_block = [&](int K) {
        if (K >= 0) prefetch_rows(V, f, ro, K * RB, min(n, K * RB + RB));
    };
    if (warp > 0) {
        int tf;
        long long tro;
        table_load(nblk - 1, tf, tro);
        table_store(nblk - 1, tf, tro);
        table_load(nblk - 2, tf, tro);
        table_store(nblk - 2, tf, tro);
        if (ptid == 0)
            for (int q = 1; q <= pf; ++q) prefetch_block(nblk - q);
    }
    __syncthreads();
    if (warp > 0) {
        double sv[kStash];
        stash_load(nblk - 1, sv);
        stash_store(sv, (nblk - 1) & 1);
    }
    __syncthreads();
    for (int K = nblk - 1; K >= 0; --K) {
        const int cur = K & 1;
        const int c0 = K * RB;
        if (warp == 0) {
            const int i = c0 + lane;
            const bool live = lane < RB && i < n;
            double s = live ? y[i] : 0.0;
            if (live && K + 1 < nblk) {
                const int nb1 = min(RB, n - (c0 + RB));
#pragma unroll 6
                for (int c = 0; c < nb1; ++c) s = fma(-tri[cur][lane][RB + c], y[c0 + RB + c], s);
            }
            const int cb = min(RB, n - c0);
            const double dinv = live ? __ldg(d + c0 + lane) : 0.0;  // reciprocal pivots (k_factor)
            for (int c = cb - 1; c >= 0; --c) {
                if (lane == c) s *= dinv;
                const double xc = __shfl_sync(0xffffffffu, s, c);
                if (lane < c && live) s = fma(-tri[cur][lane][c], xc, s);
            }
            if (live) y[i] = s;
        } else {
            // the columns the row updates need pf steps from now (bulk L2 prefetch
            // from a panel thread: warp 0 is on the critical path)
            if (ptid == 0 && pf > 0) prefetch_block(K - pf);
            int tf;
            long long tro;
            table_load(K - 2, tf, tro);
            double sv[kStash];
            if (K >= 1) stash_load(K - 1, sv);
            if (K + 1 < nblk) {
                // rows above block K from block K+1's columns
                const int nxt = (K + 1) & 3;
                const int cb1 = min(RB, n - (c0 + RB));
                int jmin = c0;
                for (int c = 0; c < cb1; ++c) jmin = min(jmin, cf[nxt][c]);
                // one thread per row pair (16-byte loads down each column: columns
                // start at even rows and c0 is even), all RB columns in three
                // batches of ten loads issued before their FMAs
                for (int base = jmin & ~1; base < c0; base += 2 * pthreads) {
                    const int jr = base + 2 * ptid;
                    const bool ok = jr < c0;
                    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                    for (int cb = 0; cb < RB; cb += 10) {
                        double2 a[10];
#pragma unroll
                        for (int u = 0; u < 10; ++u) {
                            const int c = cb + u;
                            a[u] = (ok && c < cb1 && jr >= cf[nxt][c])
                                       ? ld_stream(reinterpret_cast<const double2*>(V + cro[nxt][c] + (jr - cf[nxt][c])))
                                       : make_double2(0.0, 0.0);
                        }
#pragma unroll
                        for (int u = 0; u < 10; ++u) {
                            const int c = cb + u;
                            if (c < cb1) {
                                const double xc = y[c0 + RB + c];
                                acc0 = fma(a[u].x, xc, acc0);
                                acc1 = fma(a[u].y, xc, acc1);
                            }
                        }
                    }
                    if (ok) {
                        y[jr] -= acc0;
                        y[jr + 1] -= acc1;
                    }
                }
            }
            if (K >= 1) stash_store(sv, cur ^ 1);
            table_store(K - 2, tf, tro);  // slot (K-2) & 3 == (K+2) & 3: no longer read
        }
        __syncthreads();
    }
}

/** Record backward solve on U's column envelope (far parts only: column c
 *  keeps rows [f_c, (c / RB - 1) RB), the rest is in the block records).
 *  Step K: warp 0 forms x_K = U_KK^-1 y_K - W_K x_{K+1} from the record in
 *  the stash; the panel warps apply block K+1's columns to every row above
 *  block K -- lane = (row pair, group of 8 columns), 16-byte loads down the
 *  columns, the four groups of a pair combined by a fixed butterfly (results
 *  are bitwise reproducible) -- and bring in block K-1's record (cp.async)
 *  and block K's column tables (shared ring of two).  Streams each stored
 *  entry of U exactly once; one barrier per block. */
template <class SH>
__device__ __forceinline__ void upper_solve_rec(int n, const int* __restrict__ f, const std::int64_t* __restrict__ ro,
                                                const double* __restrict__ V, const double* __restrict__ rec,
                                                double* y, double (*tri)[SH::RB][SH::TS], int (*cf)[SH::RB],
                                                long long (*cro)[SH::RB]) {
    constexpr int RB = SH::RB;
    constexpr int kPanelWarps = SH::kWarps - 1;
    constexpr int NG = (RB + 7) / 8;  // groups of eight columns per block
    constexpr int PPW = 32 / NG;      // row pairs per warp pass
    static_assert(NG == 1 || NG == 2 || NG == 4, "one, two or four groups of eight columns cover a block");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - 32;
    const int nblk = (n + RB - 1) / RB;
    auto load_rec = [&](int K, int buf) {
        const double* src = rec + static_cast<std::int64_t>(K) * rec_pitch(RB);
        const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(&tri[buf][0][0]));
        for (int e = 2 * ptid; e < rec_size(RB); e += 2 * (blockDim.x - 32))
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + 8 * e), "l"(src + e) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto load_table = [&](int K, int slot) {
        if (K >= 0 && ptid < RB) {
            const int c = K * RB + ptid;
            cf[slot][ptid] = c < n ? __ldg(f + c) : INT_MAX;
            cro[slot][ptid] = c < n ? __ldg(ro + c) : 0;
        }
    };
    // columns of block K: contiguous far parts [ro_{K RB}, end of the last
    // column), from the shared table of block K
    auto prefetch_block = [&](int K, int slot) {
        if (K >= 1) {
            const int l = min(RB, n - K * RB) - 1;
            const long long lo = cro[slot][0];
            const long long hi = cro[slot][l] + max(0, (K - 1) * RB - cf[slot][l]);
            if (hi > lo) prefetch_l2(V + lo, (hi - lo) * 8);
        }
    };
    if (warp > 0) {
        load_rec(nblk - 1, (nblk - 1) & 1);
        load_table(nblk - 1, (nblk - 1) & 1);
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    if (ptid == 0) prefetch_block(nblk - 1, (nblk - 1) & 1);
    for (int K = nblk - 1; K >= 0; --K) {
        const int cur = K & 1;
        const int r0 = K * RB;
        if (warp == 0) {
            const int i = r0 + lane;
            const bool live = lane < RB && i < n;
            const double t = live ? y[i] : 0.0;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            const double* trow = tri[cur][lane < RB ? lane : 0];
#pragma unroll
            for (int c = 0; c < RB; c += 2) {
                const double t0 = __shfl_sync(0xffffffffu, t, c);
                const double t1 = __shfl_sync(0xffffffffu, t, c + 1);
                a2 = fma(trow[RB + c], t0, a2);
                a3 = fma(trow[RB + c + 1], t1, a3);
            }
            if (K + 1 < nblk) {
                const int nb = min(RB, n - (r0 + RB));
                for (int c = 0; c < nb; ++c) (c & 1 ? a1 : a0) = fma(trow[c], y[r0 + RB + c], c & 1 ? a1 : a0);
            }
            if (live) y[i] = (a2 + a3) - (a0 + a1);
        } else {
            if (K >= 1) load_rec(K - 1, cur ^ 1);
            if (ptid == 0 && K >= 2)
                prefetch_l2(rec + static_cast<std::int64_t>(K - 2) * rec_pitch(RB), 8LL * rec_size(RB));
            // block K's column table, for step K - 1 (slot cur was last read at
            // step K + 1); loaded now, stored after this step's loads
            int tfv = INT_MAX;
            long long trv = 0;
            if (K >= 0 && ptid < RB && K * RB + ptid < n) {
                tfv = __ldg(f + K * RB + ptid);
                trv = __ldg(ro + K * RB + ptid);
            }
            if (K + 1 < nblk) {
                const int slot = cur ^ 1;
                const int c0 = r0 + RB;
                const int g = lane % NG, pp = lane / NG;
                int jmin = r0;
                for (int c = 0; c < RB; ++c) jmin = min(jmin, cf[slot][c]);
                double xc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = g * 8 + u;
                    xc[u] = c < RB && c0 + c < n ? y[c0 + c] : 0.0;
                }
                for (int base = (jmin & ~1) + 2 * PPW * (warp - 1); base < r0; base += 2 * PPW * kPanelWarps) {
                    const int r = base + 2 * pp;
                    double2 a[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int c = g * 8 + u;
                        const int fc = c < RB ? cf[slot][c] : INT_MAX;
                        a[u] = (r < r0 && r >= fc)
                                   ? ld_stream(reinterpret_cast<const double2*>(V + cro[slot][c] + (r - fc)))
                                   : make_double2(0.0, 0.0);
                    }
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        s0 = fma(a[u].x, xc[u], s0);
                        s1 = fma(a[u].y, xc[u], s1);
                    }
#pragma unroll
                    for (int m = 1; m < NG; m <<= 1) {
                        s0 += __shfl_xor_sync(0xffffffffu, s0, m);
                        s1 += __shfl_xor_sync(0xffffffffu, s1, m);
                    }
                    if (g == 0 && r < r0) {
                        y[r] -= s0;
                        y[r + 1] -= s1;
                    }
                }
            }
            if (ptid < RB) {
                cf[cur][ptid] = tfv;
                cro[cur][ptid] = trv;
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        __syncthreads();
        // block K's columns are applied at step K - 1: bulk-prefetch them now
        if (ptid == 0 && K >= 1) prefetch_block(K, cur);
    }
}

// MODE 0: full apply; 1: forward only; 2: backward only (profiling);
// 3: factor probe -- r / z are per-row arrays in factor order (vbase
//    indexing) instead of global vectors, no gather / scatter.
// UROWS: backward on reversed U rows (k_reverse_u) instead of U columns.
// INV: record solve (k_block_records) on the compacted far rows.
template <int MODE, bool UROWS, class SH, bool INV>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks) k_solve(const int* __restrict__ order,
                                                            const int* __restrict__ n_rows,
                                                            const std::int64_t* __restrict__ vbase,
                                                            const std::int64_t* __restrict__ ebase,
                                                            const int* __restrict__ first_all,
                                                            const std::int64_t* __restrict__ roff_all,
                                                            const std::int64_t* __restrict__ ebaseU,
                                                            const int* __restrict__ firstU_all,
                                                            const std::int64_t* __restrict__ roffU_all,
                                                            const double* __restrict__ diag_all,
                                                            const double* __restrict__ L_all,
                                                            const double* __restrict__ U_all,
                                                            const int* __restrict__ gidx_all,
                                                            const int* __restrict__ sidx_all,
                                                            const double* __restrict__ r, double* z,
                                                            int accumulate, int pf,
                                                            const std::int64_t* __restrict__ ubase,
                                                            const int* __restrict__ ufirst_all,
                                                            const std::int64_t* __restrict__ uroff_all,
                                                            const double* __restrict__ drev_all, int dbg,
                                                            const std::int64_t* __restrict__ rbase,
                                                            const double* __restrict__ recL_all,
                                                            const double* __restrict__ recU_all) {
    const int j = order[blockIdx.x];
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    extern __shared__ double y[];
    __shared__ double part[2][SH::RB + 2];
    __shared__ __align__(16) double tri[2][SH::RB][SH::TS];
    const int tid = threadIdx.x;
    // development (CPDDG_SOLVE_DEBUG & 32): per-CTA start / end (globaltimer ns), SM, subdomain
    const bool ctr = (dbg & 32) && tid == 0 && blockIdx.x < 1024;
    if (ctr) {
        long long t0;
        unsigned sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace[blockIdx.x][0] = t0;
        g_trace[blockIdx.x][2] = sm;
        g_trace[blockIdx.x][3] = j;
    }

    for (int p = tid; p < n; p += blockDim.x) {
        if (MODE == 3) {
            y[p] = r[vb + p];
        } else {
            const int g = __ldg(gidx_all + vb + p);
            y[p] = g >= 0 ? __ldg(r + g) : 0.0;
        }
    }
    __syncthreads();
    // forward: L y = b (unit lower)
    __shared__ int tf[4][SH::RB];
    __shared__ long long tro[4][SH::RB];
    if (MODE != 2) {
        if constexpr (INV)
            lower_solve_rec<SH>(n, first_all + vb, roff_all + vb, L_all + ebase[j], recL_all + rbase[j], y, part, tri,
                                tf, tro, dbg);
        else
            lower_solve<SH>(n, first_all + vb, roff_all + vb, L_all + ebase[j], nullptr, y, part, tri, dbg);
    }
    if constexpr (UROWS) {
        // backward: U x = y as a forward solve on the reversed system
        for (int p = tid; p < n / 2; p += blockDim.x) {
            const double t = y[p];
            y[p] = y[n - 1 - p];
            y[n - 1 - p] = t;
        }
        __syncthreads();
        if (MODE != 1)
        {
            if constexpr (INV)
                lower_solve_rec<SH>(n, ufirst_all + vb, uroff_all + vb, U_all + ubase[j], recU_all + rbase[j], y, part,
                                    tri, tf, tro, dbg);
            else
                lower_solve<SH>(n, ufirst_all + vb, uroff_all + vb, U_all + ubase[j], drev_all + vb, y, part, tri, dbg);
        }
        for (int p = tid; p < n; p += blockDim.x) {
            if (MODE == 3) {
                z[vb + p] = y[n - 1 - p];
                continue;
            }
            const int s = __ldg(sidx_all + vb + p);
            if (s >= 0) {
                const double v = y[n - 1 - p];
                z[s] = accumulate ? z[s] + v : v;
            }
        }
        if (ctr) {
            long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_trace[blockIdx.x][1] = t1;
        }
    } else {
        if constexpr (INV) {
            // backward: U x = y on the far parts of U's columns + block records
            __shared__ int cf[2][SH::RB];
            __shared__ long long cro[2][SH::RB];
            if (MODE != 1)
                upper_solve_rec<SH>(n, firstU_all + vb, roffU_all + vb, U_all + ebaseU[j], recU_all + rbase[j], y, tri,
                                    cf, cro);
        } else {
            static_assert(INV || std::is_same_v<SH, ShapeMid>, "the column-layout backward is built for ShapeMid");
            // backward: U x = y, column-oriented on the factorisation's U layout
            __shared__ int cf[4][RB];
            __shared__ long long cro[4][RB];
            if (MODE != 1)
                upper_solve_cols(n, firstU_all + vb, roffU_all + vb, U_all + ebaseU[j], diag_all + vb, y, tri, cf, cro,
                                 pf);
        }
        for (int p = tid; p < n; p += blockDim.x) {
            if (MODE == 3) {
                z[vb + p] = y[p];
                continue;
            }
            const int s = __ldg(sidx_all + vb + p);
            if (s >= 0) z[s] = accumulate ? z[s] + y[p] : y[p];
        }
        if (ctr) {
            long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_trace[blockIdx.x][1] = t1;
        }
    }
}

// ------------------------------------------------- persistent TMA-streamed solve
//
// The register-staged k_solve keeps one wave of factor loads in flight per
// warp and waits, every block step, for the slowest of its warps' loads: a
// latency-bound 4.6 TB/s.  k_solve_tma decouples the stream from the steps:
// one CTA per SM walks its subdomains (assigned longest-processing-time first
// with a measured per-step cost model) and, per subdomain, the forward then
// the backward record solve (blocks of RB = 8 rows).  Every step is an *item*
// -- the far rows (forward) or far columns (backward) its consumers apply, its
// block record, its row descriptor -- that one producer thread (warp 1,
// item table prefetched one item ahead) copies with cp.async.bulk into a
// 128 KB shared ring (6 item slots with an mbarrier each), as far ahead as the
// ring allows and across pass and subdomain boundaries.  Warp 0 solves the
// step's block from the record; 8 consumer warps apply the staged item from
// shared memory; one named barrier per step (the producer is not part of it).
// Measured: 2.43 ms per headline apply, DRAM traffic = algorithmic bytes; a
// step (~1.8 k cycles) is bound by its instruction issue, not the stream
// (K2-K4).
namespace tmas {
constexpr int RB = 8;                   // block rows (records built for it; ShapeRec8 is the fallback)
constexpr int NB = 6;                   // item slots
constexpr int RING = 128 * 1024;        // staging ring, bytes (power of two)
constexpr int kMask = RING / 8 - 1;     // ring index mask, doubles
constexpr int kConsumers = RB;          // consumer warps 2 .. RB + 1 (one per block row)
constexpr int kThreads = 32 * (2 + kConsumers);
constexpr int kStep = kThreads - 32;    // warp 0 + consumers: named barrier 1
constexpr int TS = rec_stride(RB);
constexpr int kRec = rec_size(RB);      // doubles per record
constexpr int kDesc = 16;               // ints per descriptor (64 B): f and offset per row
static_assert(2 * RB <= kDesc, "descriptor holds RB f values and RB offsets");
struct Item {
    const double* data;  // far rows / columns of the step's data block (contiguous)
    long long bytes;     // 0 when the step applies nothing
    const double* rec;   // the solved block's record
    const int* desc;     // [0, RB): f of the data block's rows / columns (INT_MAX past n);
                         // [RB, 2 RB): their offsets in the item (doubles)
};
static_assert(sizeof(Item) == 32, "items are 32 bytes");
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void bulk_copy(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
/** bulk_copy with an L2 eviction-priority policy (createpolicy): the factor
 *  stream of a preconditioner apply (10.5 GB at the headline) is read once, so
 *  it is marked evict_first and does not push the operator tables, the
 *  Krylov basis and the vectors out of L2. */
__device__ __forceinline__ void bulk_copy_hint(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                               unsigned long long policy) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy) : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void step_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kStep) : "memory"); }
}  // namespace tmas

template <int MODE>
__global__ void __launch_bounds__(tmas::kThreads, 1) k_solve_tma(const int* __restrict__ cta_begin,
                                                                 const int* __restrict__ cta_subs,
                                                                 const int* __restrict__ n_rows,
                                                                 const std::int64_t* __restrict__ vbase,
                                                                 const std::int64_t* __restrict__ itbase,
                                                                 const tmas::Item* __restrict__ items,
                                                                 const int* __restrict__ gidx_all,
                                                                 const int* __restrict__ sidx_all,
                                                                 const double* __restrict__ r, double* z,
                                                                 int accumulate, int dbg) {
    constexpr int RB = tmas::RB, NB = tmas::NB, RING = tmas::RING, kMask = tmas::kMask;
    constexpr int kConsumers = tmas::kConsumers, kStep = tmas::kStep, TS = tmas::TS, kRec = tmas::kRec,
                  kDesc = tmas::kDesc;
    using tmas::Item;
    using tmas::smem_u32;
    using tmas::mbar_wait;
    using tmas::bulk_copy;
    using tmas::step_bar;
    extern __shared__ __align__(128) unsigned char smem[];
    double* ring = reinterpret_cast<double*>(smem);
    double* recs = reinterpret_cast<double*>(smem + RING);       // [NB][RB][TS]
    int* descs = reinterpret_cast<int*>(recs + NB * kRec);        // [NB][kDesc]
    double* y = reinterpret_cast<double*>(descs + NB * kDesc);    // [max_rows]
    __shared__ __align__(8) unsigned long long mbar[NB];
    __shared__ long long prod_start[NB];
    __shared__ int item_pos[NB];
    __shared__ volatile int done;  // steps completed (written by thread 0 after the step barrier)
    __shared__ double red[2][tmas::kConsumers][tmas::RB];  // forward partial dots per consumer warp
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int s0 = cta_begin[blockIdx.x], s1 = cta_begin[blockIdx.x + 1];
    constexpr bool kFwd = MODE != 2, kBwd = MODE != 1;
    if (tid == 0) {
        for (int q = 0; q < NB; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        done = 0;
    }
    __syncthreads();

    if (warp == 1) {
        // ---------------- producer (one thread): items of every step, in step order;
        // the next item's 32-byte descriptor is loaded one item ahead
        if (lane != 0) return;
        unsigned long long head = 0;
        int t = 0;
        auto item_at = [&](int si, int pass, int q) -> const Item* {
            const int j = cta_subs[si];
            const int nblk = (n_rows[j] + RB - 1) / RB;
            return items + itbase[j] + static_cast<std::int64_t>(pass) * nblk + q;
        };
        // step order: subdomains, then (enabled) passes, then blocks
        int si = s0, pass = kFwd ? 0 : 1, q = 0;
        int nblk = si < s1 ? (n_rows[cta_subs[si]] + RB - 1) / RB : 0;
        auto advance = [&]() {
            if (++q < nblk) return;
            q = 0;
            if (pass == 0 && kBwd) {
                pass = 1;
                return;
            }
            pass = kFwd ? 0 : 1;
            if (++si < s1) nblk = (n_rows[cta_subs[si]] + RB - 1) / RB;
        };
        Item cur{};
        if (si < s1) cur = *item_at(si, pass, q);
        while (si < s1) {
            advance();
            Item nxt{};
            if (si < s1) nxt = *item_at(si, pass, q);  // in flight while this item is issued
            const long long bytes = cur.bytes;
            const bool ptr = (dbg & 16) && blockIdx.x == (dbg >> 16) && t < 1024;
            if (ptr) g_trace[t][6] = clock64();
            const int slot = t % NB;
            // spins back off: a tight loop of shared loads slows the consumers' traffic
            while (done < t - NB + 1) __nanosleep(64);  // slot's previous item consumed
            if (ptr) g_trace[t][7] = clock64();
            for (;;) {                                  // ring space
                const int d = done;
                const unsigned long long freed = d >= t ? head : prod_start[d % NB];
                if (head + ((bytes + 127) & ~127LL) - freed <= static_cast<unsigned long long>(RING)) break;
                __nanosleep(64);
            }
            if (ptr) g_trace[t][8] = clock64();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            prod_start[slot] = static_cast<long long>(head);
            const unsigned off = static_cast<unsigned>(head & (RING - 1));
            item_pos[slot] = static_cast<int>(off / 8);
            const unsigned bar = smem_u32(&mbar[slot]);
            const bool small = !(dbg & 2);  // dbg & 2: data only (timing experiment)
            const unsigned tx = static_cast<unsigned>(bytes) + (small ? 8u * kRec + 4u * kDesc : 0u);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
            if (bytes > 0) {
                const unsigned first = static_cast<unsigned>(min(bytes, static_cast<long long>(RING - off)));
                bulk_copy(smem_u32(smem + off), cur.data, first, bar);
                if (first < bytes)
                    bulk_copy(smem_u32(smem), reinterpret_cast<const char*>(cur.data) + first,
                              static_cast<unsigned>(bytes) - first, bar);
            }
            if (small) {
                bulk_copy(smem_u32(recs + slot * kRec), cur.rec, 8u * kRec, bar);
                bulk_copy(smem_u32(descs + slot * kDesc), cur.desc, 4u * kDesc, bar);
            }
            head += static_cast<unsigned long long>((bytes + 127) & ~127LL);
            if (ptr) {
                g_trace[t][5] = clock64();
                g_trace[t][9] = bytes;
            }
            cur = nxt;
            ++t;
        }
        return;
    }

    // ---------------- warp 0 (block solves) + consumer warps
    const bool ctr = (dbg & 32) && tid == 0 && blockIdx.x < 1024;
    if (ctr) {
        long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        g_trace[blockIdx.x][0] = t0;
        g_trace[blockIdx.x][2] = s1 - s0;
    }
    const int stid = warp == 0 ? lane : tid - 32;  // 0 .. kStep-1
    const int cw = warp - 2;                       // consumer warp 0 .. 13
    const int ct = tid - 64;                       // consumer thread 0 .. 447
    int t = 0;
    const double2* ring2 = reinterpret_cast<const double2*>(ring);
    for (int si = s0; si < s1; ++si) {
        const int j = cta_subs[si];
        const int n = n_rows[j];
        const std::int64_t vb = vbase[j];
        const int nblk = (n + RB - 1) / RB;
        for (int p = stid; p < n; p += kStep) {
            if (MODE == 3) {
                y[p] = r[vb + p];
            } else {
                const int g = __ldg(gidx_all + vb + p);
                y[p] = g >= 0 ? __ldg(r + g) : 0.0;
            }
        }
        step_bar();
        if constexpr (kFwd) {
            for (int k = 0; k < nblk; ++k, ++t) {
                const int slot = t % NB;
                const bool tr = (dbg & 16) && blockIdx.x == (dbg >> 16) && t < 1024;
                if (tr && stid == 0) g_trace[t][0] = clock64();
                mbar_wait(smem_u32(&mbar[slot]), static_cast<unsigned>((t / NB) & 1));
                if (tr && stid == 0) g_trace[t][1] = clock64();
                const double* R = recs + slot * kRec;
                const int r0 = k * RB;
                if (dbg & 1) {
                    // timing experiment: stream only (no solve work)
                } else if (warp == 0) {
                    if (tr && lane == 0) g_trace[t][10] = clock64();
                    const int i = r0 + lane;
                    const bool live = lane < RB && i < n;
                    double pk = 0.0;
                    if (k > 0 && lane < RB) {
#pragma unroll
                        for (int w = 0; w < kConsumers; ++w) pk += red[k & 1][w][lane];
                    }
                    const double tv = live ? y[i] - pk : 0.0;
                    const double* trow = R + (lane < RB ? lane : 0) * TS;
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int c = 0; c < RB; c += 2) {
                        a2 = fma(trow[RB + c], __shfl_sync(0xffffffffu, tv, c), a2);
                        a3 = fma(trow[RB + c + 1], __shfl_sync(0xffffffffu, tv, c + 1), a3);
                    }
                    if (tr && lane == 0) g_trace[t][11] = clock64();
                    if (r0 >= RB) {
#pragma unroll
                        for (int c = 0; c < RB; c += 2) {
                            a0 = fma(trow[c], y[r0 - RB + c], a0);
                            a1 = fma(trow[c + 1], y[r0 - RB + c + 1], a1);
                        }
                    }
                    if (live) y[i] = (a2 + a3) - (a0 + a1);
                } else if (k + 1 < nblk) {
                    // partial dots of block k+1's rows over columns [f_r, k RB) of the
                    // staged far rows: thread per column pair, y read once for all
                    // RB rows, per-warp sums by a multi-value butterfly into red[]
                    // (summed by warp 0 next step in warp order: deterministic)
                    const int* D = descs + slot * kDesc;
                    const int lim = r0;
                    int fr[RB], orr[RB];
                    int fmin = lim;
                    const int ipos = item_pos[slot];
                    static_assert(RB % 4 == 0, "descriptor read as int4");
#pragma unroll
                    for (int q = 0; q < RB; q += 4) {  // 16-byte descriptor reads
                        const int4 f4 = *reinterpret_cast<const int4*>(D + q);
                        const int4 o4 = *reinterpret_cast<const int4*>(D + RB + q);
                        fr[q] = f4.x, fr[q + 1] = f4.y, fr[q + 2] = f4.z, fr[q + 3] = f4.w;
                        orr[q] = ipos + o4.x - f4.x, orr[q + 1] = ipos + o4.y - f4.y;
                        orr[q + 2] = ipos + o4.z - f4.z, orr[q + 3] = ipos + o4.w - f4.w;
                    }
#pragma unroll
                    for (int q = 0; q < RB; ++q) fmin = min(fmin, fr[q]);
                    double acc[RB];
#pragma unroll
                    for (int q = 0; q < RB; ++q) acc[q] = 0.0;
                    const double2* y2 = reinterpret_cast<const double2*>(y);
                    for (int c = (fmin & ~1) + 2 * ct; c < lim; c += 2 * 32 * kConsumers) {
                        const double2 yy = y2[c >> 1];
#pragma unroll
                        for (int q = 0; q < RB; ++q) {
                            if (c >= fr[q]) {
                                const double2 v = ring2[((orr[q] + c) & kMask) >> 1];
                                acc[q] = fma(v.x, yy.x, acc[q]);
                                acc[q] = fma(v.y, yy.y, acc[q]);
                            }
                        }
                    }
                    static_assert(RB == 8, "the butterfly below reduces eight rows");
                    // 8 values over 32 lanes: xor 16 / 8 / 4 halve the set, xor 2 / 1 finish
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool hi = lane & 16;
                        const double send = hi ? acc[q] : acc[q + 4];
                        const double keep = hi ? acc[q + 4] : acc[q];
                        acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const bool hi = lane & 8;
                        const double send = hi ? acc[q] : acc[q + 2];
                        const double keep = hi ? acc[q + 2] : acc[q];
                        acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    {
                        const bool hi = lane & 4;
                        const double send = hi ? acc[0] : acc[1];
                        const double keep = hi ? acc[1] : acc[0];
                        acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                    }
                    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
                    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
                    if ((lane & 3) == 0) {
                        const int row = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                        red[(k + 1) & 1][cw][row] = acc[0];
                    }
                }
                if (tr && lane == 0 && warp == 0) g_trace[t][2] = clock64();
                if (tr && lane == 0 && warp == 2) g_trace[t][3] = clock64();
                step_bar();
                if (tr && stid == 0) g_trace[t][4] = clock64();
                if (stid == 0) done = t + 1;
            }
        }
        if constexpr (kBwd) {
            for (int K = nblk - 1; K >= 0; --K, ++t) {
                const int slot = t % NB;
                const bool tr = (dbg & 16) && blockIdx.x == (dbg >> 16) && t < 1024;
                if (tr && stid == 0) g_trace[t][0] = clock64();
                mbar_wait(smem_u32(&mbar[slot]), static_cast<unsigned>((t / NB) & 1));
                if (tr && stid == 0) g_trace[t][1] = clock64();
                const double* R = recs + slot * kRec;
                const int r0 = K * RB;
                if (dbg & 1) {
                    // timing experiment: stream only (no solve work)
                } else if (warp == 0) {
                    const int i = r0 + lane;
                    const bool live = lane < RB && i < n;
                    const double tv = live ? y[i] : 0.0;
                    const double* trow = R + (lane < RB ? lane : 0) * TS;
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int c = 0; c < RB; c += 2) {
                        a2 = fma(trow[RB + c], __shfl_sync(0xffffffffu, tv, c), a2);
                        a3 = fma(trow[RB + c + 1], __shfl_sync(0xffffffffu, tv, c + 1), a3);
                    }
                    if (K + 1 < nblk) {
                        const int nb = min(RB, n - (r0 + RB));
                        for (int c = 0; c < nb; ++c) {
                            if (c & 1)
                                a1 = fma(trow[c], y[r0 + RB + c], a1);
                            else
                                a0 = fma(trow[c], y[r0 + RB + c], a0);
                        }
                    }
                    if (live) y[i] = (a2 + a3) - (a0 + a1);
                } else if (K + 1 < nblk) {
                    // block K+1's far columns onto rows [jmin, K RB): thread per row pair
                    const int* D = descs + slot * kDesc;
                    const int c0 = r0 + RB;
                    int fc[RB], oc[RB];
                    double xc[RB];
                    int jmin = r0;
#pragma unroll
                    for (int c = 0; c < RB; c += 4) {  // 16-byte descriptor reads
                        const int4 f4 = *reinterpret_cast<const int4*>(D + c);
                        const int4 o4 = *reinterpret_cast<const int4*>(D + RB + c);
                        fc[c] = f4.x, fc[c + 1] = f4.y, fc[c + 2] = f4.z, fc[c + 3] = f4.w;
                        oc[c] = o4.x - f4.x, oc[c + 1] = o4.y - f4.y, oc[c + 2] = o4.z - f4.z, oc[c + 3] = o4.w - f4.w;
                    }
#pragma unroll
                    for (int c = 0; c < RB; ++c) jmin = fc[c] < r0 ? min(jmin, fc[c]) : jmin;
                    if (c0 + RB <= n) {  // x of block K+1 (16-byte aligned: c0 is a multiple of RB)
#pragma unroll
                        for (int c = 0; c < RB; c += 2) {
                            const double2 x2 = *reinterpret_cast<const double2*>(y + c0 + c);
                            xc[c] = x2.x, xc[c + 1] = x2.y;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < RB; ++c) xc[c] = c0 + c < n ? y[c0 + c] : 0.0;
                    }
                    const int base = item_pos[slot];
                    for (int row = (jmin & ~1) + 2 * ct; row < r0; row += 2 * 32 * kConsumers) {
                        double q0 = 0.0, q1 = 0.0;
#pragma unroll
                        for (int c = 0; c < RB; ++c) {
                            if (row >= fc[c]) {
                                const double2 v = ring2[((base + oc[c] + row) & kMask) >> 1];
                                q0 = fma(v.x, xc[c], q0);
                                q1 = fma(v.y, xc[c], q1);
                            }
                        }
                        y[row] -= q0;
                        y[row + 1] -= q1;
                    }
                }
                if (tr && lane == 0 && warp == 0) g_trace[t][2] = clock64();
                if (tr && lane == 0 && warp == 2) g_trace[t][3] = clock64();
                step_bar();
                if (tr && stid == 0) g_trace[t][4] = clock64();
                if (stid == 0) done = t + 1;
            }
        }
        for (int p = stid; p < n; p += kStep) {
            if (MODE == 3) {
                z[vb + p] = y[p];
            } else {
                const int sx = __ldg(sidx_all + vb + p);
                if (sx >= 0) z[sx] = accumulate ? z[sx] + y[p] : y[p];
            }
        }
        step_bar();
    }
    if (ctr) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        g_trace[blockIdx.x][1] = t1;
    }
}

// ---------------------------------------------- persistent windowed streamed solve
//
// k_solve_win is the default preconditioner apply.  Like k_solve_tma it is
// persistent (one CTA per SM over LPT-balanced subdomain lists) and streams
// every step's item -- descriptor, block record and the far rows (forward) or
// far columns (backward) of one block -- with cp.async.bulk into a shared
// ring, one producer thread running ahead of the solve.  What changes:
//
//  * the local vector y lives in a circular WINDOW of W = 2^m entries in
//    shared memory instead of whole: row i sits in slot i & (W - 1).  W covers
//    the longest envelope row / column (+ a few blocks), 16 KB at the
//    headline against up to 54 KB for the whole vector, so the ring grows to
//    ~200 KB and the block is RB = 16 rows (half the sequential steps of
//    RB = 8 for the same bytes).  Subdomain size is no longer bounded by
//    shared memory: rows enter and leave the window as the solve moves.
//  * R_j r and the results travel through a per-row buffer ybuf (factor
//    order, concatenated over subdomains): a gather kernel fills it, the
//    forward pass overwrites it with L^-1 b, the backward pass with the
//    solution, and a scatter kernel applies Rt_j^T.  Rows enter the window
//    from ybuf through "helper" lanes of warp 0 (lanes RB .. 2RB-1, idle
//    during the block solve) whose loads are issued two steps before the
//    value is stored, so no step waits on a global load: forward step k
//    stores block k+1's right-hand side; backward step K stores the forward
//    result of block K - D, D blocks below the lowest row any later column
//    update touches (D RB > longest U column).
//  * items are placed contiguously in the ring (no wrap inside an item), so
//    the consumers index it without masking; an item larger than the ring
//    is read by the consumers straight from HBM (header still staged).
//
// Step structure per block (unchanged from k_solve_tma): warp 0 forms
// x_k = T_kk^-1 s_k - W_k x_{k-1} from the record; the 8 consumer warps
// apply the staged far part of the NEXT block (forward: partial dots of its
// rows, thread per column pair, fixed butterfly; backward: its columns onto
// every row above, thread per row pair); one named barrier per step.
// GY = true keeps y in ybuf itself (global memory, no window): the fallback
// for windows that do not fit shared memory.
//
// Work units are SEGMENTS: a range [t0, t1) of the 2 nblk steps of one
// subdomain (t < nblk: forward step k = t; else backward step
// K = 2 nblk - 1 - t; the item of step t is items[itbase[j] + t]).  The
// default table balances the SMs exactly by McNaughton's wrap-around rule
// (setup_win): a subdomain may be cut once, its first part at the head of one
// CTA's list and its second part at the tail of the previous CTA's, with the
// state handed over through global memory -- ybuf holds every solved row; a
// cut inside the forward pass adds the partial dots of the next block
// (red[][]), a cut inside the backward pass the window itself (pending column
// updates) -- behind a release / acquire flag that the receiver clears.  The
// handed-over values are the ones the unsplit kernel would hold, so results
// are bitwise independent of the cuts.
namespace win {
struct Seg {
    int j, t0, t1;  // subdomain, step range
    int hand;       // hand-over slot (flag + scratch) of the subdomain's cut, -1: none
};
static_assert(sizeof(Seg) == 16, "segments are 16 bytes");
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr int kConsumers = 8;                     // consumer warps 1 .. 8
constexpr int kThreads = 32 * (kConsumers + 2);   // + warp 0 (solve, helpers) + producer warp
constexpr int kStep = kThreads - 32;              // warps 0 .. 8: named barrier 1
constexpr int NS = 8;                             // item slots (one mbarrier each)
constexpr int kMaxSmem = 227 * 1024;
struct Item {
    const double* data;  // far rows / columns of the step's data block (contiguous)
    long long bytes;     // 0 when the step applies nothing
    const double* rec;   // the solved block's record
    const int* desc;     // [0, RB): f of the data block's rows / columns (INT_MAX past n);
                         // [RB, 2 RB): their offsets in the item's data (doubles)
};
static_assert(sizeof(Item) == 32, "items are 32 bytes");
template <int RB>
struct Geo {
    static constexpr int TS = rec_stride(RB), kRec = rec_size(RB), kDesc = 2 * RB;
    static constexpr int kHdr = 4 * kDesc + 8 * kRec;  // staged header: descriptor, record
    static_assert(kHdr % 128 == 0, "item data starts 128-byte aligned");
};
__device__ __forceinline__ void step_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kStep) : "memory"); }
__device__ __forceinline__ double2 lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2(unsigned a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
}  // namespace win

template <int RB, bool GY>
__global__ void __launch_bounds__(win::kThreads, 1) k_solve_win(const int* __restrict__ cta_begin,
                                                                const win::Seg* __restrict__ segs,
                                                                const int* __restrict__ n_rows,
                                                                const std::int64_t* __restrict__ vbase,
                                                                const std::int64_t* __restrict__ itbase,
                                                                const win::Item* __restrict__ items,
                                                                double* ybuf, int wmask, int dback, int ring_bytes,
                                                                int mode, int* hand_flag, double* hand_buf,
                                                                int hand_stride, int dbg) {
    using G = win::Geo<RB>;
    constexpr int TS = G::TS, kDesc = G::kDesc, kHdr = G::kHdr, NS = win::NS, kC = win::kConsumers;
    using tmas::smem_u32;
    using tmas::mbar_wait;
    using tmas::bulk_copy;
    using tmas::bulk_copy_hint;
    using win::step_bar;
    using win::lds2;
    using win::sts2;
    static_assert(RB == 8 || RB == 16, "butterfly below reduces 8 or 16 rows");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    __shared__ __align__(8) unsigned long long mbar[NS];
    __shared__ unsigned long long prod_start[NS];
    __shared__ int item_pos[NS];
    __shared__ const double* item_g[NS];
    __shared__ volatile int done;  // steps completed (thread 0, after the step barrier)
    __shared__ double red[2][kC][RB];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int s0 = cta_begin[blockIdx.x], s1 = cta_begin[blockIdx.x + 1];
    // mode 1 / 2 (timing experiments): the forward / backward steps only, no hand-overs
    auto clip = [&](const win::Seg& g, int nblk, int& a, int& b) {
        a = mode == 2 ? max(g.t0, nblk) : g.t0;
        b = mode == 1 ? min(g.t1, nblk) : g.t1;
    };
    if (tid == 0) {
        for (int q = 0; q < NS; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        done = 0;
    }
    __syncthreads();

    if (warp == kC + 1) {
        // ---------------- producer (one thread): every step's item in step order
        if (lane != 0) return;
        const unsigned long long pol = tmas::policy_evict_first();
        const unsigned long long RING = static_cast<unsigned long long>(ring_bytes);
        unsigned long long head = 0;  // virtual ring position (bytes)
        int t = 0;
        int si = s0, q = 0, qe = 0;  // segment, its current and end step
        const win::Item* ibase = nullptr;
        auto open_seg = [&]() {  // first non-empty segment at or after si
            for (; si < s1; ++si) {
                const win::Seg g = segs[si];
                clip(g, (n_rows[g.j] + RB - 1) / RB, q, qe);
                if (q < qe) {
                    ibase = items + itbase[g.j];
                    return;
                }
            }
        };
        auto advance = [&]() {
            if (++q < qe) return;
            ++si;
            open_seg();
        };
        open_seg();
        win::Item cur{};
        if (si < s1) cur = ibase[q];
        while (si < s1) {
            advance();
            win::Item nxt{};
            if (si < s1) nxt = ibase[q];  // in flight while this item is issued
            const int slot = t % NS;
            const bool big = kHdr + cur.bytes > ring_bytes;  // data read from HBM by the consumers
            const unsigned long long need = (kHdr + (big ? 0 : cur.bytes) + 127) & ~127ULL;
            unsigned long long start = head;
            if (start % RING + need > RING) start += RING - start % RING;  // items never wrap
            while (done < t - NS + 1) __nanosleep(64);                       // slot's previous item consumed
            for (;;) {                                                       // ring space
                const int d = done;
                const unsigned long long freed = d >= t ? start : prod_start[d % NS];
                if (start + need - freed <= RING) break;
                __nanosleep(64);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            prod_start[slot] = start;
            const unsigned off = static_cast<unsigned>(start % RING);
            item_pos[slot] = static_cast<int>(off);
            item_g[slot] = big ? cur.data : nullptr;
            const unsigned bar = smem_u32(&mbar[slot]);
            const unsigned tx = static_cast<unsigned>(kHdr + (big ? 0 : cur.bytes));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
            bulk_copy_hint(smem_u32(ring + off), cur.desc, 4u * kDesc, bar, pol);
            bulk_copy_hint(smem_u32(ring + off + 4 * kDesc), cur.rec, 8u * G::kRec, bar, pol);
            if (!big && cur.bytes > 0)
                bulk_copy_hint(smem_u32(ring + off + kHdr), cur.data, static_cast<unsigned>(cur.bytes), bar, pol);
            head = start + need;
            cur = nxt;
            ++t;
        }
        return;
    }

    // ---------------- warp 0 (block solves + helper lanes) and consumer warps 1 .. kC
#if __CUDA_ARCH__ >= 900
    // launched as a programmatic dependent of k_win_gather: the producer above reads only the
    // factors and the setup tables; everything below touches ybuf / the hand-over state
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    double* ywin = reinterpret_cast<double*>(smem + ring_bytes);
    const unsigned ywin_u = smem_u32(ywin);
    const unsigned ring_u = smem_u32(ring);
    const int cw = warp - 1;   // consumer warp 0 .. kC-1
    const int ct = tid - 32;   // consumer thread 0 .. 32 kC - 1
    const bool helper = warp == 0 && lane >= RB && lane < 2 * RB;
    const int h = lane - RB;   // helper row within a block
    const int li = lane & (RB - 1);  // warp 0: the block row this lane solves (lanes >= RB mirror, unused)
    int t = 0;
    double hv0 = 0.0, hv1 = 0.0;  // helper registers: hv[b & 1] holds block b's entering value
    for (int si = s0; si < s1; ++si) {
        const win::Seg sg = segs[si];
        const int j = sg.j;
        const int n = n_rows[j];
        const int nblk = (n + RB - 1) / RB;
        int t0, t1;
        clip(sg, nblk, t0, t1);
        if (t0 >= t1) continue;
        const bool handover = mode == 0 && sg.hand >= 0;
        const bool resume = handover && sg.t0 > 0;          // another CTA ran steps [0, t0)
        const bool publish = handover && sg.t1 < 2 * nblk;  // another CTA runs steps [t1, 2 nblk)
        int* hflag = hand_flag + (handover ? sg.hand : 0);
        double* hbuf = hand_buf + static_cast<std::int64_t>(handover ? sg.hand : 0) * hand_stride;
        double* yb = ybuf + vbase[j];
        double* y = GY ? yb : ywin;
        const int wm = GY ? -1 : wmask;
        // y of a row (rows past n read 0: the window holds zeros there, ybuf the next subdomain)
        auto yv = [&](int row) -> double { return GY && row >= n ? 0.0 : y[row & wm]; };
        // y of the row pair (row, row + 1), row even
        auto y2 = [&](int row) -> double2 {
            if constexpr (GY)
                return make_double2(y[row], y[row + 1]);
            else
                return lds2(ywin_u + 8u * static_cast<unsigned>(row & wm));
        };
        // ybuf is read past L1 (rows next to another CTA's subdomain share its lines)
        auto ldblk = [&](int b) -> double {  // row b RB + h of ybuf (0 past the ends)
            const int row = b * RB + h;
            return b >= 0 && row < n ? __ldcg(yb + row) : 0.0;
        };
        if (resume) {
            // the first part's rows, partial dots / window are published before its flag
            if (tid == 0) {
                while (win::ld_acquire(hflag) == 0) __nanosleep(100);
                *hflag = 0;  // one waiter per cut: ready for the next apply
                __threadfence();
            }
            step_bar();
        }
        if (t0 < nblk) {
            const int k1 = min(t1, nblk);
            if (t0 == 0) {
                if (!GY && helper) {
                    ywin[h & wm] = ldblk(0);
                    hv1 = ldblk(1);
                    hv0 = ldblk(2);
                }
                if (warp == 0) __syncwarp();
            } else {
                // resume at forward step t0: the window's rows below block t0 + 1 (solved rows,
                // block t0's right-hand side), the next two entering blocks, block t0's partial dots
                if (!GY) {
                    const int hi = (t0 + 1) * RB;
                    for (int row = max(0, hi - (wm + 1)) + (warp == 0 ? lane : 32 + ct); row < hi; row += win::kStep)
                        ywin[row & wm] = row < n ? __ldcg(yb + row) : 0.0;
                    if (helper) {
                        if (t0 & 1) {
                            hv0 = ldblk(t0 + 1);
                            hv1 = ldblk(t0 + 2);
                        } else {
                            hv1 = ldblk(t0 + 1);
                            hv0 = ldblk(t0 + 2);
                        }
                    }
                }
                for (int e = (warp == 0 ? lane : 32 + ct); e < kC * RB; e += win::kStep)
                    (&red[t0 & 1][0][0])[e] = __ldcg(hbuf + e);
                step_bar();
            }
            for (int k = t0; k < k1; ++k, ++t) {
                const int slot = t % NS;
                mbar_wait(smem_u32(&mbar[slot]), static_cast<unsigned>((t / NS) & 1));
                const int hoff = item_pos[slot];
                const int r0 = k * RB;
                if (dbg & 1) {
                    // timing experiment: stream only
                } else if (warp == 0) {
                    // x_k = T_kk^-1 (y_k - partial dots) - W_k x_{k-1}
                    const double* R = reinterpret_cast<const double*>(ring + hoff + 4 * kDesc) + li * TS;
                    const int i = r0 + li;
                    double pk = 0.0;
                    if (k > 0) {
#pragma unroll
                        for (int w = 0; w < kC; ++w) pk += red[k & 1][w][li];
                    }
                    const double tv = yv(i) - pk;
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int c = 0; c < RB; c += 2) {
                        a2 = fma(R[RB + c], __shfl_sync(0xffffffffu, tv, c), a2);
                        a3 = fma(R[RB + c + 1], __shfl_sync(0xffffffffu, tv, c + 1), a3);
                    }
                    if (k > 0) {
#pragma unroll
                        for (int c = 0; c < RB; c += 2) {
                            const double2 xp = y2(r0 - RB + c);
                            a0 = fma(R[c], xp.x, a0);
                            a1 = fma(R[c + 1], xp.y, a1);
                        }
                    }
                    const double x = i < n ? (a2 + a3) - (a0 + a1) : 0.0;
                    if (lane < RB) {
                        if (!GY || i < n) y[i & wm] = x;
                        if (!GY && i < n) yb[i] = x;
                    } else if (!GY && helper) {
                        // block k+1's right-hand side into the window; block k+3's load
                        const int b = k + 1;
                        if (b & 1) {
                            if (b < nblk) ywin[(b * RB + h) & wm] = hv1;
                            hv1 = ldblk(k + 3);
                        } else {
                            if (b < nblk) ywin[(b * RB + h) & wm] = hv0;
                            hv0 = ldblk(k + 3);
                        }
                    }
                } else if (k + 1 < nblk) {
                    // partial dots of block k+1's rows over columns [f_r, k RB) of the staged
                    // far rows: thread per column pair, y read once for all RB rows
                    const int* D = reinterpret_cast<const int*>(ring + hoff);
                    const int lim = r0;
                    int fr[RB], orr[RB];
                    int fmin = lim;
#pragma unroll
                    for (int q = 0; q < RB; q += 4) {
                        const int4 f4 = *reinterpret_cast<const int4*>(D + q);
                        const int4 o4 = *reinterpret_cast<const int4*>(D + RB + q);
                        fr[q] = f4.x, fr[q + 1] = f4.y, fr[q + 2] = f4.z, fr[q + 3] = f4.w;
                        orr[q] = o4.x - f4.x, orr[q + 1] = o4.y - f4.y;
                        orr[q + 2] = o4.z - f4.z, orr[q + 3] = o4.w - f4.w;
                    }
#pragma unroll
                    for (int q = 0; q < RB; ++q) fmin = min(fmin, fr[q]);
                    double acc[RB];
#pragma unroll
                    for (int q = 0; q < RB; ++q) acc[q] = 0.0;
                    auto dots = [&](auto load) {
                        for (int c = (fmin & ~1) + 2 * ct; c < lim; c += 64 * kC) {
                            const double2 yy = y2(c);
#pragma unroll
                            for (int q = 0; q < RB; ++q) {
                                if (c >= fr[q]) {
                                    const double2 v = load(orr[q] + c);
                                    acc[q] = fma(v.x, yy.x, acc[q]);
                                    acc[q] = fma(v.y, yy.y, acc[q]);
                                }
                            }
                        }
                    };
                    if (const double* g = item_g[slot])
                        dots([&](int e) { return ld_stream(reinterpret_cast<const double2*>(g + e)); });
                    else {
                        const unsigned db = ring_u + static_cast<unsigned>(hoff + kHdr);
                        dots([&](int e) { return lds2(db + 8u * static_cast<unsigned>(e)); });
                    }
                    // RB values over 32 lanes: halve the set at xor 16, 8, ... (the lane
                    // bit keeps the upper half), then plain adds; fixed order, so the
                    // result is bitwise reproducible
#pragma unroll
                    for (int s = 0; s < 5; ++s) {
                        const int o = 16 >> s;
                        const int half = RB >> (s + 1);
                        if (half >= 1) {
                            const bool hi = lane & o;
#pragma unroll
                            for (int q = 0; q < half; ++q) {
                                const double send = hi ? acc[q] : acc[q + half];
                                const double keep = hi ? acc[q + half] : acc[q];
                                acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                            }
                        } else {
                            acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
                        }
                    }
                    // row = lane bits 4, 3, ... (most significant first): (lane >> kSel) & (RB - 1)
                    constexpr int kSel = RB == 16 ? 1 : 2;
                    if ((lane & ((1 << kSel) - 1)) == 0) red[(k + 1) & 1][cw][(lane >> kSel) & (RB - 1)] = acc[0];
                }
                step_bar();
                if (tid == 0) done = t + 1;
            }
            if (publish && t1 <= nblk) {
                // cut inside (or at the end of) the forward pass: block t1's partial dots
                if (t1 < nblk)
                    for (int e = (warp == 0 ? lane : 32 + ct); e < kC * RB; e += win::kStep)
                        hbuf[e] = (&red[t1 & 1][0][0])[e];
                step_bar();
                if (tid == 0) {
                    __threadfence();
                    win::st_release(hflag, 1);
                }
            }
        }
        if (t1 > nblk) {
            const int Khi = 2 * nblk - 1 - max(t0, nblk), Klo = 2 * nblk - t1;
            if (!GY) {
                if (t0 <= nblk) {
                    // window: the last D + 2 blocks (the forward results, 0 past n)
                    const int lo = max(0, (nblk - 2 - dback) * RB);
                    for (int row = lo + (warp == 0 ? lane : 32 + ct); row < nblk * RB; row += win::kStep)
                        ywin[row & wm] = row < n ? __ldcg(yb + row) : 0.0;
                } else {
                    // resume inside the backward pass: the first part's window (pending column updates)
                    for (int e = (warp == 0 ? lane : 32 + ct); e <= wm; e += win::kStep) ywin[e] = __ldcg(hbuf + e);
                }
                if (helper) {
                    const int e = Khi - dback;
                    if (e & 1) {
                        hv1 = ldblk(e);
                        hv0 = ldblk(e - 1);
                    } else {
                        hv0 = ldblk(e);
                        hv1 = ldblk(e - 1);
                    }
                }
                step_bar();
            }
            for (int K = Khi; K >= Klo; --K, ++t) {
                const int slot = t % NS;
                mbar_wait(smem_u32(&mbar[slot]), static_cast<unsigned>((t / NS) & 1));
                const int hoff = item_pos[slot];
                const int r0 = K * RB;
                if (dbg & 1) {
                } else if (warp == 0) {
                    // x_K = U_KK^-1 y_K - W_K x_{K+1}
                    const double* R = reinterpret_cast<const double*>(ring + hoff + 4 * kDesc) + li * TS;
                    const int i = r0 + li;
                    const double tv = yv(i);
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int c = 0; c < RB; c += 2) {
                        a2 = fma(R[RB + c], __shfl_sync(0xffffffffu, tv, c), a2);
                        a3 = fma(R[RB + c + 1], __shfl_sync(0xffffffffu, tv, c + 1), a3);
                    }
                    if (K + 1 < nblk) {
#pragma unroll
                        for (int c = 0; c < RB; c += 2) {
                            a0 = fma(R[c], yv(r0 + RB + c), a0);
                            a1 = fma(R[c + 1], yv(r0 + RB + c + 1), a1);
                        }
                    }
                    const double x = i < n ? (a2 + a3) - (a0 + a1) : 0.0;
                    if (lane < RB) {
                        if (!GY || i < n) y[i & wm] = x;
                        if (!GY && i < n) yb[i] = x;
                    } else if (!GY && helper) {
                        const int e = K - dback;  // entering block (forward result)
                        if (e >= 0) {
                            if (e & 1) {
                                ywin[(e * RB + h) & wm] = hv1;
                                hv1 = ldblk(e - 2);
                            } else {
                                ywin[(e * RB + h) & wm] = hv0;
                                hv0 = ldblk(e - 2);
                            }
                        }
                    }
                } else if (K + 1 < nblk) {
                    // block K+1's far columns onto rows [jmin, K RB): thread per row pair
                    const int* D = reinterpret_cast<const int*>(ring + hoff);
                    const int c0 = r0 + RB;
                    int fc[RB], oc[RB];
                    double xc[RB];
                    int jmin = r0;
#pragma unroll
                    for (int c = 0; c < RB; c += 4) {
                        const int4 f4 = *reinterpret_cast<const int4*>(D + c);
                        const int4 o4 = *reinterpret_cast<const int4*>(D + RB + c);
                        fc[c] = f4.x, fc[c + 1] = f4.y, fc[c + 2] = f4.z, fc[c + 3] = f4.w;
                        oc[c] = o4.x - f4.x, oc[c + 1] = o4.y - f4.y, oc[c + 2] = o4.z - f4.z, oc[c + 3] = o4.w - f4.w;
                    }
#pragma unroll
                    for (int c = 0; c < RB; ++c) jmin = fc[c] < r0 ? min(jmin, fc[c]) : jmin;
#pragma unroll
                    for (int c = 0; c < RB; ++c) xc[c] = yv(c0 + c);  // x of block K+1 (0 past n)
                    auto update = [&](auto load) {
                        for (int row = (jmin & ~1) + 2 * ct; row < r0; row += 64 * kC) {
                            double q0 = 0.0, q1 = 0.0;
#pragma unroll
                            for (int c = 0; c < RB; ++c) {
                                if (row >= fc[c]) {
                                    const double2 v = load(oc[c] + row);
                                    q0 = fma(v.x, xc[c], q0);
                                    q1 = fma(v.y, xc[c], q1);
                                }
                            }
                            if constexpr (GY) {
                                y[row] -= q0;
                                y[row + 1] -= q1;
                            } else {
                                const unsigned a = ywin_u + 8u * static_cast<unsigned>(row & wm);
                                double2 yy = lds2(a);
                                yy.x -= q0;
                                yy.y -= q1;
                                sts2(a, yy);
                            }
                        }
                    };
                    if (const double* g = item_g[slot])
                        update([&](int e) { return ld_stream(reinterpret_cast<const double2*>(g + e)); });
                    else {
                        const unsigned db = ring_u + static_cast<unsigned>(hoff + kHdr);
                        update([&](int e) { return lds2(db + 8u * static_cast<unsigned>(e)); });
                    }
                }
                step_bar();
                if (tid == 0) done = t + 1;
            }
            if (publish) {
                // cut inside the backward pass: the window goes with the flag
                if (!GY)
                    for (int e = (warp == 0 ? lane : 32 + ct); e <= wm; e += win::kStep) hbuf[e] = ywin[e];
                step_bar();
                if (tid == 0) {
                    __threadfence();
                    win::st_release(hflag, 1);
                }
            }
        }
    }
}

/** ybuf[p] = r[gidx[p]] (0 for rows outside the overlap: Dirichlet closures). */
__global__ void k_win_gather(std::int64_t rows, const int* __restrict__ gidx, const double* __restrict__ r,
                             double* __restrict__ ybuf) {
#if __CUDA_ARCH__ >= 900
    // k_solve_win may start: its producer streams factor items while this kernel still gathers
    // (everything that reads ybuf waits in griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    for (std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; p < rows;
         p += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int g = gidx[p];
        ybuf[p] = g >= 0 ? __ldg(r + g) : 0.0;
    }
}

/** z[sidx[p]] (+)= ybuf[p] over the owned rows (Rt_j^T; disjoint writes). */
__global__ void k_win_scatter(std::int64_t rows, const int* __restrict__ sidx, const double* __restrict__ ybuf,
                              double* __restrict__ z, int accumulate) {
#if __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of k_solve_win
#endif
    for (std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; p < rows;
         p += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int s = sidx[p];
        if (s >= 0) z[s] = accumulate ? z[s] + ybuf[p] : ybuf[p];
    }
}

// ------------------------------------------------------ small systems: dense inverses
//
// For a handful of small subdomains (BASELINE config 1: 8 systems of ~400
// unknowns) the envelope solve is one CTA per subdomain walking a chain of
// n dependent substitution steps (~60 us), with most of the GPU idle.  The
// local inverses A_j^-1 (n_j^2 entries, formed once at setup from the
// factors, column by column) turn the apply into a batched dense
// matrix-vector product spread over many CTAs: each CTA gathers R_j r into
// shared memory and produces kDenseRows rows of A_j^-1 (R_j r), then the
// restricted scatter.  Rows are in factor order like everything else.

constexpr int kDenseRows = 16;     // rows of one subdomain per CTA (one warp per 2 rows)
constexpr int kDenseThreads = 256;

__global__ void __launch_bounds__(kDenseThreads) k_solve_dense(const int* __restrict__ tile_sub,
                                                               const int* __restrict__ tile_row0,
                                                               const int* __restrict__ n_rows,
                                                               const std::int64_t* __restrict__ vbase,
                                                               const std::int64_t* __restrict__ dbase,
                                                               const double* __restrict__ Ainv,
                                                               const int* __restrict__ gidx_all,
                                                               const int* __restrict__ sidx_all,
                                                               const double* __restrict__ r, double* z,
                                                               int accumulate, int mode3) {
    extern __shared__ double b[];
    const int j = tile_sub[blockIdx.x], row0 = tile_row0[blockIdx.x];
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j];
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        if (mode3) {
            b[p] = r[vb + p];
        } else {
            const int g = __ldg(gidx_all + vb + p);
            b[p] = g >= 0 ? __ldg(r + g) : 0.0;
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* M = Ainv + dbase[j];
    for (int rr = warp; rr < kDenseRows; rr += kDenseThreads / 32) {
        const int i = row0 + rr;
        if (i >= n) break;
        const double* row = M + static_cast<std::int64_t>(i) * n;
        double s0 = 0.0, s1 = 0.0;
        int c = lane;
        for (; c + 32 < n; c += 64) {
            s0 = fma(ld_stream(row + c), b[c], s0);
            s1 = fma(ld_stream(row + c + 32), b[c + 32], s1);
        }
        if (c < n) s0 = fma(ld_stream(row + c), b[c], s0);
        const double v = warp_sum(s0 + s1);
        if (lane == 0) {
            if (mode3) {
                z[vb + i] = v;
            } else {
                const int sg = __ldg(sidx_all + vb + i);
                if (sg >= 0) z[sg] = accumulate ? z[sg] + v : v;
            }
        }
    }
}

/** e_k probe right-hand sides (factor order, per-row arrays): r[vb + k] = 1. */
__global__ void k_unit_rhs(int n_sub, const int* __restrict__ n_rows, const std::int64_t* __restrict__ vbase,
                           int k, double* __restrict__ r) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n_sub && k < n_rows[j]) r[vbase[j] + k] = 1.0;
}
__global__ void k_unit_clear(int n_sub, const int* __restrict__ n_rows, const std::int64_t* __restrict__ vbase,
                             int k, double* __restrict__ r) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n_sub && k < n_rows[j]) r[vbase[j] + k] = 0.0;
}
/** Column k of every A_j^-1 (z, factor order) into the row-major inverses. */
__global__ void __launch_bounds__(256) k_store_column(int k, const int* __restrict__ n_rows,
                                                      const std::int64_t* __restrict__ vbase,
                                                      const std::int64_t* __restrict__ dbase,
                                                      const double* __restrict__ z, double* __restrict__ Ainv) {
    const int j = blockIdx.x;
    const int n = n_rows[j];
    if (k >= n) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        Ainv[dbase[j] + static_cast<std::int64_t>(i) * n + k] = z[vbase[j] + i];
}

template <class T>
void append(std::vector<T>& dst, const std::vector<T>& src) {
    dst.insert(dst.end(), src.begin(), src.end());
}

}  // namespace

template <bool UROWS, class SH, bool INV>
static void launch_solve(const cpddg_pc* pc, int grid, const double* r, double* z, bool accumulate, int mode,
                         int dbg, cudaStream_t st) {
    auto kern = mode == 1 ? k_solve<1, UROWS, SH, INV> : mode == 2 ? k_solve<2, UROWS, SH, INV>
              : mode == 3 ? k_solve<3, UROWS, SH, INV> : k_solve<0, UROWS, SH, INV>;
    kern<<<grid, SH::kThreads, pc->solve_smem, st>>>(
        pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(), pc->first.get(), pc->roff.get(),
        pc->ebaseU.get(), pc->firstU.get(), pc->roffU.get(),
        pc->dinv.get(), pc->L.get(), pc->U.get(), pc->gidx.get(), pc->sidx.get(), r, z, accumulate ? 1 : 0,
        pc->bwd_prefetch, pc->ubase.get(), pc->ufirst.get(), pc->uroff.get(), pc->drev.get(), dbg,
        pc->rbase.get(), pc->recL.get(), pc->recU.get());
    CPDDG_CUDA(cudaGetLastError());
}

/** cudaFuncAttributeMaxDynamicSharedMemorySize is per kernel, not per
 *  preconditioner: raise it to the largest request seen so far, so that a
 *  preconditioner built earlier with larger subdomains still launches after
 *  a smaller one was built. */
static void raise_smem_limit(const void* kern, int bytes) {
    static std::mutex m;
    static std::vector<std::pair<const void*, int>> seen;
    std::lock_guard<std::mutex> lk(m);
    for (auto& [k, b] : seen)
        if (k == kern) {
            if (bytes <= b) return;
            b = bytes;
            CPDDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            return;
        }
    seen.emplace_back(kern, bytes);
    CPDDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <bool UROWS, class SH, bool INV>
static void set_solve_smem(int bytes) {
    for (auto kern : {k_solve<0, UROWS, SH, INV>, k_solve<1, UROWS, SH, INV>, k_solve<2, UROWS, SH, INV>,
                      k_solve<3, UROWS, SH, INV>})
        raise_smem_limit(reinterpret_cast<const void*>(kern), std::max(bytes, 1));
}

void pc_apply_mode(const cpddg_pc* pc, const double* r, double* z, bool accumulate, int mode, cudaStream_t st) {
    static const int dbg_flags = [] {
        const char* e = std::getenv("CPDDG_SOLVE_DEBUG");  // development: timing experiments only
        return e ? std::atoi(e) : 0;
    }();
    static const int limit = [] {
        const char* e = std::getenv("CPDDG_SOLVE_LIMIT");  // development: solve only the first k subdomains
        return e ? std::atoi(e) : 0;
    }();
    const int grid = (limit > 0 && mode != 3) ? std::min(limit, pc->n_sub) : pc->n_sub;
    const int dbg = mode == 3 ? 0 : dbg_flags;
    if (pc->dense && (mode == 0 || (mode == 3 && pc->dense_probe))) {
        k_solve_dense<<<pc->dense_tiles, kDenseThreads, sizeof(double) * pc->max_rows, st>>>(
            pc->dense_tile_sub.get(), pc->dense_tile_row0.get(), pc->n_rows.get(), pc->vbase.get(),
            pc->dense_base.get(), pc->Ainv.get(), pc->gidx.get(), pc->sidx.get(), r, z, accumulate ? 1 : 0,
            mode == 3 ? 1 : 0);
        CPDDG_CUDA(cudaGetLastError());
        return;
    }
    if (pc->win) {
        const int rb = pc->win_rb;
        const std::int64_t rows = pc->rows_total;
        const int gblocks = static_cast<int>(std::min<std::int64_t>((rows + 255) / 256, 8LL * sm_count()));
        double* yb = pc->ybuf.get();
        if (mode == 3) {  // probe / unit solves: r and z are already per-row (factor order)
            CPDDG_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * static_cast<std::size_t>(rows), cudaMemcpyDeviceToDevice, st));
            yb = z;
        } else {
            k_win_gather<<<gblocks, 256, 0, st>>>(rows, pc->gidx.get(), r, yb);
        }
        const int m = mode == 3 ? 0 : mode;
        // balanced (cut) lists for full applies with the shared-memory window
        const bool bal = m == 0 && !pc->win_gy && pc->win_cuts > 0;
        auto pick = [&](auto rbc) {
            constexpr int RB = decltype(rbc)::value;
            return pc->win_gy ? k_solve_win<RB, true> : k_solve_win<RB, false>;
        };
        auto kern = rb == 8 ? pick(std::integral_constant<int, 8>{}) : pick(std::integral_constant<int, 16>{});
        // gather -> solve -> scatter as programmatic dependents (CPDDG_PC_PDL=0: plain stream order)
        const char* pe = std::getenv("CPDDG_PC_PDL");
        const bool pdl = mode != 3 && !(pe && std::string(pe) == "0");
        cudaLaunchAttribute pattr{};
        pattr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pattr.val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(pc->win_grid);
        cfg.blockDim = dim3(win::kThreads);
        cfg.dynamicSmemBytes = static_cast<std::size_t>(pc->win_smem);
        cfg.stream = st;
        cfg.attrs = &pattr;
        cfg.numAttrs = pdl ? 1 : 0;
        CPDDG_CUDA(cudaLaunchKernelEx(
            &cfg, kern, static_cast<const int*>((bal ? pc->win_bal_begin : pc->win_cta_begin).get()),
            reinterpret_cast<const win::Seg*>((bal ? pc->win_bal_segs : pc->win_cta_subs).get()),
            static_cast<const int*>(pc->n_rows.get()), static_cast<const std::int64_t*>(pc->vbase.get()),
            static_cast<const std::int64_t*>(pc->win_itbase.get()),
            reinterpret_cast<const win::Item*>(pc->win_items.get()), yb, pc->win_wmask, pc->win_dback, pc->win_ring, m,
            pc->win_hand_flag.get(), pc->win_hand_buf.get(), pc->win_hand_stride, dbg));
        if (mode != 3) {
            cudaLaunchConfig_t sc = {};
            sc.gridDim = dim3(gblocks);
            sc.blockDim = dim3(256);
            sc.stream = st;
            sc.attrs = &pattr;
            sc.numAttrs = pdl ? 1 : 0;
            CPDDG_CUDA(cudaLaunchKernelEx(&sc, k_win_scatter, rows, static_cast<const int*>(pc->sidx.get()),
                                          static_cast<const double*>(yb), z, accumulate ? 1 : 0));
        }
        return;
    }
    if (pc->tma) {
        auto kern = mode == 1 ? k_solve_tma<1> : mode == 2 ? k_solve_tma<2> : mode == 3 ? k_solve_tma<3> : k_solve_tma<0>;
        kern<<<pc->tma_grid, tmas::kThreads, pc->tma_smem, st>>>(
            pc->tma_cta_begin.get(), pc->tma_cta_subs.get(), pc->n_rows.get(), pc->vbase.get(), pc->tma_itbase.get(),
            reinterpret_cast<const tmas::Item*>(pc->tma_items.get()), pc->gidx.get(), pc->sidx.get(), r, z,
            accumulate ? 1 : 0, dbg);
        CPDDG_CUDA(cudaGetLastError());
        return;
    }
    if (!pc->urows && pc->blockinv) {
        if (pc->shape == 0)
            launch_solve<false, ShapeBig, true>(pc, grid, r, z, accumulate, mode, dbg, st);
        else if (pc->shape == 1)
            launch_solve<false, ShapeMid, true>(pc, grid, r, z, accumulate, mode, dbg, st);
        else if (pc->shape == 4)
            launch_solve<false, ShapeRec8, true>(pc, grid, r, z, accumulate, mode, dbg, st);
        else
            launch_solve<false, ShapeRec, true>(pc, grid, r, z, accumulate, mode, dbg, st);
    } else if (!pc->urows)
        launch_solve<false, ShapeMid, false>(pc, grid, r, z, accumulate, mode, dbg, st);
    else if (pc->blockinv) {
        if (pc->shape == 0)
            launch_solve<true, ShapeBig, true>(pc, grid, r, z, accumulate, mode, dbg, st);
        else if (pc->shape == 1)
            launch_solve<true, ShapeMid, true>(pc, grid, r, z, accumulate, mode, dbg, st);
        else
            launch_solve<true, ShapeRec, true>(pc, grid, r, z, accumulate, mode, dbg, st);
    } else if (pc->shape == 0)
        launch_solve<true, ShapeBig, false>(pc, grid, r, z, accumulate, mode, dbg, st);
    else if (pc->shape == 1)
        launch_solve<true, ShapeMid, false>(pc, grid, r, z, accumulate, mode, dbg, st);
    else
        launch_solve<true, ShapeSmall, false>(pc, grid, r, z, accumulate, mode, dbg, st);
}

void pc_apply(const cpddg_pc* pc, const double* r, double* z, bool accumulate, cudaStream_t st) {
    pc_apply_mode(pc, r, z, accumulate, 0, st);
}

/** Items, descriptors and the per-CTA subdomain lists of k_solve_tma (see
 *  there).  Subdomains go to CTAs (one per SM) longest-processing-time first
 *  by streamed bytes; the path is left off if an item would not fit the ring. */
static void setup_tma(cpddg_pc* pc, const std::vector<int>& n_rows, const std::vector<std::int64_t>& vbase,
                      const std::vector<int>& fL, const std::vector<int>& fU, const std::vector<std::int64_t>& rocL,
                      const std::vector<std::int64_t>& cbL, const std::vector<std::int64_t>& rocU,
                      const std::vector<std::int64_t>& cbU, const std::vector<std::int64_t>& rbase) {
    using tmas::RB;
    const int n_sub = pc->n_sub;
    std::vector<std::int64_t> itbase(static_cast<std::size_t>(n_sub)), cost(static_cast<std::size_t>(n_sub), 0);
    std::int64_t n_items = 0;
    for (int j = 0; j < n_sub; ++j) {
        itbase[static_cast<std::size_t>(j)] = n_items;
        n_items += 2 * ((n_rows[static_cast<std::size_t>(j)] + RB - 1) / RB);
    }
    std::vector<tmas::Item> items(static_cast<std::size_t>(n_items));
    std::vector<int> desc(static_cast<std::size_t>(n_items) * tmas::kDesc, INT_MAX);
    DevBuf<int> ddesc(desc.size());
    const double* Lc = pc->L.get();
    const double* Uc = pc->U.get();
    long long max_bytes = 0;
    for (int j = 0; j < n_sub; ++j) {
        const int n = n_rows[static_cast<std::size_t>(j)];
        const int nblk = (n + RB - 1) / RB;
        const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
        for (int pass = 0; pass < 2; ++pass) {
            const std::vector<int>& f = pass ? fU : fL;
            const std::vector<std::int64_t>& roc = pass ? rocU : rocL;
            const double* V = (pass ? Uc : Lc) + (pass ? cbU : cbL)[static_cast<std::size_t>(j)];
            const double* rec = (pass ? pc->recU.get() : pc->recL.get()) + rbase[static_cast<std::size_t>(j)];
            for (int q = 0; q < nblk; ++q) {
                const int k = pass ? nblk - 1 - q : q;  // the block solved at this step
                const int B = k + 1;                    // the block whose far part the step applies
                const std::int64_t it = itbase[static_cast<std::size_t>(j)] + static_cast<std::int64_t>(pass) * nblk + q;
                tmas::Item& I = items[static_cast<std::size_t>(it)];
                I.rec = rec + static_cast<std::int64_t>(k) * rec_pitch(RB);
                I.desc = ddesc.get() + it * tmas::kDesc;
                I.data = V;
                I.bytes = 0;
                for (int c = 0; c < RB; ++c) desc[static_cast<std::size_t>(it * tmas::kDesc + RB + c)] = 0;
                if (B < nblk) {
                    const int lim = (B - 1) * RB;
                    long long len = 0;
                    for (int c = 0; c < RB && B * RB + c < n; ++c) {
                        const int fc = f[static_cast<std::size_t>(v0 + B * RB + c)];
                        desc[static_cast<std::size_t>(it * tmas::kDesc + c)] = fc;
                        desc[static_cast<std::size_t>(it * tmas::kDesc + RB + c)] = static_cast<int>(len);
                        len += std::max(0, lim - fc);
                    }
                    I.data = V + roc[static_cast<std::size_t>(v0 + B * RB)];
                    I.bytes = 8 * len;
                    max_bytes = std::max(max_bytes, I.bytes);
                }
                // measured step cost (scripts/trace_tma_steps.py): ~1,060 cycles + ~27 cycles per KB
                cost[static_cast<std::size_t>(j)] += 1060 * 1024 + 27 * I.bytes;
            }
        }
    }
    if (std::getenv("CPDDG_VERBOSE")) {
        std::vector<long long> sz;
        for (const auto& I : items) sz.push_back(I.bytes);
        std::sort(sz.begin(), sz.end());
        auto over = [&](long long b) { return static_cast<long long>(sz.end() - std::upper_bound(sz.begin(), sz.end(), b)); };
        std::fprintf(stderr, "[cpddg] tma items %zu: p50 %lld p99 %lld max %lld bytes; over 64K %lld, over 96K %lld, over 128K %lld\n",
                     sz.size(), sz[sz.size() / 2], sz[sz.size() * 99 / 100], sz.back(), over(65536), over(98304),
                     over(131072));
    }
    // an item exceeds the ring: keep the register-staged solve (ShapeRec8 over the same
    // records); CPDDG_TMA_RING_LIMIT (bytes) lowers the limit to exercise that fallback
    long long limit = tmas::RING;
    if (const char* e = std::getenv("CPDDG_TMA_RING_LIMIT")) limit = std::min(limit, std::atoll(e));
    if (max_bytes > limit) return;
    // longest processing time first onto min(#SMs, n_sub) CTAs
    const int grid = std::min(sm_count(), n_sub);
    std::vector<int> by_cost(static_cast<std::size_t>(n_sub));
    std::iota(by_cost.begin(), by_cost.end(), 0);
    std::stable_sort(by_cost.begin(), by_cost.end(),
                     [&](int a, int b) { return cost[static_cast<std::size_t>(a)] > cost[static_cast<std::size_t>(b)]; });
    std::vector<std::int64_t> load(static_cast<std::size_t>(grid), 0);
    std::vector<std::vector<int>> lists(static_cast<std::size_t>(grid));
    for (int j : by_cost) {
        const auto m = std::min_element(load.begin(), load.end()) - load.begin();
        lists[static_cast<std::size_t>(m)].push_back(j);
        load[static_cast<std::size_t>(m)] += cost[static_cast<std::size_t>(j)];
    }
    std::vector<int> begin{0}, subs;
    for (const auto& L : lists) {
        subs.insert(subs.end(), L.begin(), L.end());
        begin.push_back(static_cast<int>(subs.size()));
    }
    CPDDG_CUDA(cudaMemcpy(ddesc.get(), desc.data(), desc.size() * sizeof(int), cudaMemcpyHostToDevice));
    pc->tma_desc = std::move(ddesc);
    pc->tma_items.alloc(items.size() * sizeof(tmas::Item));
    CPDDG_CUDA(cudaMemcpy(pc->tma_items.get(), items.data(), items.size() * sizeof(tmas::Item), cudaMemcpyHostToDevice));
    pc->tma_itbase.upload(itbase);
    pc->tma_cta_begin.upload(begin);
    pc->tma_cta_subs.upload(subs);
    pc->tma_grid = grid;
    pc->tma_smem = tmas::RING + 8 * tmas::NB * tmas::kRec + 4 * tmas::NB * tmas::kDesc + 8 * pc->max_rows;
    for (auto kern : {k_solve_tma<0>, k_solve_tma<1>, k_solve_tma<2>, k_solve_tma<3>})
        raise_smem_limit(reinterpret_cast<const void*>(kern), pc->tma_smem);
    pc->tma = true;
}

/** Window geometry of k_solve_win for blocks of RB rows: W (power of two)
 *  covers the longest far row (forward) and the D-block entering lookahead
 *  below the backward front (D RB > longest U column); the ring takes the
 *  rest of shared memory, or all of it when the window goes to HBM. */
struct WinGeometry {
    int W = 0, dback = 0, ring = 0;
    bool gy = false;
};
static WinGeometry win_geometry(int rb, int reachL, int reachU) {
    WinGeometry g;
    g.dback = (reachU + rb - 1) / rb + 1;
    g.W = 4 * rb;
    while (g.W < reachL + 2 * rb || g.W < (g.dback + 3) * rb) g.W *= 2;
    if (const char* e = std::getenv("CPDDG_WIN_W")) g.W = std::max(g.W, std::atoi(e));  // development: larger windows
    const int kStatic = 4096;  // static shared memory of the kernel (mbarriers, slots, partial dots)
    const int avail = (win::kMaxSmem - kStatic) & ~127;
    g.gy = 8 * g.W > avail - 64 * 1024;  // keep at least a 64 KB ring, else y stays in ybuf
    if (const char* e = std::getenv("CPDDG_WIN_GY")) g.gy = g.gy || std::string(e) == "1";
    g.ring = g.gy ? avail : (avail - 8 * g.W) & ~127;
    if (const char* e = std::getenv("CPDDG_WIN_RING")) g.ring = std::min(g.ring, std::atoi(e) & ~127);
    return g;
}

/** Block size of k_solve_win: RB = 16 halves the sequential steps of RB = 8
 *  (1.89 vs 2.44 ms per headline apply, where the largest RB = 16 item is
 *  170 KB of a 212 KB ring) but doubles the items; when more than 0.5 % of
 *  the RB = 16 items would come near the ring size (long envelope rows:
 *  large subdomains), RB = 8 keeps the stream in the ring instead of reading
 *  those items from HBM (2.7x slower per byte, measured). */
static int win_choose_rb(const std::vector<int>& n_rows, const std::vector<std::int64_t>& vbase,
                         const std::vector<int>& fL, const std::vector<int>& fU) {
    constexpr int RB = 16;
    int reachL = 0, reachU = 0;
    std::int64_t items = 0, large = 0;
    for (std::size_t j = 0; j < n_rows.size(); ++j)
        for (int i = 0; i < n_rows[j]; ++i) {
            reachL = std::max(reachL, i - fL[static_cast<std::size_t>(vbase[j] + i)]);
            reachU = std::max(reachU, i - fU[static_cast<std::size_t>(vbase[j] + i)]);
        }
    const WinGeometry g = win_geometry(RB, reachL, reachU);
    for (std::size_t j = 0; j < n_rows.size(); ++j) {
        const int n = n_rows[j], nblk = (n + RB - 1) / RB;
        for (const auto* f : {&fL, &fU})
            for (int B = 1; B < nblk; ++B) {
                long long len = 0;
                for (int i = B * RB; i < std::min(n, B * RB + RB); ++i)
                    len += std::max(0, (B - 1) * RB - (*f)[static_cast<std::size_t>(vbase[j] + i)]);
                ++items;
                large += win::Geo<RB>::kHdr + 8 * len > g.ring * 85LL / 100 ? 1 : 0;
            }
    }
    return 200 * large > items ? 8 : 16;
}

/** Items, descriptors, per-CTA subdomain lists, window and ring geometry of
 *  k_solve_win (see there) for blocks of RB rows.  Returns false (path left
 *  off) only if not even the global-memory variant fits. */
template <int RB>
static bool setup_win(cpddg_pc* pc, const std::vector<int>& n_rows, const std::vector<std::int64_t>& vbase,
                      const std::vector<int>& fL, const std::vector<int>& fU, const std::vector<std::int64_t>& rocL,
                      const std::vector<std::int64_t>& cbL, const std::vector<std::int64_t>& rocU,
                      const std::vector<std::int64_t>& cbU, const std::vector<std::int64_t>& rbase) {
    using G = win::Geo<RB>;
    constexpr int kDesc = G::kDesc;
    const int n_sub = pc->n_sub;
    // window: the longest far row (forward) and column (backward) plus the
    // blocks in flight; D blocks of entering lookahead below the backward front
    int reachL = 0, reachU = 0;
    for (int j = 0; j < n_sub; ++j)
        for (int i = 0; i < n_rows[static_cast<std::size_t>(j)]; ++i) {
            const std::size_t g = static_cast<std::size_t>(vbase[static_cast<std::size_t>(j)] + i);
            reachL = std::max(reachL, i - fL[g]);
            reachU = std::max(reachU, i - fU[g]);
        }
    const WinGeometry geo = win_geometry(RB, reachL, reachU);
    const int dback = geo.dback, W = geo.W, ring = geo.ring;
    const bool gy = geo.gy;
    if (ring < 2 * G::kHdr) return false;

    std::vector<std::int64_t> itbase(static_cast<std::size_t>(n_sub)), cost(static_cast<std::size_t>(n_sub), 0);
    std::int64_t n_items = 0;
    for (int j = 0; j < n_sub; ++j) {
        itbase[static_cast<std::size_t>(j)] = n_items;
        n_items += 2 * ((n_rows[static_cast<std::size_t>(j)] + RB - 1) / RB);
    }
    std::vector<win::Item> items(static_cast<std::size_t>(n_items));
    std::vector<int> desc(static_cast<std::size_t>(n_items) * kDesc, INT_MAX);
    DevBuf<int> ddesc(desc.size());
    long long n_big = 0, max_bytes = 0;
    // step cost model for the LPT assignment (cycles; CPDDG_WIN_COST="c0,c1" per step and per KB)
    long long c0 = 2000, c1 = 30;
    if (const char* e = std::getenv("CPDDG_WIN_COST")) std::sscanf(e, "%lld,%lld", &c0, &c1);
    for (int j = 0; j < n_sub; ++j) {
        const int n = n_rows[static_cast<std::size_t>(j)];
        const int nblk = (n + RB - 1) / RB;
        const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
        for (int pass = 0; pass < 2; ++pass) {
            const std::vector<int>& f = pass ? fU : fL;
            const std::vector<std::int64_t>& roc = pass ? rocU : rocL;
            const double* V = (pass ? pc->U.get() : pc->L.get()) + (pass ? cbU : cbL)[static_cast<std::size_t>(j)];
            const double* rec = (pass ? pc->recU.get() : pc->recL.get()) + rbase[static_cast<std::size_t>(j)];
            for (int q = 0; q < nblk; ++q) {
                const int k = pass ? nblk - 1 - q : q;  // the block solved at this step
                const int B = k + 1;                    // the block whose far part the step applies
                const std::int64_t it = itbase[static_cast<std::size_t>(j)] + static_cast<std::int64_t>(pass) * nblk + q;
                win::Item& I = items[static_cast<std::size_t>(it)];
                I.rec = rec + static_cast<std::int64_t>(k) * rec_pitch(RB);
                I.desc = ddesc.get() + it * kDesc;
                I.data = V;
                I.bytes = 0;
                for (int c = 0; c < RB; ++c) desc[static_cast<std::size_t>(it * kDesc + RB + c)] = 0;
                if (B < nblk) {
                    const int lim = (B - 1) * RB;
                    long long len = 0;
                    for (int c = 0; c < RB && B * RB + c < n; ++c) {
                        const int fc = f[static_cast<std::size_t>(v0 + B * RB + c)];
                        desc[static_cast<std::size_t>(it * kDesc + c)] = fc;
                        desc[static_cast<std::size_t>(it * kDesc + RB + c)] = static_cast<int>(len);
                        len += std::max(0, lim - fc);
                    }
                    I.data = V + roc[static_cast<std::size_t>(v0 + B * RB)];
                    I.bytes = 8 * len;
                    max_bytes = std::max(max_bytes, I.bytes);
                    n_big += G::kHdr + I.bytes > ring ? 1 : 0;
                }
                cost[static_cast<std::size_t>(j)] += c0 * 1024 + c1 * (G::kHdr + I.bytes);
            }
        }
    }
    if (std::getenv("CPDDG_VERBOSE")) {
        std::vector<long long> sz;
        for (const auto& I : items) sz.push_back(I.bytes);
        std::sort(sz.begin(), sz.end());
        std::fprintf(stderr, "[cpddg] win RB %d: items %zu, p50 %lld p99 %lld max %lld bytes, %lld from HBM (ring %d B); "
                     "window %d rows (%s), reach L %d U %d, lookahead %d blocks\n",
                     RB, sz.size(), sz[sz.size() / 2], sz[sz.size() * 99 / 100], sz.back(), n_big, ring, W,
                     gy ? "global" : "shared", reachL, reachU, dback);
    }
    const int grid = std::min(sm_count(), n_sub);
    std::vector<int> by_cost(static_cast<std::size_t>(n_sub));
    std::iota(by_cost.begin(), by_cost.end(), 0);
    std::stable_sort(by_cost.begin(), by_cost.end(),
                     [&](int a, int b) { return cost[static_cast<std::size_t>(a)] > cost[static_cast<std::size_t>(b)]; });
    std::vector<std::int64_t> load(static_cast<std::size_t>(grid), 0);
    std::vector<std::vector<int>> lists(static_cast<std::size_t>(grid));
    for (int j : by_cost) {
        const auto m = std::min_element(load.begin(), load.end()) - load.begin();
        lists[static_cast<std::size_t>(m)].push_back(j);
        load[static_cast<std::size_t>(m)] += cost[static_cast<std::size_t>(j)];
    }
    // whole-subdomain segments (modes 1 / 2, the global-y variant, CPDDG_WIN_SPLIT=0)
    std::vector<int> begin{0}, segs;
    std::int64_t total = 0, lpt_span = 0, chain = 0;
    for (std::size_t m = 0; m < lists.size(); ++m) {
        for (int j : lists[m]) {
            const int nblk = (n_rows[static_cast<std::size_t>(j)] + RB - 1) / RB;
            segs.insert(segs.end(), {j, 0, 2 * nblk, -1});
        }
        begin.push_back(static_cast<int>(segs.size() / 4));
        lpt_span = std::max(lpt_span, load[m]);
    }
    for (int j = 0; j < n_sub; ++j) {
        total += cost[static_cast<std::size_t>(j)];
        chain = std::max(chain, cost[static_cast<std::size_t>(j)]);
    }
    pc->win_lpt_eff = static_cast<double>(total) / (static_cast<double>(grid) * static_cast<double>(lpt_span));
    // balanced segments: McNaughton's wrap-around rule.  The subdomains lie end
    // to end on a line cut every `quota` (>= the longest chain); a subdomain
    // across a cut runs its FIRST steps at the head of the next CTA's list and
    // its LAST steps at the tail of this CTA's, so the two parts never overlap
    // in time (cost <= quota) and the tail part finds its flag set.
    {
        const std::int64_t quota = std::max((total + grid - 1) / grid, chain);
        std::vector<std::vector<int>> bl(static_cast<std::size_t>(grid));
        std::vector<std::int64_t> bload(static_cast<std::size_t>(grid), 0);
        auto step_cost = [&](int j, int t) {
            return c0 * 1024 + c1 * (G::kHdr + items[static_cast<std::size_t>(itbase[static_cast<std::size_t>(j)] + t)].bytes);
        };
        std::int64_t pos = 0;
        int cuts = 0;
        for (int j : by_cost) {
            const int nsteps = 2 * ((n_rows[static_cast<std::size_t>(j)] + RB - 1) / RB);
            const std::int64_t cj = cost[static_cast<std::size_t>(j)];
            const int m = static_cast<int>(std::min<std::int64_t>(pos / quota, grid - 1));
            const std::int64_t room = static_cast<std::int64_t>(m + 1) * quota - pos;  // left on CTA m
            int x = 0;  // steps [x, nsteps) stay on CTA m, [0, x) go to CTA m + 1
            if (cj > room && m + 1 < grid) {
                std::int64_t tail = 0;
                x = nsteps;
                while (x > 0 && tail + step_cost(j, x - 1) <= room) tail += step_cost(j, --x);
                // nearest step boundary to the cut
                if (x > 0 && room - tail > (tail + step_cost(j, x - 1)) - room) tail += step_cost(j, --x);
                if (x == 0) x = 0;
            }
            if (x == 0) {
                bl[static_cast<std::size_t>(m)].insert(bl[static_cast<std::size_t>(m)].end(), {j, 0, nsteps, -1});
                bload[static_cast<std::size_t>(m)] += cj;
            } else if (x == nsteps) {
                bl[static_cast<std::size_t>(m) + 1].insert(bl[static_cast<std::size_t>(m) + 1].end(), {j, 0, nsteps, -1});
                bload[static_cast<std::size_t>(m) + 1] += cj;
            } else {
                std::int64_t headc = 0;
                for (int t = 0; t < x; ++t) headc += step_cost(j, t);
                bl[static_cast<std::size_t>(m)].insert(bl[static_cast<std::size_t>(m)].end(), {j, x, nsteps, cuts});
                bl[static_cast<std::size_t>(m) + 1].insert(bl[static_cast<std::size_t>(m) + 1].end(), {j, 0, x, cuts});
                bload[static_cast<std::size_t>(m)] += cj - headc;
                bload[static_cast<std::size_t>(m) + 1] += headc;
                ++cuts;
            }
            pos += cj;
        }
        // a CTA's list: the head part (pushed by the previous CTA's last subdomain)
        // first, then whole subdomains, then the tail part
        std::vector<int> bbegin{0}, bsegs;
        for (auto& L : bl) {
            std::vector<int> headp, mid, tailp;
            for (std::size_t e = 0; e < L.size(); e += 4) {
                std::vector<int>& dst = L[e + 3] < 0 ? mid : L[e + 1] == 0 ? headp : tailp;
                dst.insert(dst.end(), L.begin() + static_cast<std::ptrdiff_t>(e), L.begin() + static_cast<std::ptrdiff_t>(e) + 4);
            }
            bsegs.insert(bsegs.end(), headp.begin(), headp.end());
            bsegs.insert(bsegs.end(), mid.begin(), mid.end());
            bsegs.insert(bsegs.end(), tailp.begin(), tailp.end());
            bbegin.push_back(static_cast<int>(bsegs.size() / 4));
        }
        const std::int64_t bal_span = *std::max_element(bload.begin(), bload.end());
        pc->win_bal_eff = static_cast<double>(total) / (static_cast<double>(grid) * static_cast<double>(bal_span));
        pc->win_cuts = cuts;
        if (const char* e = std::getenv("CPDDG_WIN_SPLIT"))  // development: 0 = whole subdomains per CTA (LPT)
            if (std::atoi(e) == 0) pc->win_cuts = 0;
        pc->win_hand_stride = std::max(W, win::kConsumers * RB);
        pc->win_bal_begin.upload(bbegin);
        pc->win_bal_segs.upload(bsegs);
        std::vector<int> zero(static_cast<std::size_t>(std::max(cuts, 1)), 0);
        pc->win_hand_flag.upload(zero);
        pc->win_hand_buf.alloc(static_cast<std::size_t>(std::max(cuts, 1)) * static_cast<std::size_t>(pc->win_hand_stride));
        if (std::getenv("CPDDG_VERBOSE"))
            std::fprintf(stderr, "[cpddg] win schedule: %d CTAs, modelled efficiency LPT %.3f, balanced %.3f (%d cuts)\n", grid,
                         pc->win_lpt_eff, pc->win_bal_eff, cuts);
    }
    CPDDG_CUDA(cudaMemcpy(ddesc.get(), desc.data(), desc.size() * sizeof(int), cudaMemcpyHostToDevice));
    pc->win_desc = std::move(ddesc);
    pc->win_items.alloc(items.size() * sizeof(win::Item));
    CPDDG_CUDA(cudaMemcpy(pc->win_items.get(), items.data(), items.size() * sizeof(win::Item), cudaMemcpyHostToDevice));
    pc->win_itbase.upload(itbase);
    pc->win_cta_begin.upload(begin);
    pc->win_cta_subs.upload(segs);
    pc->win_grid = grid;
    pc->win_gy = gy;
    pc->win_wmask = W - 1;
    pc->win_dback = dback;
    pc->win_ring = ring;
    pc->win_smem = ring + (gy ? 0 : 8 * W);
    pc->win_reach_l = reachL;
    pc->win_reach_u = reachU;
    pc->ybuf.alloc(static_cast<std::size_t>(std::max<std::int64_t>(pc->rows_total, 1)));
    for (auto kern : {k_solve_win<RB, false>, k_solve_win<RB, true>})
        raise_smem_limit(reinterpret_cast<const void*>(kern), pc->win_smem);
    pc->win = true;
    return true;
}

/** Thrown by pc_build when local systems need the pivoted host factorisation:
 *  a zero / non-finite pivot or a failed probe of the no-pivot device LU. */
struct NeedPivot {
    std::vector<int> subs;
};

static cpddg_pc* pc_build(int n_global, int n_sub, const cpddg_local_desc* locals, const cpddg_pc_options* opt,
                          const std::vector<char>& pivot_set) {
    if (n_global <= 0 || n_sub <= 0 || !locals) throw InternalError("empty preconditioner");
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<HostSub> subs(static_cast<std::size_t>(n_sub));
    parallel_for(n_sub, opt ? opt->workers : 0, [&](int j, int) {
        subs[static_cast<std::size_t>(j)] = analyse(locals[j], n_global, pivot_set[static_cast<std::size_t>(j)] != 0, j);
    });
    std::vector<int> pre(static_cast<std::size_t>(n_sub), 0);
    for (int j = 0; j < n_sub; ++j) pre[static_cast<std::size_t>(j)] = subs[static_cast<std::size_t>(j)].pivoted ? 1 : 0;
    if (std::getenv("CPDDG_VERBOSE")) {
        std::int64_t eL = 0, eU = 0;
        int reachL = 0, reachU = 0;  // longest row / column of the envelopes (a y window must cover it)
        for (const auto& S : subs) {
            eL += S.ne;
            eU += S.neU;
            for (int i = 0; i < S.n; ++i) {
                reachL = std::max(reachL, i - S.first[static_cast<std::size_t>(i)]);
                reachU = std::max(reachU, i - S.firstU[static_cast<std::size_t>(i)]);
            }
        }
        std::fprintf(stderr, "[cpddg] envelopes: L rows %lld, U columns %lld entries; longest L row %d, U column %d\n",
                     static_cast<long long>(eL), static_cast<long long>(eU), reachL, reachU);
    }
    // owned slots must be a disjoint cover (partition of unity, solve.hpp:62-63)
    std::vector<char> owned(static_cast<std::size_t>(n_global), 0);
    for (const auto& S : subs)
        for (int g : S.sidx)
            if (g >= 0) {
                if (owned[static_cast<std::size_t>(g)]) throw InternalError("restricted scatters overlap");
                owned[static_cast<std::size_t>(g)] = 1;
            }
    auto pc = std::make_unique<cpddg_pc>();
    pc->n_global = n_global;
    pc->n_sub = n_sub;
    std::vector<int> n_rows, first, firstU, rlast, urlast, gidx, sidx;
    std::vector<std::int64_t> vbase, ebase, ebaseU, roff, roffU;
    std::vector<double> probe_all, probe_dev;
    std::vector<std::vector<int>> invs;
    std::int64_t vb = 0, ebs = 0, ebsU = 0;
    for (auto& S : subs) {
        n_rows.push_back(S.n);
        vbase.push_back(vb);
        ebase.push_back(ebs);
        ebaseU.push_back(ebsU);
        vb += S.n;
        ebs += S.ne;
        ebsU += S.neU;
        pc->max_rows = std::max(pc->max_rows, S.n);
        pc->n_reduced += S.reduced ? 1 : 0;
    }
    pc->rows_total = vb;
    // values: scattered per subdomain into scratch and copied straight into
    // the device arrays (no host-side concatenation of the factor storage)
    pc->L.alloc(static_cast<std::size_t>(std::max<std::int64_t>(ebs, 1)));
    pc->U.alloc(static_cast<std::size_t>(std::max<std::int64_t>(ebsU, 1)));
    pc->diag.alloc(static_cast<std::size_t>(vb));
    const auto t_an = std::chrono::steady_clock::now();

    {
        // A_j's entries as (destination, value) pairs, scattered on the device
        std::vector<std::int64_t> pbase(static_cast<std::size_t>(n_sub) + 1, 0);
        for (int j = 0; j < n_sub; ++j) {
            const HostSub& S = subs[static_cast<std::size_t>(j)];
            pbase[static_cast<std::size_t>(j) + 1] =
                pbase[static_cast<std::size_t>(j)] + (S.pivoted ? S.ne + S.neU + S.n : locals[j].row_ptr[S.n]);
        }
        const std::int64_t cap = std::max<std::int64_t>(pbase.back(), 1);
        DevBuf<std::int64_t> pdst(static_cast<std::size_t>(cap));
        DevBuf<double> pval(static_cast<std::size_t>(cap));
        std::vector<std::int64_t> used(static_cast<std::size_t>(n_sub), 0);
        CPDDG_CUDA(cudaMemset(pc->L.get(), 0, sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(ebs, 1))));
        CPDDG_CUDA(cudaMemset(pc->U.get(), 0, sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(ebsU, 1))));
        CPDDG_CUDA(cudaMemset(pc->diag.get(), 0, sizeof(double) * static_cast<std::size_t>(vb)));
        // the workers copy on the caller's device (a new host thread starts on
        // device 0); the legacy default stream orders those copies before
        // k_scatter_pairs, and the synchronize below makes it explicit
        int dev = 0;
        CPDDG_CUDA(cudaGetDevice(&dev));
        parallel_for(n_sub, opt ? opt->workers : 0, [&](int j, int) {
            CPDDG_CUDA(cudaSetDevice(dev));
            const HostSub& S = subs[static_cast<std::size_t>(j)];
            const std::int64_t room = pbase[static_cast<std::size_t>(j) + 1] - pbase[static_cast<std::size_t>(j)];
            std::vector<std::int64_t> dst(static_cast<std::size_t>(room));
            std::vector<double> val(static_cast<std::size_t>(room));
            std::int64_t m = 0;
            if (S.pivoted) {  // the host factors, slot by slot
                const std::int64_t eb = ebase[static_cast<std::size_t>(j)], ebu = ebaseU[static_cast<std::size_t>(j)];
                const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
                for (std::int64_t e = 0; e < S.ne; ++e, ++m) {
                    dst[static_cast<std::size_t>(m)] = eb + e;
                    val[static_cast<std::size_t>(m)] = S.preL[static_cast<std::size_t>(e)];
                }
                for (std::int64_t e = 0; e < S.neU; ++e, ++m) {
                    dst[static_cast<std::size_t>(m)] = (1LL << kTagShift) | (ebu + e);
                    val[static_cast<std::size_t>(m)] = S.preU[static_cast<std::size_t>(e)];
                }
                for (int i = 0; i < S.n; ++i, ++m) {
                    dst[static_cast<std::size_t>(m)] = (2LL << kTagShift) | (v0 + i);
                    val[static_cast<std::size_t>(m)] = S.prediag[static_cast<std::size_t>(i)];
                }
            } else {
                m = scatter_pairs(locals[j], S, ebase[static_cast<std::size_t>(j)], ebaseU[static_cast<std::size_t>(j)],
                                  vbase[static_cast<std::size_t>(j)], dst.data(), val.data());
            }
            used[static_cast<std::size_t>(j)] = m;
            const std::size_t o = static_cast<std::size_t>(pbase[static_cast<std::size_t>(j)]);
            if (m) {
                CPDDG_CUDA(cudaMemcpy(pdst.get() + o, dst.data(), sizeof(std::int64_t) * m, cudaMemcpyHostToDevice));
                CPDDG_CUDA(cudaMemcpy(pval.get() + o, val.data(), sizeof(double) * m, cudaMemcpyHostToDevice));
            }
        });
        // unused tails of each subdomain's range: point them at a harmless zero add
        for (int j = 0; j < n_sub; ++j) {
            const std::int64_t o = pbase[static_cast<std::size_t>(j)] + used[static_cast<std::size_t>(j)];
            const std::int64_t rest = pbase[static_cast<std::size_t>(j) + 1] - o;
            if (rest > 0) {
                CPDDG_CUDA(cudaMemset(pdst.get() + o, 0, sizeof(std::int64_t) * static_cast<std::size_t>(rest)));
                CPDDG_CUDA(cudaMemset(pval.get() + o, 0, sizeof(double) * static_cast<std::size_t>(rest)));
            }
        }
        CPDDG_CUDA(cudaDeviceSynchronize());
        const int blocks = 4 * sm_count();
        k_scatter_pairs<<<blocks, 256>>>(pbase.back(), pdst.get(), pval.get(), pc->L.get(), pc->U.get(),
                                         pc->diag.get());
        CPDDG_CUDA(cudaGetLastError());
        CPDDG_CUDA(cudaDeviceSynchronize());
    }
    first.reserve(static_cast<std::size_t>(vb));
    int max_reach = 0;  // longest trailing window of the factorisation (k_factor2's block list)
    for (auto& S : subs) {
        for (int i = 0; i < S.n; ++i) max_reach = std::max(max_reach, S.rlast[static_cast<std::size_t>(i)] - i);
        append(first, S.first);
        append(firstU, S.firstU);
        append(rlast, S.rlast);
        append(urlast, S.urlast);
        append(roffU, S.roffU);
        append(gidx, S.gidx);
        append(sidx, S.sidx);
        append(roff, S.roff);
        append(probe_all, S.probe);
        if (S.pivoted)  // the device solves L U z = P b: its probe right-hand side is permuted
            for (int i = 0; i < S.n; ++i) probe_dev.push_back(S.probe[static_cast<std::size_t>(S.rowperm[static_cast<std::size_t>(i)])]);
        else
            append(probe_dev, S.probe);
        invs.push_back(std::move(S.inv));
        S = HostSub{};
    }
    std::vector<int> order(static_cast<std::size_t>(n_sub));
    std::iota(order.begin(), order.end(), 0);
    {
        std::vector<std::int64_t> subs_cost(static_cast<std::size_t>(n_sub));
        for (int j = 0; j < n_sub; ++j)
            subs_cost[static_cast<std::size_t>(j)] =
                (j + 1 < n_sub ? ebase[static_cast<std::size_t>(j) + 1] : ebs) - ebase[static_cast<std::size_t>(j)] +
                (j + 1 < n_sub ? ebaseU[static_cast<std::size_t>(j) + 1] : ebsU) - ebaseU[static_cast<std::size_t>(j)];
        std::vector<std::int64_t> cost(static_cast<std::size_t>(n_sub));
        for (int j = 0; j < n_sub; ++j)
            cost[static_cast<std::size_t>(j)] = subs_cost[static_cast<std::size_t>(j)];
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[static_cast<std::size_t>(a)] > cost[static_cast<std::size_t>(b)]; });
        // SM balance for the solve (2 resident CTAs per SM, blocks dealt to SMs
        // round-robin): with n_sub = S + P subdomains on S SMs, the S - P SMs that
        // get one CTA take the largest systems, and each remaining SM pairs a
        // large system with a small one.
        const int S = sm_count();
        const char* bal = std::getenv("CPDDG_BALANCE");
        if (n_sub > S && n_sub <= 2 * S && !(bal && std::string(bal) == "0")) {
            const int P = n_sub - S;          // SMs with two CTAs
            const int singles = S - P;        // SMs with one CTA
            std::vector<int> sorted = order, o(static_cast<std::size_t>(n_sub));
            for (int k = 0; k < singles; ++k) o[static_cast<std::size_t>(P + k)] = sorted[static_cast<std::size_t>(k)];
            for (int i = 0; i < P; ++i) {
                o[static_cast<std::size_t>(i)] = sorted[static_cast<std::size_t>(singles + i)];
                o[static_cast<std::size_t>(S + i)] = sorted[static_cast<std::size_t>(n_sub - 1 - i)];
            }
            order = o;
        }
    }
    pc->n_rows.upload(n_rows);
    pc->vbase.upload(vbase);
    pc->ebase.upload(ebase);
    pc->order.upload(order);
    pc->first.upload(first);
    pc->roff.upload(roff);
    pc->ebaseU.upload(ebaseU);
    pc->firstU.upload(firstU);
    pc->roffU.upload(roffU);
    pc->rlast.upload(rlast);
    pc->gidx.upload(gidx);
    pc->sidx.upload(sidx);

    const auto t1 = std::chrono::steady_clock::now();
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] pc analyse %.3f s, scatter+upload %.3f s\n",
                     std::chrono::duration<double>(t_an - t0).count(), std::chrono::duration<double>(t1 - t_an).count());
    pc->analyse_seconds = std::chrono::duration<double>(t1 - t0).count();

    // device factorisation
    const char* fenv = std::getenv("CPDDG_FACTOR");  // v1: the round-1 kernel (two CTAs per SM, no pipelining)
    const bool factor_v1_env = fenv && std::string(fenv) == "v1";
    const bool factor_v1 = factor_v1_env || max_reach + NB > kF2MaxBlk * TILE;
    const int fsm = factor_v1 ? static_cast<int>(sizeof(double)) * (NB * (NB + 1) + 4 * NB * kTS)
                              : static_cast<int>(sizeof(double)) * (NB * (NB + 1) + 2 * kF2Buf);
    if (factor_v1) {
        CPDDG_CUDA(cudaFuncSetAttribute(k_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm));
        // two CTAs per SM (256 subdomains in one wave on 148 SMs): full shared-memory carveout
        CPDDG_CUDA(cudaFuncSetAttribute(k_factor, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    } else {
        CPDDG_CUDA(cudaFuncSetAttribute(k_factor2, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm));
    }
    DevBuf<int> status(static_cast<std::size_t>(n_sub));
    status.zero();
    pc->dinv.alloc(static_cast<std::size_t>(vb));
    cudaEvent_t e0, e1;
    CPDDG_CUDA(cudaEventCreate(&e0));
    CPDDG_CUDA(cudaEventCreate(&e1));
    CPDDG_CUDA(cudaEventRecord(e0));
    DevBuf<int> dpre;
    dpre.upload(pre);
    if (factor_v1)
        k_factor<<<n_sub, kFactorThreads, fsm>>>(pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(),
                                               pc->ebaseU.get(), pc->first.get(), pc->roff.get(), pc->firstU.get(),
                                               pc->roffU.get(), pc->rlast.get(), pc->diag.get(),
                                               pc->L.get(), pc->U.get(), pc->dinv.get(), status.get(), dpre.get());
    else
        k_factor2<<<n_sub, kF2Threads, fsm>>>(pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(),
                                             pc->ebaseU.get(), pc->first.get(), pc->roff.get(), pc->firstU.get(),
                                             pc->roffU.get(), pc->rlast.get(), pc->diag.get(),
                                             pc->L.get(), pc->U.get(), pc->dinv.get(), status.get(), dpre.get());
    CPDDG_CUDA(cudaGetLastError());
    CPDDG_CUDA(cudaEventRecord(e1));
    CPDDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    CPDDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    pc->factor_seconds = ms * 1e-3;
    auto t_lap = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {  // CPDDG_VERBOSE: host wall time of the setup phases after the factorisation
        if (!std::getenv("CPDDG_VERBOSE")) return;
        CPDDG_CUDA(cudaDeviceSynchronize());
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[cpddg] pc %s: %.3f s\n", what, std::chrono::duration<double>(t - t_lap).count());
        t_lap = t;
    };
    std::vector<int> st(static_cast<std::size_t>(n_sub));
    CPDDG_CUDA(cudaMemcpy(st.data(), status.get(), st.size() * sizeof(int), cudaMemcpyDeviceToHost));
    {
        NeedPivot np;
        for (int j = 0; j < n_sub; ++j)
            if (st[static_cast<std::size_t>(j)]) {
                // a zero pivot of the pivoted host factor was already reported by piv_lu
                if (pre[static_cast<std::size_t>(j)]) throw DivergenceError("singular factorization of subdomain " + std::to_string(j));
                np.subs.push_back(j);
            }
        if (!np.subs.empty()) throw np;  // retry those subdomains with partial pivoting
    }
    pc->n_pivoted = static_cast<int>(std::count(pre.begin(), pre.end(), 1));

    pc->u_entries = ebsU;
    // record solve (default): U by columns; substitution-chain solve
    // (CPDDG_BLOCKINV=0): reversed U rows.  CPDDG_BWD_LAYOUT=rows|cols overrides.
    {
        const char* e = std::getenv("CPDDG_BLOCKINV");
        pc->blockinv = !(e && std::string(e) == "0");
    }
    pc->urows = !pc->blockinv;
    if (const char* e = std::getenv("CPDDG_BWD_LAYOUT")) pc->urows = std::string(e) != "cols";
    std::vector<int> ufirst;
    std::vector<std::int64_t> uroff, ubase;
    if (pc->urows) {
        ufirst.assign(static_cast<std::size_t>(vb), 0);
        uroff.assign(static_cast<std::size_t>(vb), 0);
        ubase.assign(static_cast<std::size_t>(n_sub), 0);
        std::int64_t ub = 0;
        for (int j = 0; j < n_sub; ++j) {
            const int nj = n_rows[static_cast<std::size_t>(j)];
            const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
            ubase[static_cast<std::size_t>(j)] = ub;
            std::int64_t off = 0;
            for (int ip = 0; ip < nj; ++ip) {
                const int i = nj - 1 - ip;
                const int fpr = (nj - 1 - urlast[static_cast<std::size_t>(v0 + i)]) & ~1;
                ufirst[static_cast<std::size_t>(v0 + ip)] = fpr;
                uroff[static_cast<std::size_t>(v0 + ip)] = off;
                off += (ip + (ip & 1)) - fpr;
            }
            ub += off;
        }
        pc->u_entries = ub;
        pc->ufirst.upload(ufirst);
        pc->uroff.upload(uroff);
        pc->ubase.upload(ubase);
        DevBuf<double> urev(static_cast<std::size_t>(std::max<std::int64_t>(ub, 1)));
        pc->drev.alloc(static_cast<std::size_t>(vb));
        k_reverse_u<<<n_sub, 256>>>(pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebaseU.get(),
                                    pc->ubase.get(), pc->firstU.get(), pc->roffU.get(), pc->ufirst.get(),
                                    pc->uroff.get(), pc->dinv.get(), pc->U.get(), urev.get(), pc->drev.get());
        CPDDG_CUDA(cudaGetLastError());
        CPDDG_CUDA(cudaDeviceSynchronize());
        pc->U = std::move(urev);
    }
    pc->entries = ebs + pc->u_entries + vb;
    pc->profile_entries = ebs + ebsU + vb;
    pc->solve_smem = static_cast<int>(sizeof(double)) * pc->max_rows;
    if (const char* e = std::getenv("CPDDG_BWD_PREFETCH")) pc->bwd_prefetch = std::atoi(e);
    // solve path: CPDDG_SOLVE=win (default; windowed streamed solve, any
    // subdomain size), tma (k_solve_tma, whole y in shared memory) or reg
    // (register-staged k_solve); the last two need y in shared memory
    const std::string solve_path = [] {
        const char* e = std::getenv("CPDDG_SOLVE");
        const char* t = std::getenv("CPDDG_TMA");  // round-1 switch: CPDDG_TMA=0 = register-staged
        return e ? std::string(e) : (t && std::string(t) == "0") ? std::string("reg") : std::string("win");
    }();
    const bool smem_y = pc->solve_smem <= 200 * 1024;
    if (solve_path != "win" && !smem_y)
        throw ConfigError("subdomain system too large for the shared-memory solve (CPDDG_SOLVE=" + solve_path + ")");
    // the shared-memory-y kernels can only run (and only need their limit raised) when y fits
    const int solve_smem_set = smem_y ? pc->solve_smem : 1;
    set_solve_smem<false, ShapeMid, false>(solve_smem_set);
    set_solve_smem<true, ShapeBig, false>(solve_smem_set);
    set_solve_smem<true, ShapeMid, false>(solve_smem_set);
    set_solve_smem<true, ShapeSmall, false>(solve_smem_set);
    set_solve_smem<true, ShapeBig, true>(solve_smem_set);
    set_solve_smem<true, ShapeMid, true>(solve_smem_set);
    set_solve_smem<true, ShapeRec, true>(solve_smem_set);
    set_solve_smem<false, ShapeBig, true>(solve_smem_set);
    set_solve_smem<false, ShapeMid, true>(solve_smem_set);
    set_solve_smem<false, ShapeRec, true>(solve_smem_set);
    set_solve_smem<false, ShapeRec8, true>(solve_smem_set);
    lap("pivot check, kernel attributes");
    // block shape: one CTA per subdomain, all resident in one wave
    {
        const int S = sm_count();
        // measured: two waves of ShapeMid beat one wave of ShapeSmall; the
        // record solve uses ShapeRec (shape 3) when n_sub > #SMs
        pc->shape = pc->blockinv ? 3 : n_sub <= S ? 0 : 1;  // record solve: streamed (measured faster at 64 and 256 subdomains)
        if (const char* e = std::getenv("CPDDG_SOLVE_SHAPE")) {
            const std::string v(e);
            pc->shape = v == "big" ? 0 : v == "mid" ? 1 : v == "small" ? 2 : v == "rec" ? 3 : pc->shape;
        }
    }
    // record solve: block records from the full rows, then the rows compacted
    // to their far parts (CPDDG_BLOCKINV=0 keeps the substitution-chain solve)
    // persistent TMA-streamed solve (k_solve_tma): U by columns, records for tmas::RB
    bool want_tma = false, want_win = false;
    {
        const int tma_smem = tmas::RING + 8 * tmas::NB * tmas::kRec + 4 * tmas::NB * tmas::kDesc + 8 * pc->max_rows;
        const bool streamable = pc->blockinv && !pc->urows && pc->shape == 3;
        want_win = streamable && solve_path == "win";
        want_tma = streamable && solve_path == "tma" && tma_smem <= 227 * 1024;
        if (want_tma) pc->shape = 4;  // the streamed path's RB; ShapeRec8 if an item would not fit the ring
        if (want_win) {
            pc->shape = 5;
            pc->win_rb = win_choose_rb(n_rows, vbase, first, firstU);
            if (const char* e = std::getenv("CPDDG_WIN_RB")) pc->win_rb = std::atoi(e) == 8 ? 8 : 16;
        }
        if (!want_win && !smem_y) throw ConfigError("subdomain system too large for the shared-memory solve");
    }
    if (pc->blockinv) {
        const int rb = pc->shape == 5 ? pc->win_rb : pc->shape == 4 ? tmas::RB : pc->shape >= 2 ? ShapeRec::RB : ShapeMid::RB;
        static_assert(ShapeBig::RB == ShapeMid::RB && ShapeSmall::RB == ShapeRec::RB,
                      "records are built for RB = 30 or RB = 14");
        std::vector<std::int64_t> rbase(static_cast<std::size_t>(n_sub));
        std::int64_t rt = 0;
        for (int j = 0; j < n_sub; ++j) {
            rbase[static_cast<std::size_t>(j)] = rt;
            rt += static_cast<std::int64_t>((n_rows[static_cast<std::size_t>(j)] + rb - 1) / rb) * rec_pitch(rb);
        }
        pc->rec_entries = 2 * rt;
        pc->rbase.upload(rbase);
        pc->recL.alloc(static_cast<std::size_t>(std::max<std::int64_t>(rt, 1)));
        pc->recU.alloc(static_cast<std::size_t>(std::max<std::int64_t>(rt, 1)));
        const dim3 rgrid(static_cast<unsigned>(n_sub), 16);
        auto records = rb == 30 ? k_block_records<30> : rb == 14 ? k_block_records<14> : rb == 16 ? k_block_records<16>
                                                                                   : k_block_records<8>;
        auto compact = rb == 30 ? k_compact_rows<30> : rb == 14 ? k_compact_rows<14> : rb == 16 ? k_compact_rows<16>
                                                                                  : k_compact_rows<8>;
        records<<<rgrid, 64>>>(pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(), pc->first.get(), pc->roff.get(),
                               pc->L.get(), nullptr, pc->rbase.get(), pc->recL.get());
        if (pc->urows)
            records<<<rgrid, 64>>>(pc->n_rows.get(), pc->vbase.get(), pc->ubase.get(), pc->ufirst.get(),
                                   pc->uroff.get(), pc->U.get(), pc->drev.get(), pc->rbase.get(), pc->recU.get());
        else
            (rb == 30 ? k_block_records_upper<30> : rb == 14 ? k_block_records_upper<14>
                                  : rb == 16 ? k_block_records_upper<16> : k_block_records_upper<8>)<<<rgrid, 64>>>(
                pc->n_rows.get(), pc->vbase.get(), pc->ebaseU.get(), pc->firstU.get(), pc->roffU.get(), pc->U.get(),
                pc->dinv.get(), pc->rbase.get(), pc->recU.get());
        CPDDG_CUDA(cudaGetLastError());
        // far parts: row i keeps [f_i, max(f_i, (i / rb - 1) rb))
        auto far_layout = [&](const std::vector<int>& f, std::vector<std::int64_t>& roc, std::vector<std::int64_t>& cb) {
            roc.assign(static_cast<std::size_t>(vb), 0);
            cb.assign(static_cast<std::size_t>(n_sub), 0);
            std::int64_t tot = 0;
            for (int j = 0; j < n_sub; ++j) {
                cb[static_cast<std::size_t>(j)] = tot;
                const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
                std::int64_t off = 0;
                for (int i = 0; i < n_rows[static_cast<std::size_t>(j)]; ++i) {
                    if (i % rb == 0) off = (off + 15) / 16 * 16;  // blocks start on 128-byte lines
                    const int fi = f[static_cast<std::size_t>(v0 + i)];
                    roc[static_cast<std::size_t>(v0 + i)] = off;
                    off += std::max(0, (i / rb - 1) * rb - fi);
                }
                tot += (off + 15) / 16 * 16;
            }
            return tot;
        };
        if (std::getenv("CPDDG_VERBOSE")) {
            // layout study: U far entries by columns vs per-block rectangles
            std::int64_t cols = 0, rect = 0, lrows = 0;
            for (int j = 0; j < n_sub; ++j) {
                const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
                const int nj = n_rows[static_cast<std::size_t>(j)];
                for (int K = 1; K * rb < nj; ++K) {
                    int fmin = INT_MAX;
                    for (int c = K * rb; c < std::min(nj, K * rb + rb); ++c) {
                        const int fc = firstU[static_cast<std::size_t>(v0 + c)];
                        fmin = std::min(fmin, fc);
                        cols += std::max(0, (K - 1) * rb - fc);
                        lrows += std::max(0, (K - 1) * rb - first[static_cast<std::size_t>(v0 + c)]);
                    }
                    rect += static_cast<std::int64_t>(rb) * std::max(0, (K - 1) * rb - fmin);
                }
            }
            std::fprintf(stderr, "[cpddg] far entries: L rows %lld, U cols %lld, U block rectangles %lld\n",
                         static_cast<long long>(lrows), static_cast<long long>(cols), static_cast<long long>(rect));
        }
        std::vector<std::int64_t> rocL, cbL, rocU, cbU;
        const std::int64_t nL = far_layout(first, rocL, cbL), nU = far_layout(pc->urows ? ufirst : firstU, rocU, cbU);
        DevBuf<std::int64_t> drocL, dcbL, drocU, dcbU;
        drocL.upload(rocL);
        dcbL.upload(cbL);
        drocU.upload(rocU);
        dcbU.upload(cbU);
        DevBuf<double> Lc(static_cast<std::size_t>(std::max<std::int64_t>(nL, 1))),
            Uc(static_cast<std::size_t>(std::max<std::int64_t>(nU, 1)));
        compact<<<n_sub, 256>>>(pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(), pc->first.get(), pc->roff.get(),
                                pc->L.get(), dcbL.get(), drocL.get(), Lc.get());
        if (pc->urows)
            compact<<<n_sub, 256>>>(pc->n_rows.get(), pc->vbase.get(), pc->ubase.get(), pc->ufirst.get(),
                                    pc->uroff.get(), pc->U.get(), dcbU.get(), drocU.get(), Uc.get());
        else  // U columns: the same far-part rule, [f_c, (c / rb - 1) rb)
            compact<<<n_sub, 256>>>(pc->n_rows.get(), pc->vbase.get(), pc->ebaseU.get(), pc->firstU.get(),
                                    pc->roffU.get(), pc->U.get(), dcbU.get(), drocU.get(), Uc.get());
        CPDDG_CUDA(cudaGetLastError());
        CPDDG_CUDA(cudaDeviceSynchronize());
        pc->L = std::move(Lc);
        pc->U = std::move(Uc);
        pc->roff = std::move(drocL);
        pc->ebase = std::move(dcbL);
        if (pc->urows) {
            pc->uroff = std::move(drocU);
            pc->ubase = std::move(dcbU);
        } else {
            pc->roffU = std::move(drocU);
            pc->ebaseU = std::move(dcbU);
        }
        pc->far_entries = nL + nU;
        if (want_tma) setup_tma(pc.get(), n_rows, vbase, first, firstU, rocL, cbL, rocU, cbU, rbase);
        if (want_win) {
            const bool ok = pc->win_rb == 8 ? setup_win<8>(pc.get(), n_rows, vbase, first, firstU, rocL, cbL, rocU, cbU, rbase)
                                            : setup_win<16>(pc.get(), n_rows, vbase, first, firstU, rocL, cbL, rocU, cbU, rbase);
            if (!ok) throw ConfigError("preconditioner blocks do not fit the streamed solve's shared memory");
        }
    }
    lap("records, far parts, solve tables and schedule");
    // factor probe (cpddg_pc_options::check_residual): solve A_j z = A_j x_probe
    // on the device for every subdomain and check the residual on the host --
    // the DirectSolver contract of the reference (residual ~1e-12,
    // tests/test_transmission.cpp:307-334) made observable.
    if (opt && opt->check_residual) {
        DevBuf<double> pb, pz(static_cast<std::size_t>(vb));
        pb.upload(probe_dev);
        pc_apply_mode(pc.get(), pb.get(), pz.get(), false, 3, nullptr);
        std::vector<double> z(static_cast<std::size_t>(vb));
        CPDDG_CUDA(cudaMemcpy(z.data(), pz.get(), z.size() * sizeof(double), cudaMemcpyDeviceToHost));
        std::vector<double> res(static_cast<std::size_t>(n_sub), 0.0);
        parallel_for(n_sub, opt->workers, [&](int j, int) {
            const cpddg_local_desc& d = locals[j];
            const std::vector<int>& inv = invs[static_cast<std::size_t>(j)];
            const int n = n_rows[static_cast<std::size_t>(j)];
            const std::int64_t v0 = vbase[static_cast<std::size_t>(j)];
            double rmax = 0.0, bmax = 0.0;
            for (int r = 0; r < n; ++r) {
                double acc = 0.0;
                for (std::int64_t k = d.row_ptr[r]; k < d.row_ptr[r + 1]; ++k) {
                    const int c = d.col[k];
                    if (c >= n) continue;
                    acc += d.val[k] * z[static_cast<std::size_t>(v0 + inv[static_cast<std::size_t>(c)])];
                }
                const double b = probe_all[static_cast<std::size_t>(v0 + inv[static_cast<std::size_t>(r)])];
                rmax = std::max(rmax, std::abs(acc - b));
                bmax = std::max(bmax, std::abs(b));
            }
            res[static_cast<std::size_t>(j)] = bmax > 0 ? rmax / bmax : rmax;
        });
        pc->max_probe_residual = *std::max_element(res.begin(), res.end());
        NeedPivot np;
        for (int j = 0; j < n_sub; ++j)
            if (!(res[static_cast<std::size_t>(j)] <= 1e-8)) {
                if (pre[static_cast<std::size_t>(j)])
                    throw DivergenceError("inaccurate factorization of subdomain " + std::to_string(j) +
                                          " (probe residual " + std::to_string(res[static_cast<std::size_t>(j)]) + ")");
                np.subs.push_back(j);
            }
        if (!np.subs.empty()) throw np;  // no-pivot factors not accurate enough: pivot those
    }
    lap("probe solves");
    // small systems: dense inverses (k_solve_dense) when the envelope solve
    // would be a latency-bound chain on a mostly idle GPU
    {
        std::int64_t dense_entries = 0;
        for (int nj : n_rows) dense_entries += static_cast<std::int64_t>(nj) * nj;
        const char* e = std::getenv("CPDDG_DENSE");
        const bool auto_dense = pc->max_rows <= 1024 && n_sub <= sm_count() && 8 * dense_entries <= (256LL << 20);
        pc->dense = e ? std::string(e) == "1" && 8 * dense_entries <= (4LL << 30) : auto_dense;
        if (pc->dense) {
            std::vector<std::int64_t> dbase(static_cast<std::size_t>(n_sub));
            std::vector<int> tsub, trow;
            std::int64_t acc = 0;
            for (int j = 0; j < n_sub; ++j) {
                dbase[static_cast<std::size_t>(j)] = acc;
                acc += static_cast<std::int64_t>(n_rows[static_cast<std::size_t>(j)]) * n_rows[static_cast<std::size_t>(j)];
                for (int r0 = 0; r0 < n_rows[static_cast<std::size_t>(j)]; r0 += kDenseRows) {
                    tsub.push_back(j);
                    trow.push_back(r0);
                }
            }
            pc->dense_base.upload(dbase);
            pc->dense_tile_sub.upload(tsub);
            pc->dense_tile_row0.upload(trow);
            pc->dense_tiles = static_cast<int>(tsub.size());
            pc->Ainv.alloc(static_cast<std::size_t>(std::max<std::int64_t>(acc, 1)));
            if (static_cast<int>(sizeof(double)) * pc->max_rows > 48 * 1024)
                raise_smem_limit(reinterpret_cast<const void*>(k_solve_dense),
                                 static_cast<int>(sizeof(double)) * pc->max_rows);
            // column k of A_j^-1 = the envelope solve of e_k, for all subdomains at once
            DevBuf<double> er(static_cast<std::size_t>(vb)), ez(static_cast<std::size_t>(vb));
            er.zero();
            const int ub = (n_sub + 127) / 128;
            for (int k = 0; k < pc->max_rows; ++k) {
                k_unit_rhs<<<ub, 128>>>(n_sub, pc->n_rows.get(), pc->vbase.get(), k, er.get());
                pc_apply_mode(pc.get(), er.get(), ez.get(), false, 3, nullptr);  // envelope path (dense_probe off)
                k_store_column<<<n_sub, 256>>>(k, pc->n_rows.get(), pc->vbase.get(), pc->dense_base.get(), ez.get(),
                                               pc->Ainv.get());
                k_unit_clear<<<ub, 128>>>(n_sub, pc->n_rows.get(), pc->vbase.get(), k, er.get());
            }
            CPDDG_CUDA(cudaGetLastError());
            CPDDG_CUDA(cudaDeviceSynchronize());
            pc->dense_entries = acc;
            // the inverses reproduce the envelope solve on the probe right-hand sides
            if (!probe_all.empty()) {
                DevBuf<double> pb, z1(static_cast<std::size_t>(vb)), z2(static_cast<std::size_t>(vb));
                pb.upload(probe_dev);
                pc_apply_mode(pc.get(), pb.get(), z1.get(), false, 3, nullptr);
                pc->dense_probe = true;
                pc_apply_mode(pc.get(), pb.get(), z2.get(), false, 3, nullptr);
                pc->dense_probe = false;
                std::vector<double> a(static_cast<std::size_t>(vb)), c(static_cast<std::size_t>(vb));
                CPDDG_CUDA(cudaMemcpy(a.data(), z1.get(), a.size() * sizeof(double), cudaMemcpyDeviceToHost));
                CPDDG_CUDA(cudaMemcpy(c.data(), z2.get(), c.size() * sizeof(double), cudaMemcpyDeviceToHost));
                double dmax = 0.0, amax = 0.0;
                for (std::size_t q = 0; q < a.size(); ++q) {
                    dmax = std::max(dmax, std::abs(a[q] - c[q]));
                    amax = std::max(amax, std::abs(a[q]));
                }
                if (!(dmax <= 1e-10 * amax)) pc->dense = false;  // keep the envelope solve
            }
        }
    }
    // bytes one apply streams: L, U, diag, first, roff per row, gather/scatter maps, r gathers, z writes
    // streamed per apply: L and reversed-U values, diagonal, and the per-row
    // tables (first + offset) of both passes
    if (pc->blockinv) pc->entries = pc->far_entries + pc->rec_entries;
    pc->factor_bytes = pc->dense      ? 8 * pc->dense_entries
                       : pc->blockinv ? 8 * (pc->far_entries + pc->rec_entries) + 2 * 12 * vb
                                      : 8 * (ebs + pc->u_entries + vb) + 2 * 12 * vb;
    std::int64_t gathers = 0, scatters = 0;
    for (int g : gidx) gathers += g >= 0 ? 1 : 0;
    for (int s : sidx) scatters += s >= 0 ? 1 : 0;
    // B_pc = stored factor bytes + 12 |Sigma_j| (gather) + 12 N_A (scatter)
    pc->alg_bytes = pc->factor_bytes + 12 * gathers + 12 * scatters;
    return pc.release();
}

/** A local system without the unknowns nothing depends on.
 *
 *  An ORAS closure holds the Robin ring and the ghost-type closure nodes
 *  (transmission.hpp:84-92: "only ever referenced by their own transmission
 *  row"): unknown q appears in no row but its own, it is not scattered back
 *  (only owned overlap slots are, transmission.hpp:66-69), and so no value the
 *  preconditioner returns depends on it -- row q only defines x_q from the
 *  others.  Deleting row and column q leaves every other unknown's equation,
 *  hence its solution, unchanged (the system is block triangular with the
 *  nonzero a_qq on the diagonal, so it is singular exactly when the reduced
 *  one is).  Dropped rows may hold the only references to further closure
 *  unknowns: iterated to the fixed point with a work list.  At the headline
 *  this removes ~17 % of the local unknowns and ~20 % of the envelope entries
 *  every apply streams.  CPDDG_DROP=0 keeps the systems whole (parity test). */
struct OwnedLocal {
    std::vector<std::int64_t> ptr;
    std::vector<int> col, scl;
    std::vector<double> val;
};

/** gone[q] = 1 for every unknown drop_unreferenced removes; returns their count
 *  (0 for malformed input, which analyse() reports). */
static int mark_unreferenced(const cpddg_local_desc& d, std::vector<char>& gone) {
    const int nl = d.n_overlap + d.n_bc;
    gone.assign(static_cast<std::size_t>(std::max(nl, 0)), 0);
    if (d.n_overlap < 0 || d.n_bc <= 0 || !d.row_ptr || !d.col || !d.val) return 0;
    const std::int64_t* rp = d.row_ptr;
    // malformed input is left for analyse() to report
    for (int r = 0; r < nl; ++r)
        if (rp[r + 1] < rp[r]) return 0;
    for (std::int64_t k = rp[0]; k < rp[nl]; ++k)
        if (d.col[k] < 0 || d.col[k] >= nl) return 0;
    for (int k = 0; k < d.n_scatter; ++k)
        if (d.scatter_local[k] < 0 || d.scatter_local[k] >= nl) return 0;
    std::vector<int> ref(static_cast<std::size_t>(nl), 0);     // off-diagonal entries of column c in live rows
    std::vector<double> dg(static_cast<std::size_t>(nl), 0.0);  // a_cc (duplicates summed, as the solver does)
    for (int r = 0; r < nl; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            if (d.col[k] == r)
                dg[static_cast<std::size_t>(r)] += d.val[k];
            else
                ++ref[static_cast<std::size_t>(d.col[k])];
        }
    std::vector<char> fixed(static_cast<std::size_t>(nl), 0);
    for (int k = 0; k < d.n_scatter; ++k) fixed[static_cast<std::size_t>(d.scatter_local[k])] = 1;
    auto free_unknown = [&](int c) {
        return c >= d.n_overlap && !fixed[static_cast<std::size_t>(c)] && !gone[static_cast<std::size_t>(c)] &&
               ref[static_cast<std::size_t>(c)] == 0 && dg[static_cast<std::size_t>(c)] != 0.0 &&
               std::isfinite(dg[static_cast<std::size_t>(c)]);
    };
    std::vector<int> work;
    for (int c = d.n_overlap; c < nl; ++c)
        if (free_unknown(c)) {
            gone[static_cast<std::size_t>(c)] = 1;
            work.push_back(c);
        }
    int dropped = 0;
    while (!work.empty()) {
        const int q = work.back();
        work.pop_back();
        ++dropped;
        for (std::int64_t k = rp[q]; k < rp[q + 1]; ++k) {
            const int c = d.col[k];
            if (c == q) continue;
            --ref[static_cast<std::size_t>(c)];
            if (free_unknown(c)) {
                gone[static_cast<std::size_t>(c)] = 1;
                work.push_back(c);
            }
        }
    }
    return dropped;
}

static int drop_unreferenced(const cpddg_local_desc& d, OwnedLocal& o, cpddg_local_desc& out) {
    std::vector<char> gone;
    const int dropped = mark_unreferenced(d, gone);
    if (dropped == 0) return 0;
    const int nl = d.n_overlap + d.n_bc;
    const std::int64_t* rp = d.row_ptr;
    std::vector<int> id(static_cast<std::size_t>(nl));
    int m = 0;
    std::int64_t nnz = 0;
    for (int c = 0; c < nl; ++c) {
        id[static_cast<std::size_t>(c)] = gone[static_cast<std::size_t>(c)] ? -1 : m++;
        if (!gone[static_cast<std::size_t>(c)]) nnz += rp[c + 1] - rp[c];
    }
    o.ptr.assign(1, 0);
    o.ptr.reserve(static_cast<std::size_t>(m) + 1);
    o.col.resize(static_cast<std::size_t>(nnz));
    o.val.resize(static_cast<std::size_t>(nnz));
    std::int64_t w = 0;
    for (int r = 0; r < nl; ++r) {
        if (gone[static_cast<std::size_t>(r)]) continue;
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k, ++w) {
            o.col[static_cast<std::size_t>(w)] = id[static_cast<std::size_t>(d.col[k])];  // live rows hold live columns only
            o.val[static_cast<std::size_t>(w)] = d.val[k];
        }
        o.ptr.push_back(w);
    }
    o.scl.resize(static_cast<std::size_t>(std::max(d.n_scatter, 0)));
    for (int k = 0; k < d.n_scatter; ++k) o.scl[static_cast<std::size_t>(k)] = id[static_cast<std::size_t>(d.scatter_local[k])];
    out = d;
    out.n_bc = d.n_bc - dropped;
    out.scatter_local = o.scl.data();
    out.row_ptr = o.ptr.data();
    out.col = o.col.data();
    out.val = o.val.data();
    return dropped;
}

/** pc_build with the DirectSolver's robustness (direct.hpp:41-52: Eigen
 *  SparseLU pivots): local systems whose no-pivot device factorisation hits
 *  a zero / non-finite pivot or misses the probe-residual contract are
 *  factored on the host with partial pivoting (piv_lu) and the whole
 *  preconditioner is rebuilt with them.  CPDDG_PIVOT=all pivots every
 *  subdomain (testing). */
static cpddg_pc* pc_build_pivoting(int n_global, int n_sub, const cpddg_local_desc* locals_in,
                                   const cpddg_pc_options* opt) {
    // unknowns nothing depends on leave the local systems first (drop_unreferenced)
    std::vector<OwnedLocal> owned;
    std::vector<cpddg_local_desc> reduced;
    std::int64_t n_dropped = 0;
    const cpddg_local_desc* locals = locals_in;
    const char* de = std::getenv("CPDDG_DROP");
    const auto t_drop = std::chrono::steady_clock::now();
    if (n_sub > 0 && locals_in && !(de && std::string(de) == "0")) {
        owned.resize(static_cast<std::size_t>(n_sub));
        reduced.assign(locals_in, locals_in + n_sub);
        std::vector<int> cnt(static_cast<std::size_t>(n_sub), 0);
        parallel_for(n_sub, opt ? opt->workers : 0, [&](int j, int) {
            cnt[static_cast<std::size_t>(j)] =
                drop_unreferenced(locals_in[j], owned[static_cast<std::size_t>(j)], reduced[static_cast<std::size_t>(j)]);
        });
        for (int c : cnt) n_dropped += c;
        if (n_dropped > 0) locals = reduced.data();
        if (std::getenv("CPDDG_VERBOSE"))
            std::fprintf(stderr, "[cpddg] pc reduce: %lld unreferenced unknowns dropped in %.3f s\n",
                         static_cast<long long>(n_dropped),
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_drop).count());
    }
    std::vector<char> pivot(static_cast<std::size_t>(std::max(n_sub, 0)), 0);
    if (const char* e = std::getenv("CPDDG_PIVOT"); e && std::string(e) == "all") std::fill(pivot.begin(), pivot.end(), 1);
    for (int attempt = 0;; ++attempt) {
        try {
            cpddg_pc* pc = pc_build(n_global, n_sub, locals, opt, pivot);
            pc->n_dropped = n_dropped;
            return pc;
        } catch (const NeedPivot& np) {
            if (attempt > 0 && std::none_of(np.subs.begin(), np.subs.end(), [&](int j) { return !pivot[static_cast<std::size_t>(j)]; }))
                throw DivergenceError("inaccurate factorization of subdomain " + std::to_string(np.subs.front()));
            for (int j : np.subs) pivot[static_cast<std::size_t>(j)] = 1;
            if (std::getenv("CPDDG_VERBOSE"))
                std::fprintf(stderr, "[cpddg] %zu local system(s) refactored with partial pivoting (first: %d)\n",
                             np.subs.size(), np.subs.front());
        }
    }
}

}  // namespace cpddg

using namespace cpddg;

namespace cpddg {
__global__ void k_zero_stats(std::int64_t n, const double* __restrict__ a, unsigned long long* out) {
    unsigned long long z = 0, zs = 0;
    for (std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; s < (n + 15) / 16;
         s += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int cnt = 0, len = 0;
        for (int q = 0; q < 16; ++q) {
            const std::int64_t i = 16 * s + q;
            if (i < n) {
                ++len;
                if (a[i] == 0.0) ++cnt;
            }
        }
        z += cnt;
        zs += cnt == len ? 1 : 0;
    }
    atomicAdd(out, z);
    atomicAdd(out + 1, zs);
}
}  // namespace cpddg

extern "C" {

int cpddg_pc_create(int n_global, int n_sub, const cpddg_local_desc* locals, const cpddg_pc_options* opt,
                    cpddg_pc** out) {
    return guarded([&] {
        if (!out) throw InternalError("null argument");
        *out = pc_build_pivoting(n_global, n_sub, locals, opt);
    });
}

int cpddg_local_unreferenced(const cpddg_local_desc* d, unsigned char* dropped, int* n_dropped) {
    return guarded([&] {
        if (!d || !dropped || !n_dropped) throw InternalError("null argument");
        std::vector<char> gone;
        *n_dropped = mark_unreferenced(*d, gone);
        for (std::size_t q = 0; q < gone.size(); ++q) dropped[q] = static_cast<unsigned char>(gone[q]);
    });
}

int cpddg_pc_create_from_setup(const cpddg_setup* s, const cpddg_pc_options* opt, cpddg_pc** out) {
    return guarded([&] {
        if (!s || !out) throw InternalError("null argument");
        const std::vector<LocalSystem>* locs = nullptr;
        int n_global = 0;
        if (s->dim == 2) {
            locs = &impl_of<2>(s).locals;
            n_global = impl_of<2>(s).band.n_active;
        } else {
            locs = &impl_of<3>(s).locals;
            n_global = impl_of<3>(s).band.n_active;
        }
        if (locs->empty()) throw ConfigError("setup has no subdomains: call cpddg_setup_decompose first");
        std::vector<cpddg_local_desc> d(locs->size());
        for (std::size_t j = 0; j < locs->size(); ++j) {
            const LocalSystem& L = (*locs)[j];
            d[j] = {L.n_overlap, L.n_bc, L.overlap.data(), static_cast<int>(L.scatter_local.size()),
                    L.scatter_local.data(), L.scatter_global.data(), L.A.ptr.data(), L.A.col.data(), L.A.val.data()};
        }
        *out = pc_build_pivoting(n_global, static_cast<int>(d.size()), d.data(), opt);
    });
}

int cpddg_pc_apply(cpddg_pc* pc, const double* r, double* z, void* stream) {
    return guarded([&] {
        if (!pc || !r || !z) throw InternalError("null argument");
        pc_apply(pc, r, z, false, static_cast<cudaStream_t>(stream));
    });
}

int cpddg_pc_stats_get(const cpddg_pc* pc, cpddg_pc_stats* st) {
    return guarded([&] {
        if (!pc || !st) throw InternalError("null argument");
        st->n_sub = pc->n_sub;
        st->n_reduced = pc->n_reduced;
        st->n_rows_total = pc->rows_total;
        st->factor_entries = pc->entries;
        st->profile_entries = pc->profile_entries;
        st->factor_bytes = pc->factor_bytes;
        st->algorithmic_bytes = pc->alg_bytes;
        st->max_rows = pc->max_rows;
        st->factor_seconds = pc->factor_seconds;
        st->analyse_seconds = pc->analyse_seconds;
        st->max_probe_residual = pc->max_probe_residual;
        st->apply_mode = pc->dense ? 1 : pc->tma ? 2 : pc->win ? (pc->win_gy ? 4 : 3) : 0;
        st->n_pivoted = pc->n_pivoted;
        st->n_dropped = pc->n_dropped;
        st->win_cuts = pc->win && !pc->win_gy ? pc->win_cuts : 0;
        st->win_lpt_efficiency = pc->win ? pc->win_lpt_eff : 0.0;
        st->win_bal_efficiency = pc->win ? pc->win_bal_eff : 0.0;
    });
}

/** Development hooks (include/cpddg.h, last section): the per-block trace and
 *  one pass of the preconditioner (mode 1 forward, 2 backward, 0 both, 3 probe). */

/** Development: exact zeros among the stored factor entries (L, U arrays as
 *  streamed by the solve) and all-zero 16-entry segments: out[6] = L size,
 *  L zeros, L zero segments, U size, U zeros, U zero segments. */
int cpddg_pc_debug_zero_stats(const cpddg_pc* pc, int64_t* out) {
    return guarded([&] {
        if (!pc || !out) throw InternalError("null argument");
        DevBuf<unsigned long long> d(4);
        d.zero();
        const std::int64_t nl = static_cast<std::int64_t>(pc->L.size()), nu = static_cast<std::int64_t>(pc->U.size());
        k_zero_stats<<<4 * sm_count(), 256>>>(nl, pc->L.get(), d.get());
        k_zero_stats<<<4 * sm_count(), 256>>>(nu, pc->U.get(), d.get() + 2);
        CPDDG_CUDA(cudaGetLastError());
        unsigned long long h[4];
        CPDDG_CUDA(cudaMemcpy(h, d.get(), sizeof(h), cudaMemcpyDeviceToHost));
        out[0] = nl;
        out[1] = static_cast<int64_t>(h[0]);
        out[2] = static_cast<int64_t>(h[1]);
        out[3] = nu;
        out[4] = static_cast<int64_t>(h[2]);
        out[5] = static_cast<int64_t>(h[3]);
    });
}

int cpddg_dev_trace(long long* out) {  // development: copy g_trace
    return guarded([&] { CPDDG_CUDA(cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * 1024 * 20)); });
}

int cpddg_pc_apply_mode(cpddg_pc* pc, const double* r, double* z, int mode, void* stream) {
    return guarded([&] {
        if (!pc || !r || !z) throw InternalError("null argument");
        pc_apply_mode(pc, r, z, false, mode, static_cast<cudaStream_t>(stream));
    });
}

int cpddg_pc_destroy(cpddg_pc* pc) {
    delete pc;
    return CPDDG_OK;
}

}  // extern "C"
