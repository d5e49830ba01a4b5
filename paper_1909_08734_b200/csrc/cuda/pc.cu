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
#include "../host/setup.hpp"
#include "common.cuh"
#include "op.cuh"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <numeric>

namespace cpddg {

namespace {

constexpr int NB = 32;    // factor panel width
constexpr int TILE = 64;  // trailing-update tile
constexpr int SB = 32;    // solve block

struct HostSub {
    int n = 0;
    bool reduced = false;
    std::vector<int> first, rlast, gidx, sidx;
    std::vector<std::int64_t> roff;
    std::vector<double> L, U, diag;
};

/** Reverse Cuthill-McKee of a symmetric pattern (sorted, no diagonal).
 *  Components in order of their lowest-degree node; each starts at a
 *  pseudo-peripheral node (repeated BFS, min-degree node of the last level);
 *  neighbours enqueued by (degree, index).  Returns perm[new] = old. */
std::vector<int> rcm(const std::vector<std::vector<int>>& adj) {
    const int n = static_cast<int>(adj.size());
    std::vector<int> order;
    order.reserve(static_cast<std::size_t>(n));
    std::vector<char> done(static_cast<std::size_t>(n), 0);
    std::vector<int> level(static_cast<std::size_t>(n), -1);
    auto deg = [&](int v) { return static_cast<int>(adj[static_cast<std::size_t>(v)].size()); };
    auto far_node = [&](int s, int& ecc) {
        std::vector<int> q{s};
        level[static_cast<std::size_t>(s)] = 0;
        for (std::size_t h = 0; h < q.size(); ++h) {
            const int v = q[h];
            for (int w : adj[static_cast<std::size_t>(v)])
                if (!done[static_cast<std::size_t>(w)] && level[static_cast<std::size_t>(w)] < 0) {
                    level[static_cast<std::size_t>(w)] = level[static_cast<std::size_t>(v)] + 1;
                    q.push_back(w);
                }
        }
        ecc = level[static_cast<std::size_t>(q.back())];
        int best = -1;
        for (int v : q)
            if (level[static_cast<std::size_t>(v)] == ecc && (best < 0 || deg(v) < deg(best) || (deg(v) == deg(best) && v < best)))
                best = v;
        for (int v : q) level[static_cast<std::size_t>(v)] = -1;
        return best;
    };
    std::vector<int> by_deg(static_cast<std::size_t>(n));
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg(a) < deg(b); });
    std::vector<int> nb;
    for (int s0 : by_deg) {
        if (done[static_cast<std::size_t>(s0)]) continue;
        int ecc = 0, s = s0;
        int cand = far_node(s, ecc);
        for (int it = 0; it < 6; ++it) {
            int ecc2 = 0;
            const int nxt = far_node(cand, ecc2);
            if (ecc2 <= ecc) break;
            ecc = ecc2;
            s = cand;
            cand = nxt;
        }
        s = cand;
        const std::size_t start = order.size();
        order.push_back(s);
        done[static_cast<std::size_t>(s)] = 1;
        for (std::size_t h = start; h < order.size(); ++h) {
            nb.clear();
            for (int w : adj[static_cast<std::size_t>(order[h])])
                if (!done[static_cast<std::size_t>(w)]) nb.push_back(w);
            std::sort(nb.begin(), nb.end(), [&](int a, int b) { return deg(a) != deg(b) ? deg(a) < deg(b) : a < b; });
            for (int w : nb) {
                done[static_cast<std::size_t>(w)] = 1;
                order.push_back(w);
            }
        }
    }
    std::reverse(order.begin(), order.end());
    return order;
}

HostSub analyse(const cpddg_local_desc& d, int n_global) {
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
    std::vector<std::vector<int>> adj(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = d.col[k];
            if (c >= n || c == r) continue;
            adj[static_cast<std::size_t>(r)].push_back(c);
            adj[static_cast<std::size_t>(c)].push_back(r);
        }
    for (auto& a : adj) {
        std::sort(a.begin(), a.end());
        a.erase(std::unique(a.begin(), a.end()), a.end());
    }
    const std::vector<int> perm = rcm(adj);
    std::vector<int> inv(static_cast<std::size_t>(n));
    for (int k = 0; k < n; ++k) inv[static_cast<std::size_t>(perm[static_cast<std::size_t>(k)])] = k;
    S.first.assign(static_cast<std::size_t>(n), 0);
    for (int o = 0; o < n; ++o) {
        const int i = inv[static_cast<std::size_t>(o)];
        int f = i;
        for (int w : adj[static_cast<std::size_t>(o)]) f = std::min(f, inv[static_cast<std::size_t>(w)]);
        S.first[static_cast<std::size_t>(i)] = f;
    }
    S.roff.assign(static_cast<std::size_t>(n) + 1, 0);
    for (int i = 0; i < n; ++i) S.roff[static_cast<std::size_t>(i) + 1] = S.roff[static_cast<std::size_t>(i)] + (i - S.first[static_cast<std::size_t>(i)]);
    std::vector<int> maxrow(static_cast<std::size_t>(n), -1);
    for (int i = 0; i < n; ++i) maxrow[static_cast<std::size_t>(S.first[static_cast<std::size_t>(i)])] = std::max(maxrow[static_cast<std::size_t>(S.first[static_cast<std::size_t>(i)])], i);
    S.rlast.assign(static_cast<std::size_t>(n), 0);
    int run = -1;
    for (int i = 0; i < n; ++i) {
        run = std::max(run, maxrow[static_cast<std::size_t>(i)]);
        S.rlast[static_cast<std::size_t>(i)] = std::max(run, i);
    }
    const std::size_t ne = static_cast<std::size_t>(S.roff[static_cast<std::size_t>(n)]);
    S.L.assign(ne, 0.0);
    S.U.assign(ne, 0.0);
    S.diag.assign(static_cast<std::size_t>(n), 0.0);
    for (int r = 0; r < n; ++r)
        for (std::int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = d.col[k];
            if (c >= n) continue;  // eliminated Dirichlet closure column (z_b = 0)
            const int pi = inv[static_cast<std::size_t>(r)], pj = inv[static_cast<std::size_t>(c)];
            const double v = d.val[k];
            if (pi == pj)
                S.diag[static_cast<std::size_t>(pi)] += v;
            else if (pj < pi)
                S.L[static_cast<std::size_t>(S.roff[static_cast<std::size_t>(pi)] + (pj - S.first[static_cast<std::size_t>(pi)]))] += v;
            else
                S.U[static_cast<std::size_t>(S.roff[static_cast<std::size_t>(pj)] + (pi - S.first[static_cast<std::size_t>(pj)]))] += v;
        }
    S.gidx.assign(static_cast<std::size_t>(n), -1);
    S.sidx.assign(static_cast<std::size_t>(n), -1);
    for (int o = 0; o < std::min(n, d.n_overlap); ++o) {
        const int g = d.overlap[o];
        if (g < 0 || g >= n_global) throw InternalError("overlap index out of range");
        S.gidx[static_cast<std::size_t>(inv[static_cast<std::size_t>(o)])] = g;
    }
    for (int k = 0; k < d.n_scatter; ++k) {
        const int lo = d.scatter_local[k], g = d.scatter_global[k];
        if (lo < 0 || lo >= n || g < 0 || g >= n_global) throw InternalError("scatter index out of range");
        S.sidx[static_cast<std::size_t>(inv[static_cast<std::size_t>(lo)])] = g;
    }
    S.roff.pop_back();
    return S;
}

struct SubPtrs {
    int n;
    const int* first;
    const std::int64_t* roff;
    const int* rlast;
    double* diag;
    double* L;
    double* U;
};

__device__ __forceinline__ SubPtrs sub_ptrs(int j, const int* n_rows, const std::int64_t* vbase,
                                            const std::int64_t* ebase, const int* first,
                                            const std::int64_t* roff, const int* rlast, double* diag,
                                            double* L, double* U) {
    const std::int64_t vb = vbase[j], eb = ebase[j];
    return {n_rows[j], first + vb, roff + vb, rlast + vb, diag + vb, L + eb, U + eb};
}

// ------------------------------------------------------------ factorisation

constexpr int kFactorThreads = 256;
constexpr int kTS = TILE + 1;  // padded tile row stride (doubles) -- tiles are [NB][TILE+1]

__global__ void __launch_bounds__(kFactorThreads) k_factor(const int* __restrict__ order,
                                                           const int* __restrict__ n_rows,
                                                           const std::int64_t* __restrict__ vbase,
                                                           const std::int64_t* __restrict__ ebase,
                                                           const int* __restrict__ first_all,
                                                           const std::int64_t* __restrict__ roff_all,
                                                           const int* __restrict__ rlast_all,
                                                           double* diag_all, double* L_all, double* U_all,
                                                           int* status) {
    const int j = order[blockIdx.x];
    const SubPtrs S = sub_ptrs(j, n_rows, vbase, ebase, first_all, roff_all, rlast_all, diag_all, L_all, U_all);
    extern __shared__ double sm[];
    double* A11 = sm;                            // [NB][NB+1]
    double* Xi = A11 + NB * (NB + 1);            // [NB][TILE+1]: X rows of tile i, transposed (p-major)
    double* Yi = Xi + NB * kTS;
    double* Xj = Yi + NB * kTS;
    double* Yj = Xj + NB * kTS;
    const int tid = threadIdx.x;
    const int n = S.n;
    __shared__ int skip_tile;

    for (int k0 = 0; k0 < n; k0 += NB) {
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
                    const int f = S.first[gc];
                    if (gr >= f) v = S.U[S.roff[gc] + gr - f];
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
                const int f = S.first[gc];
                if (gr >= f) S.U[S.roff[gc] + gr - f] = v;
            }
        }
        // (3)+(4) panels: rows i in [k1, R]
        for (int i = k1 + tid; i <= R; i += blockDim.x) {
            const int f = S.first[i];
            if (f >= k1) continue;  // no entries in the panel columns
            const std::int64_t ro = S.roff[i] - f;
            double x[NB], u[NB];
#pragma unroll
            for (int p = 0; p < NB; ++p) {
                const int gc = k0 + p;
                const bool in = p < kb && gc >= f;
                x[p] = in ? S.L[ro + gc] : 0.0;
                u[p] = in ? S.U[ro + gc] : 0.0;
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
                if (p < kb && gc >= f) {
                    S.L[ro + gc] = x[p];
                    S.U[ro + gc] = u[p];
                }
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
                        if (i0 + q <= R) mi = min(mi, S.first[i0 + q]);
                        if (j0 + q <= R) mj = min(mj, S.first[j0 + q]);
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
                            const int f = S.first[gi];
                            if (gc >= f) {
                                xi = S.L[S.roff[gi] + gc - f];
                                yi = S.U[S.roff[gi] + gc - f];
                            }
                        }
                        if (gj <= R) {
                            const int f = S.first[gj];
                            if (gc >= f) {
                                xj = S.L[S.roff[gj] + gc - f];
                                yj = S.U[S.roff[gj] + gc - f];
                            }
                        }
                    }
                    Xi[p * kTS + r] = xi;
                    Yi[p * kTS + r] = yi;
                    Xj[p * kTS + r] = xj;
                    Yj[p * kTS + r] = yj;
                }
                __syncthreads();
                const int ty = tid / 16, tx = tid % 16;  // rows ty*4.., cols tx*4..
                double aL[4][4], aU[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) aL[a][b] = aU[a][b] = 0.0;
                for (int p = 0; p < kb; ++p) {
                    double xr[4], yr[4], yc[4], xc[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        xr[a] = Xi[p * kTS + ty * 4 + a];
                        yr[a] = Yi[p * kTS + ty * 4 + a];
                        yc[a] = Yj[p * kTS + tx * 4 + a];
                        xc[a] = Xj[p * kTS + tx * 4 + a];
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            aL[a][b] = fma(xr[a], yc[b], aL[a][b]);
                            aU[a][b] = fma(yr[a], xc[b], aU[a][b]);
                        }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int gi = i0 + ty * 4 + a;
                    if (gi > R) continue;
                    const int f = S.first[gi];
                    const std::int64_t ro = S.roff[gi] - f;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int gc = j0 + tx * 4 + b;
                        if (gc > R) continue;
                        if (gc < gi) {
                            if (gc >= f) {
                                S.L[ro + gc] -= aL[a][b];
                                S.U[ro + gc] -= aU[a][b];
                            }
                        } else if (gc == gi) {
                            S.diag[gi] -= aL[a][b];
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    // pivot check: a zero or non-finite pivot is a singular factorisation
    int bad = 0;
    for (int i = tid; i < n; i += blockDim.x) {
        const double d = S.diag[i];
        if (!(fabs(d) > 0.0) || !isfinite(d)) bad = 1;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) status[j] = bad;
}

// ---------------------------------------------------------------- solve

constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;

__global__ void __launch_bounds__(kSolveThreads) k_solve(const int* __restrict__ order,
                                                         const int* __restrict__ n_rows,
                                                         const std::int64_t* __restrict__ vbase,
                                                         const std::int64_t* __restrict__ ebase,
                                                         const int* __restrict__ first_all,
                                                         const std::int64_t* __restrict__ roff_all,
                                                         const double* __restrict__ diag_all,
                                                         const double* __restrict__ L_all,
                                                         const double* __restrict__ U_all,
                                                         const int* __restrict__ gidx_all,
                                                         const int* __restrict__ sidx_all,
                                                         const double* __restrict__ r, double* z,
                                                         int accumulate) {
    const int j = order[blockIdx.x];
    const int n = n_rows[j];
    const std::int64_t vb = vbase[j], eb = ebase[j];
    const int* first = first_all + vb;
    const std::int64_t* roff = roff_all + vb;
    const double* diag = diag_all + vb;
    const double* L = L_all + eb;
    const double* U = U_all + eb;
    extern __shared__ double y[];
    __shared__ double part[SB];
    __shared__ double tri[SB][SB + 1];
    __shared__ int sf[SB];
    __shared__ long long sro[SB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int p = tid; p < n; p += blockDim.x) {
        const int g = gidx_all[vb + p];
        y[p] = g >= 0 ? __ldg(r + g) : 0.0;
    }
    __syncthreads();

    // ---- forward: L y = b (unit lower), 32-row blocks
    for (int r0 = 0; r0 < n; r0 += SB) {
        const int rb = min(SB, n - r0);
        for (int rr = warp; rr < rb; rr += kSolveWarps) {
            const int i = r0 + rr;
            const int f = __ldg(first + i);
            const double* Li = L + (__ldg(roff + i) - f);
            double s = 0.0;
            for (int c = f + lane; c < r0; c += 32) s = fma(__ldg(Li + c), y[c], s);
            const int c = r0 + lane;
            tri[rr][lane] = (c >= f && c < i) ? __ldg(Li + c) : 0.0;
            s = warp_sum(s);
            if (lane == 0) part[rr] = s;
        }
        __syncthreads();
        if (warp == 0) {
            const int i = r0 + lane;
            double val = lane < rb ? y[i] - part[lane] : 0.0;
            for (int k = 0; k < rb; ++k) {
                const double xk = __shfl_sync(0xffffffffu, val, k);
                if (lane > k) val -= tri[lane][k] * xk;
            }
            if (lane < rb) y[i] = val;
        }
        __syncthreads();
    }

    // ---- backward: U x = y, U column i stored contiguously over [f_i, i)
    for (int c0 = ((n - 1) / SB) * SB; c0 >= 0; c0 -= SB) {
        const int cb = min(SB, n - c0);
        if (tid < SB) {
            sf[tid] = tid < cb ? __ldg(first + c0 + tid) : c0 + SB;
            sro[tid] = tid < cb ? __ldg(roff + c0 + tid) : 0;
        }
        __syncthreads();
        for (int e = tid; e < SB * SB; e += blockDim.x) {
            const int kk = e / SB, t = e % SB;  // tri[kk][t] = U(c0+t, c0+kk)
            double v = 0.0;
            if (kk < cb && t < kk && c0 + t >= sf[kk]) v = __ldg(U + sro[kk] + (c0 + t - sf[kk]));
            tri[kk][t] = v;
        }
        __syncthreads();
        if (warp == 0) {
            double val = lane < cb ? y[c0 + lane] : 0.0;
            for (int kk = cb - 1; kk >= 0; --kk) {
                if (lane == kk) val = val / __ldg(diag + c0 + kk);
                const double xk = __shfl_sync(0xffffffffu, val, kk);
                if (lane < kk) val -= tri[kk][lane] * xk;
            }
            if (lane < cb) y[c0 + lane] = val;
        }
        __syncthreads();
        int fmin = c0;
        for (int kk = 0; kk < cb; ++kk) fmin = min(fmin, sf[kk]);
        for (int jc = fmin + tid; jc < c0; jc += blockDim.x) {
            double acc = 0.0;
#pragma unroll 8
            for (int kk = 0; kk < cb; ++kk)
                if (jc >= sf[kk]) acc = fma(__ldg(U + sro[kk] + (jc - sf[kk])), y[c0 + kk], acc);
            y[jc] -= acc;
        }
        __syncthreads();
    }

    for (int p = tid; p < n; p += blockDim.x) {
        const int s = sidx_all[vb + p];
        if (s >= 0) z[s] = accumulate ? z[s] + y[p] : y[p];
    }
}

template <class T>
void append(std::vector<T>& dst, const std::vector<T>& src) {
    dst.insert(dst.end(), src.begin(), src.end());
}

}  // namespace

void pc_apply(const cpddg_pc* pc, const double* r, double* z, bool accumulate, cudaStream_t st) {
    k_solve<<<pc->n_sub, kSolveThreads, pc->solve_smem, st>>>(
        pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(), pc->first.get(), pc->roff.get(),
        pc->diag.get(), pc->L.get(), pc->U.get(), pc->gidx.get(), pc->sidx.get(), r, z, accumulate ? 1 : 0);
    CPDDG_CUDA(cudaGetLastError());
}

static cpddg_pc* pc_build(int n_global, int n_sub, const cpddg_local_desc* locals, const cpddg_pc_options* opt) {
    if (n_global <= 0 || n_sub <= 0 || !locals) throw InternalError("empty preconditioner");
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<HostSub> subs(static_cast<std::size_t>(n_sub));
    parallel_for(n_sub, opt ? opt->workers : 0,
                 [&](int j, int) { subs[static_cast<std::size_t>(j)] = analyse(locals[j], n_global); });
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
    std::vector<int> n_rows, first, rlast, gidx, sidx;
    std::vector<std::int64_t> vbase, ebase, roff;
    std::vector<double> L, U, diag;
    std::int64_t vb = 0, ebs = 0;
    for (auto& S : subs) {
        n_rows.push_back(S.n);
        vbase.push_back(vb);
        ebase.push_back(ebs);
        vb += S.n;
        ebs += static_cast<std::int64_t>(S.L.size());
        pc->max_rows = std::max(pc->max_rows, S.n);
        pc->n_reduced += S.reduced ? 1 : 0;
    }
    pc->rows_total = vb;
    pc->entries = 2 * ebs + vb;
    first.reserve(static_cast<std::size_t>(vb));
    L.reserve(static_cast<std::size_t>(ebs));
    U.reserve(static_cast<std::size_t>(ebs));
    for (auto& S : subs) {
        append(first, S.first);
        append(rlast, S.rlast);
        append(gidx, S.gidx);
        append(sidx, S.sidx);
        append(roff, S.roff);
        append(diag, S.diag);
        append(L, S.L);
        append(U, S.U);
        S = HostSub{};
    }
    std::vector<int> order(static_cast<std::size_t>(n_sub));
    std::iota(order.begin(), order.end(), 0);
    {
        std::vector<std::int64_t> cost(static_cast<std::size_t>(n_sub));
        for (int j = 0; j < n_sub; ++j)
            cost[static_cast<std::size_t>(j)] = (j + 1 < n_sub ? ebase[static_cast<std::size_t>(j) + 1] : ebs) - ebase[static_cast<std::size_t>(j)];
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[static_cast<std::size_t>(a)] > cost[static_cast<std::size_t>(b)]; });
    }
    pc->n_rows.upload(n_rows);
    pc->vbase.upload(vbase);
    pc->ebase.upload(ebase);
    pc->order.upload(order);
    pc->first.upload(first);
    pc->roff.upload(roff);
    pc->rlast.upload(rlast);
    pc->gidx.upload(gidx);
    pc->sidx.upload(sidx);
    pc->diag.upload(diag);
    pc->L.upload(L);
    pc->U.upload(U);
    const auto t1 = std::chrono::steady_clock::now();
    pc->analyse_seconds = std::chrono::duration<double>(t1 - t0).count();

    // device factorisation
    const int fsm = static_cast<int>(sizeof(double)) * (NB * (NB + 1) + 4 * NB * kTS);
    CPDDG_CUDA(cudaFuncSetAttribute(k_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm));
    DevBuf<int> status(static_cast<std::size_t>(n_sub));
    status.zero();
    cudaEvent_t e0, e1;
    CPDDG_CUDA(cudaEventCreate(&e0));
    CPDDG_CUDA(cudaEventCreate(&e1));
    CPDDG_CUDA(cudaEventRecord(e0));
    k_factor<<<n_sub, kFactorThreads, fsm>>>(pc->order.get(), pc->n_rows.get(), pc->vbase.get(), pc->ebase.get(),
                                           pc->first.get(), pc->roff.get(), pc->rlast.get(), pc->diag.get(),
                                           pc->L.get(), pc->U.get(), status.get());
    CPDDG_CUDA(cudaGetLastError());
    CPDDG_CUDA(cudaEventRecord(e1));
    CPDDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    CPDDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    pc->factor_seconds = ms * 1e-3;
    std::vector<int> st(static_cast<std::size_t>(n_sub));
    CPDDG_CUDA(cudaMemcpy(st.data(), status.get(), st.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int j = 0; j < n_sub; ++j)
        if (st[static_cast<std::size_t>(j)]) throw DivergenceError("singular factorization of subdomain " + std::to_string(j));

    pc->solve_smem = static_cast<int>(sizeof(double)) * pc->max_rows;
    if (pc->solve_smem > 200 * 1024) throw ConfigError("subdomain system too large for the shared-memory solve");
    CPDDG_CUDA(cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(pc->solve_smem, 1)));
    // bytes one apply streams: L, U, diag, first, roff per row, gather/scatter maps, r gathers, z writes
    pc->factor_bytes = 16 * ebs + 8 * vb;
    std::int64_t gathers = 0, scatters = 0;
    for (int g : gidx) gathers += g >= 0 ? 1 : 0;
    for (int s : sidx) scatters += s >= 0 ? 1 : 0;
    // B_pc = stored factor bytes + 12 |Sigma_j| (gather) + 12 N_A (scatter)
    pc->alg_bytes = pc->factor_bytes + 12 * gathers + 12 * scatters;
    return pc.release();
}

}  // namespace cpddg

using namespace cpddg;

extern "C" {

int cpddg_pc_create(int n_global, int n_sub, const cpddg_local_desc* locals, const cpddg_pc_options* opt,
                    cpddg_pc** out) {
    return guarded([&] {
        if (!out) throw InternalError("null argument");
        *out = pc_build(n_global, n_sub, locals, opt);
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
        *out = pc_build(n_global, static_cast<int>(d.size()), d.data(), opt);
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
        st->factor_bytes = pc->factor_bytes;
        st->algorithmic_bytes = pc->alg_bytes;
        st->max_rows = pc->max_rows;
        st->factor_seconds = pc->factor_seconds;
        st->analyse_seconds = pc->analyse_seconds;
        st->max_probe_residual = pc->max_probe_residual;
    });
}

int cpddg_pc_destroy(cpddg_pc* pc) {
    delete pc;
    return CPDDG_OK;
}

}  // extern "C"
