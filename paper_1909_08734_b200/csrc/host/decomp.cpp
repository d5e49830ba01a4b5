// Assembled operators and the subdomain machinery (see decomp.hpp).
#include "decomp.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <string>
#include <thread>

namespace cpddg {

void Csr::append_row(std::vector<std::pair<int, double>>& scratch) {
    std::sort(scratch.begin(), scratch.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    for (std::size_t k = 0; k < scratch.size(); ++k) {
        const auto& [c, v] = scratch[k];
        if (c < 0 || c >= cols) throw InternalError("sparse: column out of range");
        if (k > 0 && scratch[k - 1].first == c)
            val.back() += v;
        else {
            col.push_back(c);
            val.push_back(v);
        }
    }
    ptr.push_back(static_cast<std::int64_t>(col.size()));
    scratch.clear();
}

int resolve_workers(int workers) {
    return workers > 0 ? workers : std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
}

void parallel_for(int n, int workers, const std::function<void(int, int)>& f) {
    if (n <= 0) return;
    const int nw = std::max(1, std::min(resolve_workers(workers), n));
    if (nw == 1) {
        for (int i = 0; i < n; ++i) f(i, 0);
        return;
    }
    std::atomic<int> next{0};
    std::exception_ptr err;
    std::mutex m;
    auto run = [&](int w) {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n) return;
            try {
                f(i, w);
            } catch (...) {
                std::lock_guard<std::mutex> lk(m);
                if (!err) err = std::current_exception();
                next.store(n);
            }
        }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < nw; ++w) th.emplace_back(run, w);
    run(0);
    for (auto& t : th) t.join();
    if (err) std::rethrow_exception(err);
}

namespace {

/** Rows [r0, r1) of a row-built matrix, assembled independently per chunk
 *  then concatenated in order (identical to serial append_row). */
struct RowChunk {
    std::vector<std::int64_t> len;
    std::vector<int> col;
    std::vector<double> val;
};

Csr concat_chunks(int rows, int cols, std::vector<RowChunk>& chunks) {
    Csr M;
    M.rows = rows;
    M.cols = cols;
    std::size_t nnz = 0;
    for (auto& c : chunks) nnz += c.col.size();
    M.ptr.reserve(static_cast<std::size_t>(rows) + 1);
    M.col.reserve(nnz);
    M.val.reserve(nnz);
    for (auto& c : chunks) {
        for (auto l : c.len) M.ptr.push_back(M.ptr.back() + l);
        M.col.insert(M.col.end(), c.col.begin(), c.col.end());
        M.val.insert(M.val.end(), c.val.begin(), c.val.end());
        c = RowChunk{};
    }
    return M;
}

template <class RowFn>
Csr build_rows(int rows, int cols, int workers, RowFn&& row_fn) {
    const int chunk = 4096;
    const int nchunks = (rows + chunk - 1) / chunk;
    std::vector<RowChunk> chunks(static_cast<std::size_t>(nchunks));
    parallel_for(nchunks, workers, [&](int c, int) {
        Csr local;
        local.rows = 0;
        local.cols = cols;
        std::vector<std::pair<int, double>> scratch;
        RowChunk& out = chunks[static_cast<std::size_t>(c)];
        const int r1 = std::min(rows, (c + 1) * chunk);
        for (int r = c * chunk; r < r1; ++r) {
            row_fn(r, scratch);
            const std::size_t before = local.col.size();
            local.append_row(scratch);
            out.len.push_back(static_cast<std::int64_t>(local.col.size() - before));
        }
        out.col = std::move(local.col);
        out.val = std::move(local.val);
    });
    return concat_chunks(rows, cols, chunks);
}

}  // namespace

// operators.hpp:30-51
template <int D>
Csr build_extension(const Band<D>& g, int workers) {
    const int na = g.n_active, total = g.n_band();
    const int pp = g.p + 1;
    int count = 1;
    for (int a = 0; a < D; ++a) count *= pp;
    return build_rows(total, na, workers, [&](int code, std::vector<std::pair<int, double>>& row) {
        const Stencil1D<D> s = stencil_of<D>(g.cp[static_cast<std::size_t>(code)], g.h, g.p);
        for (int k = 0; k < count; ++k) {
            Ix<D> q;
            double w = 1.0;
            int rem = k;
            for (int a = 0; a < D; ++a) {
                const int o = rem % pp;
                rem /= pp;
                q[a] = s.base[a] + o;
                w *= s.w[a][o];
            }
            const std::int64_t c = g.lookup(q);
            if (!g.is_active(c))
                throw InternalError("extension stencil node is not active: band closure violated");
            row.emplace_back(static_cast<int>(c), w);
        }
    });
}

// operators.hpp:79-112
template <int D>
Csr assemble_helmholtz(const Band<D>& g, const Csr& E, double c, int workers) {
    if (c <= 0) throw ConfigError("Helmholtz constant c must be positive");
    if (E.rows != g.n_band() || E.cols != g.n_active)
        throw InternalError("extension operator shape does not match the band");
    const double gamma = 2.0 * D / (g.h * g.h);
    const double ih2 = 1.0 / (g.h * g.h);
    return build_rows(g.n_active, g.n_active, workers,
                      [&](int i, std::vector<std::pair<int, double>>& row) {
                          row.emplace_back(i, c + gamma);
                          Ix<D> nbr[2 * D];
                          neighbors_of<D>(g.ix[static_cast<std::size_t>(i)], nbr);
                          for (int k = 0; k < 2 * D; ++k) {
                              const std::int64_t code = g.lookup(nbr[k]);
                              if (code < 0)
                                  throw InternalError("finite-difference neighbor missing from band");
                              for (std::int64_t m = E.ptr[static_cast<std::size_t>(code)];
                                   m < E.ptr[static_cast<std::size_t>(code) + 1]; ++m)
                                  row.emplace_back(E.col[static_cast<std::size_t>(m)],
                                                   -ih2 * E.val[static_cast<std::size_t>(m)]);
                          }
                      });
}

int validate_partition(const std::vector<int>& part, int n_active) {
    if (static_cast<int>(part.size()) != n_active)
        throw ConfigError("partition file has " + std::to_string(part.size()) +
                          " entries but the mesh has " + std::to_string(n_active) +
                          " active nodes");
    int mx = -1;
    for (int v : part) {
        if (v < 0) throw ConfigError("partition file contains a negative label");
        mx = std::max(mx, v);
    }
    std::vector<char> present(static_cast<std::size_t>(mx + 1), 0);
    for (int v : part) present[static_cast<std::size_t>(v)] = 1;
    for (int q = 0; q <= mx; ++q)
        if (!present[static_cast<std::size_t>(q)])
            throw ConfigError("partition labels skip part " + std::to_string(q));
    return mx + 1;
}

// partition.hpp:474-508
template <int D>
int align_interfaces(const Band<D>& g, std::vector<int>& part, int interp_degree) {
    if (static_cast<int>(part.size()) != g.n_active)
        throw InternalError("partition size does not match grid");
    const int n_parts = *std::max_element(part.begin(), part.end()) + 1;
    int total = 0;
    Ix<D> around[2 * D];
    for (int sweep = 0; sweep < interp_degree + 1; ++sweep) {
        std::vector<std::pair<int, int>> moves;
        for (int i = 0; i < g.n_active; ++i) {
            bool iface = false;
            neighbors_of<D>(g.ix[static_cast<std::size_t>(i)], around);
            for (int k = 0; k < 2 * D; ++k) {
                const std::int64_t code = g.lookup(around[k]);
                if (g.is_active(code) && part[static_cast<std::size_t>(code)] != part[static_cast<std::size_t>(i)]) {
                    iface = true;
                    break;
                }
            }
            if (!iface) continue;
            const Ix<D> xbar = nearest_node<D>(g.cp[static_cast<std::size_t>(i)], g.h);
            const std::int64_t code = g.lookup(xbar);
            if (!g.is_active(code)) continue;
            if (part[static_cast<std::size_t>(code)] != part[static_cast<std::size_t>(i)])
                moves.emplace_back(i, part[static_cast<std::size_t>(code)]);
        }
        if (moves.empty()) break;
        for (const auto& [i, q] : moves) part[static_cast<std::size_t>(i)] = q;
        total += static_cast<int>(moves.size());
    }
    std::vector<int> cnt(static_cast<std::size_t>(n_parts), 0);
    for (int v : part) ++cnt[static_cast<std::size_t>(v)];
    for (int q = 0; q < n_parts; ++q)
        if (cnt[static_cast<std::size_t>(q)] == 0)
            throw ConfigError("interface alignment emptied part " + std::to_string(q) +
                              "; use fewer subdomains or a finer grid");
    return total;
}

// subdomain.hpp:59-79
template <int D>
std::vector<int> find_cross_points(const Band<D>& g, const std::vector<int>& part) {
    std::vector<int> cross;
    Ix<D> around[2 * D];
    for (int i = 0; i < g.n_active; ++i) {
        neighbors_of<D>(g.ix[static_cast<std::size_t>(i)], around);
        int sa = -1, sb = -1;
        for (int k = 0; k < 2 * D; ++k) {
            const std::int64_t code = g.lookup(around[k]);
            if (!g.is_active(code)) continue;
            const int q = part[static_cast<std::size_t>(code)];
            if (q == part[static_cast<std::size_t>(i)] || q == sa || q == sb) continue;
            if (sa < 0)
                sa = q;
            else
                sb = q;
        }
        if (sb >= 0) cross.push_back(i);
    }
    return cross;
}

namespace {

template <int D>
std::uint64_t bin_key(const Vec<D>& q, double cell, const int* off = nullptr) {
    Ix<D> b;
    for (int a = 0; a < D; ++a) b[a] = static_cast<int>(std::floor(q[a] / cell)) + (off ? off[a] : 0);
    return LatticeMap::pack(b.data(), D);
}

/** Uniform bins of points: bin key -> point ids in insertion order. */
template <int D>
struct Bins {
    double cell = 1.0;
    LatticeMap head;                 // key -> slot in `lists`
    std::vector<std::vector<int>> lists;
    void build(const std::vector<Vec<D>>& pts, double c) {
        cell = c;
        head.clear();
        lists.clear();
        head.reserve(pts.size());
        for (int k = 0; k < static_cast<int>(pts.size()); ++k) {
            const std::uint64_t key = bin_key<D>(pts[static_cast<std::size_t>(k)], cell);
            std::int64_t s = head.find(key);
            if (s < 0) {
                s = static_cast<std::int64_t>(lists.size());
                head.insert(key, s);
                lists.emplace_back();
            }
            lists[static_cast<std::size_t>(s)].push_back(k);
        }
    }
    /** Call f(k) for every point in the 3^D bins around x (odometer order,
     *  axis 0 fastest, as LambdaIndex::query, subdomain.hpp:104-128). */
    template <class F>
    void around(const Vec<D>& x, F&& f) const {
        int off[D];
        for (int a = 0; a < D; ++a) off[a] = -1;
        for (;;) {
            const std::int64_t s = head.find(bin_key<D>(x, cell, off));
            if (s >= 0)
                for (int k : lists[static_cast<std::size_t>(s)]) f(k);
            int a = 0;
            while (a < D && off[a] == 1) off[a++] = -1;
            if (a == D) break;
            ++off[a];
        }
    }
};

}  // namespace

// subdomain.hpp:153-313
template <int D>
std::vector<Subdomain<D>> build_subdomains(const Band<D>& g, const Surface<D>& surface,
                                           const std::vector<int>& part, const Csr& E,
                                           int n_overlap, bool robin_ring, int workers) {
    if (n_overlap < 1) throw ConfigError("overlap width must be at least 1 layer");
    if (static_cast<int>(part.size()) != g.n_active)
        throw InternalError("partition size does not match grid");
    const int n_parts = *std::max_element(part.begin(), part.end()) + 1;
    const double anchor_radius = stencil_reach<D>(g.h, g.p) + g.h;

    const std::vector<int> cross = find_cross_points<D>(g, part);
    std::vector<Vec<D>> cross_x;
    cross_x.reserve(cross.size());
    for (int i : cross) cross_x.push_back(g.x(i));
    const double cross_radius = 2.0 * n_overlap * g.h;
    Bins<D> cross_bins;
    cross_bins.build(cross_x, cross_radius);

    std::vector<std::vector<int>> owned(static_cast<std::size_t>(n_parts));
    for (int i = 0; i < g.n_active; ++i) owned[static_cast<std::size_t>(part[static_cast<std::size_t>(i)])].push_back(i);

    std::vector<Subdomain<D>> subs(static_cast<std::size_t>(n_parts));
    const int nthreads = resolve_workers(workers);
    struct Scratch {
        std::vector<int> ov, bc, gh;  // generation stamps per band code
        int gen = 0;
    };
    std::vector<Scratch> scratch(static_cast<std::size_t>(nthreads));

    parallel_for(n_parts, nthreads, [&](int j, int w) {
        Scratch& sc = scratch[static_cast<std::size_t>(w)];
        if (sc.ov.empty()) {
            sc.ov.assign(static_cast<std::size_t>(g.n_band()), 0);
            sc.bc.assign(static_cast<std::size_t>(g.n_band()), 0);
            sc.gh.assign(static_cast<std::size_t>(g.n_band()), 0);
        }
        const int gen = ++sc.gen;
        auto in_ov = [&](std::int64_t c) { return sc.ov[static_cast<std::size_t>(c)] == gen; };
        auto in_bc = [&](std::int64_t c) { return sc.bc[static_cast<std::size_t>(c)] == gen; };

        Subdomain<D>& S = subs[static_cast<std::size_t>(j)];
        S.id = j;
        S.disjoint = owned[static_cast<std::size_t>(j)];
        Ix<D> around[2 * D];

        // ---- overlap: N_O breadth-first layers over active axis neighbours
        std::vector<int> members = S.disjoint;
        for (int i : S.disjoint) sc.ov[static_cast<std::size_t>(i)] = gen;
        std::vector<int> frontier = S.disjoint, last_layer;
        for (int layer = 0; layer < n_overlap; ++layer) {
            std::vector<int> next;
            for (int i : frontier) {
                neighbors_of<D>(g.ix[static_cast<std::size_t>(i)], around);
                for (int k = 0; k < 2 * D; ++k) {
                    const std::int64_t code = g.lookup(around[k]);
                    if (!g.is_active(code)) continue;
                    if (!in_ov(code)) {
                        sc.ov[static_cast<std::size_t>(code)] = gen;
                        next.push_back(static_cast<int>(code));
                        members.push_back(static_cast<int>(code));
                    }
                }
            }
            if (!next.empty()) last_layer = next;
            frontier = std::move(next);
            if (frontier.empty()) break;
        }
        std::sort(members.begin(), members.end());
        S.overlap = std::move(members);
        std::sort(last_layer.begin(), last_layer.end());
        S.final_layer = std::move(last_layer);

        // ---- ghosts adjacent to the overlap, FD-completion actives
        std::vector<int> ghost_list, bc_list, fd;
        for (int i : S.overlap) {
            neighbors_of<D>(g.ix[static_cast<std::size_t>(i)], around);
            for (int k = 0; k < 2 * D; ++k) {
                const std::int64_t code = g.lookup(around[k]);
                if (code < 0) throw InternalError("band closure missed a neighbour");
                if (g.is_active(code)) {
                    if (!in_ov(code) && !in_bc(code)) {
                        sc.bc[static_cast<std::size_t>(code)] = gen;
                        bc_list.push_back(static_cast<int>(code));
                        fd.push_back(static_cast<int>(code));
                    }
                } else if (sc.gh[static_cast<std::size_t>(code)] != gen) {
                    sc.gh[static_cast<std::size_t>(code)] = gen;
                    ghost_list.push_back(static_cast<int>(code));
                }
            }
        }
        // ---- extension-row references of overlap rows, ghosts, FD completion
        auto add_row_refs = [&](int code) {
            for (std::int64_t m = E.ptr[static_cast<std::size_t>(code)]; m < E.ptr[static_cast<std::size_t>(code) + 1]; ++m) {
                const int col = E.col[static_cast<std::size_t>(m)];
                if (!in_ov(col) && !in_bc(col)) {
                    sc.bc[static_cast<std::size_t>(col)] = gen;
                    bc_list.push_back(col);
                }
            }
        };
        for (int i : S.overlap) add_row_refs(i);
        for (int q : ghost_list) add_row_refs(q);
        for (int b : fd) add_row_refs(b);
        std::sort(ghost_list.begin(), ghost_list.end());
        S.ghosts = ghost_list;

        S.bc.reserve(bc_list.size());
        for (int b : bc_list) {
            BoundaryNode<D> node;
            node.ix = g.ix[static_cast<std::size_t>(b)];
            node.x = g.x(b);
            node.global_active = b;
            node.cp = g.cp[static_cast<std::size_t>(b)];
            S.bc.push_back(node);
        }

        // ---- ghost-type ring around the BC actives (Robin only)
        if (robin_ring) {
            LatticeMap ring_seen;
            ring_seen.reserve(bc_list.size());
            std::vector<BoundaryNode<D>> ring;
            for (int b : bc_list) {
                neighbors_of<D>(g.ix[static_cast<std::size_t>(b)], around);
                for (int k = 0; k < 2 * D; ++k) {
                    const std::int64_t code = g.lookup(around[k]);
                    if (g.is_active(code) && (in_ov(code) || in_bc(code))) continue;
                    if (code >= 0 && !g.is_active(code) && sc.gh[static_cast<std::size_t>(code)] == gen) continue;
                    if (!ring_seen.insert(LatticeMap::pack(around[k].data(), D), 0)) continue;
                    BoundaryNode<D> node;
                    node.ix = around[k];
                    node.is_ghost_type = true;
                    if (code >= 0) {
                        node.x = g.x(code);
                        node.cp = g.cp[static_cast<std::size_t>(code)];
                        node.global_active = g.is_active(code) ? static_cast<int>(code) : -1;
                    } else {
                        node.x = index_to_point<D>(around[k], g.h);
                        node.cp = surface.closest_point(node.x).cp;
                    }
                    ring.push_back(node);
                }
            }
            S.bc.insert(S.bc.end(), ring.begin(), ring.end());
        }
        std::sort(S.bc.begin(), S.bc.end(),
                  [](const BoundaryNode<D>& a, const BoundaryNode<D>& b) { return a.ix < b.ix; });

        // ---- interface anchors: closest points of the final overlap layer
        std::vector<Vec<D>> pts, nrms;
        pts.reserve(S.final_layer.size());
        for (int i : S.final_layer) {
            pts.push_back(g.cp[static_cast<std::size_t>(i)]);
            nrms.push_back(g.normal[static_cast<std::size_t>(i)]);
        }
        S.n_lambda = static_cast<int>(pts.size());
        if (!S.bc.empty() && pts.empty())
            throw InternalError("subdomain has boundary nodes but no interface anchors");
        Bins<D> lam;
        lam.build(pts, anchor_radius);
        const double excl = 1e-12 * g.h;
        for (BoundaryNode<D>& node : S.bc) {
            int best = -1;
            double bd = anchor_radius;
            lam.around(node.x, [&](int k) {
                const double d = norm<D>(sub<D>(pts[static_cast<std::size_t>(k)], node.x));
                if (d <= excl) return;
                if (d < bd || (d == bd && (best < 0 || k < best))) {
                    bd = d;
                    best = k;
                }
            });
            if (best < 0) {
                double gd = std::numeric_limits<double>::infinity();
                for (int k = 0; k < static_cast<int>(pts.size()); ++k) {
                    const double d = norm<D>(sub<D>(pts[static_cast<std::size_t>(k)], node.x));
                    if (d <= excl) continue;
                    if (d < gd) {
                        gd = d;
                        best = k;
                    }
                }
                node.fallback = true;
                ++S.fallback_count;
            }
            if (best < 0) throw InternalError("no usable interface anchor for a boundary node");
            node.cp_local = pts[static_cast<std::size_t>(best)];
            const Vec<D> dv = sub<D>(node.x, node.cp_local);
            const Vec<D>& nrm = nrms[static_cast<std::size_t>(best)];
            const double dn = dot<D>(dv, nrm);
            Vec<D> tang;
            for (int a = 0; a < D; ++a) tang[a] = dv[a] - dn * nrm[a];
            const double tn = norm<D>(tang);
            if (tn > 1e-12 * norm<D>(dv)) {
                node.conormal = divide<D>(tang, tn);
                node.dq = tn;
            }
            bool flag = false;
            cross_bins.around(node.x, [&](int k) {
                if (!flag && norm<D>(sub<D>(node.x, cross_x[static_cast<std::size_t>(k)])) <= cross_radius) flag = true;
            });
            node.cross_flagged = flag;
        }
    });
    return subs;
}

// transmission.hpp:73-138
template <int D>
LocalSystem assemble_local(const Band<D>& g, const Csr& A, const Subdomain<D>& S,
                           const TransmissionSpec& spec, std::vector<int>& colmap) {
    if (A.rows != g.n_active || A.cols != g.n_active)
        throw InternalError("global operator shape does not match the band");
    LocalSystem L;
    L.id = S.id;
    L.n_overlap = static_cast<int>(S.overlap.size());
    L.n_bc = static_cast<int>(S.bc.size());
    L.overlap = S.overlap;
    if (colmap.size() != static_cast<std::size_t>(g.n_active)) colmap.assign(static_cast<std::size_t>(g.n_active), -1);
    for (int k = 0; k < L.n_overlap; ++k) colmap[static_cast<std::size_t>(S.overlap[static_cast<std::size_t>(k)])] = k;
    for (int b = 0; b < L.n_bc; ++b)
        if (!S.bc[static_cast<std::size_t>(b)].is_ghost_type && S.bc[static_cast<std::size_t>(b)].global_active >= 0)
            colmap[static_cast<std::size_t>(S.bc[static_cast<std::size_t>(b)].global_active)] = L.n_overlap + b;
    auto local_col = [&](int a) {
        const int c = colmap[static_cast<std::size_t>(a)];
        if (c < 0) throw InternalError("subdomain closure missed an active reference");
        return c;
    };
    auto reset = [&] {
        for (int i : S.overlap) colmap[static_cast<std::size_t>(i)] = -1;
        for (const auto& b : S.bc)
            if (b.global_active >= 0) colmap[static_cast<std::size_t>(b.global_active)] = -1;
    };
    try {
        for (int i : S.disjoint) {
            L.scatter_local.push_back(local_col(i));
            L.scatter_global.push_back(i);
        }
        L.A.rows = L.A.cols = L.n_local();
        std::vector<std::pair<int, double>> row;
        for (int k = 0; k < L.n_overlap; ++k) {
            const int i = L.overlap[static_cast<std::size_t>(k)];
            for (std::int64_t m = A.ptr[static_cast<std::size_t>(i)]; m < A.ptr[static_cast<std::size_t>(i) + 1]; ++m)
                row.emplace_back(local_col(A.col[static_cast<std::size_t>(m)]), A.val[static_cast<std::size_t>(m)]);
            L.A.append_row(row);
        }
        const int pp = g.p + 1;
        int count = 1;
        for (int a = 0; a < D; ++a) count *= pp;
        for (int b = 0; b < L.n_bc; ++b) {
            const BoundaryNode<D>& node = S.bc[static_cast<std::size_t>(b)];
            row.emplace_back(L.n_overlap + b, 1.0);
            if (spec.robin) {
                if (node.dq < 0) throw InternalError("negative tangential offset");
                const double alpha = node.cross_flagged ? spec.alpha_cross : spec.alpha;
                const double s = 1.0 / (1.0 + alpha * node.dq);
                const Stencil1D<D> st = stencil_of<D>(node.cp_local, g.h, g.p);
                for (int k = 0; k < count; ++k) {
                    Ix<D> q;
                    double w = 1.0;
                    int rem = k;
                    for (int a = 0; a < D; ++a) {
                        const int o = rem % pp;
                        rem /= pp;
                        q[a] = st.base[a] + o;
                        w *= st.w[a][o];
                    }
                    const std::int64_t code = g.lookup(q);
                    if (!g.is_active(code))
                        throw InternalError("interface anchor stencil leaves the active set");
                    row.emplace_back(local_col(static_cast<int>(code)), -s * w);
                }
            }
            L.A.append_row(row);
        }
    } catch (...) {
        reset();
        throw;
    }
    reset();
    return L;
}

template <int D>
std::vector<LocalSystem> assemble_locals(const Band<D>& g, const Csr& A,
                                         const std::vector<Subdomain<D>>& subs,
                                         const TransmissionSpec& spec, int workers) {
    std::vector<LocalSystem> out(subs.size());
    const int nthreads = resolve_workers(workers);
    std::vector<std::vector<int>> maps(static_cast<std::size_t>(nthreads));
    parallel_for(static_cast<int>(subs.size()), nthreads, [&](int j, int w) {
        out[static_cast<std::size_t>(j)] =
            assemble_local<D>(g, A, subs[static_cast<std::size_t>(j)], spec, maps[static_cast<std::size_t>(w)]);
    });
    return out;
}

#define CPDDG_INST(D)                                                                              \
    template Csr build_extension<D>(const Band<D>&, int);                                          \
    template Csr assemble_helmholtz<D>(const Band<D>&, const Csr&, double, int);                   \
    template int align_interfaces<D>(const Band<D>&, std::vector<int>&, int);                      \
    template std::vector<int> find_cross_points<D>(const Band<D>&, const std::vector<int>&);       \
    template std::vector<Subdomain<D>> build_subdomains<D>(const Band<D>&, const Surface<D>&,      \
                                                           const std::vector<int>&, const Csr&,    \
                                                           int, bool, int);                        \
    template LocalSystem assemble_local<D>(const Band<D>&, const Csr&, const Subdomain<D>&,        \
                                           const TransmissionSpec&, std::vector<int>&);            \
    template std::vector<LocalSystem> assemble_locals<D>(const Band<D>&, const Csr&,               \
                                                         const std::vector<Subdomain<D>>&,         \
                                                         const TransmissionSpec&, int);
CPDDG_INST(2)
CPDDG_INST(3)

}  // namespace cpddg
