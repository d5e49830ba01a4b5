// Fill-reducing orderings of a local system's symmetric pattern for the
// envelope (profile) LU of csrc/cuda/pc.cu.  The reference factors with Eigen
// SparseLU + COLAMD (direct.hpp:36-52); the device LU keeps its fill inside
// the row / column envelopes, so the ordering's profile is the number of
// factor entries every preconditioner apply streams.
#pragma once

#include <algorithm>
#include <numeric>
#include <vector>

namespace cpddg {

/** Symmetric pattern in CSR form: neighbours of v are adj[xadj[v] .. xadj[v+1]), sorted. */
struct Graph {
    std::vector<int> xadj, adj;
    int size() const { return static_cast<int>(xadj.size()) - 1; }
    const int* begin(int v) const { return adj.data() + xadj[static_cast<std::size_t>(v)]; }
    const int* end(int v) const { return adj.data() + xadj[static_cast<std::size_t>(v) + 1]; }
    int degree(int v) const { return xadj[static_cast<std::size_t>(v) + 1] - xadj[static_cast<std::size_t>(v)]; }
};

namespace ordering_detail {

/** BFS over the not-yet-numbered nodes from s: fills level[] for the nodes
 *  reached (the caller resets them through `reached`), returns the
 *  eccentricity and the min-degree node of the last level. */
inline int bfs_far(const Graph& g, const std::vector<char>& done, int s, std::vector<int>& level,
                   std::vector<int>& reached, int& ecc) {
    reached.assign(1, s);
    level[static_cast<std::size_t>(s)] = 0;
    for (std::size_t h = 0; h < reached.size(); ++h) {
        const int v = reached[h];
        for (const int* pw = g.begin(v); pw != g.end(v); ++pw)
            if (const int w = *pw; !done[static_cast<std::size_t>(w)] && level[static_cast<std::size_t>(w)] < 0) {
                level[static_cast<std::size_t>(w)] = level[static_cast<std::size_t>(v)] + 1;
                reached.push_back(w);
            }
    }
    ecc = level[static_cast<std::size_t>(reached.back())];
    int best = -1;
    for (int v : reached)
        if (level[static_cast<std::size_t>(v)] == ecc &&
            (best < 0 || g.degree(v) < g.degree(best) || (g.degree(v) == g.degree(best) && v < best)))
            best = v;
    return best;
}

/** Pseudo-peripheral pair of s0's component (repeated BFS, min-degree node
 *  of the last level): returns the start node, `far` its antipode. */
inline int peripheral_pair(const Graph& g, const std::vector<char>& done, int s0, std::vector<int>& level,
                           std::vector<int>& reached, int& far) {
    int ecc = 0, s = s0;
    int cand = bfs_far(g, done, s, level, reached, ecc);
    for (int v : reached) level[static_cast<std::size_t>(v)] = -1;
    for (int it = 0; it < 6; ++it) {
        int ecc2 = 0;
        const int nxt = bfs_far(g, done, cand, level, reached, ecc2);
        for (int v : reached) level[static_cast<std::size_t>(v)] = -1;
        if (ecc2 <= ecc) break;
        ecc = ecc2;
        s = cand;
        cand = nxt;
    }
    far = s;
    return cand;
}

}  // namespace ordering_detail

/** Reverse Cuthill-McKee of a symmetric pattern (sorted, no diagonal).
 *  Components in order of their lowest-degree node; each starts at a
 *  pseudo-peripheral node; neighbours enqueued by (degree, index).
 *  Returns perm[new] = old. */
inline std::vector<int> rcm(const Graph& g) {
    const int n = g.size();
    std::vector<int> order;
    order.reserve(static_cast<std::size_t>(n));
    std::vector<char> done(static_cast<std::size_t>(n), 0);
    std::vector<int> level(static_cast<std::size_t>(n), -1), reached;
    auto deg = [&](int v) { return g.degree(v); };
    std::vector<int> by_deg(static_cast<std::size_t>(n));
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg(a) < deg(b); });
    std::vector<int> nb;
    for (int s0 : by_deg) {
        if (done[static_cast<std::size_t>(s0)]) continue;
        int far = 0;
        const int s = ordering_detail::peripheral_pair(g, done, s0, level, reached, far);
        const std::size_t start = order.size();
        order.push_back(s);
        done[static_cast<std::size_t>(s)] = 1;
        for (std::size_t h = start; h < order.size(); ++h) {
            nb.clear();
            for (const int* pw = g.begin(order[h]); pw != g.end(order[h]); ++pw)
                if (!done[static_cast<std::size_t>(*pw)]) nb.push_back(*pw);
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

/** Sloan's profile-reducing ordering (S. W. Sloan, IJNME 23 (1986), the
 *  published algorithm restated): per component a pseudo-peripheral pair
 *  (s, e); nodes are numbered from s by the priority
 *      P(v) = w1 * dist(v, e) - w2 * (current degree of v + 1),
 *  where the current degree counts the neighbours that are neither numbered
 *  nor in the front; numbering a node makes its neighbours active and their
 *  neighbours preactive.  The candidate with the highest priority is taken by
 *  a linear scan (ties: lowest index), so the result is deterministic.
 *  Returns perm[new] = old (numbered forward: row envelopes [first_i, i)
 *  follow the front). */
inline std::vector<int> sloan(const Graph& g, int w1, int w2) {
    const int n = g.size();
    std::vector<int> order;
    order.reserve(static_cast<std::size_t>(n));
    enum : char { INACTIVE = 0, PREACTIVE = 1, ACTIVE = 2, NUMBERED = 3 };
    std::vector<char> status(static_cast<std::size_t>(n), INACTIVE), done(static_cast<std::size_t>(n), 0);
    std::vector<int> level(static_cast<std::size_t>(n), -1), reached, cand;
    std::vector<long long> prio(static_cast<std::size_t>(n), 0);
    std::vector<int> by_deg(static_cast<std::size_t>(n));
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return g.degree(a) < g.degree(b); });
    for (int s0 : by_deg) {
        if (done[static_cast<std::size_t>(s0)]) continue;
        int e = 0, ecc = 0;
        const int s = ordering_detail::peripheral_pair(g, done, s0, level, reached, e);
        ordering_detail::bfs_far(g, done, e, level, reached, ecc);  // level = dist(., e) over the component
        for (int v : reached)
            prio[static_cast<std::size_t>(v)] =
                static_cast<long long>(w1) * level[static_cast<std::size_t>(v)] - static_cast<long long>(w2) * (g.degree(v) + 1);
        const std::vector<int> comp = reached;
        cand.assign(1, s);
        status[static_cast<std::size_t>(s)] = PREACTIVE;
        while (!cand.empty()) {
            std::size_t bi = 0;
            for (std::size_t k = 1; k < cand.size(); ++k) {
                const int a = cand[k], b = cand[bi];
                if (prio[static_cast<std::size_t>(a)] > prio[static_cast<std::size_t>(b)] ||
                    (prio[static_cast<std::size_t>(a)] == prio[static_cast<std::size_t>(b)] && a < b))
                    bi = k;
            }
            const int v = cand[bi];
            cand[bi] = cand.back();
            cand.pop_back();
            if (status[static_cast<std::size_t>(v)] == PREACTIVE)
                for (const int* pw = g.begin(v); pw != g.end(v); ++pw) {
                    const int w = *pw;
                    prio[static_cast<std::size_t>(w)] += w2;
                    if (status[static_cast<std::size_t>(w)] == INACTIVE) {
                        status[static_cast<std::size_t>(w)] = PREACTIVE;
                        cand.push_back(w);
                    }
                }
            status[static_cast<std::size_t>(v)] = NUMBERED;
            done[static_cast<std::size_t>(v)] = 1;
            order.push_back(v);
            for (const int* pw = g.begin(v); pw != g.end(v); ++pw) {
                const int w = *pw;
                if (status[static_cast<std::size_t>(w)] != PREACTIVE) continue;
                status[static_cast<std::size_t>(w)] = ACTIVE;
                prio[static_cast<std::size_t>(w)] += w2;
                for (const int* px = g.begin(w); px != g.end(w); ++px) {
                    const int x = *px;
                    if (status[static_cast<std::size_t>(x)] == NUMBERED) continue;
                    prio[static_cast<std::size_t>(x)] += w2;
                    if (status[static_cast<std::size_t>(x)] == INACTIVE) {
                        status[static_cast<std::size_t>(x)] = PREACTIVE;
                        cand.push_back(x);
                    }
                }
            }
        }
        for (int v : comp) level[static_cast<std::size_t>(v)] = -1;
    }
    return order;
}

}  // namespace cpddg
