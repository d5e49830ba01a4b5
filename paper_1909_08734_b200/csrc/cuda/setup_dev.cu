// Device setup: the computational band with its
// closest points, interface alignment and the subdomain index sets, built on
// the GPU and bit-identical to the host restatement (csrc/host/band.cpp,
// decomp.cpp), which is itself bit-exact with the reference:
//
//   build_band_device   build_band_tube (band.hpp:150-182): level-synchronous
//                       flood fill from the node nearest the surface sample,
//                       closest points of a whole level per launch (circle,
//                       sphere, torus, TriMesh ring search), closure under CP
//                       stencils (band.hpp:124-142) in rounds, finalize
//                       (band.hpp:78-118): actives and ghosts sorted
//                       lexicographically by radix sort of the packed
//                       lattice key (its numeric order is the lexicographic
//                       order of the index).
//
// Sets are hash tables keyed by packed lattice index (dhash.cuh); set
// semantics make the results independent of thread scheduling, and every
// ordered output is produced by a sort.  Compiled with --fmad=false.
#include "../host/setup_dev.hpp"
#include "setup_dev.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

namespace cpddg {

struct DevMesh {
    DevBuf<double> verts, vert_n, face_n, edge_n;
    DevBuf<int> tris, cell_start, cell_tris;
    DevBuf<unsigned char> face_ok;
    DevHashTable cells;
};

namespace {

constexpr int kThr = 256;
inline int blocks_for(long long n) { return static_cast<int>(std::max(1LL, (n + kThr - 1) / kThr)); }

struct BandCounters {
    int n_act, n_next, n_ghost, overflow, err;
};

__global__ void k_mesh_cells(DHash cells, const unsigned long long* keys, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cells.insert(keys[i] + 1, i);
}

/** One BFS level (band.hpp:158-176): closest points of the level's nodes;
 *  accepted nodes (dist <= radius) join the active set and push their unseen
 *  axis neighbours onto the next level. */
template <int D>
__global__ void k_bfs_level(DSurf S, double h, double radius, int n_level, const std::uint64_t* __restrict__ level,
                            std::uint64_t* __restrict__ next, int cap, DHash seen, DHash act,
                            std::uint64_t* act_keys, double* act_cp, double* act_n, double* act_d,
                            BandCounters* cnt) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_level) return;
    const std::uint64_t key = level[q];
    int ix[D];
    lat_unpack<D>(key, ix);
    double x[D];
    d_point<D>(ix, h, x);
    const DCp<D> r = d_closest_point<D>(S, x, &cnt->err);
    if (r.dist > radius) return;
    const int pos = atomicAdd(&cnt->n_act, 1);
    if (pos >= cap) {
        cnt->overflow = 1;
        return;
    }
    act_keys[pos] = key;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        act_cp[static_cast<std::size_t>(pos) * D + a] = r.cp[a];
        act_n[static_cast<std::size_t>(pos) * D + a] = r.n[a];
    }
    act_d[pos] = r.dist;
    act.insert(key, pos);
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        int nb[D];
#pragma unroll
        for (int a = 0; a < D; ++a) nb[a] = ix[a];
        nb[k >> 1] += (k & 1) ? 1 : -1;
        const std::uint64_t nk = lat_pack<D>(nb);
        if (seen.insert(nk, 0)) {
            const int np = atomicAdd(&cnt->n_next, 1);
            if (np < cap)
                next[np] = nk;
            else
                cnt->overflow = 1;
        }
    }
}

/** Closure round (band.hpp:124-142): every stencil node of the CPs of actives
 *  [begin, end) that is not yet active joins the active set. */
template <int D>
__global__ void k_close(double h, int p, int begin, int end, int cap, DHash act, std::uint64_t* act_keys,
                        const double* __restrict__ act_cp, BandCounters* cnt) {
    const int w = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= end) return;
    int base[D];
#pragma unroll
    for (int a = 0; a < D; ++a) base[a] = d_stencil_base(act_cp[static_cast<std::size_t>(w) * D + a], h, p);
    const int pp = p + 1;
    int count = 1;
    for (int a = 0; a < D; ++a) count *= pp;
    for (int k = 0; k < count; ++k) {
        int q[D], rem = k;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            q[a] = base[a] + rem % pp;
            rem /= pp;
        }
        const std::uint64_t key = lat_pack<D>(q);
        if (act.contains(key)) continue;
        const int pos = act.insert_claim(key, &cnt->n_act);
        if (pos < 0) continue;
        if (pos >= cap)
            cnt->overflow = 1;
        else
            act_keys[pos] = key;
    }
}

/** Closest points of nodes [begin, end) of a key list (no acceptance test). */
template <int D>
__global__ void k_cp_keys(DSurf S, double h, int begin, int end, const std::uint64_t* __restrict__ keys, double* cp,
                          double* nrm, double* dist, BandCounters* cnt) {
    const int w = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= end) return;
    int ix[D];
    lat_unpack<D>(keys[w], ix);
    double x[D];
    d_point<D>(ix, h, x);
    const DCp<D> r = d_closest_point<D>(S, x, &cnt->err);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        cp[static_cast<std::size_t>(w) * D + a] = r.cp[a];
        nrm[static_cast<std::size_t>(w) * D + a] = r.n[a];
    }
    dist[w] = r.dist;
}

template <int D>
__global__ void k_gather_band(int n, const int* __restrict__ perm, const double* __restrict__ cp_in,
                              const double* __restrict__ n_in, const double* __restrict__ d_in, double* cp,
                              double* nrm, double* dist) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = perm[k];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        cp[static_cast<std::size_t>(k) * D + a] = cp_in[static_cast<std::size_t>(s) * D + a];
        nrm[static_cast<std::size_t>(k) * D + a] = n_in[static_cast<std::size_t>(s) * D + a];
    }
    dist[k] = d_in[s];
}

/** Ghosts (band.hpp:96-105): axis neighbours of actives that are not active. */
template <int D>
__global__ void k_ghosts(int na, const std::uint64_t* __restrict__ keys, DHash act, DHash gseen,
                         std::uint64_t* gkeys, int cap, BandCounters* cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int ix[D];
    lat_unpack<D>(keys[i], ix);
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        int nb[D];
#pragma unroll
        for (int a = 0; a < D; ++a) nb[a] = ix[a];
        nb[k >> 1] += (k & 1) ? 1 : -1;
        const std::uint64_t nk = lat_pack<D>(nb);
        if (act.contains(nk)) continue;
        if (gseen.insert(nk, 0)) {
            const int g = atomicAdd(&cnt->n_ghost, 1);
            if (g < cap)
                gkeys[g] = nk;
            else
                cnt->overflow = 1;
        }
    }
}

__global__ void k_iota(int n, int* v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

__global__ void k_map_insert(DHash map, const std::uint64_t* __restrict__ keys, int n, int offset) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) map.insert(keys[i], offset + i);
}

/** Radix sort of packed keys (numeric order = lexicographic order of the
 *  lattice index) with the permutation. */
void sort_keys(int n, int dim, const std::uint64_t* keys_in, std::uint64_t* keys_out, int* perm_out,
               cudaStream_t st) {
    DevBuf<int> iota(static_cast<std::size_t>(std::max(n, 1)));
    k_iota<<<blocks_for(n), kThr, 0, st>>>(n, iota.get());
    std::size_t tmp = 0;
    const int bits = 21 * dim;
    CPDDG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys_in, keys_out, iota.get(), perm_out, n, 0, bits, st));
    DevBuf<unsigned char> scratch(std::max<std::size_t>(tmp, 1));
    CPDDG_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(), tmp, keys_in, keys_out, iota.get(), perm_out, n, 0,
                                               bits, st));
}

template <class T>
std::vector<T> download(const T* p, std::size_t n, cudaStream_t st) {
    std::vector<T> h(n);
    if (n) CPDDG_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    CPDDG_CUDA(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

DSurf DevBand::surf() const {
    DSurf S;
    S.kind = kind;
    S.radius = radius;
    S.R = major_R;
    S.r = minor_r;
    if (mesh) {
        S.verts = mesh->verts.get();
        S.tris = mesh->tris.get();
        S.face_n = mesh->face_n.get();
        S.vert_n = mesh->vert_n.get();
        S.edge_n = mesh->edge_n.get();
        S.face_ok = mesh->face_ok.get();
        S.cells = mesh->cells.view();
        S.cell_start = mesh->cell_start.get();
        S.cell_tris = mesh->cell_tris.get();
        S.n_tris = n_tris;
        S.max_ring = max_ring;
        S.cell = cell;
    }
    return S;
}

DevBand::~DevBand() = default;
DevBand::DevBand() = default;

template <int D>
static void upload_surface(const Surface<D>& surface, DevBand& B) {
    B.kind = static_cast<int>(surface.kind);
    B.radius = surface.radius;
    B.major_R = surface.major_R;
    B.minor_r = surface.minor_r;
    if constexpr (D == 3) {
        if (surface.kind == SurfaceKind::trimesh) {
            const TriMeshTables T = surface.mesh->tables();
            B.mesh = std::make_unique<DevMesh>();
            DevMesh& M = *B.mesh;
            M.verts.upload(T.verts);
            M.vert_n.upload(T.vert_n);
            M.face_n.upload(T.face_n);
            M.edge_n.upload(T.edge_n);
            M.tris.upload(T.tris);
            M.face_ok.upload(T.face_ok);
            M.cell_start.upload(T.cell_start);
            M.cell_tris.upload(T.cell_tris);
            const int nc = static_cast<int>(T.cell_keys.size());
            M.cells.init(static_cast<std::size_t>(nc));
            DevBuf<unsigned long long> ck;
            std::vector<unsigned long long> keys(T.cell_keys.begin(), T.cell_keys.end());
            ck.upload(keys);
            k_mesh_cells<<<blocks_for(nc), kThr>>>(M.cells.view(), ck.get(), nc);
            CPDDG_CUDA(cudaGetLastError());
            CPDDG_CUDA(cudaDeviceSynchronize());
            B.n_tris = static_cast<int>(T.face_ok.size());
            B.max_ring = T.max_ring;
            B.cell = T.cell;
        }
    }
}

template <int D>
Band<D> build_band_device(const Surface<D>& surface, double h, int p, double tube_radius,
                          std::shared_ptr<DevBand>* keep) {
    if (h <= 0) throw ConfigError("grid spacing h must be positive");
    if (p < 1) throw ConfigError("interpolation degree must be at least 1");
    const auto t0 = std::chrono::steady_clock::now();
    auto B = std::make_shared<DevBand>();
    B->dim = D;
    B->h = h;
    B->p = p;
    upload_surface<D>(surface, *B);
    const DSurf S = B->surf();
    Band<D> g;
    g.h = h;
    g.p = p;
    g.tube_radius = tube_radius > 0 ? tube_radius : stencil_reach<D>(h, p);
    cudaStream_t st = nullptr;
    DevBuf<BandCounters> cnt(1);
    BandCounters hc{};
    const Ix<D> seed = nearest_node<D>(surface.sample_point(), h);
    const std::uint64_t seed_key = lat_pack<D>(seed.data());

    // flood fill + closure; restarted with twice the capacity on overflow
    int cap = 1 << 20;
    DevBuf<std::uint64_t> act_keys, lv[2];
    DevBuf<double> act_cp, act_n, act_d;
    DevHashTable seen, act;
    int levels = 0;
    for (;;) {
        act_keys.alloc(static_cast<std::size_t>(cap));
        lv[0].alloc(static_cast<std::size_t>(cap));
        lv[1].alloc(static_cast<std::size_t>(cap));
        act_cp.alloc(static_cast<std::size_t>(cap) * D);
        act_n.alloc(static_cast<std::size_t>(cap) * D);
        act_d.alloc(static_cast<std::size_t>(cap));
        seen.init(2 * static_cast<std::size_t>(cap), st);
        act.init(static_cast<std::size_t>(cap), st);
        CPDDG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(BandCounters), st));
        CPDDG_CUDA(cudaMemcpyAsync(lv[0].get(), &seed_key, sizeof(seed_key), cudaMemcpyHostToDevice, st));
        k_map_insert<<<1, 1, 0, st>>>(seen.view(), lv[0].get(), 1, 0);  // the seed is seen
        int n_level = 1, cur = 0;
        levels = 0;
        hc = BandCounters{};
        while (n_level > 0 && !hc.overflow) {
            CPDDG_CUDA(cudaMemsetAsync(&cnt.get()->n_next, 0, sizeof(int), st));
            k_bfs_level<D><<<blocks_for(n_level), kThr, 0, st>>>(S, h, g.tube_radius, n_level, lv[cur].get(),
                                                                  lv[cur ^ 1].get(), cap, seen.view(), act.view(),
                                                                  act_keys.get(), act_cp.get(), act_n.get(),
                                                                  act_d.get(), cnt.get());
            CPDDG_CUDA(cudaGetLastError());
            CPDDG_CUDA(cudaMemcpyAsync(&hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
            CPDDG_CUDA(cudaStreamSynchronize(st));
            n_level = std::min(hc.n_next, cap);
            cur ^= 1;
            ++levels;
        }
        if (!hc.overflow && hc.n_act > 0) {
            // closure rounds
            int begin = 0;
            while (begin < hc.n_act && !hc.overflow) {
                const int end = hc.n_act;
                k_close<D><<<blocks_for(end - begin), kThr, 0, st>>>(h, p, begin, end, cap, act.view(),
                                                                      act_keys.get(), act_cp.get(), cnt.get());
                CPDDG_CUDA(cudaMemcpyAsync(&hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
                CPDDG_CUDA(cudaStreamSynchronize(st));
                if (hc.overflow) break;
                if (hc.n_act > end)
                    k_cp_keys<D><<<blocks_for(hc.n_act - end), kThr, 0, st>>>(S, h, end, hc.n_act, act_keys.get(),
                                                                            act_cp.get(), act_n.get(), act_d.get(),
                                                                            cnt.get());
                CPDDG_CUDA(cudaGetLastError());
                begin = end;
            }
        }
        if (!hc.overflow) break;
        cap *= 2;
    }
    if (hc.err) throw InternalError("closest-point query found no triangle");
    if (hc.n_act == 0) throw ConfigError("band is empty: grid spacing too large for the surface");
    const int na = hc.n_act;

    // finalize: sorted actives, ghosts, sorted ghosts
    DevBuf<std::uint64_t> keys_sorted(static_cast<std::size_t>(na));
    DevBuf<int> perm(static_cast<std::size_t>(na));
    sort_keys(na, D, act_keys.get(), keys_sorted.get(), perm.get(), st);
    DevHashTable gseen;
    gseen.init(static_cast<std::size_t>(na), st);
    DevBuf<std::uint64_t> gkeys;
    int gcap = std::max(1024, na);
    for (;;) {
        gkeys.alloc(static_cast<std::size_t>(gcap));
        gseen.init(static_cast<std::size_t>(gcap), st);
        CPDDG_CUDA(cudaMemsetAsync(&cnt.get()->n_ghost, 0, sizeof(int), st));
        CPDDG_CUDA(cudaMemsetAsync(&cnt.get()->overflow, 0, sizeof(int), st));
        k_ghosts<D><<<blocks_for(na), kThr, 0, st>>>(na, keys_sorted.get(), act.view(), gseen.view(), gkeys.get(),
                                                      gcap, cnt.get());
        CPDDG_CUDA(cudaMemcpyAsync(&hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
        if (!hc.overflow) break;
        gcap *= 2;
    }
    const int ng = hc.n_ghost;
    const int nb = na + ng;
    B->keys.alloc(static_cast<std::size_t>(nb));
    B->cp.alloc(static_cast<std::size_t>(nb) * D);
    B->normal.alloc(static_cast<std::size_t>(nb) * D);
    B->dist.alloc(static_cast<std::size_t>(nb));
    CPDDG_CUDA(cudaMemcpyAsync(B->keys.get(), keys_sorted.get(), sizeof(std::uint64_t) * na, cudaMemcpyDeviceToDevice, st));
    k_gather_band<D><<<blocks_for(na), kThr, 0, st>>>(na, perm.get(), act_cp.get(), act_n.get(), act_d.get(),
                                                       B->cp.get(), B->normal.get(), B->dist.get());
    if (ng > 0) {
        DevBuf<int> gperm(static_cast<std::size_t>(ng));
        sort_keys(ng, D, gkeys.get(), B->keys.get() + na, gperm.get(), st);
        k_cp_keys<D><<<blocks_for(ng), kThr, 0, st>>>(S, h, na, nb, B->keys.get(), B->cp.get(), B->normal.get(),
                                                       B->dist.get(), cnt.get());
    }
    CPDDG_CUDA(cudaGetLastError());
    B->map.init(static_cast<std::size_t>(nb), st);
    k_map_insert<<<blocks_for(nb), kThr, 0, st>>>(B->map.view(), B->keys.get(), nb, 0);
    CPDDG_CUDA(cudaGetLastError());
    CPDDG_CUDA(cudaMemcpyAsync(&hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
    CPDDG_CUDA(cudaStreamSynchronize(st));
    if (hc.err) throw InternalError("closest-point query found no triangle");
    B->na = na;
    B->ng = ng;
    const auto t1 = std::chrono::steady_clock::now();

    // host copy of the band (the host setup -- E, A, local systems -- and the
    // operator tables consume it)
    const std::vector<std::uint64_t> hk = download(B->keys.get(), static_cast<std::size_t>(nb), st);
    const std::vector<double> hcp = download(B->cp.get(), static_cast<std::size_t>(nb) * D, st);
    const std::vector<double> hn = download(B->normal.get(), static_cast<std::size_t>(nb) * D, st);
    g.dist = download(B->dist.get(), static_cast<std::size_t>(nb), st);
    g.n_active = na;
    g.n_ghost = ng;
    g.ix.resize(static_cast<std::size_t>(nb));
    g.cp.resize(static_cast<std::size_t>(nb));
    g.normal.resize(static_cast<std::size_t>(nb));
    for (int k = 0; k < nb; ++k) {
        lat_unpack<D>(hk[static_cast<std::size_t>(k)], g.ix[static_cast<std::size_t>(k)].data());
        for (int a = 0; a < D; ++a) {
            g.cp[static_cast<std::size_t>(k)][a] = hcp[static_cast<std::size_t>(k) * D + a];
            g.normal[static_cast<std::size_t>(k)][a] = hn[static_cast<std::size_t>(k) * D + a];
        }
    }
    g.map.reserve(static_cast<std::size_t>(nb));
    for (int k = 0; k < nb; ++k) g.map.insert(hk[static_cast<std::size_t>(k)], static_cast<std::int64_t>(k));
    const double kappa = surface.curvature_bound();
    if (kappa > 0) {
        const double ghost_reach = g.tube_radius + std::sqrt(double(D)) * h;
        if (ghost_reach >= 1.0 / kappa) g.tube_radius_warning = true;
    }
    const auto t2 = std::chrono::steady_clock::now();
    B->levels = levels;
    B->device_seconds = std::chrono::duration<double>(t1 - t0).count();
    B->copy_seconds = std::chrono::duration<double>(t2 - t1).count();
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] device band: N_A %d N_G %d, %d BFS levels, device %.3f s, host copy %.3f s\n", na,
                     ng, levels, B->device_seconds, B->copy_seconds);
    if (keep) *keep = B;
    return g;
}

template Band<2> build_band_device<2>(const Surface<2>&, double, int, double, std::shared_ptr<DevBand>*);
template Band<3> build_band_device<3>(const Surface<3>&, double, int, double, std::shared_ptr<DevBand>*);

}  // namespace cpddg
