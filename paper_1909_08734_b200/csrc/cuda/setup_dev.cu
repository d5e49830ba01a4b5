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
//   decompose_device    align_interfaces (partition.hpp:474-508): p + 1
//                       simultaneous-move sweeps; find_cross_points
//                       (subdomain.hpp:59-79); build_subdomains
//                       (subdomain.hpp:153-313) for ALL subdomains at once:
//                       (subdomain, node) membership hash sets, N_O
//                       breadth-first overlap layers, FD completion and
//                       ghosts, extension-row references, the Robin ring
//                       (fresh closest points for non-band ring nodes),
//                       interface anchors (lexicographic (distance, index)
//                       minimum over the final layer, as the host's binned
//                       search with its tie rule) and cross flags (the
//                       host's cross-point bins).
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

// ------------------------------------------------------------ subdomain sets

namespace {

struct SetCounters {
    int moves, n_ov, n_bc, n_fd, n_gh, n_ring, overflow, err;
};

constexpr int kErrNbr = 1, kErrStencil = 2, kErrAnchor = 4, kErrRange = 8, kErrCp = 16;

__host__ __device__ __forceinline__ std::uint64_t pair_key(int j, int i) {
    return ((static_cast<std::uint64_t>(j) << 32) | static_cast<std::uint32_t>(i)) + 1;
}
__host__ __device__ __forceinline__ int pair_j(std::uint64_t k) { return static_cast<int>((k - 1) >> 32); }
__host__ __device__ __forceinline__ int pair_i(std::uint64_t k) { return static_cast<int>((k - 1) & 0xffffffffu); }

/** (subdomain, lattice index) key for the Robin ring and the BC sort: 10
 *  bits of subdomain, 18 bits per axis; numeric order = (j, lexicographic). */
template <int D>
__host__ __device__ __forceinline__ std::uint64_t ring_key(int j, const int* ix) {
    std::uint64_t k = static_cast<std::uint64_t>(j);
    for (int a = 0; a < 3; ++a) {
        const int v = a < D ? ix[a] : 0;
        k = (k << 18) | (static_cast<std::uint64_t>(static_cast<std::uint32_t>(v + (1 << 17))) & 0x3FFFFu);
    }
    return k;
}

template <int D>
__global__ void k_nbr_codes(int na, const std::uint64_t* __restrict__ keys, DHash map, int* nbr) {
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
        nbr[static_cast<std::size_t>(k) * na + i] = map.find(lat_pack<D>(nb));
    }
}

/** One align_interfaces sweep (partition.hpp:474-508): moves decided on the
 *  old labels, applied simultaneously. */
template <int D>
__global__ void k_align(int na, double h, const int* __restrict__ nbr, const double* __restrict__ cp, DHash map,
                        const int* __restrict__ part, int* part_new, SetCounters* cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int pi = part[i];
    int out = pi;
    bool iface = false;
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        const int c = nbr[static_cast<std::size_t>(k) * na + i];
        if (c >= 0 && c < na && part[c] != pi) iface = true;
    }
    if (iface) {
        int xb[D];
#pragma unroll
        for (int a = 0; a < D; ++a) xb[a] = static_cast<int>(floor((cp[static_cast<std::size_t>(i) * D + a] - 0.0) / h + 0.5));
        const int c = map.find(lat_pack<D>(xb));
        if (c >= 0 && c < na && part[c] != pi) {
            out = part[c];
            atomicAdd(&cnt->moves, 1);
        }
    }
    part_new[i] = out;
}

__global__ void k_part_hist(int na, const int* __restrict__ part, int* hist) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) atomicAdd(hist + part[i], 1);
}

/** find_cross_points (subdomain.hpp:59-79). */
template <int D>
__global__ void k_cross(int na, const int* __restrict__ nbr, const int* __restrict__ part, int* flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int sa = -1, sb = -1;
    const int pi = part[i];
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        const int c = nbr[static_cast<std::size_t>(k) * na + i];
        if (c < 0 || c >= na) continue;
        const int q = part[c];
        if (q == pi || q == sa || q == sb) continue;
        if (sa < 0)
            sa = q;
        else
            sb = q;
    }
    flag[i] = sb >= 0;
}

/** Bin key of a point (decomp.cpp Bins::bin_key): floor(q / cell) + off. */
template <int D>
__device__ __forceinline__ std::uint64_t d_bin_key(const double* q, double cell, const int* off) {
    int b[D];
#pragma unroll
    for (int a = 0; a < D; ++a) b[a] = static_cast<int>(floor(q[a] / cell)) + off[a];
    return lat_pack<D>(b);
}

template <int D>
__global__ void k_cross_bins(int n, const int* __restrict__ cross, const std::uint64_t* __restrict__ keys, double h,
                             double cell, std::uint64_t* bkey) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    int ix[D];
    lat_unpack<D>(keys[cross[s]], ix);
    double x[D];
    d_point<D>(ix, h, x);
    const int off[D] = {};
    bkey[s] = d_bin_key<D>(x, cell, off);
}

__global__ void k_run_heads(int n, const std::uint64_t* __restrict__ sk, DHash heads) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n && (s == 0 || sk[s] != sk[s - 1])) heads.insert(sk[s], s);
}

__global__ void k_pairs_init(int na, const int* __restrict__ part, DHash ov, std::uint64_t* ovl, int* ovlay) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const std::uint64_t k = pair_key(part[i], i);
    ov.insert(k, 0);
    ovl[i] = k;
    ovlay[i] = 0;
}

/** One overlap layer (subdomain.hpp:186-207) for every subdomain at once. */
template <int D>
__global__ void k_ov_layer(int f0, int f1, int layer, int na, const int* __restrict__ nbr, DHash ov,
                           std::uint64_t* ovl, int* ovlay, int cap, SetCounters* cnt) {
    const int s = f0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= f1) return;
    const std::uint64_t k0 = ovl[s];
    const int j = pair_j(k0), i = pair_i(k0);
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        const int c = nbr[static_cast<std::size_t>(k) * na + i];
        if (c < 0 || c >= na) continue;
        const std::uint64_t kk = pair_key(j, c);
        if (ov.insert(kk, layer)) {
            const int pos = atomicAdd(&cnt->n_ov, 1);
            if (pos < cap) {
                ovl[pos] = kk;
                ovlay[pos] = layer;
            } else {
                cnt->overflow = 1;
            }
        }
    }
}

__device__ __forceinline__ void push_pair(std::uint64_t k, std::uint64_t* list, int* counter, int cap,
                                          SetCounters* cnt) {
    const int pos = atomicAdd(counter, 1);
    if (pos < cap)
        list[pos] = k;
    else
        cnt->overflow = 1;
}

/** FD completion and adjacent ghosts of the overlap (subdomain.hpp:212-230). */
template <int D>
__global__ void k_fd_ghosts(int n_ov, int na, const int* __restrict__ nbr, const std::uint64_t* __restrict__ ovl,
                            DHash ov, DHash bc, DHash gh, std::uint64_t* bcl, std::uint64_t* ghl, int cap_bc,
                            int cap_gh, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_ov) return;
    const std::uint64_t k0 = ovl[s];
    const int j = pair_j(k0), i = pair_i(k0);
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        const int c = nbr[static_cast<std::size_t>(k) * na + i];
        if (c < 0) {
            atomicOr(&cnt->err, kErrNbr);
            continue;
        }
        const std::uint64_t kk = pair_key(j, c);
        if (c < na) {
            if (!ov.contains(kk) && bc.insert(kk, 1)) push_pair(kk, bcl, &cnt->n_bc, cap_bc, cnt);
        } else if (gh.insert(kk, 0)) {
            push_pair(kk, ghl, &cnt->n_gh, cap_gh, cnt);
        }
    }
}

/** Extension-row references (subdomain.hpp:232-244) of the pairs in list. */
template <int D>
__global__ void k_ext_refs(int n, const std::uint64_t* __restrict__ list, int na, double h, int p,
                           const double* __restrict__ cp, DHash map, DHash ov, DHash bc, std::uint64_t* bcl,
                           int cap_bc, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const std::uint64_t k0 = list[s];
    const int j = pair_j(k0), code = pair_i(k0);
    int base[D];
#pragma unroll
    for (int a = 0; a < D; ++a) base[a] = d_stencil_base(cp[static_cast<std::size_t>(code) * D + a], h, p);
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
        const int c = map.find(lat_pack<D>(q));
        if (c < 0 || c >= na) {
            atomicOr(&cnt->err, kErrStencil);
            continue;
        }
        const std::uint64_t kk = pair_key(j, c);
        if (!ov.contains(kk) && bc.insert(kk, 0)) push_pair(kk, bcl, &cnt->n_bc, cap_bc, cnt);
    }
}

/** Ghost-type Robin ring around the BC actives (subdomain.hpp:249-273). */
template <int D>
__global__ void k_ring(int n_bc, int na, const std::uint64_t* __restrict__ bcl, const std::uint64_t* __restrict__ keys,
                       DHash map, DHash ov, DHash bc, DHash gh, DHash ring, std::uint64_t* rkey, int* rcode,
                       int cap, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_bc) return;
    const std::uint64_t k0 = bcl[s];
    const int j = pair_j(k0), b = pair_i(k0);
    int ix[D];
    lat_unpack<D>(keys[b], ix);
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) {
        int nb[D];
#pragma unroll
        for (int a = 0; a < D; ++a) nb[a] = ix[a];
        nb[k >> 1] += (k & 1) ? 1 : -1;
        const int c = map.find(lat_pack<D>(nb));
        if (c >= 0 && c < na) {
            const std::uint64_t kk = pair_key(j, c);
            if (ov.contains(kk) || bc.contains(kk)) continue;
        }
        if (c >= na && gh.contains(pair_key(j, c))) continue;
        const std::uint64_t rk = ring_key<D>(j, nb) + 1;
        if (!ring.insert(rk, 0)) continue;
        const int pos = atomicAdd(&cnt->n_ring, 1);
        if (pos < cap) {
            rkey[pos] = rk - 1;
            rcode[pos] = c;
        } else {
            cnt->overflow = 1;
        }
    }
}

/** Sort keys of the BC entries: BC actives (tag = index into bcl) and ring
 *  nodes (tag = n_bc + index into the ring list). */
template <int D>
__global__ void k_bc_keys(int n_bc, int n_ring, const std::uint64_t* __restrict__ bcl,
                          const std::uint64_t* __restrict__ keys, const std::uint64_t* __restrict__ rkey,
                          std::uint64_t* skey, int* tag, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_bc + n_ring) return;
    if (s < n_bc) {
        const std::uint64_t k0 = bcl[s];
        int ix[D];
        lat_unpack<D>(keys[pair_i(k0)], ix);
#pragma unroll
        for (int a = 0; a < D; ++a)
            if (ix[a] <= -(1 << 17) || ix[a] >= (1 << 17) - 1) atomicOr(&cnt->err, kErrRange);
        skey[s] = ring_key<D>(pair_j(k0), ix);
    } else {
        skey[s] = rkey[s - n_bc];
    }
    tag[s] = s;
}

__global__ void k_final_max(int n_ov, const std::uint64_t* __restrict__ ovl, const int* __restrict__ ovlay, int* maxl) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n_ov) atomicMax(maxl + pair_j(ovl[s]), ovlay[s]);
}

__global__ void k_final_flag(int n_ov, const std::uint64_t* __restrict__ ovl, const int* __restrict__ ovlay,
                             const int* __restrict__ maxl, std::uint64_t* fkey) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_ov) return;
    const int j = pair_j(ovl[s]);
    fkey[s] = (ovlay[s] >= 1 && ovlay[s] == maxl[j]) ? ovl[s] : ~0ULL;
}

/** Interface anchor, conormal, dq and cross flag of every BC entry
 *  (subdomain.hpp:276-311, host decomp.cpp). */
template <int D>
__global__ void k_anchor(int n, double h, double anchor_radius, double excl, double cross_radius,
                         const std::uint64_t* __restrict__ skey, const int* __restrict__ fstart,
                         const int* __restrict__ fcode, const double* __restrict__ cp, const double* __restrict__ nrm,
                         const double* __restrict__ cross_x, const std::uint64_t* __restrict__ cross_bkey,
                         DHash cross_heads, int n_cross, double* out, unsigned char* flags, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const std::uint64_t k = skey[s];
    const int j = static_cast<int>(k >> 54);
    int ix[D];
    {
        std::uint64_t r = k;
        int t[3];
        for (int a = 2; a >= 0; --a) {
            t[a] = static_cast<int>(r & 0x3FFFFu) - (1 << 17);
            r >>= 18;
        }
#pragma unroll
        for (int a = 0; a < D; ++a) ix[a] = t[a];
    }
    double x[D];
    d_point<D>(ix, h, x);
    const int f0 = fstart[j], f1 = fstart[j + 1];
    int best = -1;
    double bd = anchor_radius;
    for (int q = f0; q < f1; ++q) {
        const double d = ddist<D>(cp + static_cast<std::size_t>(fcode[q]) * D, x);
        if (d <= excl) continue;
        if (d < bd || (d == bd && best < 0)) {
            bd = d;
            best = q - f0;
        }
    }
    unsigned char fl = 0;
    if (best < 0) {
        double gd = __longlong_as_double(0x7ff0000000000000LL);
        for (int q = f0; q < f1; ++q) {
            const double d = ddist<D>(cp + static_cast<std::size_t>(fcode[q]) * D, x);
            if (d <= excl) continue;
            if (d < gd) {
                gd = d;
                best = q - f0;
            }
        }
        fl |= 1;  // fallback
    }
    double* o = out + static_cast<std::size_t>(s) * (2 * D + 1);
    if (best < 0) {
        atomicOr(&cnt->err, kErrAnchor);
        return;
    }
    const double* pl = cp + static_cast<std::size_t>(fcode[f0 + best]) * D;
    const double* nl = nrm + static_cast<std::size_t>(fcode[f0 + best]) * D;
    double dv[D], tang[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dv[a] = x[a] - pl[a];
    const double dn = ddot<D>(dv, nl);
#pragma unroll
    for (int a = 0; a < D; ++a) tang[a] = dv[a] - dn * nl[a];
    const double tn = dnorm<D>(tang);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        o[a] = pl[a];
        o[D + a] = 0.0;
    }
    o[2 * D] = 0.0;
    if (tn > 1e-12 * dnorm<D>(dv)) {
#pragma unroll
        for (int a = 0; a < D; ++a) o[D + a] = tang[a] / tn;
        o[2 * D] = tn;
    }
    // cross flag: any cross point within cross_radius in the 3^D bins around x
    int off[D];
#pragma unroll
    for (int a = 0; a < D; ++a) off[a] = -1;
    bool flag = false;
    for (;;) {
        const std::uint64_t bk = d_bin_key<D>(x, cross_radius, off);
        const int h0 = cross_heads.find(bk);
        if (h0 >= 0)
            for (int q = h0; q < n_cross && cross_bkey[q] == bk && !flag; ++q)
                if (ddist<D>(x, cross_x + static_cast<std::size_t>(q) * D) <= cross_radius) flag = true;
        int a = 0;
        while (a < D && off[a] == 1) off[a++] = -1;
        if (a == D) break;
        ++off[a];
    }
    if (flag) fl |= 2;
    flags[s] = fl;
}

/** Closest points of the non-band ring nodes (subdomain.hpp:262-263). */
template <int D>
__global__ void k_ring_cp(DSurf S, double h, int n_ring, const std::uint64_t* __restrict__ rkey,
                          const int* __restrict__ rcode, double* rcp, SetCounters* cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_ring || rcode[s] >= 0) return;
    std::uint64_t r = rkey[s];
    int t[3];
    for (int a = 2; a >= 0; --a) {
        t[a] = static_cast<int>(r & 0x3FFFFu) - (1 << 17);
        r >>= 18;
    }
    double x[D];
    d_point<D>(t, h, x);
    int err = 0;
    const DCp<D> c = d_closest_point<D>(S, x, &err);
    if (err) atomicOr(&cnt->err, kErrCp);
#pragma unroll
    for (int a = 0; a < D; ++a) rcp[static_cast<std::size_t>(s) * D + a] = c.cp[a];
}

template <class T>
void sort_u64(int n, const std::uint64_t* in, std::uint64_t* out, int bits, cudaStream_t st) {
    std::size_t tmp = 0;
    CPDDG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in, out, n, 0, bits, st));
    DevBuf<unsigned char> scratch(std::max<std::size_t>(tmp, 1));
    CPDDG_CUDA(cub::DeviceRadixSort::SortKeys(scratch.get(), tmp, in, out, n, 0, bits, st));
}

void sort_u64_pairs(int n, const std::uint64_t* kin, std::uint64_t* kout, const int* vin, int* vout, int bits,
                    cudaStream_t st) {
    std::size_t tmp = 0;
    CPDDG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, bits, st));
    DevBuf<unsigned char> scratch(std::max<std::size_t>(tmp, 1));
    CPDDG_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(), tmp, kin, kout, vin, vout, n, 0, bits, st));
}

/** Split keys sorted by (j, i) into per-subdomain lists of i. */
void split_pairs(const std::vector<std::uint64_t>& k, int n_parts, std::vector<std::vector<int>>& out) {
    out.assign(static_cast<std::size_t>(n_parts), {});
    for (std::uint64_t v : k) {
        if (v == ~0ULL) break;
        out[static_cast<std::size_t>(pair_j(v))].push_back(pair_i(v));
    }
}

}  // namespace

template <int D>
int decompose_device(const DevBand& B, const Band<D>& g, std::vector<int>& part, int n_overlap, bool robin_ring,
                     std::vector<Subdomain<D>>& subs, double* t_align, double* t_sets) {
    if (n_overlap < 1) throw ConfigError("overlap width must be at least 1 layer");
    const int na = B.na;
    if (static_cast<int>(part.size()) != na) throw InternalError("partition size does not match grid");
    const int n_parts = *std::max_element(part.begin(), part.end()) + 1;
    if (n_parts > 1023) throw DeviceSetLimit("device subdomain sets support at most 1023 subdomains");
    cudaStream_t st = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const double h = B.h;
    const DSurf S = B.surf();
    DevBuf<SetCounters> cnt(1);
    SetCounters hc{};
    auto pull = [&] {
        CPDDG_CUDA(cudaMemcpyAsync(&hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
    };
    DevBuf<int> nbr(static_cast<std::size_t>(2 * D) * na);
    k_nbr_codes<D><<<blocks_for(na), kThr, 0, st>>>(na, B.keys.get(), B.map.view(), nbr.get());

    // ---- align_interfaces
    DevBuf<int> pa, pb(static_cast<std::size_t>(na));
    pa.upload(part);
    int total = 0;
    for (int sweep = 0; sweep < B.p + 1; ++sweep) {
        CPDDG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(SetCounters), st));
        k_align<D><<<blocks_for(na), kThr, 0, st>>>(na, h, nbr.get(), B.cp.get(), B.map.view(), pa.get(), pb.get(),
                                                     cnt.get());
        pull();
        if (hc.moves == 0) break;
        std::swap(pa, pb);
        total += hc.moves;
    }
    {
        DevBuf<int> hist(static_cast<std::size_t>(n_parts));
        hist.zero(st);
        k_part_hist<<<blocks_for(na), kThr, 0, st>>>(na, pa.get(), hist.get());
        const std::vector<int> hh = download(hist.get(), static_cast<std::size_t>(n_parts), st);
        for (int q = 0; q < n_parts; ++q)
            if (hh[static_cast<std::size_t>(q)] == 0)
                throw ConfigError("interface alignment emptied part " + std::to_string(q) +
                                  "; use fewer subdomains or a finer grid");
    }
    part = download(pa.get(), static_cast<std::size_t>(na), st);
    const auto t1 = std::chrono::steady_clock::now();

    // ---- cross points and their bins
    const double cross_radius = 2.0 * n_overlap * h;
    DevBuf<int> cflag(static_cast<std::size_t>(na));
    k_cross<D><<<blocks_for(na), kThr, 0, st>>>(na, nbr.get(), pa.get(), cflag.get());
    std::vector<int> cross;
    {
        const std::vector<int> hf = download(cflag.get(), static_cast<std::size_t>(na), st);
        for (int i = 0; i < na; ++i)
            if (hf[static_cast<std::size_t>(i)]) cross.push_back(i);
    }
    const int nc = static_cast<int>(cross.size());
    DevBuf<std::uint64_t> cbk_sorted(static_cast<std::size_t>(std::max(nc, 1)));
    DevBuf<double> cross_x(static_cast<std::size_t>(std::max(nc, 1)) * D);
    DevHashTable cross_heads;
    cross_heads.init(static_cast<std::size_t>(std::max(nc, 1)), st);
    if (nc > 0) {
        DevBuf<int> dcross, cperm(static_cast<std::size_t>(nc)), iota(static_cast<std::size_t>(nc));
        dcross.upload(cross);
        DevBuf<std::uint64_t> cbk(static_cast<std::size_t>(nc));
        k_cross_bins<D><<<blocks_for(nc), kThr, 0, st>>>(nc, dcross.get(), B.keys.get(), h, cross_radius, cbk.get());
        k_iota<<<blocks_for(nc), kThr, 0, st>>>(nc, iota.get());
        sort_u64_pairs(nc, cbk.get(), cbk_sorted.get(), iota.get(), cperm.get(), 63, st);
        k_run_heads<<<blocks_for(nc), kThr, 0, st>>>(nc, cbk_sorted.get(), cross_heads.view());
        const std::vector<int> hp = download(cperm.get(), static_cast<std::size_t>(nc), st);
        std::vector<double> hx(static_cast<std::size_t>(nc) * D);
        for (int s2 = 0; s2 < nc; ++s2) {
            const Vec<D> xx = g.x(cross[static_cast<std::size_t>(hp[static_cast<std::size_t>(s2)])]);
            for (int a = 0; a < D; ++a) hx[static_cast<std::size_t>(s2) * D + a] = xx[a];
        }
        cross_x.upload(hx);
    }

    // ---- overlap layers, FD completion, ghosts, extension refs, ring
    int cap_ov = 4 * na, cap_bc = 2 * na, cap_gh = na, cap_ring = na;
    DevBuf<std::uint64_t> ovl, bcl, ghl, rkey;
    DevBuf<int> ovlay, rcode;
    DevHashTable ov, bc, gh, ring;
    for (;;) {
        ovl.alloc(static_cast<std::size_t>(cap_ov));
        ovlay.alloc(static_cast<std::size_t>(cap_ov));
        bcl.alloc(static_cast<std::size_t>(cap_bc));
        ghl.alloc(static_cast<std::size_t>(cap_gh));
        rkey.alloc(static_cast<std::size_t>(cap_ring));
        rcode.alloc(static_cast<std::size_t>(cap_ring));
        ov.init(static_cast<std::size_t>(cap_ov), st);
        bc.init(static_cast<std::size_t>(cap_bc), st);
        gh.init(static_cast<std::size_t>(cap_gh), st);
        ring.init(static_cast<std::size_t>(cap_ring), st);
        CPDDG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(SetCounters), st));
        CPDDG_CUDA(cudaMemcpyAsync(&cnt.get()->n_ov, &na, sizeof(int), cudaMemcpyHostToDevice, st));
        k_pairs_init<<<blocks_for(na), kThr, 0, st>>>(na, pa.get(), ov.view(), ovl.get(), ovlay.get());
        int f0 = 0, f1 = na;
        for (int layer = 1; layer <= n_overlap && f1 > f0; ++layer) {
            k_ov_layer<D><<<blocks_for(f1 - f0), kThr, 0, st>>>(f0, f1, layer, na, nbr.get(), ov.view(), ovl.get(),
                                                               ovlay.get(), cap_ov, cnt.get());
            pull();
            if (hc.overflow) break;
            f0 = f1;
            f1 = hc.n_ov;
        }
        if (!hc.overflow) {
            const int n_ov = hc.n_ov;
            k_fd_ghosts<D><<<blocks_for(n_ov), kThr, 0, st>>>(n_ov, na, nbr.get(), ovl.get(), ov.view(), bc.view(),
                                                             gh.view(), bcl.get(), ghl.get(), cap_bc, cap_gh,
                                                             cnt.get());
            pull();
            const int n_fd = std::min(hc.n_bc, cap_bc), n_gh = std::min(hc.n_gh, cap_gh);
            if (!hc.overflow) {
                k_ext_refs<D><<<blocks_for(n_ov), kThr, 0, st>>>(n_ov, ovl.get(), na, h, B.p, B.cp.get(),
                                                                B.map.view(), ov.view(), bc.view(), bcl.get(), cap_bc,
                                                                cnt.get());
                k_ext_refs<D><<<blocks_for(n_gh), kThr, 0, st>>>(n_gh, ghl.get(), na, h, B.p, B.cp.get(),
                                                                B.map.view(), ov.view(), bc.view(), bcl.get(), cap_bc,
                                                                cnt.get());
                // the FD nodes' rows: bcl[0, n_fd) is not rewritten (appends only)
                k_ext_refs<D><<<blocks_for(n_fd), kThr, 0, st>>>(n_fd, bcl.get(), na, h, B.p, B.cp.get(),
                                                                B.map.view(), ov.view(), bc.view(), bcl.get(), cap_bc,
                                                                cnt.get());
                pull();
            }
            if (!hc.overflow && robin_ring) {
                k_ring<D><<<blocks_for(hc.n_bc), kThr, 0, st>>>(hc.n_bc, na, bcl.get(), B.keys.get(), B.map.view(),
                                                               ov.view(), bc.view(), gh.view(), ring.view(), rkey.get(),
                                                               rcode.get(), cap_ring, cnt.get());
                pull();
            }
        }
        if (!hc.overflow) break;
        cap_ov *= 2;
        cap_bc *= 2;
        cap_gh *= 2;
        cap_ring *= 2;
    }
    if (hc.err & kErrNbr) throw InternalError("band closure missed a neighbour");
    if (hc.err & kErrStencil) throw InternalError("extension stencil node is not active: band closure violated");
    const int n_ov = hc.n_ov, n_bc = hc.n_bc, n_gh = hc.n_gh, n_ring = robin_ring ? hc.n_ring : 0;

    // ---- sorted lists
    DevBuf<std::uint64_t> ovs(static_cast<std::size_t>(n_ov)), ghs(static_cast<std::size_t>(std::max(n_gh, 1)));
    sort_u64<int>(n_ov, ovl.get(), ovs.get(), 64, st);
    if (n_gh) sort_u64<int>(n_gh, ghl.get(), ghs.get(), 64, st);
    DevBuf<int> maxl(static_cast<std::size_t>(n_parts));
    maxl.zero(st);
    k_final_max<<<blocks_for(n_ov), kThr, 0, st>>>(n_ov, ovl.get(), ovlay.get(), maxl.get());
    DevBuf<std::uint64_t> fk(static_cast<std::size_t>(n_ov)), fks(static_cast<std::size_t>(n_ov));
    k_final_flag<<<blocks_for(n_ov), kThr, 0, st>>>(n_ov, ovl.get(), ovlay.get(), maxl.get(), fk.get());
    sort_u64<int>(n_ov, fk.get(), fks.get(), 64, st);
    const int n_be = n_bc + n_ring;
    DevBuf<std::uint64_t> bkey(static_cast<std::size_t>(std::max(n_be, 1))), bkey_s(static_cast<std::size_t>(std::max(n_be, 1)));
    DevBuf<int> btag(static_cast<std::size_t>(std::max(n_be, 1))), btag_s(static_cast<std::size_t>(std::max(n_be, 1)));
    CPDDG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(SetCounters), st));
    if (n_be) {
        k_bc_keys<D><<<blocks_for(n_be), kThr, 0, st>>>(n_bc, n_ring, bcl.get(), B.keys.get(), rkey.get(), bkey.get(),
                                                       btag.get(), cnt.get());
        sort_u64_pairs(n_be, bkey.get(), bkey_s.get(), btag.get(), btag_s.get(), 64, st);
    }
    pull();
    if (hc.err & kErrRange) throw DeviceSetLimit("lattice index out of the device subdomain-set range");

    const std::vector<std::uint64_t> h_ov = download(ovs.get(), static_cast<std::size_t>(n_ov), st);
    const std::vector<std::uint64_t> h_gh = download(ghs.get(), static_cast<std::size_t>(n_gh), st);
    const std::vector<std::uint64_t> h_fl = download(fks.get(), static_cast<std::size_t>(n_ov), st);
    std::vector<std::vector<int>> ovj, ghj, flj;
    split_pairs(h_ov, n_parts, ovj);
    split_pairs(h_gh, n_parts, ghj);
    split_pairs(h_fl, n_parts, flj);

    // final-layer CSR for the anchors
    std::vector<int> fstart(static_cast<std::size_t>(n_parts) + 1, 0), fcode;
    for (int j = 0; j < n_parts; ++j) {
        fcode.insert(fcode.end(), flj[static_cast<std::size_t>(j)].begin(), flj[static_cast<std::size_t>(j)].end());
        fstart[static_cast<std::size_t>(j) + 1] = static_cast<int>(fcode.size());
    }
    DevBuf<int> d_fstart, d_fcode;
    d_fstart.upload(fstart);
    d_fcode.upload(fcode.empty() ? std::vector<int>{0} : fcode);
    DevBuf<double> rcp(static_cast<std::size_t>(std::max(n_ring, 1)) * D);
    if (n_ring)
        k_ring_cp<D><<<blocks_for(n_ring), kThr, 0, st>>>(S, h, n_ring, rkey.get(), rcode.get(), rcp.get(), cnt.get());
    const double anchor_radius = stencil_reach<D>(h, B.p) + h;
    const double excl = 1e-12 * h;
    DevBuf<double> aout(static_cast<std::size_t>(std::max(n_be, 1)) * (2 * D + 1));
    DevBuf<unsigned char> aflag(static_cast<std::size_t>(std::max(n_be, 1)));
    // subdomains with BC nodes but no anchors are an error (checked below)
    std::vector<std::uint64_t> h_bk = download(bkey_s.get(), static_cast<std::size_t>(n_be), st);
    for (std::uint64_t k : h_bk) {
        const int j = static_cast<int>(k >> 54);
        if (fstart[static_cast<std::size_t>(j) + 1] == fstart[static_cast<std::size_t>(j)])
            throw InternalError("subdomain has boundary nodes but no interface anchors");
    }
    if (n_be)
        k_anchor<D><<<blocks_for(n_be), kThr, 0, st>>>(n_be, h, anchor_radius, excl, cross_radius, bkey_s.get(),
                                                      d_fstart.get(), d_fcode.get(), B.cp.get(), B.normal.get(),
                                                      cross_x.get(), cbk_sorted.get(), cross_heads.view(), nc,
                                                      aout.get(), aflag.get(), cnt.get());
    CPDDG_CUDA(cudaGetLastError());
    pull();
    if (hc.err & kErrAnchor) throw InternalError("no usable interface anchor for a boundary node");
    if (hc.err & kErrCp) throw InternalError("closest-point query found no triangle");
    const std::vector<int> h_tag = download(btag_s.get(), static_cast<std::size_t>(n_be), st);
    const std::vector<std::uint64_t> h_bcl = download(bcl.get(), static_cast<std::size_t>(n_bc), st);
    const std::vector<int> h_rcode = download(rcode.get(), static_cast<std::size_t>(n_ring), st);
    const std::vector<double> h_rcp = download(rcp.get(), static_cast<std::size_t>(n_ring) * D, st);
    const std::vector<double> h_out = download(aout.get(), static_cast<std::size_t>(n_be) * (2 * D + 1), st);
    const std::vector<unsigned char> h_fl2 = download(aflag.get(), static_cast<std::size_t>(n_be), st);

    // ---- host Subdomain structures
    subs.assign(static_cast<std::size_t>(n_parts), Subdomain<D>{});
    for (int j = 0; j < n_parts; ++j) subs[static_cast<std::size_t>(j)].id = j;
    for (int i = 0; i < na; ++i) subs[static_cast<std::size_t>(part[static_cast<std::size_t>(i)])].disjoint.push_back(i);
    for (int j = 0; j < n_parts; ++j) {
        Subdomain<D>& Sj = subs[static_cast<std::size_t>(j)];
        Sj.overlap = std::move(ovj[static_cast<std::size_t>(j)]);
        Sj.ghosts = std::move(ghj[static_cast<std::size_t>(j)]);
        Sj.final_layer = std::move(flj[static_cast<std::size_t>(j)]);
        Sj.n_lambda = static_cast<int>(Sj.final_layer.size());
    }
    for (int s2 = 0; s2 < n_be; ++s2) {
        const std::uint64_t k = h_bk[static_cast<std::size_t>(s2)];
        const int j = static_cast<int>(k >> 54);
        const int tag = h_tag[static_cast<std::size_t>(s2)];
        BoundaryNode<D> node;
        std::uint64_t r = k;
        int t[3];
        for (int a = 2; a >= 0; --a) {
            t[a] = static_cast<int>(r & 0x3FFFFu) - (1 << 17);
            r >>= 18;
        }
        for (int a = 0; a < D; ++a) node.ix[a] = t[a];
        node.x = index_to_point<D>(node.ix, h);
        if (tag < n_bc) {
            const int b = pair_i(h_bcl[static_cast<std::size_t>(tag)]);
            node.global_active = b;
            node.cp = g.cp[static_cast<std::size_t>(b)];
        } else {
            const int q = tag - n_bc;
            const int c = h_rcode[static_cast<std::size_t>(q)];
            node.is_ghost_type = true;
            if (c >= 0) {
                node.cp = g.cp[static_cast<std::size_t>(c)];
                node.global_active = c < na ? c : -1;
            } else {
                for (int a = 0; a < D; ++a) node.cp[a] = h_rcp[static_cast<std::size_t>(q) * D + a];
            }
        }
        const double* o = h_out.data() + static_cast<std::size_t>(s2) * (2 * D + 1);
        for (int a = 0; a < D; ++a) {
            node.cp_local[a] = o[a];
            node.conormal[a] = o[D + a];
        }
        node.dq = o[2 * D];
        node.fallback = h_fl2[static_cast<std::size_t>(s2)] & 1;
        node.cross_flagged = (h_fl2[static_cast<std::size_t>(s2)] & 2) != 0;
        Subdomain<D>& Sj = subs[static_cast<std::size_t>(j)];
        if (node.fallback) ++Sj.fallback_count;
        Sj.bc.push_back(node);
    }
    const auto t2 = std::chrono::steady_clock::now();
    if (t_align) *t_align = std::chrono::duration<double>(t1 - t0).count();
    if (t_sets) *t_sets = std::chrono::duration<double>(t2 - t1).count();
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] device sets: align %.3f s (%d moves), sets %.3f s (ov %d bc %d ring %d gh %d)\n",
                     std::chrono::duration<double>(t1 - t0).count(), total,
                     std::chrono::duration<double>(t2 - t1).count(), n_ov, n_bc, n_ring, n_gh);
    return total;
}

template int decompose_device<2>(const DevBand&, const Band<2>&, std::vector<int>&, int, bool,
                                 std::vector<Subdomain<2>>&, double*, double*);
template int decompose_device<3>(const DevBand&, const Band<3>&, std::vector<int>&, int, bool,
                                 std::vector<Subdomain<3>>&, double*, double*);

}  // namespace cpddg
