// Matrix-free CPM operator on the device.
//
// Replaces SparseOperator::apply on the assembled Helmholtz matrix
// (proj/include/cpdd/sparse.hpp:65-75; A from operators.hpp:96-112):
//
//   (A x)_i = (c + 2d/h^2) x_i - h^-2 sum_{k in 2d axis nbrs of i} (E x)_k
//
// Two streaming kernels, both HBM-bound:
//   k_extend : v_k = (E x)_k for every band node (actives + ghosts).  The
//              (p+1)^d stencil of cp_k is (p+1)^(d-1) runs of p+1
//              CONSECUTIVE active ordinals (lexicographic band order, last
//              axis fastest -- verified at create time), so a node stores
//              one int32 start per run plus its d stencil offsets t_a; the
//              1-D barycentric weights are recomputed from t_a in registers
//              (interp.hpp:35-54, same exact-hit rule) instead of loading
//              (p+1)^d weights.
//   k_helm   : y_i = (c+gamma) x_i - ih2 sum_k v[nbr_k(i)], optionally fused
//              with r = b - y and a deterministic ||r||^2 partial sum.
// Layout: every per-node table is structure-of-arrays ([entry][node]) so a
// warp's loads of one table entry are one contiguous 128-byte line.
#include "../host/setup.hpp"
#include "common.cuh"
#include "op.cuh"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>

namespace cpddg {

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        CPDDG_CUDA(cudaGetDevice(&dev));
        CPDDG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

int reduction_blocks() { return 4 * sm_count(); }

void ReduceWork::ensure(int s) {
    if (s <= slots) return;
    partials.alloc(static_cast<std::size_t>(s) * reduction_blocks());
    counter.alloc(static_cast<std::size_t>(s));
    counter.zero();
    CPDDG_CUDA(cudaDeviceSynchronize());
    slots = s;
}

namespace {

/** interp_weights_1d (interp.hpp:35-54) for a compile-time degree. */
template <int P>
__device__ __forceinline__ void weights_1d(double t, double* w) {
#pragma unroll
    for (int j = 0; j <= P; ++j) w[j] = 0.0;
    int hit = -1;
#pragma unroll
    for (int j = 0; j <= P; ++j)
        if (hit < 0 && fabs(t - j) < 1e-12) hit = j;
    if (hit >= 0) {
#pragma unroll
        for (int j = 0; j <= P; ++j) w[j] = (j == hit) ? 1.0 : 0.0;
        return;
    }
    double sum = 0.0, b = 1.0;
#pragma unroll
    for (int j = 0; j <= P; ++j) {
        w[j] = __ddiv_rn(b, __dsub_rn(t, static_cast<double>(j)));
        sum = __dadd_rn(sum, w[j]);
        b *= -static_cast<double>(P - j) / (j + 1);
    }
#pragma unroll
    for (int j = 0; j <= P; ++j) w[j] = __ddiv_rn(w[j], sum);
}

template <int D, int P>
__global__ void __launch_bounds__(256) k_extend(int nb, const double* __restrict__ t,
                                                const int* __restrict__ lines,
                                                const double* __restrict__ x, double* __restrict__ v) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nb) return;
    constexpr int Q = P + 1;
    double wl[Q];  // weights along the contiguous (last) axis
    weights_1d<P>(__ldg(t + static_cast<std::size_t>(D - 1) * nb + k), wl);
    double acc = 0.0;
    if constexpr (D == 2) {
        double w0[Q];
        weights_1d<P>(__ldg(t + k), w0);
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            const int o = __ldg(lines + static_cast<std::size_t>(a) * nb + k);
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c) s = fma(wl[c], __ldg(x + o + c), s);
            acc = fma(w0[a], s, acc);
        }
    } else {
        double w0[Q], w1[Q];
        weights_1d<P>(__ldg(t + k), w0);
        weights_1d<P>(__ldg(t + static_cast<std::size_t>(nb) + k), w1);
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double sa = 0.0;
#pragma unroll
            for (int b = 0; b < Q; ++b) {
                const int o = __ldg(lines + static_cast<std::size_t>(a * Q + b) * nb + k);
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < Q; ++c) s = fma(wl[c], __ldg(x + o + c), s);
                sa = fma(w1[b], s, sa);
            }
            acc = fma(w0[a], sa, acc);
        }
    }
    v[k] = acc;
}

/** Cubic (p = 3) weights in product (Lagrange) form -- no divisions -- with
 *  the reference's exact-hit rule (interp.hpp:39-44).  Differs from the
 *  barycentric evaluation only in the last bits; operator parity is 1e-12. */
__device__ __forceinline__ void weights_p3_nohit(double t, double* w) {
    const double t0 = t, t1 = t - 1.0, t2 = t - 2.0, t3 = t - 3.0;
    w[0] = -(t1 * t2 * t3) * (1.0 / 6.0);
    w[1] = (t0 * t2 * t3) * 0.5;
    w[2] = -(t0 * t1 * t3) * 0.5;
    w[3] = (t0 * t1 * t2) * (1.0 / 6.0);
}
__device__ __forceinline__ void weights_p3(double t, double* w) {
    const double t0 = t, t1 = t - 1.0, t2 = t - 2.0, t3 = t - 3.0;
    weights_p3_nohit(t, w);
    // exact hit: at most one |t - j| < 1e-12; branch-free selects
    const bool h0 = fabs(t0) < 1e-12, h1 = fabs(t1) < 1e-12, h2 = fabs(t2) < 1e-12, h3 = fabs(t3) < 1e-12;
    const bool any = h0 || h1 || h2 || h3;
    w[0] = h0 ? 1.0 : (any ? 0.0 : w[0]);
    w[1] = h1 ? 1.0 : (any ? 0.0 : w[1]);
    w[2] = h2 ? 1.0 : (any ? 0.0 : w[2]);
    w[3] = h3 ? 1.0 : (any ? 0.0 : w[3]);
}

/** v = E x for p = 3 with four threads per band node (one per offset a of
 *  axis 0): each thread gathers its (p+1)^(d-2) runs of 4 consecutive x,
 *  the quad reduces with two shuffles.  4x the threads of one-node-per-thread
 *  and no divisions: the gather from L2 is the only latency left. */
template <int D>
__global__ void __launch_bounds__(256) k_extend_p3(int nb, const double* __restrict__ t,
                                                   const int* __restrict__ lines, const double* __restrict__ x,
                                                   double* __restrict__ v) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = gt >> 2, a = gt & 3;
    double acc = 0.0;
    if (k < nb) {
        double wl[4], w0[4];
        weights_p3(__ldg(t + static_cast<std::size_t>(D - 1) * nb + k), wl);
        weights_p3(__ldg(t + k), w0);
        if constexpr (D == 2) {
            const int o = __ldg(lines + static_cast<std::size_t>(a) * nb + k);
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) s = fma(wl[c], __ldg(x + o + c), s);
            acc = (a == 0 ? w0[0] : a == 1 ? w0[1] : a == 2 ? w0[2] : w0[3]) * s;
        } else {
            double w1[4];
            weights_p3(__ldg(t + static_cast<std::size_t>(nb) + k), w1);
            int o[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) o[b] = __ldg(lines + static_cast<std::size_t>(a * 4 + b) * nb + k);
            double xv[4][4];
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) xv[b][c] = __ldg(x + o[b] + c);
            double sa = 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) s = fma(wl[c], xv[b][c], s);
                sa = fma(w1[b], s, sa);
            }
            acc = (a == 0 ? w0[0] : a == 1 ? w0[1] : a == 2 ? w0[2] : w0[3]) * sa;
        }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (k < nb && a == 0) v[k] = acc;
}

#ifndef CPDDG_EXT_UNROLL
#define CPDDG_EXT_UNROLL 8
#endif
#ifndef CPDDG_EXT_MINB
#define CPDDG_EXT_MINB 5
#endif
/** v = E x for d = 3, p = 3, staged: one CTA per tile of kExtTile
 *  consecutive band nodes, one thread per node.  The CTA first copies the
 *  x entries its 16 x 256 stencil runs touch (sorted unique active
 *  ordinals, ~9 per node at the headline) into shared memory with coalesced
 *  loads, then every thread reads its 64 stencil values from the stage at
 *  16-bit tile-local run starts.  Consecutive band nodes share most of their
 *  runs, so the L2 gather of 64 values per node (the bound of k_extend_p3:
 *  L1 wavefronts) becomes ~9 streamed loads per node.  The summation order
 *  is k_extend_p3's ((a0 + a1) + (a2 + a3)), so v is bit-identical. */
__global__ void __launch_bounds__(kExtTile, CPDDG_EXT_MINB) k_extend_staged(int nb, const double* __restrict__ t,
                                                           const std::uint16_t* __restrict__ lines16,
                                                           const int* __restrict__ perm,
                                                           const int* __restrict__ tile_k0,
                                                           const int* __restrict__ stage_base,
                                                           const int* __restrict__ stage_idx,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ v) {
    extern __shared__ double xs[];
    const int k = __ldg(tile_k0 + blockIdx.x) + threadIdx.x;
    const bool live = k < __ldg(tile_k0 + blockIdx.x + 1);
    // the node's offsets first: their latency overlaps the stage copy
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    if (live) {
        t0 = __ldg(t + k);
        t1 = __ldg(t + static_cast<std::size_t>(nb) + k);
        t2 = __ldg(t + 2 * static_cast<std::size_t>(nb) + k);
    }
    const int s0 = __ldg(stage_base + blockIdx.x), s1 = __ldg(stage_base + blockIdx.x + 1);
    constexpr int U = CPDDG_EXT_UNROLL;  // one round covers U * kExtTile staged entries
    for (int j = s0 + threadIdx.x; j < s1; j += U * kExtTile) {
        int src[U];
#pragma unroll
        for (int u = 0; u < U; ++u) src[u] = j + u * kExtTile < s1 ? __ldg(stage_idx + j + u * kExtTile) : -1;
        double val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = src[u] >= 0 ? __ldg(x + src[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (src[u] >= 0) xs[j - s0 + u * kExtTile] = val[u];
    }
    double wl[4], w0[4], w1[4];
    weights_p3(t2, wl);
    weights_p3(t0, w0);
    weights_p3(t1, w1);
    __syncthreads();
    if (!live) return;
    double part[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double sa = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* r = xs + __ldg(lines16 + static_cast<std::size_t>(a * 4 + b) * nb + k);
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) s = fma(wl[c], r[c], s);
            sa = fma(w1[b], s, sa);
        }
        part[a] = __dmul_rn(w0[a], sa);
    }
    v[__ldg(perm + k)] = (part[0] + part[1]) + (part[2] + part[3]);  // k is the tile slot
}

/** v = E x for d = 3, p = 3, grouped by stencil base: band nodes sorted by
 *  their stencil base (~8.6 nodes share one at the headline: the nodes along
 *  a surface normal have nearly the same closest point), two nodes of one
 *  base per thread; chunk c is the threads' slot pairs [c kGrpNodes,
 *  (c+1) kGrpNodes) and touches <= kGrpMax bases whose 16 run starts sit at
 *  a fixed stride.  A CTA stages the 64 x values of each of its bases ONCE
 *  into shared memory (~7.5 values per node instead of 64); each thread
 *  reads its base's 4x4x4 block once (128-bit loads; the lanes of one base
 *  read the same words) and contracts it against both nodes' weights.
 *  Summation order is k_extend_p3's ((p0 + p1) + (p2 + p3)), so v is
 *  bit-identical; v is written in band order (the neighbour gathers of
 *  k_helm stay coalesced along lattice lines).
 *
 *  Persistent and software-pipelined (one chunk at a time is load-latency
 *  bound: run starts -> x gather -> shared -> compute): while chunk c is
 *  contracted, the x values of the CTA's next chunk are in flight by
 *  cp.async into the other stage buffer, and the run starts and offsets of
 *  the chunk after that are in flight into registers. */
__global__ void __launch_bounds__(kGrpThreads, 4) k_extend_grouped(int nchunks, int ns, const double* __restrict__ t,
                                                                const unsigned char* __restrict__ gslot,
                                                                const int* __restrict__ perm,
                                                                const int* __restrict__ grp_lines,
                                                                const double* __restrict__ x,
                                                                double* __restrict__ v) {
    __shared__ __align__(16) double xs[2][kGrpMax * kGrpSS];
    constexpr int NT = kGrpThreads, RUNS = kGrpMax * 16, RW = RUNS / (NT / 32), UR = (RW + 31) / 32;
    static_assert(RW % 8 == 0, "runs per warp must be a multiple of 8");
    const int G = gridDim.x, lane = threadIdx.x & 31, wr0 = (threadIdx.x >> 5) * RW;
    int o[UR];  // run starts of this warp's runs wr0 + lane + 32 k
    double2 tt[3];
    int gs = 0;
    int2 pp = make_int2(-1, -1);
    auto load_meta = [&](int c) {  // run starts, offsets, base slot, band codes of chunk c (registers)
#pragma unroll
        for (int u = 0; u < UR; ++u) {
            const int r = wr0 + lane + 32 * u;
            o[u] = (c < nchunks && lane + 32 * u < RW) ? __ldg(grp_lines + static_cast<std::size_t>(c) * RUNS + r) : -1;
        }
        if (c < nchunks) {
            const int th = c * kGrpThreads + threadIdx.x;  // slots 2 th, 2 th + 1
#pragma unroll
            for (int a = 0; a < 3; ++a) tt[a] = __ldg(reinterpret_cast<const double2*>(t + static_cast<std::size_t>(a) * ns) + th);
            gs = __ldg(gslot + th);
            pp = __ldg(reinterpret_cast<const int2*>(perm) + th);
        }
    };
    // x values of the chunk whose run starts are in o: lanes 4q..4q+3 copy
    // the 4 consecutive values of one run (8 runs, 256 contiguous shared bytes
    // per instruction), the run start shuffled from the lane that loaded it
    // x values of the chunk whose run starts are in o: lanes 4q..4q+3 copy
    // the 4 consecutive values of one run (8 runs, 256 contiguous shared bytes
    // per instruction), the run start shuffled from the lane that loaded it.
    // Warp-local run rl = 8 j + lane / 4 is base wr0 / 16 + j / 2, axis-0
    // offset 2 (j % 2) + lane / 16, axis-1 offset (lane / 4) % 4.
    static_assert(RW % 16 == 0, "a warp's runs must cover whole bases");
    const unsigned lane_off = static_cast<unsigned>(
        ((wr0 >> 4) * kGrpSS + (lane >> 4) * kGrpAS + ((lane >> 2) & 3) * 4 + (lane & 3)) * sizeof(double));
    const unsigned xs_base = static_cast<unsigned>(__cvta_generic_to_shared(&xs[0][0]));
    auto issue_stage = [&](int buf) {
        const unsigned b0 = xs_base + buf * (kGrpMax * kGrpSS * sizeof(double)) + lane_off;
#pragma unroll
        for (int j = 0; j < RW / 8; ++j) {
            const int src = __shfl_sync(0xffffffffu, o[(8 * j) / 32], (8 * j + (lane >> 2)) & 31);
            const unsigned dst = b0 + ((j >> 1) * kGrpSS + (j & 1) * 2 * kGrpAS) * sizeof(double);
            if (src >= 0)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(x + src + (lane & 3)) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int c = blockIdx.x;
    load_meta(c);
    issue_stage(0);
    double2 tc[3] = {tt[0], tt[1], tt[2]};
    int gc = gs;
    int2 pc = pp;
    load_meta(c + G);
    for (int it = 0; c < nchunks; ++it, c += G) {
        issue_stage((it + 1) & 1);  // chunk c + G (empty group past the end)
        const double2 tn[3] = {tt[0], tt[1], tt[2]};
        const int gn = gs;
        const int2 pn = pp;
        load_meta(c + 2 * G);
        double wl[2][4], w1[2][4], w0[2][4];
        weights_p3(tc[2].x, wl[0]);
        weights_p3(tc[1].x, w1[0]);
        weights_p3(tc[0].x, w0[0]);
        weights_p3(tc[2].y, wl[1]);
        weights_p3(tc[1].y, w1[1]);
        weights_p3(tc[0].y, w0[1]);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        double part[2][4];
        const unsigned X0 = xs_base + ((it & 1) * (kGrpMax * kGrpSS) + gc * kGrpSS) * sizeof(double);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double sa[2] = {0.0, 0.0};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                double2 lo, hi;
                const unsigned ad = X0 + (a * kGrpAS + b * 4) * sizeof(double);
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(lo.x), "=d"(lo.y) : "r"(ad));
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(hi.x), "=d"(hi.y) : "r"(ad + 16));
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    double s4 = fma(wl[n][0], lo.x, 0.0);
                    s4 = fma(wl[n][1], lo.y, s4);
                    s4 = fma(wl[n][2], hi.x, s4);
                    s4 = fma(wl[n][3], hi.y, s4);
                    sa[n] = fma(w1[n][b], s4, sa[n]);
                }
            }
#pragma unroll
            for (int n = 0; n < 2; ++n) part[n][a] = __dmul_rn(w0[n][a], sa[n]);
        }
        if (pc.x >= 0) v[pc.x] = (part[0][0] + part[0][1]) + (part[0][2] + part[0][3]);
        if (pc.y >= 0) v[pc.y] = (part[1][0] + part[1][1]) + (part[1][2] + part[1][3]);
        __syncthreads();  // cur is refilled two iterations on
#pragma unroll
        for (int a = 0; a < 3; ++a) tc[a] = tn[a];
        gc = gn;
        pc = pn;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#if __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

/** v = E x for d = 3, p = 3, grouped by stencil base with a UNION stage:
 *  slots as k_extend_grouped (two nodes of one stencil base per thread,
 *  chunks of kGrpThreads threads), but a chunk stages the union of its
 *  bases' x runs -- consecutive bases share most of their lattice lines, so
 *  ~2.8 staged values per node instead of 64 per base (11 per node) -- as one
 *  sorted list of active ordinals at a fixed stride (coalesced cp.async,
 *  mostly consecutive sources); each base addresses its 16 runs by 16-bit
 *  offsets into the stage.  Same pipeline (next chunk's x in flight by
 *  cp.async, the one after's tables in registers) and the same summation
 *  order: v is bit-identical to the gather kernel. */
__global__ void __launch_bounds__(kGrpThreads, 4) k_extend_union(int nchunks, int ns, const double* __restrict__ t,
                                                              const unsigned char* __restrict__ gslot,
                                                              const int* __restrict__ perm,
                                                              const int* __restrict__ stage,
                                                              const unsigned short* __restrict__ roff,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ v) {
    __shared__ __align__(16) double xs[2][kUnionMax];
    constexpr int NT = kGrpThreads, UR = kUnionMax / NT;
    const int G = gridDim.x;
    int o[UR];
    double2 tt[3];
    uint4 ro[2];
    int2 pp = make_int2(-1, -1);
    unsigned hb = 0;  // exact-hit flags of the two slots (bits 6, 7 of the slot byte)
    auto load_meta = [&](int c) {
        if (c >= nchunks) {
#pragma unroll
            for (int u = 0; u < UR; ++u) o[u] = -1;
            return;
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) o[u] = __ldg(stage + static_cast<std::size_t>(c) * kUnionMax + threadIdx.x + u * NT);
        const int th = c * kGrpThreads + threadIdx.x;  // slots 2 th, 2 th + 1
#pragma unroll
        for (int a = 0; a < 3; ++a) tt[a] = __ldg(reinterpret_cast<const double2*>(t + static_cast<std::size_t>(a) * ns) + th);
        const unsigned gb = __ldg(gslot + th);
        const int gs = static_cast<int>(gb & 63u);
        hb = gb >> 6;
        const uint4* rp = reinterpret_cast<const uint4*>(roff + (static_cast<std::size_t>(c) * kGrpMax + gs) * 16);
        ro[0] = __ldg(rp);
        ro[1] = __ldg(rp + 1);
        pp = __ldg(reinterpret_cast<const int2*>(perm) + th);
    };
    const unsigned xs_base = static_cast<unsigned>(__cvta_generic_to_shared(&xs[0][0]));
    auto issue_stage = [&](int buf) {
        const unsigned b0 = xs_base + static_cast<unsigned>((buf * kUnionMax + threadIdx.x) * 8);
#pragma unroll
        for (int u = 0; u < UR; ++u)
            if (o[u] >= 0)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(b0 + static_cast<unsigned>(u * NT * 8)),
                             "l"(x + o[u])
                             : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int c = blockIdx.x;
    load_meta(c);
    issue_stage(0);
    double2 tc[3] = {tt[0], tt[1], tt[2]};
    uint4 rc[2] = {ro[0], ro[1]};
    int2 pc = pp;
    unsigned hc = hb;
    load_meta(c + G);
    for (int it = 0; c < nchunks; ++it, c += G) {
        issue_stage((it + 1) & 1);  // chunk c + G (nothing past the end)
        const double2 tn[3] = {tt[0], tt[1], tt[2]};
        const uint4 rn[2] = {ro[0], ro[1]};
        const int2 pn = pp;
        const unsigned hn = hb;
        load_meta(c + 2 * G);
        double wl[2][4], w1[2][4], w0[2][4];
        // the exact-hit rule only where setup flagged a hit (same bits either
        // way; ~12 % fewer instructions)
        if (hc & 1u) {
            weights_p3(tc[2].x, wl[0]);
            weights_p3(tc[1].x, w1[0]);
            weights_p3(tc[0].x, w0[0]);
        } else {
            weights_p3_nohit(tc[2].x, wl[0]);
            weights_p3_nohit(tc[1].x, w1[0]);
            weights_p3_nohit(tc[0].x, w0[0]);
        }
        if (hc & 2u) {
            weights_p3(tc[2].y, wl[1]);
            weights_p3(tc[1].y, w1[1]);
            weights_p3(tc[0].y, w0[1]);
        } else {
            weights_p3_nohit(tc[2].y, wl[1]);
            weights_p3_nohit(tc[1].y, w1[1]);
            weights_p3_nohit(tc[0].y, w0[1]);
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const double* X = xs[it & 1];
        const unsigned rw[8] = {rc[0].x, rc[0].y, rc[0].z, rc[0].w, rc[1].x, rc[1].y, rc[1].z, rc[1].w};
        double part[2][4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double sa[2] = {0.0, 0.0};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int r = a * 4 + b;
                const int off = (rw[r >> 1] >> (16 * (r & 1))) & 0xffff;
                const double x0 = X[off], x1 = X[off + 1], x2 = X[off + 2], x3 = X[off + 3];
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    double s4 = fma(wl[n][0], x0, 0.0);
                    s4 = fma(wl[n][1], x1, s4);
                    s4 = fma(wl[n][2], x2, s4);
                    s4 = fma(wl[n][3], x3, s4);
                    sa[n] = fma(w1[n][b], s4, sa[n]);
                }
            }
#pragma unroll
            for (int n = 0; n < 2; ++n) part[n][a] = __dmul_rn(w0[n][a], sa[n]);
        }
        if (pc.x >= 0) v[pc.x] = (part[0][0] + part[0][1]) + (part[0][2] + part[0][3]);
        if (pc.y >= 0) v[pc.y] = (part[1][0] + part[1][1]) + (part[1][2] + part[1][3]);
        __syncthreads();  // this buffer is refilled two iterations on
#pragma unroll
        for (int a = 0; a < 3; ++a) tc[a] = tn[a];
        rc[0] = rn[0];
        rc[1] = rn[1];
        pc = pn;
        hc = hn;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#if __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

/** y = cg x - ih2 sum_k v[nbr_k], one active node per thread, the 2d
 *  neighbour codes of a node contiguous ([N_A][2d], 8-byte loads: a warp's
 *  codes are one contiguous 768-byte run).  Launched with programmatic
 *  stream serialization after the extension: codes and x are loaded before
 *  griddepcontrol.wait, so their latency overlaps the extension's tail; only
 *  the v gathers wait for it.  Same summation order as k_helm. */
template <int D>
__global__ void __launch_bounds__(256) k_helm_pdl(int na, double cg, double ih2, const int2* __restrict__ nbr2,
                                                  const double* __restrict__ v, const double* __restrict__ x,
                                                  double* __restrict__ y) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    int2 nb[D];
    double xi = 0.0;
    if (i < na) {
#pragma unroll
        for (int k = 0; k < D; ++k) nb[k] = __ldg(nbr2 + static_cast<std::size_t>(i) * D + k);
        xi = __ldg(x + i);
    }
#if __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    if (i >= na) return;
    double vv[2 * D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        vv[2 * k] = v[nb[k].x];  // written by the preceding kernel: no __ldg
        vv[2 * k + 1] = v[nb[k].y];
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) s += vv[k];
    y[i] = cg * xi - ih2 * s;
}

/** y = cg x - ih2 sum v[nbr]; if b != nullptr: y <- b - y and partial ||y||^2. */
template <int D, bool RESID>
__global__ void __launch_bounds__(kRedThreads) k_helm(int na, double cg, double ih2,
                                                      const int* __restrict__ nbr,
                                                      const double* __restrict__ v,
                                                      const double* __restrict__ x,
                                                      const double* __restrict__ b,
                                                      double* __restrict__ y, double* partials,
                                                      unsigned int* counter, double* result) {
    double local = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 2 * D; ++k) s += __ldg(v + __ldg(nbr + static_cast<std::size_t>(k) * na + i));
        const double ax = cg * __ldg(x + i) - ih2 * s;
        if constexpr (RESID) {
            const double r = __ldg(b + i) - ax;
            y[i] = r;
            local = fma(r, r, local);
        } else {
            y[i] = ax;
        }
    }
    if constexpr (RESID) {
        __shared__ double sh[kRedThreads / 32];
        __shared__ bool last;
        const double bs = block_sum<kRedThreads>(local, sh);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = bs;
            __threadfence();
            last = atomicInc(counter, gridDim.x - 1) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            double acc = 0.0;
            for (int q = threadIdx.x; q < static_cast<int>(gridDim.x); q += blockDim.x)
                acc += static_cast<volatile double*>(partials)[q];
            const double tot = block_sum<kRedThreads>(acc, sh);
            if (threadIdx.x == 0) *result = tot;
        }
    }
}

}  // namespace

// ---------------------------------------------------------------- host side

/** Stage lists of the staged extension (k_extend_staged): band nodes are cut
 *  into tiles of at most kExtTile consecutive nodes (halved until a tile's
 *  stage fits kExtStageCap entries, so several CTAs fit one SM); per tile, the
 *  sorted unique active ordinals its runs cover and every run's 16-bit start
 *  inside that list.  Left empty (gather kernel) if even a 32-node tile
 *  overflows the cap. */
static void build_stage(cpddg_op* op, const std::vector<int>& lines, const std::vector<double>& t, int nb) {
    constexpr int R = 16, Q = 4;
    // within a tile, threads take the nodes in order of their first stencil
    // run (x, y, z of the stencil base): the lanes of a warp then read the
    // same few stage rows, so a stencil read is ~1-2 shared-memory wavefronts
    // instead of one per column group in the warp
    std::vector<int> perm(static_cast<std::size_t>(nb));
    std::vector<double> tp(static_cast<std::size_t>(3) * nb);
    const int groups = (nb + kExtTile - 1) / kExtTile;
    struct Tile {
        int k0, k1;
        std::vector<int> u;
    };
    std::vector<std::vector<Tile>> parts(static_cast<std::size_t>(groups));
    std::vector<int> fail(static_cast<std::size_t>(groups), 0);
    std::vector<std::uint16_t> l16(static_cast<std::size_t>(R) * nb);
    auto stage_of = [&](int k0, int k1) {
        std::vector<int> st;
        st.reserve(static_cast<std::size_t>(R) * (k1 - k0));
        for (int l = 0; l < R; ++l)
            for (int k = k0; k < k1; ++k) st.push_back(lines[static_cast<std::size_t>(l) * nb + k]);
        std::sort(st.begin(), st.end());
        st.erase(std::unique(st.begin(), st.end()), st.end());
        std::vector<int> u;
        for (int o : st)  // union of [o, o + Q), runs sorted by start
            for (int c = (u.empty() ? 0 : std::max(0, u.back() - o + 1)); c < Q; ++c) u.push_back(o + c);
        return u;
    };
    parallel_for(groups, 0, [&](int g, int) {
        std::vector<std::pair<int, int>> todo{{g * kExtTile, std::min(nb, (g + 1) * kExtTile)}};
        auto& out = parts[static_cast<std::size_t>(g)];
        while (!todo.empty()) {
            const auto [k0, k1] = todo.back();
            todo.pop_back();
            std::vector<int> u = stage_of(k0, k1);
            if (static_cast<int>(u.size()) > kExtStageCap) {
                if (k1 - k0 <= 32) {
                    fail[static_cast<std::size_t>(g)] = 1;
                    return;
                }
                const int mid = k0 + (k1 - k0) / 2;
                todo.push_back({mid, k1});  // popped after [k0, mid): tiles stay in order
                todo.push_back({k0, mid});
                continue;
            }
            std::vector<int> ord(static_cast<std::size_t>(k1 - k0));
            std::iota(ord.begin(), ord.end(), k0);
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lines[a] < lines[b]; });
            for (int q = 0; q < k1 - k0; ++q) {
                const int k = ord[static_cast<std::size_t>(q)], slot = k0 + q;
                perm[static_cast<std::size_t>(slot)] = k;
                for (int a = 0; a < 3; ++a)
                    tp[static_cast<std::size_t>(a) * nb + slot] = t[static_cast<std::size_t>(a) * nb + k];
                for (int l = 0; l < R; ++l) {
                    const int o = lines[static_cast<std::size_t>(l) * nb + k];
                    l16[static_cast<std::size_t>(l) * nb + slot] =
                        static_cast<std::uint16_t>(std::lower_bound(u.begin(), u.end(), o) - u.begin());
                }
            }
            out.push_back({k0, k1, std::move(u)});
        }
    });
    for (int f : fail)
        if (f) return;
    std::vector<int> k0s, base{0}, idx;
    for (auto& ts : parts)
        for (auto& tl : ts) {
            k0s.push_back(tl.k0);
            idx.insert(idx.end(), tl.u.begin(), tl.u.end());
            base.push_back(static_cast<int>(idx.size()));
        }
    k0s.push_back(nb);
    op->lines16.upload(l16);
    op->ext_perm.upload(perm);
    op->ext_t.upload(tp);
    op->tile_k0.upload(k0s);
    op->stage_base.upload(base);
    op->stage_idx.upload(idx);
    op->ext_tiles = static_cast<int>(k0s.size()) - 1;
    op->ext_smem = kExtStageCap * static_cast<int>(sizeof(double));
    CPDDG_CUDA(cudaFuncSetAttribute(k_extend_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, op->ext_smem));
}

/** Slots of the grouped extension (k_extend_grouped): band nodes sorted by
 *  stencil base (the run start of offset (0, 0), an active ordinal unique to
 *  the base), then by code, taken two of one base per thread; chunks of
 *  kGrpThreads threads touching <= kGrpMax bases (a chunk closes early,
 *  padded with idle threads, when one more base would not fit; a base cut by
 *  a chunk boundary is staged in both). */
static void build_groups(cpddg_op* op, const std::vector<int>& lines, const std::vector<double>& t, int nb) {
    constexpr int R = 16;
    std::vector<int> ord(static_cast<std::size_t>(nb));
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lines[a] < lines[b]; });
    std::vector<int> perm;     // band code per slot (2 per thread), -1 idle
    std::vector<int> glines;   // [chunks][kGrpMax][16], -1 unused
    std::vector<unsigned char> gslot;  // per thread
    int nbase = 0, used = 0;   // bases / threads of the open chunk
    for (int q = 0; q < nb;) {
        const int k = ord[static_cast<std::size_t>(q)];
        const bool new_base = q == 0 || lines[k] != lines[ord[static_cast<std::size_t>(q) - 1]];
        if (q == 0 || used == kGrpThreads || (new_base && nbase == kGrpMax)) {
            perm.resize(perm.size() + 2 * kGrpThreads, -1);
            gslot.resize(gslot.size() + kGrpThreads, 0);
            glines.resize(glines.size() + kGrpMax * R, -1);
            nbase = used = 0;
        }
        if (new_base || nbase == 0) {  // first node of a base, or a base continued into a new chunk
            const std::size_t g = glines.size() - static_cast<std::size_t>(kGrpMax) * R + static_cast<std::size_t>(nbase) * R;
            for (int l = 0; l < R; ++l) glines[g + l] = lines[static_cast<std::size_t>(l) * nb + k];
            ++nbase;
        }
        const std::size_t th = gslot.size() - kGrpThreads + static_cast<std::size_t>(used++);
        gslot[th] = static_cast<unsigned char>(nbase - 1);
        perm[2 * th] = k;
        ++q;
        if (q < nb && lines[ord[static_cast<std::size_t>(q)]] == lines[k]) {  // second node of the same base
            perm[2 * th + 1] = ord[static_cast<std::size_t>(q)];
            ++q;
        }
    }
    const std::size_t ns = perm.size();
    std::vector<double> ts(3 * ns, 0.0);
    for (std::size_t sl = 0; sl < ns; ++sl)
        if (perm[sl] >= 0)
            for (int a = 0; a < 3; ++a) ts[static_cast<std::size_t>(a) * ns + sl] = t[static_cast<std::size_t>(a) * nb + perm[sl]];
    op->grp_t.upload(ts);
    op->grp_slot.upload(gslot);
    op->grp_perm.upload(perm);
    op->grp_lines.upload(glines);
    op->grp_chunks = static_cast<int>(gslot.size() / kGrpThreads);
    op->grp_slots = static_cast<int>(ns);
    int per_sm = 0;
    CPDDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extend_grouped, kGrpThreads, 0));
    op->grp_grid = std::max(1, std::min(op->grp_chunks, std::max(1, per_sm) * sm_count()));
}

/** Slots and union stages of k_extend_union: band nodes sorted by stencil
 *  base (then by code), two of one base per thread; a chunk closes when its
 *  kGrpThreads threads are used, at kGrpMax bases, or when the next base's
 *  runs would push the union stage past kUnionMax values (a base cut by a
 *  chunk boundary is staged in both).  The sorted sequence is cut at base
 *  boundaries into segments chunked independently on the host threads (a
 *  segment's last chunk may stay partly empty); v does not depend on the
 *  chunking. */
static void build_union(cpddg_op* op, const std::vector<int>& lines, const std::vector<double>& t, int nb) {
    constexpr int R = 16;
    std::vector<int> ord(static_cast<std::size_t>(nb));
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lines[a] < lines[b]; });
    struct Part {
        std::vector<int> perm, stage;      // per slot / [chunks][kUnionMax]
        std::vector<unsigned short> roff;  // [chunks][kGrpMax][16]
        std::vector<unsigned char> gslot;  // per thread
    };
    // segments of ~16 k nodes, cut where the base changes
    const int target = 16384;
    std::vector<int> cut{0};
    for (int q = target; q < nb; q += target) {
        int c = q;
        while (c < nb && lines[ord[static_cast<std::size_t>(c)]] == lines[ord[static_cast<std::size_t>(c) - 1]]) ++c;
        if (c < nb && c > cut.back()) cut.push_back(c);
    }
    cut.push_back(nb);
    const int nseg = static_cast<int>(cut.size()) - 1;
    std::vector<Part> parts(static_cast<std::size_t>(nseg));
    const int nworkers = std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
    std::vector<std::vector<int>> marks(static_cast<std::size_t>(nworkers));
    auto run_start = [&](int k, int l) { return lines[static_cast<std::size_t>(l) * nb + k]; };
    parallel_for(nseg, nworkers, [&](int sg, int w) {
        Part& P = parts[static_cast<std::size_t>(sg)];
        std::vector<int>& mark = marks[static_cast<std::size_t>(w)];
        if (mark.empty()) mark.assign(static_cast<std::size_t>(op->na), -1);
        std::vector<int> members, base_nodes;
        int nbase = 0, used = 0, chunk = -1;
        auto new_values = [&](int k) {  // staged values base k would add to the open chunk
            int add = 0;
            for (int l = 0; l < R; ++l)
                for (int q = 0; q < 4; ++q) {
                    const int ov = run_start(k, l) + q;
                    if (mark[static_cast<std::size_t>(ov)] != chunk) {
                        mark[static_cast<std::size_t>(ov)] = -2 - chunk;  // provisional
                        ++add;
                    }
                }
            for (int l = 0; l < R; ++l)
                for (int q = 0; q < 4; ++q) {
                    const int ov = run_start(k, l) + q;
                    if (mark[static_cast<std::size_t>(ov)] == -2 - chunk) mark[static_cast<std::size_t>(ov)] = -1;
                }
            return add;
        };
        auto close_chunk = [&] {
            if (chunk < 0) return;
            std::sort(members.begin(), members.end());
            const std::size_t s0 = static_cast<std::size_t>(chunk) * kUnionMax;
            for (std::size_t q = 0; q < members.size(); ++q) P.stage[s0 + q] = members[q];
            for (int b = 0; b < nbase; ++b)
                for (int l = 0; l < R; ++l) {
                    const int o = run_start(base_nodes[static_cast<std::size_t>(b)], l);
                    const std::size_t pos = static_cast<std::size_t>(std::lower_bound(members.begin(), members.end(), o) - members.begin());
                    P.roff[(static_cast<std::size_t>(chunk) * kGrpMax + b) * R + l] = static_cast<unsigned short>(pos);
                }
            for (int m : members) mark[static_cast<std::size_t>(m)] = -1;
            members.clear();
            base_nodes.clear();
        };
        auto open_chunk = [&] {
            close_chunk();
            ++chunk;
            P.perm.resize(P.perm.size() + 2 * kGrpThreads, -1);
            P.gslot.resize(P.gslot.size() + kGrpThreads, 0);
            P.stage.resize(P.stage.size() + kUnionMax, -1);
            P.roff.resize(P.roff.size() + static_cast<std::size_t>(kGrpMax) * R, 0);
            nbase = used = 0;
        };
        const int q0 = cut[static_cast<std::size_t>(sg)], q1 = cut[static_cast<std::size_t>(sg) + 1];
        for (int q = q0; q < q1;) {
            const int k = ord[static_cast<std::size_t>(q)];
            const bool new_base = q == q0 || lines[k] != lines[ord[static_cast<std::size_t>(q) - 1]];
            if (chunk < 0 || used == kGrpThreads || (new_base && nbase == kGrpMax) ||
                ((new_base || nbase == 0) && static_cast<int>(members.size()) + new_values(k) > kUnionMax))
                open_chunk();
            if (new_base || nbase == 0) {
                for (int l = 0; l < R; ++l)
                    for (int c = 0; c < 4; ++c) {
                        const int ov = run_start(k, l) + c;
                        if (mark[static_cast<std::size_t>(ov)] != chunk) {
                            mark[static_cast<std::size_t>(ov)] = chunk;
                            members.push_back(ov);
                        }
                    }
                if (static_cast<int>(members.size()) > kUnionMax)
                    throw InternalError("one stencil base exceeds the union stage");
                base_nodes.push_back(k);
                ++nbase;
            }
            const std::size_t th = P.gslot.size() - kGrpThreads + static_cast<std::size_t>(used++);
            P.gslot[th] = static_cast<unsigned char>(nbase - 1);
            P.perm[2 * th] = k;
            ++q;
            if (q < q1 && lines[ord[static_cast<std::size_t>(q)]] == lines[k]) {
                P.perm[2 * th + 1] = ord[static_cast<std::size_t>(q)];
                ++q;
            }
        }
        close_chunk();
        // exact-hit flags (bits 6 and 7 of the slot byte): the kernel applies
        // interp.hpp:39-44's rule only to flagged slots -- same test, same doubles
        for (std::size_t th = 0; th < P.gslot.size(); ++th)
            for (int n = 0; n < 2; ++n) {
                const int k = P.perm[2 * th + static_cast<std::size_t>(n)];
                if (k < 0) continue;
                bool hit = false;
                for (int a = 0; a < 3; ++a)
                    for (int j = 0; j <= 3; ++j)
                        hit = hit || std::fabs(t[static_cast<std::size_t>(a) * nb + k] - static_cast<double>(j)) < 1e-12;
                if (hit) P.gslot[th] = static_cast<unsigned char>(P.gslot[th] | (64u << n));
            }
    });
    std::vector<int> perm, stage;
    std::vector<unsigned short> roff;
    std::vector<unsigned char> gslot;
    for (const Part& P : parts) {
        perm.insert(perm.end(), P.perm.begin(), P.perm.end());
        stage.insert(stage.end(), P.stage.begin(), P.stage.end());
        roff.insert(roff.end(), P.roff.begin(), P.roff.end());
        gslot.insert(gslot.end(), P.gslot.begin(), P.gslot.end());
    }
    const std::size_t ns = perm.size();
    std::vector<double> ts(3 * ns, 0.0);
    parallel_for(static_cast<int>((ns + 65535) / 65536), 0, [&](int c, int) {
        const std::size_t e = std::min(ns, (static_cast<std::size_t>(c) + 1) * 65536);
        for (std::size_t sl = static_cast<std::size_t>(c) * 65536; sl < e; ++sl)
            if (perm[sl] >= 0)
                for (int a = 0; a < 3; ++a) ts[static_cast<std::size_t>(a) * ns + sl] = t[static_cast<std::size_t>(a) * nb + perm[sl]];
    });
    op->grp_t.upload(ts);
    op->grp_slot.upload(gslot);
    op->grp_perm.upload(perm);
    op->uni_stage.upload(stage);
    op->uni_roff.upload(roff);
    op->grp_chunks = static_cast<int>(gslot.size() / kGrpThreads);
    op->grp_slots = static_cast<int>(ns);
    op->uni = true;
    int per_sm = 0;
    CPDDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extend_union, kGrpThreads, 0));
    op->grp_grid = std::max(1, std::min(op->grp_chunks, std::max(1, per_sm) * sm_count()));
}

/** The union kernel's tables, the node-major neighbour codes and v move into
 *  one slab, and the device sets aside persisting L2 for it: launch_apply puts
 *  an access-policy window over the slab (hits persist, everything else the
 *  two kernels touch streams), so the ~50 MB the operator re-reads every
 *  iteration survive the preconditioner's and the orthogonalisation's traffic.
 *  CPDDG_OP_L2=0 leaves the tables where they are (no window). */
static void pack_tables(cpddg_op* op) {
    const char* e = std::getenv("CPDDG_OP_L2");
    if (e && std::string(e) == "0") return;
    int dev = 0;
    cudaDeviceProp prop{};
    CPDDG_CUDA(cudaGetDevice(&dev));
    CPDDG_CUDA(cudaGetDeviceProperties(&prop, dev));
    auto up = [](std::size_t b) { return (b + 255) / 256 * 256; };
    const std::size_t total = up(op->grp_t.bytes()) + up(op->grp_slot.bytes()) + up(op->grp_perm.bytes()) +
                              up(op->uni_stage.bytes()) + up(op->uni_roff.bytes()) + up(op->nbr_aos.bytes()) +
                              up(op->v.bytes());
    if (prop.persistingL2CacheMaxSize <= 0 || prop.accessPolicyMaxWindowSize <= 0 ||
        total > static_cast<std::size_t>(prop.accessPolicyMaxWindowSize) ||
        total > static_cast<std::size_t>(prop.persistingL2CacheMaxSize))
        return;  // does not fit a window / the carve-out: stay with the separate buffers
    op->slab.alloc(total);
    std::size_t at = 0;
    auto move = [&](auto& buf) {
        using T = std::remove_pointer_t<decltype(buf.get())>;
        const std::size_t n = buf.size();
        T* dst = reinterpret_cast<T*>(op->slab.get() + at);
        if (n) CPDDG_CUDA(cudaMemcpy(dst, buf.get(), n * sizeof(T), cudaMemcpyDeviceToDevice));
        at += up(n * sizeof(T));
        buf.view(dst, n);
    };
    move(op->grp_t);
    move(op->grp_slot);
    move(op->grp_perm);
    move(op->uni_stage);
    move(op->uni_roff);
    move(op->nbr_aos);
    move(op->v);
    std::size_t have = 0;
    CPDDG_CUDA(cudaDeviceGetLimit(&have, cudaLimitPersistingL2CacheSize));
    if (have < total) CPDDG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, total));
    op->l2_window = total;
}

template <int D>
static void build_tables(cpddg_op* op, const Ix<D>* ix, const Vec<D>* cp, const LatticeMap& map) {
    const int nb = op->na + op->ng, p = op->p, Q = p + 1;
    int nlines = 1;
    for (int a = 0; a < D - 1; ++a) nlines *= Q;
    std::vector<double> t(static_cast<std::size_t>(D) * nb);
    std::vector<int> lines(static_cast<std::size_t>(nlines) * nb);
    auto lookup = [&](const Ix<D>& q) { return map.find(LatticeMap::pack(q.data(), D)); };
    auto t_lap = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {  // CPDDG_VERBOSE: host wall time of the table phases
        if (!std::getenv("CPDDG_VERBOSE")) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[cpddg] op tables, %s: %.3f s\n", what, std::chrono::duration<double>(now - t_lap).count());
        t_lap = now;
    };
    parallel_for((nb + 8191) / 8192, 0, [&](int chunk, int) {
        const int k1 = std::min(nb, (chunk + 1) * 8192);
        for (int k = chunk * 8192; k < k1; ++k) {
            const Stencil1D<D> s = stencil_of<D>(cp[k], op->h, p);
            for (int a = 0; a < D; ++a) {
                const double g = (cp[k][a] - 0.0) / op->h;
                t[static_cast<std::size_t>(a) * nb + k] = g - s.base[a];
            }
            for (int l = 0; l < nlines; ++l) {
                Ix<D> q;
                int rem = l;
                for (int a = D - 2; a >= 0; --a) {
                    q[a] = s.base[a] + rem % Q;
                    rem /= Q;
                }
                q[D - 1] = s.base[D - 1];
                const std::int64_t o = lookup(q);
                if (o < 0 || o >= op->na)
                    throw InternalError("extension stencil node is not active: band closure violated");
                for (int c = 1; c < Q; ++c) {
                    Ix<D> r = q;
                    r[D - 1] += c;
                    if (lookup(r) != o + c)
                        throw InternalError("stencil run is not contiguous in band order");
                }
                lines[static_cast<std::size_t>(l) * nb + k] = static_cast<int>(o);
            }
        }
    });
    lap("stencil offsets and run starts");
    std::vector<int> nbr(static_cast<std::size_t>(2 * D) * op->na);
    std::vector<int> aos(nbr.size());  // node-major copy for k_helm_pdl
    parallel_for((op->na + 8191) / 8192, 0, [&](int chunk, int) {
        const int i1 = std::min(op->na, (chunk + 1) * 8192);
        for (int i = chunk * 8192; i < i1; ++i) {
            Ix<D> around[2 * D];
            neighbors_of<D>(ix[i], around);
            for (int k = 0; k < 2 * D; ++k) {
                const std::int64_t c = lookup(around[k]);
                if (c < 0) throw InternalError("finite-difference neighbor missing from band");
                nbr[static_cast<std::size_t>(k) * op->na + i] = static_cast<int>(c);
                aos[static_cast<std::size_t>(i) * 2 * D + k] = static_cast<int>(c);
            }
        }
    });
    lap("neighbour codes");
    if constexpr (D == 3) {
        // default: grouped by stencil base; CPDDG_EXT=staged / CPDDG_EXT_GATHER=1
        // keep the round-1 tiled-stage and gather kernels (same v bits)
        const char* ext = std::getenv("CPDDG_EXT");
        if (p == 3 && !std::getenv("CPDDG_EXT_GATHER")) {
            if (ext && std::string(ext) == "staged") {
                build_stage(op, lines, t, nb);
            } else if (ext && std::string(ext) == "grouped") {
                build_groups(op, lines, t, nb);
            } else {
                build_union(op, lines, t, nb);
            }
        }
    }
    lap("extension slots and stages");
    op->t.upload(t);
    op->lines.upload(lines);
    op->nbr.upload(nbr);
    op->nbr_aos.upload(aos);
    op->v.alloc(static_cast<std::size_t>(nb));
    if (op->uni) pack_tables(op);
    lap("uploads");
    op->nlines = nlines;
    // B_op = 16 N_A + [8d + 4 (p+1)^(d-1)] N_B + 8d N_A
    op->alg_bytes = 16LL * op->na + (8LL * D + 4LL * nlines) * nb + 8LL * D * op->na;
    // streamed: x read + y write, t + lines per band node, v write+read, nbr
    op->streamed_bytes = 16LL * op->na + (8LL * D + 4LL * nlines) * nb + 16LL * nb + 8LL * D * op->na;
    if (op->ext_tiles)  // staged: 16-bit run starts + one int per staged x
        op->streamed_bytes += (2LL - 4LL) * nlines * nb + 4LL * static_cast<long long>(op->stage_idx.size());
    if (op->uni)  // union: t + code per slot, a byte per thread, the stage list and 16-bit run offsets
        op->streamed_bytes = 16LL * op->na + (8LL * D + 4) * op->grp_slots + op->grp_slots / 2 + 16LL * nb +
                             8LL * D * op->na + 4LL * static_cast<long long>(op->uni_stage.size()) +
                             2LL * static_cast<long long>(op->uni_roff.size());
    else if (op->grp_chunks)  // grouped: t + one byte per slot, kGrpMax x 16 run starts per chunk
        op->streamed_bytes = 16LL * op->na + (8LL * D + 4) * op->grp_slots + op->grp_slots / 2 + 16LL * nb +
                             8LL * D * op->na + 4LL * static_cast<long long>(op->grp_lines.size());
}

template <int D>
static void launch_apply(const cpddg_op* op, const double* x, const double* b, double* y, double* rn2,
                         cudaStream_t st, bool pdl = true) {
    const int nb = op->na + op->ng;
    const int thr = 256;
    cudaLaunchAttribute l2attr{};
    l2attr.id = cudaLaunchAttributeAccessPolicyWindow;
    l2attr.val.accessPolicyWindow.base_ptr = op->slab.get();
    l2attr.val.accessPolicyWindow.num_bytes = op->l2_window;
    l2attr.val.accessPolicyWindow.hitRatio = 1.0f;
    l2attr.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    l2attr.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (op->uni) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(op->grp_grid);
        cfg.blockDim = dim3(kGrpThreads);
        cfg.stream = st;
        cfg.attrs = &l2attr;
        cfg.numAttrs = op->l2_window ? 1 : 0;
        CPDDG_CUDA(cudaLaunchKernelEx(&cfg, k_extend_union, op->grp_chunks, op->grp_slots,
                                      static_cast<const double*>(op->grp_t.get()),
                                      static_cast<const unsigned char*>(op->grp_slot.get()),
                                      static_cast<const int*>(op->grp_perm.get()),
                                      static_cast<const int*>(op->uni_stage.get()),
                                      static_cast<const unsigned short*>(op->uni_roff.get()), x, op->v.get()));
    } else if (op->grp_chunks) {
        k_extend_grouped<<<op->grp_grid, kGrpThreads, 0, st>>>(op->grp_chunks, op->grp_slots, op->grp_t.get(),
                                                                  op->grp_slot.get(), op->grp_perm.get(),
                                                                  op->grp_lines.get(), x, op->v.get());
    } else if (op->ext_tiles) {
        k_extend_staged<<<op->ext_tiles, kExtTile, op->ext_smem, st>>>(nb, op->ext_t.get(), op->lines16.get(),
                                                                       op->ext_perm.get(), op->tile_k0.get(),
                                                                       op->stage_base.get(), op->stage_idx.get(), x,
                                                                       op->v.get());
    } else if (op->p == 3) {
        const long long threads = 4LL * nb;
        k_extend_p3<D><<<static_cast<int>((threads + thr - 1) / thr), thr, 0, st>>>(nb, op->t.get(), op->lines.get(), x,
                                                                                  op->v.get());
    } else switch (op->p) {
#define CPDDG_EXT(PP) \
    case PP: k_extend<D, PP><<<(nb + thr - 1) / thr, thr, 0, st>>>(nb, op->t.get(), op->lines.get(), x, op->v.get()); break;
        CPDDG_EXT(1) CPDDG_EXT(2) CPDDG_EXT(3) CPDDG_EXT(4) CPDDG_EXT(5) CPDDG_EXT(6) CPDDG_EXT(7)
#undef CPDDG_EXT
        default: throw ConfigError("interpolation degree must be in [1,7]");
    }
    CPDDG_CUDA(cudaGetLastError());
    const int rb = reduction_blocks();
    const int grid = std::min(rb, (op->na + kRedThreads - 1) / kRedThreads);
    if (!b && op->grp_chunks) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((op->na + 255) / 256);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        int na_ = 0;
        if (pdl) {
            attr[na_].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[na_].val.programmaticStreamSerializationAllowed = 1;
            ++na_;
        }
        if (op->l2_window) attr[na_++] = l2attr;
        cfg.attrs = attr;
        cfg.numAttrs = na_;
        CPDDG_CUDA(cudaLaunchKernelEx(&cfg, k_helm_pdl<D>, op->na, op->cg, op->ih2,
                                      reinterpret_cast<const int2*>(op->nbr_aos.get()),
                                      static_cast<const double*>(op->v.get()), x, y));
    } else if (b)
        k_helm<D, true><<<rb, kRedThreads, 0, st>>>(op->na, op->cg, op->ih2, op->nbr.get(), op->v.get(), x,
                                                    b, y, op->red.partials.get(), op->red.counter.get(), rn2);
    else
        k_helm<D, false><<<std::max(grid, 1), kRedThreads, 0, st>>>(op->na, op->cg, op->ih2, op->nbr.get(),
                                                                   op->v.get(), x, nullptr, y, nullptr,
                                                                   nullptr, nullptr);
    CPDDG_CUDA(cudaGetLastError());
}

void op_apply(const cpddg_op* op, const double* x, double* y, cudaStream_t st, bool pdl) {
    if (op->dim == 2)
        launch_apply<2>(op, x, nullptr, y, nullptr, st, pdl);
    else
        launch_apply<3>(op, x, nullptr, y, nullptr, st, pdl);
}

void op_residual(const cpddg_op* op, const double* b, const double* x, double* r, double* rn2_dev,
                 cudaStream_t st) {
    if (op->dim == 2)
        launch_apply<2>(op, x, b, r, rn2_dev, st);
    else
        launch_apply<3>(op, x, b, r, rn2_dev, st);
}

template <int D>
static cpddg_op* create_from(int p, int na, int ng, double h, double c, const Ix<D>* ix, const Vec<D>* cp,
                             const LatticeMap* map_in) {
    if (c <= 0) throw ConfigError("Helmholtz constant c must be positive");
    if (!(h > 0)) throw ConfigError("grid spacing h must be positive");
    if (p < 1 || p > 7) throw ConfigError("interpolation degree must be in [1,7]");
    auto op = std::make_unique<cpddg_op>();
    op->dim = D;
    op->p = p;
    op->na = na;
    op->ng = ng;
    op->h = h;
    op->c = c;
    op->cg = c + 2.0 * D / (h * h);
    op->ih2 = 1.0 / (h * h);
    LatticeMap own;
    const LatticeMap* map = map_in;
    if (!map) {
        own.reserve(static_cast<std::size_t>(na + ng));
        for (int k = 0; k < na + ng; ++k)
            if (!own.insert(LatticeMap::pack(ix[k].data(), D), k))
                throw InternalError("duplicate lattice index in band description");
        map = &own;
    }
    const auto t0 = std::chrono::steady_clock::now();
    build_tables<D>(op.get(), ix, cp, *map);
    if (std::getenv("CPDDG_VERBOSE"))
        std::fprintf(stderr, "[cpddg] op tables: %.3f s\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    op->red.ensure(1);
    op->rn2.alloc(1);
    return op.release();
}

}  // namespace cpddg

using namespace cpddg;

extern "C" {

int cpddg_op_create(const cpddg_band_desc* d, cpddg_op** out) {
    return guarded([&] {
        if (!d || !out || !d->ix || !d->cp) throw InternalError("null argument");
        if (d->n_active <= 0) throw ConfigError("band is empty");
        const int nb = d->n_active + d->n_ghost;
        if (d->dim == 2) {
            std::vector<Ix<2>> ix(static_cast<std::size_t>(nb));
            std::vector<Vec<2>> cp(static_cast<std::size_t>(nb));
            for (int k = 0; k < nb; ++k)
                for (int a = 0; a < 2; ++a) {
                    ix[static_cast<std::size_t>(k)][a] = d->ix[2 * k + a];
                    cp[static_cast<std::size_t>(k)][a] = d->cp[2 * k + a];
                }
            *out = create_from<2>(d->p, d->n_active, d->n_ghost, d->h, d->c, ix.data(), cp.data(), nullptr);
        } else if (d->dim == 3) {
            std::vector<Ix<3>> ix(static_cast<std::size_t>(nb));
            std::vector<Vec<3>> cp(static_cast<std::size_t>(nb));
            for (int k = 0; k < nb; ++k)
                for (int a = 0; a < 3; ++a) {
                    ix[static_cast<std::size_t>(k)][a] = d->ix[3 * k + a];
                    cp[static_cast<std::size_t>(k)][a] = d->cp[3 * k + a];
                }
            *out = create_from<3>(d->p, d->n_active, d->n_ghost, d->h, d->c, ix.data(), cp.data(), nullptr);
        } else {
            throw ConfigError("dimension must be 2 or 3");
        }
    });
}

int cpddg_op_create_from_setup(const cpddg_setup* s, cpddg_op** out) {
    return guarded([&] {
        if (!s || !out) throw InternalError("null argument");
        if (s->dim == 2) {
            auto& I = impl_of<2>(s);
            *out = create_from<2>(I.band.p, I.band.n_active, I.band.n_ghost, I.band.h, s->c, I.band.ix.data(),
                                  I.band.cp.data(), &I.band.map);
        } else {
            auto& I = impl_of<3>(s);
            *out = create_from<3>(I.band.p, I.band.n_active, I.band.n_ghost, I.band.h, s->c, I.band.ix.data(),
                                  I.band.cp.data(), &I.band.map);
        }
    });
}

int cpddg_op_apply(cpddg_op* op, const double* x, double* y, void* stream) {
    return guarded([&] {
        if (!op || !x || !y) throw InternalError("null argument");
        op_apply(op, x, y, static_cast<cudaStream_t>(stream));
    });
}

int cpddg_op_residual(cpddg_op* op, const double* b, const double* x, double* r, double* rnorm, void* stream) {
    return guarded([&] {
        if (!op || !b || !x || !r) throw InternalError("null argument");
        auto st = static_cast<cudaStream_t>(stream);
        op_residual(op, b, x, r, op->rn2.get(), st);
        double h = 0;
        CPDDG_CUDA(cudaMemcpyAsync(&h, op->rn2.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
        if (rnorm) *rnorm = std::sqrt(h);
    });
}

int cpddg_op_size(const cpddg_op* op) { return op ? op->na : -1; }

int cpddg_op_bytes(const cpddg_op* op, int64_t* alg, int64_t* streamed) {
    return guarded([&] {
        if (!op) throw InternalError("null argument");
        if (alg) *alg = op->alg_bytes;
        if (streamed) *streamed = op->streamed_bytes;
    });
}

int cpddg_op_destroy(cpddg_op* op) {
    if (op && op->l2_window) cudaCtxResetPersistingL2Cache();  // its persisting lines return to normal use
    delete op;
    return CPDDG_OK;
}

}  // extern "C"
