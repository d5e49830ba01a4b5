// Device-resident Krylov drivers: restarted right-preconditioned GMRES with
// modified Gram-Schmidt (solve.hpp:128-214) and the stationary Schwarz
// iteration (solve.hpp:95-123).
//
// All vectors (basis V, w, r, u) live in HBM; the host keeps only the
// (m+2)-entry Hessenberg column, the Givens rotations and the residual
// history -- the reference's own scalar arithmetic, in the same order, so
// the rotated estimates follow the reference step for step.  Each MGS step
// is one fused streaming pass `w -= h_{i-1} V_{i-1}; h_i = V_i . w`
// (deterministic two-level reduction, last-block-done), the norm of the
// operator image rides on the first pass, and the correction
// u += M^-1 (V y) scatters straight into u (owned slots are disjoint).
#include "../host/setup.hpp"
#include "common.cuh"
#include "op.cuh"
#include "setup_dev.cuh"

#include <cooperative_groups.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace cpddg {

namespace {

/** One MGS pass over w.  If vprev: w -= (*hprev) * vprev.  Then
 *  out[0] = vnext . w (or w . w when vnext == nullptr); if out2:
 *  out2[0] = w . w as well.  Deterministic: fixed grid, fixed-order sums. */
__global__ void __launch_bounds__(kRedThreads) k_mgs(int n, const double* __restrict__ hprev,
                                                     const double* __restrict__ vprev, double* __restrict__ w,
                                                     const double* __restrict__ vnext, double* partials,
                                                     unsigned int* counter, double* out, double* out2) {
    const double h = vprev ? *hprev : 0.0;
    double a1 = 0.0, a2 = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double wi = w[i];
        if (vprev) {
            wi -= h * __ldg(vprev + i);
            w[i] = wi;
        }
        a1 = fma(vnext ? __ldg(vnext + i) : wi, wi, a1);
        if (out2) a2 = fma(wi, wi, a2);
    }
    __shared__ double sh[kRedThreads / 32];
    __shared__ bool last;
    const double b1 = block_sum<kRedThreads>(a1, sh);
    const double b2 = out2 ? block_sum<kRedThreads>(a2, sh) : 0.0;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = b1;
        partials[gridDim.x + blockIdx.x] = b2;
        __threadfence();
        last = atomicInc(counter, gridDim.x - 1) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double s1 = 0.0, s2 = 0.0;
        for (int q = threadIdx.x; q < static_cast<int>(gridDim.x); q += blockDim.x) {
            s1 += static_cast<volatile double*>(partials)[q];
            s2 += static_cast<volatile double*>(partials)[gridDim.x + q];
        }
        const double t1 = block_sum<kRedThreads>(s1, sh);
        const double t2 = out2 ? block_sum<kRedThreads>(s2, sh) : 0.0;
        if (threadIdx.x == 0) {
            *out = t1;
            if (out2) *out2 = t2;
        }
    }
}

/** The whole modified Gram-Schmidt step of one Arnoldi iteration in one
 *  cooperative launch (solve.hpp:162-169, then the basis scaling of :195):
 *    pass 0:        h_0 = V_0 . w,  ||w||^2 (before orthogonalisation)
 *    pass i=1..m:   w -= h_{i-1} V_{i-1};  h_i = V_i . w
 *    pass m+1:      w -= h_m V_m;  h_{m+1} = w . w
 *    then           V_{m+1} = w / sqrt(h_{m+1})   (speculative; unused if the host stops)
 *  Passes are separated by grid-wide barriers; every block re-sums the
 *  per-block partials of a pass in the same fixed order, so all blocks hold
 *  the identical h_i without a second barrier and results are bitwise
 *  deterministic (fixed grid).  h[0..m+1] and ||w0||^2 land in `hout`. */
__global__ void __launch_bounds__(kRedThreads) k_mgs_all(int n, int m, const double* const* __restrict__ V,
                                                         double* __restrict__ w, double* __restrict__ vnext,
                                                         double* partials, double* hout, double* wn0,
                                                         const int* __restrict__ mdev, double* __restrict__ vin) {
    if (mdev) {  // device-driven Arnoldi: step from the solver state, V_{m+1} and ||w0||^2 slot follow
        m = *mdev;
        vnext = const_cast<double*>(V[m + 1]);
        wn0 = hout + m + 2;
    }
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kRedThreads / 32];
    __shared__ double hb;
    const int nb = gridDim.x;
    const int stride = gridDim.x * blockDim.x;
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    double hprev = 0.0;
    for (int pass = 0; pass <= m + 1; ++pass) {
        const double* vp = pass > 0 ? V[pass - 1] : nullptr;
        const double* vn = pass <= m ? V[pass] : nullptr;
        double a1 = 0.0, a2 = 0.0;
        for (int i = i0; i < n; i += stride) {
            double wi = w[i];
            if (vp) {
                wi -= hprev * vp[i];
                w[i] = wi;
            }
            a1 = fma(vn ? vn[i] : wi, wi, a1);
            if (pass == 0) a2 = fma(wi, wi, a2);
        }
        const double b1 = block_sum<kRedThreads>(a1, sh);
        const double b2 = pass == 0 ? block_sum<kRedThreads>(a2, sh) : 0.0;
        double* slot = partials + static_cast<std::size_t>(pass) * 2 * nb;
        if (threadIdx.x == 0) {
            slot[blockIdx.x] = b1;
            slot[nb + blockIdx.x] = b2;
        }
        grid.sync();
        double s1 = 0.0, s2 = 0.0;
        for (int q = threadIdx.x; q < nb; q += blockDim.x) {
            s1 += slot[q];
            if (pass == 0) s2 += slot[nb + q];
        }
        const double t1 = block_sum<kRedThreads>(s1, sh);
        const double t2 = pass == 0 ? block_sum<kRedThreads>(s2, sh) : 0.0;
        if (threadIdx.x == 0) {
            hb = t1;
            if (blockIdx.x == 0) {
                hout[pass] = t1;
                if (pass == 0) *wn0 = t2;
            }
        }
        __syncthreads();
        hprev = hb;
    }
    // hprev = ||w||^2 after the last pass: speculative next basis vector
    const double sub = sqrt(hprev);
    if (vnext)
        for (int i = i0; i < n; i += stride) {
            const double v = w[i] / sub;
            vnext[i] = v;
            if (vin) vin[i] = v;
        }
}

/** k_mgs_all with the thread's slice of w and of the previous basis vector
 *  held in registers across passes (EPT elements per thread, same index
 *  mapping, same summation order -- bit-identical results): a pass streams
 *  one basis vector (8n bytes) instead of w twice and two basis vectors
 *  (32n bytes). */
template <int EPT>
__global__ void __launch_bounds__(kRedThreads) k_mgs_reg(int n, int m, const double* const* __restrict__ V,
                                                         double* __restrict__ w, double* __restrict__ vnext,
                                                         double* partials, double* hout, double* wn0,
                                                         const int* __restrict__ mdev, double* __restrict__ vin) {
    if (mdev) {
        m = *mdev;
        vnext = const_cast<double*>(V[m + 1]);
        wn0 = hout + m + 2;
    }
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kRedThreads / 32];
    __shared__ double hb;
    const int nb = gridDim.x;
    const int stride = gridDim.x * blockDim.x;
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    // vc: this pass's basis vector slice, loaded during the previous pass
    // (before its grid barrier: the loads do not depend on h)
    double wr[EPT], vr[EPT], vc[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int i = i0 + k * stride;
        wr[k] = i < n ? w[i] : 0.0;
        vr[k] = 0.0;
        vc[k] = (i < n && m >= 0) ? __ldcg(V[0] + i) : 0.0;
    }
    double hprev = 0.0;
    for (int pass = 0; pass <= m + 1; ++pass) {
        const bool has_v = pass <= m;
        double a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int i = i0 + k * stride;
            if (i < n) {
                double wi = wr[k];
                if (pass > 0) {
                    wi -= hprev * vr[k];
                    wr[k] = wi;
                }
                const double vi = has_v ? vc[k] : wi;
                vr[k] = vi;
                a1 = fma(vi, wi, a1);
                if (pass == 0) a2 = fma(wi, wi, a2);
            }
        }
        if (pass + 1 <= m) {
            const double* vn = V[pass + 1];
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const int i = i0 + k * stride;
                vc[k] = i < n ? __ldcg(vn + i) : 0.0;
            }
        }
        const double b1 = block_sum<kRedThreads>(a1, sh);
        const double b2 = pass == 0 ? block_sum<kRedThreads>(a2, sh) : 0.0;
        double* slot = partials + static_cast<std::size_t>(pass) * 2 * nb;
        if (threadIdx.x == 0) {
            slot[blockIdx.x] = b1;
            slot[nb + blockIdx.x] = b2;
        }
        grid.sync();
        double s1 = 0.0, s2 = 0.0;
        for (int q = threadIdx.x; q < nb; q += blockDim.x) {
            s1 += slot[q];
            if (pass == 0) s2 += slot[nb + q];
        }
        const double t1 = block_sum<kRedThreads>(s1, sh);
        const double t2 = pass == 0 ? block_sum<kRedThreads>(s2, sh) : 0.0;
        if (threadIdx.x == 0) {
            hb = t1;
            if (blockIdx.x == 0) {
                hout[pass] = t1;
                if (pass == 0) *wn0 = t2;
            }
        }
        __syncthreads();
        hprev = hb;
    }
    const double sub = sqrt(hprev);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int i = i0 + k * stride;
        if (i < n) {
            w[i] = wr[k];
            if (vnext) {
                const double v = wr[k] / sub;
                vnext[i] = v;
                if (vin) vin[i] = v;
            }
        }
    }
}

/** Three block sums behind one pair of barriers (results valid in thread 0). */
template <int NT>
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sh /* [3 NT / 32] */) {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[w] = a;
        sh[NT / 32 + w] = b;
        sh[2 * (NT / 32) + w] = c;
    }
    __syncthreads();
    if (w == 0) {
        a = warp_sum(l < NT / 32 ? sh[l] : 0.0);
        b = warp_sum(l < NT / 32 ? sh[NT / 32 + l] : 0.0);
        c = warp_sum(l < NT / 32 ? sh[2 * (NT / 32) + l] : 0.0);
    }
    __syncthreads();
}

/** k_mgs_reg with TWO projections per grid barrier.  A pass loads the basis
 *  vectors V_a, V_b (a = 2 pass, b = a + 1) and reduces
 *      d1 = V_a . w,   d2 = V_b . w,   c = V_b . V_a
 *  together; then h_a = d1 and h_b = d2 - h_a c, which IS the modified
 *  Gram-Schmidt coefficient V_b . (w - h_a V_a) with the subtraction moved
 *  across the dot product (exact algebra; c is the basis' own loss of
 *  orthogonality, ~1e-16).  w is then updated as MGS does, one vector after
 *  the other.  Half the grid barriers of k_mgs_reg (the barriers, not the
 *  bytes, are what an MGS step costs: ~3.4 us each, j + 2 of them at step j);
 *  coefficients agree with k_mgs_reg to rounding (tests/test_gpu_parity.py).
 *  Pass 0 also reduces ||w||^2; the last pass reduces ||w||^2 of the
 *  orthogonalised w.  Same index mapping and fixed summation orders: bitwise
 *  reproducible run to run. */
template <int EPT, int NT = kRedThreads>
__global__ void __launch_bounds__(NT, NT == kRedThreads ? 2 : 1) k_mgs_pair(int n, int m, const double* const* __restrict__ V,
                                                          double* __restrict__ w, double* __restrict__ vnext,
                                                          double* partials, double* hout, double* wn0,
                                                          const int* __restrict__ mdev, double* __restrict__ vin) {
    if (mdev) {
        m = *mdev;
        vnext = const_cast<double*>(V[m + 1]);
        wn0 = hout + m + 2;
    }
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[3 * (NT / 32)];
    __shared__ double hb[3];
    const int nb = gridDim.x;
    const int stride = gridDim.x * blockDim.x;
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    const int npair = (m + 2) / 2;  // dot passes: vectors (0, 1), (2, 3), ...; the last may be single
    double wr[EPT], pa[EPT], pb[EPT], ca[EPT], cb[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int i = i0 + k * stride;
        wr[k] = i < n ? w[i] : 0.0;
        pa[k] = pb[k] = 0.0;
        ca[k] = (i < n && m >= 0) ? __ldcg(V[0] + i) : 0.0;
        cb[k] = (i < n && m >= 1) ? __ldcg(V[1] + i) : 0.0;
    }
    double ha = 0.0, hbv = 0.0;  // the previous pair's coefficients
    for (int pass = 0; pass <= npair; ++pass) {
        const bool dots = pass < npair;
        const bool two = dots && 2 * pass + 1 <= m;
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int i = i0 + k * stride;
            if (i < n) {
                double wi = wr[k];
                if (pass > 0) {  // MGS update with the previous pair, one vector after the other
                    wi -= ha * pa[k];
                    wi -= hbv * pb[k];
                    wr[k] = wi;
                }
                if (dots) {
                    s1 = fma(ca[k], wi, s1);
                    if (two) {
                        s2 = fma(cb[k], wi, s2);
                        s3 = fma(cb[k], ca[k], s3);
                    }
                } else {
                    s1 = fma(wi, wi, s1);  // ||w||^2 after the last update
                }
            }
        }
        // pass 0 carries ||w0||^2 in a fourth sum
        double s4 = 0.0;
        if (pass == 0) {
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const int i = i0 + k * stride;
                if (i < n) s4 = fma(wr[k], wr[k], s4);
            }
        }
        if (dots) {
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                pa[k] = ca[k];
                pb[k] = two ? cb[k] : 0.0;
            }
            const int na = 2 * pass + 2, nbv = 2 * pass + 3;
            if (na <= m) {
                const double* va = V[na];
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int i = i0 + k * stride;
                    ca[k] = i < n ? __ldcg(va + i) : 0.0;
                }
            }
            if (nbv <= m) {
                const double* vb = V[nbv];
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int i = i0 + k * stride;
                    cb[k] = i < n ? __ldcg(vb + i) : 0.0;
                }
            }
        }
        block_sum3<NT>(s1, s2, s3, sh);
        const double b4 = pass == 0 ? block_sum<NT>(s4, sh) : 0.0;
        double* slot = partials + static_cast<std::size_t>(pass) * 4 * nb;
        if (threadIdx.x == 0) {
            slot[blockIdx.x] = s1;
            slot[nb + blockIdx.x] = s2;
            slot[2 * nb + blockIdx.x] = s3;
            slot[3 * nb + blockIdx.x] = b4;
        }
        grid.sync();
        double t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0;
        for (int q = threadIdx.x; q < nb; q += blockDim.x) {
            t1 += slot[q];
            if (two) {
                t2 += slot[nb + q];
                t3 += slot[2 * nb + q];
            }
            if (pass == 0) t4 += slot[3 * nb + q];
        }
        block_sum3<NT>(t1, t2, t3, sh);
        if (pass == 0) t4 = block_sum<NT>(t4, sh);
        if (threadIdx.x == 0) {
            const double h1 = t1;
            const double h2 = two ? t2 - h1 * t3 : 0.0;
            hb[0] = h1;
            hb[1] = h2;
            if (blockIdx.x == 0) {
                if (dots) {
                    hout[2 * pass] = h1;
                    if (two) hout[2 * pass + 1] = h2;
                } else {
                    hout[m + 1] = h1;
                }
                if (pass == 0) *wn0 = t4;
            }
        }
        __syncthreads();
        ha = hb[0];
        hbv = hb[1];
    }
    // ha = ||w||^2 after the last pass: speculative next basis vector
    const double sub = sqrt(ha);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int i = i0 + k * stride;
        if (i < n) {
            w[i] = wr[k];
            if (vnext) {
                const double v = wr[k] / sub;
                vnext[i] = v;
                if (vin) vin[i] = v;
            }
        }
    }
}

/** Single-CTA variant of k_mgs_all for small systems (n below a few 10^4):
 *  the same passes and fixed-order sums with __syncthreads instead of grid
 *  barriers, so a whole Arnoldi orthogonalisation costs a few microseconds. */
template <int NT>
__global__ void __launch_bounds__(NT) k_mgs_block(int n, int m, const double* const* __restrict__ V,
                                                  double* __restrict__ w, double* __restrict__ vnext,
                                                  double* hout, double* wn0, const int* __restrict__ mdev,
                                                  double* __restrict__ vin) {
    if (mdev) {
        m = *mdev;
        vnext = const_cast<double*>(V[m + 1]);
        wn0 = hout + m + 2;
    }
    __shared__ double sh[NT / 32];
    __shared__ double hb;
    double hprev = 0.0;
    for (int pass = 0; pass <= m + 1; ++pass) {
        const double* vp = pass > 0 ? V[pass - 1] : nullptr;
        const double* vn = pass <= m ? V[pass] : nullptr;
        double a1 = 0.0, a2 = 0.0;
        for (int i = threadIdx.x; i < n; i += NT) {
            double wi = w[i];
            if (vp) {
                wi -= hprev * vp[i];
                w[i] = wi;
            }
            a1 = fma(vn ? vn[i] : wi, wi, a1);
            if (pass == 0) a2 = fma(wi, wi, a2);
        }
        const double t1 = block_sum<NT>(a1, sh);
        const double t2 = pass == 0 ? block_sum<NT>(a2, sh) : 0.0;
        if (threadIdx.x == 0) {
            hb = t1;
            hout[pass] = t1;
            if (pass == 0) *wn0 = t2;
        }
        __syncthreads();
        hprev = hb;
        __syncthreads();
    }
    const double sub = sqrt(hprev);
    if (vnext)
        for (int i = threadIdx.x; i < n; i += NT) {
            const double v = w[i] / sub;
            vnext[i] = v;
            if (vin) vin[i] = v;
        }
}

/** k_mgs_block for n <= NT E with the latency trimmed out of its passes
 *  (small systems, BASELINE config 1, are bound by the m + 2 sequential
 *  passes of the orthogonalisation):
 *   - w in registers (E entries per thread, i = tid + e NT: k_mgs_block's
 *     per-thread order), the subtraction w -= h_p V_p folded into the end of
 *     pass p;
 *   - the basis pointers staged in shared memory once, V_{p+2} copied into
 *     a 3-slice shared ring by cp.async while pass p reduces (each thread
 *     copies and reads only its own entries);
 *   - two barriers per pass instead of four (warp partials; block_sum's
 *     final butterfly in warp 0, h broadcast) and no global store inside the
 *     loop -- the h values go out together at the end.
 *  NT = 1024: same partition, same butterflies, so h, ||w||^2 and V_{m+1}
 *  are bitwise those of k_mgs_block (tests/test_gpu_parity.py). */
template <int NT, int E>
__global__ void __launch_bounds__(NT) k_mgs_block_reg(int n, int m, const double* const* __restrict__ V,
                                                      double* __restrict__ w, double* __restrict__ vnext,
                                                      double* hout, double* wn0, const int* __restrict__ mdev,
                                                      double* __restrict__ vin) {
    static_assert(NT % 32 == 0 && NT <= 1024, "warp partials fit one warp");
    constexpr int kMaxV = 64;
    extern __shared__ __align__(16) double vs[];  // [3][E][NT]: V_p, V_{p+1}, V_{p+2} slices
    __shared__ double sh[2][2][NT / 32];
    __shared__ double hs[kMaxV + 2];  // h of every pass; [kMaxV + 1]: ||w||^2
    __shared__ const double* vp_s[kMaxV];
    if (mdev) m = *mdev;
    if (threadIdx.x <= m && threadIdx.x < kMaxV) vp_s[threadIdx.x] = V[threadIdx.x];
    if (mdev) {
        vnext = const_cast<double*>(V[m + 1]);
        wn0 = hout + m + 2;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double wr[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x + e * NT;
        wr[e] = i < n ? w[i] : 0.0;
    }
    __syncthreads();
    // each thread copies (cp.async, 8 bytes) and later reads only its own
    // entries: no barrier orders the slices, and -- unlike register
    // prefetches -- the copies in flight do not hold up the pass barriers
    const unsigned vs_u = static_cast<unsigned>(__cvta_generic_to_shared(vs));
    auto fetch = [&](int q) {
        if (q <= m) {
            const double* src = vp_s[q];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = threadIdx.x + e * NT;
                if (i < n)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                     vs_u + 8u * static_cast<unsigned>(((q % 3) * E + e) * NT + threadIdx.x)),
                                 "l"(src + i)
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(0);
    fetch(1);
    for (int pass = 0; pass <= m + 1; ++pass) {
        const bool has_v = pass <= m;  // pass m + 1: the norm of the orthogonalised w
        fetch(pass + 2);
        asm volatile("cp.async.wait_group 2;" ::: "memory");  // V_pass has landed
        const double* cur = vs + (pass % 3) * E * NT + threadIdx.x;
        double a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (threadIdx.x + e * NT < n) {
                a1 = fma(has_v ? cur[e * NT] : wr[e], wr[e], a1);
                if (pass == 0) a2 = fma(wr[e], wr[e], a2);
            }
        }
        a1 = warp_sum(a1);
        if (pass == 0) a2 = warp_sum(a2);
        if (lane == 0) {
            sh[pass & 1][0][warp] = a1;
            sh[pass & 1][1][warp] = a2;
        }
        __syncthreads();
        if (warp == 0) {  // block_sum's final butterfly, then broadcast
            const double t1 = warp_sum(lane < NT / 32 ? sh[pass & 1][0][lane] : 0.0);
            const double t2 = pass == 0 ? warp_sum(lane < NT / 32 ? sh[0][1][lane] : 0.0) : 0.0;
            if (lane == 0) {
                hs[pass] = t1;  // to hout after the loop: a global store before
                if (pass == 0) hs[kMaxV + 1] = t2;  // the next barrier would hold it up
            }
        }
        __syncthreads();
        const double h = hs[pass];
        if (has_v) {
#pragma unroll
            for (int e = 0; e < E; ++e) wr[e] -= h * cur[e * NT];
        } else {
            const double sub = sqrt(h);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = threadIdx.x + e * NT;
                if (i < n) {
                    w[i] = wr[e];
                    if (vnext) {
                        const double v = wr[e] / sub;
                        vnext[i] = v;
                        if (vin) vin[i] = v;
                    }
                }
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (threadIdx.x <= m + 1) hout[threadIdx.x] = hs[threadIdx.x];
    if (threadIdx.x == 0) *wn0 = hs[kMaxV + 1];
}

__global__ void k_scale(int n, const double* __restrict__ src, double s, double* __restrict__ dst) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i] / s;
}

/** out = sum_k y[k] V_k  (V_k at vbase[k]). */
__global__ void k_combine(int n, int m, const double* const* __restrict__ vptr, const double* __restrict__ y,
                          double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < m; ++k) s = fma(y[k], __ldg(vptr[k] + i), s);
        out[i] = s;
    }
}

__global__ void k_axpy1(int n, const double* __restrict__ x, double* __restrict__ y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] += x[i];
}

/** dst = src / s and dst2 = src / s (the first basis vector and the fixed
 *  preconditioner input of the device-driven Arnoldi loop). */
__global__ void k_scale2(int n, const double* __restrict__ src, double s, double* __restrict__ dst,
                         double* __restrict__ dst2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = src[i] / s;
        dst[i] = v;
        dst2[i] = v;
    }
}

/** Device state of one GMRES cycle run as a CUDA graph (layout of the
 *  solver-state buffer, in doubles: [0, 8) this struct, then H (cap x cap,
 *  column k = rotated Hessenberg column of step k), cs, sn (cap), g
 *  (cap + 1), est (cap: |g_{k+1}| after step k), stamps (4 cap int64). */
struct GState {
    int m, total, cycle, max_iter, status, pad;
    double target, pad2;
};
constexpr int kGHead = 8;
static_assert(sizeof(GState) <= kGHead * sizeof(double), "GState layout");
enum { kGRun = 0, kGBasisNonFinite = 1, kGEstNonFinite = 2, kGConverged = 3 };

__global__ void k_gstate_init(double* gb, int cap, int total, int cycle, int max_iter, double target, double beta) {
    GState* S = reinterpret_cast<GState*>(gb);
    S->m = 0;
    S->total = total;
    S->cycle = cycle;
    S->max_iter = max_iter;
    S->status = kGRun;
    S->target = target;
    double* g = gb + kGHead + static_cast<std::size_t>(cap) * cap + 2 * cap;
    g[0] = beta;
}

/** Arnoldi step m's Givens update on the device (the host loop of
 *  solve.hpp:165-200 / gmres() below, same operations in the same order,
 *  round-to-nearest intrinsics: no contraction, so the rotated estimates are
 *  bitwise those of the host loop; hypot is glibc's algorithm, as the host's
 *  std::hypot).  Sets the while-condition of the cycle graph: continue while
 *  not converged, no breakdown, m < cycle and total < max_iter. */
__global__ void k_givens(double* gb, int cap, const double* __restrict__ hd, cudaGraphConditionalHandle cond) {
    if (threadIdx.x != 0) return;
    GState* S = reinterpret_cast<GState*>(gb);
    double* H = gb + kGHead;
    double* cs = H + static_cast<std::size_t>(cap) * cap;
    double* sn = cs + cap;
    double* g = sn + cap;
    double* est = g + cap + 1;
    const int m = S->m;
    double* h = H + static_cast<std::size_t>(m) * cap;
    for (int i = 0; i <= m; ++i) h[i] = hd[i];
    h[m + 1] = sqrt(hd[m + 1]);
    const double wnorm0 = sqrt(hd[m + 2]);
    const double subdiag = h[m + 1];
    int status = kGRun;
    if (!isfinite(subdiag)) {
        status = kGBasisNonFinite;
    } else {
        for (int i = 0; i < m; ++i) {
            const double t = __dadd_rn(__dmul_rn(cs[i], h[i]), __dmul_rn(sn[i], h[i + 1]));
            h[i + 1] = __dadd_rn(__dmul_rn(-sn[i], h[i]), __dmul_rn(cs[i], h[i + 1]));
            h[i] = t;
        }
        const double denom = hypot_glibc(h[m], h[m + 1]);
        cs[m] = denom == 0 ? 1.0 : __ddiv_rn(h[m], denom);
        sn[m] = denom == 0 ? 0.0 : __ddiv_rn(h[m + 1], denom);
        h[m] = denom;
        g[m + 1] = __dmul_rn(-sn[m], g[m]);
        g[m] = __dmul_rn(cs[m], g[m]);
        S->m = m + 1;
        S->total += 1;
        const double e = fabs(g[m + 1]);
        est[m] = e;
        if (!isfinite(e))
            status = kGEstNonFinite;
        else if (e <= S->target || subdiag <= __dmul_rn(1e-14, wnorm0))
            status = kGConverged;
    }
    S->status = status;
    const bool more = status == kGRun && S->m < S->cycle && S->total < S->max_iter;
    cudaGraphSetConditional(cond, more ? 1u : 0u);
}

/** Stationary iteration state (stationary_graph): [0, 8) this struct, then
 *  the residual history (max_iter + 1 entries). */
struct SState {
    int it, max_iter, status, pad;
    double r0, target;
};
enum { kSRun = 0, kSNonFinite = 1, kSDiverged = 2, kSConverged = 3 };

/** One stationary step's checks on the device (solve.hpp:112-121, the host
 *  loop's order): rn = sqrt(||r||^2), finite, divergence (> 1e8 r0),
 *  convergence (<= rel_tol r0); sets the loop condition. */
__global__ void k_stat_check(double* sb, const double* __restrict__ rn2, cudaGraphConditionalHandle cond) {
    if (threadIdx.x != 0) return;
    SState* S = reinterpret_cast<SState*>(sb);
    const double rn = sqrt(*rn2);
    const int it = S->it + 1;
    S->it = it;
    sb[8 + it] = rn;
    int status = kSRun;
    if (!isfinite(rn))
        status = kSNonFinite;
    else if (rn > __dmul_rn(1e8, S->r0))
        status = kSDiverged;
    else if (rn <= S->target)
        status = kSConverged;
    S->status = status;
    cudaGraphSetConditional(cond, (status == kSRun && it < S->max_iter) ? 1u : 0u);
}

__global__ void k_sstate_init(double* sb, int max_iter, double r0, double target) {
    SState* S = reinterpret_cast<SState*>(sb);
    S->it = 0;
    S->max_iter = max_iter;
    S->status = kSRun;
    S->r0 = r0;
    S->target = target;
}

/** Device timestamp (profiling of the graph loop): stamps[4 m + slot]. */
__global__ void k_stamp(const double* gb, long long* stamps, int slot) {
    if (threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[4 * reinterpret_cast<const GState*>(gb)->m + slot] = static_cast<long long>(t);
}

void check_finite(double v, const char* what) {
    if (!std::isfinite(v)) throw DivergenceError(std::string(what) + " is not finite");
}

struct Pinned {
    double* p = nullptr;
    explicit Pinned(std::size_t n) { CPDDG_CUDA(cudaMallocHost(&p, n * sizeof(double))); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Timer {
    cudaEvent_t a, b;
    cudaStream_t s;
    explicit Timer(cudaStream_t st) : s(st) {
        CPDDG_CUDA(cudaEventCreate(&a));
        CPDDG_CUDA(cudaEventCreate(&b));
        CPDDG_CUDA(cudaEventRecord(a, s));
    }
    double stop() {
        CPDDG_CUDA(cudaEventRecord(b, s));
        CPDDG_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        CPDDG_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms * 1e-3;
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

/** Optional per-launch CUDA-event timing of the preconditioner and operator
 *  applies (events recorded around each launch on the solve stream; the
 *  elapsed times are collected at the per-iteration host synchronisation). */
struct KernelTimer {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<cudaEvent_t>& pool;  // owned by the operator's KrylovCache: reused across solves
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pc_pending, op_pending;
    double pc_s = 0, op_s = 0;
    std::int64_t pc_n = 0, op_n = 0;
    std::size_t used = 0;
    cudaEvent_t ev() {
        if (used == pool.size()) {
            cudaEvent_t e;
            CPDDG_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    template <class F>
    void time(bool is_pc, F&& f) {
        if (!on) {
            f();
            return;
        }
        cudaEvent_t a = ev(), b = ev();
        CPDDG_CUDA(cudaEventRecord(a, st));
        f();
        CPDDG_CUDA(cudaEventRecord(b, st));
        (is_pc ? pc_pending : op_pending).emplace_back(a, b);
    }
    /** Call after a stream synchronisation. */
    void collect() {
        if (!on) return;
        for (auto& [a, b] : pc_pending) {
            float ms = 0;
            CPDDG_CUDA(cudaEventElapsedTime(&ms, a, b));
            pc_s += ms * 1e-3;
            ++pc_n;
        }
        for (auto& [a, b] : op_pending) {
            float ms = 0;
            CPDDG_CUDA(cudaEventElapsedTime(&ms, a, b));
            op_s += ms * 1e-3;
            ++op_n;
        }
        pc_pending.clear();
        op_pending.clear();
        used = 0;
    }
    explicit KernelTimer(std::vector<cudaEvent_t>& p) : pool(p) {}
};

constexpr int kSmallMgs = 16384;  // single-CTA orthogonalisation below this size

struct Workspace {
    int n;
    cudaStream_t st;
    int grid;
    KrylovCache& kc;
    ReduceWork& red;
    std::int64_t launches = 0;
    Workspace(int n_, cudaStream_t s, KrylovCache& c) : n(n_), st(s), kc(c), red(c.red) {
        grid = reduction_blocks();
        red.ensure(2);
        auto need = [&](DevBuf<double>& b, std::size_t cnt) {
            if (b.size() < cnt) b.alloc(cnt);
        };
        need(kc.w, static_cast<std::size_t>(n));
        need(kc.r, static_cast<std::size_t>(n));
        need(kc.tmp, static_cast<std::size_t>(n));
    }
    /** Scalar slots and pinned host scratch for `cap` Hessenberg entries. */
    void reserve(int cap) {
        if (kc.scal.size() < static_cast<std::size_t>(cap) + 4) kc.scal.alloc(static_cast<std::size_t>(cap) + 4);
        if (kc.yd.size() < static_cast<std::size_t>(cap)) kc.yd.alloc(static_cast<std::size_t>(cap));
        if (kc.vptr.size() < static_cast<std::size_t>(cap)) {
            kc.vptr.alloc(static_cast<std::size_t>(cap) + 64);
            kc.vptr_valid = 0;
        }
        // three regions: two alternating Hessenberg columns (pipelined
        // Arnoldi steps) and the update coefficients y
        if (kc.host_cap < 3 * (cap + 4)) {
            if (kc.host) cudaFreeHost(kc.host);
            CPDDG_CUDA(cudaMallocHost(&kc.host, sizeof(double) * 3 * (cap + 4)));
            kc.host_cap = 3 * (cap + 4);
        }
    }
    double* basis(int k) {
        while (static_cast<int>(kc.V.size()) <= k) kc.V.emplace_back(static_cast<std::size_t>(n));
        return kc.V[static_cast<std::size_t>(k)].get();
    }
    /** out = (vnext ? vnext . w : w . w) after the optional update. */
    void mgs(const double* hprev, const double* vprev, double* w, const double* vnext, double* out,
             double* out2) {
        k_mgs<<<grid, kRedThreads, 0, st>>>(n, hprev, vprev, w, vnext, red.partials.get(), red.counter.get(), out,
                                            out2);
        CPDDG_CUDA(cudaGetLastError());
        ++launches;
    }
    // persistent (KrylovCache): the cycle graph keeps pointers into them
    DevBuf<double>& mgs_partials = kc.mgs_partials;
    int& coop_grid = kc.coop_grid;
    /** mgs_all with the step read from *mdev on the device (V_{m+1} and the
     *  ||w0||^2 slot follow from it; the new basis vector is also copied to
     *  vin): the launch parameters do not depend on the step, so it can sit
     *  in a captured loop body.  The basis table must cover V_0..V_{cap}. */
    void mgs_all_dev(int mmax, double* w, double* hout, const int* mdev, double* vin) {
        mgs_all(mmax, w, nullptr, hout, nullptr, mdev, vin);
    }
    void mgs_all(int m, double* w, double* vnext, double* hout, double* wn0, const int* mdev = nullptr,
                 double* vin = nullptr) {
        prepare_mgs(m);
        int nn = n, mm = m;
        const double* const* vpd = kc.vptr.get();
        const char* me = std::getenv("CPDDG_MGS");  // development: "block" = k_mgs_block for every small n
        const bool block_only = me && std::string(me) == "block";
        if (n <= 4 * 1024 && !block_only && m < 60) {  // k_mgs_block_reg stages <= 64 basis pointers
            static const bool attr = [] {
                for (const void* k : {reinterpret_cast<const void*>(k_mgs_block_reg<1024, 1>),
                                      reinterpret_cast<const void*>(k_mgs_block_reg<1024, 2>),
                                      reinterpret_cast<const void*>(k_mgs_block_reg<1024, 4>)})
                    CPDDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4 * 1024 * 8));
                return true;
            }();
            (void)attr;
            if (n <= 1024)
                k_mgs_block_reg<1024, 1><<<1, 1024, 3 * 1 * 1024 * 8, st>>>(nn, mm, vpd, w, vnext, hout, wn0, mdev, vin);
            else if (n <= 2 * 1024)
                k_mgs_block_reg<1024, 2><<<1, 1024, 3 * 2 * 1024 * 8, st>>>(nn, mm, vpd, w, vnext, hout, wn0, mdev, vin);
            else
                k_mgs_block_reg<1024, 4><<<1, 1024, 3 * 4 * 1024 * 8, st>>>(nn, mm, vpd, w, vnext, hout, wn0, mdev, vin);
            CPDDG_CUDA(cudaGetLastError());
            ++launches;
            return;
        }
        if (n <= kSmallMgs) {
            k_mgs_block<1024><<<1, 1024, 0, st>>>(nn, mm, vpd, w, vnext, hout, wn0, mdev, vin);
            CPDDG_CUDA(cudaGetLastError());
            ++launches;
            return;
        }
        double* part = mgs_partials.get();
        void* args[] = {&nn, &mm, &vpd, &w, &vnext, &part, &hout, &wn0, &mdev, &vin};
        // register-resident w: up to 8 elements per thread of the cooperative grid
        static const bool streamed = [] {
            const char* e = std::getenv("CPDDG_MGS");  // development: "stream" = k_mgs_all
            return e && std::string(e) == "stream";
        }();
        const long long threads = static_cast<long long>(coop_grid) * kRedThreads;
        const int ept = static_cast<int>((n + threads - 1) / threads);
        const char* se = std::getenv("CPDDG_MGS");  // "single" = one projection per grid barrier (k_mgs_reg)
        const bool single = se && std::string(se) == "single";
        const void* kern = reinterpret_cast<const void*>(k_mgs_all);
        if (!streamed && !single && ept <= 8)
            kern = ept <= 1   ? reinterpret_cast<const void*>(k_mgs_pair<1>)
                   : ept <= 2 ? reinterpret_cast<const void*>(k_mgs_pair<2>)
                   : ept <= 4 ? reinterpret_cast<const void*>(k_mgs_pair<4>)
                              : reinterpret_cast<const void*>(k_mgs_pair<8>);
        else if (!streamed && ept <= 16)
            kern = ept <= 1   ? reinterpret_cast<const void*>(k_mgs_reg<1>)
                   : ept <= 2 ? reinterpret_cast<const void*>(k_mgs_reg<2>)
                   : ept <= 4 ? reinterpret_cast<const void*>(k_mgs_reg<4>)
                   : ept <= 8 ? reinterpret_cast<const void*>(k_mgs_reg<8>)
                              : reinterpret_cast<const void*>(k_mgs_reg<16>);
        // fewer, larger blocks make the grid barrier cheaper: one 512-thread block per SM when its
        // slice still fits 8 elements per thread (CPDDG_MGS_WIDE=0: kRedThreads-thread blocks)
        const char* we = std::getenv("CPDDG_MGS_WIDE");
        const bool wide_ok = !(we && std::string(we) == "0") && !streamed && !single && coop_grid >= sm_count() &&
                             static_cast<long long>(sm_count()) * 512 * 8 >= n &&
                             static_cast<long long>(sm_count()) * 512 * 4 < n;
        if (wide_ok) {
            const void* wk = reinterpret_cast<const void*>(k_mgs_pair<8, 512>);
            int per_sm = 0;
            CPDDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wk, 512, 0));
            if (per_sm >= 1) {
                CPDDG_CUDA(cudaLaunchCooperativeKernel(wk, dim3(sm_count()), dim3(512), args, 0, st));
                ++launches;
                return;
            }
        }
        if (kern != reinterpret_cast<const void*>(k_mgs_all)) {
            int per_sm = 0;  // the whole grid must be resident
            CPDDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRedThreads, 0));
            if (per_sm * sm_count() < coop_grid) kern = reinterpret_cast<const void*>(k_mgs_all);
        }
        CPDDG_CUDA(cudaLaunchCooperativeKernel(kern, dim3(coop_grid), dim3(kRedThreads), args, 0, st));
        ++launches;
    }
    /** Cooperative grid size, per-pass partials (m + 2 passes) and the basis
     *  pointer table for steps up to m. */
    void prepare_mgs(int m) {
        if (coop_grid == 0) {
            int per_sm = 0;
            CPDDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs_all, kRedThreads, 0));
            // cooperative blocks per SM: the fewest (>= 2) that keep the register
            // kernel's slice at <= 8 elements per thread -- measured: 2 beats 4
            // at the headline (cheaper grid barriers); larger systems need more
            // blocks or they fall back to the streaming k_mgs_all
            const long long per_block_sm = static_cast<long long>(sm_count()) * kRedThreads * 8;
            int bps = static_cast<int>(std::max<long long>(2, (n + per_block_sm - 1) / per_block_sm));
            if (const char* e = std::getenv("CPDDG_MGS_BPS")) bps = std::max(1, std::atoi(e));  // development knob
            coop_grid = std::max(1, std::min(per_sm, bps)) * sm_count();
        }
        // k_mgs_reg / k_mgs_all: 2 sums x (m + 2) passes; k_mgs_pair: 4 sums x ((m + 2) / 2 + 1) passes
        const std::size_t need = std::max(static_cast<std::size_t>(2 * coop_grid) * (m + 2),
                                          static_cast<std::size_t>(4 * coop_grid) * ((m + 2) / 2 + 2));
        if (mgs_partials.size() < need) mgs_partials.alloc(std::max(need, static_cast<std::size_t>(2 * coop_grid) * 64));
        // basis pointer table (V_0..V_m) on the device: basis buffers never
        // move once allocated, so the table is uploaded only when it grows
        if (kc.vptr_valid < m + 1) {
            std::vector<const double*> vp(kc.V.size());
            for (std::size_t k = 0; k < kc.V.size(); ++k) vp[k] = kc.V[k].get();
            if (kc.vptr.size() < vp.size()) kc.vptr.alloc(vp.size() + 64);
            CPDDG_CUDA(cudaMemcpy(kc.vptr.get(), vp.data(), sizeof(double*) * vp.size(), cudaMemcpyHostToDevice));
            kc.vptr_valid = static_cast<int>(vp.size());
        }
    }
    /** Upload the full basis pointer table (V_0 .. V_{mmax} and beyond). */
    void refresh_vptr(int mmax) {
        for (int k = 0; k <= mmax; ++k) basis(k);
        std::vector<const double*> vp(kc.V.size());
        for (std::size_t k = 0; k < kc.V.size(); ++k) vp[k] = kc.V[k].get();
        if (kc.vptr.size() < vp.size()) kc.vptr.alloc(vp.size() + 64);
        CPDDG_CUDA(cudaMemcpyAsync(kc.vptr.get(), vp.data(), sizeof(double*) * vp.size(), cudaMemcpyHostToDevice, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
        kc.vptr_valid = static_cast<int>(vp.size());
    }
    void scale(const double* src, double s, double* dst) {
        k_scale<<<grid, kRedThreads, 0, st>>>(n, src, s, dst);
        CPDDG_CUDA(cudaGetLastError());
        ++launches;
    }
};

void record(cpddg_log* log, const std::vector<double>& res, int iters, bool conv, double final_true, double secs,
            std::int64_t launches, const KernelTimer* kt = nullptr) {
    if (!log) return;
    if (kt) {
        log->pc_seconds = kt->pc_s;
        log->pc_launches = kt->pc_n;
        log->op_seconds = kt->op_s;
        log->op_launches = kt->op_n;
    }
    log->n_residuals = static_cast<int>(res.size());
    if (log->residuals)
        for (int k = 0; k < std::min(log->capacity, log->n_residuals); ++k) log->residuals[k] = res[static_cast<std::size_t>(k)];
    log->iterations = iters;
    log->converged = conv ? 1 : 0;
    log->final_true_residual = final_true;
    log->seconds = secs;
    log->kernel_launches = launches;
}

}  // namespace

/** Build (or reuse) the cycle graph: a while-conditional node whose body is
 *  one Arnoldi step with device-resident control -- z = M^-1 vin, w = A z,
 *  the cooperative MGS (step m read from the state; V_{m+1} also into vin)
 *  and k_givens, which sets the loop condition.  A GMRES(cycle) cycle is one
 *  graph launch: no host round trip per step. */
static void ensure_cycle_graph(cpddg_op* op, cpddg_pc* pc, Workspace& ws, int cycle, int cap, bool prof) {
    KrylovCache& kc = op->kc;
    ws.refresh_vptr(cycle);  // fixed addresses for V_0..V_cycle, table uploaded before any capture
    if (kc.vin.size() < static_cast<std::size_t>(ws.n)) kc.vin.alloc(static_cast<std::size_t>(ws.n));
    const std::size_t gsz0 = kGHead + static_cast<std::size_t>(cap) * cap + 2 * cap + (cap + 1) + cap + 4 * cap;
    if (kc.gstate.size() < gsz0) kc.gstate.alloc(gsz0);
    ws.prepare_mgs(cycle);  // cooperative grid and partials allocated before any capture
    // every device address the captured body uses: a reallocation forces a rebuild
    const std::vector<const void*> sig{pc, kc.scal.get(), kc.vptr.get(), kc.gstate.get(), kc.w.get(), kc.tmp.get(),
                                       kc.vin.get(), kc.V[0].get(), kc.mgs_partials.get()};
    if (kc.gexec && kc.gcycle == cycle && kc.gprof == (prof ? 1 : 0) && kc.gn == ws.n && kc.gsig == sig) return;
    if (kc.gexec) {
        cudaGraphExecDestroy(kc.gexec);
        kc.gexec = nullptr;
    }
    if (kc.graph) {
        cudaGraphDestroy(kc.graph);
        kc.graph = nullptr;
    }
    if (!kc.gstream) CPDDG_CUDA(cudaStreamCreateWithFlags(&kc.gstream, cudaStreamNonBlocking));
    const int n = ws.n;
    const std::size_t gsz = gsz0;
    CPDDG_CUDA(cudaGraphCreate(&kc.graph, 0));
    cudaGraphConditionalHandle cond;
    CPDDG_CUDA(cudaGraphConditionalHandleCreate(&cond, kc.graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CPDDG_CUDA(cudaGraphAddNode(&node, kc.graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStream_t cs = kc.gstream;
    double* gb = kc.gstate.get();
    const int* mdev = reinterpret_cast<const int*>(gb);  // GState::m
    long long* stamps = reinterpret_cast<long long*>(gb + kGHead + static_cast<std::size_t>(cap) * cap + 2 * cap +
                                                     (cap + 1) + cap);
    double* hd = ws.kc.scal.get();
    CPDDG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const cudaStream_t saved = ws.st;
    ws.st = cs;
    try {
        if (prof) k_stamp<<<1, 32, 0, cs>>>(gb, stamps, 0);
        const double* z = kc.vin.get();
        if (pc) {
            pc_apply(pc, kc.vin.get(), kc.tmp.get(), false, cs);
            z = kc.tmp.get();
        }
        if (prof) k_stamp<<<1, 32, 0, cs>>>(gb, stamps, 1);
        // programmatic edge extension -> Helmholtz kernel also inside the captured body
        // (CPDDG_GRAPH_PDL=0: plain edge)
        const char* gp = std::getenv("CPDDG_GRAPH_PDL");
        op_apply(op, z, kc.w.get(), cs, !(gp && std::string(gp) == "0"));
        if (prof) k_stamp<<<1, 32, 0, cs>>>(gb, stamps, 2);
        ws.mgs_all_dev(cycle, kc.w.get(), hd, mdev, kc.vin.get());
        k_givens<<<1, 32, 0, cs>>>(gb, cap, hd, cond);
        CPDDG_CUDA(cudaGetLastError());
    } catch (...) {
        ws.st = saved;
        cudaGraph_t dummy;
        cudaStreamEndCapture(cs, &dummy);
        throw;
    }
    ws.st = saved;
    CPDDG_CUDA(cudaStreamEndCapture(cs, &body));
    CPDDG_CUDA(cudaGraphInstantiate(&kc.gexec, kc.graph, 0));
    // the MGS partials may have been (re)allocated by the captured launch
    kc.gsig = {pc, kc.scal.get(), kc.vptr.get(), kc.gstate.get(), kc.w.get(), kc.tmp.get(),
               kc.vin.get(), kc.V[0].get(), kc.mgs_partials.get()};
    kc.gpc = pc;
    kc.gcycle = cycle;
    kc.gprof = prof ? 1 : 0;
    kc.gn = n;
    if (kc.ghost_n < gsz) {
        if (kc.ghost) cudaFreeHost(kc.ghost);
        CPDDG_CUDA(cudaMallocHost(&kc.ghost, sizeof(double) * gsz));
        kc.ghost_n = gsz;
    }
}

/** solve.hpp:128-214 with each restart cycle run as one graph launch
 *  (ensure_cycle_graph).  Same arithmetic as the host loop below, in the
 *  same order: residual histories and solutions are bitwise identical
 *  (tests/test_gpu_parity.py::test_graph_gmres_matches_host_loop). */
static void gmres_graph(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params& prm,
                        cpddg_log* log, cudaStream_t st) {
    const int n = op->na;
    const int max_iter = prm.max_iter;
    const int cycle = std::max(1, std::min(prm.restart > 0 ? prm.restart : max_iter, max_iter));
    Workspace ws(n, st, op->kc);
    const int cap = cycle + 2;
    ws.reserve(cap);
    const bool prof = prm.profile_kernels != 0;
    ensure_cycle_graph(op, pc, ws, cycle, cap, prof);
    KrylovCache& kc = op->kc;
    double* gb = kc.gstate.get();
    double* nd = ws.kc.scal.get() + cap;  // [1] ||r||^2
    DevBuf<double>& r = ws.kc.r;
    DevBuf<double>& tmp = ws.kc.tmp;
    KernelTimer kt(op->kc.events);
    kt.on = prof;
    kt.st = st;
    Timer timer(st);
    CPDDG_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * n, st));
    CPDDG_CUDA(cudaMemcpyAsync(r.get(), b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double* hp = ws.kc.host;
    auto fetch = [&](const double* dev, int cnt) {
        CPDDG_CUDA(cudaMemcpyAsync(hp, dev, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
    };
    ws.mgs(nullptr, nullptr, r.get(), nullptr, nd + 1, nullptr);
    fetch(nd + 1, 1);
    double rnorm = std::sqrt(hp[0]);
    std::vector<double> residuals{rnorm};
    const double beta0 = rnorm;
    int total = 0;
    bool converged = false;
    if (beta0 == 0.0) {
        record(log, residuals, 0, true, 0.0, timer.stop(), ws.launches);
        return;
    }
    const double target = prm.rel_tol * beta0;
    const std::size_t off_cs = kGHead + static_cast<std::size_t>(cap) * cap;
    const std::size_t off_g = off_cs + 2 * cap, off_est = off_g + cap + 1, off_st = off_est + cap;
    const std::size_t gsz = off_st + 4 * cap;
    double pc_graph_s = 0, op_graph_s = 0;
    std::int64_t pc_graph_n = 0, op_graph_n = 0;
    std::vector<const double*> vptr_h(static_cast<std::size_t>(cap));
    while (total < max_iter && !converged) {
        const double beta = rnorm;
        check_finite(beta, "gmres residual");
        if (beta <= target) {
            converged = true;
            break;
        }
        k_scale2<<<ws.grid, kRedThreads, 0, st>>>(n, r.get(), beta, ws.basis(0), kc.vin.get());
        k_gstate_init<<<1, 1, 0, st>>>(gb, cap, total, cycle, max_iter, target, beta);
        CPDDG_CUDA(cudaGetLastError());
        CPDDG_CUDA(cudaGraphLaunch(kc.gexec, st));
        ws.launches += 2;
        CPDDG_CUDA(cudaMemcpyAsync(kc.ghost, gb, sizeof(double) * gsz, cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
        const GState* S = reinterpret_cast<const GState*>(kc.ghost);
        const int m = S->m;
        ws.launches += static_cast<std::int64_t>(m) * (4 + (prof ? 3 : 0));
        total = S->total;
        for (int k = 0; k < m; ++k) residuals.push_back(kc.ghost[off_est + k]);
        if (S->status == kGBasisNonFinite) throw DivergenceError("gmres basis norm is not finite");
        if (S->status == kGEstNonFinite) throw DivergenceError("gmres residual estimate is not finite");
        if (prof) {
            const long long* stp = reinterpret_cast<const long long*>(kc.ghost + off_st);
            for (int k = 0; k < m; ++k) {
                pc_graph_s += 1e-9 * static_cast<double>(stp[4 * k + 1] - stp[4 * k]);
                op_graph_s += 1e-9 * static_cast<double>(stp[4 * k + 2] - stp[4 * k + 1]);
            }
            pc_graph_n += pc ? m : 0;
            op_graph_n += m;
        }
        converged = S->status == kGConverged;
        if (m > 0) {
            const double* H = kc.ghost + kGHead;
            const double* g = kc.ghost + off_g;
            std::vector<double> y(static_cast<std::size_t>(m), 0.0);
            for (int i = m - 1; i >= 0; --i) {
                double sacc = g[i];
                for (int k = i + 1; k < m; ++k) sacc -= H[static_cast<std::size_t>(k) * cap + i] * y[static_cast<std::size_t>(k)];
                if (H[static_cast<std::size_t>(i) * cap + i] == 0.0)
                    throw DivergenceError("gmres encountered a singular projection");
                y[static_cast<std::size_t>(i)] = sacc / H[static_cast<std::size_t>(i) * cap + i];
            }
            double* yh = ws.kc.host + 2 * (cap + 4);
            for (int k = 0; k < m; ++k) {
                vptr_h[static_cast<std::size_t>(k)] = ws.basis(k);
                yh[k] = y[static_cast<std::size_t>(k)];
            }
            CPDDG_CUDA(cudaMemcpyAsync(ws.kc.vptr.get(), vptr_h.data(), sizeof(double*) * m, cudaMemcpyHostToDevice, st));
            CPDDG_CUDA(cudaMemcpyAsync(ws.kc.yd.get(), yh, sizeof(double) * m, cudaMemcpyHostToDevice, st));
            k_combine<<<ws.grid, kRedThreads, 0, st>>>(n, m, ws.kc.vptr.get(), ws.kc.yd.get(), tmp.get());
            CPDDG_CUDA(cudaGetLastError());
            ++ws.launches;
            if (pc) {
                kt.time(true, [&] { pc_apply(pc, tmp.get(), u, true, st); });
            } else {
                k_axpy1<<<ws.grid, kRedThreads, 0, st>>>(n, tmp.get(), u);
                CPDDG_CUDA(cudaGetLastError());
            }
            ++ws.launches;
            CPDDG_CUDA(cudaStreamSynchronize(st));
            // (the update rewrote entries 0..m-1 of the pointer table with the
            // same basis pointers the graph's MGS reads)
        }
        kt.time(false, [&] { op_residual(op, b, u, r.get(), nd + 1, st); });
        ws.launches += 2;
        fetch(nd + 1, 1);
        kt.collect();
        rnorm = std::sqrt(hp[0]);
    }
    const double secs = timer.stop();
    kt.collect();
    kt.pc_s += pc_graph_s;
    kt.pc_n += pc_graph_n;
    kt.op_s += op_graph_s;
    kt.op_n += op_graph_n;
    record(log, residuals, total, converged, rnorm, secs, ws.launches, &kt);
}

// solve.hpp:128-214
static void gmres(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params& prm,
                  cpddg_log* log, cudaStream_t st) {
    const int n = op->na;
    if (pc && pc->n_global != n) throw InternalError("preconditioner size does not match the operator");
    {
        // default: device-driven cycles (one CUDA graph launch per restart
        // cycle); CPDDG_GMRES_GRAPH=0 or CPDDG_GMRES_SYNC=1 select the host
        // loop.  Kernel profiling (per-launch CUDA events) runs the host loop
        // unless CPDDG_GMRES_GRAPH=1 (then device timestamps in the graph)
        const char* ge = std::getenv("CPDDG_GMRES_GRAPH");
        const char* se = std::getenv("CPDDG_GMRES_SYNC");
        const bool forced = ge && std::string(ge) == "1";
        const bool host_loop = (ge && std::string(ge) == "0") || (se && std::string(se) == "1") ||
                               (prm.profile_kernels && !forced);
        if (!host_loop && prm.max_iter > 0) {
            gmres_graph(op, pc, b, u, prm, log, st);
            return;
        }
    }
    const int max_iter = prm.max_iter;
    const int cycle = prm.restart > 0 ? prm.restart : max_iter;
    Workspace ws(n, st, op->kc);
    const int cap = std::max(std::min(cycle, max_iter), 1) + 2;
    ws.reserve(cap);
    double* hd = ws.kc.scal.get();   // h[0..m+1]
    double* nd = hd + cap;           // [0] ||w0||^2, [1] ||r||^2
    struct {
        double* p;
    } hh{ws.kc.host};
    double* hslot[2] = {hh.p, hh.p + (cap + 4)};
    struct Events {
        cudaEvent_t e[2];
        Events() {
            for (auto& x : e) CPDDG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        }
        ~Events() {
            for (auto& x : e) cudaEventDestroy(x);
        }
    } hevs;
    cudaEvent_t* hev = hevs.e;
    DevBuf<double>& w = ws.kc.w;
    DevBuf<double>& r = ws.kc.r;
    DevBuf<double>& tmp = ws.kc.tmp;
    auto basis = [&](int k) { return ws.basis(k); };
    DevBuf<const double*>& vptr = ws.kc.vptr;
    DevBuf<double>& yd = ws.kc.yd;
    std::vector<const double*> vptr_h(static_cast<std::size_t>(cap));

    KernelTimer kt(op->kc.events);
    kt.on = prm.profile_kernels != 0;
    kt.st = st;
    Timer timer(st);
    CPDDG_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * n, st));
    CPDDG_CUDA(cudaMemcpyAsync(r.get(), b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    auto fetch = [&](const double* dev, int cnt) {
        CPDDG_CUDA(cudaMemcpyAsync(hh.p, dev, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
    };
    ws.mgs(nullptr, nullptr, r.get(), nullptr, nd + 1, nullptr);
    fetch(nd + 1, 1);
    double rnorm = std::sqrt(hh.p[0]);
    std::vector<double> residuals{rnorm};
    const double beta0 = rnorm;
    int total = 0;
    bool converged = false;
    if (beta0 == 0.0) {
        record(log, residuals, 0, true, 0.0, timer.stop(), ws.launches);
        return;
    }
    const double target = prm.rel_tol * beta0;
    while (total < max_iter && !converged) {
        const double beta = rnorm;
        check_finite(beta, "gmres residual");
        if (beta <= target) {
            converged = true;
            break;
        }
        ws.scale(r.get(), beta, basis(0));
        std::vector<std::vector<double>> H;
        std::vector<double> cs, sn, g{beta};
        int m = 0;
        bool breakdown = false;
        // Arnoldi step mm on the device: z = M^-1 V_mm, w = A z, MGS (all
        // mm+2 passes and the next basis vector in one cooperative launch),
        // the Hessenberg column to pinned host slot `slot`, event.
        auto enqueue = [&](int mm, int slot) {
            const double* z = basis(mm);
            if (pc) {
                kt.time(true, [&] { pc_apply(pc, basis(mm), tmp.get(), false, st); });
                ++ws.launches;
                z = tmp.get();
            }
            kt.time(false, [&] { op_apply(op, z, w.get(), st); });
            ws.launches += 2;
            double* vnext = (mm + 1 <= cycle) ? basis(mm + 1) : nullptr;
            ws.mgs_all(mm, w.get(), vnext, hd, hd + mm + 2);
            CPDDG_CUDA(cudaMemcpyAsync(hslot[slot], hd, sizeof(double) * (mm + 3), cudaMemcpyDeviceToHost, st));
            CPDDG_CUDA(cudaEventRecord(hev[slot], st));
        };
        int slot = 0;
        bool queued = false;  // step m already enqueued (speculatively, by step m-1)
        const char* sync_env = std::getenv("CPDDG_GMRES_SYNC");  // tests: the synchronous loop
        const bool pipelined = !(sync_env && std::string(sync_env) == "1");
        while (m < cycle && total < max_iter) {
            if (!queued) enqueue(m, slot);
            // pipelining: enqueue step m+1 before the host reads step m's
            // column, so the device never waits for the host's Givens update.
            // Only while the residual trend says step m will not converge (a
            // wasted step costs a preconditioner apply); step m+1 depends on
            // V_{m+1}, which step m writes on the device.
            bool spec = pipelined && m + 1 < cycle && total + 1 < max_iter;
            if (spec) {
                const std::size_t nr = residuals.size();
                const double last = residuals[nr - 1];
                const double rate = nr >= 2 && m >= 1 ? std::min(1.0, last / residuals[nr - 2]) : 1.0;
                spec = last * rate > 4.0 * target;
            }
            if (spec) enqueue(m + 1, slot ^ 1);
            CPDDG_CUDA(cudaEventSynchronize(hev[slot]));
            // kernel timings (profile_kernels) are collected after the next full
            // stream synchronisation: a speculative step may still be in flight
            const double* hp = hslot[slot];
            std::vector<double> h(hp, hp + m + 2);
            h[static_cast<std::size_t>(m) + 1] = std::sqrt(h[static_cast<std::size_t>(m) + 1]);
            const double wnorm0 = std::sqrt(hp[m + 2]);
            const double subdiag = h[static_cast<std::size_t>(m) + 1];
            check_finite(subdiag, "gmres basis norm");
            for (int i = 0; i < m; ++i) {
                const double t = cs[static_cast<std::size_t>(i)] * h[static_cast<std::size_t>(i)] + sn[static_cast<std::size_t>(i)] * h[static_cast<std::size_t>(i) + 1];
                h[static_cast<std::size_t>(i) + 1] = -sn[static_cast<std::size_t>(i)] * h[static_cast<std::size_t>(i)] + cs[static_cast<std::size_t>(i)] * h[static_cast<std::size_t>(i) + 1];
                h[static_cast<std::size_t>(i)] = t;
            }
            const double denom = std::hypot(h[static_cast<std::size_t>(m)], h[static_cast<std::size_t>(m) + 1]);
            cs.push_back(denom == 0 ? 1.0 : h[static_cast<std::size_t>(m)] / denom);
            sn.push_back(denom == 0 ? 0.0 : h[static_cast<std::size_t>(m) + 1] / denom);
            h[static_cast<std::size_t>(m)] = denom;
            g.push_back(-sn[static_cast<std::size_t>(m)] * g[static_cast<std::size_t>(m)]);
            g[static_cast<std::size_t>(m)] = cs[static_cast<std::size_t>(m)] * g[static_cast<std::size_t>(m)];
            H.push_back(std::move(h));
            ++m;
            ++total;
            slot ^= 1;
            queued = spec;
            const double est = std::abs(g[static_cast<std::size_t>(m)]);
            check_finite(est, "gmres residual estimate");
            residuals.push_back(est);
            if (subdiag <= 1e-14 * wnorm0) breakdown = true;
            if (est <= target || breakdown) {
                converged = true;
                break;
            }
            // V[m] = w / subdiag was written by k_mgs_all (same sqrt of the same h)
        }
        if (m > 0) {
            std::vector<double> y(static_cast<std::size_t>(m), 0.0);
            for (int i = m - 1; i >= 0; --i) {
                double s = g[static_cast<std::size_t>(i)];
                for (int k = i + 1; k < m; ++k) s -= H[static_cast<std::size_t>(k)][static_cast<std::size_t>(i)] * y[static_cast<std::size_t>(k)];
                if (H[static_cast<std::size_t>(i)][static_cast<std::size_t>(i)] == 0.0)
                    throw DivergenceError("gmres encountered a singular projection");
                y[static_cast<std::size_t>(i)] = s / H[static_cast<std::size_t>(i)][static_cast<std::size_t>(i)];
            }
            double* yh = hh.p + 2 * (cap + 4);  // not a Hessenberg slot: a speculative step may still write those
            for (int k = 0; k < m; ++k) {
                vptr_h[static_cast<std::size_t>(k)] = basis(k);
                yh[k] = y[static_cast<std::size_t>(k)];
            }
            CPDDG_CUDA(cudaMemcpyAsync(vptr.get(), vptr_h.data(), sizeof(double*) * m, cudaMemcpyHostToDevice, st));
            CPDDG_CUDA(cudaMemcpyAsync(yd.get(), yh, sizeof(double) * m, cudaMemcpyHostToDevice, st));
            k_combine<<<ws.grid, kRedThreads, 0, st>>>(n, m, vptr.get(), yd.get(), tmp.get());
            CPDDG_CUDA(cudaGetLastError());
            ++ws.launches;
            if (pc) {
                kt.time(true, [&] { pc_apply(pc, tmp.get(), u, true, st); });
            } else {
                k_axpy1<<<ws.grid, kRedThreads, 0, st>>>(n, tmp.get(), u);
                CPDDG_CUDA(cudaGetLastError());
            }
            ++ws.launches;
            // keep the host copy of y alive until the transfer completed
            CPDDG_CUDA(cudaStreamSynchronize(st));
        }
        kt.time(false, [&] { op_residual(op, b, u, r.get(), nd + 1, st); });
        ws.launches += 2;
        fetch(nd + 1, 1);
        kt.collect();
        rnorm = std::sqrt(hh.p[0]);
    }
    // final_true_residual = ||b - A u|| (solve.hpp:212): r was just recomputed from u
    const double secs = timer.stop();
    kt.collect();
    record(log, residuals, total, converged, rnorm, secs, ws.launches, &kt);
}

/** solve.hpp:95-123 as one CUDA-graph launch: a while-conditional node whose
 *  body is u += M r, r = b - A u with ||r||^2, and the device checks
 *  (k_stat_check).  The graph is built per call (b, u are captured); the
 *  residual history comes back once at the end.  Bitwise equal to the host
 *  loop below (tests/test_gpu_parity.py::test_graph_stationary_matches_host_loop). */
static void stationary_graph(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params& prm,
                             cpddg_log* log, cudaStream_t st) {
    const int n = op->na;
    Workspace ws(n, st, op->kc);
    ws.reserve(2);
    KrylovCache& kc = op->kc;
    DevBuf<double>& r = ws.kc.r;
    double* rn2 = ws.kc.scal.get();
    Timer timer(st);
    CPDDG_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * n, st));
    CPDDG_CUDA(cudaMemcpyAsync(r.get(), b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    ws.mgs(nullptr, nullptr, r.get(), nullptr, rn2, nullptr);
    double* hp = ws.kc.host;
    CPDDG_CUDA(cudaMemcpyAsync(hp, rn2, sizeof(double), cudaMemcpyDeviceToHost, st));
    CPDDG_CUDA(cudaStreamSynchronize(st));
    const double r0 = std::sqrt(hp[0]);
    std::vector<double> residuals{r0};
    if (r0 == 0.0) {
        record(log, residuals, 0, true, 0.0, timer.stop(), ws.launches);
        return;
    }
    const std::size_t ssz = 8 + static_cast<std::size_t>(prm.max_iter) + 1;
    DevBuf<double> sb(ssz);
    if (!kc.gstream) CPDDG_CUDA(cudaStreamCreateWithFlags(&kc.gstream, cudaStreamNonBlocking));
    cudaGraph_t graph;
    CPDDG_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphExec_t exec = nullptr;
    struct Guard {
        cudaGraph_t& g;
        cudaGraphExec_t& e;
        ~Guard() {
            if (e) cudaGraphExecDestroy(e);
            cudaGraphDestroy(g);
        }
    } guard{graph, exec};
    cudaGraphConditionalHandle cond;
    CPDDG_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CPDDG_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStream_t cs = kc.gstream;
    CPDDG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
        pc_apply(pc, r.get(), u, true, cs);
        op_residual(op, b, u, r.get(), rn2, cs);
        k_stat_check<<<1, 32, 0, cs>>>(sb.get(), rn2, cond);
        CPDDG_CUDA(cudaGetLastError());
    } catch (...) {
        cudaGraph_t dummy;
        cudaStreamEndCapture(cs, &dummy);
        throw;
    }
    CPDDG_CUDA(cudaStreamEndCapture(cs, &body));
    CPDDG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    k_sstate_init<<<1, 1, 0, st>>>(sb.get(), prm.max_iter, r0, prm.rel_tol * r0);
    CPDDG_CUDA(cudaGetLastError());
    if (prm.max_iter > 0) CPDDG_CUDA(cudaGraphLaunch(exec, st));
    std::vector<double> hs(ssz);
    CPDDG_CUDA(cudaMemcpyAsync(hs.data(), sb.get(), sizeof(double) * ssz, cudaMemcpyDeviceToHost, st));
    CPDDG_CUDA(cudaStreamSynchronize(st));
    const SState* S = reinterpret_cast<const SState*>(hs.data());
    const int iters = S->it;
    for (int k = 1; k <= iters; ++k) residuals.push_back(hs[8 + static_cast<std::size_t>(k)]);
    ws.launches += 2 + static_cast<std::int64_t>(iters) * 4;
    if (S->status == kSNonFinite) throw DivergenceError("stationary residual is not finite");
    if (S->status == kSDiverged) throw DivergenceError("stationary iteration diverged");
    const double rn = residuals.back();
    const double secs = timer.stop();
    record(log, residuals, iters, S->status == kSConverged, iters ? rn : r0, secs, ws.launches);
}

// solve.hpp:95-123
static void stationary(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params& prm,
                       cpddg_log* log, cudaStream_t st) {
    const int n = op->na;
    if (!pc) throw InternalError("stationary iteration needs a preconditioner");
    if (pc->n_global != n) throw InternalError("preconditioner size does not match the operator");
    {
        // default: one graph launch for the whole iteration (see gmres() for the switches)
        const char* ge = std::getenv("CPDDG_GMRES_GRAPH");
        const bool forced = ge && std::string(ge) == "1";
        const bool host_loop = (ge && std::string(ge) == "0") || (prm.profile_kernels && !forced);
        if (!host_loop) {
            stationary_graph(op, pc, b, u, prm, log, st);
            return;
        }
    }
    Workspace ws(n, st, op->kc);
    ws.reserve(2);
    struct {
        double* p;
    } hh{ws.kc.host};
    DevBuf<double>& r = ws.kc.r;
    KernelTimer kt(op->kc.events);
    kt.on = prm.profile_kernels != 0;
    kt.st = st;
    Timer timer(st);
    CPDDG_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * n, st));
    CPDDG_CUDA(cudaMemcpyAsync(r.get(), b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    ws.mgs(nullptr, nullptr, r.get(), nullptr, ws.kc.scal.get(), nullptr);
    CPDDG_CUDA(cudaMemcpyAsync(hh.p, ws.kc.scal.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
    CPDDG_CUDA(cudaStreamSynchronize(st));
    const double r0 = std::sqrt(hh.p[0]);
    std::vector<double> residuals{r0};
    if (r0 == 0.0) {
        record(log, residuals, 0, true, 0.0, timer.stop(), ws.launches);
        return;
    }
    bool converged = false;
    int iters = 0;
    double rn = r0;
    for (int it = 1; it <= prm.max_iter; ++it) {
        kt.time(true, [&] { pc_apply(pc, r.get(), u, true, st); });
        kt.time(false, [&] { op_residual(op, b, u, r.get(), ws.kc.scal.get(), st); });
        ws.launches += 3;
        CPDDG_CUDA(cudaMemcpyAsync(hh.p, ws.kc.scal.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
        CPDDG_CUDA(cudaStreamSynchronize(st));
        kt.collect();
        rn = std::sqrt(hh.p[0]);
        check_finite(rn, "stationary residual");
        residuals.push_back(rn);
        iters = it;
        if (rn > 1e8 * r0) throw DivergenceError("stationary iteration diverged");
        if (rn <= prm.rel_tol * r0) {
            converged = true;
            break;
        }
    }
    const double secs = timer.stop();
    kt.collect();
    record(log, residuals, iters, converged, rn, secs, ws.launches, &kt);
}

}  // namespace cpddg

using namespace cpddg;

extern "C" {

int cpddg_gmres(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params* prm,
                cpddg_log* log, void* stream) {
    return guarded([&] {
        if (!op || !b || !u || !prm) throw InternalError("null argument");
        if (prm->max_iter < 0 || prm->restart < 0) throw ConfigError("max_iter and restart must be >= 0");
        if (!(prm->rel_tol > 0 && prm->rel_tol < 1)) throw ConfigError("rel_tol must lie strictly between 0 and 1");
        // CPDDG_VERBOSE: host time between two solve calls and inside this call beyond the device time
        static std::chrono::steady_clock::time_point last_exit{};
        const auto t_in = std::chrono::steady_clock::now();
        gmres(op, pc, b, u, *prm, log, static_cast<cudaStream_t>(stream));
        const auto t_out = std::chrono::steady_clock::now();
        if (std::getenv("CPDDG_VERBOSE") && log) {
            const double between = last_exit.time_since_epoch().count() ? std::chrono::duration<double>(t_in - last_exit).count() : 0.0;
            const double inside = std::chrono::duration<double>(t_out - t_in).count() - log->seconds;
            if (between > 2e-3 || inside > 2e-3)
                std::fprintf(stderr, "[cpddg] gmres call: %.1f ms since the previous call returned, %.1f ms in the call beyond the device time\n",
                             1e3 * between, 1e3 * inside);
        }
        last_exit = t_out;
    });
}

int cpddg_stationary(cpddg_op* op, cpddg_pc* pc, const double* b, double* u, const cpddg_solve_params* prm,
                     cpddg_log* log, void* stream) {
    return guarded([&] {
        if (!op || !b || !u || !prm) throw InternalError("null argument");
        if (!(prm->rel_tol > 0 && prm->rel_tol < 1)) throw ConfigError("rel_tol must lie strictly between 0 and 1");
        stationary(op, pc, b, u, *prm, log, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
