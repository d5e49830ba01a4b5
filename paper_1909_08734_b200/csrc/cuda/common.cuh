// Shared device plumbing: error checks, owning device buffers, and
// deterministic (fixed-order) block reductions.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cpddg {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CPDDG_CUDA(call) ::cpddg::cuda_check((call), #call)

/** Owning device allocation. */
template <class T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), owns_(o.owns_) {
        o.p_ = nullptr;
        o.n_ = 0;
        o.owns_ = true;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            owns_ = o.owns_;
            o.p_ = nullptr;
            o.n_ = 0;
            o.owns_ = true;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(std::size_t n) {
        release();
        if (n) CPDDG_CUDA(cudaMalloc(&p_, n * sizeof(T)));
        n_ = n;
    }
    void upload(const std::vector<T>& h) {
        alloc(h.size());
        if (!h.empty()) CPDDG_CUDA(cudaMemcpy(p_, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    }
    void upload(const T* h, std::size_t n) {
        alloc(n);
        if (n) CPDDG_CUDA(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice));
    }
    void zero(cudaStream_t s = nullptr) {
        if (n_) CPDDG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }
    std::size_t bytes() const { return n_ * sizeof(T); }
    /** Become a non-owning view of n elements at p (storage owned by a slab that outlives this). */
    void view(T* p, std::size_t n) {
        release();
        p_ = p;
        n_ = n;
        owns_ = false;
    }

private:
    void release() {
        if (p_ && owns_) cudaFree(p_);
        owns_ = true;
        p_ = nullptr;
        n_ = 0;
    }
    T* p_ = nullptr;
    std::size_t n_ = 0;
    bool owns_ = true;
};

/** Number of SMs of the current device (148 on B200). */
int sm_count();

/** Grid size used by every reduction kernel: a fixed multiple of the SM
 *  count, so partial sums (and hence results) do not depend on the launch
 *  history. */
int reduction_blocks();

constexpr int kRedThreads = 256;
constexpr int kExtTile = 256;      // max band nodes per staged-extension tile (one per thread)
#ifndef CPDDG_EXT_CAP
#define CPDDG_EXT_CAP 4096
#endif
constexpr int kExtStageCap = CPDDG_EXT_CAP; // max staged x entries per tile (8 B of shared memory each)
// grouped extension (k_extend_grouped): chunks of kGrpThreads threads (two
// band nodes of one stencil base each) touching <= kGrpMax bases; a base's
// 4x4x4 x block sits at stride kGrpSS doubles, its axis-0 slices at stride
// kGrpAS (the pads put up to 8 bases' 16-byte words in distinct shared banks)
constexpr int kGrpThreads = 128;
constexpr int kUnionMax = 768;   // staged x values per chunk of k_extend_union
constexpr int kGrpMax = 36;
static_assert(kGrpMax <= 64, "k_extend_union packs the base slot in 6 bits of the slot byte");
constexpr int kGrpSS = 82;
constexpr int kGrpAS = 18;

// Fixed-order block sum: warp shuffles (xor tree) then warp 0 over the 8
// warp partials.  Deterministic for a fixed blockDim.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NT / 32 ? sh[l] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

/** Device scalar slots used by the Krylov kernels. */
struct ReduceWork {
    DevBuf<double> partials;      // reduction_blocks() entries per slot
    DevBuf<unsigned int> counter; // last-block-done tickets
    void ensure(int slots);
    int slots = 0;
};

}  // namespace cpddg
