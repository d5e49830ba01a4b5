// Per-SM intake of cp.async.bulk (global -> shared, mbarrier complete_tx) with a
// ring of NS slots of CH bytes; one producer thread, all threads "consume"
// (touch one word per slot) -- development microbenchmark.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                 ::"r"(smem_u32(b)), "r"(phase) : "memory");
}
template <int NS, int CH>
__global__ void __launch_bounds__(512) k(const char* __restrict__ g, long long bytes_per_cta, double* out) {
    extern __shared__ __align__(128) char ring[];
    __shared__ uint64_t full[NS];
    const char* src = g + blockIdx.x * bytes_per_cta;
    const int nchunks = static_cast<int>(bytes_per_cta / CH);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int c = 0; c < NS && c < nchunks; ++c) {
            mbar_expect_tx(&full[c], CH);
            bulk_g2s(ring + c * CH, src + static_cast<long long>(c) * CH, CH, &full[c]);
        }
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const int s = c % NS;
        mbar_wait(&full[s], (c / NS) & 1);
        acc += reinterpret_cast<const double*>(ring + s * CH)[threadIdx.x % (CH / 8)];
        __syncthreads();  // slot consumed
        if (threadIdx.x == 0 && c + NS < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[s], CH);
            bulk_g2s(ring + s * CH, src + static_cast<long long>(c + NS) * CH, CH, &full[s]);
        }
    }
    if (acc == 1.2345) out[0] = acc;
}
template <int NS, int CH>
void run(const char* g, double* out, int ctas, long long bpc) {
    auto kern = k<NS, CH>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * CH);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<ctas, 512, NS * CH>>>(g, bpc, out); cudaDeviceSynchronize();
    cudaEventRecord(e0); kern<<<ctas, 512, NS * CH>>>(g, bpc, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("NS %d CH %6d ctas %3d: %.1f GB/s total, %.1f GB/s per CTA %s\n", NS, CH, ctas, bpc * ctas / ms / 1e6,
           bpc / ms / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
}
int main() {
    const long long bpc = 32LL << 20;
    char* g; double* out;
    cudaMalloc(&g, bpc * 296); cudaMalloc(&out, 8); cudaMemset(g, 0, bpc * 296);
    for (int ctas : {1, 148, 296}) {
        run<2, 32768>(g, out, ctas, bpc);
        run<4, 32768>(g, out, ctas, bpc);
        if (ctas != 296) run<6, 32768>(g, out, ctas, bpc);
        run<4, 16384>(g, out, ctas, bpc);
        if (ctas != 296) run<3, 65536>(g, out, ctas, bpc);
    }
}
