// Single-CTA streaming rate for load flavours (development microbenchmark):
// ld.global.cs (__ldcs), ld.global.nc (__ldg), ld.global.nc.L1::no_allocate.L2::256B.
#include <cstdio>
template <int KIND>
__device__ __forceinline__ double2 ld2(const double2* p) {
    if constexpr (KIND == 0) return __ldcs(p);
    if constexpr (KIND == 1) return __ldg(p);
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int KIND, int U>
__global__ void __launch_bounds__(512) k(const double2* __restrict__ p, long long n2, double* out) {
    const double2* q = p + blockIdx.x * n2;
    double acc = 0.0;
    for (long long b = threadIdx.x; b < n2; b += 512LL * U) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = (b + u * 512 < n2) ? ld2<KIND>(q + b + u * 512) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y;
    }
    if (acc == 1.2345) out[0] = acc;
}
template <int KIND>
void run(const double2* p, double* out, int ctas, long long bytes) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<KIND, 8><<<ctas, 512>>>(p, bytes / 16, out); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<KIND, 8><<<ctas, 512>>>(p, bytes / 16, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("kind %d ctas %3d: %.1f GB/s per CTA, %.0f GB/s total\n", KIND, ctas, bytes / ms / 1e6, bytes * ctas / ms / 1e6);
}
int main() {
    const long long bytes = 32LL << 20;
    double2* p; double* out;
    cudaMalloc(&p, bytes * 296); cudaMalloc(&out, 8); cudaMemset(p, 0, bytes * 296);
    for (int ctas : {1, 296}) { run<0>(p, out, ctas, bytes); run<1>(p, out, ctas, bytes); run<2>(p, out, ctas, bytes); }
}
