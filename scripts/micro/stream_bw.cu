// Single-SM / full-chip streaming read bandwidth (development microbenchmark):
// each CTA streams its own contiguous slice with 16-byte __ldcs loads,
// U loads in flight per lane.
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void __launch_bounds__(512) k_stream(const double2* __restrict__ p, long long n2_per_cta, double* out) {
    const double2* q = p + blockIdx.x * n2_per_cta;
    double acc = 0.0;
    for (long long b = threadIdx.x; b < n2_per_cta; b += 512LL * U) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = (b + u * 512 < n2_per_cta) ? __ldcs(q + b + u * 512) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y;
    }
    if (acc == 12345.0) out[0] = acc;
}
int main() {
    const long long bytes_per_cta = 64LL << 20;  // 64 MB per CTA
    const int maxc = 296;
    double2* p; double* out;
    cudaMalloc(&p, bytes_per_cta * maxc); cudaMalloc(&out, 8);
    cudaMemset(p, 0, bytes_per_cta * maxc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int ctas : {1, 2, 148, 296}) {
        for (int U : {4, 8, 16}) {
            auto run = [&] {
                if (U == 4) k_stream<4><<<ctas, 512>>>(p, bytes_per_cta / 16, out);
                if (U == 8) k_stream<8><<<ctas, 512>>>(p, bytes_per_cta / 16, out);
                if (U == 16) k_stream<16><<<ctas, 512>>>(p, bytes_per_cta / 16, out);
            };
            run(); cudaDeviceSynchronize();
            cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("ctas %3d U %2d: %.3f ms  %.1f GB/s total, %.1f GB/s per CTA\n", ctas, U, ms,
                   bytes_per_cta * ctas / ms / 1e6, bytes_per_cta / ms / 1e6);
        }
    }
    return 0;
}
