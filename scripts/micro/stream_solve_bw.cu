// Full-chip streaming read bandwidth with the k_solve load pattern (development
// microbenchmark): G CTAs of T threads, each streaming its own contiguous
// slice with 16-byte ld.global.nc.L1::no_allocate loads, U loads in flight per
// lane, no dependencies.  The ceiling of a register-staged solve.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double2 ldn(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int U>
__global__ void __launch_bounds__(512, 2) k_stream(const double2* __restrict__ p, long long n2_per_cta, double* out) {
    const double2* q = p + blockIdx.x * n2_per_cta;
    double acc = 0.0;
    const int T = blockDim.x;
    for (long long b = threadIdx.x; b < n2_per_cta; b += (long long)T * U) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = (b + u * T < n2_per_cta) ? ldn(q + b + u * T) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y;
    }
    if (acc == 12345.0) out[0] = acc;
}
int main(int argc, char** argv) {
    const bool one = argc > 1;  // one config (256 x 512, U 4) for profiling
    const long long total = 10LL << 30;  // 10 GB
    double2* p; double* out;
    cudaMalloc(&p, total); cudaMalloc(&out, 8);
    cudaMemset(p, 0, total);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int ctas : {148, 256, 296}) {
        for (int T : {256, 512}) {
            for (int U : {4, 8}) {
                if (one && !(ctas == 256 && T == 512 && U == 4)) continue;
                const long long per = total / ctas / 16 / 1024 * 1024;
                auto run = [&] {
                    if (U == 4) k_stream<4><<<ctas, T>>>(p, per, out);
                    if (U == 8) k_stream<8><<<ctas, T>>>(p, per, out);
                };
                run(); cudaDeviceSynchronize();
                cudaEventRecord(e0);
                for (int r = 0; r < 3; ++r) run();
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                printf("ctas %d threads %d U %d: %.0f GB/s\n", ctas, T, U, 3.0 * per * 16 * ctas / (ms * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
