// Round-trip latency of one batch of independent 16-byte loads per thread
// (single CTA of 512 threads; development microbenchmark).
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void k_rt(const double2* __restrict__ p, long long stride2, int rounds, long long* out, double* sink) {
    double acc = 0.0;
    long long tsum = 0;
    const double2* q = p + threadIdx.x;
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();
        const long long t0 = clock64();
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = __ldcs(q + (static_cast<long long>(r) * U + u) * stride2);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u].x;
        __syncthreads();
        tsum += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = tsum / rounds;
    if (acc == 1.2345) sink[0] = acc;
}
int main() {
    const long long bytes = 1LL << 30;
    double2* p; long long* out; double* sink;
    cudaMalloc(&p, bytes); cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
    cudaMemset(p, 0, bytes);
    long long h;
    for (int threads : {32, 512}) {
        // stride: each round's loads hit fresh memory (DRAM); 1 MB apart
        for (int U : {1, 4, 8}) {
            const long long stride2 = (1 << 20) / 16;
            const int rounds = 64;
            if (U == 1) k_rt<1><<<1, threads>>>(p, stride2, rounds, out, sink);
            if (U == 4) k_rt<4><<<1, threads>>>(p, stride2, rounds, out, sink);
            if (U == 8) k_rt<8><<<1, threads>>>(p, stride2, rounds, out, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("threads %3d U %d: %lld cycles per round (DRAM, cold)\n", threads, U, h);
        }
        // L2-resident: same small buffer every round
        for (int U : {1, 4, 8}) {
            const long long stride2 = 4096 / 16;
            if (U == 1) k_rt<1><<<1, threads>>>(p, stride2, 64, out, sink);
            if (U == 4) k_rt<4><<<1, threads>>>(p, stride2, 64, out, sink);
            if (U == 8) k_rt<8><<<1, threads>>>(p, stride2, 64, out, sink);
            cudaDeviceSynchronize();
            if (U == 1) k_rt<1><<<1, threads>>>(p, stride2, 64, out, sink);
            if (U == 4) k_rt<4><<<1, threads>>>(p, stride2, 64, out, sink);
            if (U == 8) k_rt<8><<<1, threads>>>(p, stride2, 64, out, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("threads %3d U %d: %lld cycles per round (L2 warm)\n", threads, U, h);
        }
    }
    return 0;
}
