// Dependent-chain latencies on one warp: DFMA, SHFL.IDX, LDS.64 (development microbenchmark).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sh[64];
    sh[threadIdx.x] = threadIdx.x;
    __syncwarp();
    double s = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) s = fma(s, a, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (i + threadIdx.x) & 31);
    long long t2 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) idx = static_cast<int>(sh[idx & 31]) ^ 1;
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) { s = fma(s, a, b); s = __shfl_sync(0xffffffffu, s, i & 31); }
    long long t4 = clock64();
    out[threadIdx.x] = s + idx;
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    k<<<1, 32>>>(o, c, 0.999, 0.001, 4096); cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("DFMA %lld  SHFL %lld  LDS(dep) %lld  DFMA+SHFL %lld cycles\n", h[0], h[1], h[2], h[3]);
}
