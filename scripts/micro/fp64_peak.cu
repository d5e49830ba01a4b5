// Measured FP64 peaks of this B200 (denominators for k_factor's DMMA
// fraction): DFMA (CUDA cores) and DMMA
// (mma.sync.m8n8k4.f64, the FP64 tensor path; tcgen05 has no f64 kind).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma(double* out) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[0] = s;
}

// DFMA and DMMA interleaved in one instruction stream: if the two paths are
// separate pipes, the combined rate exceeds either alone.
__global__ void k_mixed(double* out, double fa, double fb) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
    double c[8][2], x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0, x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = fma(x[q], fa, fb);
        }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + x[k];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best_fma = 0, best_mma = 0;
    for (int rep = 0; rep < 5; ++rep) {
        const int blocks = sms * 8, threads = 256;
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * kIters * 8 * double(blocks) * threads;
        if (rep) best_fma = fmax(best_fma, flops / (ms * 1e-3) / 1e12);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double mflops = 512.0 * kIters * 8 * double(blocks) * (threads / 32);
        if (rep) best_mma = fmax(best_mma, mflops / (ms * 1e-3) / 1e12);
    }
    double best_mix = 0, mix_ms = 0;
    for (int rep = 0; rep < 5; ++rep) {
        const int blocks = sms * 8, threads = 256;
        cudaEventRecord(e0);
        k_mixed<<<blocks, threads>>>(out, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 512.0 * kIters * 8 * double(blocks) * (threads / 32) + 2.0 * kIters * 64 * double(blocks) * threads;
        if (rep && flops / (ms * 1e-3) / 1e12 > best_mix) best_mix = flops / (ms * 1e-3) / 1e12, mix_ms = ms;
    }
    std::printf("{\"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"mixed_tflops\": %.2f, \"mixed_ms\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n", best_fma,
                best_mma, best_mix, mix_ms, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
