// Microbenchmark: FP32 FMA issue rates on this GPU (scalar FFMA 3-reg form vs packed FFMA2).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, float a, float b, int iters) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ unsigned long long f2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long x, unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(a), "l"(b));
    return r;
}

__global__ void ffma2_kernel(float* out, float a, float b, int iters) {
    const unsigned long long A = f2(a, a), B = f2(b, b);
    unsigned long long x0 = f2(threadIdx.x, 1), x1 = f2(2, 3), x2 = f2(4, 5), x3 = f2(6, 7);
    unsigned long long x4 = f2(8, 9), x5 = f2(10, 11), x6 = f2(12, 13), x7 = f2(14, 15);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = fma2(x0, A, B); x1 = fma2(x1, A, B); x2 = fma2(x2, A, B); x3 = fma2(x3, A, B);
            x4 = fma2(x4, A, B); x5 = fma2(x5, A, B); x6 = fma2(x6, A, B); x7 = fma2(x7, A, B);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = float((x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7) & 0xff);
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float) * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms1, ms2;
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventRecord(e0);
        ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms2, e0, e1);
        const double lanes = double(blocks) * threads * iters * 64;   // FMA lane-ops (ffma); x2 for ffma2
        printf("FFMA : %.3f ms  %.2f T lane-FMA/s\n", ms1, lanes / ms1 / 1e9);
        printf("FFMA2: %.3f ms  %.2f T lane-FMA/s\n", ms2, 2 * lanes / ms2 / 1e9);
    }
    return 0;
}
