// Throughput of scalar FFMA vs packed FFMA2 on sm_100a (diagnostics).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void k_scalar(float* out, int iters, float s) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], s, a[(i + 1) & 15]);
    float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_packed(float* out, int iters, float s) {
    f32x2 a[8];
    f32x2 ss; asm("mov.b64 %0, {%1, %2};" : "=l"(ss) : "f"(s), "f"(s));
    for (int i = 0; i < 8; ++i) { float x = threadIdx.x * 0.001f + i; asm("mov.b64 %0, {%1, %2};" : "=l"(a[i]) : "f"(x), "f"(x + 0.5f)); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], ss, a[(i + 1) & 7]);
    float r = 0; for (int i = 0; i < 8; ++i) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i])); r += lo + hi; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_scalar<<<148 * 8, 256>>>(d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 148.0 * 8 * 256 * iters * 16;
        printf("scalar FFMA: %.2f ms, %.1f TFMA/s, %.2f FMA/clk/SM at 1.965 GHz\n", ms, fl / ms / 1e9, fl / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(e0); k_packed<<<148 * 8, 256>>>(d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2: %.2f ms, %.1f TFMA/s, %.2f FMA/clk/SM\n", ms, fl / ms / 1e9, fl / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
