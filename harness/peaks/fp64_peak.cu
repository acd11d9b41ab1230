// Micro-benchmark: fp64 peak of the CUDA-core pipe (DFMA) and of the fp64 tensor-core
// path (DMMA.8x8x4 via mma.sync.m8n8k4.f64) on the current GPU. Many independent
// accumulator chains per warp, all SMs busy; CUDA-event timed. Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
    double d[8][2];
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
    const double a = 1e-3 * (threadIdx.x & 31), b = 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
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
    const int threads = 512, blocks = sms * 4, iters = 4096;
    float ms = 0;
    dfma_kernel<<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma_tf = 2.0 * blocks * threads * iters * 16 / (ms * 1e-3) / 1e12;
    dmma_kernel<<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * (threads / 32.0);
    const double dmma_tf = 2.0 * warps * iters * 8 * 256 / (ms * 1e-3) / 1e12;
    printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"sms\": %d}\n", dfma_tf, dmma_tf, sms);
    return 0;
}
