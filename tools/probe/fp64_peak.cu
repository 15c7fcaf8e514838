// FP64 peak microbenchmarks for B200 (sm_100a): DFMA and DMMA (mma.sync m8n8k4 f64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) out[i] = in[i];
}

int main() {
    int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
    int sms = prop.multiProcessorCount;
    printf("device %s SMs %d clock %d kHz\n", prop.name, sms, prop.clockRate);
    double* out; cudaMalloc(&out, 1 << 26);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        int blocks = sms * (2048 / threads);
        int iters = 2000;
        dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 64 * iters * (double)blocks * threads;
        printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
    for (int warps : {4, 8, 16}) {
        int threads = warps * 32, blocks = sms * (2048 / threads) / 2;
        int iters = 4000;
        dmma_kernel<<<blocks, threads>>>(out, 10);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * blocks * warps;
        printf("DMMA m8n8k4 warps/blk=%d blocks=%d: %.2f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    }
    size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("copy: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
    }
    cudaError_t err = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(err));
    return 0;
}
