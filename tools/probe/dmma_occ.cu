// DMMA.8x8x4 throughput vs resident warps per SM and independent accumulator chains per warp
// (one CTA per SM; operands in registers, or re-read from shared memory every k-step like the LU update).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, bool SMEM>
__global__ void k(double* out, int iters, long long* cyc) {
    __shared__ double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-6;
    __syncthreads();
    double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
    double c[CH][2];
#pragma unroll
    for (int t = 0; t < CH; ++t) { c[t][0] = 0; c[t][1] = 0; }
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (SMEM) {
            a = sm[(i * 64 + lane * 2) & 4095];
            b = sm[(i * 64 + lane * 2 + 1024) & 4095];
        }
#pragma unroll
        for (int t = 0; t < CH; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH, bool SMEM>
void run(int warps, int sms, double* out, long long* cyc) {
    const int iters = 2000;
    k<CH, SMEM><<<sms, warps * 32>>>(out, 10, cyc);
    cudaDeviceSynchronize();
    k<CH, SMEM><<<sms, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double dmma_per_sm = (double)iters * CH * warps;
    printf("warps/SM %2d chains %2d smem %d: %.2f cycles per DMMA per SM (floor 4.0)\n", warps, CH, (int)SMEM,
           c / dmma_per_sm);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 1 << 24);
    long long* cyc; cudaMalloc(&cyc, 8);
    for (int w : {1, 4, 8, 16, 32}) {
        run<8, false>(w, sms, out, cyc);
        run<16, false>(w, sms, out, cyc);
        run<8, true>(w, sms, out, cyc);
    }
    run<1, false>(1, 1, out, cyc);
}
