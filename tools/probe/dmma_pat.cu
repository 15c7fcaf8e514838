// DMMA (mma.sync m8n8k4 f64) throughput vs. issue pattern, one CTA per SM (148 CTAs):
// warps per CTA, independent accumulator chains per warp, operands from registers or shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// NC chains; SMEM: operands (1 a per chain-column group, 1 b per row group) loaded from smem every k-step
template <int NC, int SMEM>
__global__ void k(double* out, int iters, long long* cyc) {
    __shared__ double sa[64 * 64];
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sa[i] = 1e-3 * (i % 17);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double c[NC][2];
#pragma unroll
    for (int t = 0; t < NC; ++t) c[t][0] = c[t][1] = 0;
    double a = lane * 1e-3, b = lane * 2e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (SMEM) {
            // 16x32 tile pattern: NC = 8 -> 2 b (rows) x 4 a (cols) operands per k-step
            double av[NC / 2 > 0 ? NC / 2 : 1], bv[2];
            const int kk = (i & 7) * 4 + (lane & 3);
#pragma unroll
            for (int q = 0; q < NC / 2; ++q) av[q] = sa[kk * 64 + q * 8 + (lane >> 2)];
            bv[0] = sa[2048 + kk * 64 + (lane >> 2)];
            bv[1] = sa[2048 + kk * 64 + 8 + (lane >> 2)];
#pragma unroll
            for (int q = 0; q < NC / 2; ++q) {
                mma(c[2 * q][0], c[2 * q][1], av[q], bv[0]);
                mma(c[2 * q + 1][0], c[2 * q + 1][1], av[q], bv[1]);
            }
        } else {
#pragma unroll
            for (int t = 0; t < NC; ++t) mma(c[t][0], c[t][1], a, b);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int t = 0; t < NC; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NC, int SMEM>
void run(int threads, double* out, long long* cyc) {
    const int iters = 2000;
    k<NC, SMEM><<<148, threads>>>(out, 10, cyc);
    cudaDeviceSynchronize();
    k<NC, SMEM><<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    const double dmma_per_sm = (double)iters * NC * (threads / 32);
    printf("warps %2d chains %2d %s: %.2f clk per DMMA per SM (4.0 = peak)  %s\n", threads / 32, NC,
           SMEM ? "smem operands" : "reg operands ", (double)mx / dmma_per_sm, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMallocManaged(&cyc, 148 * 8);
    for (int th : {128, 256, 512, 1024}) {
        run<4, 0>(th, out, cyc);
        run<8, 0>(th, out, cyc);
        run<16, 0>(th, out, cyc);
        run<8, 1>(th, out, cyc);
        run<16, 1>(th, out, cyc);
    }
    return 0;
}
