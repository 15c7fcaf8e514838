// df_u12 (lu.cu: U12 = L11^{-1} A12 for nc columns) timed alone in a 256-thread CTA (cycles per call).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      -I paper_1509_07919_b200/csrc tools/probe/u12_probe.cu -o tools/probe/u12_probe
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <cstdio>

namespace sapgpu {
long long g_launch_count = 0;
}
using namespace sapgpu;

__device__ long long g_cyc[8];

__global__ void __launch_bounds__(256, 2) k_u12(int nc, double* gbuf, int slot, int reps) {
    extern __shared__ __align__(16) double smem[];
    const int pld = 236, uld = 100;
    double* P = smem;
    double* U = smem + 32 * pld;
    for (int i = threadIdx.x; i < 32 * pld; i += 256) P[i] = (i % pld == i / pld) ? 1.0 : 0.001 * ((i * 7) % 13 - 6);
    __syncthreads();
    Lu L{gbuf, 1, 401, 4000, 200, 32, pld, uld, 0.0, gbuf};
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
        for (int i = threadIdx.x; i < 32 * uld; i += 256) U[i] = 0.01 * ((i * 5 + r) % 11 - 5);
        __syncthreads();
        const long long t0 = clock64();
        df_u12<256>(L, 0, 32, 0, nc, nc, P, pld, U, uld);
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) g_cyc[slot] = tot / reps;
}

int main() {
    double* g;
    cudaMalloc(&g, sizeof(double) * 4000 * 401);
    const size_t smem = sizeof(double) * (32 * 236 + 32 * 100);
    cudaFuncSetAttribute(k_u12, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_u12<<<1, 256, smem>>>(32, g, 0, 50);
    k_u12<<<1, 256, smem>>>(96, g, 1, 50);
    cudaDeviceSynchronize();
    long long c[8];
    cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
    printf("df_u12 cycles per call: nc=32 %lld, nc=96 %lld (%s)\n", c[0], c[1], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
