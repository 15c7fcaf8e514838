// panel_diag (lu.cu) timed alone on one SM vs beside a DMMA-saturating CTA on the same SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      -I paper_1509_07919_b200/csrc tools/probe/diag_probe.cu -o tools/probe/diag_probe
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <cstdio>

namespace sapgpu {
long long g_launch_count = 0;
}
using namespace sapgpu;

__device__ long long g_cyc[4];
__device__ double g_sink;

// blockIdx 0: panel_diag x reps (warp 0); blockIdx 1 (mode 1): DMMA loop on all warps; mode 2: DFMA loop
__global__ void __launch_bounds__(512, 1) k_probe(int mode, int reps) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(16) double s_ut[kUtSize];
    __shared__ double s_rcp[64];
    __shared__ int s_b;
    const int pld = 236;
    for (int i = threadIdx.x; i < 32 * pld; i += 512) smem[i] = (i % pld == i / pld) ? 40.0 : 0.01 * ((i * 7) % 13 - 6);
    if (threadIdx.x == 0) s_b = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            panel_diag<32, true>(smem, pld, s_ut, s_rcp, 32, 1e-10, &s_b);
            __syncwarp();
        }
        if (threadIdx.x == 0) g_cyc[mode] = (clock64() - t0) / reps;
        if (threadIdx.x == 0) g_sink = smem[5];
    } else if (threadIdx.x >= 256 && mode == 1) {
        double a = threadIdx.x, b = 1.0, c0 = 0, c1 = 0;
        for (int r = 0; r < reps * 2000; ++r) dmma_m8n8k4(c0, c1, a, b, c0, c1);
        if (c0 == 12345.0) g_sink = c1;
    } else if (threadIdx.x >= 256 && mode == 2) {
        double x = threadIdx.x, y = 1.0, z = 0.5, w = 0.25;
        for (int r = 0; r < reps * 2000; ++r) { x = fma(x, y, z); w = fma(w, y, z); }
        if (x == 12345.0) g_sink = w;
    }
}

int main() {
    const size_t smem = 32 * 236 * 8 + 32 * 36 * 8;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 3; ++mode) {
        k_probe<<<1, 512, smem>>>(mode, 200);
        cudaDeviceSynchronize();
    }
    long long c[4];
    cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
    printf("panel_diag cycles per call: alone %lld, beside DMMA CTA %lld, beside DFMA CTA %lld (%s)\n", c[0], c[1], c[2],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
