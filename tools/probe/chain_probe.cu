// The dataflow LU chain item's compute phases (lu.cu) on one SM, timed per phase with clock64 (no dependency
// waits, no other SMs busy): top-rows update, panel_diag (warp 0) beside the rows-[32, R) update (warps 1-7),
// then the L21 rows. Compare with the in-kernel phase trace (tools/lu_df_trace.py) to see what the
// environment adds.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      -I paper_1509_07919_b200/csrc tools/probe/chain_probe.cu -o tools/probe/chain_probe
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <cstdio>

namespace sapgpu {
long long g_launch_count = 0;
}
using namespace sapgpu;

__device__ long long g_ph[4];

__global__ void __launch_bounds__(256, 1) k_chain(double* band, int reps) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(16) double s_ut[kUtSize];
    __shared__ double s_rcp[64];
    __shared__ int s_b;
    constexpr int K = 200, B = 32;
    const int pld = 236, uld = 100, m = 4000;
    double* P = smem;
    double* U = smem + 32 * pld;
    const int tid = threadIdx.x, warp = tid >> 5;
    Lu L{band, 1, 2 * K + 1, m, K, B, pld, uld, 1e-10, band};  // column-major band: (i, c) at i + c (2K+1)
    const DfTile T{64, K, 0, 32, 0};
    long long acc[4] = {0, 0, 0, 0};
    if (tid == 0) s_b = 0;
    for (int r = 0; r < reps; ++r) {
        for (int i = tid; i < 32 * pld; i += 256) P[i] = (i % pld == i / pld) ? 40.0 + r : 0.01 * ((i * 7 + r) % 13 - 6);
        for (int i = tid; i < 32 * uld; i += 256) U[i] = 0.01 * ((i * 5 + r) % 11 - 5);
        __syncthreads();
        long long t0 = clock64();
        df_upd_top<256>(L, T, P, pld, U, uld);  // ends with a barrier
        long long t1 = clock64(), t2 = 0;
        if (warp == 0) {
            panel_diag<B, true>(P, pld, s_ut, s_rcp, 32, 1e-10, &s_b);
            t2 = clock64();
        } else {
            df_upd_rest<256>(L, T, P, pld, U, uld);
        }
        __syncthreads();
        const long long t3 = clock64();
        df_rows<B, true, 256>(P, pld, s_ut, s_rcp, 32, 32 + K);
        __syncthreads();
        const long long t4 = clock64();
        if (tid == 0) {
            acc[0] += t1 - t0;
            acc[1] += t2 - t1;
            acc[2] += t3 - t1;
            acc[3] += t4 - t3;
        }
    }
    if (tid == 0)
        for (int q = 0; q < 4; ++q) g_ph[q] = acc[q] / reps;
}

int main() {
    double* band;
    const size_t n = (size_t)4000 * 401;
    cudaMalloc(&band, n * sizeof(double));
    cudaMemset(band, 0, n * sizeof(double));
    const size_t smem = sizeof(double) * (32 * 236 + 32 * 100);
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_chain<<<1, 256, smem>>>(band, 50);
    cudaDeviceSynchronize();
    long long ph[4];
    cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
    printf("cycles: top update %lld, panel_diag %lld (diag || rest: %lld), rows %lld (%s)\n", ph[0], ph[1], ph[2],
           ph[3], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
