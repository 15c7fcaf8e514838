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
__device__ long long g_groups[8];

__global__ void __launch_bounds__(256, 1) k_chain(double* band, int reps, int nchain, int* flag, double* wbuf,
                                                  int marks) {
    extern __shared__ __align__(16) double smem[];
    __shared__ unsigned long long s_marks[10];
    if ((int)blockIdx.x >= nchain) {  // the other SMs: DMMA + L2 traffic (like the worker strips) until done
        double a = threadIdx.x, b = 1.0, c0 = 0, c1 = 0, s = 0;
        const size_t nw = (size_t)1 << 24;
        size_t off = ((size_t)blockIdx.x * 256 + threadIdx.x) * 2;
        while (*(volatile int*)flag < nchain) {
            for (int r = 0; r < 200; ++r) dmma_m8n8k4(c0, c1, a, b, c0, c1);
            s += __ldcg(wbuf + off % nw);
            wbuf[(off + 4096) % nw] = c0;
            off += 148 * 256 * 2;
        }
        if (c0 == 12345.0 || s == 12345.0) band[0] = c1;
        return;
    }
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
            panel_diag<B, true>(P, pld, s_ut, s_rcp, 32, 1e-10, &s_b, marks ? s_marks : nullptr);
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
    if (tid == 0 && blockIdx.x == 0) {
        for (int q = 0; q < 4; ++q) g_ph[q] = acc[q] / reps;
        if (marks)
            for (int q = 0; q < 8; ++q) g_groups[q] = s_marks[q + 1] - s_marks[q];  // the last call's 4-pivot groups
    }
    if (tid == 0) atomicAdd(flag, 1);
}

int main() {
    double* band;
    const size_t n = (size_t)4000 * 401;
    cudaMalloc(&band, n * sizeof(double));
    cudaMemset(band, 0, n * sizeof(double));
    const size_t smem = sizeof(double) * (32 * 236 + 32 * 100);
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int* flag;
    double* wbuf;
    cudaMalloc(&flag, sizeof(int));
    cudaMalloc(&wbuf, sizeof(double) << 24);
    cudaMemset(wbuf, 0, sizeof(double) << 24);
    for (int busy = 0; busy < 3; ++busy) {
        cudaMemset(flag, 0, sizeof(int));
        k_chain<<<busy == 1 ? 148 : 1, 256, smem>>>(band, 50, busy == 1 ? 50 : 1, flag, wbuf, busy == 2);
        cudaDeviceSynchronize();
        long long ph[4];
        cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
        printf("%s cycles: top update %lld, panel_diag %lld (diag || rest: %lld), rows %lld (%s)\n",
               busy == 1 ? "50 chains + 98 SMs DMMA/L2:" : busy ? "1 CTA, trace marks on:" : "1 CTA alone:", ph[0], ph[1], ph[2], ph[3],
               cudaGetErrorString(cudaGetLastError()));
    }
    long long gr[8];
    cudaMemcpyFromSymbol(gr, g_groups, sizeof(gr));
    printf("4-pivot groups (us at 1.965 GHz):");
    for (int q = 0; q < 8; ++q) printf(" %.2f", gr[q] / 1965.0);
    printf("\n");
    return 0;
}
