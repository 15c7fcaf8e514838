// Per-call panel_diag (lu.cu) cycles on warp 0 of a 256-thread CTA, in the dataflow LU chain's settings:
//   mode 0: warps 1-7 idle;  mode 1: warps 1-7 run a DFMA burst (~the chain's rows-[32, R) update) beside it;
//   mode 2: the burst first, then the pivot chain (serial);
// on `nchain` CTAs (one per SM), optionally with the remaining SMs running DMMA loops (the worker strips).
// Prints the per-call distribution: the chain trace (tools/lu_df_trace.py) shows a bimodal panel_diag.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      -I paper_1509_07919_b200/csrc tools/probe/diag_throttle.cu -o tools/probe/diag_throttle
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <algorithm>
#include <cstdio>
#include <vector>

namespace sapgpu {
long long g_launch_count = 0;
}
using namespace sapgpu;

__device__ double g_sink;
constexpr int kCalls = 200;

__device__ __forceinline__ void burst(int n) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
    const double y = 0.999, z = 0.5;
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], y, z);
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += x[q];
    if (s == 12345.0) g_sink = s;
}

// rule < 0: CTAs [0, nchain) run chains, the rest DMMA. rule >= 0: by %smid -- chain if smid % 4 == 0, DMMA if
// smid % 4 == rule (1: the TPC sibling SM 4t + 1, 2: an SM of the next TPC), the others idle
__global__ void __launch_bounds__(256, 1) k_probe(int mode, int nchain, int burst_n, long long* out, int* flag,
                                                  int rule, int* n_started) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(16) double s_ut[kUtSize];
    __shared__ double s_rcp[64];
    __shared__ int s_b;
    const int pld = 236;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    bool chain = blockIdx.x < nchain, dmma = !chain;
    int slot = blockIdx.x;
    if (rule >= 0) {
        chain = smid % 4 == 0;
        dmma = (int)(smid % 4) == rule;
        if (!chain && !dmma) return;
        if (chain) {
            __shared__ int s_slot;
            if (threadIdx.x == 0) s_slot = atomicAdd(n_started, 1);
            __syncthreads();
            slot = s_slot;
        }
    }
    if (dmma && mode == 7) {  // other SMs stream a large code footprint (panel_diag<32, false>, ~72 KB) until done
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int i = threadIdx.x; i < 32 * pld; i += 256) smem[i] = (i % pld == i / pld) ? 40.0 : 0.001;
        __syncthreads();
        do {
            if (threadIdx.x < 32) panel_diag<32, false>(smem, pld, s_ut, s_rcp, 31, 1e-10, &s_b);
            __syncthreads();
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        } while (*(volatile int*)flag < nchain && t1 - t0 < 3000000000ull);
        return;
    }
    if (dmma) {  // worker SM: DMMA until the chains are done
        double a = threadIdx.x, b = 1.0, c0 = 0, c1 = 0;
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {  // (bounded: 3 s)
            for (int r = 0; r < 1000; ++r) dmma_m8n8k4(c0, c1, a, b, c0, c1);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        } while (*(volatile int*)flag < nchain && t1 - t0 < 3000000000ull);
        if (c0 == 12345.0) g_sink = c1;
        return;
    }
    if (threadIdx.x == 0) s_b = 0;
    for (int call = 0; call < kCalls; ++call) {
        for (int i = threadIdx.x; i < 32 * pld; i += 256)
            smem[i] = (i % pld == i / pld) ? 40.0 + call : 0.01 * ((i * 7 + call) % 13 - 6);
        __syncthreads();
        if (mode == 2 && threadIdx.x >= 32) burst(burst_n);
        if (mode == 2) __syncthreads();
        if (mode == 3) {  // ~72 KB of other code through the instruction caches first (panel_diag<32, false>)
            if (threadIdx.x >= 32 && threadIdx.x < 64)
                panel_diag<32, false>(smem + 32 * pld, pld, s_ut, s_rcp, 31, 1e-10, &s_b);
            __syncthreads();
            for (int i = threadIdx.x; i < 32 * pld; i += 256)
                smem[i] = (i % pld == i / pld) ? 40.0 + call : 0.01 * ((i * 7 + call) % 13 - 6);
            __syncthreads();
        }
        if (threadIdx.x < 32) {
            const long long t0 = clock64();
            panel_diag<32, true>(smem, pld, s_ut, s_rcp, 32, 1e-10, &s_b);
            __syncwarp();
            if (threadIdx.x == 0) out[(size_t)slot * kCalls + call] = clock64() - t0;
        } else if (mode == 1 || (mode == 4 && (threadIdx.x >> 5) % 4 != 0)) {
            burst(burst_n);  // mode 4: not on warp 0's SM sub-partition (warps 4, 8, ...)
        } else if (mode == 5 || (mode == 6 && (threadIdx.x >> 5) % 4 != 0)) {
            double a = threadIdx.x, b = 1.0, c0 = 0, c1 = 0;  // DMMA (mode 6: off warp 0's sub-partition)
            for (int r = 0; r < burst_n; ++r) dmma_m8n8k4(c0, c1, a, b, c0, c1);
            if (c0 == 12345.0) g_sink = c1;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicAdd(flag, 1);
}

static void run(const char* name, int mode, int nchain, int grid, int burst_n, int rule = -1) {
    const size_t smem = 120 * 1024;  // one CTA per SM
    long long* d;
    int* flag;
    cudaMalloc(&d, sizeof(long long) * grid * kCalls);
    cudaMalloc(&flag, 2 * sizeof(int));
    cudaMemset(flag, 0, 2 * sizeof(int));
    k_probe<<<grid, 256, smem>>>(mode, nchain, burst_n, d, flag, rule, flag + 1);
    cudaDeviceSynchronize();
    std::vector<long long> h((size_t)nchain * kCalls);
    cudaMemcpy(h.data(), d, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost);
    std::vector<long long> v;
    for (int b = 0; b < nchain; ++b)
        for (int c = 10; c < kCalls; ++c) v.push_back(h[(size_t)b * kCalls + c]);
    std::sort(v.begin(), v.end());
    const long long med = v[v.size() / 2];
    size_t slow = 0;
    for (long long x : v) slow += x > 2 * med;
    printf("%-44s p10 %6lld  p50 %6lld  p90 %6lld  p99 %6lld  >2x median %.1f%%  (%s)\n", name, v[v.size() / 10], med,
           v[v.size() * 9 / 10], v[v.size() * 99 / 100], 100.0 * slow / v.size(), cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(flag);
}

int main() {
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int bn = 1500;  // ~the chain's update burst
    run("1 CTA, alone", 0, 1, 1, bn);
    run("1 CTA, beside DFMA burst", 1, 1, 1, bn);
    run("1 CTA, after DFMA burst", 2, 1, 1, bn);
    run("1 CTA, after 72 KB of other code", 3, 1, 1, bn);
    run("1 CTA, beside DFMA burst, warp 4 idle", 4, 1, 1, bn);
    run("1 CTA, beside DMMA burst", 5, 1, 1, bn);
    run("1 CTA, beside DMMA burst, warp 4 idle", 6, 1, 1, bn);
    run("50 CTAs alone, 98 SMs big code", 7, 50, nsm, bn);
    run("50 CTAs, beside DFMA burst", 1, 50, 50, bn);
    run("50 CTAs, beside burst, 98 SMs DMMA", 1, 50, nsm, bn);
    run("50 CTAs, alone, 98 SMs DMMA", 0, 50, nsm, bn);
    run("50 CTAs, after burst, 98 SMs DMMA", 2, 50, nsm, bn);
    run("148 CTAs, beside DFMA burst", 1, nsm, nsm, bn);
    // chains on smid % 4 == 0 (37 of them): DMMA on the TPC sibling vs on another TPC
    run("smid%4==0 chains, DMMA on smid%4==1", 0, 37, nsm, bn, 1);
    run("smid%4==0 chains, DMMA on smid%4==2", 0, 37, nsm, bn, 2);
    run("smid%4==0 chains, DMMA on smid%4==3", 0, 37, nsm, bn, 3);
    run("smid%4==0 chains+burst, DMMA on smid%4==1", 1, 37, nsm, bn, 1);
    return 0;
}
