// Isolated timing of the LU panel factorization routine (one CTA, clock64), with variants.
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <cstdio>
#include <vector>
namespace sapgpu { long long g_launch_count = 0; }
using namespace sapgpu;

template <int B>
__device__ __noinline__ void panel_nodiv(const Lu& L, double* Pn, double* prow, int* bc, int np, int ph, int ptid) {
    const int pld = L.pld;
    double row[B];
#pragma unroll
    for (int c = 0; c < B; ++c) row[c] = ptid < ph ? Pn[c * pld + ptid] : 0.0;
#pragma unroll
    for (int C = 0; C < B; ++C) {
        named_sync(kBarPg, kPgThreads);
        const double* pr = prow + (C & 1) * (B + 1);
        if (ptid > C && ptid < ph) {
            const double l = row[C] * pr[C];
            row[C] = l;
#pragma unroll
            for (int cc = C + 1; cc < B; ++cc) row[cc] = fma(-l, pr[cc], row[cc]);
            if (ptid == C + 1) {
                double* q = prow + ((C + 1) & 1) * (B + 1);
                q[C + 1] = row[C + 1] * 0.999;
#pragma unroll
                for (int cc = C + 2; cc < B; ++cc) q[cc] = row[cc];
            }
        }
    }
    if (ptid < ph)
#pragma unroll
        for (int c = 0; c < B; ++c) Pn[c * pld + ptid] = row[c];
}

template <int VARIANT>
__global__ void __launch_bounds__(512, 1) k_probe(double* gpanel, int K, int np, int ph, int pld, long long* out) {
    extern __shared__ double sm[];
    __shared__ __align__(16) double prow[2 * 34];
    __shared__ int boosts;
    const int tid = threadIdx.x;
    for (int i = tid; i < 32 * pld; i += blockDim.x) sm[i] = gpanel[i];
    if (tid == 0) boosts = 0;
    __syncthreads();
    Lu L{nullptr, 1, 2LL * K, 4000, K, 32, pld, 0, 1e-10};
    long long t0 = clock64();
    if (tid < kPgThreads) {
        if (VARIANT == 0) {
            pg_factor_panel<32>(L, sm, prow, &boosts, np, ph, tid);
        } else if (VARIANT == 3) {  // register panel, reciprocal replaced by a multiply (no DDIV)
            panel_nodiv<32>(L, sm, prow, &boosts, np, ph, tid);
        } else if (VARIANT == 1) {  // barriers only
            for (int c = 0; c < np; ++c) named_sync(kBarPg, kPgThreads);
        } else if (VARIANT == 2) {  // barriers + row update, no publish
            double* my = sm + tid;
            for (int c = 0; c < np; ++c) {
                named_sync(kBarPg, kPgThreads);
                if (tid > c && tid < ph) {
                    const double l = my[c * pld] * 0.5;
                    my[c * pld] = l;
                    for (int cc = c + 1; cc < np; ++cc) my[cc * pld] = fma(-l, prow[cc & 31], my[cc * pld]);
                }
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) out[VARIANT] = t1 - t0;
}

int main() {
    const int K = 200, np = 32, ph = 232, pld = 244;
    std::vector<double> h(32 * pld);
    for (int c = 0; c < 32; ++c)
        for (int r = 0; r < pld; ++r) h[c * pld + r] = (r == c) ? 50.0 : (r < ph ? 0.01 * ((r * 7 + c * 3) % 13 - 6) : 0.0);
    double* d; cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    long long* o; cudaMalloc(&o, 8 * 8); cudaMemset(o, 0, 64);
    size_t sm = 32 * pld * 8;
    cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int rep = 0; rep < 2; ++rep) {
        k_probe<0><<<1, 512, sm>>>(d, K, np, ph, pld, o);
        k_probe<1><<<1, 512, sm>>>(d, K, np, ph, pld, o);
        k_probe<2><<<1, 512, sm>>>(d, K, np, ph, pld, o);
        k_probe<3><<<1, 512, sm>>>(d, K, np, ph, pld, o);
    }
    cudaDeviceSynchronize();
    long long ho[8]; cudaMemcpy(ho, o, 64, cudaMemcpyDeviceToHost);
    printf("no-div register panel: %lld (%.0f/col)\n", ho[3], ho[3] / 32.0);
    printf("full panel: %lld cycles (%.0f/col)\nbarriers only: %lld (%.0f/col)\nbarrier+update: %lld (%.0f/col)\nerr %s\n",
           ho[0], ho[0] / 32.0, ho[1], ho[1] / 32.0, ho[2], ho[2] / 32.0, cudaGetErrorString(cudaGetLastError()));
}
