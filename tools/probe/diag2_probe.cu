// panel_diag (lu.cu) vs a shuffle-broadcast form (panel_diag_shfl): cycles alone and bitwise equality of every
// output (the factored block, packed U11 rows, pivots / reciprocals, boost count) on random blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      -I paper_1509_07919_b200/csrc tools/probe/diag2_probe.cu -o tools/probe/diag2_probe
#include "../../paper_1509_07919_b200/csrc/lu.cu"
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace sapgpu {
long long g_launch_count = 0;
}
using namespace sapgpu;

// candidate: lane r owns row r; pivot row entries by shuffle from lane c; the (uniform) boosted pivot and its
// reciprocal computed by every lane; lane c publishes its final row to the packed U11 and the pivots
template <int B, bool FULL>
__device__ __noinline__ void panel_diag_shfl(double* __restrict__ P, int pld, double* __restrict__ Ut,
                                             double* __restrict__ s_piv, int nb_rt, double bv, int* boost_ctr) {
    const int nb = FULL ? B : nb_rt;
    const int r = threadIdx.x & 31;
    const bool own = r < nb;
    double a[B];
#pragma unroll
    for (int j = 0; j < B; ++j) a[j] = (own && j < nb) ? P[j * pld + r] : 0.0;
    int boosts = 0;
#pragma unroll
    for (int c = 0; c < B; ++c) {
        if (FULL || c < nb) {
            double p = __shfl_sync(0xffffffffu, a[c], c);
            const bool boost = fabs(p) < bv;
            p = boost ? (p < 0.0 ? -bv : bv) : p;
            if (boost && r == c) ++boosts;
            const double rc = rcp2(p);
            if (r == c) a[c] = p;
            const bool below = own && r > c;
            const double lq = div_rcp(a[c], p, rc);
            const double l = below ? lq : 0.0;
            if (below) a[c] = lq;
#pragma unroll
            for (int j = c + 1; j < B; ++j) {
                const double u = __shfl_sync(0xffffffffu, a[j], c);
                a[j] = fma(-l, u, a[j]);
            }
            if (r == c) {
                s_piv[c] = p;
                s_piv[B + c] = rc;
#pragma unroll
                for (int j = ut_lo(c); j < B; j += 2)
                    *reinterpret_cast<double2*>(Ut + ut_off(c) + j - ut_lo(c)) = make_double2(a[j], a[j + 1]);
            }
            if (own) P[c * pld + r] = a[c];
        }
    }
    if (boosts) atomicAdd(boost_ctr, boosts);
}

__device__ long long g_cyc[2];

template <int MODE>
__global__ void __launch_bounds__(32, 1) k_probe(double* blocks, double* out, int nblk, int reps, double bv, int pld) {
    __shared__ __align__(16) double sm[32 * 40];
    __shared__ __align__(16) double s_ut[kUtSize];
    __shared__ double s_piv[64];
    __shared__ int s_b;
    const int r = threadIdx.x;
    long long tot = 0;
    for (int b = 0; b < nblk; ++b) {
        for (int rep = 0; rep < reps; ++rep) {
            for (int i = r; i < 32 * pld; i += 32) sm[i] = blocks[(size_t)b * 32 * 32 + (i / pld) * 32 + (i % pld) % 32];
            for (int i = r; i < kUtSize; i += 32) s_ut[i] = 0.0;
            if (r == 0) s_b = 0;
            __syncwarp();
            const long long t0 = clock64();
            if (MODE == 0)
                panel_diag<32, true>(sm, pld, s_ut, s_piv, 32, bv, &s_b);
            else
                panel_diag_shfl<32, true>(sm, pld, s_ut, s_piv, 32, bv, &s_b);
            __syncwarp();
            tot += clock64() - t0;
        }
        double* o = out + (size_t)b * (32 * 32 + kUtSize + 64 + 1);
        for (int i = r; i < 32 * 32; i += 32) o[i] = sm[(i / 32) * pld + (i % 32)];
        for (int i = r; i < kUtSize; i += 32) o[1024 + i] = s_ut[i];
        for (int i = r; i < 64; i += 32) o[1024 + kUtSize + i] = s_piv[i];
        if (r == 0) o[1024 + kUtSize + 64] = s_b;
    }
    if (r == 0) g_cyc[MODE] = tot / (nblk * reps);
}

int main() {
    const int nblk = 64, reps = 20, pld = 36;
    const size_t bn = (size_t)nblk * 1024, on = (size_t)nblk * (1024 + kUtSize + 65);
    double* h = (double*)malloc(bn * 8);
    srand(7);
    for (int b = 0; b < nblk; ++b)
        for (int i = 0; i < 1024; ++i) {
            const int row = i % 32, col = i / 32;
            double v = (rand() / (double)RAND_MAX) * 2 - 1;
            if (row == col) v = (b % 8 == 3 && row == 5) ? 1e-14 : (b % 2 ? 40.0 : 3.0) * (v < 0 ? -1 : 1);
            h[(size_t)b * 1024 + col * 32 + row] = v;
        }
    double *d, *o0, *o1;
    cudaMalloc(&d, bn * 8);
    cudaMalloc(&o0, on * 8);
    cudaMalloc(&o1, on * 8);
    cudaMemcpy(d, h, bn * 8, cudaMemcpyHostToDevice);
    k_probe<0><<<1, 32>>>(d, o0, nblk, reps, 1e-10 * 50, pld);
    k_probe<1><<<1, 32>>>(d, o1, nblk, reps, 1e-10 * 50, pld);
    cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
    double* a = (double*)malloc(on * 8);
    double* bb = (double*)malloc(on * 8);
    cudaMemcpy(a, o0, on * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(bb, o1, on * 8, cudaMemcpyDeviceToHost);
    long long diff = 0;
    for (size_t i = 0; i < on; ++i) diff += memcmp(&a[i], &bb[i], 8) != 0;
    printf("panel_diag %lld cycles, panel_diag_shfl %lld cycles; differing output words %lld of %zu (%s)\n", c[0], c[1],
           diff, on, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
