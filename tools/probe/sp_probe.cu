// Standalone timing of a one-warp 32x32 register-row LU (substitution-panel experiment).
#include <cstdio>
__device__ __forceinline__ double fast_rcp(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0); r = fma(r, e, r); e = fma(-p, r, 1.0); r = fma(r, e, r); e = fma(-p, r, 1.0);
    return fma(r, e, r);
}
template <int V>
__device__ __noinline__ void diag(double* __restrict__ P, int pld, double bv, double* __restrict__ s_rcp,
                                  double* __restrict__ s_u, int* boost_ctr) {
    constexpr int B = 32;
    const int i = threadIdx.x & 31;
    double a[B];
#pragma unroll
    for (int c = 0; c < B; ++c) a[c] = P[c * pld + i];
#pragma unroll
    for (int c = 0; c < B; ++c) {
        if (V == 0) {
            if (i == c) {
                double p = a[c];
                if (fabs(p) < bv) { p = p < 0.0 ? -bv : bv; a[c] = p; atomicAdd(boost_ctr, 1); }
                s_rcp[c] = fast_rcp(p);
#pragma unroll
                for (int j = c; j < B; ++j) s_u[c * B + j] = a[j];
            }
            __syncwarp();
            if (i > c) {
                const double l = a[c] * s_rcp[c];
                a[c] = l;
#pragma unroll
                for (int j = c + 1; j < B; ++j) a[j] = fma(-l, s_u[c * B + j], a[j]);
            }
        } else {
            // pivot row by shuffles, no smem
            double p = __shfl_sync(0xffffffffu, a[c], c);
            if (fabs(p) < bv) p = p < 0.0 ? -bv : bv;
            const double rc = fast_rcp(p);
            const double l = a[c] * rc;
            if (i > c) a[c] = l;
            if (i == c) a[c] = p;
#pragma unroll
            for (int j = c + 1; j < B; ++j) {
                const double u = __shfl_sync(0xffffffffu, a[j], c);
                if (i > c) a[j] = fma(-l, u, a[j]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < B; ++c) P[c * pld + i] = a[c];
}
template <int V>
__global__ void kt(const double* g, long long* cyc, double* out) {
    __shared__ double P[32 * 36];
    __shared__ double s_rcp[32];
    __shared__ __align__(16) double s_u[32 * 32];
    __shared__ int boosts;
    for (int i = threadIdx.x; i < 32 * 36; i += 32) P[i] = g[i];
    boosts = 0;
    __syncwarp();
    long long t0 = clock64();
    diag<V>(P, 36, 1e-10, s_rcp, s_u, &boosts);
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    for (int i = threadIdx.x; i < 32 * 36; i += 32) out[i] = P[i];
}
int main() {
    const int n = 32 * 36;
    double h[n];
    for (int i = 0; i < n; ++i) h[i] = 1e-3 * ((i * 37) % 101) - 0.05;
    for (int c = 0; c < 32; ++c) h[c * 36 + c] = 10.0;
    double *g, *o; long long* cyc;
    cudaMalloc(&g, n * 8); cudaMalloc(&o, n * 8); cudaMallocManaged(&cyc, 16);
    cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
        kt<0><<<1, 32>>>(g, cyc, o); cudaDeviceSynchronize(); long long a = cyc[0];
        kt<1><<<1, 32>>>(g, cyc, o); cudaDeviceSynchronize(); long long b = cyc[0];
        printf("diag smem-publish %lld cycles, shuffle %lld cycles  %s\n", a, b, cudaGetErrorString(cudaGetLastError()));
    }
}
