// Dependent-chain latency of DFMA / DADD / LDS+DFMA on one warp, and DFMA issue with 4 independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe/fp64_lat.cu -o tools/probe/fp64_lat
#include <cstdio>
__device__ long long g_r[8];
__device__ double g_sink;
__global__ void k(double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = 1.0 + i * 1e-9;
    __syncwarp();
    double x = threadIdx.x * 1e-3, y = x, z = x, w = x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) y = y + b;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) z = fma(sm[(i * 33 + threadIdx.x) & 1023], z, b);
    long long t3 = clock64();
    double u0 = x, u1 = y, u2 = z, u3 = w;
    for (int i = 0; i < n; ++i) {
        u0 = fma(u0, a, b); u1 = fma(u1, a, b); u2 = fma(u2, a, b); u3 = fma(u3, a, b);
    }
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        g_r[0] = (t1 - t0); g_r[1] = (t2 - t1); g_r[2] = (t3 - t2); g_r[3] = (t4 - t3);
    }
    g_sink = x + y + z + w + u0 + u1 + u2 + u3;
}
int main() {
    const int n = 4096;
    k<<<1, 32>>>(0.999999, 1e-7, n);
    cudaDeviceSynchronize();
    long long r[8];
    cudaMemcpyFromSymbol(r, g_r, sizeof(r));
    printf("cycles per op: DFMA chain %.1f, DADD chain %.1f, LDS+DFMA chain %.1f, 4 independent DFMA chains %.1f per round\n",
           r[0] / (double)n, r[1] / (double)n, r[2] / (double)n, r[3] / (double)n);
    return 0;
}
