// Dependent-chain latencies on B200: DFMA, DMUL, MUFU.RCP64H (rcp.approx.ftz.f64), SHFL (64-bit), LDS.64.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed, int n) {
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = seed + threadIdx.x;
    __syncthreads();
    double a = seed, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = a * b;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r; }
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
    long long t4 = clock64();
    int idx = threadIdx.x & 63;
    for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v) & 63; a += v; }
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) a = a / (b + a * 1e-300);
    long long t6 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMallocManaged(&c, 8 * 8);
    const int n = 1024;
    k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
    const char* nm[] = {"DFMA", "DMUL", "MUFU.RCP64H", "SHFL f64", "LDS.64 (+DADD)", "IEEE div"};
    for (int i = 0; i < 6; ++i) printf("%-16s %.1f cycles/op\n", nm[i], (double)c[i] / n);
}
