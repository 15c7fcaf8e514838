// Trailing-update tile-shape probe: 100 CTAs x 512 threads, each updates its own 200 x 200 window of a
// tall-thin band (C from/to global through L2, 16-byte accesses) with operands in shared memory
// (panel column-major ld 236, U12 row-major ld 204), DMMA m8n8k4. Warp tile TM x 32 (TM = 16, 24, 32).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int TM>
__global__ void __launch_bounds__(512, 1) k(double* band, int K, int steps, long long* cyc) {
    constexpr int pld = 236, uld = 204, R = 200, TA = TM / 8;
    extern __shared__ __align__(16) double sm[];
    double* P = sm;
    double* U = sm + 32 * pld;
    for (int i = threadIdx.x; i < 32 * pld + 32 * uld; i += 512) sm[i] = 1e-3 * ((i * 37) % 101);
    __syncthreads();
    const long long ld = 2LL * K;
    double* base = band + (long long)blockIdx.x * 4000 * (2 * K + 1) + K + 64 * (ld + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int trows = (R + TM - 1) / TM, tcols = (R + 31) / 32, ntiles = trows * tcols;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        for (int t = warp; t < ntiles; t += 16) {
            const int row0 = (t / tcols) * TM, col0 = (t % tcols) * 32;
            double acc[TA][4][2];
            const int ib = row0 + 2 * lc, cb = col0 + lr;
            double* p00 = base + (long long)cb * ld + ib;
#pragma unroll
            for (int a = 0; a < TA; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool ok = row0 + 8 * a < R && col0 + 8 * q < R;
                    double2 v = ok ? __ldcg(reinterpret_cast<const double2*>(p00 + 8 * a + 8 * q * ld)) : make_double2(0, 0);
                    acc[a][q][0] = v.x;
                    acc[a][q][1] = v.y;
                }
            const double* pk = P + 32 + row0 + lr;
            const double* uk = U + col0 + lr;
#pragma unroll 2
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = ks * 4 + lc;
                double b[TA], aq[4];
#pragma unroll
                for (int a = 0; a < TA; ++a) b[a] = -pk[kk * pld + 8 * a];
#pragma unroll
                for (int q = 0; q < 4; ++q) aq[q] = uk[kk * uld + 8 * q];
#pragma unroll
                for (int a = 0; a < TA; ++a)
#pragma unroll
                    for (int q = 0; q < 4; ++q) mma(acc[a][q][0], acc[a][q][1], aq[q], b[a]);
            }
#pragma unroll
            for (int a = 0; a < TA; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (row0 + 8 * a < R && col0 + 8 * q < R)
                        __stcg(reinterpret_cast<double2*>(p00 + 8 * a + 8 * q * ld), make_double2(acc[a][q][0], acc[a][q][1]));
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / steps;
}
template <int TM>
void run(double* band, long long* cyc) {
    const size_t bytes = sizeof(double) * (32 * 236 + 32 * 204 + 512);
    cudaFuncSetAttribute(k<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    k<TM><<<100, 512, bytes>>>(band, 200, 5, cyc);
    cudaDeviceSynchronize();
    k<TM><<<100, 512, bytes>>>(band, 200, 50, cyc);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < 100; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    printf("tile %2d x 32: %lld cycles/step (DMMA-peak bound ~20000)  %s\n", TM, mx, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double* band;
    long long* cyc;
    const size_t n = (size_t)100 * 4000 * 401;
    cudaMalloc(&band, n * 8);
    cudaMemset(band, 0, n * 8);
    cudaMallocManaged(&cyc, 100 * 8);
    run<16>(band, cyc);
    run<24>(band, cyc);
    run<32>(band, cyc);
}
