// Does __syncthreads wait for the CTA's outstanding global stores? 148 CTAs x 512 threads; per iteration every
// warp stores one 256-byte line (streaming through L2/HBM), then (a) nothing, (b) __syncthreads, (c) a
// __syncthreads after 2000 cycles of independent ALU work. Cycles per iteration.
#include <cstdio>
__global__ void k(double* out, int iters, int mode, long long* cyc) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    double* p = out + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double acc = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __stcg(p + (long long)i * stride, acc);
        if (mode == 2) {
            long long w = clock64();
            while (clock64() - w < 2000) acc = acc * 1.0000001 + 1e-9;
        }
        if (mode >= 1) __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
    if (acc == -1.0) out[0] = acc;
}
int main() {
    const int iters = 2000;
    double* out;
    cudaMalloc(&out, (size_t)148 * 512 * iters * 8);
    long long* cyc;
    cudaMallocManaged(&cyc, 148 * 8);
    const char* nm[] = {"store only", "store + __syncthreads", "store + 2000-cycle ALU + __syncthreads"};
    for (int mode = 0; mode < 3; ++mode) {
        k<<<148, 512>>>(out, 100, mode, cyc);
        cudaDeviceSynchronize();
        k<<<148, 512>>>(out, iters, mode, cyc);
        cudaDeviceSynchronize();
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
        printf("%-42s %lld cycles/iter  %s\n", nm[mode], mx, cudaGetErrorString(cudaGetLastError()));
    }
}
