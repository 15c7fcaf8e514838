// Banded SpMV variants at config 2 (N = 200000, K = 200), same per-row summation order (ascending columns, one
// FMA chain from zero): V0 = k_band_spmv (spmv.cu), V1 = 16 loads batched ahead of their FMAs, V2 = two row
// groups per warp (rows r0 + lane and r0 + 32 + lane: two independent chains). Prints us / GB/s and bitwise checks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe/spmv_probe.cu -o tools/probe/spmv_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__global__ void __launch_bounds__(256) v0(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
#pragma unroll 8
        for (int j = clo; j <= chi; ++j, col += ld) {
            const double xv = __ldg(x + j);
            if (i < n && i - j <= k && j - i <= k) acc = fma(*col, xv, acc);
        }
        if (i < n) y[i] = acc;
    }
}

template <int NB>
__global__ void __launch_bounds__(256) v1(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        for (int j0 = clo; j0 <= chi; j0 += NB) {
            double v[NB], xv[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int j = j0 + u;
                const bool ok = j <= chi && i < n && i - j <= k && j - i <= k;
                v[u] = ok ? __ldcs(col + (long long)u * ld) : 0.0;
                xv[u] = j <= chi ? __ldg(x + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int j = j0 + u;
                if (j <= chi && i < n && i - j <= k && j - i <= k) acc = fma(v[u], xv[u], acc);
            }
            col += NB * ld;
        }
        if (i < n) y[i] = acc;
    }
}

__global__ void __launch_bounds__(256) v2(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 64; r0 < n; r0 += nw * 64) {
        const int i0 = r0 + lane, i1 = r0 + 32 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 63 + k, n - 1);
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = a + (long long)clo * ld + i0 + k;
#pragma unroll 8
        for (int j = clo; j <= chi; ++j, col += ld) {
            const double xv = __ldg(x + j);
            if (i0 < n && i0 - j <= k && j - i0 <= k) acc0 = fma(col[0], xv, acc0);
            if (i1 < n && i1 - j <= k && j - i1 <= k) acc1 = fma(col[32], xv, acc1);
        }
        if (i0 < n) y[i0] = acc0;
        if (i1 < n) y[i1] = acc1;
    }
}

// V3: the CTA's 8 warps (rows rb .. rb + 255) walk one common column range in lock-step (a barrier every SYNC
// columns), each warp active on its own window, so at any time the CTA reads ~2 KB contiguous of one column
// block instead of 8 scattered 256-byte pieces (same per-row order)
template <int SYNC>
__global__ void __launch_bounds__(256) v3(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long ld = 2LL * k;
    for (int rb = blockIdx.x * 256; rb < n; rb += gridDim.x * 256) {
        const int r0 = rb + 32 * warp, i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        const int blo = max(rb - k, 0), bhi = min(rb + 255 + k, n - 1);
        double acc = 0.0;
        for (int j0 = blo; j0 <= bhi; j0 += SYNC) {
            const int ja = max(j0, clo), jb = min(j0 + SYNC - 1, chi);
            const double* col = a + (long long)ja * ld + i + k;
#pragma unroll 8
            for (int j = ja; j <= jb; ++j, col += ld) {
                const double xv = __ldg(x + j);
                if (i < n && i - j <= k && j - i <= k) acc = fma(*col, xv, acc);
            }
            __syncthreads();
        }
        if (i < n) y[i] = acc;
    }
}

int main() {
    const int n = 200000, k = 200;
    const size_t w = 2 * k + 1, total = (size_t)n * w;
    std::vector<double> ha(total, 0.0), hx(n);
    srand(3);
    for (size_t j = 0; j < (size_t)n; ++j)
        for (int s = 0; s < (int)w; ++s) {
            const long long i = (long long)j - k + s;
            if (i >= 0 && i < n) ha[j * w + s] = rand() / (double)RAND_MAX - 0.5;
        }
    for (int i = 0; i < n; ++i) hx[i] = rand() / (double)RAND_MAX - 0.5;
    double *a, *x, *y0, *y1;
    cudaMalloc(&a, total * 8);
    cudaMalloc(&x, n * 8);
    cudaMalloc(&y0, n * 8);
    cudaMalloc(&y1, n * 8);
    cudaMemcpy(a, ha.data(), total * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice);
    const double bytes = 8.0 * total + 16.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 5; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 50; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 50;
        std::vector<double> h0(n), h1(n);
        cudaMemcpy(h0.data(), y0, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(h1.data(), y1, n * 8, cudaMemcpyDeviceToHost);
        printf("%-28s %7.1f us  %6.0f GB/s  bitwise vs v0: %s\n", name, us, bytes / (us * 1e-6) / 1e9,
               memcmp(h0.data(), h1.data(), n * 8) == 0 ? "yes" : "NO");
    };
    const int warps = (n + 31) / 32;
    auto g = [](int warps_, int per) { return std::min((warps_ + per - 1) / per, 148 * 64); };
    v0<<<g(warps, 8), 256>>>(a, n, k, x, y0);
    timeit("v0 (current)", [&] { v0<<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v1 batch 16", [&] { v1<16><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v1 batch 32", [&] { v1<32><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v2 two row groups", [&] { v2<<<g((n + 63) / 64, 8), 256>>>(a, n, k, x, y1); });
    timeit("v0 128-thread blocks", [&] { v0<<<g(warps, 4), 128>>>(a, n, k, x, y1); });
    timeit("v3 lock-step, sync 16", [&] { v3<16><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v3 lock-step, sync 32", [&] { v3<32><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v3 lock-step, sync 64", [&] { v3<64><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
