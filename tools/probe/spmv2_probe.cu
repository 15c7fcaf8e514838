// Probe: dual banded SpMV (y0 = A x0, y1 = A x1) at config 2 (n 200000, k 200): the product kernel's
// load-then-use loop vs batches of B band loads issued ahead of their FMAs (same per-row FMA order, so the
// outputs must be bitwise equal). nvcc -O3 -gencode arch=compute_100a,code=sm_100a spmv2_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void __launch_bounds__(256) base2(const double* __restrict__ a, int n, int k, const double* __restrict__ x0,
                                             double* __restrict__ y0, const double* __restrict__ x1, double* __restrict__ y1) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
#pragma unroll 8
        for (int j = clo; j <= chi; ++j, col += ld) {
            const double xv0 = __ldg(x0 + j), xv1 = __ldg(x1 + j);
            if (i < n && i - j <= k && j - i <= k) {
                const double av = *col;
                acc0 = fma(av, xv0, acc0);
                acc1 = fma(av, xv1, acc1);
            }
        }
        if (i < n) { y0[i] = acc0; y1[i] = acc1; }
    }
}

template <int B>
__global__ void __launch_bounds__(256) batch2(const double* __restrict__ a, int n, int k, const double* __restrict__ x0,
                                              double* __restrict__ y0, const double* __restrict__ x1, double* __restrict__ y1) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        int j = clo;
        for (; j + B - 1 <= chi; j += B, col += B * ld) {
            double av[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int jj = j + u;
                av[u] = (i < n && i - jj <= k && jj - i <= k) ? __ldg(col + u * ld) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int jj = j + u;
                if (i < n && i - jj <= k && jj - i <= k) {
                    acc0 = fma(av[u], __ldg(x0 + jj), acc0);
                    acc1 = fma(av[u], __ldg(x1 + jj), acc1);
                }
            }
        }
        for (; j <= chi; ++j, col += ld)
            if (i < n && i - j <= k && j - i <= k) {
                const double av = __ldg(col);
                acc0 = fma(av, __ldg(x0 + j), acc0);
                acc1 = fma(av, __ldg(x1 + j), acc1);
            }
        if (i < n) { y0[i] = acc0; y1[i] = acc1; }
    }
}

template <int B>
__global__ void __launch_bounds__(256) batch1(const double* __restrict__ a, int n, int k, const double* __restrict__ x0,
                                              double* __restrict__ y0) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc0 = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        int j = clo;
        for (; j + B - 1 <= chi; j += B, col += B * ld) {
            double av[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int jj = j + u;
                av[u] = (i < n && i - jj <= k && jj - i <= k) ? __ldg(col + u * ld) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int jj = j + u;
                if (i < n && i - jj <= k && jj - i <= k) acc0 = fma(av[u], __ldg(x0 + jj), acc0);
            }
        }
        for (; j <= chi; ++j, col += ld)
            if (i < n && i - j <= k && j - i <= k) acc0 = fma(__ldg(col), __ldg(x0 + j), acc0);
        if (i < n) y0[i] = acc0;
    }
}

__global__ void base1(const double* __restrict__ a, int n, int k, const double* __restrict__ x, double* __restrict__ y) {
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

int main() {
    const int n = 200000, k = 200;
    const size_t ne = (size_t)n * (2 * k + 1);
    std::vector<double> h(ne), hx(n), hx1(n);
    unsigned s = 1;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (double)(s >> 8) / (1 << 24) - 0.5; };
    for (auto& v : h) v = rnd();
    for (auto& v : hx) v = rnd();
    for (auto& v : hx1) v = rnd();
    double *a, *x0, *x1, *y0, *y1, *z0, *z1;
    CK(cudaMalloc(&a, ne * 8));
    CK(cudaMalloc(&x0, n * 8)); CK(cudaMalloc(&x1, n * 8));
    CK(cudaMalloc(&y0, n * 8)); CK(cudaMalloc(&y1, n * 8)); CK(cudaMalloc(&z0, n * 8)); CK(cudaMalloc(&z1, n * 8));
    CK(cudaMemcpy(a, h.data(), ne * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x0, hx.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x1, hx1.data(), n * 8, cudaMemcpyHostToDevice));
    const int grid = (n / 32 + 7) / 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<double> r0(n), r1(n), q0(n), q1(n);
    auto timeit = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-22s %8.1f us\n", name, ms * 1e3 / 20);
    };
    timeit("base1", [&] { base1<<<grid, 256>>>(a, n, k, x0, y0); });
    CK(cudaMemcpy(r0.data(), y0, n * 8, cudaMemcpyDeviceToHost));
    for (int B : {4, 8, 16}) {
        char nm[32]; snprintf(nm, 32, "batch1<%d>", B);
        if (B == 4) timeit(nm, [&] { batch1<4><<<grid, 256>>>(a, n, k, x0, z0); });
        if (B == 8) timeit(nm, [&] { batch1<8><<<grid, 256>>>(a, n, k, x0, z0); });
        if (B == 16) timeit(nm, [&] { batch1<16><<<grid, 256>>>(a, n, k, x0, z0); });
        CK(cudaMemcpy(q0.data(), z0, n * 8, cudaMemcpyDeviceToHost));
        printf("   bitwise %s\n", memcmp(q0.data(), r0.data(), n * 8) == 0 ? "equal" : "DIFFERENT");
    }
    timeit("base2", [&] { base2<<<grid, 256>>>(a, n, k, x0, y0, x1, y1); });
    CK(cudaMemcpy(r0.data(), y0, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r1.data(), y1, n * 8, cudaMemcpyDeviceToHost));
    for (int B : {4, 8, 16}) {
        char nm[32]; snprintf(nm, 32, "batch2<%d>", B);
        if (B == 4) timeit(nm, [&] { batch2<4><<<grid, 256>>>(a, n, k, x0, z0, x1, z1); });
        if (B == 8) timeit(nm, [&] { batch2<8><<<grid, 256>>>(a, n, k, x0, z0, x1, z1); });
        if (B == 16) timeit(nm, [&] { batch2<16><<<grid, 256>>>(a, n, k, x0, z0, x1, z1); });
        CK(cudaMemcpy(q0.data(), z0, n * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(q1.data(), z1, n * 8, cudaMemcpyDeviceToHost));
        printf("   bitwise %s\n",
               memcmp(q0.data(), r0.data(), n * 8) == 0 && memcmp(q1.data(), r1.data(), n * 8) == 0 ? "equal" : "DIFFERENT");
    }
    return 0;
}
