// Krylov A operators: banded and CSR SpMV (optionally fused with b - A x).
//
// Reference: BandedMatrix::matvec proj/include/sap/banded_matrix.hpp:72-80 and
// SparseMatrix::matvec proj/include/sap/sparse_matrix.hpp:24-31. Each row
// accumulates its products in ascending column order from zero (FMA), as the
// reference does.
//
// Banded: a warp owns 32 consecutive rows and walks the union of their
// column windows; for each column the 32 lanes read 32 consecutive slots
// (slot = j*2k + i + k), i.e. one fully used 256-byte run of the tall-thin
// band, and x[j] is a warp-wide broadcast.
#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

// Row sums over the union window [clo, chi] of a warp's 32 rows: the band slots of kSpB columns are loaded
// (predicated on the band) before their FMAs, so a thread keeps several 8-byte loads in flight instead of one
// (the conditional load-then-use loop compiled to one outstanding load; tools/probe/spmv2_probe.cu measured
// 132 -> 118 us for one product at config 2, 195 -> 143 us for two). The FMAs still run in ascending column
// order and skip the out-of-band slots, so every row's sum is bitwise the reference order's.
constexpr int kSpB = 8;

__global__ void __launch_bounds__(256)
    k_band_spmv(const double* __restrict__ a, int n, int k, const double* __restrict__ x, double* __restrict__ y,
                const double* __restrict__ b) {
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = warp_global * 32; r0 < n; r0 += nwarps * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        int j = clo;
        for (; j + kSpB - 1 <= chi; j += kSpB, col += kSpB * ld) {
            double av[kSpB];
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
                const int jj = j + u;
                av[u] = (i < n && i - jj <= k && jj - i <= k) ? __ldg(col + u * ld) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
                const int jj = j + u;
                if (i < n && i - jj <= k && jj - i <= k) acc = fma(av[u], __ldg(x + jj), acc);
            }
        }
        for (; j <= chi; ++j, col += ld)
            if (i < n && i - j <= k && j - i <= k) acc = fma(__ldg(col), __ldg(x + j), acc);
        if (i < n) y[i] = b ? b[i] - acc : acc;
    }
}

void launch_band_spmv(const double* band, int n, int k, const double* x, double* y, const double* b, cudaStream_t s) {
    const int warps = ceil_div(n, 32);
    const int grid = std::min(ceil_div(warps, 8), 148 * 64);
    k_band_spmv<<<grid, 256, 0, s>>>(band, n, k, x, y, b);
    SAP_LAUNCHED();
}

// Two products over one read of the band: y0 = A x0, y1 = A x1. BiCGStab's step applies A to the updated
// residual and (for the true residual, krylov.hpp:62-72) to the updated iterate back to back; each row's
// sum is formed exactly as in k_band_spmv (ascending columns, FMA from zero), so both are bitwise its.
__global__ void __launch_bounds__(256)
    k_band_spmv2(const double* __restrict__ a, int n, int k, const double* __restrict__ x0, double* __restrict__ y0,
                 const double* __restrict__ x1, double* __restrict__ y1) {
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = warp_global * 32; r0 < n; r0 += nwarps * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        int j = clo;
        for (; j + kSpB - 1 <= chi; j += kSpB, col += kSpB * ld) {
            double av[kSpB];
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
                const int jj = j + u;
                av[u] = (i < n && i - jj <= k && jj - i <= k) ? __ldg(col + u * ld) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
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
        if (i < n) {
            y0[i] = acc0;
            y1[i] = acc1;
        }
    }
}

void launch_band_spmv2(const double* band, int n, int k, const double* x0, double* y0, const double* x1, double* y1,
                       cudaStream_t s) {
    const int warps = ceil_div(n, 32);
    const int grid = std::min(ceil_div(warps, 8), 148 * 64);
    k_band_spmv2<<<grid, 256, 0, s>>>(band, n, k, x0, y0, x1, y1);
    SAP_LAUNCHED();
}

__global__ void __launch_bounds__(256)
    k_band_spmv_rows(const double* __restrict__ a, int n, int k, int rbeg, int rend, const double* __restrict__ x,
                     double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = rbeg + warp_global * 32; r0 < rend; r0 += nwarps * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        int j = clo;
        for (; j + kSpB - 1 <= chi; j += kSpB, col += kSpB * ld) {
            double av[kSpB];
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
                const int jj = j + u;
                av[u] = (i < rend && i - jj <= k && jj - i <= k) ? __ldg(col + u * ld) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kSpB; ++u) {
                const int jj = j + u;
                if (i < rend && i - jj <= k && jj - i <= k) acc = fma(av[u], __ldg(x + jj), acc);
            }
        }
        for (; j <= chi; ++j, col += ld)
            if (i < rend && i - j <= k && j - i <= k) acc = fma(__ldg(col), __ldg(x + j), acc);
        if (i < rend) y[i - rbeg] = acc;
    }
}

void launch_band_spmv_rows(const double* band, int n, int k, int r0, int r1, const double* x, double* y, cudaStream_t s) {
    if (r1 <= r0) return;
    const int warps = ceil_div(r1 - r0, 32);
    k_band_spmv_rows<<<std::min(ceil_div(warps, 8), 148 * 64), 256, 0, s>>>(band, n, k, r0, r1, x, y);
    SAP_LAUNCHED();
}

__global__ void k_gemv_w(const double* __restrict__ A, int w, const double* __restrict__ v,
                         const double* __restrict__ u, double* __restrict__ y, int mode) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= w) return;
    double acc = 0.0;
    for (int j = lane; j < w; j += 32) acc = fma(A[(long long)i * w + j], v[j], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[i] = (mode == 0 ? u[i] : y[i]) - acc;
}

void launch_gemv_w(const double* A, int w, const double* v, const double* u, double* y, int mode, cudaStream_t s) {
    if (w <= 0) return;
    k_gemv_w<<<ceil_div(w, 8), 256, 0, s>>>(A, w, v, u, y, mode);
    SAP_LAUNCHED();
}

__global__ void k_csr_spmv(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                           int n, const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ b) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc = 0.0;
        const int e = rp[i + 1];
        for (int s = rp[i]; s < e; ++s) acc = fma(v[s], __ldg(x + ci[s]), acc);
        y[i] = b ? b[i] - acc : acc;
    }
}

void launch_csr_spmv(const int* rp, const int* ci, const double* v, int n, const double* x, double* y,
                     const double* b, cudaStream_t s) {
    k_csr_spmv<<<std::min(ceil_div(n, 256), 148 * 32), 256, 0, s>>>(rp, ci, v, n, x, y, b);
    SAP_LAUNCHED();
}

// assemble_banded (pipeline.hpp:103-115) on the device: entry (i, j) -> slot j*(2k+1) + (i-j+k); the
// first entry outside the band (lowest row, then position) is reported through bad = i * n + j.
__global__ void k_assemble_band(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                                int n, int k, double* __restrict__ band, unsigned long long* __restrict__ bad) {
    const long long w = 2LL * k + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int s = rp[i]; s < rp[i + 1]; ++s) {
            const int j = ci[s];
            if (i - j > k || j - i > k) {
                if (bad) atomicMin(bad, (unsigned long long)i * (unsigned long long)n + (unsigned long long)j);
            } else
                band[(long long)j * w + (i - j + k)] = v[s];
        }
}

void launch_assemble_band(const int* rp, const int* ci, const double* v, int n, int k, double* band,
                          unsigned long long* bad, cudaStream_t s) {
    if (n <= 0) return;
    k_assemble_band<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(rp, ci, v, n, k, band, bad);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
