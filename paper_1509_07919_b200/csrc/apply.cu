// Preconditioner application M^{-1} b (SaP-D and SaP-C).
//
// Reference: block_solve / band_lu_solve proj/include/sap/block_factors.hpp:74-90,
// :210-236 and apply_preconditioner proj/include/sap/spike.hpp:304-351.
//
// Block solve: one CTA per partition walks its rows in 32-row chunks. For a
// chunk, the 16 warps form the off-chunk part of every row's dot product
// (each warp a strided subset of the previous K columns, lane = row, so every
// load is a contiguous 256-byte run of the column-major band), the partials
// are summed in fixed order, and warp 0 finishes the 32x32 triangle with
// shuffles. The backward (U) sweep mirrors it from the bottom chunk up.
#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

constexpr int kSolveThreads = 512;
constexpr int kSolveWarps = kSolveThreads / 32;

template <class T>
__global__ void __launch_bounds__(kSolveThreads)
    k_block_solve(const T* __restrict__ lu, const int* __restrict__ offs, int k, T* __restrict__ x) {
    const int b = blockIdx.x;
    const int off = offs[b], m = offs[b + 1] - off;
    const T* f = lu + (long long)off * (2 * k + 1);
    const long long ld = 2LL * k;
    T* xb = x + off;
    __shared__ T part[kSolveWarps][33];
    __shared__ T tri[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nchunks = (m + 31) / 32;

    // forward: L unit lower, x_i -= sum_{j<i} L(i,j) x_j
    for (int ch = 0; ch < nchunks; ++ch) {
        const int i0 = ch * 32, rows = min(32, m - i0);
        const int i = i0 + lane;
        T s = T(0);
        const int jlo = max(i0 - k, 0);
#pragma unroll 4
        for (int j = jlo + warp; j < i0; j += kSolveWarps)
            if (lane < rows && i - j <= k) s = fma(f[(long long)j * ld + i + k], xb[j], s);
        part[warp][lane] = s;
        for (int jj = warp; jj < rows; jj += kSolveWarps)
            tri[lane][jj] = (lane > jj && lane < rows && lane - jj <= k) ? f[(long long)(i0 + jj) * ld + i + k] : T(0);
        __syncthreads();
        if (warp == 0) {
            T tot = T(0);
#pragma unroll
            for (int q = 0; q < kSolveWarps; ++q) tot += part[q][lane];
            T y = lane < rows ? xb[i] - tot : T(0);
            for (int jj = 0; jj < rows; ++jj) {
                const T xj = __shfl_sync(0xffffffffu, y, jj);
                if (lane > jj) y = fma(-tri[lane][jj], xj, y);
            }
            if (lane < rows) xb[i] = y;
        }
        __syncthreads();
    }
    // backward: U with diagonal, x_i = (x_i - sum_{j>i} U(i,j) x_j) / U(i,i)
    for (int ch = nchunks - 1; ch >= 0; --ch) {
        const int i0 = ch * 32, rows = min(32, m - i0);
        const int i = i0 + lane;
        T s = T(0);
        const int jhi = min(i0 + 31 + k, m - 1);
#pragma unroll 4
        for (int j = i0 + rows + warp; j <= jhi; j += kSolveWarps)
            if (lane < rows && j - i <= k) s = fma(f[(long long)j * ld + i + k], xb[j], s);
        part[warp][lane] = s;
        for (int jj = warp; jj < rows; jj += kSolveWarps)
            tri[lane][jj] = (lane <= jj && lane < rows && jj - lane <= k) ? f[(long long)(i0 + jj) * ld + i + k] : T(0);
        __syncthreads();
        if (warp == 0) {
            T tot = T(0);
#pragma unroll
            for (int q = 0; q < kSolveWarps; ++q) tot += part[q][lane];
            T y = lane < rows ? xb[i] - tot : T(0);
            for (int jj = rows - 1; jj >= 0; --jj) {
                if (lane == jj) y = y / tri[lane][lane];
                const T xj = __shfl_sync(0xffffffffu, y, jj);
                if (lane < jj) y = fma(-tri[lane][jj], xj, y);
            }
            if (lane < rows) xb[i] = y;
        }
        __syncthreads();
    }
}

template <class T>
void launch_block_solve(const T* lu, const int* d_offsets, int p, int k, T* x, cudaStream_t s) {
    k_block_solve<T><<<p, kSolveThreads, 0, s>>>(lu, d_offsets, k, x);
    SAP_LAUNCHED();
}
template void launch_block_solve<double>(const double*, const int*, int, int, double*, cudaStream_t);
template void launch_block_solve<float>(const float*, const int*, int, int, float*, cudaStream_t);

// ---------------------------------------------------------------------------
// SaP-C interface step, one CTA per interface t (spike.hpp:323-347):
//   rhs = g[e:e+w] - W^t g[e-w:e];  R xt = rhs;  xb = g[e-w:e] - V^b xt;
//   b2[e-w:e] -= B xt;  b2[e:e+w] -= C xb.
// Interfaces write disjoint rows of b2 (every block has >= 2K rows).
template <class T>
__device__ void gemv_sub_warps(const T* __restrict__ a, int w, const T* xv, T* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < w; i += nw) {
        T acc = T(0);
        for (int j = lane; j < w; j += 32) acc = fma(a[(long long)i * w + j], xv[j], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[i] -= acc;
    }
}

template <class T>
__global__ void __launch_bounds__(256)
    k_interfaces(const T* __restrict__ g, const int* __restrict__ offs, int k, const T* __restrict__ wt,
                 const T* __restrict__ vb, const T* __restrict__ rbar, const T* __restrict__ bblk,
                 const T* __restrict__ cblk, T* __restrict__ b2) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* gb = reinterpret_cast<T*>(smraw);
    T* rhs = gb + k;
    const int t = blockIdx.x, w = k;
    const int e = offs[t + 1];
    const long long ww = (long long)w * w;
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        gb[i] = g[e - w + i];
        rhs[i] = g[e + i];
    }
    __syncthreads();
    gemv_sub_warps(wt + t * ww, w, gb, rhs);
    __syncthreads();
    const T* R = rbar + t * ww;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        for (int i = 0; i < w; ++i) {  // unit lower
            T acc = T(0);
            for (int j = lane; j < i; j += 32) acc = fma(R[(long long)i * w + j], rhs[j], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) rhs[i] -= acc;
            __syncwarp();
        }
        for (int i = w - 1; i >= 0; --i) {  // upper with diagonal
            T acc = T(0);
            for (int j = i + 1 + lane; j < w; j += 32) acc = fma(R[(long long)i * w + j], rhs[j], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) rhs[i] = (rhs[i] - acc) / R[(long long)i * w + i];
            __syncwarp();
        }
    }
    __syncthreads();
    gemv_sub_warps(vb + t * ww, w, rhs, gb);  // gb becomes xb
    __syncthreads();
    gemv_sub_warps(bblk + t * ww, w, rhs, b2 + e - w);
    gemv_sub_warps(cblk + t * ww, w, gb, b2 + e);
}

template <class T>
void launch_interfaces(const T* g, const int* d_offsets, int p, int k, const T* wt, const T* vb, const T* rbar,
                       const T* bblk, const T* cblk, T* b2, cudaStream_t s) {
    if (p < 2 || k == 0) return;
    k_interfaces<T><<<p - 1, 256, 2 * k * sizeof(T), s>>>(g, d_offsets, k, wt, vb, rbar, bblk, cblk, b2);
    SAP_LAUNCHED();
}
template void launch_interfaces<double>(const double*, const int*, int, int, const double*, const double*,
                                        const double*, const double*, const double*, double*, cudaStream_t);
template void launch_interfaces<float>(const float*, const int*, int, int, const float*, const float*,
                                       const float*, const float*, const float*, float*, cudaStream_t);

// ---------------------------------------------------------------------------
// Diagonal preconditioner (build_precond_op's `diagonal` branch, pipeline.hpp:151-161).
__global__ void k_boosted_diag(const double* __restrict__ a, int n, int k, const double* __restrict__ scale,
                               double eps, double* __restrict__ diag) {
    const double sc = *scale;
    const double bv = eps * (sc > 0 ? sc : 1.0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double d = a[(long long)i * (2 * k + 1) + k];
        if (fabs(d) < bv) d = d < 0.0 ? -bv : bv;
        diag[i] = d;
    }
}

void launch_boosted_diag(const double* band, int n, int k, const double* scale, double boost_eps, double* diag,
                         cudaStream_t s) {
    k_boosted_diag<<<ceil_div(n, 256), 256, 0, s>>>(band, n, k, scale, boost_eps, diag);
    SAP_LAUNCHED();
}

__global__ void k_diag_apply(const double* __restrict__ in, const double* __restrict__ diag,
                             double* __restrict__ out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] / diag[i];
}

void launch_diag_apply(const double* in, const double* diag, double* out, int n, cudaStream_t s) {
    k_diag_apply<<<ceil_div(n, 256), 256, 0, s>>>(in, diag, out, n);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
