// The FP32 SaP preconditioner of KrylovOptions::mixed_precision: build_precond_op<float>
// (proj/include/sap/pipeline.hpp:140-202) factors banded_cast<float>(A) (banded_matrix.hpp:129-136) in
// single precision -- factor_blocks<float> (block_factors.hpp:138-206: block norms accumulated in double
// over the float entries, boost value float(boost_eps * norm)), compute_spike_tips<float>
// (spike.hpp:178-254), finish_reduced_blocks<float> (spike.hpp:143-170: R = I - W V in float,
// dense_lu_nopivot_boosted<float> with its norm in double) -- and applies it in float between casts.
//
// These kernels are that factorization on the device. Every element receives its updates in the
// reference's order (pivot by pivot, j ascending); the GPU contracts a - l * u into one FMA where the
// reference rounds the product first, so results agree to FP32 rounding, not bitwise.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

namespace {

// Block band copies cast to float (banded_cast then factor_blocks' per-block copy; k_copy_blocks at
// T = float): slot o of block b is local column o / (2k+1), local row c - k + o % (2k+1); zero outside.
__global__ void k_copy_blocks_f32(const double* __restrict__ a, int k, const int* __restrict__ offs,
                                  long long pstride, int pad, long long total, float* __restrict__ lu,
                                  float* __restrict__ ul) {
    const long long w = 2LL * k + 1;
    for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < total;
         d += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(d / pstride);
        const long long o = d - (long long)b * pstride - pad;
        const int off = offs[b], m = offs[b + 1] - off;
        float v = 0.0f;
        if (o >= 0 && o < (long long)m * w) {
            const long long c = o / w, slot = o - c * w, r = c - k + slot;
            if (r >= 0 && r < m) v = (float)a[(off + c) * w + slot];
        }
        lu[d] = v;
        if (ul) ul[d] = v;
    }
}

constexpr int kF32Threads = 256;
constexpr int kF32B = 32;

// band_lu_inplace<float> / band_ul_inplace<float> (block_factors.hpp:22-71) of one job per CTA on a strided
// view (UL = LU of the flipped system, as in the FP64 kernels), blocked by 32 columns:
//   panel: unblocked column loop (boost, l = a / p, rank-1 update of the panel columns);
//   U12 <- L11^{-1} A12, thread per column, j ascending; A22 -= L21 U12, 4 x 4 register tiles, k ascending.
// A zero u_jc is skipped like the reference (its `if (ujc == 0) continue`).
__global__ void __launch_bounds__(kF32Threads)
    k_band_lu_f32(const FactorJobF* __restrict__ jobs, double eps, int pld, int uld) {
    extern __shared__ __align__(16) float fsm[];
    float* P = fsm;              // panel, column-major P[c * pld + r]
    float* U = fsm + kF32B * pld;  // U12, row-major U[r * uld + c]
    __shared__ int s_boosts;
    const FactorJobF J = jobs[blockIdx.x];
    const int m = J.m, K = J.k, tid = threadIdx.x;
    const long long rs = J.rs, cs = J.cs;
    float* const base = J.base;
    const double scale = *J.scale;
    const float bv = (float)(eps * (scale > 0 ? scale : 1.0));
    if (tid == 0) s_boosts = 0;
    for (int jb = 0; jb < m; jb += kF32B) {
        const int nb = min(kF32B, m - jb), ph = min(nb + K, m - jb), R = ph - nb;
        __syncthreads();
        for (int idx = tid; idx < kF32B * ph; idx += kF32Threads) {
            const int c = idx / ph, r = idx - c * ph;
            P[c * pld + r] = (c < nb && r - c <= K && c - r <= K) ? base[(jb + r) * rs + (jb + c) * cs] : 0.0f;
        }
        for (int idx = tid; idx < nb * R; idx += kF32Threads) {
            const int r = idx / R, c = idx - r * R;
            U[r * uld + c] = (nb + c - r <= K) ? base[(jb + r) * rs + (jb + nb + c) * cs] : 0.0f;
        }
        __syncthreads();
        for (int c = 0; c < nb; ++c) {
            if (tid == 0) {
                float p = P[c * pld + c];
                if (fabsf(p) < bv) {
                    P[c * pld + c] = p < 0.0f ? -bv : bv;
                    ++s_boosts;
                }
            }
            __syncthreads();
            const float p = P[c * pld + c];
            const int hi = min(c + K, ph - 1);
            for (int r = c + 1 + tid; r <= hi; r += kF32Threads) P[c * pld + r] = P[c * pld + r] / p;
            __syncthreads();
            const int rows = hi - c, cols = nb - 1 - c;
            for (int idx = tid; idx < rows * cols; idx += kF32Threads) {
                const int q = idx / rows, cc = c + 1 + q, r = c + 1 + (idx - q * rows);
                const float u = P[cc * pld + c];
                if (u != 0.0f) P[cc * pld + r] = fmaf(-P[c * pld + r], u, P[cc * pld + r]);
            }
            __syncthreads();
        }
        for (int c = tid; c < R; c += kF32Threads) {
            for (int r = 1; r < nb; ++r) {
                float acc = U[r * uld + c];
                for (int j = 0; j < r; ++j) {
                    const float u = U[j * uld + c];
                    if (u != 0.0f) acc = fmaf(-P[j * pld + r], u, acc);
                }
                U[r * uld + c] = acc;
            }
        }
        __syncthreads();
        for (int idx = tid; idx < kF32B * ph; idx += kF32Threads) {
            const int c = idx / ph, r = idx - c * ph;
            if (c < nb && r - c <= K && c - r <= K) base[(jb + r) * rs + (jb + c) * cs] = P[c * pld + r];
        }
        for (int idx = tid; idx < nb * R; idx += kF32Threads) {
            const int r = idx / R, c = idx - r * R;
            if (nb + c - r <= K) base[(jb + r) * rs + (jb + nb + c) * cs] = U[r * uld + c];
        }
        // A22 (R x R at (jb + nb, jb + nb), all inside the band) -= L21 U12
        const int T4 = (R + 3) >> 2;
        float* const a22 = base + (jb + nb) * rs + (jb + nb) * cs;
        for (int t = tid; t < T4 * T4; t += kF32Threads) {
            const int i0 = 4 * (t % T4), c0 = 4 * (t / T4);
            float acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    acc[a][b] = (i0 + a < R && c0 + b < R) ? a22[(i0 + a) * rs + (c0 + b) * cs] : 0.0f;
            for (int j = 0; j < nb; ++j) {
                float l[4], u[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) l[a] = P[j * pld + nb + i0 + a];
#pragma unroll
                for (int b = 0; b < 4; ++b) u[b] = U[j * uld + c0 + b];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = u[b] != 0.0f ? fmaf(-l[a], u[b], acc[a][b]) : acc[a][b];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (i0 + a < R && c0 + b < R) a22[(i0 + a) * rs + (c0 + b) * cs] = acc[a][b];
        }
    }
    __syncthreads();
    if (tid == 0) *J.boosts = s_boosts;
}

// compute_spike_tips<float> (spike.hpp:190-250), one CTA per tip, thread per right-hand-side column, the
// w columns in shared memory (col[r * w + c]). which 0: V^b = U^{-1} L^{-1} B on the trailing w x w corner of
// block t's LU; which 1: W^t = L^{-1} U^{-1} C on the leading corner of block t+1's UL. Every corner entry is
// used as the reference's lu_at / ul_at gives it (zero outside the band), sums in j order.
__global__ void __launch_bounds__(kF32Threads)
    k_spike_tips_f32(const TipJobF* __restrict__ jobs, int k, int* __restrict__ nonfinite) {
    extern __shared__ float col[];
    const TipJobF J = jobs[blockIdx.x];
    const int w = k, ld = 2 * k;  // entry (i, j) of the block at f[j * 2k + i + k]
    const float* f = J.f + k;
    auto at = [&](int i, int j) -> float {  // corner coordinates
        const int gi = J.corner + i, gj = J.corner + j;
        return (gi - gj > k || gj - gi > k) ? 0.0f : f[(long long)gj * ld + gi];
    };
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) col[e] = J.rhs[e];
    __syncthreads();
    bool bad = false;
    for (int c = threadIdx.x; c < w; c += blockDim.x) {
        if (J.which == 0) {
            for (int i = 0; i < w; ++i) {  // unit lower, forward
                float acc = col[i * w + c];
                for (int j = 0; j < i; ++j) acc = fmaf(-at(i, j), col[j * w + c], acc);
                col[i * w + c] = acc;
            }
            for (int i = w - 1; i >= 0; --i) {  // upper, backward
                float acc = col[i * w + c];
                for (int j = i + 1; j < w; ++j) acc = fmaf(-at(i, j), col[j * w + c], acc);
                col[i * w + c] = acc / at(i, i);
            }
        } else {
            for (int i = w - 1; i >= 0; --i) {  // unit upper, backward
                float acc = col[i * w + c];
                for (int j = i + 1; j < w; ++j) acc = fmaf(-at(i, j), col[j * w + c], acc);
                col[i * w + c] = acc;
            }
            for (int i = 0; i < w; ++i) {  // lower with the diagonal, forward
                float acc = col[i * w + c];
                for (int j = 0; j < i; ++j) acc = fmaf(-at(i, j), col[j * w + c], acc);
                col[i * w + c] = acc / at(i, i);
            }
        }
        for (int r = 0; r < w; ++r) bad |= !isfinite(col[r * w + c]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) J.out[e] = col[e];
    if (bad) atomicOr(nonfinite + J.flag, 1);
}

// finish_reduced_blocks<float> (spike.hpp:143-170): R = I - W V (float sums, l ascending), the non-finite
// check, dense_lu_nopivot_boosted<float> (spike.hpp:20-45: norm accumulated in double, bv = float(eps * norm),
// row-major no-pivot LU, rows with a zero multiplier skipped); the factors are written in the reduced-block
// BandStore layout (k' = w - 1) of the FP32 sweep plan. One CTA per interface, R in shared memory.
__global__ void __launch_bounds__(kF32Threads)
    k_rbar_f32(const float* __restrict__ wt, const float* __restrict__ vb, int w, double eps, float* __restrict__ rbar,
               long long rstride, int rpad, int* __restrict__ boosts, int* __restrict__ nonfinite) {
    extern __shared__ float a[];
    __shared__ double s_norm;
    __shared__ int s_bad, s_boosts;
    const int t = blockIdx.x, tid = threadIdx.x;
    const float* W = wt + (size_t)t * w * w;
    const float* V = vb + (size_t)t * w * w;
    if (tid == 0) {
        s_norm = 0.0;
        s_bad = 0;
        s_boosts = 0;
    }
    __syncthreads();
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int i = e / w, j = e - i * w;
        float acc = 0.0f;
        for (int l = 0; l < w; ++l) acc = fmaf(W[i * w + l], V[l * w + j], acc);
        const float r = (i == j ? 1.0f : 0.0f) - acc;
        a[e] = r;
        if (!isfinite(r)) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) nonfinite[t] = 1;
        return;
    }
    for (int i = tid; i < w; i += blockDim.x) {
        double row = 0.0;
        for (int j = 0; j < w; ++j) row += fabs((double)a[i * w + j]);
        // non-negative doubles order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(&s_norm), (unsigned long long)__double_as_longlong(row));
    }
    __syncthreads();
    const float bv = (float)(eps * (s_norm > 0 ? s_norm : 1.0));
    for (int j = 0; j < w; ++j) {
        if (tid == 0) {
            const float p = a[j * w + j];
            if (fabsf(p) < bv) {
                a[j * w + j] = p < 0.0f ? -bv : bv;
                ++s_boosts;
            }
        }
        __syncthreads();
        const float p = a[j * w + j];
        for (int i = j + 1 + tid; i < w; i += blockDim.x) {
            const float l = a[i * w + j] / p;
            a[i * w + j] = l;
            if (l == 0.0f) continue;
            for (int c = j + 1; c < w; ++c) a[i * w + c] = fmaf(-l, a[j * w + c], a[i * w + c]);
        }
        __syncthreads();
    }
    // band layout, k' = w - 1: entry (i, j) at j * (2k' + 1) + (i - j + k')
    float* out = rbar + (long long)t * rstride + rpad;
    const int kp = w - 1, bw = 2 * kp + 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int i = e / w, j = e - i * w;
        out[(long long)j * bw + (i - j + kp)] = a[e];
    }
    if (tid == 0) boosts[t] = s_boosts;
}

}  // namespace

void launch_copy_blocks_f32(const double* band, int k, const int* d_offsets, int p, const BandStore& st, float* lu,
                            float* ul, cudaStream_t s) {
    const long long total = st.pstride * (long long)p;
    const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    k_copy_blocks_f32<<<grid, 256, 0, s>>>(band, k, d_offsets, st.pstride, st.pad, total, lu, ul);
    SAP_LAUNCHED();
}

void launch_band_lu_f32(const FactorJobF* d_jobs, int njobs, int max_k, double boost_eps, cudaStream_t s) {
    if (njobs <= 0) return;
    const int pld = kF32B + max_k + 1, uld = max_k + 1;
    const size_t bytes = sizeof(float) * (size_t)(kF32B * pld + kF32B * uld);
    if (bytes > 227 * 1024) throw InvalidArgument("band LU (FP32): half-bandwidth too large for the shared-memory panel");
    SAP_CUDA(cudaFuncSetAttribute(k_band_lu_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_band_lu_f32<<<njobs, kF32Threads, bytes, s>>>(d_jobs, boost_eps, pld, uld);
    SAP_LAUNCHED();
}

void launch_spike_tips_f32(const TipJobF* d_jobs, int njobs, int k, int* nonfinite, cudaStream_t s) {
    if (njobs <= 0) return;
    const size_t bytes = sizeof(float) * (size_t)k * k;
    if (bytes > 227 * 1024) throw InvalidArgument("spike tips (FP32): interface too wide for shared memory");
    SAP_CUDA(cudaFuncSetAttribute(k_spike_tips_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_spike_tips_f32<<<njobs, kF32Threads, bytes, s>>>(d_jobs, k, nonfinite);
    SAP_LAUNCHED();
}

void launch_rbar_f32(const float* wt, const float* vb, int w, int ni, double boost_eps, float* rbar,
                     const BandStore& rst, int* boosts, int* nonfinite, cudaStream_t s) {
    if (ni <= 0) return;
    const size_t bytes = sizeof(float) * (size_t)w * w;
    if (bytes > 227 * 1024) throw InvalidArgument("reduced blocks (FP32): interface too wide for shared memory");
    SAP_CUDA(cudaFuncSetAttribute(k_rbar_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_rbar_f32<<<ni, kF32Threads, bytes, s>>>(wt, vb, w, boost_eps, rbar, rst.pstride, rst.pad, boosts, nonfinite);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
