// Truncated-SPIKE coupling: corners, spike tips and reduced-block products.
//
// Reference: extract_coupling proj/include/sap/spike.hpp:95-116,
// compute_spike_tips :178-254, finish_reduced_blocks :143-170.
//
// Tips. V^b_t = U_BB^{-1} L_BB^{-1} B_t uses the trailing w x w corner of
// LU_t; W^t_t = L_TT^{-1} U_TT^{-1} C_t the leading corner of UL_{t+1}. Each
// CTA owns one tip and a chunk of right-hand-side columns held in smem and
// runs the triangular solves right-looking: at step j every (row, column)
// element below (above) j is updated in parallel. For the forward solves this
// applies each element's updates in the reference's ascending-j order; the
// backward solves apply them in descending j (within tolerance).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

// One 32 x 32 tile of B_t and C_t per CTA, through shared memory: the band is read down its columns (for a fixed
// corner column the corner rows are consecutive band slots) and the row-major corners are written along rows, so
// both sides are coalesced (element-per-thread in corner order read the band at a 2K-double stride).
__global__ void __launch_bounds__(256)
    k_extract_coupling(const double* __restrict__ a, int n, int k, const int* __restrict__ offs,
                       double* __restrict__ bblk, double* __restrict__ cblk, const int* __restrict__ wid) {
    __shared__ double tb[32][33], tc[32][33];  // [corner column j][corner row r]
    const int t = blockIdx.z;
    const int w = k;
    const int wt = wid ? wid[t] : k;  // third stage: the reference's width, embedded (third.cu)
    const int e = offs[t + 1];
    const long long ld = 2LL * k;
    const int r0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = j0 + ty + 8 * q, r = r0 + tx;
        // B_t[r][j] = A(e-w+r, e+j); C_t[r][j] = A(e+r, e-w+j)  (zero outside the band)
        const int bi = e - w + r, bj = e + j, ci = e + r, cj = e - w + j;
        const bool ok = r < w && j < w;
        const bool bin = ok && bi >= 0 && bi < n && bj >= 0 && bj < n && bi - bj <= k && bj - bi <= k;
        const bool cin = ok && ci >= 0 && ci < n && cj >= 0 && cj < n && ci - cj <= k && cj - ci <= k;
        const bool bw = r >= w - wt && j < wt, cw = r < wt && j >= w - wt;
        tb[ty + 8 * q][tx] = bin && bw ? a[(long long)bj * ld + bi + k] : 0.0;
        tc[ty + 8 * q][tx] = cin && cw ? a[(long long)cj * ld + ci + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int r = r0 + ty + 8 * q, j = j0 + tx;
        if (r < w && j < w) {
            bblk[(long long)t * w * w + (long long)r * w + j] = tb[tx][ty + 8 * q];
            cblk[(long long)t * w * w + (long long)r * w + j] = tc[tx][ty + 8 * q];
        }
    }
}

void launch_extract_coupling(const double* band, int n, int k, const int* d_offsets, int p, double* bblk,
                             double* cblk, cudaStream_t s, const int* d_wid) {
    if (p < 2 || k == 0) return;
    dim3 grid(ceil_div(k, 32), ceil_div(k, 32), p - 1);
    k_extract_coupling<<<grid, 256, 0, s>>>(band, n, k, d_offsets, bblk, cblk, d_wid);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
constexpr int kTipCols = 32;
constexpr int kTipThreads = 256;

// grid: (column chunks, jobs). X is w x kTipCols row-major in smem.
__global__ void __launch_bounds__(kTipThreads)
    k_spike_tips(const TipJob* __restrict__ jobs, int k, int* __restrict__ nonfinite) {
    extern __shared__ double sm[];
    const int w = k;
    const TipJob J = jobs[blockIdx.y];
    const int which = J.which, c0 = blockIdx.x * kTipCols;
    const int nc = min(kTipCols, w - c0);
    double* X = sm;                    // [w][kTipCols]
    double* colv = sm + w * kTipCols;  // factor column j, [w]
    const long long ld = 2LL * k;      // band: (i, j) at j*2k + i + k
    const double* f = J.f;
    const int corner = J.corner;       // first row/col of the corner inside the block band
    const double* rhs = J.rhs;
    for (int idx = threadIdx.x; idx < w * kTipCols; idx += blockDim.x) {
        const int r = idx / kTipCols, c = idx - r * kTipCols;
        X[idx] = c < nc ? rhs[(long long)r * w + c0 + c] : 0.0;
    }
    auto F = [&](int i, int j) -> double {  // corner entry (i, j); all |i-j| < w <= k are in band
        return f[(long long)(corner + j) * ld + (corner + i) + k];
    };
    if (which == 0) {
        // forward, unit lower L: X[i] -= L(i,j) X[j], j ascending
        for (int j = 0; j < w - 1; ++j) {
            __syncthreads();
            for (int i = j + 1 + threadIdx.x; i < w; i += blockDim.x) colv[i] = F(i, j);
            __syncthreads();
            const int rows = w - 1 - j;
            for (int idx = threadIdx.x; idx < rows * kTipCols; idx += blockDim.x) {
                const int i = j + 1 + idx / kTipCols, c = idx % kTipCols;
                X[i * kTipCols + c] = fma(-colv[i], X[j * kTipCols + c], X[i * kTipCols + c]);
            }
        }
        // backward, upper U with diagonal
        for (int j = w - 1; j >= 0; --j) {
            __syncthreads();
            for (int i = threadIdx.x; i <= j; i += blockDim.x) colv[i] = F(i, j);
            __syncthreads();
            if (threadIdx.x < kTipCols) X[j * kTipCols + threadIdx.x] = X[j * kTipCols + threadIdx.x] / colv[j];
            __syncthreads();
            for (int idx = threadIdx.x; idx < j * kTipCols; idx += blockDim.x) {
                const int i = idx / kTipCols, c = idx % kTipCols;
                X[i * kTipCols + c] = fma(-colv[i], X[j * kTipCols + c], X[i * kTipCols + c]);
            }
        }
    } else {
        // backward, unit upper U (UL's U): X[i] -= U(i,j) X[j] for i < j, j descending
        for (int j = w - 1; j >= 1; --j) {
            __syncthreads();
            for (int i = threadIdx.x; i < j; i += blockDim.x) colv[i] = F(i, j);
            __syncthreads();
            for (int idx = threadIdx.x; idx < j * kTipCols; idx += blockDim.x) {
                const int i = idx / kTipCols, c = idx % kTipCols;
                X[i * kTipCols + c] = fma(-colv[i], X[j * kTipCols + c], X[i * kTipCols + c]);
            }
        }
        // forward, lower L with diagonal, j ascending
        for (int j = 0; j < w; ++j) {
            __syncthreads();
            for (int i = j + threadIdx.x; i < w; i += blockDim.x) colv[i] = F(i, j);
            __syncthreads();
            if (threadIdx.x < kTipCols) X[j * kTipCols + threadIdx.x] = X[j * kTipCols + threadIdx.x] / colv[j];
            __syncthreads();
            const int rows = w - 1 - j;
            for (int idx = threadIdx.x; idx < rows * kTipCols; idx += blockDim.x) {
                const int i = j + 1 + idx / kTipCols, c = idx % kTipCols;
                X[i * kTipCols + c] = fma(-colv[i], X[j * kTipCols + c], X[i * kTipCols + c]);
            }
        }
    }
    __syncthreads();
    double* out = J.out;
    int bad = 0;
    for (int idx = threadIdx.x; idx < w * kTipCols; idx += blockDim.x) {
        const int r = idx / kTipCols, c = idx - r * kTipCols;
        if (c < nc) {
            const double v = X[idx];
            if (!isfinite(v)) bad = 1;
            out[(long long)r * w + c0 + c] = v;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite + J.flag, 1);
}

// ---------------------------------------------------------------------------
// Blocked tips: X (w x 32 columns of the right-hand side, row-major in smem) is solved in 32-row blocks.
// For block rb the already-solved blocks contribute X_rb -= F_rb,cb X_cb on DMMA (m8n8k4, factor block
// staged in smem, accumulators in registers over all cb), then one warp finishes the diagonal block with
// a lane per column (substitution in the reference's order within the block). Phases:
//   which 0 (V^b = U^{-1} L^{-1} B): lower unit (forward), then upper with diagonal (backward);
//   which 1 (W^t = L^{-1} U^{-1} C): upper unit (backward), then lower with diagonal (forward).
constexpr int kTB = 32;        // row block
constexpr int kTC = 32;        // right-hand-side columns per CTA
constexpr int kTXld = kTC + 4;  // X row stride (doubles): conflict-free DMMA B fragments
constexpr int kTSld = kTB + 4;  // staged factor block stride: conflict-free A fragments

struct TipCorner {
    const double* f;
    int corner;
    long long ld;
    int k;
    __device__ __forceinline__ const double* col(int j) const { return f + (long long)(corner + j) * ld + corner + k; }
};

// stage F[i0:i0+ni, j0:j0+nj] into S[i][j] (zero-padded to 32 x 32)
__device__ __forceinline__ void tip_stage(const TipCorner& F, double* __restrict__ S, int i0, int ni, int j0, int nj) {
    for (int idx = threadIdx.x; idx < kTB * kTB; idx += blockDim.x) {
        const int j = idx >> 5, i = idx & 31;  // lanes walk a factor column (contiguous rows)
        S[i * kTSld + j] = (i < ni && j < nj) ? F.col(j0 + j)[i0 + i] : 0.0;
    }
}

// acc (this warp's two 8 x 8 tiles of X_rb) -= S (32 x 32) * X[j0:j0+32, :]
__device__ __forceinline__ void tip_mma(double (&acc)[2][2], const double* __restrict__ S,
                                        const double* __restrict__ X, int j0, int nj, int tm, int tn0) {
    const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
#pragma unroll
    for (int ks = 0; ks < kTB / 4; ++ks) {
        const int kk = ks * 4 + lc;
        const double a = -S[(tm * 8 + lr) * kTSld + kk];
        const double bx0 = kk < nj ? X[(j0 + kk) * kTXld + tn0 * 8 + lr] : 0.0;
        const double bx1 = kk < nj ? X[(j0 + kk) * kTXld + (tn0 + 1) * 8 + lr] : 0.0;
        dmma_m8n8k4(acc[0][0], acc[0][1], a, bx0, acc[0][0], acc[0][1]);
        dmma_m8n8k4(acc[1][0], acc[1][1], a, bx1, acc[1][0], acc[1][1]);
    }
}

// One triangular phase over all row blocks. LOWER: blocks top-down, else bottom-up. UNIT: no division.
template <bool LOWER, bool UNIT>
__device__ __forceinline__ void tip_phase(const TipCorner& F, double* __restrict__ X, double* __restrict__ S, int w) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int nrb = (w + kTB - 1) / kTB;
    // 16 DMMA tiles (8 x 8) of a 32 x 32 block: warp -> row tile tm, column tiles tn0, tn0+1
    const int tm = warp >> 1, tn0 = (warp & 1) * 2;
    for (int bi = 0; bi < nrb; ++bi) {
        const int rb = LOWER ? bi : nrb - 1 - bi;
        const int r0 = rb * kTB, nr = min(kTB, w - r0);
        double acc[2][2];
        const int ri = r0 + tm * 8 + lr;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int c = (tn0 + t) * 8 + 2 * lc;
            acc[t][0] = ri < w ? X[ri * kTXld + c] : 0.0;
            acc[t][1] = ri < w ? X[ri * kTXld + c + 1] : 0.0;
        }
        // acc layout: D[m = lr][n = 2 lc + e] = X(r0 + tm*8 + lr, (tn0+t)*8 + 2lc + e)
        // the diagonal block's loads are issued first: their latency hides behind the off-diagonal work
        double dpre[kTB * kTB / 256];
#pragma unroll
        for (int u = 0; u < kTB * kTB / 256; ++u) {
            const int idx = threadIdx.x + 256 * u, j = idx >> 5, i = idx & 31;
            dpre[u] = (i < nr && j < nr) ? F.col(r0 + j)[r0 + i] : 0.0;
        }
        // off-diagonal blocks: the next factor block loads into registers while this one multiplies
        double pre[kTB * kTB / 256];
        auto fetch = [&](int bj) {
            const int cb = LOWER ? bj : nrb - 1 - bj;
            const int c0 = cb * kTB, nc = min(kTB, w - c0);
#pragma unroll
            for (int u = 0; u < kTB * kTB / 256; ++u) {
                const int idx = threadIdx.x + 256 * u, j = idx >> 5, i = idx & 31;
                pre[u] = (i < nr && j < nc) ? F.col(c0 + j)[r0 + i] : 0.0;
            }
        };
        auto put = [&](double* Sb) {
#pragma unroll
            for (int u = 0; u < kTB * kTB / 256; ++u) {
                const int idx = threadIdx.x + 256 * u, j = idx >> 5, i = idx & 31;
                Sb[i * kTSld + j] = pre[u];
            }
        };
        if (bi > 0) {
            fetch(0);
            __syncthreads();
            put(S);
        }
        for (int bj = 0; bj < bi; ++bj) {
            const int cb = LOWER ? bj : nrb - 1 - bj;
            const int c0 = cb * kTB, nc = min(kTB, w - c0);
            if (bj + 1 < bi) fetch(bj + 1);
            __syncthreads();
            tip_mma(acc, S, X, c0, nc, tm, tn0);
            if (bj + 1 < bi) {
                __syncthreads();
                put(S);
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int c = (tn0 + t) * 8 + 2 * lc;
            if (ri < w) {
                X[ri * kTXld + c] = acc[t][0];
                X[ri * kTXld + c + 1] = acc[t][1];
            }
        }
#pragma unroll
        for (int u = 0; u < kTB * kTB / 256; ++u) {  // tip_stage(F, S, r0, nr, r0, nr) from the registers
            const int idx = threadIdx.x + 256 * u, j = idx >> 5, i = idx & 31;
            S[i * kTSld + j] = dpre[u];
        }
        __syncthreads();
        if (warp == 0) {
            // lane = column: substitution inside the diagonal block. 1/diag comes from one IEEE division per
            // lane up front (shuffled), so the chain carries a multiply instead of a division.
            double rd = 1.0;
            if (!UNIT) rd = lane < nr ? 1.0 / S[lane * kTSld + lane] : 1.0;
            double x[kTB];
#pragma unroll
            for (int i = 0; i < kTB; ++i) x[i] = i < nr ? X[(r0 + i) * kTXld + lane] : 0.0;
            if (LOWER) {
#pragma unroll
                for (int j = 0; j < kTB; ++j) {
                    if (!UNIT) x[j] *= __shfl_sync(0xffffffffu, rd, j);
#pragma unroll
                    for (int i = j + 1; i < kTB; ++i) x[i] = fma(-S[i * kTSld + j], x[j], x[i]);
                }
            } else {
#pragma unroll
                for (int jj = 0; jj < kTB; ++jj) {
                    const int j = kTB - 1 - jj;
                    if (!UNIT) x[j] *= __shfl_sync(0xffffffffu, rd, j);
#pragma unroll
                    for (int i = 0; i < j; ++i) x[i] = fma(-S[i * kTSld + j], x[j], x[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < kTB; ++i)
                if (i < nr) X[(r0 + i) * kTXld + lane] = x[i];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256, 3)
    k_spike_tips_blk(const TipJob* __restrict__ jobs, int k, int* __restrict__ nonfinite) {
    extern __shared__ __align__(16) double sm[];
    const int w = k;
    const TipJob J = jobs[blockIdx.y];
    const int c0 = blockIdx.x * kTC, nc = min(kTC, w - c0);
    double* X = sm;                  // [w][kTXld]
    double* S = sm + (size_t)w * kTXld;  // [32][kTSld]
    const TipCorner F{J.f, J.corner, 2LL * k, k};
    // the right-hand sides in batches of 8 loads per thread issued before their stores (a load-then-store
    // loop keeps one global load in flight: ~25 serial round trips per CTA at w = 200)
    for (int base = 0; base < w * kTC; base += 8 * 256) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + threadIdx.x + 256 * u;
            const int r = idx / kTC, c = idx - r * kTC;
            v[u] = (idx < w * kTC && c < nc) ? J.rhs[(long long)r * w + c0 + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + threadIdx.x + 256 * u;
            const int r = idx / kTC, c = idx - r * kTC;
            if (idx < w * kTC) X[r * kTXld + c] = v[u];
        }
    }
    __syncthreads();
    if (J.which == 0) {
        tip_phase<true, true>(F, X, S, w);
        tip_phase<false, false>(F, X, S, w);
    } else {
        tip_phase<false, true>(F, X, S, w);
        tip_phase<true, false>(F, X, S, w);
    }
    int bad = 0;
    for (int idx = threadIdx.x; idx < w * kTC; idx += blockDim.x) {
        const int r = idx / kTC, c = idx - r * kTC;
        if (c < nc) {
            const double v = X[r * kTXld + c];
            if (!isfinite(v)) bad = 1;
            J.out[(long long)r * w + c0 + c] = v;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite + J.flag, 1);
}

void launch_spike_tips(const TipJob* d_jobs, int njobs, int k, int* nonfinite, cudaStream_t s) {
    if (njobs <= 0 || k == 0) return;
    {
        const size_t bytes = sizeof(double) * ((size_t)k * kTXld + kTB * kTSld);
        if (bytes <= 200 * 1024) {
            SAP_CUDA(cudaFuncSetAttribute(k_spike_tips_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
            SAP_CUDA(cudaFuncSetAttribute(k_spike_tips_blk, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            k_spike_tips_blk<<<dim3(ceil_div(k, kTC), njobs), 256, bytes, s>>>(d_jobs, k, nonfinite);
            SAP_LAUNCHED();
            return;
        }
    }
    const size_t bytes = sizeof(double) * ((size_t)k * kTipCols + k);
    if (bytes > 227 * 1024) throw InvalidArgument("spike tips: half-bandwidth too large");
    SAP_CUDA(cudaFuncSetAttribute(k_spike_tips, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    dim3 grid(ceil_div(k, kTipCols), njobs);
    k_spike_tips<<<grid, kTipThreads, bytes, s>>>(d_jobs, k, nonfinite);
    SAP_LAUNCHED();
}

// One coupling corner at block boundary e (band coordinates): which 0 -> B[r][j] = A(e-w+r, e+j),
// which 1 -> C[r][j] = A(e+r, e-w+j) (extract_coupling, spike.hpp:107-111).
__global__ void k_extract_one(const double* __restrict__ a, int n, int k, int e, int which, double* __restrict__ out) {
    const int w = k;
    const long long ld = 2LL * k;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w * w; idx += gridDim.x * blockDim.x) {
        const int r = idx / w, j = idx - r * w;
        const int i = which == 0 ? e - w + r : e + r;
        const int c = which == 0 ? e + j : e - w + j;
        const bool in = i >= 0 && i < n && c >= 0 && c < n && i - c <= k && c - i <= k;
        out[idx] = in ? a[(long long)c * ld + i + k] : 0.0;
    }
}

void launch_extract_one(const double* band, int n, int k, int e, int which, double* out, cudaStream_t s) {
    if (k == 0) return;
    k_extract_one<<<ceil_div((long long)k * k, 256), 256, 0, s>>>(band, n, k, e, which, out);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// rbar[t] = I - wt[t] vb[t] (finish_reduced_blocks, spike.hpp:154-160).
// On DMMA (m8n8k4): 32 x 32 output tile per CTA, W and V staged 32 columns / rows at a
// time, each warp two 8 x 8 tiles. The k-sum runs in groups of 4 inside the MMA (within the SURVEY §8c
// tolerance of finish_reduced_blocks' ascending FMA order).
constexpr int kRbLd = 36;
__global__ void __launch_bounds__(256) k_rbar_mma(const double* __restrict__ wt, const double* __restrict__ vb, int w,
                                                  double* __restrict__ rbar, long long rpstride, int rpad,
                                                  int* __restrict__ nonfinite) {
    __shared__ double As[32 * kRbLd];  // As[i][l] = W(i0 + i, l0 + l)
    __shared__ double Bs[32 * kRbLd];  // Bs[l][j] = V(l0 + l, j0 + j)
    const int t = blockIdx.z, i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int tm = warp >> 1, tn0 = (warp & 1) * 2;
    const double* A = wt + (long long)t * w * w;
    const double* Bm = vb + (long long)t * w * w;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int l0 = 0; l0 < w; l0 += 32) {
        // all 8 of this thread's W / V entries in flight before the stores (one at a time before)
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = threadIdx.x + 256 * u, r = idx >> 5, c = idx & 31;
            av[u] = (i0 + r < w && l0 + c < w) ? A[(long long)(i0 + r) * w + l0 + c] : 0.0;
            bv[u] = (l0 + r < w && j0 + c < w) ? Bm[(long long)(l0 + r) * w + j0 + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = threadIdx.x + 256 * u, r = idx >> 5, c = idx & 31;
            As[r * kRbLd + c] = av[u];
            Bs[r * kRbLd + c] = bv[u];
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int kk = ks * 4 + lc;
            const double a = As[(tm * 8 + lr) * kRbLd + kk];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const double b = Bs[kk * kRbLd + (tn0 + q) * 8 + lr];
                dmma_m8n8k4(acc[q][0], acc[q][1], a, b, acc[q][0], acc[q][1]);
            }
        }
        __syncthreads();
    }
    int bad = 0;
    const long long bw = 2LL * w - 1;
    const int i = i0 + tm * 8 + lr;
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = j0 + (tn0 + q) * 8 + 2 * lc + e;
            if (i < w && j < w) {
                const double v = (i == j ? 1.0 : 0.0) - acc[q][e];
                if (!isfinite(v)) bad = 1;
                rbar[(long long)t * rpstride + rpad + (long long)j * bw + (i - j + w - 1)] = v;
            }
        }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite + t, 1);
}

void launch_rbar(const double* wt, const double* vb, int w, int ni, double* rbar, const BandStore& rst,
                 int* nonfinite, cudaStream_t s) {
    if (ni <= 0 || w == 0) return;
    dim3 grid(ceil_div(w, 32), ceil_div(w, 32), ni);
    k_rbar_mma<<<grid, 256, 0, s>>>(wt, vb, w, rbar, rst.pstride, rst.pad, nonfinite);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
