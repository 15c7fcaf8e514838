// Per-partition banded factorization (SaP split step).
//
// Reference: factor_blocks / band_lu_inplace / band_ul_inplace,
// proj/include/sap/block_factors.hpp:22-71, :138-206; dense reduced-block LU
// dense_lu_nopivot_boosted, proj/include/sap/spike.hpp:20-45.
//
// One kernel factors all three: it works on a strided view (FactorJob) so
//   LU of a band   : rs = 1,  cs = 2k   (tall-thin slot j*2k + i + k)
//   UL of a band   : the same LU on the flipped system J A J (rs = -1, cs = -2k);
//                    the reference's UL is bitwise rev(LU(rev(band)))
//   dense R = LU   : rs = w,  cs = 1, k = w-1
// Algorithm: right-looking blocked LU, panel width B. For panel columns
// [jb, jb+nb):
//   1. the (nb+K) x nb panel and the nb x K block row U12 are staged in smem;
//   2. the panel is factored column by column (pivot boosting exactly as the
//      reference: |p| < eps*scale -> ±eps*scale, sign of zero is +);
//   3. U12 <- L11^{-1} U12 (per-column forward substitution, reference order);
//   4. the K x K trailing block A22 -= L21 U12 is applied with FP64 tensor
//      cores (mma.sync m8n8k4 f64 -> DMMA.8x8x4), accumulators initialised
//      from A22 so every element receives the reference's updates in the
//      reference's column order (FMA-contracted).
// A22 streams through L2 (ld/st.global.cg); a partition's K x K window is
// 320 KB at K = 200, so 100 concurrent factorizations keep ~32 MB hot in the
// 126 MB L2 while the band itself is read from and written to HBM once.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

long long g_launch_count = 0;

// ---------------------------------------------------------------------------
// Block infinity norms: row r of block b sums |A(off+r, off+c)| over in-block
// columns c in ascending order (bitwise the reference's row loop,
// block_factors.hpp:196-203). A warp owns 32 consecutive rows of one block and
// walks the union of their column ranges so that, for each column, the 32
// loads are one contiguous run (slot = c*2k + r + k). The per-block max is
// order-independent: non-negative doubles compare like their bit patterns,
// so atomicMax on the bits is exact; NaN rows are skipped like the
// reference's `row > norm` test.
// F32: the norm of the band cast to float (build_precond_op<float>'s banded_cast, pipeline.hpp:150; the
// row sums stay double, banded_matrix.hpp:90).
template <bool F32>
__global__ void __launch_bounds__(256)
    k_block_norms(const double* __restrict__ a, int k, const int* __restrict__ offs, long long pstride, int pad,
                  unsigned long long* __restrict__ norms_bits, int* __restrict__ nonfinite, int p,
                  const int* __restrict__ nrows) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int off = offs[b], m = offs[b + 1] - off;
    const int r0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
    if (r0 >= m) return;
    const long long ld = 2LL * k;
    const double* base = a + (pstride > 0 ? (long long)b * pstride + pad : (long long)off * (2LL * k + 1));
    const int r = r0 + lane;
    const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, m - 1);
    double row = 0.0;
    const double* col = base + (long long)clo * ld + r + k;
#pragma unroll 8
    for (int c = clo; c <= chi; ++c, col += ld)
        if (r < m && r - c <= k && c - r <= k) row += fabs(F32 ? (double)(float)*col : *col);
    if (nonfinite && r < m) {
        // finiteness of every stored entry of global row off + r (the Krylov solver may then take
        // b - A*0 = b exactly for the zero initial guess): the in-block entries through the row sum
        // (a non-finite |a| makes it inf/NaN), the coupling columns outside the block here
        bool bad = !isfinite(row);
        const int n = offs[p];
        for (int c = max(r - k, -off); c < 0; ++c) bad |= !isfinite(base[(long long)c * ld + r + k]);
        for (int c = m; c <= min(r + k, n - 1 - off); ++c) bad |= !isfinite(base[(long long)c * ld + r + k]);
        if (bad) atomicOr(nonfinite, 1);
    }
    double best = (r < m && row > 0.0 && (!nrows || r < nrows[b])) ? row : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0 && best > 0.0) atomicMax(norms_bits + b, (unsigned long long)__double_as_longlong(best));
}

void launch_block_norms(const double* band, int max_m, int k, const int* d_offsets, int p, const BandStore* store,
                        double* norms, cudaStream_t s, int* nonfinite, const int* d_nrows, bool f32) {
    SAP_CUDA(cudaMemsetAsync(norms, 0, sizeof(double) * p, s));
    dim3 grid(ceil_div(ceil_div(max_m, 32), 8), p);
    (f32 ? k_block_norms<true> : k_block_norms<false>)<<<grid, 256, 0, s>>>(band, k, d_offsets, store ? store->pstride : 0, store ? store->pad : 0,
                                        reinterpret_cast<unsigned long long*>(norms), store ? nullptr : nonfinite, p,
                                        d_nrows);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Block band copies into a BandStore: slot o of block b (o < m_b*(2k+1)) is
// local column c = o / (2k+1), local row r = c - k + o % (2k+1); it takes the
// global band's value when r lies inside the block and zero otherwise;
// padding slots are zeroed.
__global__ void k_copy_blocks(const double* __restrict__ a, int k, const int* __restrict__ offs, long long pstride,
                              int pad, long long total, double* __restrict__ lu, double* __restrict__ ul) {
    const long long w = 2LL * k + 1;
    for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < total;
         d += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(d / pstride);
        const long long o = d - (long long)b * pstride - pad;
        const int off = offs[b], m = offs[b + 1] - off;
        double v = 0.0;
        if (o >= 0 && o < (long long)m * w) {
            const long long c = o / w;
            const long long slot = o - c * w;
            const long long r = c - k + slot;
            if (r >= 0 && r < m) v = a[(off + c) * w + slot];
        }
        lu[d] = v;
        if (ul) ul[d] = v;
    }
}

void launch_copy_blocks(const double* band, int k, const int* d_offsets, int p, const BandStore& st, double* lu,
                             double* ul, cudaStream_t s) {
    const long long total = st.pstride * (long long)p;
    const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    k_copy_blocks<<<grid, 256, 0, s>>>(band, k, d_offsets, st.pstride, st.pad, total, lu, ul);
    SAP_LAUNCHED();
}

// The slots of a BandStore block that lie outside the block's matrix (the top-left and bottom-right
// corner triangles of its band, the leading pad and the trailing slack) zeroed: what k_copy_blocks
// leaves in them, for the LU kernels that read the unfactored band from its source instead.
__global__ void k_zero_pad(int k, const int* __restrict__ offs, long long pstride, int pad, double* __restrict__ lu,
                           double* __restrict__ ul) {
    const int b = blockIdx.y;
    const long long w = 2LL * k + 1;
    const int m = offs[b + 1] - offs[b];
    double* f0 = lu + (long long)b * pstride;
    double* f1 = ul ? ul + (long long)b * pstride : nullptr;
    const long long corner = (long long)k * w;
    const long long tail0 = pad + (long long)m * w;
    const long long n_items = 2 * corner + pad + (pstride - tail0);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n_items;
         q += (long long)gridDim.x * blockDim.x) {
        long long d = -1;
        if (q < 2 * corner) {
            const long long qq = q < corner ? q : q - corner;
            const long long c0 = qq / w, slot = qq - c0 * w;
            const long long c = q < corner ? c0 : m - 1 - c0;
            if (c < 0 || c >= m) continue;
            const long long r = c - k + slot;
            if (r >= 0 && r < m) continue;
            d = pad + c * w + slot;
        } else {
            const long long t = q - 2 * corner;
            d = t < pad ? t : tail0 + (t - pad);
        }
        f0[d] = 0.0;
        if (f1) f1[d] = 0.0;
    }
}

void launch_zero_pad(int k, const int* d_offsets, int p, const BandStore& st, double* lu, double* ul, cudaStream_t s) {
    const long long items = 2LL * k * (2LL * k + 1) + st.pstride;
    dim3 grid((unsigned)std::min<long long>((items + 255) / 256, 64), (unsigned)p);
    k_zero_pad<<<grid, 256, 0, s>>>(k, d_offsets, st.pstride, st.pad, lu, ul);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Blocked LU.

template <int B, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_band_lu(const FactorJob* __restrict__ jobs, double eps, int pld, int uld) {
    extern __shared__ __align__(16) double smem[];
    double* P = smem;             // panel, column-major: P[c*pld + r]
    double* U = smem + B * pld;   // U12, row-major:      U[r*uld + c]
    __shared__ int s_boosts;

    const FactorJob J = jobs[blockIdx.x];
    const int m = J.m, K = J.k, tid = threadIdx.x;
    const long long rs = J.rs, cs = J.cs;
    double* const base = J.base;
    const double scale = *J.scale;
    const double bv = eps * (scale > 0 ? scale : 1.0);
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int NW = NT / 32;
    if (tid == 0) s_boosts = 0;

    for (int jb = 0; jb < m; jb += B) {
        const int nb = min(B, m - jb);
        const int ph = min(nb + K, m - jb);  // panel rows jb .. jb+ph-1
        const int R = ph - nb;               // trailing block order = min(K, m-jb-nb)
        __syncthreads();

        // 1. stage panel and U12 (zero outside the band and beyond the block)
        for (int idx = tid; idx < B * pld; idx += NT) {
            const int c = idx / pld, r = idx - c * pld;
            double v = 0.0;
            if (c < nb && r < ph && r - c <= K && c - r <= K)
                v = __ldcg(base + (long long)(jb + r) * rs + (long long)(jb + c) * cs);
            P[idx] = v;
        }
        for (int idx = tid; idx < B * uld; idx += NT) {
            const int r = idx / uld, c = idx - r * uld;
            double v = 0.0;
            if (r < nb && c < R && nb + c - r <= K)
                v = __ldcg(base + (long long)(jb + r) * rs + (long long)(jb + nb + c) * cs);
            U[idx] = v;
        }
        __syncthreads();

        // 2. unblocked panel factorization (reference column loop)
        for (int c = 0; c < nb; ++c) {
            if (tid == 0) {
                double p = P[c * pld + c];
                if (fabs(p) < bv) {
                    p = p < 0.0 ? -bv : bv;
                    P[c * pld + c] = p;
                    ++s_boosts;
                }
            }
            __syncthreads();
            const double p = P[c * pld + c];
            const int hi = min(c + K, ph - 1);
            for (int r = c + 1 + tid; r <= hi; r += NT) P[c * pld + r] = P[c * pld + r] / p;
            __syncthreads();
            const int rows = hi - c, cols = nb - 1 - c;
            for (int idx = tid; idx < rows * cols; idx += NT) {
                const int q = idx / rows;
                const int cc = c + 1 + q, r = c + 1 + (idx - q * rows);
                const double u = P[cc * pld + c];
                if (u != 0.0) P[cc * pld + r] = fma(-P[c * pld + r], u, P[cc * pld + r]);
            }
            __syncthreads();
        }

        // 3. U12 <- L11^{-1} U12, one column per thread, j ascending
        for (int c = tid; c < R; c += NT) {
            for (int r = 1; r < nb; ++r) {
                double acc = U[r * uld + c];
                for (int j = 0; j < r; ++j) {
                    const double u = U[j * uld + c];
                    if (u != 0.0) acc = fma(-P[j * pld + r], u, acc);
                }
                U[r * uld + c] = acc;
            }
        }
        // write back the panel (L11\U11, L21); U12 after the solve
        for (int idx = tid; idx < B * pld; idx += NT) {
            const int c = idx / pld, r = idx - c * pld;
            if (c < nb && r < ph && r - c <= K && c - r <= K)
                __stcg(base + (long long)(jb + r) * rs + (long long)(jb + c) * cs, P[idx]);
        }
        __syncthreads();
        for (int idx = tid; idx < B * uld; idx += NT) {
            const int r = idx / uld, c = idx - r * uld;
            if (r < nb && c < R && nb + c - r <= K)
                __stcg(base + (long long)(jb + r) * rs + (long long)(jb + nb + c) * cs, U[idx]);
        }

        // 4. A22 -= L21 * U12 on DMMA. Warp tile = 2 x 4 mma tiles (16 x 32).
        if (R > 0) {
            const int TT = (R + 7) >> 3;
            const int WR = (TT + 1) >> 1, WC = (TT + 3) >> 2;
            const int ksteps = (nb + 3) >> 2;
            const int lr = lane >> 2, lc = lane & 3;
            double* const a22 = base + (long long)(jb + nb) * rs + (long long)(jb + nb) * cs;
            for (int wt = warp; wt < WR * WC; wt += NW) {
                const int wr = wt % WR, wc = wt / WR;
                double acc[2][4][2];
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int i = (wr * 2 + a) * 8 + lr;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c0 = (wc * 4 + q) * 8 + 2 * lc;
                        acc[a][q][0] = (i < R && c0 < R) ? __ldcg(a22 + i * rs + c0 * cs) : 0.0;
                        acc[a][q][1] = (i < R && c0 + 1 < R) ? __ldcg(a22 + i * rs + (c0 + 1) * cs) : 0.0;
                    }
                }
                const bool row1 = (wr * 2 + 1) < TT;
                for (int ks = 0; ks < ksteps; ++ks) {
                    const int kk = ks * 4 + lc;
                    const double a0 = -P[kk * pld + nb + (wr * 2) * 8 + lr];
                    const double a1 = row1 ? -P[kk * pld + nb + (wr * 2 + 1) * 8 + lr] : 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (wc * 4 + q < TT) {
                            const double bq = U[kk * uld + (wc * 4 + q) * 8 + lr];
                            dmma_m8n8k4(acc[0][q][0], acc[0][q][1], a0, bq, acc[0][q][0], acc[0][q][1]);
                            if (row1) dmma_m8n8k4(acc[1][q][0], acc[1][q][1], a1, bq, acc[1][q][0], acc[1][q][1]);
                        }
                    }
                }
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int i = (wr * 2 + a) * 8 + lr;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c0 = (wc * 4 + q) * 8 + 2 * lc;
                        if (i < R && c0 < R) __stcg(a22 + i * rs + c0 * cs, acc[a][q][0]);
                        if (i < R && c0 + 1 < R) __stcg(a22 + i * rs + (c0 + 1) * cs, acc[a][q][1]);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0) *J.boosts = s_boosts;
}

static int pad16_4(int x) { return x + (((4 - x) % 16) + 16) % 16; }

template <int B>
static void launch_lu_b(const FactorJob* jobs, int njobs, int max_k, double eps, cudaStream_t s) {
    constexpr int NT = 512;
    const int k8 = ((max_k + 7) / 8) * 8;
    const int pld = pad16_4(B + k8);
    const int uld = pad16_4(k8 > 0 ? k8 : 8);
    const size_t bytes = sizeof(double) * (size_t)(B * pld + B * uld);
    if (bytes > 227 * 1024) throw InvalidArgument("band LU: half-bandwidth too large for the shared-memory panel");
    SAP_CUDA(cudaFuncSetAttribute(k_band_lu<B, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_band_lu<B, NT><<<njobs, NT, bytes, s>>>(jobs, eps, pld, uld);
    SAP_LAUNCHED();
}

void launch_band_lu(const FactorJob* d_jobs, int njobs, int max_k, double boost_eps, cudaStream_t s, bool streamed,
                    int m_max, int* df_scratch, int lu_kernel) {
    if (njobs <= 0) return;
    const bool df = lu_kernel == 1   ? false
                    : lu_kernel == 2 ? (max_k >= 64 && max_k <= 512)
                                     : lu_df_applies(max_k, njobs, m_max);
    if (df_scratch && m_max > 0 && df) {
        launch_band_lu_df(d_jobs, njobs, m_max, max_k, boost_eps, s, streamed, df_scratch);
        return;
    }
    if (launch_band_lu_ws(d_jobs, njobs, max_k, boost_eps, s, streamed)) return;
    if (streamed) throw CudaFailure("streamed factorization needs k_band_lu_res");
    if (max_k >= 48 && max_k <= 360)
        launch_lu_b<32>(d_jobs, njobs, max_k, boost_eps, s);
    else if (max_k > 360 && max_k <= 820)
        launch_lu_b<16>(d_jobs, njobs, max_k, boost_eps, s);
    else if (max_k > 820)
        launch_lu_b<8>(d_jobs, njobs, max_k, boost_eps, s);
    else
        launch_lu_b<16>(d_jobs, njobs, max_k, boost_eps, s);
}

// ---------------------------------------------------------------------------
// Streamed-upload check: job j (block j mod p) was factored without boosting; the reference would have
// boosted iff some |pivot| < boost_eps * ||A_b|| (block_factors.hpp:29). One CTA per job reads the
// pivots off U's diagonal; bad |= 1 then, |= 2 on a stalled upload (the kernel left minpiv[j] = -1).
__global__ void k_stream_check(const FactorJob* __restrict__ jobs, const double* __restrict__ minpiv,
                               const double* __restrict__ norms, int p, double eps, int* __restrict__ bad) {
    const int j = blockIdx.x;
    const FactorJob J = jobs[j];
    const double sc = norms[j % p];
    const double bv = eps * (sc > 0 ? sc : 1.0);
    int f = 0;
    for (int i = threadIdx.x; i < J.m; i += blockDim.x)
        if (fabs(J.base[(long long)i * (J.rs + J.cs)]) < bv) f = 1;
    if (threadIdx.x == 0 && minpiv[j] < 0.0) f |= 2;
    f = __syncthreads_or(f & 1) | (threadIdx.x == 0 ? (f & 2) : 0);
    if (threadIdx.x == 0 && f) atomicOr(bad, f);
}

void launch_stream_check(const FactorJob* d_jobs, const double* minpiv, const double* norms, int njobs, int p,
                         double eps, int* bad, cudaStream_t s) {
    SAP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    k_stream_check<<<njobs, 256, 0, s>>>(d_jobs, minpiv, norms, p, eps, bad);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Dense reduced blocks: infinity norm (row sums, ascending j as in
// dense_lu_nopivot_boosted spike.hpp:22-27) and the all_finite check (:162).
__global__ void k_dense_norms(const double* __restrict__ a, int w, double* norms, int* nonfinite) {
    const double* blk = a + (long long)blockIdx.x * w * w;
    double best = 0.0;
    int bad = 0;
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        double row = 0.0;
        for (int j = 0; j < w; ++j) {
            const double v = blk[(long long)i * w + j];
            if (!isfinite(v)) bad = 1;
            row += fabs(v);
        }
        best = fmax(best, row);
    }
    __shared__ double red[32];
    __shared__ int rbad[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
        red[warp] = best;
        rbad[warp] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        int f = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
            v = fmax(v, red[q]);
            f |= rbad[q];
        }
        norms[blockIdx.x] = v;
        nonfinite[blockIdx.x] = f;
    }
}

void launch_dense_norms(const double* a, int w, int ni, double* norms, int* nonfinite, cudaStream_t s) {
    if (ni <= 0) return;
    k_dense_norms<<<ni, 256, 0, s>>>(a, w, norms, nonfinite);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
