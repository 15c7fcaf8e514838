// Third stage on the device: per-block reordering. The caller supplies sap::third_stage's result
// (proj/include/sap/reorder_cm.hpp:227-274: a half-bandwidth K_b and an optional permutation per
// partition, computed on the host); the device applies it the way the reference does:
//   * factor_blocks (block_factors.hpp:155-180): block b is factored as P_b A_b P_b^T at bandwidth K_b;
//     a nonzero entry the permutation pushes outside K_b is an invalid_argument;
//   * compute_full_spikes (spike.hpp:258-296): with per-block permutations the tips cannot be read off
//     the factor corners, so the full spikes V_t = A_t^{-1} [0; B_t] and W_t = A_{t+1}^{-1} [C_t; 0]
//     are solved over whole blocks (w right-hand sides each, LU of both blocks) and the tips taken
//     from their ends;
//   * block_solve (block_factors.hpp:210-236): every block solve gathers into permuted order, sweeps,
//     and scatters back.
//
// Storage stays at the global half-bandwidth k. A block with K_b < k is factored in the k-wide band
// with zeros outside K_b: the no-pivot LU never fills outside the band, and the extra terms are exact
// zeros, so every entry inside K_b is the one the K_b-wide factorization produces. Interface widths
// w_t = max(K_t, K_{t+1}) (extract_coupling, spike.hpp:102) are embedded in k x k corners:
// B' = A(e-k+r, e+j) restricted to r >= k-w, j < w and C' = A(e+r, e-k+j) restricted to r < w,
// j >= k-w hold the reference's B_t, C_t and zeros elsewhere, so V' and W' carry the reference's
// spikes in columns [0, w) and [k-w, k). With the rows >= w of W'^t zeroed, R' = I - W'^t V'^b is
// diag(R_t, I) exactly, and the interface solve's x^t rows [0, w) - the only ones the apply reads -
// are the reference's.
#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

// ---------------------------------------------------------------------------
// P_b A_b P_b^T into the LU BandStore (zeroed by the caller). gperm[off + r] = off + pm[r]
// (off + r for blocks without a permutation).
__global__ void k_assemble_blocks(const double* __restrict__ a, int n, int k, const int* __restrict__ offs, int p,
                                  const int* __restrict__ gperm, const int* __restrict__ has_perm,
                                  const int* __restrict__ kb, BandStore st, double* __restrict__ lu,
                                  int* __restrict__ bad) {
    const long long w = 2LL * k + 1, total = (long long)n * w;
    for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < total;
         d += (long long)gridDim.x * blockDim.x) {
        const int cg = (int)(d / w);
        const int rg = cg - k + (int)(d - (long long)cg * w);
        if (rg < 0 || rg >= n) continue;
        int lo = 0, hi = p;  // block of column cg: offs[lo] <= cg < offs[lo + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (offs[mid] <= cg) lo = mid; else hi = mid;
        }
        const int b = lo, off = offs[b], m = offs[b + 1] - off;
        if (rg < off || rg >= off + m) continue;
        const double v = a[d];
        const bool perm = has_perm[b] != 0;
        const int pr = (perm ? gperm[rg] : rg) - off, pc = (perm ? gperm[cg] : cg) - off;
        const int kk = kb[b];
        if (pr - pc > kk || pc - pr > kk) {
            if (perm && v != 0.0) atomicMin(bad, b);
            continue;
        }
        if (perm && v == 0.0) continue;  // block_factors.hpp:169
        lu[(long long)b * st.pstride + st.pad + (long long)pc * w + (pr - pc + k)] = v;
    }
}

void launch_assemble_blocks(const double* band, int n, int k, const int* d_offsets, int p, const int* d_gperm,
                            const int* d_has_perm, const int* d_kb, const BandStore& st, double* lu, int* bad,
                            cudaStream_t s) {
    const long long total = (long long)n * (2LL * k + 1);
    if (total == 0) return;
    const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    k_assemble_blocks<<<grid, 256, 0, s>>>(band, n, k, d_offsets, p, d_gperm, d_has_perm, d_kb, st, lu, bad);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Right-hand sides of the full spikes, in each block's permuted row order (spike.hpp:269-276):
// V_t rows gperm[e-k+r] <- B'[r][:], W_t rows gperm[e+r] <- C'[r][:]. vfull / wfull are zeroed,
// n x k row-major, indexed by global (permuted) row.
__global__ void k_full_rhs(const double* __restrict__ bblk, const double* __restrict__ cblk, int k,
                           const int* __restrict__ offs, const int* __restrict__ gperm, double* __restrict__ vfull,
                           double* __restrict__ wfull) {
    const int t = blockIdx.y, e = offs[t + 1];
    const long long kk = (long long)k * k;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kk; idx += gridDim.x * blockDim.x) {
        const int r = idx / k, c = idx - r * k;
        vfull[(long long)gperm[e - k + r] * k + c] = bblk[t * kk + idx];
        wfull[(long long)gperm[e + r] * k + c] = cblk[t * kk + idx];
    }
}

// Tips off the full spikes: V'^b = the last k rows of V_t (original order), W'^t = the first k rows of
// W_t with rows >= w_t zeroed (see the header).
__global__ void k_full_tips(const double* __restrict__ vfull, const double* __restrict__ wfull, int k,
                            const int* __restrict__ offs, const int* __restrict__ gperm, const int* __restrict__ wid,
                            double* __restrict__ vb, double* __restrict__ wt) {
    const int t = blockIdx.y, e = offs[t + 1], w = wid[t];
    const long long kk = (long long)k * k;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kk; idx += gridDim.x * blockDim.x) {
        const int r = idx / k, c = idx - r * k;
        vb[t * kk + idx] = vfull[(long long)gperm[e - k + r] * k + c];
        wt[t * kk + idx] = r < w ? wfull[(long long)gperm[e + r] * k + c] : 0.0;
    }
}

void launch_full_rhs(const double* bblk, const double* cblk, int k, const int* d_offsets, int ni,
                     const int* d_gperm, double* vfull, double* wfull, cudaStream_t s) {
    if (ni <= 0 || k == 0) return;
    k_full_rhs<<<dim3(ceil_div((long long)k * k, 256), ni), 256, 0, s>>>(bblk, cblk, k, d_offsets, d_gperm, vfull,
                                                                         wfull);
    SAP_LAUNCHED();
}

void launch_full_tips(const double* vfull, const double* wfull, int k, const int* d_offsets, int ni,
                      const int* d_gperm, const int* d_wid, double* vb, double* wt, cudaStream_t s) {
    if (ni <= 0 || k == 0) return;
    k_full_tips<<<dim3(ceil_div((long long)k * k, 256), ni), 256, 0, s>>>(vfull, wfull, k, d_offsets, d_gperm,
                                                                          d_wid, vb, wt);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Full spikes: L U X = R over a whole block for a group of 32 right-hand-side columns
// (band_lu_solve, block_factors.hpp:74-90, applied to w columns at once).
//
// One CTA per (job, 32 columns), 256 threads: lane = column, warp = 4 rows of the current 32-row
// chunk. The chunk's update from the k rows before it (after it, backward) runs as a sequence of
// 32 x 32 factor tiles, double-buffered in smem (the next tile's loads in flight during the current
// tile's FMAs); the solved rows of X sit in a ring of smem rows (ceil(k/32)+1 chunks), so X is read
// from global memory once per sweep. The chunk's own 32 x 32 triangle is then solved by warp 0 in
// registers. Forward: each element accumulates its terms in ascending column order, as the reference;
// backward: the off-chunk terms first, then the in-chunk ones (descending), then the division by the
// pivot (within the SURVEY §8c tolerance of the reference's ascending order).
constexpr int kFS = 32;
constexpr int kFSThreads = 256;

__device__ __forceinline__ void fs_tile_load(const FullSpikeJob& J, long long ld, int k, int r0, int j0, bool fwd,
                                             double (&pf)[4], const double* dinv_b = nullptr) {
    if (dinv_b && j0 == r0) {  // diagonal tile: the chunk triangle's inverse (column-major, like the tiles)
        const double* src = dinv_b + ((long long)(r0 / kFS) * 2 + (fwd ? 0 : 1)) * kFS * kFS;
#pragma unroll
        for (int q = 0; q < 4; ++q) pf[q] = __ldg(src + threadIdx.x + kFSThreads * q);
        return;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int idx = threadIdx.x + kFSThreads * q;
        const int i = r0 + (idx & 31), j = j0 + (idx >> 5);
        const bool ok = i < J.m && j >= 0 && j < J.m && (fwd ? (j < i && i - j <= k) : (j >= i && j - i <= k));
        pf[q] = ok ? __ldg(J.f + (long long)j * ld + i) : 0.0;
    }
}

__device__ __forceinline__ void fs_tile_store(double* Lt, const double (&pf)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) Lt[threadIdx.x + kFSThreads * q] = pf[q];
}

__global__ void __launch_bounds__(kFSThreads, 2)
    k_full_spike_solve(const FullSpikeJob* __restrict__ jobs, int k, int* __restrict__ nonfinite,
                       const double* __restrict__ dinv, int nch_max, const unsigned long long* __restrict__ kappa,
                       double kappa_max) {
    extern __shared__ __align__(16) double sm[];
    const FullSpikeJob J = jobs[blockIdx.y];
    if (blockIdx.x * kFS >= J.col_hi || (blockIdx.x + 1) * kFS <= J.col_lo) return;  // all-zero columns
    const int RB = (k + kFS - 1) / kFS + 1;  // ring chunks
    const int T = (J.kb + kFS - 1) / kFS;    // off-chunk tiles per chunk: the block's own bandwidth
    double* Lt = sm;                    // [2][32 cols j][32 rows i]
    double* Xr = sm + 2 * kFS * kFS;    // [RB * 32 rows][32 columns]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = blockIdx.x * kFS, col = c0 + lane;
    const bool colok = col < k;
    const long long ld = 2LL * k;
    const int m = J.m, nch = (m + kFS - 1) / kFS;
    auto slot = [&](int row) { return ((row / kFS) % RB) * kFS + (row % kFS); };
    double pf[4];
    int bad = 0;
    // the chunk triangles through their precomputed inverses (the sweeps' k_chunk_inverses, same 32-row
    // chunks) unless they are ill-conditioned: then warp 0 substitutes (as the substitution sweeps)
    const bool use_inv = dinv != nullptr && __longlong_as_double((long long)*kappa) <= kappa_max;
    const double* dinv_b = use_inv ? dinv + (long long)J.blk * nch_max * 2 * kFS * kFS : nullptr;
    for (int pass = 0; pass < 2; ++pass) {
        const bool fwd = pass == 0;
        for (int i = threadIdx.x; i < RB * kFS * kFS; i += kFSThreads) Xr[i] = 0.0;
        // tile t < T: off-chunk columns (forward: j0 = r0 - 32 (T - t), ascending; backward:
        // j0 = r0 + 32 (t + 1)); tile T: the diagonal tile j0 = r0
        auto tile_j0 = [&](int r0, int t) {
            return t == T ? r0 : (fwd ? r0 - kFS * (T - t) : r0 + kFS * (t + 1));
        };
        auto first_tile = [&](int r0) {
            int t = 0;
            while (t < T && (fwd ? tile_j0(r0, t) + kFS <= 0 : tile_j0(r0, t) >= m)) ++t;
            return t;
        };
        auto load_rhs = [&](int r0, double (&a)[4]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int row = r0 + warp * 4 + q;
                a[q] = (row < m && colok) ? J.x[(long long)row * k + col] : 0.0;
            }
        };
        const int ch_first = fwd ? J.first_row / kFS : nch - 1, step = fwd ? 1 : -1;
        // the next chunk's first tile and right-hand sides are loaded while this chunk's triangle is
        // solved (the loads overlap warp 0's substitution)
        double accn[4];
        load_rhs(ch_first * kFS, accn);
        fs_tile_load(J, ld, k, ch_first * kFS, tile_j0(ch_first * kFS, first_tile(ch_first * kFS)), fwd, pf, dinv_b);
        for (int ch = ch_first; fwd ? ch < nch : ch >= 0; ch += step) {
            const int r0 = ch * kFS, chn = ch + step;
            const bool has_next = fwd ? chn < nch : chn >= 0;
            double acc[4] = {accn[0], accn[1], accn[2], accn[3]};
            int t = first_tile(r0);
            fs_tile_store(Lt + (t & 1) * kFS * kFS, pf);
            __syncthreads();
            for (; t <= T; ++t) {
                const double* L = Lt + (t & 1) * kFS * kFS;
                if (t < T) {
                    fs_tile_load(J, ld, k, r0, tile_j0(r0, t + 1), fwd, pf, dinv_b);
                    const int j0 = tile_j0(r0, t);
                    const double* xr = Xr + slot(max(j0, 0)) * kFS + lane;
#pragma unroll 8
                    for (int jj = 0; jj < kFS; ++jj) {
                        const double xv = xr[jj * kFS];
                        const double2 l01 = *reinterpret_cast<const double2*>(L + jj * kFS + warp * 4);
                        const double2 l23 = *reinterpret_cast<const double2*>(L + jj * kFS + warp * 4 + 2);
                        acc[0] = fma(-l01.x, xv, acc[0]);
                        acc[1] = fma(-l01.y, xv, acc[1]);
                        acc[2] = fma(-l23.x, xv, acc[2]);
                        acc[3] = fma(-l23.y, xv, acc[3]);
                    }
                    fs_tile_store(Lt + ((t + 1) & 1) * kFS * kFS, pf);
                } else {
                    double* xc = Xr + slot(r0) * kFS;
#pragma unroll
                    for (int q = 0; q < 4; ++q) xc[(warp * 4 + q) * kFS + lane] = acc[q];
                    if (has_next) {
                        load_rhs(chn * kFS, accn);
                        fs_tile_load(J, ld, k, chn * kFS, tile_j0(chn * kFS, first_tile(chn * kFS)), fwd, pf, dinv_b);
                    }
                    __syncthreads();
                    if (use_inv) {
                        // x = T^{-1} acc: every warp, 4 rows each
                        double y[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
                        for (int jj = 0; jj < kFS; ++jj) {
                            const double xv = xc[jj * kFS + lane];
                            const double2 l01 = *reinterpret_cast<const double2*>(L + jj * kFS + warp * 4);
                            const double2 l23 = *reinterpret_cast<const double2*>(L + jj * kFS + warp * 4 + 2);
                            y[0] = fma(l01.x, xv, y[0]);
                            y[1] = fma(l01.y, xv, y[1]);
                            y[2] = fma(l23.x, xv, y[2]);
                            y[3] = fma(l23.y, xv, y[3]);
                        }
                        __syncthreads();
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = warp * 4 + q;
                            xc[i * kFS + lane] = y[q];
                            if (r0 + i < m && colok) {
                                J.x[(long long)(r0 + i) * k + col] = y[q];
                                if (!fwd && !isfinite(y[q])) bad = 1;
                            }
                        }
                    } else if (warp == 0) {
                        // substitution in shared memory (lane = column): ill-conditioned triangles only
                        if (fwd) {
                            for (int j = 0; j < kFS - 1; ++j) {
                                const double xj = xc[j * kFS + lane];
                                for (int i = j + 1; i < kFS; ++i)
                                    xc[i * kFS + lane] = fma(-L[j * kFS + i], xj, xc[i * kFS + lane]);
                            }
                        } else {
                            // the 32 pivot reciprocals in parallel (lane i: row r0 + i), then
                            // x / d = fma(fma(-q, d, x), 1/d, q), q = x / d rounded through 1/d
                            const double rcl = r0 + lane < m ? 1.0 / L[lane * kFS + lane] : 0.0;
                            for (int j = kFS - 1; j >= 0; --j) {
                                const double rc = __shfl_sync(0xffffffffu, rcl, j), d = L[j * kFS + j];
                                const double xv = xc[j * kFS + lane], q = xv * rc;
                                const double xj = r0 + j < m ? fma(fma(-q, d, xv), rc, q) : 0.0;
                                xc[j * kFS + lane] = xj;
                                for (int i = 0; i < j; ++i)
                                    xc[i * kFS + lane] = fma(-L[j * kFS + i], xj, xc[i * kFS + lane]);
                            }
                        }
                        for (int i = 0; i < kFS; ++i) {
                            const double xi = xc[i * kFS + lane];
                            if (r0 + i < m && colok) {
                                J.x[(long long)(r0 + i) * k + col] = xi;
                                if (!fwd && !isfinite(xi)) bad = 1;
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite + J.flag, 1);
}

size_t full_spike_smem(int k) {
    const int T = (k + kFS - 1) / kFS;
    return sizeof(double) * (2 * kFS * kFS + (size_t)(T + 1) * kFS * kFS);
}

void launch_full_spikes(const FullSpikeJob* d_jobs, int njobs, int k, int* nonfinite, const double* dinv, int nch_max,
                        const unsigned long long* kappa, double kappa_max, cudaStream_t s) {
    if (njobs <= 0 || k == 0) return;
    const size_t bytes = full_spike_smem(k);
    if (bytes > 227 * 1024) throw InvalidArgument("third stage: half-bandwidth too large for the full-spike solve");
    SAP_CUDA(cudaFuncSetAttribute(k_full_spike_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_full_spike_solve<<<dim3(ceil_div(k, kFS), njobs), kFSThreads, bytes, s>>>(d_jobs, k, nonfinite, dinv, nch_max,
                                                                              kappa, kappa_max);
    SAP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Block permutations of a vector (block_solve, block_factors.hpp:222-229):
// scatter: out[gperm[i]] = in[i]; gather: out[i] = in[gperm[i]].
template <class T>
__global__ void k_permute(const int* __restrict__ gperm, const T* __restrict__ in, T* __restrict__ out, int n,
                          int scatter) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int g = gperm[i];
        if (scatter)
            out[g] = in[i];
        else
            out[i] = in[g];
    }
}

template <class T>
void launch_permute(const int* d_gperm, const T* in, T* out, int n, bool scatter, cudaStream_t s) {
    if (n <= 0) return;
    k_permute<T><<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(d_gperm, in, out, n, scatter ? 1 : 0);
    SAP_LAUNCHED();
}
template void launch_permute<double>(const int*, const double*, double*, int, bool, cudaStream_t);
template void launch_permute<float>(const int*, const float*, float*, int, bool, cudaStream_t);

}  // namespace sapgpu
