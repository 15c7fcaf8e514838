// Preconditioner application M^{-1} b (SaP-D and SaP-C).
//
// Reference: block_solve / band_lu_solve proj/include/sap/block_factors.hpp:74-90,
// :210-236 and apply_preconditioner proj/include/sap/spike.hpp:304-351.
//
// Band sweeps, TMA path (k_sweep_tma). One CTA per block walks the rows in
// TR-row chunks. The factor slab a chunk needs -- rows [i0, i0+TR) of the K
// columns left of it (forward, L) or right of it (backward, U) -- is ONE 2-D
// TMA box of an overlapping tensor view of the tall-thin band (element (i, c)
// at c*2k + i + k: dim0 = row, stride1 = 2k doubles), streamed S chunks ahead
// into a shared-memory ring under an mbarrier, with deeper L2 prefetches.
// The chunk's diagonal TRxTR triangle is not walked serially: its inverse
// (unit-lower L^{-1} / upper U^{-1}, precomputed once at setup by
// k_chunk_inverses) arrives with the slab, so finishing a chunk is a TRxTR
// mat-vec on warp 0 instead of a TR-step shuffle chain. Per chunk:
//   phase 1: warp 0 finishes chunk ch-1 (x = D^{-1} z) while warps 1..15 form
//            the part of chunk ch's row sums that only needs older x;
//   phase 2: all warps add the TR columns that need chunk ch-1's x.
// x lives in a circular shared-memory window of the last K+2TR rows.
// Padding/out-of-band slab entries are masked in registers; entries beyond the
// block are zero in the BandStore or zero-filled by TMA.
//
// k == 0 (or a band too wide for the TMA ring) uses k_sweep_ldgsts: the same
// chunking with cp.async slabs and a shuffle triangle solve.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

constexpr int kSwThreads = 512;
constexpr int kSwWarps = kSwThreads / 32;

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier, TMA, bulk copies, cp.async.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = smem_u32(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(a), "r"(parity)
                     : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x0, int x1, int x2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x0), "r"(x1), "r"(x2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x0, int x1, int x2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(x0), "r"(x1),
                 "r"(x2)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
template <class T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// Diagonal-chunk inverses: dinv[((b*nch_max + q)*2 + dir)*TR*TR + j*TR + i] =
// (L_qq^{-1})(i, j) for dir 0 (unit lower), (U_qq^{-1})(i, j) for dir 1.
// Rows beyond the block are padded with the identity. One warp per inverse,
// lane j builds column j by substitution on e_j.
// UL: the chunk triangles of a UL store (A = U'L', U' unit upper, L' lower with the diagonal; the UL
// job's factors at their original positions): dir 0 (top-down) inverts the lower triangle with its
// diagonal, dir 1 (bottom-up) the unit upper one; no substitution triangles (UL sweeps use inverses only).
template <class T, int TR, bool UL = false>
__global__ void k_chunk_inverses(const T* __restrict__ f0, long long pstride, int pad, const int* __restrict__ offs,
                                 int k, T* __restrict__ dinv, int nch_max, T* __restrict__ tri,
                                 unsigned long long* __restrict__ kappa_bits) {
    __shared__ T blk[TR][TR + 1];       // blk[j][i] = F(i0+i, i0+j)
    __shared__ T X[2][TR][TR + 1];      // X[dir][j][i]
    const int b = blockIdx.y, q = blockIdx.x;
    const int m = offs[b + 1] - offs[b];
    const int i0 = q * TR;
    if (i0 >= m) return;
    const int rows = min(TR, m - i0);
    const T* f = f0 + (long long)b * pstride + pad;
    const long long ld = 2LL * k;
    // every thread's TR*TR/64 chunk entries are loaded before any is stored (the conditional load-then-store
    // loop kept one global load in flight per thread: ~16 serial L2/HBM round trips per CTA)
    constexpr int kPer = TR * TR / 64;
    T v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int idx = threadIdx.x + u * 64;
        const int j = idx / TR, i = idx % TR;
        const bool in = i < rows && j < rows && i - j <= k && j - i <= k;
        v[u] = in ? f[(long long)(i0 + j) * ld + i0 + i + k] : T(0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int idx = threadIdx.x + u * 64;
        const int j = idx / TR, i = idx % TR;
        blk[j][i] = (i < rows && j < rows) ? v[u] : ((i == j) ? T(1) : T(0));
    }
    __syncthreads();
    const int dir = threadIdx.x >> 5, j = threadIdx.x & 31;
    // UL: the top-down (lower) inverses are read only by the tip sweeps' stopped second sweep, i.e. for the
    // chunks covering the first k rows; the others are not formed (half the kernel's work on the side stream)
    const bool skip = UL && dir == 0 && q >= (k + TR - 1) / TR;
    if (UL && j < TR && !skip) {
        if (dir == 0) {  // lower with diagonal
            for (int i = 0; i < TR; ++i) X[0][j][i] = T(0);
            X[0][j][j] = T(1) / blk[j][j];
            for (int i = j + 1; i < TR; ++i) {
                T acc = T(0);
                for (int l = j; l < i; ++l) acc = fma(blk[l][i], X[0][j][l], acc);
                X[0][j][i] = -acc / blk[i][i];
            }
        } else {  // unit upper
            for (int i = 0; i < TR; ++i) X[1][j][i] = (i == j) ? T(1) : T(0);
            for (int i = j - 1; i >= 0; --i) {
                T acc = T(0);
                for (int l = i + 1; l <= j; ++l) acc = fma(blk[l][i], X[1][j][l], acc);
                X[1][j][i] = -acc;
            }
        }
    } else if (!UL && j < TR) {
        if (dir == 0) {  // unit lower
            for (int i = 0; i < TR; ++i) X[0][j][i] = (i == j) ? T(1) : T(0);
            for (int i = j + 1; i < TR; ++i) {
                T acc = T(0);
                for (int l = j; l < i; ++l) acc = fma(blk[l][i], X[0][j][l], acc);
                X[0][j][i] = -acc;
            }
        } else {  // upper with diagonal
            for (int i = 0; i < TR; ++i) X[1][j][i] = T(0);
            X[1][j][j] = T(1) / blk[j][j];
            for (int i = j - 1; i >= 0; --i) {
                T acc = T(0);
                for (int l = i + 1; l <= j; ++l) acc = fma(blk[l][i], X[1][j][l], acc);
                X[1][j][i] = -acc / blk[i][i];
            }
        }
    }
    __syncthreads();
    T* out = dinv + ((long long)b * nch_max + q) * 2 * TR * TR;
    T* tout = tri + ((long long)b * nch_max + q) * 2 * TR * TR;
    for (int idx = threadIdx.x; idx < 2 * TR * TR; idx += blockDim.x) {
        const int d = idx / (TR * TR), r = idx % (TR * TR), jj = r / TR, ii = r % TR;
        out[idx] = X[d][jj][ii];
        if (UL) continue;
        // the triangle itself (unit lower / upper with diagonal), for the substitution sweeps; the upper
        // triangle's unused strictly-lower slots carry 1/d_ii (tri_rcp_slot) for the quotient
        T v = d == 0 ? (jj < ii ? blk[jj][ii] : (jj == ii ? T(1) : T(0))) : (jj >= ii ? blk[jj][ii] : T(0));
        if (d == 1) {
            const int r = jj == 0 ? ii : -1;  // column 0 rows 1..TR-1 hold 1/d for rows 1..TR-1
            if (r >= 1) v = X[1][r][r];
            if (jj == TR - 2 && ii == TR - 1) v = X[1][0][0];  // 1/d_00
        }
        tout[idx] = v;
    }
    // infinity-norm condition estimate ||T|| ||T^{-1}|| of both triangles (max over chunks, as double bits)
    {
        const int d = threadIdx.x >> 5, i = threadIdx.x & 31;
        double rt = 0.0, ri = 0.0;
        if (i < TR && !skip)
            for (int jj = 0; jj < TR; ++jj) {
                const T tv = UL ? (d == 0 ? (jj <= i ? blk[jj][i] : T(0)) : (jj > i ? blk[jj][i] : (jj == i ? T(1) : T(0))))
                                : (d == 0 ? (jj < i ? blk[jj][i] : (jj == i ? T(1) : T(0))) : (jj >= i ? blk[jj][i] : T(0)));
                rt += fabs((double)tv);
                ri += fabs((double)X[d][jj][i]);
            }
        for (int o = 16; o > 0; o >>= 1) {
            rt = fmax(rt, __shfl_xor_sync(0xffffffffu, rt, o));
            ri = fmax(ri, __shfl_xor_sync(0xffffffffu, ri, o));
        }
        const double kap = rt * ri;
        if (i == 0 && isfinite(kap)) atomicMax(kappa_bits, (unsigned long long)__double_as_longlong(kap));
    }
}

// ---------------------------------------------------------------------------
#ifdef SAP_SWEEP_TRACE
__device__ long long g_sw_trace[24];
void read_sweep_trace(long long* out) { SAP_CUDA(cudaMemcpyFromSymbol(out, g_sw_trace, sizeof(long long) * 18)); }
#define SWT(var) long long var = clock64()
#else
#define SWT(var) do { } while (0)
#endif
// Row r's sum over the slab's CONTIGUOUS columns [c_lo, c_hi) against x (ring xs). The common case (no
// band-edge masking, no ring wrap) is two FMA chains over constant-offset shared loads: ~3 instructions
// per column. The sweep's per-chunk time is instruction-issue bound (ncu: helper loop stalls are
// not_selected / selected / wait), and warp 0's finishing step shares its SMSP with three helpers.
template <class T, int TR>
__device__ __forceinline__ T slab_range(const T* __restrict__ L, const T* __restrict__ xs, int xm, int cbase, int c_lo,
                                        int c_hi, int r, int k, bool fwd) {
    if (c_lo >= c_hi) return T(0);
    const bool masked = fwd ? (c_lo < TR) : (c_hi - 1 > k - TR + r || c_hi - 1 > k - TR);
    const int xb = (cbase + c_lo) & xm;
    if (!masked && xb + (c_hi - c_lo) <= xm + 1) {
        const T* __restrict__ xp = xs + xb - c_lo;  // xp[c] = x(cbase + c)
        const T* __restrict__ lp = L + r;           // lp[c * TR] = slab(r, c)
        T s0 = T(0), s1 = T(0);
        int c = c_lo;
#pragma unroll 4
        for (; c + 1 < c_hi; c += 2) {
            s0 = fma(lp[c * TR], xp[c], s0);
            s1 = fma(lp[(c + 1) * TR], xp[c + 1], s1);
        }
        if (c < c_hi) s0 = fma(lp[c * TR], xp[c], s0);
        return s0 + s1;
    }
    T s0 = T(0);
    for (int c = c_lo; c < c_hi; ++c) {
        const bool mk = fwd ? (c < TR && r > c) : (TR + c - r > k);
        s0 = fma(mk ? T(0) : L[c * TR + r], xs[(cbase + c) & xm], s0);
    }
    return s0;
}

// TR = 32 paired form: lane = (half h, row pair rp) -- rows rp, rp+1 of the slab in one 16-byte load, the
// half-warps h = 0/1 take the two halves of [c_lo, c_hi); sums of the two halves are combined by the
// caller. ~2 instructions per FMA instead of ~8 (the sweep is instruction-issue bound).
template <class T>
struct Vec2;
template <>
struct Vec2<double> {
    using type = double2;
};
template <>
struct Vec2<float> {
    using type = float2;
};
template <class T>
__device__ __forceinline__ void slab_range_pair(const T* __restrict__ L, const T* __restrict__ xs, int xm, int cbase,
                                                int c_lo, int c_hi, int lane, int k, bool fwd, T& s0, T& s1) {
    constexpr int TR = 32;
    const int h = lane >> 4, rp = (lane & 15) * 2;
    const int mid = c_lo + ((c_hi - c_lo + 1) >> 1);
    const int a = h ? mid : c_lo, b = h ? c_hi : mid;
    if (a >= b) return;
    const bool masked = fwd ? (a < TR) : (b - 1 > k - TR);
    const int xb = (cbase + a) & xm;
    if (!masked && xb + (b - a) <= xm + 1) {
        using V = typename Vec2<T>::type;
        const V* __restrict__ lp = reinterpret_cast<const V*>(L + rp);  // lp[c * 16] = rows rp, rp+1 of column c
        const T* __restrict__ xp = xs + xb - a;
        T t0 = T(0), t1 = T(0);
#pragma unroll 4
        for (int c = a; c < b; ++c) {
            const V v = lp[c * (TR / 2)];
            const T xv = xp[c];
            s0 = fma(v.x, xv, s0);
            s1 = fma(v.y, xv, s1);
        }
        (void)t0;
        (void)t1;
        return;
    }
    for (int c = a; c < b; ++c) {
        const T xv = xs[(cbase + c) & xm];
        const bool m0 = fwd ? (c < TR && rp > c) : (TR + c - rp > k);
        const bool m1 = fwd ? (c < TR && rp + 1 > c) : (TR + c - rp - 1 > k);
        s0 = fma(m0 ? T(0) : L[c * TR + rp], xv, s0);
        s1 = fma(m1 ? T(0) : L[c * TR + rp + 1], xv, s1);
    }
}

template <class T, int TR, int S>
struct SweepSmem {
    static constexpr int SD = S + 1;  // inverse ring outlives the slab by one chunk
};

// SUBST: the chunk's triangle T (bulk-loaded in place of D^{-1}) is solved by substitution on warp 0
// (32 broadcast steps; the reference's band_lu_solve order within the chunk, a / p as IEEE division).
// Chosen at setup when the chunk triangles are ill conditioned (element growth at low diagonal
// dominance, max ||T|| ||T^-1|| > 1e4): a product with an explicit inverse is not backward stable there
// and moves the Krylov iteration counts (measured: config 3 at d = 0.06, 20.25 vs the reference's 1.5);
// well-conditioned factors keep the 32x32 inverse mat-vec (one dependent step instead of 32).
// UL: a UL store (A = U'L'): the bottom-up sweep (unit upper U') runs first, then the top-down one (L' with
// its diagonal); the slabs are the LU sweeps' (strictly upper / strictly lower entries beyond the chunk),
// only the chunk inverses differ (k_chunk_inverses<UL>).
// tip_rows > 0: the second sweep stops once the tip_rows rows it reaches first are final (LU: the block's
// last rows, UL: its first rows) -- the SaP-C apply needs only those rows of its first block solve.
template <class T, int TR, int S, bool SUBST, bool UL>
__global__ void __launch_bounds__(kSwThreads, 1)
    k_sweep_tma(const __grid_constant__ CUtensorMap map, const T* __restrict__ dinv, int nch_max,
                const int* __restrict__ offs, int k, T* __restrict__ xbase, int xw, int slab_cols, int box_c,
                int nbox, const T* __restrict__ tri, const int* __restrict__ kbs, int tip_rows,
                const T* __restrict__ xsrc) {
    constexpr int SD = SweepSmem<T, TR, S>::SD;
    constexpr int CG = 32 / TR;  // column groups per warp
    constexpr int PF = 6;        // L2 prefetch distance (chunks)
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smraw);  // S barriers (128 B reserved)
    T* slab = reinterpret_cast<T*>(smraw + 128);
    const size_t slab_elems = (size_t)TR * slab_cols;
    T* dv = slab + S * slab_elems;                 // SD x TR*TR
    T* xs = dv + SD * TR * TR;                     // xw
    T* part = xs + xw;                             // kSwWarps x TR
    T* zb = part + kSwWarps * TR;                  // TR: warp 0's z broadcast

    const int b = blockIdx.x;
    const int off = offs[b], m = offs[b + 1] - off;
    // third stage: block b's own half-bandwidth K_b <= k (block_factors.hpp:155-180); its factor lives in the
    // k-wide store with zeros beyond K_b, so only the slab boxes and columns within K_b are loaded and summed
    const int kb = kbs ? min(max(kbs[b], 0), k) : k;
    const int qf0 = (k - kb) / box_c;          // forward: first box reaching a column in [k - kb, k)
    const int qb1 = (kb + box_c - 1) / box_c;  // backward: boxes covering columns [0, kb)
    T* x = xbase + off;
    // xsrc: the right-hand side when it is not x itself (the first sweep reads it, every sweep writes x)
    const T* x1 = xsrc ? xsrc + off : x;
    const int xm = xw - 1;
    const int nch = (m + TR - 1) / TR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane % TR, cg = lane / TR;
    const T* dvb = dinv + (long long)b * nch_max * 2 * TR * TR;
    const unsigned slab_bytes = (unsigned)(slab_elems * sizeof(T));
    const unsigned dv_bytes = (unsigned)(TR * TR * sizeof(T));
    // TMA producer: lane 0 of the last warp, which forms no phase-1 sums (issuing a slab's TMA takes ~500
    // cycles, measured; on a helper warp that delayed every chunk's phase 1)
    const bool producer = (warp == kSwWarps - 1 && lane == 0);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < xw; i += kSwThreads) xs[i] = T(0);
    __syncthreads();

    // g = global chunk sequence number (first sweep 0..nch-1, second nch..; LU: forward first, UL: backward)
    auto chunk_of = [&](int g, bool& fwd) {
        const bool first = g < nch;
        fwd = first != UL;
        const int q = first ? g : g - nch;
        return fwd ? q : nch - 1 - q;
    };
    auto issue = [&](int g) {
        bool fwd;
        const int ch = chunk_of(g, fwd);
        const int i0 = ch * TR;
        const int c0 = fwd ? i0 - k : i0 + TR;
        const int st = g % S;
#ifdef SAP_ABL_NOTMA
        if (g >= S) {  // timing study only: no slab traffic after the first ring pass (results invalid)
            mbar_expect_tx(bar + st, 0);
            return;
        }
#endif
        const int q0 = fwd ? qf0 : 0, q1 = fwd ? nbox : min(qb1, nbox);
        mbar_expect_tx(bar + st, (unsigned)(max(q1 - q0, 0) * TR * box_c * sizeof(T)) + dv_bytes);
        T* dst = slab + st * slab_elems;
        for (int q = q0; q < q1; ++q) tma_load_3d(dst + (size_t)q * TR * box_c, &map, i0, c0 + q * box_c, b, bar + st);
        const long long o = ((long long)ch * 2 + (fwd ? 0 : 1)) * TR * TR;
        bulk_load(dv + (g % SD) * TR * TR, (SUBST ? tri : dinv) + (long long)b * nch_max * 2 * TR * TR + o, dv_bytes,
                  bar + st);
    };
    auto prefetch = [&](int g) {
        bool fwd;
        const int ch = chunk_of(g, fwd);
        const int i0 = ch * TR;
        const int c0 = fwd ? i0 - k : i0 + TR;
        const int q0 = fwd ? qf0 : 0, q1 = fwd ? nbox : min(qb1, nbox);
        for (int q = q0; q < q1; ++q) tma_prefetch_3d(&map, i0, c0 + q * box_c, b);
    };

    for (int dir = 0; dir < 2; ++dir) {
        const bool fwd = (dir == 0) != UL;
        const int gbase = dir == 0 ? 0 : nch;
        // chunks this sweep finishes (all, or the second sweep's first tip_rows rows)
        const int nl = (dir == 1 && tip_rows > 0)
                           ? (fwd ? min(nch, (tip_rows + TR - 1) / TR) : nch - max(m - tip_rows, 0) / TR)
                           : nch;
        if (producer) {
            for (int q = 0; q < S - 1 && q < nl; ++q) issue(gbase + q);
            for (int q = S - 1; q < S - 1 + PF && q < nl; ++q) prefetch(gbase + q);
        }
        T yprev = T(0);  // y of the chunk warp 0 finishes next (warp 0 only)
        if (warp == 0) {
            const int ch0 = fwd ? 0 : nch - 1;
            const int in = ch0 * TR + lane;
            yprev = (lane < TR && in < m) ? (dir == 0 ? x1 : x)[in] : T(0);
        }
        int prev_rows = 0;
#ifdef SAP_SWEEP_TRACE
        long long acc_wait = 0, acc_p1 = 0, acc_p2 = 0, acc_a = 0, t_loop0 = clock64();
#endif
        for (int t = 0; t <= nl; ++t) {
            const int g = gbase + t;
            const int ch = fwd ? t : nch - 1 - t;   // chunk whose row sums are formed now
            const int pch = fwd ? t - 1 : nch - t;  // chunk finished now by warp 0
            SWT(tw0);
            if (t < nl) mbar_wait(bar + g % S, (unsigned)((g / S) & 1));
            SWT(tw1);
            __syncthreads();  // A
            SWT(tw2);
#ifdef SAP_SWEEP_TRACE
            acc_wait += tw1 - tw0;
            acc_a += tw2 - tw1;
#endif
            if (producer && t + S - 1 < nl) {
                issue(g + S - 1);
                if (t + S - 1 + PF < nl) prefetch(g + S - 1 + PF);
            }
            const T* L = slab + (g % S) * slab_elems;
            const int i0 = ch * TR;
            // ---- phase 1 ----
            T sA = T(0), sA2 = T(0);  // TR = 32: rows 2*(lane&15), +1 (paired form); else row r
            if (warp == 0) {
                if (t >= 1) {
                    const int p0 = pch * TR;
                    T z = T(0);
                    if (lane < TR) {
                        T t0 = T(0), t1 = T(0), t2 = T(0), t3 = T(0);
#pragma unroll
                        for (int q = 0; q < kSwWarps; q += 4) {
                            t0 += part[q * TR + lane];
                            t1 += part[(q + 1) * TR + lane];
                            t2 += part[(q + 2) * TR + lane];
                            t3 += part[(q + 3) * TR + lane];
                        }
                        z = yprev - ((t0 + t1) + (t2 + t3));
                    }
                    const T* D = dv + ((g - 1) % SD) * TR * TR;
                    T xv;
                    if constexpr (SUBST) {
                        // D holds the triangle itself: forward unit lower (column j after x_j), backward upper
                        T zz = z;
                        if (fwd) {
#pragma unroll 4
                            for (int jj = 0; jj < TR; ++jj) {
                                const T xj = __shfl_sync(0xffffffffu, zz, jj);
                                if (lane > jj && lane < TR) zz = fma(-D[jj * TR + lane], xj, zz);
                            }
                        } else {
                            // 1/d of this lane's row (precomputed, see k_chunk_inverses), quotient corrected
                            // once: the correctly rounded z / d of band_lu_solve without a 140-cycle
                            // division on each of the 32 dependent steps
                            const T dl = lane < TR ? D[lane * TR + lane] : T(1);
                            const T rl = lane < TR ? (lane == 0 ? D[(TR - 2) * TR + TR - 1] : D[lane]) : T(1);
#pragma unroll 4
                            for (int jj = TR - 1; jj >= 0; --jj) {
                                if (lane == jj) {
                                    const T q = zz * rl;
                                    zz = fma(fma(-q, dl, zz), rl, q);
                                }
                                const T xj = __shfl_sync(0xffffffffu, zz, jj);
                                if (lane < jj) zz = fma(-D[jj * TR + lane], xj, zz);
                            }
                        }
                        xv = zz;
                    } else {
                        // z broadcast through shared memory (measured: the SHFL version of this mat-vec
                        // was ~1.4K cycles of the ~2.1K-cycle chunk)
                        if (lane < TR) zb[lane] = z;
                        __syncwarp();
                        T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
                        if (lane < TR) {
#pragma unroll
                            for (int jj = 0; jj < TR; jj += 4) {
                                a0 = fma(D[jj * TR + lane], zb[jj], a0);
                                a1 = fma(D[(jj + 1) * TR + lane], zb[jj + 1], a1);
                                a2 = fma(D[(jj + 2) * TR + lane], zb[jj + 2], a2);
                                a3 = fma(D[(jj + 3) * TR + lane], zb[jj + 3], a3);
                            }
                        }
                        xv = (a0 + a1) + (a2 + a3);
                        __syncwarp();
                    }
                    if (lane < prev_rows) {
                        xs[(p0 + lane) & xm] = xv;
                        x[p0 + lane] = xv;
                    }
                }
                if (t < nl) {  // y of chunk ch, finished in the next iteration
                    const int in = i0 + lane;
                    yprev = (lane < TR && in < m) ? (dir == 0 ? x1 : x)[in] : T(0);
                    prev_rows = min(TR, m - i0);
                }
            } else if (t < nl && warp < kSwWarps - 1) {
                // columns needing only x older than chunk pch (within K_b)
                const int ca = fwd ? k - kb : TR, cb = fwd ? k - TR : kb;
                const int cbase = fwd ? i0 - k : i0 + TR;
                // contiguous column ranges: helper warp (warp-1) of 14, column group cg of CG
                if constexpr (TR == 32) {
                    const int nparts = kSwWarps - 2, part_id = warp - 1;
                    const int len = (cb - ca + nparts - 1) / nparts;
                    const int lo = ca + part_id * len, hi = min(lo + len, cb);
                    slab_range_pair<T>(L, xs, xm, cbase, lo, hi, lane, k, fwd, sA, sA2);
                } else {
                    const int nparts = (kSwWarps - 2) * CG, part_id = (warp - 1) * CG + cg;
                    const int len = (cb - ca + nparts - 1) / nparts;
                    const int lo = ca + part_id * len, hi = min(lo + len, cb);
                    sA = slab_range<T, TR>(L, xs, xm, cbase, lo, hi, r, k, fwd);
                }
            }
            SWT(tw3);
            __syncthreads();  // B
            SWT(tw4);
#ifdef SAP_SWEEP_TRACE
            acc_p1 += tw3 - tw2;
#endif
            // ---- phase 2: the TR columns of chunk pch ----
            if (t < nl) {
                const int ca = fwd ? max(max(k - TR, 0), k - kb) : 0, cb = fwd ? k : min(TR, kb);
                const int cbase = fwd ? i0 - k : i0 + TR;
                if constexpr (TR == 32) {
                    const int len = (cb - ca + kSwWarps - 1) / kSwWarps;
                    const int lo = ca + warp * len, hi = min(lo + len, cb);
                    slab_range_pair<T>(L, xs, xm, cbase, lo, hi, lane, k, fwd, sA, sA2);
                    sA += __shfl_xor_sync(0xffffffffu, sA, 16);
                    sA2 += __shfl_xor_sync(0xffffffffu, sA2, 16);
                    if (lane < 16) {
                        part[warp * TR + 2 * lane] = sA;
                        part[warp * TR + 2 * lane + 1] = sA2;
                    }
                } else {
                    const int nparts = kSwWarps * CG, part_id = warp * CG + cg;
                    const int len = (cb - ca + nparts - 1) / nparts;
                    const int lo = ca + part_id * len, hi = min(lo + len, cb);
                    const T sB = slab_range<T, TR>(L, xs, xm, cbase, lo, hi, r, k, fwd);
                    T s = sA + sB;
                    if constexpr (CG > 1) {
#pragma unroll
                        for (int o = TR; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    }
                    if (cg == 0) part[warp * TR + r] = s;
                }
            }
#ifdef SAP_SWEEP_TRACE
            acc_p2 += clock64() - tw4;
#endif
        }
#ifdef SAP_SWEEP_TRACE
        if (blockIdx.x == 0 && fwd && (tid == 0 || tid == 32 || tid == kSwThreads - 32)) {
            const int o = tid == 0 ? 0 : tid == 32 ? 6 : 12;
            g_sw_trace[o + 0] = clock64() - t_loop0;
            g_sw_trace[o + 1] = acc_wait;
            g_sw_trace[o + 2] = acc_a;
            g_sw_trace[o + 3] = acc_p1;
            g_sw_trace[o + 4] = acc_p2;
            g_sw_trace[o + 5] = nch;
        }
#endif
        __syncthreads();
        for (int i = tid; i < xw; i += kSwThreads) xs[i] = T(0);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Fallback sweep (k == 0, or bands too wide for the TMA ring): cp.async slabs,
// shuffle triangle solves. TR = 32.
template <class T, int S>
__global__ void __launch_bounds__(kSwThreads, 1)
    k_sweep_ldgsts(const T* __restrict__ f0, long long pstride, int pad, const int* __restrict__ offs, int k,
                   T* __restrict__ xbase, int xw) {
    constexpr int TR = 32;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int ncol = k + TR;
    T* ring = reinterpret_cast<T*>(smraw);
    T* xs = ring + (size_t)S * ncol * TR;
    T* part = xs + xw;
    const int b = blockIdx.x;
    const int off = offs[b], m = offs[b + 1] - off;
    const T* f = f0 + (long long)b * pstride + pad;
    T* x = xbase + off;
    const long long ld = 2LL * k;
    const int xm = xw - 1;
    const int nch = (m + TR - 1) / TR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < xw; i += kSwThreads) xs[i] = T(0);
    for (int dir = 0; dir < 2; ++dir) {
        const bool fwd = dir == 0;
        auto issue = [&](int t) {
            const int ch = fwd ? t : nch - 1 - t;
            T* dst = ring + (size_t)(t % S) * ncol * TR;
            const int i0 = ch * TR, c0 = fwd ? i0 - k : i0;
            for (int idx = tid; idx < ncol * TR; idx += kSwThreads) {
                const int cc = idx >> 5, rr = idx & 31;
                const int c = c0 + cc, i = i0 + rr;
                const bool ok = fwd ? (c >= 0 && i < m && c < i && i - c <= k) : (i < m && c < m && c >= i && c - i <= k);
                if (ok)
                    cp_async_elem(dst + idx, f + (long long)c * ld + i + k);
                else
                    dst[idx] = T(0);
            }
        };
        __syncthreads();
#pragma unroll
        for (int s = 0; s < S - 1; ++s) {
            if (s < nch) issue(s);
            cp_async_commit();
        }
        for (int t = 0; t < nch; ++t) {
            const int ch = fwd ? t : nch - 1 - t;
            cp_async_wait<S - 2>();
            __syncthreads();
            if (t + S - 1 < nch) issue(t + S - 1);
            cp_async_commit();
            const T* Lc = ring + (size_t)(t % S) * ncol * TR;
            const int i0 = ch * TR;
            T s = T(0);
            if (fwd) {
                for (int cc = warp; cc < k; cc += kSwWarps) s = fma(Lc[cc * TR + lane], xs[(i0 - k + cc) & xm], s);
            } else {
                for (int cc = TR + warp; cc < ncol; cc += kSwWarps) s = fma(Lc[cc * TR + lane], xs[(i0 + cc) & xm], s);
            }
            part[warp * 33 + lane] = s;
            __syncthreads();
            if (warp == 0) {
                T tot = T(0);
#pragma unroll
                for (int q = 0; q < kSwWarps; ++q) tot += part[q * 33 + lane];
                const int rows = min(TR, m - i0);
                T y = lane < rows ? x[i0 + lane] - tot : T(0);
                if (fwd) {
                    const T* tri = Lc + (size_t)k * TR;
                    for (int jj = 0; jj < rows; ++jj) {
                        const T xj = __shfl_sync(0xffffffffu, y, jj);
                        if (lane > jj) y = fma(-tri[jj * TR + lane], xj, y);
                    }
                } else {
                    for (int jj = rows - 1; jj >= 0; --jj) {
                        if (lane == jj) y = y / Lc[jj * TR + jj];
                        const T xj = __shfl_sync(0xffffffffu, y, jj);
                        if (lane < jj) y = fma(-Lc[jj * TR + lane], xj, y);
                    }
                }
                if (lane < rows) {
                    xs[(i0 + lane) & xm] = y;
                    x[i0 + lane] = y;
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();
        for (int i = tid; i < xw; i += kSwThreads) xs[i] = T(0);
    }
}

// ---------------------------------------------------------------------------
static int pow2_at_least(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        SAP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaFailure("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

template <class T, int TR, int S>
static size_t tma_smem_bytes(int slab_cols, int xw) {
    return 128 + sizeof(T) * ((size_t)S * TR * slab_cols + (size_t)(S + 1) * TR * TR + xw + (kSwWarps + 1) * TR);
}

template <class T>
static void choose_tma(SweepPlan<T>& pl) {
    pl.tma = false;
    const int k = pl.k;
    if (k < 1) return;
    const int xw = pow2_at_least(k + 96);
    pl.xw = xw;
    for (int tr : {32, 16}) {
        const int nbox = (k + 255) / 256;
        const int box_c = ((k + nbox - 1) / nbox + 7) / 8 * 8;
        const int cols = box_c * nbox;
        for (int s : {3, 2}) {
            size_t bytes = 0;
            if (tr == 32)
                bytes = s == 3 ? tma_smem_bytes<T, 32, 3>(cols, xw) : tma_smem_bytes<T, 32, 2>(cols, xw);
            else
                bytes = s == 3 ? tma_smem_bytes<T, 16, 3>(cols, xw) : tma_smem_bytes<T, 16, 2>(cols, xw);
            if (bytes <= 225 * 1024) {
                pl.tma = true;
                pl.tr = tr;
                pl.stages = s;
                pl.nbox = nbox;
                pl.box_c = box_c;
                pl.smem = bytes;
                return;
            }
        }
    }
}

template <class T>
void plan_sweeps(SweepPlan<T>& pl, T* dinv_storage) {
    choose_tma(pl);
    if (!pl.tma) return;
    const int tr = pl.tr;
    pl.nch_max = (pl.st.m_max + tr - 1) / tr;
    pl.dinv = dinv_storage;
    pl.tri = dinv_storage + (size_t)pl.p * pl.nch_max * 2 * tr * tr;
    // overlapping 3-D view: (row i, column c, block b) -> base + b*pstride + pad + k + c*2k + i
    cuuint64_t dims[3] = {(cuuint64_t)pl.st.m_max, (cuuint64_t)pl.st.m_max, (cuuint64_t)pl.p};
    cuuint64_t strides[2] = {(cuuint64_t)2 * pl.k * sizeof(T), (cuuint64_t)pl.st.pstride * sizeof(T)};
    cuuint32_t box[3] = {(cuuint32_t)tr, (cuuint32_t)pl.box_c, 1};
    cuuint32_t es[3] = {1, 1, 1};
    void* base = const_cast<T*>(pl.f) + pl.st.pad + pl.k;
    const CUresult rc = encode_fn()(&pl.map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                    3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) {
        pl.tma = false;
        return;
    }
}
template void plan_sweeps<double>(SweepPlan<double>&, double*);
template void plan_sweeps<float>(SweepPlan<float>&, float*);

template <class T>
size_t sweep_dinv_elems(const SweepPlan<T>& pl) {
    SweepPlan<T> tmp = pl;
    choose_tma(tmp);
    if (!tmp.tma) return 0;
    const int nch_max = (pl.st.m_max + tmp.tr - 1) / tmp.tr;
    return 2 * (size_t)pl.p * nch_max * 2 * tmp.tr * tmp.tr;  // inverses, then the triangles (substitution)
}
template size_t sweep_dinv_elems<double>(const SweepPlan<double>&);
template size_t sweep_dinv_elems<float>(const SweepPlan<float>&);

template <class T>
void launch_chunk_inverses(const SweepPlan<T>& pl, cudaStream_t s) {
    if (!pl.tma) return;
    dim3 grid(pl.nch_max, pl.p);
    if (pl.ul && pl.tr != 32) throw InvalidArgument("UL sweeps need 32-row chunks");
    if (pl.ul)
        k_chunk_inverses<T, 32, true><<<grid, 64, 0, s>>>(pl.f, pl.st.pstride, pl.st.pad, pl.offs, pl.k, pl.dinv,
                                                          pl.nch_max, pl.tri, pl.kappa);
    else if (pl.tr == 32)
        k_chunk_inverses<T, 32><<<grid, 64, 0, s>>>(pl.f, pl.st.pstride, pl.st.pad, pl.offs, pl.k, pl.dinv, pl.nch_max,
                                                    pl.tri, pl.kappa);
    else
        k_chunk_inverses<T, 16><<<grid, 64, 0, s>>>(pl.f, pl.st.pstride, pl.st.pad, pl.offs, pl.k, pl.dinv, pl.nch_max,
                                                    pl.tri, pl.kappa);
    SAP_LAUNCHED();
}
template void launch_chunk_inverses<double>(const SweepPlan<double>&, cudaStream_t);
template void launch_chunk_inverses<float>(const SweepPlan<float>&, cudaStream_t);

template <class T, int TR, int S>
static void run_tma(const SweepPlan<T>& pl, T* x, int tip_rows, const T* xsrc, cudaStream_t s) {
    const int cols = pl.box_c * pl.nbox;
    auto kern = pl.ul ? k_sweep_tma<T, TR, S, false, true>
                      : (pl.subst ? k_sweep_tma<T, TR, S, true, false> : k_sweep_tma<T, TR, S, false, false>);
    SAP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    kern<<<pl.p, kSwThreads, pl.smem, s>>>(pl.map, pl.dinv, pl.nch_max, pl.offs, pl.k, x, pl.xw, cols, pl.box_c,
                                           pl.nbox, pl.tri, pl.kb, tip_rows, xsrc);
    SAP_LAUNCHED();
}

template <class T, int S>
static bool try_ldgsts(const SweepPlan<T>& pl, T* x, cudaStream_t s) {
    const int xw = pow2_at_least(pl.k + 64);
    const size_t bytes = sizeof(T) * ((size_t)S * (pl.k + 32) * 32 + xw + kSwWarps * 33);
    if (bytes > 200 * 1024) return false;
    SAP_CUDA(cudaFuncSetAttribute(k_sweep_ldgsts<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_sweep_ldgsts<T, S><<<pl.p, kSwThreads, bytes, s>>>(pl.f, pl.st.pstride, pl.st.pad, pl.offs, pl.k, x, xw);
    SAP_LAUNCHED();
    return true;
}

template <class T>
void launch_block_solve(const SweepPlan<T>& pl, T* x, cudaStream_t s, int tip_rows, const T* xsrc) {
    if (pl.p <= 0) return;
    if (xsrc && !pl.tma) throw InvalidArgument("out-of-place band solve needs the TMA sweep");  // fallback: in place
    if ((pl.ul || tip_rows > 0) && !(pl.tma && pl.tr == 32 && !pl.subst && !pl.kb))
        throw InvalidArgument("tip sweeps need the 32-row inverse-product TMA path");
    if (pl.tma) {
        if (pl.tr == 32)
            pl.stages == 3 ? run_tma<T, 32, 3>(pl, x, tip_rows, xsrc, s) : run_tma<T, 32, 2>(pl, x, tip_rows, xsrc, s);
        else
            pl.stages == 3 ? run_tma<T, 16, 3>(pl, x, tip_rows, xsrc, s) : run_tma<T, 16, 2>(pl, x, tip_rows, xsrc, s);
        return;
    }
    if (try_ldgsts<T, 4>(pl, x, s)) return;
    if (try_ldgsts<T, 3>(pl, x, s)) return;
    if (try_ldgsts<T, 2>(pl, x, s)) return;
    throw InvalidArgument("band solve: half-bandwidth too large for the shared-memory chunk ring");
}
template void launch_block_solve<double>(const SweepPlan<double>&, double*, cudaStream_t, int, const double*);
template void launch_block_solve<float>(const SweepPlan<float>&, float*, cudaStream_t, int, const float*);

// ---------------------------------------------------------------------------
// SaP-C interface step (spike.hpp:323-347), split into wide GEMV kernels:
//   pre   : XT[t] = g[e:e+w] - W^t_t g[e-w:e]
//   solve : rbar_t XT[t] = ... (band sweep over the reduced blocks)
//   post1 : XB[t] = g[e-w:e] - V^b_t XT[t];  b2[e-w:e] -= B_t XT[t]
//   post2 : b2[e:e+w] -= C_t XB[t]
// A warp owns one output row (lanes stride the row, fixed-order shuffle tree).
template <class T>
__device__ __forceinline__ T row_dot(const T* __restrict__ a, const T* __restrict__ v, int w, int lane) {
    T acc = T(0);
    int j0 = 0;
    // a lane's terms 8 at a time, all loads in flight before the (same-order) FMA chain
    for (; j0 + 8 * 32 <= w; j0 += 8 * 32) {
        T av[8], vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            av[u] = a[j0 + lane + 32 * u];
            vv[u] = v[j0 + lane + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(av[u], vv[u], acc);
    }
    {
        T av[8], vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + lane + 32 * u;
            av[u] = j < w ? a[j] : T(0);
            vv[u] = j < w ? v[j] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j0 + lane + 32 * u < w) acc = fma(av[u], vv[u], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
}

// g: the first block solve's bottom rows of block t (g[e-w, e)); gt: its top rows of block t+1 (gt[e, e+w))
template <class T>
__global__ void k_iface_pre(const T* __restrict__ g, const T* __restrict__ gt, const int* __restrict__ offs, int w,
                            const T* __restrict__ wt, T* __restrict__ xt) {
    const int t = blockIdx.y, lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= w) return;
    const int e = offs[t + 1];
    const T acc = row_dot(wt + ((size_t)t * w + i) * w, g + e - w, w, lane);
    if (lane == 0) xt[(size_t)t * w + i] = gt[e + i] - acc;
}

template <class T>
__global__ void k_iface_post1(const T* __restrict__ g, const int* __restrict__ offs, int w, const T* __restrict__ vb,
                              const T* __restrict__ bblk, const T* __restrict__ xt, T* __restrict__ xb,
                              T* __restrict__ b2, int skip_first_b) {
    const int t = blockIdx.y, lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= w) return;
    if (blockIdx.z == 1 && t == 0 && skip_first_b) return;  // left rank's rows (multi-GPU cross interface)
    const int e = offs[t + 1];
    const T* v = xt + (size_t)t * w;
    if (blockIdx.z == 0) {
        const T acc = row_dot(vb + ((size_t)t * w + i) * w, v, w, lane);
        if (lane == 0) xb[(size_t)t * w + i] = g[e - w + i] - acc;
    } else {
        const T acc = row_dot(bblk + ((size_t)t * w + i) * w, v, w, lane);
        if (lane == 0) b2[e - w + i] -= acc;
    }
}

template <class T>
__global__ void k_iface_post2(const int* __restrict__ offs, int w, const T* __restrict__ cblk,
                              const T* __restrict__ xb, T* __restrict__ b2, int skip_last) {
    const int t = blockIdx.y, lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= w) return;
    if (t == (int)gridDim.y - 1 && skip_last) return;  // right rank's rows (multi-GPU cross interface)
    const int e = offs[t + 1];
    const T acc = row_dot(cblk + ((size_t)t * w + i) * w, xb + (size_t)t * w, w, lane);
    if (lane == 0) b2[e + i] -= acc;
}

template <class T>
void launch_interfaces(const T* g, const int* d_ioffs, const SweepPlan<T>& rplan, int ni, int k, const T* wt,
                       const T* vb, const T* bblk, const T* cblk, T* xt, T* xb, T* b2, bool skip_first_b,
                       bool skip_last_c, cudaStream_t s, const T* gtop) {
    if (ni < 1 || k == 0) return;
    const int w = k;
    dim3 grid(ceil_div(w, 8), ni);
    k_iface_pre<T><<<grid, 256, 0, s>>>(g, gtop ? gtop : g, d_ioffs, w, wt, xt);
    SAP_LAUNCHED();
    launch_block_solve<T>(rplan, xt, s);
    k_iface_post1<T><<<dim3(grid.x, ni, 2), 256, 0, s>>>(g, d_ioffs, w, vb, bblk, xt, xb, b2, skip_first_b);
    SAP_LAUNCHED();
    k_iface_post2<T><<<grid, 256, 0, s>>>(d_ioffs, w, cblk, xb, b2, skip_last_c);
    SAP_LAUNCHED();
}
template void launch_interfaces<double>(const double*, const int*, const SweepPlan<double>&, int, int, const double*,
                                        const double*, const double*, const double*, double*, double*, double*, bool,
                                        bool, cudaStream_t, const double*);
template void launch_interfaces<float>(const float*, const int*, const SweepPlan<float>&, int, int, const float*,
                                       const float*, const float*, const float*, float*, float*, float*, bool, bool,
                                       cudaStream_t, const float*);

// ---------------------------------------------------------------------------
// Diagonal preconditioner (build_precond_op's `diagonal` branch, pipeline.hpp:151-161).
// T = float: the band entries and the boost value rounded to float (banded_cast, pipeline.hpp:150-152); the
// float diagonal is stored exactly in double.
template <class T>
__global__ void k_boosted_diag(const double* __restrict__ a, int n, int k, const double* __restrict__ scale,
                               double eps, double* __restrict__ diag) {
    const double sc = *scale;
    const T bv = static_cast<T>(eps * (sc > 0 ? sc : 1.0));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        T d = static_cast<T>(a[(long long)i * (2 * k + 1) + k]);
        if (fabs(d) < bv) d = d < T(0) ? -bv : bv;
        diag[i] = static_cast<double>(d);
    }
}

void launch_boosted_diag(const double* band, int n, int k, const double* scale, double boost_eps, double* diag,
                         cudaStream_t s, bool f32) {
    (f32 ? k_boosted_diag<float> : k_boosted_diag<double>)<<<ceil_div(n, 256), 256, 0, s>>>(band, n, k, scale,
                                                                                            boost_eps, diag);
    SAP_LAUNCHED();
}

template <class T>
__global__ void k_diag_apply(const double* __restrict__ in, const double* __restrict__ diag,
                             double* __restrict__ out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = static_cast<double>(static_cast<T>(in[i]) / static_cast<T>(diag[i]));
}

void launch_diag_apply(const double* in, const double* diag, double* out, int n, cudaStream_t s, bool f32) {
    (f32 ? k_diag_apply<float> : k_diag_apply<double>)<<<ceil_div(n, 256), 256, 0, s>>>(in, diag, out, n);
    SAP_LAUNCHED();
}

}  // namespace sapgpu
