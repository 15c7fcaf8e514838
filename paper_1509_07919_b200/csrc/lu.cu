// Blocked band LU (the hot loop of factor_blocks) on FP64 tensor cores.
//
// Reference: band_lu_inplace / band_ul_inplace, proj/include/sap/block_factors.hpp:22-71;
// dense_lu_nopivot_boosted, proj/include/sap/spike.hpp:20-45 (same strided job
// views as factor.cu: LU, UL on the flipped system, and the reduced blocks).
//
// One CTA per factorization job, panel width B = 32. k_band_lu_res (K <= 224): panel and U12 resident
// in shared memory, trailing update A22 -= L21 U12 on DMMA.8x8x4 (mma.sync m8n8k4) with A22 streamed
// through L2. k_band_lu_seq: the same steps with the panel staged per step (K up to
// the shared-memory budget). Every element receives its rank-1 updates in the reference's column order
// (DMMA / DFMA contract mul+sub). Measured-slower variants (warp-specialized look-ahead,
// extended-row update) are in the git history (commit 4e449e9), not in the product library.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"


namespace sapgpu {

namespace {

constexpr int kLuThreads = 512;
constexpr int kPgWarps = 8;
constexpr int kPgThreads = kPgWarps * 32;
constexpr int kBarPg = 1;   // named barrier: panel group (256 threads)

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

struct Lu {
    double* base;
    long long rs, cs;
    int m, K, B, pld, uld;
    double bv;
    const double* src;  // unfactored entries (k_band_lu_res reads every never-updated entry from here)
    __device__ __forceinline__ double* at(int i, int c) const { return base + (long long)i * rs + (long long)c * cs; }
    __device__ __forceinline__ const double* src_at(int i, int c) const {
        return src + (long long)i * rs + (long long)c * cs;
    }
    __device__ __forceinline__ bool inband(int i, int c) const { return i - c <= K && c - i <= K; }
};

// C -= L21 * U12 over A22 tiles rows [r_lo, r_hi) x cols [c_lo, c_hi) (A22 coordinates, origin (ja, ja)).
// Warp tiles are 16 x 32, enumerated row-major; this warp takes every nw-th from widx.
// The MMA computes the transposed tile C^T -= U12^T L21^T (m8n8k4 row.col:
// A' = U12^T fragment, B' = -L21^T fragment) so that each thread's two
// accumulator elements are rows (i, i+1) of one column: adjacent in the
// tall-thin band (|rs| == 1), moved with one 16-byte access when aligned.
// Tiles are software-pipelined: the next tile's accumulators load while the
// current tile computes. Pn != nullptr: results go to the next panel buffer.
// A DMMA update region: region rows [r_lo, r_hi) x cols [c_lo, c_hi), region
// (i, c) = global (row_org + i, col_org + c); the B' operand row of region row
// i is P[poff + i]. Region rows i < band_top are panel rows whose entries are
// in the band only when nbk + c - i <= K (masked on load and store).
// Pn != nullptr: results go to smem Pn[c*pld + i - dst_off] instead of global.
struct TileCtx {
    int r_lo, r_hi, c_lo, c_hi, tcols;
    int row_org, col_org, poff, band_top, nbk, dst_off;
};
constexpr int kTileR = 16, kTileC = 32;  // warp tile: 2 x 4 DMMA tiles
constexpr int kTQ = kTileC / 8;

// L2 residency of the trailing-update window: the A22 tiles go out and come back every step, so their
// loads / stores carry an evict_last policy; the final factor columns (written once) stream out with .cs.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_keep2(const double* a) {
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(l2_keep_policy()));
    return v;
}
__device__ __forceinline__ double ld_keep(const double* a) {
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(l2_keep_policy()));
    return v;
}
__device__ __forceinline__ void st_keep2(double* a, double2 v) {
    asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y),
                 "l"(l2_keep_policy()) : "memory");
}
__device__ __forceinline__ void st_keep(double* a, double v) {
    asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(l2_keep_policy()) : "memory");
}

// final factor entries that were last written with evict_last: stored with evict_first so that the
// priority does not stay on lines the factorization is done with (the L2 would fill with them)
__device__ __forceinline__ unsigned long long l2_first_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_first(double* a, double v) {
    asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(l2_first_policy()) : "memory");
}
__device__ __forceinline__ unsigned long long l2_normal_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_normal(double* a, double v) {
    asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(l2_normal_policy()) : "memory");
}

__device__ __forceinline__ bool tile_ok(const Lu& L, const TileCtx& T, int i, int c) {
    return i < T.r_hi && c < T.c_hi && (i >= T.band_top || T.nbk + c - i <= L.K);
}

__device__ __forceinline__ void tile_load(const Lu& L, const TileCtx& T, int t, double (&acc)[2][kTQ][2]) {
    const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int row0 = T.r_lo + (t / T.tcols) * kTileR, col0 = T.c_lo + (t % T.tcols) * kTileC;
    const int ib = row0 + 2 * lc, cb = col0 + lr;
    const long long rs = L.rs, ra8 = 8 * rs, cq8 = 8 * L.cs;
    const double* p00 = L.at(T.row_org + ib, T.col_org + cb);
    const double* lo00 = rs > 0 ? p00 : p00 - 1;
    const bool full = row0 + kTileR <= T.r_hi && col0 + kTileC <= T.c_hi && row0 >= T.band_top;
    if (full && (rs == 1 || rs == -1) && ((reinterpret_cast<uintptr_t>(lo00) & 15) == 0)) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q) {
                const double2 v = ld_keep2(lo00 + a * ra8 + q * cq8);
                acc[a][q][0] = rs > 0 ? v.x : v.y;
                acc[a][q][1] = rs > 0 ? v.y : v.x;
            }
    } else {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = ib + a * 8 + e, c = cb + q * 8;
                    acc[a][q][e] = tile_ok(L, T, i, c) ? ld_keep(p00 + a * ra8 + e * rs + q * cq8) : 0.0;
                }
    }
}

__device__ __forceinline__ void tile_compute_store(const Lu& L, const TileCtx& T, int t, double (&acc)[2][kTQ][2],
                                                   const double* __restrict__ P, const double* __restrict__ U, int nb,
                                                   double* Pn) {
    const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int row0 = T.r_lo + (t / T.tcols) * kTileR, col0 = T.c_lo + (t % T.tcols) * kTileC;
    const int ib = row0 + 2 * lc, cb = col0 + lr;
    const int pld = L.pld, uld = L.uld;
    const int ksteps = (nb + 3) >> 2;
    const bool a1 = row0 + 8 < T.r_hi;
    bool qv[kTQ];
#pragma unroll
    for (int q = 0; q < kTQ; ++q) qv[q] = col0 + q * 8 < T.c_hi;
    const double* pk = P + T.poff + row0 + lr;
    const double* uk = U + col0 + lr;
    for (int ks = 0; ks < ksteps; ++ks) {
        const int kk = ks * 4 + lc;
        const double b0 = -pk[kk * pld];
        const double b1 = -pk[kk * pld + 8];
#pragma unroll
        for (int q = 0; q < kTQ; ++q) {
            if (qv[q]) {
                const double aq = uk[kk * uld + q * 8];
                dmma_m8n8k4(acc[0][q][0], acc[0][q][1], aq, b0, acc[0][q][0], acc[0][q][1]);
                if (a1) dmma_m8n8k4(acc[1][q][0], acc[1][q][1], aq, b1, acc[1][q][0], acc[1][q][1]);
            }
        }
    }
    if (Pn) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = ib + a * 8 + e, c = cb + q * 8;
                    if (tile_ok(L, T, i, c)) Pn[c * pld + i - T.dst_off] = acc[a][q][e];
                }
        return;
    }
    const long long rs = L.rs, ra8 = 8 * rs, cq8 = 8 * L.cs;
    double* p00 = L.at(T.row_org + ib, T.col_org + cb);
    double* lo00 = rs > 0 ? p00 : p00 - 1;
    const bool full = row0 + kTileR <= T.r_hi && col0 + kTileC <= T.c_hi && row0 >= T.band_top;
    if (full && (rs == 1 || rs == -1) && ((reinterpret_cast<uintptr_t>(lo00) & 15) == 0)) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q) {
                double2 v;
                v.x = rs > 0 ? acc[a][q][0] : acc[a][q][1];
                v.y = rs > 0 ? acc[a][q][1] : acc[a][q][0];
                __stcg(reinterpret_cast<double2*>(lo00 + a * ra8 + q * cq8), v);
            }
    } else {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = ib + a * 8 + e, c = cb + q * 8;
                    if (tile_ok(L, T, i, c)) __stcg(p00 + a * ra8 + e * rs + q * cq8, acc[a][q][e]);
                }
    }
}

__device__ __noinline__ void dmma_tiles(const Lu& L, const TileCtx& T, const double* __restrict__ P,
                                        const double* __restrict__ U, int nb, int widx, int nw, double* Pn) {
    if (T.r_lo >= T.r_hi || T.c_lo >= T.c_hi) return;
    const int ntiles = ((T.r_hi - T.r_lo + kTileR - 1) / kTileR) * T.tcols;
    double A[2][kTQ][2];
    for (int t = widx; t < ntiles; t += nw) {
        tile_load(L, T, t, A);
        tile_compute_store(L, T, t, A, P, U, nb, Pn);
    }
}

__device__ __forceinline__ TileCtx make_tiles(int r_lo, int r_hi, int c_lo, int c_hi, int row_org, int col_org,
                                              int poff, int band_top, int nbk, int dst_off) {
    return TileCtx{r_lo, r_hi, c_lo, c_hi, (c_hi - c_lo + kTileC - 1) / kTileC, row_org, col_org, poff, band_top, nbk,
                   dst_off};
}

// The classic A22 region (origin (ja, ja), B' rows offset by nb).
__device__ __forceinline__ void dmma_region(const Lu& L, const double* __restrict__ P, const double* __restrict__ U,
                                            int nb, int ja, int r_lo, int r_hi, int c_lo, int c_hi, int widx, int nw,
                                            double* Pn) {
    dmma_tiles(L, make_tiles(r_lo, r_hi, c_lo, c_hi, ja, ja, nb, 0, 0, 0), P, U, nb, widx, nw, Pn);
}

// Panel group: stage the parts of panel (jp, np) that phase (a) did not
// produce (rows >= ra or columns >= ca), zero everything outside the band.
__device__ __forceinline__ void pg_stage_panel(const Lu& L, double* Pn, int jp, int np, int ph, int ra, int ca,
                                               int ptid) {
    const int pld = L.pld;
    for (int r = ptid; r < pld; r += kPgThreads)
        for (int c = 0; c < L.B; ++c) {
            if (c < np && r < ph && r < ra && c < ca) continue;  // written by phase (a)
            if (c < np && r < ph && L.inband(r, c))
                cp_async8(Pn + c * pld + r, L.at(jp + r, jp + c));
            else
                Pn[c * pld + r] = 0.0;
        }
    cp_async_wait_all();
}

// Panel group: unblocked factorization of the staged panel. Thread ptid owns
// panel row ptid (ph <= kPgThreads) in registers; per column the pivot row's
// owner publishes it (double-buffered) and one named barrier follows.
// Panel group: unblocked factorization of the staged panel. Thread ptid owns
// panel row ptid (ph <= kPgThreads; its entries Pn[c*pld + ptid] are private
// to it, conflict-free). Per column the pivot row's owner publishes it with
// the reciprocal of the (boosted) pivot, double buffered, then one named
// barrier; multipliers are l = a * (1/p).
// Panel group: unblocked factorization of the staged panel. Thread ptid owns
// panel row ptid (ph <= kPgThreads) in REGISTERS (compile-time column
// indices). Per column the owner of the pivot row boosts the pivot
// (block_factors.hpp:26-34) and publishes 1/p and the row's remaining entries
// (double-buffered smem), right after updating that row so the division
// overlaps the other rows' work; one named barrier per column; l = a * (1/p).
// 1/p without the IEEE division routine: MUFU.RCP64H seed + three Newton steps
// (~2^-23 -> full double precision; the multipliers l = a * (1/p) already
// differ from the reference's a / p by rounding only).
__device__ __forceinline__ double fast_rcp(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    return fma(r, e, r);
}

// a / p from a precomputed 1/p: q = a * (1/p) plus one residual correction (e = a - q p exactly by FMA,
// q += e * (1/p)) -- the correctly rounded quotient in all but rare ties, i.e. the reference's l = a / p
// (block_factors.hpp:36), not a * (1/p) with its second rounding (growth at low d amplifies the difference).
__device__ __forceinline__ double div_rcp(double a, double p, double rc) {
    const double q = a * rc;
    return fma(fma(-q, p, a), rc, q);
}

template <int B, int C>
__device__ __forceinline__ double pg_recip(const Lu& L, double (&row)[B], int* boost_ctr) {
    double p = row[C];
    if (fabs(p) < L.bv) {
        p = p < 0.0 ? -L.bv : L.bv;
        row[C] = p;
        atomicAdd(boost_ctr, 1);
    }
    return fast_rcp(p);
}

// prow layout per buffer (B + 2 doubles, 16-byte aligned): [0] = 1/p, [2 + cc] = row entry cc
template <int B>
struct Prow {
    static constexpr int kStride = B + 2;
};

template <int B, int C>
__device__ __forceinline__ void pg_pub(const double (&row)[B], double rcp, double* __restrict__ prow) {
    double* __restrict__ pr = prow + (C & 1) * Prow<B>::kStride;
    pr[0] = rcp;
    constexpr int c0 = (C + 1) & ~1;  // publish pairs from an even column
#pragma unroll
    for (int cc = c0; cc < B; cc += 2) {
        double2 v;
        v.x = row[cc];
        v.y = cc + 1 < B ? row[cc + 1] : 0.0;
        *reinterpret_cast<double2*>(pr + 2 + cc) = v;
    }
}

template <int B, int C>
__device__ __forceinline__ void pg_col(const Lu& L, double (&row)[B], double* __restrict__ prow, int* boost_ctr,
                                       int np, int ph, int ptid) {
    if constexpr (C < B) {
        if (C < np) {
            named_sync(kBarPg, kPgThreads);
            const double* __restrict__ pr = prow + (C & 1) * Prow<B>::kStride;
            if (ptid > C && ptid < ph) {
                double u[B];
                constexpr int c0 = (C + 1) & ~1;
#pragma unroll
                for (int cc = c0; cc < B; cc += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(pr + 2 + cc);
                    u[cc] = v.x;
                    if (cc + 1 < B) u[cc + 1] = v.y;
                }
                const double l = row[C] * pr[0];
                row[C] = l;
                if constexpr (C + 1 < B) {
                    row[C + 1] = fma(-l, u[C + 1], row[C + 1]);
                    // the next pivot's owner starts its reciprocal now; its row is published
                    // only after the whole update of this column
                    const bool owner = ptid == C + 1 && C + 1 < np;
                    double rcp = 0.0;
                    if (owner) rcp = pg_recip<B, C + 1>(L, row, boost_ctr);
#pragma unroll
                    for (int cc = C + 2; cc < B; ++cc) row[cc] = fma(-l, u[cc], row[cc]);
                    if (owner) pg_pub<B, C + 1>(row, rcp, prow);
                }
            }
            pg_col<B, C + 1>(L, row, prow, boost_ctr, np, ph, ptid);
        }
    }
}

template <int B>
__device__ __noinline__ void pg_factor_panel(const Lu& L, double* __restrict__ Pn, double* __restrict__ prow,
                                             int* boost_ctr, int np, int ph, int ptid) {
    const int pld = L.pld;
    double row[B];
#pragma unroll
    for (int c = 0; c < B; ++c) row[c] = ptid < ph ? Pn[c * pld + ptid] : 0.0;
    if (ptid == 0 && np > 0) pg_pub<B, 0>(row, pg_recip<B, 0>(L, row, boost_ctr), prow);
    pg_col<B, 0>(L, row, prow, boost_ctr, np, ph, ptid);
    if (ptid < ph) {
#pragma unroll
        for (int c = 0; c < B; ++c) Pn[c * pld + ptid] = row[c];
    }
    named_sync(kBarPg, kPgThreads);
}

__device__ __forceinline__ void pg_store_panel(const Lu& L, const double* Pn, int jp, int np, int ph, int ptid) {
    const int pld = L.pld;
    for (int r = ptid; r < ph; r += kPgThreads)
        for (int c = 0; c < np; ++c)
            if (L.inband(r, c)) __stcg(L.at(jp + r, jp + c), Pn[c * pld + r]);
}

// Panel group: U12 of panel (jp, np): rows [0, np) x cols [0, Rn) at (jp, jp+np),
// staged from global, solved with the panel's unit-lower L11 (thread = column,
// register accumulators; element (r, c) receives j = 0..r-1 in order as in
// block_factors.hpp:246-250), written back.
template <int B>
__device__ __noinline__ void pg_u12(const Lu& L, const double* __restrict__ Pn, double* __restrict__ Un, int jp, int np,
                                    int Rn, int ptid) {
    constexpr int H = 8;
    static_assert(B % H == 0, "B must be a multiple of 8");
    const int pld = L.pld, uld = L.uld;
    for (int idx = ptid; idx < 32 * uld; idx += kPgThreads) {
        const int r = idx & 31, c = idx >> 5;  // lanes walk a column: contiguous in the band
        if (r >= B) continue;
        if (r < np && c < Rn && np + c - r <= L.K)
            cp_async8(Un + r * uld + c, L.at(jp + r, jp + np + c));
        else
            Un[r * uld + c] = 0.0;
    }
    cp_async_wait_all();
    named_sync(kBarPg, kPgThreads);
    // element (r, c) receives j = 0..r-1 in ascending order (block_factors.hpp:246-250);
    // rows in blocks of H: contributions of the solved rows above, then the block's own triangle
    for (int c = ptid; c < Rn; c += kPgThreads) {
#pragma unroll 1
        for (int b0 = 0; b0 < B; b0 += H) {
            double x[H];
#pragma unroll
            for (int r = 0; r < H; ++r) x[r] = Un[(b0 + r) * uld + c];
#pragma unroll 4
            for (int j = 0; j < b0; ++j) {
                const double uj = Un[j * uld + c];
                const double* __restrict__ lj = Pn + j * pld + b0;
#pragma unroll
                for (int r = 0; r < H; ++r) x[r] = fma(-lj[r], uj, x[r]);
            }
#pragma unroll
            for (int j = 0; j + 1 < H; ++j) {
                const double* __restrict__ lj = Pn + (b0 + j) * pld + b0;
#pragma unroll
                for (int r = j + 1; r < H; ++r) x[r] = fma(-lj[r], x[j], x[r]);
            }
#pragma unroll
            for (int r = 0; r < H; ++r) Un[(b0 + r) * uld + c] = x[r];
        }
    }
    named_sync(kBarPg, kPgThreads);
    for (int idx = ptid; idx < 32 * Rn; idx += kPgThreads) {
        const int r = idx & 31, c = idx >> 5;
        if (r < np && np + c - r <= L.K) __stcg(L.at(jp + r, jp + np + c), Un[r * uld + c]);
    }
}

}  // namespace

// Optional phase trace (build with -DSAP_LU_TRACE): CTA 0 records clock64 at
// phase boundaries for the first kTraceSteps steps (PG thread 0, UG warp 4 lane 0).
constexpr int kTraceSteps = 16;
constexpr int kTraceSlots = 12;
__device__ long long g_lu_trace[kTraceSteps * kTraceSlots];
__device__ long long g_lu_wtrace[64];  // per-warp timestamps of one step (SAP_LU_TRACE builds)
#ifdef SAP_LU_TRACE
#define LU_TRACE(step, slot, cond)                                                        \
    do {                                                                                  \
        if (blockIdx.x == 0 && (cond) && (step) < kTraceSteps) g_lu_trace[(step)*kTraceSlots + (slot)] = clock64(); \
    } while (0)
#else
#define LU_TRACE(step, slot, cond) do { } while (0)
#endif

template <int B>
__global__ void __launch_bounds__(kLuThreads, 1)
    k_band_lu_seq(const FactorJob* __restrict__ jobs, double eps, int pld, int uld) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_boosts;
    __shared__ __align__(16) double s_prow[2 * (B + 2)];
    const FactorJob J = jobs[blockIdx.x];
    const double scale = *J.scale;
    Lu L{J.base, J.rs, J.cs, J.m, J.k, B, pld, uld, eps * (scale > 0 ? scale : 1.0), J.src ? J.src : J.base};
    double* P = smem;
    double* U = smem + B * pld;
    const int tid = threadIdx.x, warp = tid >> 5;
    const bool pg = tid < kPgThreads;
    const int m = L.m, K = L.K;
    if (tid == 0) s_boosts = 0;
    __syncthreads();
    int step = 0;
    for (int jb = 0; jb < m; jb += B, ++step) {
        const int nb = min(B, m - jb);
        const int ph = min(nb + K, m - jb);
        const int ja = jb + nb;
        const int R = min(K, m - ja);
        LU_TRACE(step, 0, tid == 0);
        if (pg) {
            pg_stage_panel(L, P, jb, nb, ph, 0, 0, tid);
            named_sync(kBarPg, kPgThreads);
            LU_TRACE(step, 2, tid == 0);
            pg_factor_panel<B>(L, P, s_prow, &s_boosts, nb, ph, tid);
            LU_TRACE(step, 3, tid == 0);
            pg_store_panel(L, P, jb, nb, ph, tid);
            LU_TRACE(step, 4, tid == 0);
            pg_u12<B>(L, P, U, jb, nb, R, tid);
            LU_TRACE(step, 6, tid == 0);
        }
        __syncthreads();
        LU_TRACE(step, 1, tid == 0);
        dmma_region(L, P, U, nb, ja, 0, R, 0, R, warp, kLuThreads / 32, nullptr);
        LU_TRACE(step, 8, tid == 0);
        LU_TRACE(step, 9, tid == kLuThreads - 32);
        __syncthreads();
    }
    if (tid == 0) *J.boosts = s_boosts;
}

// ---------------------------------------------------------------------------
// k_band_lu_res: panel and A12 resident in shared memory.
//
// Per step s (panel columns [jb, jb+nb), A22 = the R x R window at (ja, ja), ja = jb+nb):
//   1. the nb x nb diagonal block was factored by warp 0 at the end of step s-1 (panel_diag: lane = row,
//      the pivot chain inside one warp); all threads finish L21 rows / U12 columns (panel_rows_cols);
//   2. all 16 warps run A22 -= L21 U12 on DMMA (res_bulk); the tiles that form panel s+1 (A22's first nb
//      columns) and A12(s+1) (its first rows) go straight into the other smem buffers instead of global,
//      with step s+1's new band entries, so the next step starts without staging;
//   3. warp 0 factors panel s+1's diagonal block while warps 1-15 store this step's panel and U12 to
//      global (evict-first) and L2-prefetch the band entries step s+1 meets first.
// Every element receives its updates in the reference's column order (FMA-contracted; the DMMA k-sum in
// groups of 4: the SURVEY §8c tolerances). The A22 tiles round-trip through L2 with an evict_last policy.
// Shared-memory pair load kept in program order (volatile): stops the compiler from hoisting a whole
// unrolled panel's operand loads to the top (register spills).
__device__ __forceinline__ void sts1(double* p, double v) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ double2 lds2(const double* p) {
    double2 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// Packed U11 rows: row c keeps entries j in [(c + 1) & ~1, B) (its U part plus at most one L entry),
// 16-byte aligned, 528 doubles in all for B = 32.
__host__ __device__ constexpr int ut_lo(int c) { return (c + 1) & ~1; }
__host__ __device__ constexpr int ut_off(int c) { return 32 * c - 2 * (c / 2) * ((c + 1) / 2); }
static_assert(ut_off(1) == 32 && ut_off(2) == 62 && ut_off(3) == 92 && ut_off(4) == 120, "packed U11 offsets");
constexpr int kUtSize = ut_off(32);

// 1/p from the MUFU.RCP64H seed and two Newton steps (2^-23 -> 2^-46 -> below one ulp); only ever used
// through div_rcp's residual correction and the multipliers' FMA updates.
__device__ __forceinline__ double rcp2(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    return fma(r, e, r);
}

// Pivot c of panel_diag (lane = row r, a[j] = the row's entry in column j; every index a compile-time
// constant). Stores go through explicit st.shared / ld.shared (a generic store to P here cost ~11%).
template <int c>
__device__ __forceinline__ void pd_pivot(double (&a)[32], int nb, bool full, int r, bool own, double bv, double& pl,
                                         double& rl, int& boosts, double* __restrict__ P, int pld,
                                         double* __restrict__ Ut, double* __restrict__ s_piv) {
    constexpr int B = 32;
    // pivot row c, published by its owner at the end of the previous round: the pair holding entry c + 1 (the
    // next pivot column) first
    const double* __restrict__ urow = Ut + ut_off(c) - ut_lo(c);  // urow[j] = U(c, j), j >= ut_lo(c)
    double2 un2 = make_double2(0.0, 0.0);
    if constexpr (c + 1 < B) un2 = lds2(urow + ((c + 1) & ~1));
    const double pc = __shfl_sync(0xffffffffu, pl, c);
    const double rc = __shfl_sync(0xffffffffu, rl, c);
    if (r == c) {
        s_piv[c] = pc;
        s_piv[B + c] = rc;
    }
    // rows below: multiplier (block_factors.hpp:36) and rank-1 update; other lanes apply l = 0 (rows above
    // stay as they are for finite pivot rows, the only kind a finite band produces)
    const bool below = own && r > c;
    const double lq = div_rcp(a[c], pc, rc);
    const double l = below ? lq : 0.0;
    a[c] = below ? lq : a[c];
    if (own) sts1(P + c * pld + r, a[c]);  // column c of L11\U11 is final
    if constexpr (c + 1 < B) {
        // the next pivot column first, so its reciprocal overlaps the rest of the row update
        if constexpr (c & 1) {  // pair (c + 1, c + 2)
            a[c + 1] = fma(-l, un2.x, a[c + 1]);
            if constexpr (c + 2 < B) a[c + 2] = fma(-l, un2.y, a[c + 2]);
        } else {  // pair (c, c + 1)
            a[c + 1] = fma(-l, un2.y, a[c + 1]);
        }
        if (full || c + 1 < nb) {  // boost rule block_factors.hpp:26-34; every lane inverts its own entry
            double p = a[c + 1];
            const bool boost = fabs(p) < bv;
            p = boost ? (p < 0.0 ? -bv : bv) : p;
            boosts += (boost && r == c + 1) ? 1 : 0;
            if (r == c + 1) a[c + 1] = p;
            pl = p;
            rl = rcp2(p);
        }
    }
    // the remaining pairs (aligned)
#pragma unroll
    for (int j = (c & 1) ? c + 3 : c + 2; j < B; j += 2) {
        const double2 u = lds2(urow + j);
        a[j] = fma(-l, u.x, a[j]);
        a[j + 1] = fma(-l, u.y, a[j + 1]);
    }
    // row c + 1 is final now: its owner publishes it for the next round
    if constexpr (c + 1 < B) {
        if (r == c + 1) {
#pragma unroll
            for (int j = ut_lo(c + 1); j < B; j += 2)
                *reinterpret_cast<double2*>(Ut + ut_off(c + 1) + j - ut_lo(c + 1)) = make_double2(a[j], a[j + 1]);
        }
    }
    __syncwarp();
}

template <int c, bool FULL>
__device__ __forceinline__ void pd_all(double (&a)[32], int nb, int r, bool own, double bv, double& pl, double& rl,
                                       int& boosts, double* __restrict__ P, int pld, double* __restrict__ Ut,
                                       double* __restrict__ s_piv, unsigned long long* marks) {
    if constexpr (c % 4 == 0) {
        if (marks && r == 0) marks[c >> 2] = clock64();  // tools/lu_df_trace.py: 4-pivot groups
    }
    if (FULL || c < nb) pd_pivot<c>(a, nb, FULL, r, own, bv, pl, rl, boosts, P, pld, Ut, s_piv);
    if constexpr (c + 1 < 32) pd_all<c + 1, FULL>(a, nb, r, own, bv, pl, rl, boosts, P, pld, Ut, s_piv, marks);
}

// The nb x nb diagonal block's pivot chain in one warp (lane = row), fully unrolled (rolled 2- / 4-pivot loops
// with a register shift measured 1.9x / 1.8x slower, tools/probe/diag_throttle.cu). Every element gets the
// same FMAs in the same order as a column-by-column right-looking elimination; the published U rows (Ut,
// packed) and the pivots / reciprocals (s_piv) feed the L21 rows. The calling warp must be converged (see
// df_wait).
template <int B, bool FULL>
__device__ __noinline__ void panel_diag(double* __restrict__ P, int pld, double* __restrict__ Ut,
                                        double* __restrict__ s_piv, int nb_rt, double bv, int* boost_ctr,
                                        unsigned long long* marks = nullptr) {
    static_assert(B == 32, "panel_diag: 32-column panels");
    const int nb = FULL ? B : nb_rt;
    const int r = threadIdx.x & 31;
    const bool own = r < nb;
    double a[B];
#pragma unroll
    for (int j = 0; j < B; ++j) a[j] = (own && j < nb) ? P[j * pld + r] : 0.0;
    // row 0 is final from the start: its owner publishes it (U part) before the first pivot
    if (r == 0) {
#pragma unroll
        for (int j = ut_lo(0); j < B; j += 2)
            *reinterpret_cast<double2*>(Ut + ut_off(0) + j - ut_lo(0)) = make_double2(a[j], a[j + 1]);
    }
    int boosts = 0;
    double pl, rl;
    {
        double p = a[0];
        const bool boost = fabs(p) < bv;
        p = boost ? (p < 0.0 ? -bv : bv) : p;
        boosts += (boost && r == 0) ? 1 : 0;
        if (r == 0) a[0] = p;
        pl = p;
        rl = rcp2(p);
    }
    __syncwarp();
    pd_all<0, FULL>(a, nb, r, own, bv, pl, rl, boosts, P, pld, Ut, s_piv, marks);
    if (marks && r == 0) marks[8] = clock64();
    if (boosts) atomicAdd(boost_ctr, boosts);
}

template <int B, bool FULL>
__device__ __noinline__ void panel_rows_cols(double* __restrict__ P, double* __restrict__ A, int pld, int uld,
                                             const double* __restrict__ Ut, const double* __restrict__ s_piv,
                                             int nb_rt, int ph, int R) {
    const int nb = FULL ? B : nb_rt;
    const int tid = threadIdx.x;
    if (tid < 256) {
        const int r = nb + tid;
        if (r >= ph) return;
        double x[B];
#pragma unroll
        for (int c = 0; c < B; ++c) x[c] = c < nb ? P[c * pld + r] : 0.0;
#pragma unroll
        for (int c = 0; c < B; ++c) {
            if (c < nb) {
                const double l = div_rcp(x[c], s_piv[c], s_piv[B + c]);
                x[c] = l;
                const double2* __restrict__ u2 = reinterpret_cast<const double2*>(Ut + ut_off(c) - ut_lo(c));
#pragma unroll
                for (int j = (c + 1) & ~1; j < B; j += 2) {
                    const double2 u = lds2(reinterpret_cast<const double*>(u2 + (j >> 1)));
                    if (j > c) x[j] = fma(-l, u.x, x[j]);
                    x[j + 1] = fma(-l, u.y, x[j + 1]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < B; ++c)
            if (c < nb) P[c * pld + r] = x[c];
    } else {
        const int col = tid - 256;
        if (col >= R) return;
        double y[B];
#pragma unroll
        for (int q = 0; q < B; ++q) y[q] = q < nb ? A[q * uld + col] : 0.0;
#pragma unroll
        for (int c = 0; c < B; ++c) {
            if (c < nb) {
                const double2* __restrict__ l2 = reinterpret_cast<const double2*>(P + c * pld);
#pragma unroll
                for (int q = (c + 1) & ~1; q < B; q += 2) {
                    const double2 l = lds2(reinterpret_cast<const double*>(l2 + (q >> 1)));
                    if (q > c) y[q] = fma(-l.x, y[c], y[q]);
                    y[q + 1] = fma(-l.y, y[c], y[q + 1]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (q < nb) A[q * uld + col] = y[q];
    }
}

// cp.async the entries of panel (jp, np) (rows [0, ph)) and of its A12 block (rows [0, np) x cols [0, Rn) at
// (jp, jp+np)) that the previous step's trailing update does not produce: that update covers the window
// [0, cov) x [0, cov) of panel coordinates (cov = 0 in the prologue). In-band entries only; the rest of
// the buffers stays zero.
__device__ __forceinline__ void res_fetch(const Lu& L, double* __restrict__ Pb, double* __restrict__ Ab, int jp, int np,
                                          int cov, int ph, int Rn, int t0, int nt) {
    const int pld = L.pld, uld = L.uld;
    for (int idx = threadIdx.x - t0; idx < ph * np; idx += nt) {
        const int c = idx / ph, r = idx - c * ph;
        if (r < cov && c < cov) continue;
        if (L.inband(r, c)) cp_async8(Pb + c * pld + r, L.src_at(jp + r, jp + c));
    }
    for (int idx = threadIdx.x - t0; idx < Rn * 32; idx += nt) {
        const int r = idx & 31, c = idx >> 5;
        if (r >= np || (r < cov && np + c < cov)) continue;
        if (np + c - r <= L.K) cp_async8(Ab + r * uld + c, L.src_at(jp + r, jp + np + c));
    }
}

// L2 prefetch of the unfactored entries that step s+1 reads for the first time (HBM -> L2 one step
// ahead): band rows [ja+R, ja+R+nb) of every column they meet, and columns [ja+R, ja+R+nb) of the rows
// above them. One contiguous run (|rs| == 1) per column and bulk prefetch instruction.
__device__ __forceinline__ void prefetch_run(const Lu& L, int c, int r0, int r1) {
    r0 = max(r0, c - L.K);
    r1 = min(r1, min(c + L.K + 1, L.m));
    if (r0 >= r1) return;
    const double* a = L.rs > 0 ? L.src_at(r0, c) : L.src_at(r1 - 1, c);
    uintptr_t lo = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
    uintptr_t hi = (reinterpret_cast<uintptr_t>(a) + 8 * (r1 - r0) + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo)) : "memory");
}

// tile_load for k_band_lu_res: A22 entries at window coordinates (i, c) with i >= fr or c >= fr have never
// been updated (they entered the window this step) and come from the unfactored source view; the rest
// come from the factor store, where the previous step's update left them.
__device__ __forceinline__ void tile_load_fr(const Lu& L, const TileCtx& T, int t, double (&acc)[2][kTQ][2], int fr) {
    const int row0 = T.r_lo + (t / T.tcols) * kTileR, col0 = T.c_lo + (t % T.tcols) * kTileC;
    if (row0 + kTileR <= fr && col0 + kTileC <= fr) {
        tile_load(L, T, t, acc);
        return;
    }
    const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int ib = row0 + 2 * lc, cb = col0 + lr;
    const long long rs = L.rs, ra8 = 8 * rs, cq8 = 8 * L.cs;
    const int gi = T.row_org + ib, gc = T.col_org + cb;
    const double* d00 = L.at(gi, gc);
    const double* s00 = L.src_at(gi, gc);
    const double* dlo = rs > 0 ? d00 : d00 - 1;
    const double* slo = rs > 0 ? s00 : s00 - 1;
    const bool full = row0 + kTileR <= T.r_hi && col0 + kTileC <= T.c_hi && row0 >= T.band_top;
    if (full && (rs == 1 || rs == -1) && (fr & 1) == 0 &&
        (((reinterpret_cast<uintptr_t>(dlo) | reinterpret_cast<uintptr_t>(slo)) & 15) == 0)) {
        // row pairs (ib + 8a, ib + 8a + 1) never straddle an even fr: one 16-byte load per pair from its side
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < kTQ; ++q) {
                const bool fresh = ib + a * 8 >= fr || cb + q * 8 >= fr;
                const double2 v = ld_keep2((fresh ? slo : dlo) + a * ra8 + q * cq8);
                acc[a][q][0] = rs > 0 ? v.x : v.y;
                acc[a][q][1] = rs > 0 ? v.y : v.x;
            }
        return;
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < kTQ; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = ib + a * 8 + e, c = cb + q * 8;
                const long long o = a * ra8 + e * rs + q * cq8;
                acc[a][q][e] = tile_ok(L, T, i, c) ? ld_keep((i >= fr || c >= fr ? s00 : d00) + o) : 0.0;
            }
}

// A22 -= L21 U12 over 16 x 32 warp tiles; panel-(s+1) columns -> Pn, A12(s+1) rows -> An, rest -> global.
// Also brings in step s+1's NEW band entries (panel rows [R, phn), A12 columns [R-nbn, Rn); never touched by
// an update): loaded into registers before the tile loop, stored to smem after it, so the load latency
// hides under the DMMA work (in-flight cp.async would stall the next step's shared loads).
__device__ __noinline__ void res_bulk(const Lu& L, const double* __restrict__ P, const double* __restrict__ U, int nb,
                                      int ja, int R, int nbn, int phn, int Rn, double* __restrict__ Pn,
                                      double* __restrict__ An, int fr, int step) {
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int pld = L.pld, uld = L.uld;
    constexpr int kPf = 4;  // fetch columns per warp: 64 = 32 panel + 32 A12 columns over 16 warps
    double pf[kPf];
    const bool fast = nbn > 0 && R >= nbn && nw * kPf >= 64;
#ifdef SAP_LU_TRACE
    if (step == 8 && blockIdx.x == 0 && lane == 0) g_lu_wtrace[warp] = clock64();
#endif
    if (nbn > 0 && !fast) res_fetch(L, Pn, An, ja, nbn, R, phn, Rn, 0, nw * 32);
    if (fast) {
#pragma unroll
        for (int i = 0; i < kPf; ++i) {
            const int f = warp + nw * i;
            pf[i] = 0.0;
            if (f < 32) {  // panel column f, row R + lane
                const int r = R + lane;
                if (f < nbn && r < phn && r - f <= L.K) pf[i] = __ldcs(L.src_at(ja + r, ja + f));
            } else if (f < 64) {  // A12 column R - nbn + (f - 32), row lane
                const int c = R - nbn + (f - 32);
                if (c < Rn && lane < nbn && nbn + c - lane <= L.K) pf[i] = __ldcs(L.src_at(ja + lane, ja + nbn + c));
            }
        }
    }
    if (R > 0) {
        const TileCtx T = make_tiles(0, R, 0, R, ja, ja, nb, 0, 0, 0);
        const int ntiles = ((R + kTileR - 1) / kTileR) * T.tcols;
        const int ksteps = (nb + 3) >> 2;
        double acc[2][kTQ][2];
        for (int t = warp; t < ntiles; t += nw) {
            tile_load_fr(L, T, t, acc, fr);
            const int row0 = (t / T.tcols) * kTileR, col0 = (t % T.tcols) * kTileC;
            const bool a1 = row0 + 8 < R;
            bool qv[kTQ];
#pragma unroll
            for (int q = 0; q < kTQ; ++q) qv[q] = col0 + q * 8 < R;
            const double* pk = P + nb + row0 + lr;
            const double* uk = U + col0 + lr;
            if (ksteps == 8 && a1 && qv[kTQ - 1]) {
                // full tile, full panel: operands of k-step ks+1 load while ks's DMMAs issue
                double b0 = -pk[lc * pld], b1 = -pk[lc * pld + 8], aq[kTQ];
#pragma unroll
                for (int q = 0; q < kTQ; ++q) aq[q] = uk[lc * uld + q * 8];
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    double nb0 = 0.0, nb1 = 0.0, naq[kTQ];
                    if (ks + 1 < 8) {
                        const int kn = (ks + 1) * 4 + lc;
                        nb0 = -pk[kn * pld];
                        nb1 = -pk[kn * pld + 8];
#pragma unroll
                        for (int q = 0; q < kTQ; ++q) naq[q] = uk[kn * uld + q * 8];
                    }
#pragma unroll
                    for (int q = 0; q < kTQ; ++q) {
                        dmma_m8n8k4(acc[0][q][0], acc[0][q][1], aq[q], b0, acc[0][q][0], acc[0][q][1]);
                        dmma_m8n8k4(acc[1][q][0], acc[1][q][1], aq[q], b1, acc[1][q][0], acc[1][q][1]);
                    }
                    if (ks + 1 < 8) {
                        b0 = nb0;
                        b1 = nb1;
#pragma unroll
                        for (int q = 0; q < kTQ; ++q) aq[q] = naq[q];
                    }
                }
            } else {
                for (int ks = 0; ks < ksteps; ++ks) {
                    const int kk = ks * 4 + lc;
                    const double b0 = -pk[kk * pld];
                    const double b1 = -pk[kk * pld + 8];
#pragma unroll
                    for (int q = 0; q < kTQ; ++q) {
                        if (qv[q]) {
                            const double aq = uk[kk * uld + q * 8];
                            dmma_m8n8k4(acc[0][q][0], acc[0][q][1], aq, b0, acc[0][q][0], acc[0][q][1]);
                            if (a1) dmma_m8n8k4(acc[1][q][0], acc[1][q][1], aq, b1, acc[1][q][0], acc[1][q][1]);
                        }
                    }
                }
            }
            const int ib = row0 + 2 * lc, cb = col0 + lr;
            const bool to_p = col0 < nbn, to_a = !to_p && row0 < nbn;
            if (!to_p && !to_a) {
                // global: one 16-byte store per row pair when aligned (tall-thin band, |rs| == 1)
                const long long rs = L.rs, ra8 = 8 * rs, cq8 = 8 * L.cs;
                double* p00 = L.at(ja + ib, ja + cb);
                double* lo00 = rs > 0 ? p00 : p00 - 1;
                const bool full = row0 + kTileR <= R && col0 + kTileC <= R;
                if (full && ((reinterpret_cast<uintptr_t>(lo00) & 15) == 0)) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q) {
                            double2 v;
                            v.x = rs > 0 ? acc[a][q][0] : acc[a][q][1];
                            v.y = rs > 0 ? acc[a][q][1] : acc[a][q][0];
                            st_keep2(lo00 + a * ra8 + q * cq8, v);
                        }
                } else {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int i = ib + a * 8 + e, c = cb + q * 8;
                                if (i < R && c < R) st_keep(p00 + a * ra8 + e * rs + q * cq8, acc[a][q][e]);
                            }
                }
            } else if (nbn == kTileC && row0 + kTileR <= R && col0 + kTileC <= R &&
                       (to_p || row0 + kTileR <= nbn)) {
                // whole tile inside the next panel (16-byte pairs: rows i, i+1 adjacent in Pn) or inside
                // the next U12 rows (An row-major)
                if (to_p) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q)
                            *reinterpret_cast<double2*>(Pn + (cb + q * 8) * pld + ib + a * 8) =
                                make_double2(acc[a][q][0], acc[a][q][1]);
                } else {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q) {
                            An[(ib + a * 8) * uld + (cb + q * 8 - nbn)] = acc[a][q][0];
                            An[(ib + a * 8 + 1) * uld + (cb + q * 8 - nbn)] = acc[a][q][1];
                        }
                }
            } else {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int q = 0; q < kTQ; ++q)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int i = ib + a * 8 + e, c = cb + q * 8;
                            if (i >= R || c >= R) continue;
                            if (c < nbn)
                                Pn[c * pld + i] = acc[a][q][e];
                            else if (i < nbn)
                                An[i * uld + (c - nbn)] = acc[a][q][e];
                            else
                                st_keep(L.at(ja + i, ja + c), acc[a][q][e]);
                        }
            }
        }
    }
#ifdef SAP_LU_TRACE
    if (step == 8 && blockIdx.x == 0 && lane == 0) g_lu_wtrace[16 + warp] = clock64();
#endif
    if (fast) {
#pragma unroll
        for (int i = 0; i < kPf; ++i) {
            const int f = warp + nw * i;
            if (f < 32) {
                const int r = R + lane;
                if (f < nbn && r < phn) Pn[f * pld + r] = pf[i];
            } else if (f < 64) {
                const int c = R - nbn + (f - 32);
                if (c < Rn && lane < nbn) An[lane * uld + c] = pf[i];
            }
        }
    }
}

template <int B, bool STREAM>
__global__ void __launch_bounds__(kLuThreads, 1)
    k_band_lu_res(const FactorJob* __restrict__ jobs, double eps, int pld, int uld) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_boosts;
    static_assert(B == 32, "packed U11 rows (kUtSize) assume B = 32");
    __shared__ __align__(16) double s_ut[kUtSize];  // packed U11 rows of the current panel
    __shared__ double s_rcp[2 * B];  // [0, B): 1/p, [B, 2B): p
    const FactorJob J = jobs[blockIdx.x];
    if (!STREAM && J.gate && !(*J.gate & 1)) return;  // streamed setup: no pivot fell below the threshold
    constexpr bool streamed = STREAM;  // J.ready != nullptr
    const double scale = streamed ? 0.0 : *J.scale;  // streamed: the block norm is not known yet
    Lu L{J.base, J.rs, J.cs, J.m, J.k, B, pld, uld, streamed ? 0.0 : eps * (scale > 0 ? scale : 1.0),
         J.src ? J.src : J.base};
    const int psz = B * pld, usz = B * uld;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int m = L.m, K = L.K;
    __shared__ double s_minp;
    __shared__ int s_timeout;
    for (int i = tid; i < 2 * (psz + usz); i += kLuThreads) smem[i] = 0.0;
    if (tid == 0) {
        s_boosts = 0;
        s_minp = INFINITY;
        s_timeout = 0;
    }
    // streamed upload: before a step reads the band, its columns [0, need) plus one margin column (no L1
    // line of a read column reaches unarrived bytes) must have arrived
    // s_got: the last counter value seen (shared, changed only inside the polling branch, which ends in a
    // barrier), so every thread takes the same branch and a satisfied step costs no load and no barrier
    __shared__ unsigned s_got;
    if (tid == 0) s_got = 0;
    auto wait_cols = [&](int need) {
        if constexpr (!STREAM) return;
        const long long want = min(m, need + 1);
        const long long have = (long long)s_got * J.piece;
        if (have >= want || have * J.ends >= m || s_timeout) return;
        if (tid < 32) {  // warp-uniform spin (df_wait: a lane-0 spin leaves the pivot warp diverged)
            const long long t0 = __shfl_sync(0xffffffffu, clock64(), 0);
            for (;;) {
                unsigned r;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(J.ready) : "memory");
                r = __shfl_sync(0xffffffffu, r, 0);
                const long long got = (long long)r * J.piece;
                if (got >= want || got * J.ends >= m) {
                    if (tid == 0) s_got = r;
                    break;
                }
                if (__shfl_sync(0xffffffffu, clock64(), 0) - t0 > (1LL << 36)) {  // ~35 s: the upload stalled
                    if (tid == 0) s_timeout = 1;
                    break;
                }
                __nanosleep(256);
            }
            __syncwarp();
        }
        __syncthreads();
    };
    __syncthreads();
    wait_cols(3 * B + K);
    {
        const int nb = min(B, m), ph = min(nb + K, m), R = min(K, m - nb);
        res_fetch(L, smem, smem + 2 * psz, 0, nb, 0, ph, R, 0, kLuThreads);
        cp_async_wait_all();
        __syncthreads();
        if (warp == 0) {
            if (nb == B)
                panel_diag<B, true>(smem, pld, s_ut, s_rcp, nb, L.bv, &s_boosts);
            else
                panel_diag<B, false>(smem, pld, s_ut, s_rcp, nb, L.bv, &s_boosts);
        }
    }
    __syncthreads();
    int cur = 0, step = 0;
    for (int jb = 0; jb < m; jb += B, ++step) {
        const int nb = min(B, m - jb);
        const int ph = min(nb + K, m - jb);
        const int ja = jb + nb;
        const int R = min(K, m - ja);
        const bool has_next = ja < m;
        const int nbn = has_next ? min(B, m - ja) : 0;
        const int phn = has_next ? min(nbn + K, m - ja) : 0;
        const int Rn = has_next ? min(K, m - ja - nbn) : 0;
        double* P = smem + cur * psz;
        double* A = smem + 2 * psz + cur * usz;
        double* Pn = smem + (cur ^ 1) * psz;
        double* An = smem + 2 * psz + (cur ^ 1) * usz;
        wait_cols(jb + 3 * B + K);
        LU_TRACE(step, 0, tid == 0);
        // 1-2. panel + U12: the diagonal block was factored by warp 0 during the previous step's update (or
        //      the prologue); here all threads finish L21 rows / U12 columns
        if (nb == B)
            panel_rows_cols<B, true>(P, A, pld, uld, s_ut, s_rcp, nb, ph, R);
        else
            panel_rows_cols<B, false>(P, A, pld, uld, s_ut, s_rcp, nb, ph, R);
        __syncthreads();
        LU_TRACE(step, 3, tid == 0);
        // 3. trailing update (next panel / A12 land in smem) + step s+1's new band entries; window entries at
        //    or beyond the previous step's window edge (jb + min(K, m - jb)) are fresh
        const int fr = jb == 0 ? 0 : min(K, m - jb) - nb;
        res_bulk(L, P, A, nb, ja, R, nbn, phn, Rn, Pn, An, fr, step);
        cp_async_wait_all();
        __syncthreads();
        LU_TRACE(step, 7, tid == 0);
        // 4. warp 0: the next panel's diagonal block (one warp's pivot chain); warps 1-15 meanwhile store this
        //    step's panel (L11\U11, L21) and U12 (warp per column, lanes down the rows; P, A are intact) and
        //    L2-prefetch the next step's new band entries
        if (warp == 0) {
            if (has_next) {
                if (nbn == B)
                    panel_diag<B, true>(Pn, pld, s_ut, s_rcp, nbn, L.bv, &s_boosts);
                else
                    panel_diag<B, false>(Pn, pld, s_ut, s_rcp, nbn, L.bv, &s_boosts);
            }
        } else {
            const int lane = tid & 31, w1 = warp - 1, nw1 = kLuThreads / 32 - 1;
            const long long rs = L.rs;
            for (int c = w1; c < nb; c += nw1) {
                double* g = L.at(jb, jb + c);
                const int r1 = min(ph, c + K + 1);
#pragma unroll 4
                for (int r = max(c - K, 0) + lane; r < r1; r += 32) __stcs(g + r * rs, P[c * pld + r]);
            }
            if (lane < nb) {
                double* g = L.at(jb + lane, ja);
                const long long cs = L.cs;
#pragma unroll 4
                for (int c = w1; c < R; c += nw1)
                    if (nb + c - lane <= K) __stcs(g + c * cs, A[lane * uld + c]);
            }
            if (ja < m && ja + R < m) {
                // prefetch_fresh's runs over warps 1-15
                const int e = ja + R, t1 = tid - 32;
                const int ncol = min(e + nbn, m) - ja;
                for (int t = t1; t < ncol + min(nbn, m - e); t += kLuThreads - 32) {
                    if (t < ncol)
                        prefetch_run(L, ja + t, e, e + nbn);
                    else
                        prefetch_run(L, e + t - ncol, ja + nbn, e);
                }
            }
        }
        cp_async_wait_all();
        LU_TRACE(step, 8, tid == 32);
        __syncthreads();
        cur ^= 1;
    }
    if (tid == 0) *J.boosts = s_boosts;
    if (STREAM && tid == 0 && s_timeout) *J.minpiv = -1.0;  // min |pivot| is read off U's diagonal afterwards
}

// dynamic shared memory of k_band_lu_res: 227 KB per block minus its static arrays (packed U11 rows,
// pivots, counters)
constexpr size_t kResSmemMax = 227 * 1024 - sizeof(double) * (kUtSize + 64) - 64;

static int pad_ld(int x) {
    // leading dimensions == 4 or 12 (mod 16) keep the DMMA fragment loads conflict-free
    while ((x % 16) != 4 && (x % 16) != 12) ++x;
    return x;
}

void read_lu_wtrace(long long* out) { SAP_CUDA(cudaMemcpyFromSymbol(out, g_lu_wtrace, sizeof(long long) * 64)); }
void read_lu_trace(long long* out) {
    SAP_CUDA(cudaMemcpyFromSymbol(out, g_lu_trace, sizeof(long long) * kTraceSteps * kTraceSlots));
}

bool launch_band_lu_ws(const FactorJob* d_jobs, int njobs, int max_k, double eps, cudaStream_t s, bool streamed) {
    constexpr int B = 32;
    // panel rows (<= B + K) must fit one per panel-group thread
    if (max_k < 1 || B + max_k > kPgThreads) return false;
    if (max_k <= 256 - B) {
        // panel rows: L21 by threads 0-255, U12 columns by threads 256-511
        const int pldr = pad_ld(B + max_k);
        const int uldr = pad_ld(max_k);
        const size_t rbytes = sizeof(double) * (size_t)(2 * B * pldr + 2 * B * uldr);
        if (rbytes <= kResSmemMax) {
            if (streamed) {
                SAP_CUDA(cudaFuncSetAttribute(k_band_lu_res<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)rbytes));
                k_band_lu_res<B, true><<<njobs, kLuThreads, rbytes, s>>>(d_jobs, eps, pldr, uldr);
            } else {
                SAP_CUDA(cudaFuncSetAttribute(k_band_lu_res<B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)rbytes));
                k_band_lu_res<B, false><<<njobs, kLuThreads, rbytes, s>>>(d_jobs, eps, pldr, uldr);
            }
            SAP_LAUNCHED();
            return true;
        }
    }
    const int k8 = ((max_k + 7) / 8) * 8;
    const int pld = pad_ld(B + 16 * ((max_k + 15) / 16) + 8);
    const int uld = pad_ld(k8 + 32);
    const size_t bytes = sizeof(double) * (size_t)(B * pld + B * uld);
    if (bytes > 222 * 1024) return false;
    SAP_CUDA(cudaFuncSetAttribute(k_band_lu_seq<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_band_lu_seq<B><<<njobs, kLuThreads, bytes, s>>>(d_jobs, eps, pld, uld);
    SAP_LAUNCHED();
    return true;
}

// ---------------------------------------------------------------------------
// k_band_lu_df: the same factorization as a dataflow over every SM.
//
// One 32-column step s of job J (panel columns [jb, jb + nb), trailing window [ja, ja + R)^2, ja = jb + nb)
// is split into work items:
//   panel(J, s)     the 32 x 32 diagonal block (one warp's pivot chain, panel_diag) and the L21 rows
//                   (panel_rows_cols), stored final;
//   strip(J, s, j)  window columns [32 j, 32 j + 32): the U12 slice = L11^{-1} A12 (thread per column,
//                   the reference's order) stored final, then A22 -= L21 U12 on DMMA over all R rows, stored
//                   back in place (L2, evict_last).
// Dependencies (per job): panel(s) <- strip(s-1, 0) (it produced the panel's columns); strip(s, j) <-
// panel(s) and strip(s-1, j+1) (it produced the strip's columns). Items are numbered in a topological
// order with look-ahead -- wave w: strip(w, 0) of every job, panel(w+1) of every job, strip(w, j >= 1) of
// every job -- and grabbed from one atomic counter by persistent CTAs (two per SM), so a panel's pivot chain
// overlaps other jobs' DMMA strips on the same SM and a job is no longer confined to one SM. A CTA only
// ever waits for items grabbed before its own by running CTAs, so the schedule cannot deadlock whatever
// the residency. Completion is published per job: panel_cnt[J] = s + 1, col_step[J][a] = s + 1 for the
// 32-column block a a strip updated (st.release.gpu after a CTA barrier; readers ld.acquire.gpu, then
// read the data with L1-bypassing .cg loads).
// Every element receives exactly the arithmetic of k_band_lu_res (same panel code, same DMMA fragments
// and k order): the factors are bitwise those of the single-CTA kernel.
// CTA shapes: 256 threads, two CTAs per SM for K <= 224; 512 threads, one CTA per SM up to K = 512 (the panel
// alone is (32 + K) x 32 doubles). RW row-warps x 2 column halves share a strip's C tile, NG row groups each.
template <int NT>
struct DfCfg {
    static constexpr int RW = NT / 64;
    static constexpr int NG = NT == 256 ? 7 : 8;
    static constexpr int MAXK = NT == 256 ? 224 : 512;
    static constexpr int MINB = NT == 256 ? 2 : 1;
};
constexpr int kLuDfMinK = 192;  // narrower bands: too few strips per step to pay for the item overheads
constexpr int kDfMaxSm = 256;  // %smid bound
constexpr int kDfG = 3;        // max strips per worker item (one panel load and one U12 solve for all of them)  // row groups (8 rows) per warp: 4 warps share a strip's rows, K <= 224

struct DfArgs {
    const FactorJob* jobs;
    int njobs, m_max, K, S;  // S = ceil(m_max / 32) steps; item numbering from the largest job
    unsigned* counter_p;  // chain items (panel SMs)
    unsigned* counter_w;  // worker strips
    int nps;              // the first nps SMs this launch's CTAs start on run chain items
    int excl;             // 1: one chain CTA per panel SM (its other CTAs exit); the chain's update on DMMA
    int* sm_role;         // [kDfMaxSm]: 0 undecided, 1 panel, 2 worker, 3 being decided
    int* n_panel_sm;      // SMs claimed so far
    int* n_chain;         // chain CTAs so far (a chain CTA's rank)
    int* started;         // CTAs past their role claim
    int* mode;            // chain schedule: 0 undecided, 1 job owners, 2 shared s-major queue
    int owners_ok;        // 0: always the queue (tools/lu_df_check.py A/B)
    int grp;              // strips per worker item (1..kDfG)
    int* panel_cnt;  // [njobs]
    int* col_step;   // [njobs][S]
    int* boost_acc;  // [njobs]
    int* err;        // a dependency wait timed out (never expected: reported as a CUDA failure)
    double eps;
    int pld, uld;
    unsigned long long* trace;  // tools only (lu_df_trace): per item grab / ready / end globaltimer + SM
};

__device__ __forceinline__ unsigned long long df_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire_i(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_cg(const double* a) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(a));
    return v;
}
__device__ __forceinline__ double2 ld_cg2(const double* a) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a));
    return v;
}

__device__ __forceinline__ int ld_relaxed_i(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// the acquire side of every wait of an item, once (an acquire load / fence invalidates the SM's whole L1:
// polling with it would wipe the co-resident CTA's L1 and stack on every probe)
__device__ __forceinline__ void df_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// thread 0: spin (relaxed loads) until *flag >= want (~4 s cap: a lost dependency is reported, never a hang;
// err[0] = 1, err[1..6] = the first timed-out wait: CTA, SM, the flag's word offset, want, have, tag)
// Called by all 32 lanes of one warp: the spin is warp-uniform (lane 0's value decides). A lane-0-only spin
// with __nanosleep left the warp diverged: the pivot chain it ran next took ~3.3x as long (every chain item that
// had waited, profiles/lu_df_r02.txt).
__device__ __forceinline__ int ld_relaxed_w(const int* p) { return __shfl_sync(0xffffffffu, ld_relaxed_i(p), 0); }

__device__ __forceinline__ void df_wait(const int* flag, int want, int* err, const int* base, int tag) {
    if (ld_relaxed_w(flag) >= want) return;
    const long long t0 = __shfl_sync(0xffffffffu, clock64(), 0);
    while (ld_relaxed_w(flag) < want) {
        __nanosleep(100);
        if (__shfl_sync(0xffffffffu, clock64(), 0) - t0 > (1LL << 33)) {
            if ((threadIdx.x & 31) == 0 && atomicExch(err, 1) == 0) {
                unsigned smid;
                asm("mov.u32 %0, %%smid;" : "=r"(smid));
                err[1] = blockIdx.x;
                err[2] = (int)smid;
                err[3] = (int)(flag - base);
                err[4] = want;
                err[5] = ld_relaxed_i(flag);
                err[6] = tag;
            }
            __syncwarp();
            return;
        }
    }
}

// one warp (all lanes, warp-uniform like df_wait), streamed upload: band columns [0, need) of this job's view have
// arrived (k_band_lu_res wait_cols)
__device__ __forceinline__ void df_wait_cols(const FactorJob& J, int need) {
    const long long want = min(J.m, need + 1);
    const long long t0 = __shfl_sync(0xffffffffu, clock64(), 0);
    for (;;) {
        unsigned r;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(J.ready) : "memory");
        r = __shfl_sync(0xffffffffu, r, 0);
        const long long got = (long long)r * J.piece;
        if (got >= want || got * J.ends >= J.m) return;
        if (__shfl_sync(0xffffffffu, clock64(), 0) - t0 > (1LL << 36)) {  // ~35 s: the upload stalled (minpiv)
            if ((threadIdx.x & 31) == 0) *J.minpiv = -1.0;
            __syncwarp();
            return;
        }
        __nanosleep(128);
    }
}

// element (i, c) of the job's view from the factor store (updated by an earlier item) or, when it has never
// been updated (fresh), from the unfactored source
__device__ __forceinline__ double df_ld(const Lu& L, int i, int c, bool fresh) {
    return ld_cg(fresh ? L.src_at(i, c) : L.at(i, c));
}

// trace mark (tools/lu_df_trace.py): per-CTA slot `k` of the current item
// marks go to shared memory (one global record per item at its end: tracing must not perturb the item)
__shared__ unsigned long long g_df_smark[8];
__shared__ unsigned long long g_df_pmark[10];  // trace: panel_diag's 4-pivot groups [0, 9), the update rows' end
constexpr int kDfRec = 22;                     // trace record (u64)
#define DF_MARK(k)                                                   \
    do {                                                             \
        if (A.trace && threadIdx.x == 0) g_df_smark[k] = clock64(); \
    } while (0)

// Lean staging of a 32-column panel-shaped region: rows [0, nr) of view columns cb + [0, 32) starting at view
// row i0 -> dst[c * ld + r]; rows r < rsplit come from the store, the rest from the source; entries outside the
// band (|i - c| > K) and columns >= nc are zero. Thread (c = tid / 8, k = tid % 8) takes the row pairs
// 2 (k + 8 it): one column pointer per thread, one 16-byte load per pair where the pair lies inside the band
// and is aligned (alignment is uniform per job and source for even rows); loads of a batch before any use.
template <int NT>
__device__ __forceinline__ void df_stage_panel(const Lu& L, double* __restrict__ dst, int ld, int i0, int cb, int nr,
                                               int nc, int rsplit) {
    constexpr int TPC = NT / 32;  // threads per column
    const int c = threadIdx.x / TPC, k = threadIdx.x % TPC;
    const long long rs = L.rs;
    const int gc = cb + c;
    const int lo_r = max(0, gc - L.K - i0), hi_r = min(nr, gc + L.K + 1 - i0);
    const double* ps = L.at(i0, gc);
    const double* pf = L.src_at(i0, gc);
    const bool vec = rs == 1 || rs == -1;
    // 16-byte alignment of the pair (r, r + 1), r even: uniform per pointer
    const bool al_s = vec && ((reinterpret_cast<uintptr_t>(rs > 0 ? ps : ps - 1) & 15) == 0);
    const bool al_f = vec && ((reinterpret_cast<uintptr_t>(rs > 0 ? pf : pf - 1) & 15) == 0);
    constexpr int NB = 8;
    for (int it0 = 0; 2 * (k + TPC * it0) < nr; it0 += NB) {
        double2 v[NB];
        unsigned paired = 0;
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int r = 2 * (k + TPC * (it0 + u));
            v[u] = make_double2(0.0, 0.0);
            if (c >= nc || r >= nr) continue;
            const bool in0 = r >= lo_r && r < hi_r, in1 = r + 1 >= lo_r && r + 1 < hi_r;
            const bool f0 = r >= rsplit, f1 = r + 1 >= rsplit;
            const double* p0 = (f0 ? pf : ps) + r * rs;
            if (in0 && in1 && f0 == f1 && (f0 ? al_f : al_s)) {
                v[u] = __ldcg(reinterpret_cast<const double2*>(rs > 0 ? p0 : p0 - 1));
                paired |= 1u << u;
            } else {
                if (in0) v[u].x = __ldcg(p0);
                if (in1) v[u].y = __ldcg((f1 ? pf : ps) + (r + 1) * rs);
            }
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int r = 2 * (k + TPC * (it0 + u));
            if (r >= nr) continue;
            const double2 w = (rs < 0 && (paired >> u & 1)) ? make_double2(v[u].y, v[u].x) : v[u];
            if (r + 1 < nr)
                *reinterpret_cast<double2*>(dst + c * ld + r) = w;
            else
                dst[c * ld + r] = w.x;
        }
    }
}

// ---- item helpers (256 threads) -------------------------------------------------------------------------
// The C tile of a strip: window rows [0, R) x window columns [c0, c0 + wc) of step (ja, fr). Warp w takes
// columns c0 + 16 (w >> 2) + [0, 16) and row groups (w & 3) + 4 t; the thread holds
// C(8 g + 2 lc + e, col0 + 8 q + lr) in acc[t][q][e] (k_band_lu_res' DMMA fragment layout).
struct DfTile {
    int ja, R, c0, wc, fr;
};

template <int NT>
__device__ __forceinline__ void df_c_load(const Lu& L, const DfTile& T, double (&acc)[DfCfg<NT>::NG][2][2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int col0 = T.c0 + 16 * (warp / DfCfg<NT>::RW), rw = warp % DfCfg<NT>::RW, ngr = (T.R + 7) >> 3;
    const long long rs = L.rs;
    const bool vec = rs == 1 || rs == -1;
    unsigned paired = 0;
    // all loads first (reversed pairs are swapped once every load is in flight); one column pointer per q
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int c = col0 + 8 * q + lr;
        const bool cok = c < T.c0 + T.wc, fc = c >= T.fr;
        const double* ps = L.at(T.ja, T.ja + c);
        const double* pf = L.src_at(T.ja, T.ja + c);
        const bool al_s = vec && ((reinterpret_cast<uintptr_t>(rs > 0 ? ps : ps - 1) & 15) == 0);
        const bool al_f = vec && ((reinterpret_cast<uintptr_t>(rs > 0 ? pf : pf - 1) & 15) == 0);
#pragma unroll
        for (int t = 0; t < DfCfg<NT>::NG; ++t) {
            const int g = rw + DfCfg<NT>::RW * t, i = 8 * g + 2 * lc;
            acc[t][q][0] = acc[t][q][1] = 0.0;
            if (g >= ngr || !cok || i >= T.R) continue;
            const bool f0 = fc || i >= T.fr, f1 = fc || i + 1 >= T.fr;
            const double* p0 = (f0 ? pf : ps) + i * rs;
            if (i + 1 < T.R && f0 == f1 && (f0 ? al_f : al_s)) {
                const double* lo = rs > 0 ? p0 : p0 - 1;
                const double2 v = f0 ? ld_cg2(lo) : ld_keep2(lo);
                acc[t][q][0] = v.x;
                acc[t][q][1] = v.y;
                paired |= 1u << (2 * t + q);
            } else {
                acc[t][q][0] = ld_cg(p0);
                if (i + 1 < T.R) acc[t][q][1] = ld_cg((f1 ? pf : ps) + (i + 1) * rs);
            }
        }
    }
    if (rs < 0) {
#pragma unroll
        for (int t = 0; t < DfCfg<NT>::NG; ++t)
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (paired >> (2 * t + q) & 1) {
                    const double x = acc[t][q][0];
                    acc[t][q][0] = acc[t][q][1];
                    acc[t][q][1] = x;
                }
    }
}

template <int NT>
__device__ __forceinline__ void df_c_store(const Lu& L, const DfTile& T, const double (&acc)[DfCfg<NT>::NG][2][2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int col0 = T.c0 + 16 * (warp / DfCfg<NT>::RW), rw = warp % DfCfg<NT>::RW, ngr = (T.R + 7) >> 3;
    const long long rs = L.rs;
    const bool vec = rs == 1 || rs == -1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int c = col0 + 8 * q + lr;
        if (c >= T.c0 + T.wc) continue;
        double* ps = L.at(T.ja, T.ja + c);
        const bool al = vec && ((reinterpret_cast<uintptr_t>(rs > 0 ? ps : ps - 1) & 15) == 0);
#pragma unroll
        for (int t = 0; t < DfCfg<NT>::NG; ++t) {
            const int g = rw + DfCfg<NT>::RW * t, i = 8 * g + 2 * lc;
            if (g >= ngr || i >= T.R) continue;
            double* p0 = ps + i * rs;
            if (i + 1 < T.R && al) {
                double2 v;
                v.x = rs > 0 ? acc[t][q][0] : acc[t][q][1];
                v.y = rs > 0 ? acc[t][q][1] : acc[t][q][0];
                st_keep2(rs > 0 ? p0 : p0 - 1, v);
            } else {
                st_keep(p0, acc[t][q][0]);
                if (i + 1 < T.R) st_keep(p0 + rs, acc[t][q][1]);
            }
        }
    }
}

// The C tile (DMMA fragment layout, window columns [0, wc)) into the next panel's buffer: (i, c) -> Pn[c * pld + i]
template <int NT>
__device__ __forceinline__ void df_c_to_smem(const DfTile& T, const double (&acc)[DfCfg<NT>::NG][2][2], double* Pn,
                                             int pld) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int col0 = 16 * (warp / DfCfg<NT>::RW), rw = warp % DfCfg<NT>::RW, ngr = (T.R + 7) >> 3;
#pragma unroll
    for (int t = 0; t < DfCfg<NT>::NG; ++t) {
        const int g = rw + DfCfg<NT>::RW * t;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int c = col0 + 8 * q + lr, i = 8 * g + 2 * lc;
            if (g >= ngr || c >= T.wc || i >= T.R) continue;
            if (i + 1 < T.R)
                *reinterpret_cast<double2*>(Pn + c * pld + i) = make_double2(acc[t][q][0], acc[t][q][1]);
            else
                Pn[c * pld + i] = acc[t][q][0];
        }
    }
}

// A12 rows of step (jb, ja) for window columns [c0, c0 + nc) (nc <= 32 kDfG): -> U[r * uld + c] (zero outside
// the band and for c >= wc); entries in window columns >= fr (or every entry at step 0) have never been
// updated. Column-major over the threads (coalesced band columns), four loads in flight per thread.
template <int NT>
__device__ __forceinline__ void df_a12(const Lu& L, int jb, int ja, int c0, int nc, int wc, int fr, bool first,
                                       double* __restrict__ U, int uld) {
    const int total = 32 * nc;
    for (int e0 = threadIdx.x; e0 < total; e0 += 4 * NT) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT, c = e >> 5, r = e & 31;
            v[u] = 0.0;
            if (e < total && c < wc && 32 + c0 + c - r <= L.K) {
                const int gc = ja + c0 + c;
                v[u] = __ldcg((first || c0 + c >= fr) ? L.src_at(jb + r, gc) : L.at(jb + r, gc));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            if (e < total) U[(e & 31) * uld + (e >> 5)] = v[u];
        }
    }
}

// The chain's strip(s-1, 0) on the FP64 FMA pipe (a DMMA stream on a panel SM would stall the other chain's
// pivot chain): C = window rows [0, R) x columns [0, wc) of step (ja, fr), C -= L21 U12 with the k-sum in the
// reference's order (c -= l_k u_k, k = 0..31, FMA-contracted), the result straight into the next panel
// Pn[c * pld + i] (after the barrier that ends every read of P). Thread: rows (tid % 64) + 64 h, columns
// 8 (tid / 64) + [0, 8) (a warp shares its columns: U12 loads are broadcasts).
template <int NT>
__device__ __forceinline__ void df_chain_update(const Lu& L, const DfTile& T, const double* __restrict__ P,
                                                double* __restrict__ Pn, int pld, const double* __restrict__ U,
                                                int uld) {
    constexpr int RS = NT / 4;  // rows per pass; 4 column groups of 8
    const int i0 = threadIdx.x % RS, cg = threadIdx.x / RS;
    const long long rs = L.rs;
    double c[4][8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int cc = 8 * cg + q;
        const bool fc = cc >= T.fr;
        const double* ps = L.at(T.ja, T.ja + cc);
        const double* pf = L.src_at(T.ja, T.ja + cc);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int i = i0 + RS * h;
            c[h][q] = (i < T.R && cc < T.wc) ? __ldcg(((fc || i >= T.fr) ? pf : ps) + i * rs) : 0.0;
        }
    }
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
        double u[8], l[4];
        const double2* uk = reinterpret_cast<const double2*>(U + k * uld + 8 * cg);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 w = uk[q];
            u[2 * q] = w.x;
            u[2 * q + 1] = w.y;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) l[h] = P[k * pld + 32 + i0 + RS * h];
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int q = 0; q < 8; ++q) c[h][q] = fma(-l[h], u[q], c[h][q]);
    }
    __syncthreads();  // every warp is done with panel s-1
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int i = i0 + RS * h;
        if (i >= T.R) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (8 * cg + q < T.wc) Pn[(8 * cg + q) * pld + i] = c[h][q];
    }
}

// The chain's update split so that the pivot chain overlaps most of it (same per-element FMAs, k ascending, as
// df_chain_update). Top: rows [0, 32) of the new panel -- all the pivot chain needs -- by every thread (row
// tid % 32, a warp shares its columns), written in place (they overwrite only panel s-1's L11\U11, which nobody
// reads any more); rows [R, 32) below a short last block become zeros. Ends with a barrier.
template <int NT>
__device__ __forceinline__ void df_upd_top(const Lu& L, const DfTile& T, double* __restrict__ P, int pld,
                                           const double* __restrict__ U, int uld) {
    constexpr int CPW = 32 / (NT / 32);  // columns per warp
    const int i = threadIdx.x & 31, c0 = CPW * (threadIdx.x >> 5);
    const long long rs = L.rs;
    double c[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int cc = c0 + q;
        const double* p = (cc >= T.fr || i >= T.fr) ? L.src_at(T.ja, T.ja + cc) : L.at(T.ja, T.ja + cc);
        c[q] = (i < T.R && cc < T.wc) ? __ldcg(p + i * rs) : 0.0;
    }
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
        const double l = P[k * pld + 32 + i];
#pragma unroll
        for (int q = 0; q < CPW; ++q) c[q] = fma(-l, U[k * uld + c0 + q], c[q]);
    }
#pragma unroll
    for (int q = 0; q < CPW; ++q)
        if (c0 + q < T.wc) P[(c0 + q) * pld + i] = i < T.R ? c[q] : 0.0;
    __syncthreads();
}

// Rows [32, R) of the new panel by warps 1.. (NT - 32 threads: rows 32 + (t % RS) + RS h, columns 8 (t / RS) +
// [0, 8)) while warp 0 runs the pivot chain; results are written after the group's named barrier ends every
// read of panel s-1's L21 rows (they are overwritten in place).
template <int NT>
__device__ __forceinline__ void df_upd_rest(const Lu& L, const DfTile& T, double* __restrict__ P, int pld,
                                            const double* __restrict__ U, int uld) {
    constexpr int NW = NT - 32, RS = NW / 4;  // 4 column groups of 8; RS * 4 >= MAXK - 32 rows
    const int t = threadIdx.x - 32, i0 = 32 + t % RS, cg = t / RS;
    const long long rs = L.rs;
    double c[4][8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int cc = 8 * cg + q;
        const bool fc = cc >= T.fr;
        const double* ps = L.at(T.ja, T.ja + cc);
        const double* pf = L.src_at(T.ja, T.ja + cc);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int i = i0 + RS * h;
            c[h][q] = (i < T.R && cc < T.wc) ? __ldcg(((fc || i >= T.fr) ? pf : ps) + i * rs) : 0.0;
        }
    }
    if (32 + RS * 3 >= T.R) {  // three row passes cover it (K <= 32 + 3 RS)
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            double u[8], l[3];
            const double2* uk = reinterpret_cast<const double2*>(U + k * uld + 8 * cg);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 w = uk[q];
                u[2 * q] = w.x;
                u[2 * q + 1] = w.y;
            }
#pragma unroll
            for (int h = 0; h < 3; ++h) l[h] = P[k * pld + 32 + i0 + RS * h];
#pragma unroll
            for (int h = 0; h < 3; ++h)
#pragma unroll
                for (int q = 0; q < 8; ++q) c[h][q] = fma(-l[h], u[q], c[h][q]);
        }
    } else {
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            double u[8], l[4];
            const double2* uk = reinterpret_cast<const double2*>(U + k * uld + 8 * cg);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 w = uk[q];
                u[2 * q] = w.x;
                u[2 * q + 1] = w.y;
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) l[h] = P[k * pld + 32 + i0 + RS * h];
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
                for (int q = 0; q < 8; ++q) c[h][q] = fma(-l[h], u[q], c[h][q]);
        }
    }
    named_sync(kBarPg, NW);  // every reader of panel s-1's L21 in this group is done
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int i = i0 + RS * h;
        if (i >= T.R) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (8 * cg + q < T.wc) P[(8 * cg + q) * pld + i] = c[h][q];
    }
}

// U12 = L11^{-1} A12 for nc (<= 32 kDfG) columns: a thread per column, right-looking substitution with every
// index compile-time (x in registers, L11 pairs as 16-byte broadcasts). Element (q, c) receives j = 0..q-1 in
// ascending order with the same FMAs as a column-sequential substitution (block_factors.hpp:246-250 order;
// bitwise panel_rows_cols' column half). Latency ~31 dependent FMAs (the 8-row blocked form with its barriers
// took ~4 us for 96 columns). The final U12 entries (window columns [c0, c0 + wc)) go to the store.
template <int j>
__device__ __forceinline__ void u12_col(double (&x)[32], const double* __restrict__ P, int pld) {
    const double* __restrict__ lj = P + j * pld;  // lj[q] = L11(q, j)
    constexpr int q0 = j + 1;
    if constexpr (q0 < 32 && (q0 & 1)) x[q0] = fma(-lj[q0], x[j], x[q0]);
#pragma unroll
    for (int q = (q0 + 1) & ~1; q < 32; q += 2) {
        const double2 l2 = *reinterpret_cast<const double2*>(lj + q);  // free to hoist (not lds2)
        x[q] = fma(-l2.x, x[j], x[q]);
        x[q + 1] = fma(-l2.y, x[j], x[q + 1]);
    }
    if constexpr (j + 1 < 31) u12_col<j + 1>(x, P, pld);
}

template <int NT>
__device__ __forceinline__ void df_u12(const Lu& L, int jb, int ja, int c0, int nc, int wc,
                                       const double* __restrict__ P, int pld, double* __restrict__ U, int uld) {
    constexpr int B = 32;
    const int tid = threadIdx.x;
    if (tid < nc) {
        double x[B];
#pragma unroll
        for (int q = 0; q < B; ++q) x[q] = U[q * uld + tid];
        u12_col<0>(x, P, pld);
#pragma unroll
        for (int q = 1; q < B; ++q) U[q * uld + tid] = x[q];
    }
    __syncthreads();
    // final U12 entries (the store's A12 rows; evict-first: the factorization is done with them)
    for (int e = tid; e < B * nc; e += NT) {
        const int cc = e >> 5, r = e & 31;
        if (cc < wc && B + c0 + cc - r <= L.K) st_first(L.at(jb + r, ja + c0 + cc), U[r * uld + cc]);
    }
}

// U12 = L11^{-1} A12 (the chain's 32 columns), in 8-row blocks: rows of block b first take j = 0..8b-1 (256
// threads: row 8b + tid/32, columns tid%32 + 32 g), then the block's unit-lower 8 x 8 triangle (thread per
// column). Element (q, c) receives j = 0..q-1 in ascending order with the same FMAs as a column-sequential
// substitution (block_factors.hpp:246-250 order; bitwise panel_rows_cols' column half) with dependent chains
// <= 24 + 7 long. The final U12 entries (window columns [c0, c0 + wc)) go to the store. Ends with a barrier.
template <int NT>
__device__ __forceinline__ void df_u12_blk(const Lu& L, int jb, int ja, int c0, int nc, int wc,
                                       const double* __restrict__ P, int pld, double* __restrict__ U, int uld) {
    constexpr int B = 32, H = 8;
    const int tid = threadIdx.x, rr = tid >> 5, c = tid & 31;
#pragma unroll 1
    for (int b0 = 0; b0 < B; b0 += H) {
        if (b0 > 0 && rr < H) {
            const int q = b0 + rr;
            double x[kDfG];
#pragma unroll
            for (int g = 0; g < kDfG; ++g) x[g] = c + 32 * g < nc ? U[q * uld + c + 32 * g] : 0.0;
            const double* __restrict__ lq = P + q;
#pragma unroll 4
            for (int j = 0; j < b0; ++j) {
                const double l = lq[j * pld];
#pragma unroll
                for (int g = 0; g < kDfG; ++g)
                    if (c + 32 * g < nc) x[g] = fma(-l, U[j * uld + c + 32 * g], x[g]);
            }
#pragma unroll
            for (int g = 0; g < kDfG; ++g)
                if (c + 32 * g < nc) U[q * uld + c + 32 * g] = x[g];
        }
        if (b0 > 0) __syncthreads();
        if (tid < nc) {
            double x[H];
#pragma unroll
            for (int r = 0; r < H; ++r) x[r] = U[(b0 + r) * uld + tid];
#pragma unroll
            for (int j = 0; j + 1 < H; ++j) {
                const double* __restrict__ lj = P + (b0 + j) * pld + b0;
#pragma unroll
                for (int r = j + 1; r < H; ++r) x[r] = fma(-lj[r], x[j], x[r]);
            }
#pragma unroll
            for (int r = 0; r < H; ++r) U[(b0 + r) * uld + tid] = x[r];
        }
        __syncthreads();
    }
    // final U12 entries (the store's A12 rows; evict-first: the factorization is done with them)
    for (int e = tid; e < B * nc; e += NT) {
        const int cc = e >> 5, r = e & 31;
        if (cc < wc && B + c0 + cc - r <= L.K) st_first(L.at(jb + r, ja + c0 + cc), U[r * uld + cc]);
    }
}

// C -= L21 U12 (C^T -= U12^T L21^T, k-steps of 4 in order: k_band_lu_res' fragments and order)
template <int NT>
__device__ __forceinline__ void df_dmma(const DfTile& T, const double* __restrict__ P, int pld,
                                        const double* __restrict__ U, int uld, double (&acc)[DfCfg<NT>::NG][2][2]) {
    constexpr int nb = 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    const int cp = warp / DfCfg<NT>::RW, rw = warp % DfCfg<NT>::RW, ngr = (T.R + 7) >> 3;
    const double* pk = P + nb + lr;
    const double* uk = U + 16 * cp + lr;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        const int kk = ks * 4 + lc;
        const double a0 = uk[kk * uld], a1 = uk[kk * uld + 8];
#pragma unroll
        for (int t = 0; t < DfCfg<NT>::NG; ++t) {
            const int g = rw + DfCfg<NT>::RW * t;
            if (g < ngr) {
                const double b = -pk[kk * pld + 8 * g];
                dmma_m8n8k4(acc[t][0][0], acc[t][0][1], a0, b, acc[t][0][0], acc[t][0][1]);
                dmma_m8n8k4(acc[t][1][0], acc[t][1][1], a1, b, acc[t][1][0], acc[t][1][1]);
            }
        }
    }
}

// L21 rows of a factored diagonal block: panel_rows_cols' row half (thread per row, the same operations, hence
// the same bits) for any number of rows over NT threads
template <int B, bool FULL, int NT>
__device__ __noinline__ void df_rows(double* __restrict__ P, int pld, const double* __restrict__ Ut,
                                     const double* __restrict__ s_piv, int nb_rt, int ph) {
    const int nb = FULL ? B : nb_rt;
    for (int r = nb + (int)threadIdx.x; r < ph; r += NT) {
        double x[B];
#pragma unroll
        for (int c = 0; c < B; ++c) x[c] = c < nb ? P[c * pld + r] : 0.0;
#pragma unroll
        for (int c = 0; c < B; ++c) {
            if (c < nb) {
                const double l = div_rcp(x[c], s_piv[c], s_piv[B + c]);
                x[c] = l;
                const double2* __restrict__ u2 = reinterpret_cast<const double2*>(Ut + ut_off(c) - ut_lo(c));
#pragma unroll
                for (int j0 = (c + 1) & ~1; j0 < B; j0 += 8) {  // 4 pairs per batch: one load latency each
                    double2 u[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (j0 + 2 * q < B) u[q] = lds2(reinterpret_cast<const double*>(u2 + ((j0 >> 1) + q)));
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = j0 + 2 * q;
                        if (j < B) {
                            if (j > c) x[j] = fma(-l, u[q].x, x[j]);
                            x[j + 1] = fma(-l, u[q].y, x[j + 1]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < B; ++c)
            if (c < nb) P[c * pld + r] = x[c];
    }
}

// ---- chain item (panel SMs): strip(s-1, 0) -- the update of block s -- fused with panel(s) -----------------
template <int NT, bool STREAM>
__device__ __forceinline__ void df_chain(const DfArgs& A, const FactorJob& J, int jid, int s, double* __restrict__ P,
                                         double* __restrict__ U, double* __restrict__ s_ut,
                                         double* __restrict__ s_rcp, int* s_boosts, bool have_panel) {
    constexpr int B = 32;
    const int m = J.m, K = J.k;
    if (s * B >= m) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int pld = A.pld, uld = A.uld;
    const int jb = s * B, nb = min(B, m - jb), ph = min(nb + K, m - jb), ja = jb + nb;
    const int R = min(K, m - ja);
    const int rprev = s > 0 ? min(K, m - jb) : 0;  // window s-1 rows; panel rows >= rprev are fresh
    const double scale = STREAM ? 0.0 : *J.scale;
    Lu L{J.base, J.rs, J.cs, m, K, B, pld, uld, STREAM ? 0.0 : A.eps * (scale > 0 ? scale : 1.0),
         J.src ? J.src : J.base};
    const int nbn = ja < m ? min(B, m - ja) : 0;
    // step s-1 (the strip that produces this panel)
    const int sp = s - 1, jbp = jb - B, rprevp = sp > 0 ? min(K, m - jbp) : 0;
    const DfTile T{jb, rprev, 0, min(B, rprev), sp > 0 ? rprevp - B : 0};
    if (warp == 0) {
        if (STREAM) df_wait_cols(J, ja + R + nbn + 1);
        if (s > 0) df_wait(A.panel_cnt + jid, s, A.err, A.panel_cnt, 1);
        if (sp > 0 && B < rprevp) df_wait(A.col_step + (size_t)jid * A.S + s, sp, A.err, A.panel_cnt, 2);
        if (lane == 0) {
            df_acquire();
            *s_boosts = 0;
            if (A.trace) g_df_smark[0] = clock64();
        }
    }
    __syncthreads();
    if (s > 0) {
        // panel s-1: still in shared memory when this CTA factored it (job owner), else from L2
        if (!have_panel) df_stage_panel<NT>(L, P, pld, jbp, jbp, B + rprev, B, B + rprev);
        df_a12<NT>(L, jbp, jb, 0, 32, T.wc, T.fr, sp == 0, U, uld);
        // this panel's rows that no earlier step updated (<= 32 of them), loaded now by warps 1.. and written
        // once the update has finished reading panel s-1
        constexpr int NW = NT - 32, NF = (1024 + NW - 1) / NW;
        double fv[NF];
#pragma unroll
        for (int u = 0; u < NF; ++u) {
            const int e = tid - 32 + u * NW, c = e >> 5, r = rprev + (e & 31);
            fv[u] = (warp > 0 && e < 1024 && c < nb && r < ph && L.inband(r, c)) ? __ldcg(L.src_at(jb + r, jb + c))
                                                                                  : 0.0;
        }
        __syncthreads();
        DF_MARK(1);
        df_u12_blk<NT>(L, jbp, jb, 0, 32, T.wc, P, pld, U, uld);  // all warps (the 1-warp form ran slower here)
        df_upd_top<NT>(L, T, P, pld, U, uld);
        DF_MARK(2);
        if (warp == 0) {
            if (nb == B)
                panel_diag<B, true>(P, pld, s_ut, s_rcp, nb, L.bv, s_boosts, A.trace ? g_df_pmark : nullptr);
            else
                panel_diag<B, false>(P, pld, s_ut, s_rcp, nb, L.bv, s_boosts, A.trace ? g_df_pmark : nullptr);
            DF_MARK(3);
        } else {
            df_upd_rest<NT>(L, T, P, pld, U, uld);
#pragma unroll
            for (int u = 0; u < NF; ++u) {
                const int e = tid - 32 + u * NW, c = e >> 5, r = rprev + (e & 31);
                if (e < 1024 && r < pld) P[c * pld + r] = fv[u];
            }
            if (A.trace && tid == 32) g_df_pmark[9] = clock64();
        }
    } else {
        df_stage_panel<NT>(L, P, pld, jb, jb, ph, nb, 0);
        __syncthreads();
        DF_MARK(2);
        if (warp == 0) {
            if (nb == B)
                panel_diag<B, true>(P, pld, s_ut, s_rcp, nb, L.bv, s_boosts, A.trace ? g_df_pmark : nullptr);
            else
                panel_diag<B, false>(P, pld, s_ut, s_rcp, nb, L.bv, s_boosts, A.trace ? g_df_pmark : nullptr);
            DF_MARK(3);
        }
    }
    __syncthreads();
    // L21 rows (thread per row; panel_rows_cols' row half)
    if (nb == B)
        df_rows<B, true, NT>(P, pld, s_ut, s_rcp, nb, ph);
    else
        df_rows<B, false, NT>(P, pld, s_ut, s_rcp, nb, ph);
    __syncthreads();
    DF_MARK(4);
    // the panel is final: L11\U11 and L21 to the store (the worker strips of this step read it from L2); row pairs
    // (r, r + 1), r even, as one 16-byte store where both are in the band (alignment is uniform per column)
    const long long rs = L.rs;
    const unsigned long long pol = l2_normal_policy();
    for (int c = warp; c < nb; c += NT / 32) {
        double* g = L.at(jb, jb + c);
        const int r0 = max(c - K, 0), r1 = min(ph, c + K + 1);
        const bool al = (rs == 1 || rs == -1) && ((reinterpret_cast<uintptr_t>(rs > 0 ? g : g - 1) & 15) == 0);
        const double* pc = P + c * pld;
        for (int r = 2 * lane; r < r1; r += 64) {
            const bool in0 = r >= r0, in1 = r + 1 >= r0 && r + 1 < r1;
            const double2 v = *reinterpret_cast<const double2*>(pc + r);
            if (in0 && in1 && al) {
                const double2 w = rs > 0 ? v : make_double2(v.y, v.x);
                asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(rs > 0 ? g + r : g - r - 1),
                             "d"(w.x), "d"(w.y), "l"(pol) : "memory");
            } else {
                if (in0) asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(g + r * rs), "d"(v.x),
                                      "l"(pol) : "memory");
                if (in1) asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(g + (r + 1) * rs),
                                      "d"(v.y), "l"(pol) : "memory");
            }
        }
    }
    // (no L2 prefetch of step s+1's first band entries here: 64 bulk prefetches cost the chain ~1.4 us, more than
    // the worker loads they would speed up)
    __syncthreads();
    if (tid == 0) {
        if (A.trace) g_df_smark[6] = clock64();
        const int nbst = *s_boosts;
        if (nbst) atomicAdd(A.boost_acc + jid, nbst);
        if (jb + nb >= m) *J.boosts = atomicAdd(A.boost_acc + jid, 0);  // the job's last panel
        st_release_i(A.panel_cnt + jid, s + 1);  // after the CTA barrier: publishes every thread's stores
        if (A.trace) g_df_smark[7] = clock64();
    }
}

// ---- worker item (worker SMs): strips j = 1 + kDfG g .. of step s -------------------------------------------
// One panel load, one A12 load and one U12 solve for the group; then per strip: C tile in, DMMA, C tile out and
// its column block's flag released at once (the chain two steps on waits for strip 1 only).
template <int NT, bool STREAM>
__device__ __forceinline__ void df_worker(const DfArgs& A, const FactorJob& J, int jid, int s, int g,
                                          double* __restrict__ P, double* __restrict__ U) {
    constexpr int B = 32;
    const int m = J.m, K = J.k;
    const int jb = s * B;
    if (jb + B >= m) return;  // no trailing window (a strip step always has nb = 32)
    const int nb = B, ja = jb + nb, R = min(K, m - ja), ph = nb + R;
    const int j0 = 1 + A.grp * g, c0 = 32 * j0;
    if (c0 >= R) return;
    const int j1 = min(j0 + A.grp, (R + 31) / 32);  // strips [j0, j1)
    const int tid = threadIdx.x;
    const int pld = A.pld, uld = A.uld;
    const int rprev = s > 0 ? min(K, m - jb) : 0;
    const int fr = s > 0 ? rprev - nb : 0;
    Lu L{J.base, J.rs, J.cs, m, K, B, pld, uld, 0.0, J.src ? J.src : J.base};
    if (tid < 32) {
        if (STREAM) df_wait_cols(J, ja + R + 1);
        df_wait(A.panel_cnt + jid, s + 1, A.err, A.panel_cnt, 3);
        for (int j = j0; j < j1; ++j)
            if (s > 0 && 32 * (j + 1) < rprev)
                df_wait(A.col_step + (size_t)jid * A.S + s + 1 + j, s, A.err, A.panel_cnt, 4);
        if (tid == 0) {
            df_acquire();
            if (A.trace) g_df_smark[0] = clock64();
        }
    }
    __syncthreads();
    df_stage_panel<NT>(L, P, pld, jb, jb, ph, B, ph);
    df_a12<NT>(L, jb, ja, c0, 32 * (j1 - j0), R - c0, fr, s == 0, U, uld);
    __syncthreads();
    DF_MARK(1);
    df_u12<NT>(L, jb, ja, c0, 32 * (j1 - j0), R - c0, P, pld, U, uld);
    DF_MARK(2);
    for (int j = j0; j < j1; ++j) {
        const DfTile T{ja, R, 32 * j, min(32, R - 32 * j), fr};
        double acc[DfCfg<NT>::NG][2][2];
        df_c_load<NT>(L, T, acc);
        df_dmma<NT>(T, P, pld, U + 32 * (j - j0), uld, acc);
        df_c_store<NT>(L, T, acc);
        __syncthreads();
        if (tid == 0) st_release_i(A.col_step + (size_t)jid * A.S + s + 1 + j, s + 1);
    }
    if (tid == 0) {
        DF_MARK(3);
        DF_MARK(4);
    }
}

// Panel SMs take chain items from counter_p in order (s-major); the other SMs take worker items from counter_w
// in wave order. Both orders are consistent with one topological order (chain(s) ~ 2s,
// strip(s, .) ~ 2s + 1), so the earliest unfinished item is always grabbed and runnable: no deadlock.
template <int NT, bool STREAM>
__global__ void __launch_bounds__(NT, DfCfg<NT>::MINB) k_band_lu_df(DfArgs A) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(16) double s_ut[kUtSize];
    __shared__ double s_rcp[64];
    __shared__ int s_item, s_boosts;
    {
        const int* gate = A.jobs[0].gate;
        if (!STREAM && gate && !(*gate & 1)) return;  // the streamed refactor: nothing to redo
    }
    double* P = smem;
    double* U = smem + 32 * A.pld;
    const int tid = threadIdx.x, J = A.njobs;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    // SM role: the first nps SMs on which CTAs of this launch actually start become panel SMs (placement and
    // %smid numbering are not under our control; every CTA of an SM shares its SM's role)
    __shared__ int s_role, s_rank, s_mode;
    if (tid < 32) {  // warp 0 together (lane 0 does the atomics): no divergent spin (df_wait)
        const bool l0 = tid == 0;
        int* rp = A.sm_role + (smid % kDfMaxSm);
        int r = __shfl_sync(0xffffffffu, l0 ? atomicCAS(rp, 0, 3) : 0, 0);
        if (r == 0) {
            r = __shfl_sync(0xffffffffu, l0 ? (atomicAdd(A.n_panel_sm, 1) < A.nps ? 1 : 2) : 0, 0);
            if (l0) atomicExch(rp, r);
        } else {
            while (r == 3) {
                __nanosleep(20);
                r = ld_relaxed_w(rp);
            }
            if (r == 1 && A.excl) r = 0;  // exclusive panel SM: only its deciding CTA stays
        }
        if (l0) {
            s_role = r;
            s_rank = r == 1 ? atomicAdd(A.n_chain, 1) : -1;
            __threadfence();
            atomicAdd(A.started, 1);
        }
    }
    __syncthreads();
    if (s_role == 0) {
        // spare CTA of an exclusive panel SM: it holds the slot (so no other kernel's CTAs land beside the
        // pivot chain) until every chain item has been taken
        if (tid == 0)
            while (ld_relaxed_i(reinterpret_cast<const int*>(A.counter_p)) < A.S * J) __nanosleep(4000);
        return;
    }
    const bool panel_role = s_role == 1;
    if (panel_role) {
        // Job owners when every CTA of the launch is resident and there is a chain CTA per job: chain CTA r runs
        // chain(r, 0), chain(r, 1), ... and keeps each panel in shared memory for the next step. Deadlock-free like
        // the queue (each job's items run in order on a resident CTA; the workers' queue is unchanged). Otherwise
        // (a CTA still waiting for a slot after 200 us, or fewer chain CTAs than jobs) the shared queue. The wait
        // covers the side stream's block norms / zero padding, launched just ahead of a resident-band LU: their
        // short CTAs hold some SMs for a few tens of us, and a 20 us limit sent ~1 launch in 20 to the queue
        // (LU+UL 4.1 -> 6.9 ms in that step); the loop exits as soon as every CTA has started.
        if (tid < 32) {
            int md = ld_relaxed_w(A.mode);
            if (md == 0) {
                const unsigned long long t0 = __shfl_sync(0xffffffffu, df_now(), 0);
                while (ld_relaxed_w(A.started) < (int)gridDim.x &&
                       __shfl_sync(0xffffffffu, df_now(), 0) - t0 < 200000)
                    __nanosleep(64);
                const int want =
                    A.owners_ok && ld_relaxed_w(A.started) == (int)gridDim.x && ld_relaxed_w(A.n_chain) >= J ? 1 : 2;
                md = __shfl_sync(0xffffffffu, tid == 0 ? atomicCAS(A.mode, 0, want) : 0, 0);
                if (md == 0) md = want;
            }
            if (tid == 0) s_mode = md;
        }
        __syncthreads();
        if (s_mode == 1) {
            const int jid = s_rank;
            if (jid >= J) return;
            const FactorJob Jb = A.jobs[jid];
            for (int s = 0; s < A.S && s * 32 < Jb.m; ++s) {
                unsigned long long t_grab = 0;
                if (A.trace && tid == 0) {
                    t_grab = df_now();
                    for (int q = 0; q < 8; ++q) if (q != 5) g_df_smark[q] = 0;
                    for (int q = 0; q < 10; ++q) g_df_pmark[q] = 0;
                    g_df_smark[5] = clock64();
                }
                df_chain<NT, STREAM>(A, Jb, jid, s, P, U, s_ut, s_rcp, &s_boosts, s > 0);
                __syncthreads();
                if (A.trace && tid == 0) {
                    const unsigned long long c_end = clock64();
                    unsigned long long* tr = A.trace + kDfRec * ((size_t)gridDim.x + (size_t)s * J + jid);
                    tr[0] = t_grab;
                    tr[1] = df_now();
                    tr[2] = g_df_smark[5];
                    for (int q = 0; q < 5; ++q) tr[3 + q] = g_df_smark[q];
                    tr[8] = c_end;
                    tr[9] = ((unsigned long long)smid << 32) | blockIdx.x;
                    for (int q = 0; q < 10; ++q) tr[10 + q] = g_df_pmark[q];
                    tr[20] = g_df_smark[6];
                    tr[21] = g_df_smark[7];
                }
            }
            if (tid == 0) atomicAdd(A.counter_p, (unsigned)A.S);  // releases the exclusive SMs' spare CTAs
            return;
        }
    }
    unsigned* ctr = panel_role ? A.counter_p : A.counter_w;
    if (tid == 0) s_item = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    // worker wave cursor: wave w holds strips [w0, w0 + wn) (J x (strips - 1) of step w)
    int w = 0, w0 = 0;
    auto wave_n = [&](int ww) {  // worker items of step ww: J x ceil((strips - 1) / grp)
        const int R = min(A.K, A.m_max - 32 * (ww + 1));
        return J * (((R + 31) / 32 - 1 + A.grp - 1) / A.grp);
    };
    int wn = A.S >= 2 ? wave_n(0) : 0;
    for (;;) {
        const int item = s_item;
        __syncthreads();
        if (tid == 0) s_item = (int)atomicAdd(ctr, 1u);
        unsigned long long t_grab = 0;
        if (A.trace && tid == 0) {
            t_grab = df_now();
            for (int q = 0; q < 8; ++q) if (q != 5) g_df_smark[q] = 0;
            for (int q = 0; q < 10; ++q) g_df_pmark[q] = 0;
            g_df_smark[5] = clock64();
        }
        long long rec;
        if (panel_role) {
            if (item >= A.S * J) break;
            const int s = item / J, jid = item - s * J;
            const FactorJob Jb = A.jobs[jid];
            df_chain<NT, STREAM>(A, Jb, jid, s, P, U, s_ut, s_rcp, &s_boosts, false);
            rec = item;
        } else {
            bool done = false;
            while (item >= w0 + wn) {
                w0 += wn;
                ++w;
                if (w > A.S - 2) {
                    done = true;
                    break;
                }
                wn = wave_n(w);
            }
            if (done) break;
            const int ng = wn / J, o = item - w0, jid = o / ng;
            const FactorJob Jb = A.jobs[jid];
            df_worker<NT, STREAM>(A, Jb, jid, w, o % ng, P, U);
            rec = (long long)A.S * J + item;
        }
        __syncthreads();
        if (A.trace && tid == 0) {
            // record (10 u64): grab / end (globaltimer ns), grab / ready / marks 1-4 / end (clock64), SM << 32 | CTA
            const unsigned long long c_end = clock64();
            unsigned long long* tr = A.trace + kDfRec * ((size_t)gridDim.x + rec);
            tr[0] = t_grab;
            tr[1] = df_now();
            tr[2] = g_df_smark[5];
            for (int q = 0; q < 5; ++q) tr[3 + q] = g_df_smark[q];
            tr[8] = c_end;
            tr[9] = ((unsigned long long)smid << 32) | blockIdx.x;
            for (int q = 0; q < 10; ++q) tr[10 + q] = g_df_pmark[q];
            tr[20] = g_df_smark[6];
            tr[21] = g_df_smark[7];
        }
    }
}

static int g_df_owners = 1;      // sap_dev_lu_df_owners
static int g_df_group = 0;       // sap_dev_lu_df_group (0: auto)
static int g_df_trace_mode = 0;  // sap_dev_lu_df_trace_mode: 1 trace streamed launches, 2 the others
static unsigned long long* g_df_trace = nullptr;
static size_t g_df_trace_cap = 0;
static long long g_df_trace_items = 0;
static int g_df_trace_grid = 0;

// scratch: [1..7] timeout report, [8] chain counter, [10] worker counter, [12] panel SMs claimed, [13] chain CTAs,
// [14] CTAs started, [15] chain schedule,
// [16, 16 + kDfMaxSm) SM roles, then panel_cnt[njobs], boost_acc[njobs], col_step[njobs][S]
constexpr int kDfHdr = 16 + kDfMaxSm;
size_t lu_df_scratch_ints(int njobs, int m_max) {
    const int S = (m_max + 31) / 32;
    return kDfHdr + 2 * (size_t)njobs + (size_t)njobs * S;
}

// Where the dataflow kernel beats one CTA per job (profiles/lu_df_r02.txt): wide bands (enough strips per step
// to spread), at least 16 steps per job, and no more jobs than ~0.7 x SMs (one chain CTA per job on the panel SMs, the rest for workers;
// with more jobs the single-CTA kernel's per-flop efficiency wins)
bool lu_df_applies(int max_k, int njobs, int m_max) {
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (max_k > 224) return max_k <= 512;  // no resident single-CTA kernel beyond K = 224
    // short jobs (e.g. the reduced blocks, m = w: 7 steps) do not amortize the items' latency
    return max_k >= kLuDfMinK && 10 * njobs <= 7 * nsm && m_max >= 16 * 32;
}

void launch_band_lu_df(const FactorJob* d_jobs, int njobs, int m_max, int max_k, double eps, cudaStream_t s,
                       bool streamed, int* scratch) {
    constexpr int B = 32;
    const int S = (m_max + B - 1) / B;
    // [1..7]: timeout report (cleared by lu_df_clear_error, kept across launches); [8], [10]: work counters
    SAP_CUDA(cudaMemsetAsync(scratch + 8, 0, sizeof(int) * (lu_df_scratch_ints(njobs, m_max) - 8), s));
    DfArgs A;
    A.jobs = d_jobs;
    A.njobs = njobs;
    A.m_max = m_max;
    A.K = max_k;
    A.S = S;
    A.counter_p = reinterpret_cast<unsigned*>(scratch + 8);
    A.counter_w = reinterpret_cast<unsigned*>(scratch + 10);
    A.err = scratch + 1;
    A.n_panel_sm = scratch + 12;
    A.n_chain = scratch + 13;
    A.started = scratch + 14;
    A.mode = scratch + 15;
    A.owners_ok = g_df_owners;
    A.sm_role = scratch + 16;
    A.panel_cnt = scratch + kDfHdr;
    A.boost_acc = scratch + kDfHdr + njobs;
    A.col_step = scratch + kDfHdr + 2 * njobs;
    A.eps = eps;
    A.pld = pad_ld(B + max_k);
    A.uld = pad_ld(32 * kDfG);
    A.trace = nullptr;
    const size_t bytes = sizeof(double) * (size_t)(B * A.pld + B * A.uld);
    const bool wide = max_k > DfCfg<256>::MAXK;
    if (max_k > DfCfg<512>::MAXK) throw InvalidArgument("band LU (dataflow): half-bandwidth above 512");
    const int nt = wide ? 512 : 256;
    void (*kern)(DfArgs) = wide ? (streamed ? k_band_lu_df<512, true> : k_band_lu_df<512, false>)
                                : (streamed ? k_band_lu_df<256, true> : k_band_lu_df<256, false>);
    SAP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    int dev = 0, nsm = 0, per_sm = 0;
    SAP_CUDA(cudaGetDevice(&dev));
    SAP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SAP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, bytes));
    const int grid = nsm * std::max(per_sm, 1);
    // panel SMs: one resident chain per job (chains are latency-bound), at most 40 % of the SMs; when every
    // job gets a panel SM to itself (few jobs), it is exclusive: no other chain CTA on its SM
    const int cap = (2 * nsm) / 5;
    A.excl = (njobs <= cap || per_sm <= 1) ? 1 : 0;  // one CTA per SM (wide bands) is exclusive anyway
    int nps = A.excl ? std::min(njobs, cap) : std::min((njobs + per_sm - 1) / std::max(per_sm, 1), cap);
    A.nps = std::max(1, std::min(nps, nsm - 1));
    // strips per worker item: a group waits for the previous step's group to finish (its strips shifted by one),
    // so the group's duration bounds the step period; few jobs leave worker SMs idle enough for shorter groups
    A.grp = g_df_group > 0 ? std::min(g_df_group, kDfG) : (A.excl ? 2 : kDfG);
    // chain items (one per job and step) + worker strips
    long long items = (long long)njobs * S;
    for (int w = 0; w <= S - 2; ++w)
        items += (long long)njobs * (((std::min(max_k, m_max - B * (w + 1)) + 31) / 32 - 1 + A.grp - 1) / A.grp);
    if (g_df_trace_mode && (g_df_trace_mode == 1) == streamed) {  // tools/lu_df_trace.py
        const size_t need = kDfRec * (size_t)(grid + items);
        if (g_df_trace_cap < need) {
            if (g_df_trace) cudaFree(g_df_trace);
            SAP_CUDA(cudaMalloc(&g_df_trace, need * sizeof(unsigned long long)));
            g_df_trace_cap = need;
        }
        SAP_CUDA(cudaMemsetAsync(g_df_trace, 0, need * sizeof(unsigned long long), s));
        A.trace = g_df_trace;
        g_df_trace_items = items;
        g_df_trace_grid = grid;
    }
    kern<<<grid, nt, bytes, s>>>(A);
    SAP_LAUNCHED();
}

void lu_df_clear_error(int* scratch, cudaStream_t s) { SAP_CUDA(cudaMemsetAsync(scratch, 0, sizeof(int) * 8, s)); }

int lu_df_error(const int* scratch, int* detail) {
    int e[8] = {};
    SAP_CUDA(cudaMemcpy(e, scratch + 1, sizeof(e), cudaMemcpyDeviceToHost));
    if (detail)
        for (int i = 0; i < 7; ++i) detail[i] = e[i];
    return e[0];
}

// True when launch_band_lu_ws will run k_band_lu_res for this bandwidth: that kernel reads every
// never-updated entry from FactorJob::src, so the factor stores need no initial copy of the band
// (only their out-of-matrix slots zeroed, launch_zero_pad).
bool band_lu_reads_source(int max_k) {
    constexpr int B = 32;
    if (max_k < 1 || max_k > 256 - B) return false;
    const int pldr = pad_ld(B + max_k), uldr = pad_ld(max_k);
    return sizeof(double) * (size_t)(2 * B * pldr + 2 * B * uldr) <= kResSmemMax;
}

}  // namespace sapgpu

// tools/lu_df_trace.py only (not in include/sap_gpu.h): the last traced k_band_lu_df launch, 10 u64 per item
// (grab, end: globaltimer ns; grab, dependencies met, phase marks 1-4, end: clock64; SM << 32 | CTA).
extern "C" void sap_dev_lu_df_trace_mode(int mode) { sapgpu::g_df_trace_mode = mode; }
// tools only: 0 keeps the dataflow LU's chain items on the shared queue (no job owners), 1 the default
extern "C" void sap_dev_lu_df_owners(int on) { sapgpu::g_df_owners = on; }
// tools only: strips per worker item (1..3; 0 = auto)
extern "C" void sap_dev_lu_df_group(int g) { sapgpu::g_df_group = g; }

extern "C" long long sap_dev_lu_df_trace(unsigned long long* out, long long cap) {
    using namespace sapgpu;
    if (!g_df_trace) return 0;
    const long long n = std::min<long long>(cap, g_df_trace_items);
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_df_trace + kDfRec * (size_t)g_df_trace_grid, sizeof(unsigned long long) * kDfRec * n,
               cudaMemcpyDeviceToHost);
    return n;
}
