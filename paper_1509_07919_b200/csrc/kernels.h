// Host-side launchers of the SaP sm_100a kernels. All launch on `s` and are
// asynchronous; none synchronizes.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace sapgpu {

// ---- factorization (factor.cu) ----
// Infinity norm of every diagonal block, restricted to in-block columns
// (factor_blocks' boost scale, block_factors.hpp:187-195). p blocks, offsets on device.
// store == nullptr: `band` is one contiguous band (the A operator); otherwise the
// blocks live in a BandStore.
// d_nrows (optional): only rows r < d_nrows[b] of block b count (third-stage reduced blocks diag(R_t, I)).
void launch_block_norms(const double* band, int max_m, int k, const int* d_offsets, int p, const BandStore* store,
                        double* norms, cudaStream_t s,
                        int* nonfinite = nullptr, const int* d_nrows = nullptr, bool f32 = false);
// LU (and UL) BandStores = each diagonal block's band, entries outside the block zeroed.
void launch_copy_blocks(const double* band, int k, const int* d_offsets, int p, const BandStore& st, double* lu,
                        double* ul, cudaStream_t s);
// Blocked no-pivot LU with pivot boosting of every job (one CTA per job).
// streamed: the jobs carry FactorJob::ready (k_band_lu_res<B, true>; only where band_lu_reads_source(max_k))
// df_scratch (lu_df_scratch_ints(njobs, m_max) ints, owned by the caller, one launch at a time): run the
// dataflow kernel k_band_lu_df over every SM where it applies (lu_df_applies(max_k)); m_max = largest job.
// lu_kernel: sap_options::lu_kernel (0 automatic, 1 one CTA per job, 2 dataflow where supported)
void launch_band_lu(const FactorJob* d_jobs, int njobs, int max_k, double boost_eps, cudaStream_t s,
                    bool streamed = false, int m_max = 0, int* df_scratch = nullptr, int lu_kernel = 0);
size_t lu_df_scratch_ints(int njobs, int m_max);
bool lu_df_applies(int max_k, int njobs, int m_max);
void launch_band_lu_df(const FactorJob* d_jobs, int njobs, int m_max, int max_k, double eps, cudaStream_t s,
                       bool streamed, int* scratch);
// 1 if a dependency wait of the last k_band_lu_df launch on this scratch timed out (synchronous read);
// detail (optional, 7 ints): flag, CTA, SM, flag word offset from panel_cnt, want, have, wait site
int lu_df_error(const int* scratch, int* detail = nullptr);
void lu_df_clear_error(int* scratch, cudaStream_t s);
// The warp-specialized look-ahead variant (lu.cu); false if the smem budget does not fit.
bool band_lu_reads_source(int max_k);
void launch_zero_pad(int k, const int* d_offsets, int p, const BandStore& st, double* lu, double* ul, cudaStream_t s);
// streamed upload: *bad = 1 if some job's min |pivot| < boost_eps * ||A_b|| (refactor with boosting), 2 on a stall
void launch_stream_check(const FactorJob* d_jobs, const double* minpiv, const double* norms, int njobs, int p,
                         double eps, int* bad, cudaStream_t s);
bool launch_band_lu_ws(const FactorJob* d_jobs, int njobs, int max_k, double boost_eps, cudaStream_t s,
                       bool streamed = false);
// Row-sum infinity norms of ni dense row-major w x w blocks and a non-finite flag per block.
void launch_dense_norms(const double* a, int w, int ni, double* norms, int* nonfinite, cudaStream_t s);

// ---- FP32 preconditioner (mixed.cu): build_precond_op<float> (pipeline.hpp:140-202) ----
struct FactorJobF {  // FactorJob at T = float (base = the float store's strided view)
    float* base;
    long long rs, cs;
    int m, k;
    const double* scale;  // block norm of the float band (k_block_norms<true>), device
    int* boosts;
};
struct TipJobF {  // TipJob at T = float
    const float* f;
    int corner;
    int which;
    const float* rhs;
    float* out;
    int flag;
};
void launch_copy_blocks_f32(const double* band, int k, const int* d_offsets, int p, const BandStore& st, float* lu,
                            float* ul, cudaStream_t s);
void launch_band_lu_f32(const FactorJobF* d_jobs, int njobs, int max_k, double boost_eps, cudaStream_t s);
void launch_spike_tips_f32(const TipJobF* d_jobs, int njobs, int k, int* nonfinite, cudaStream_t s);
// R_t = I - W_t V_t and its boosted dense LU, written in the reduced BandStore layout (k' = w - 1)
void launch_rbar_f32(const float* wt, const float* vb, int w, int ni, double boost_eps, float* rbar,
                     const BandStore& rst, int* boosts, int* nonfinite, cudaStream_t s);

// ---- spikes (spike.cu) ----
// d_wid (optional, third stage): interface widths w_t <= k embedded in the k x k corners (third.cu).
void launch_extract_coupling(const double* band, int n, int k, const int* d_offsets, int p, double* bblk,
                             double* cblk, cudaStream_t s, const int* d_wid = nullptr);
// One spike tip (compute_spike_tips, spike.hpp:190-250): which 0 -> V^b = U^{-1} L^{-1} rhs on the
// trailing corner of an LU block; which 1 -> W^t = L^{-1} U^{-1} rhs on the leading corner of a UL block.
struct TipJob {
    const double* f;    // the block's band (BandStore block base)
    int corner;         // first row/col of the w x w corner inside the block
    int which;
    const double* rhs;  // B or C corner, row-major w x w
    double* out;        // row-major w x w
    int flag;           // nonfinite[flag] set on a non-finite tip
};
void launch_spike_tips(const TipJob* d_jobs, int njobs, int k, int* nonfinite, cudaStream_t s);
// One coupling corner (which 0: B at boundary e, 1: C) of a band with n columns.
void launch_extract_one(const double* band, int n, int k, int e, int which, double* out, cudaStream_t s);
// rbar[t] = I - wt[t] * vb[t], written in band layout (k = w-1) of the block-diagonal
// matrix diag(rbar_0, ..., rbar_{ni-1}); nonfinite[t] flags a non-finite block.
void launch_rbar(const double* wt, const double* vb, int w, int ni, double* rbar_band, const BandStore& rst,
                 int* nonfinite, cudaStream_t s);

// ---- third stage: per-block reordering (third.cu) ----
// P_b A_b P_b^T at bandwidth kb[b] into the (zeroed) LU store; *bad = min block with an entry outside.
void launch_assemble_blocks(const double* band, int n, int k, const int* d_offsets, int p, const int* d_gperm,
                            const int* d_has_perm, const int* d_kb, const BandStore& st, double* lu, int* bad,
                            cudaStream_t s);
struct FullSpikeJob {
    const double* f;  // block LU: (i, j) at f[j * 2k + i]
    double* x;        // m x k row-major: the right-hand sides in, the spike out
    int m;
    int first_row;    // right-hand-side rows above it are zero
    int flag;         // nonfinite[flag] set on a non-finite spike entry
    int col_lo, col_hi;  // columns outside [col_lo, col_hi) have zero right-hand sides (and stay zero)
    int kb;              // the block's bandwidth K_b <= k: factor entries beyond it are zero
    int blk;             // block index (its chunk inverses)
};
void launch_full_rhs(const double* bblk, const double* cblk, int k, const int* d_offsets, int ni,
                     const int* d_gperm, double* vfull, double* wfull, cudaStream_t s);
// dinv (nullable): the LU plan's 32-row chunk inverses, used when *kappa <= kappa_max; else substitution
void launch_full_spikes(const FullSpikeJob* d_jobs, int njobs, int k, int* nonfinite, const double* dinv, int nch_max,
                        const unsigned long long* kappa, double kappa_max, cudaStream_t s);
size_t full_spike_smem(int k);
void launch_full_tips(const double* vfull, const double* wfull, int k, const int* d_offsets, int ni,
                      const int* d_gperm, const int* d_wid, double* vb, double* wt, cudaStream_t s);
template <class T>
void launch_permute(const int* d_gperm, const T* in, T* out, int n, bool scatter, cudaStream_t s);

// ---- preconditioner apply (apply.cu) ----
// Everything a block sweep needs, built once at setup: the factor BandStore,
// its overlapping 3-D TMA view and the per-chunk diagonal inverses.
template <class T>
struct SweepPlan {
    const T* f = nullptr;       // BandStore base (LU factors)
    BandStore st;
    const int* offs = nullptr;  // device block offsets (p+1)
    int p = 0, k = 0;
    bool tma = false;
    int tr = 32, stages = 3, nbox = 1, box_c = 0, xw = 0, nch_max = 0;
    size_t smem = 0;
    T* dinv = nullptr;          // [p][nch_max][2][tr*tr] chunk inverses
    T* tri = nullptr;           // [p][nch_max][2][tr*tr] the chunk triangles themselves (substitution)
    unsigned long long* kappa = nullptr;  // device: max chunk-triangle condition estimate (double bits)
    bool subst = false;         // sweeps solve chunk triangles by substitution (ill-conditioned triangles)
    const int* kb = nullptr;    // third stage: per-block half-bandwidth K_b <= k (device), nullptr = k
    bool ul = false;            // f is a UL store (A = U'L'): bottom-up sweep first (k_sweep_tma<UL>)
    CUtensorMap map;
};
// Elements of chunk-inverse storage the plan needs (0 when the TMA path is not used).
template <class T>
size_t sweep_dinv_elems(const SweepPlan<T>& pl);
// Chooses the sweep kernel and encodes the tensor map (pl.f/st/offs/p/k set by the caller).
template <class T>
void plan_sweeps(SweepPlan<T>& pl, T* dinv_storage);
template <class T>
void launch_chunk_inverses(const SweepPlan<T>& pl, cudaStream_t s);
// x <- D^{-1} x per block with the LU factors (band_lu_solve, block_factors.hpp:74-90).
// tip_rows > 0: the second sweep stops once the tip_rows rows it reaches first are final (LU: the last rows
// of every block, UL: the first); the other rows of x are then intermediate values.
// xsrc != nullptr: the right-hand side is read from xsrc (not modified) and the solution written to x.
template <class T>
void launch_block_solve(const SweepPlan<T>& pl, T* x, cudaStream_t s, int tip_rows = 0, const T* xsrc = nullptr);
// SaP-C interface step (apply_preconditioner, spike.hpp:323-347): from g (= D^{-1} b) form
// x^t (xt), x^b (xb) per interface and subtract the coupling terms from b2 (which holds b).
// rbar_band: the reduced blocks' LU in band layout (k = w-1), blocks at d_roffsets (t*w).
template <class T>
// Interface t sits at row d_ioffs[t + 1] of g / b2 (t < ni). On a multi-GPU rank the first / last
// interface may cross to a neighbour: skip_first_b / skip_last_c drop the update of the rows the
// neighbour owns (g then carries the neighbour's w rows as a halo on that side).
void launch_interfaces(const T* g, const int* d_ioffs, const SweepPlan<T>& rplan, int ni, int k, const T* wt,
                       const T* vb, const T* bblk, const T* cblk, T* xt, T* xb, T* b2, bool skip_first_b,
                       bool skip_last_c, cudaStream_t s, const T* gtop = nullptr);
// f32: build_precond_op<float>'s diagonal (pipeline.hpp:151-161 at T = float): the diagonal and the boost
// value rounded to float, the apply b / diag in float between casts (spike.hpp:304-351).
void launch_diag_apply(const double* in, const double* diag, double* out, int n, cudaStream_t s, bool f32 = false);
void launch_boosted_diag(const double* band, int n, int k, const double* scale, double boost_eps, double* diag,
                         cudaStream_t s, bool f32 = false);

// ---- operators (spmv.cu) ----
// y = A x on the band; if b != nullptr also y = b - A x.
void launch_band_spmv(const double* band, int n, int k, const double* x, double* y, const double* b, cudaStream_t s);
// y0 = A x0 and y1 = A x1 in one read of the band (each bitwise launch_band_spmv's)
void launch_band_spmv2(const double* band, int n, int k, const double* x0, double* y0, const double* x1, double* y1,
                       cudaStream_t s);
// y[i - r0] = sum_j A(i, j) x[j], rows [r0, r1) of a band with n columns (x indexed like the band's columns).
void launch_band_spmv_rows(const double* band, int n, int k, int r0, int r1, const double* x, double* y, cudaStream_t s);
// w x w row-major GEMV: mode 0: y = u - A v;  mode 1: y -= A v.
void launch_gemv_w(const double* A, int w, const double* v, const double* u, double* y, int mode, cudaStream_t s);
// bad == nullptr: entries outside k are dropped (drop_off's filter) instead of flagged
void launch_assemble_band(const int* rp, const int* ci, const double* v, int n, int k, double* band,
                          unsigned long long* bad, cudaStream_t s);
// drop_off's half-bandwidth (pipeline.hpp:59-99) of a CSR matrix on the device (synchronizes s).
int drop_off_k(const int* rp, const int* ci, const double* v, int n, int nnz, double tol, cudaStream_t s);
void launch_csr_spmv(const int* rp, const int* ci, const double* v, int n, const double* x, double* y,
                     const double* b, cudaStream_t s);

// ---- vector kernels (vec.cu) ----
// Deterministic reductions: fixed partition of [0, n) into blocks, fixed tree.
int reduce_blocks(int n);
constexpr int kMaxDots = 4;
struct DotBatch {  // up to kMaxDots dot products in one pass (kind 1: squared norm of a - b)
    const double* a[kMaxDots];
    const double* b[kMaxDots];
    int kind[kMaxDots];
    int m;
    // optional: the results also written to host-mapped memory, and *flag_dst = *flag_src, by the kernel itself
    // (the host reads them after its stream synchronisation with no device->host copy on the stream)
    double* hout;
    const int* flag_src;
    int* flag_dst;
};
void launch_dots(const DotBatch& d, int n, double* partials, unsigned* counter, double* out, cudaStream_t s);
void launch_axpy_quot(double* y, const double* num, const double* den, const double* x, int n, cudaStream_t s);
// *counter must be 0 on entry (the kernel leaves it 0).
void launch_dot(const double* a, const double* b, int n, double* partials, unsigned* counter, double* out,
                cudaStream_t s);
void launch_nonfinite(const double* a, int n, int* flag, cudaStream_t s);
void launch_cast_d2f(const double* in, float* out, int n, cudaStream_t s);
void launch_cast_f2d(const float* in, double* out, int n, cudaStream_t s);
template <class T>
void launch_cast_band(const double* in, T* out, size_t count, cudaStream_t s);

}  // namespace sapgpu
