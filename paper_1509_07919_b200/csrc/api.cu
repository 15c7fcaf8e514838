// C ABI (include/sap_gpu.h) over the SaP B200 kernels.
//
// The handle plays the role of the reference's PrecondState<T> +
// LinearOp closures (proj/include/sap/pipeline.hpp:130-202): setup builds the
// factors, coupling corners, spike tips and reduced blocks in HBM once;
// every later apply / solve reuses them (the reference rebuilds per solve;
// persisting factors across right-hand sides is the paper's stated use,
// PAPER.md:408).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/sap_gpu.h"
#include "common.cuh"
#include "kernels.h"
#include "comm_nccl.h"
#include "krylov.h"

using namespace sapgpu;

namespace {

thread_local std::string g_last_error;

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count == n && p) return;
        release();
        if (count == 0) return;
        SAP_CUDA(cudaMalloc(&p, sizeof(T) * count));
        n = count;
    }
    T* get() const { return p; }
};

struct Layout {
    int n = 0, p = 0, k = 0;
    std::vector<int> sizes, offsets;
};

// make_partition_layout (proj/include/sap/partition.hpp:42-69), same messages.
Layout make_layout(int n, int p, int k) {
    if (n <= 0) throw InvalidArgument("make_partition_layout: empty matrix");
    if (p <= 0) throw InvalidArgument("make_partition_layout: partition count must be positive");
    if (k < 0) throw InvalidArgument("make_partition_layout: negative bandwidth");
    const int base = n / p, rem = n % p;
    const int required = k == 0 ? 1 : 2 * k;
    if (base < required)
        throw InvalidArgument("make_partition_layout: " + std::to_string(p) + " partitions leave blocks under " +
                              std::to_string(required) + " rows for half-bandwidth " + std::to_string(k) +
                              "; largest feasible p is " + std::to_string(sap_max_feasible_partitions(n, k)));
    Layout L;
    L.n = n;
    L.p = p;
    L.k = k;
    L.sizes.resize(p);
    L.offsets.resize(p + 1);
    L.offsets[0] = 0;
    for (int i = 0; i < p; ++i) {
        L.sizes[i] = base + (i < rem ? 1 : 0);
        L.offsets[i + 1] = L.offsets[i] + L.sizes[i];
    }
    return L;
}

}  // namespace

struct sap_handle {
    sap_options opt{};
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    cudaEvent_t ev[12] = {};
    // SaP-C setup: the sweep chunk inverses run on `side` while extract/tips/rbar continue on `stream`
    cudaStream_t side = nullptr;
    cudaEvent_t sev[2] = {};
    // setup runs on `prio` (highest priority, joined to the caller's stream at entry) so that the side
    // stream's work (lowest priority: chunk inverses, norms, upload) fills the SMs the main chain leaves idle
    cudaStream_t prio = nullptr;
    cudaEvent_t pev = nullptr;
    // problem
    bool ready = false;
    int n = 0, k = 0;
    Layout layout;
    int kind = SAP_PRECOND_COUPLED;
    bool coupled = false;  // coupled && p > 1
    DevBuf<int> d_offsets, d_roffsets;
    const double* band_ptr = nullptr;  // A operator band (owned copy or borrowed)
    DevBuf<double> band, lu, ul, norms, bblk, cblk, vb, wt, rbar, rbar_norms, diag, scratch_g, scratch_in,
        scratch_out, dscal, xt, xb;
    DevBuf<int> boosts, rbar_boosts, nonfinite;
    DevBuf<FactorJob> jobs, rjobs;
    DevBuf<int> lu_scr;  // k_band_lu_df work counter and dependency flags (one launch at a time on the stream)
    BandStore fst, rst;                  // LU/UL and reduced-block stores
    DevBuf<double> dinv, rdinv;          // chunk inverses (+ triangles) for the sweeps
    DevBuf<unsigned long long> kappa;    // [0] LU plan, [1] reduced plan: chunk-triangle condition estimates
    DevBuf<int> op_nonfinite;            // any non-finite entry in the banded operator (single-GPU setup)
    bool op_finite = false;              // checked: the zero-guess shortcut of the Krylov solver applies
    SweepPlan<double> lplan, rplan;      // block sweeps over LU and over the reduced blocks
    // SaP-C apply, first block solve: only the rows the interfaces read are needed -- each block's last w rows
    // from an LU sweep pair whose second sweep stops there, its first w rows from a UL sweep pair (uplan over the
    // UL store) on tside, both at once (sap_options::tip_solve; used when no pivot was boosted and the chunk
    // triangles of both stores are well conditioned)
    bool ul_tips = false;
    SweepPlan<double> uplan;
    DevBuf<double> udinv, scratch_gu;
    cudaStream_t tside = nullptr;
    cudaEvent_t tev[2] = {};
    // mixed precision (KrylovOptions::mixed_precision, build_precond_op<float>): the preconditioner is
    // applied in FP32 from FP32 copies of the factors, tips and reduced factors
    bool mixed = false;
    DevBuf<float> lu_f, rbar_f, vb_f, wt_f, bblk_f, cblk_f, dinv_f, rdinv_f, g_f, o_f, xt_f, xb_f;
    // f32fac: the block preconditioner was FACTORED in FP32 (build_precond_op<float>; setup_mixed): the
    // parity getters read the FP32 factors / tips / reduced blocks
    bool f32fac = false;
    DevBuf<float> ul_f;
    DevBuf<FactorJobF> fjobs;
    DevBuf<TipJobF> ftipjobs;
    DevBuf<unsigned long long> kappa_f;
    SweepPlan<float> lplan_f, rplan_f;
    // CSR operator
    bool csr = false;
    bool diag_f32 = false;  // diagonal preconditioner built and applied in float (mixed_precision)
    int csr_n = 0;
    DevBuf<int> rp, ci;
    DevBuf<double> vals;
    DevBuf<double> asm_band;             // sap_setup_banded_from_csr: the band assembled on the device
    DevBuf<int> asm_rp, asm_ci;
    DevBuf<double> asm_v;
    DevBuf<unsigned long long> asm_bad;
    cudaEvent_t cev[3] = {};  // CSR setups: drop_off and assembly timers (T_Drop, T_Asmbl)
    DevBuf<TipJob> tipjobs;
    // third stage (sap_set_third_stage): ThirdStageResult (reorder_cm.hpp:227-231) applied at setup
    bool ts_armed = false;  // set by the caller; consumed by every following block setup
    bool ts = false;        // the current setup runs the third-stage path
    std::vector<int> ts_k, ts_has, ts_perm, widths;
    DevBuf<int> d_gperm, d_has, d_kb, d_wid, d_bad;
    DevBuf<double> vfull, wfull, norms_op, scratch_p;
    DevBuf<float> scratch_pf;
    DevBuf<FullSpikeJob> fsjobs;
    // streamed band upload (host band): LU overlapped with the host->device copy
    DevBuf<unsigned> d_ready;
    DevBuf<double> d_minpiv;
    DevBuf<int> d_sbad;
    DevBuf<FactorJob> sjobs, gjobs;  // streamed jobs, gated refactor jobs
    cudaEvent_t sev_norm = nullptr;
    // multi-GPU (sap_create_distributed): this rank owns global rows [row_lo, row_hi) = partitions
    // [pb, pe); the band slice holds global columns [c_lo, c_hi). Interface slots are ordered
    // [left cross?, local 0..p_loc-2, right cross?]; cross interfaces are solved on both ranks.
    bool dist = false;
    sap_comm comm{};
    NcclComm* nccl = nullptr;  // native data plane (sap_create_distributed_nccl); else the comm callbacks
    DevBuf<double> dred;       // device staging of host-side reductions over NCCL
    Layout glayout;
    int n_glob = 0, row_lo = 0, row_hi = 0, c_lo = 0, c_hi = 0, pb = 0, pe = 0, ni_tot = 0;
    bool has_left = false, has_right = false;
    DevBuf<int> d_ioffs, d_boffs;
    DevBuf<double> xext;
    // Krylov
    KrylovSolver krylov;
    DevBuf<double> kb, kx;
    sap_report rep{};
};

namespace {

template <class F>
sap_status guard(F&& f) {
    try {
        f();
        return SAP_OK;
    } catch (const InvalidArgument& e) {
        g_last_error = e.what();
        return SAP_ERR_INVALID_ARGUMENT;
    } catch (const PreconditionerFailure& e) {
        g_last_error = e.what();
        return SAP_ERR_PRECONDITIONER;
    } catch (const CudaFailure& e) {
        g_last_error = e.what();
        return SAP_ERR_CUDA;
    } catch (const StateError& e) {
        g_last_error = e.what();
        return SAP_ERR_STATE;
    } catch (const CommFailure& e) {
        g_last_error = e.what();
        return SAP_ERR_COMM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SAP_ERR_CUDA;
    }
}

// grows only: a launch already enqueued on the handle's stream may still use the buffer
int* lu_scratch(sap_handle* h, int njobs, int m_max) {
    const size_t need = lu_df_scratch_ints(njobs, m_max);
    if (h->lu_scr.n < need) h->lu_scr.alloc(need);
    return h->lu_scr.get();
}

// k_band_lu_df: a dependency wait that timed out (never expected) fails the setup instead of returning
// factors computed from stale data
void lu_check(sap_handle* h) {
    if (!h->lu_scr.get()) return;
    int d[7];
    if (lu_df_error(h->lu_scr.get(), d))
        throw CudaFailure("band LU (k_band_lu_df): dependency wait timed out (CTA " + std::to_string(d[1]) + ", SM " +
                          std::to_string(d[2]) + ", flag " + std::to_string(d[3]) + " want " + std::to_string(d[4]) +
                          " have " + std::to_string(d[5]) + ", site " + std::to_string(d[6]) + ")");
}

void require(bool c, const char* msg) {
    if (!c) throw InvalidArgument(msg);
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    SAP_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// M^{-1}: the reference's apply_preconditioner (spike.hpp:304-351) over the
// handle's device factors. in/out are device pointers; they may alias.
// Sweeps on ill-conditioned chunk triangles (max ||T|| ||T^-1|| over chunks above kSubstKappa: element
// growth at low diagonal dominance) solve them by substitution (k_sweep_tma<SUBST>); well conditioned
// factors keep the chunk-inverse product. sap_options::triangle_solve (1 inverse, 2 substitution) forces it.
constexpr double kSubstKappa = 1e4;
// The LU and UL tip sweeps of a SaP-C apply run side by side, one CTA per block each: they pay only while both
// launches fit on the SMs at once (with more blocks the sweeps run in waves and the pair costs about a full
// solve; config 5, P = 512, keeps the LU solve).
bool tip_sweeps_fit(int blocks) {
    int dev = 0, nsm = 0;
    SAP_CUDA(cudaGetDevice(&dev));
    SAP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    return 2 * blocks <= nsm;
}
void choose_triangle_solve(sap_handle* h) {
    int nf = 1;
    if (!h->dist && h->op_nonfinite.get())
        SAP_CUDA(cudaMemcpy(&nf, h->op_nonfinite.get(), sizeof(int), cudaMemcpyDeviceToHost));
    h->op_finite = nf == 0;
    unsigned long long kb[2] = {0, 0};
    if (h->kappa.get()) SAP_CUDA(cudaMemcpy(kb, h->kappa.get(), sizeof(kb), cudaMemcpyDeviceToHost));
    double kap[2];
    std::memcpy(kap, kb, sizeof(kap));
    const int force = h->opt.triangle_solve;
    h->lplan.subst = force ? force == 2 : kap[0] > kSubstKappa;
    h->rplan.subst = force ? force == 2 : kap[1] > kSubstKappa;
    h->rep.chunk_condition = kap[0];
    h->rep.sweep_substitution = h->lplan.subst ? 1 : 0;
    h->lplan_f.subst = h->lplan.subst;
    h->rplan_f.subst = h->rplan.subst;
}

void apply_m_dist(sap_handle* h, const double* in, double* out);
void apply_a_dist(sap_handle* h, const double* in, double* out);

// FP32 copies of everything the preconditioner apply reads (factor stores, chunk inverses recomputed in
// FP32 from the FP32 factors, tips, couplings, reduced factors). The factorization itself ran in FP64
// (the DMMA kernels): the reference's build_precond_op<float> factors in FP32, so the FP32 operands
// here differ from its by FP32 rounding -- both are FP32-accurate preconditioners.
void build_fp32_preconditioner(sap_handle* h, cudaStream_t s) {
    h->mixed = true;
    const int p = h->layout.p, k = h->k;
    h->lu_f.alloc(h->fst.total(p));
    launch_cast_band<float>(h->lu.get(), h->lu_f.get(), h->fst.total(p), s);
    h->kappa_f.alloc(2);
    SAP_CUDA(cudaMemsetAsync(h->kappa_f.get(), 0, 2 * sizeof(unsigned long long), s));
    SweepPlan<float>& lp = h->lplan_f;
    lp = SweepPlan<float>{};
    lp.f = h->lu_f.get();
    lp.st = h->fst;
    lp.offs = h->d_offsets.get();
    lp.p = p;
    lp.k = k;
    h->dinv_f.alloc(std::max<size_t>(sweep_dinv_elems(lp), 1));
    plan_sweeps(lp, h->dinv_f.get());
    lp.kappa = h->kappa_f.get();
    lp.kb = h->ts ? h->d_kb.get() : nullptr;
    launch_chunk_inverses(lp, s);
    if (h->coupled && k > 0) {
        const int ni = p - 1;
        const size_t ww = (size_t)k * k * ni;
        h->vb_f.alloc(ww);
        h->wt_f.alloc(ww);
        h->bblk_f.alloc(ww);
        h->cblk_f.alloc(ww);
        launch_cast_band<float>(h->vb.get(), h->vb_f.get(), ww, s);
        launch_cast_band<float>(h->wt.get(), h->wt_f.get(), ww, s);
        launch_cast_band<float>(h->bblk.get(), h->bblk_f.get(), ww, s);
        launch_cast_band<float>(h->cblk.get(), h->cblk_f.get(), ww, s);
        h->rbar_f.alloc(std::max<size_t>(h->rst.total(ni), 1));
        launch_cast_band<float>(h->rbar.get(), h->rbar_f.get(), h->rst.total(ni), s);
        SweepPlan<float>& rp = h->rplan_f;
        rp = SweepPlan<float>{};
        rp.f = h->rbar_f.get();
        rp.st = h->rst;
        rp.offs = h->d_roffsets.get();
        rp.p = ni;
        rp.k = k - 1;
        h->rdinv_f.alloc(std::max<size_t>(sweep_dinv_elems(rp), 1));
        plan_sweeps(rp, h->rdinv_f.get());
        rp.kappa = h->kappa_f.get() + 1;
        launch_chunk_inverses(rp, s);
        h->xt_f.alloc(std::max<size_t>((size_t)ni * k, 1));
        h->xb_f.alloc(std::max<size_t>((size_t)ni * k, 1));
    }
    h->g_f.alloc(std::max(h->n, 1));
    h->o_f.alloc(std::max(h->n, 1));
}

// M^{-1} in FP32 (apply_preconditioner<float>, spike.hpp:304-351 with pipeline.hpp:191-200's casts)
void apply_m_fp32(sap_handle* h, const double* in, double* out) {
    const cudaStream_t s = h->stream;
    const int n = h->n, p = h->layout.p, k = h->k;
    float* o = h->o_f.get();
    launch_cast_d2f(in, o, n, s);
    // block_solve with block permutations (block_factors.hpp:222-229): gather, sweep, scatter back
    auto solve = [&](float* v) {
        if (!h->ts) return launch_block_solve<float>(h->lplan_f, v, s);
        float* t = h->scratch_pf.get();
        launch_permute<float>(h->d_gperm.get(), v, t, n, true, s);
        launch_block_solve<float>(h->lplan_f, t, s);
        launch_permute<float>(h->d_gperm.get(), t, v, n, false, s);
    };
    if (h->coupled) {
        float* g = h->g_f.get();
        SAP_CUDA(cudaMemcpyAsync(g, o, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        solve(g);
        launch_interfaces<float>(g, h->d_offsets.get(), h->rplan_f, p - 1, k, h->wt_f.get(), h->vb_f.get(),
                                 h->bblk_f.get(), h->cblk_f.get(), h->xt_f.get(), h->xb_f.get(), o, false, false, s);
    }
    solve(o);
    launch_cast_f2d(o, out, n, s);
}

void apply_m(sap_handle* h, const double* in, double* out) {
    if (h->dist) return apply_m_dist(h, in, out);
    const cudaStream_t s = h->stream;
    const int n = h->n;
    const size_t bytes = sizeof(double) * (size_t)n;
    switch (h->kind) {
        case SAP_PRECOND_NONE:
            if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
            return;
        case SAP_PRECOND_DIAGONAL:
            launch_diag_apply(in, h->diag.get(), out, n, s, h->diag_f32);
            return;
        default:
            break;
    }
    if (h->mixed) return apply_m_fp32(h, in, out);
    const int p = h->layout.p, k = h->k;
    if (h->ts) {
        // block_solve with block permutations (block_factors.hpp:222-229): gather, sweep, scatter back
        double* t = h->scratch_p.get();
        launch_permute<double>(h->d_gperm.get(), in, t, n, true, s);
        launch_block_solve<double>(h->lplan, t, s);
        if (!h->coupled) return launch_permute<double>(h->d_gperm.get(), t, out, n, false, s);
        double* g = h->scratch_g.get();
        launch_permute<double>(h->d_gperm.get(), t, g, n, false, s);
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        launch_interfaces<double>(g, h->d_offsets.get(), h->rplan, p - 1, k, h->wt.get(), h->vb.get(),
                                  h->bblk.get(), h->cblk.get(), h->xt.get(), h->xb.get(), out, false, false, s);
        launch_permute<double>(h->d_gperm.get(), out, t, n, true, s);
        launch_block_solve<double>(h->lplan, t, s);
        launch_permute<double>(h->d_gperm.get(), t, out, n, false, s);
        return;
    }
    if (!h->coupled) {
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        launch_block_solve<double>(h->lplan, out, s);
        return;
    }
    double* g = h->scratch_g.get();
    if (h->ul_tips) {
        // the interfaces read g's last w rows of every block (LU sweeps, the backward one stopped there) and
        // its first w rows (UL sweeps on tside, the top-down one stopped there), computed side by side; both
        // read `in` and write their own copies
        double* gu = h->scratch_gu.get();
        SAP_CUDA(cudaEventRecord(h->tev[0], s));
        SAP_CUDA(cudaStreamWaitEvent(h->tside, h->tev[0], 0));
        launch_block_solve<double>(h->uplan, gu, h->tside, k, in);
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        launch_block_solve<double>(h->lplan, g, s, k, in);
        SAP_CUDA(cudaEventRecord(h->tev[1], h->tside));
        SAP_CUDA(cudaStreamWaitEvent(s, h->tev[1], 0));
        launch_interfaces<double>(g, h->d_offsets.get(), h->rplan, p - 1, k, h->wt.get(), h->vb.get(),
                                  h->bblk.get(), h->cblk.get(), h->xt.get(), h->xb.get(), out, false, false, s, gu);
        launch_block_solve<double>(h->lplan, out, s);
        return;
    }
    SAP_CUDA(cudaMemcpyAsync(g, in, bytes, cudaMemcpyDeviceToDevice, s));
    if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
    launch_block_solve<double>(h->lplan, g, s);
    launch_interfaces<double>(g, h->d_offsets.get(), h->rplan, p - 1, k, h->wt.get(), h->vb.get(), h->bblk.get(),
                              h->cblk.get(), h->xt.get(), h->xb.get(), out, false, false, s);
    launch_block_solve<double>(h->lplan, out, s);
}

void apply_a(sap_handle* h, const double* in, double* out) {
    if (h->dist)
        apply_a_dist(h, in, out);
    else if (h->csr)
        launch_csr_spmv(h->rp.get(), h->ci.get(), h->vals.get(), h->csr_n, in, out, nullptr, h->stream);
    else
        launch_band_spmv(h->band_ptr, h->n, h->k, in, out, nullptr, h->stream);
}

int op_n(const sap_handle* h) { return h->csr ? h->csr_n : h->n; }

// cuStreamWriteValue32 (stream memory operation: the copy engine's stream writes the round counter
// without an SM, so the factorization kernel polling it can never starve it)
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value_fn() {
    static WriteValue32Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WriteValue32Fn>(p);
        cudaGetLastError();
    }
    return fn;
}

constexpr int kUploadRounds = 24;

// Setup on the high-priority stream: it waits for the caller's stream at entry; setup_banded ends with a
// synchronize, so nothing needs joining back.
struct PrioScope {
    sap_handle* h;
    cudaStream_t user;
    explicit PrioScope(sap_handle* hh) : h(hh), user(hh->stream) {
        SAP_CUDA(cudaEventRecord(h->pev, user));
        SAP_CUDA(cudaStreamWaitEvent(h->prio, h->pev, 0));
        h->stream = h->prio;
    }
    ~PrioScope() {
        if (h->stream == h->prio) {  // on an exception: the caller's stream must still see the setup's work
            cudaEventRecord(h->pev, h->prio);
            cudaStreamWaitEvent(user, h->pev, 0);
        }
        h->stream = user;
    }
};

// build_precond_op<float> (pipeline.hpp:140-202) for the block preconditioners: banded_cast<float> of the
// resident band into the LU / UL stores, block norms over the float entries (accumulated in double,
// block_factors.hpp:187-195), FP32 LU / UL with boosting (mixed.cu), the coupling corners in float, FP32 spike
// tips and reduced blocks, then the FP32 sweep plans the apply uses (apply_m_fp32). T_* timers as in the
// FP64 setup; the FP64 factors are not built.
void setup_mixed(sap_handle* h, const Layout& L, bool want_ul) {
    const cudaStream_t s = h->stream;
    const int n = h->n, k = h->k, p = L.p;
    h->mixed = true;
    h->f32fac = true;
    SAP_CUDA(cudaEventRecord(h->ev[1], s));  // the band is resident
    h->d_offsets.alloc(p + 1);
    SAP_CUDA(cudaMemcpyAsync(h->d_offsets.get(), L.offsets.data(), sizeof(int) * (p + 1), cudaMemcpyHostToDevice, s));
    h->norms.alloc(p);
    h->boosts.alloc(2 * (size_t)p);
    SAP_CUDA(cudaMemsetAsync(h->boosts.get(), 0, sizeof(int) * 2 * p, s));
    SAP_CUDA(cudaMemsetAsync(h->norms.get(), 0, sizeof(double) * p, s));
    h->op_nonfinite.alloc(1);
    SAP_CUDA(cudaMemsetAsync(h->op_nonfinite.get(), 0, sizeof(int), s));
    const int m_max = L.sizes[0];
    h->fst = BandStore::make(m_max, k);
    h->lu.release();
    h->ul.release();
    h->lu_f.alloc(h->fst.total(p));
    if (want_ul)
        h->ul_f.alloc(h->fst.total(p));
    else
        h->ul_f.release();
    launch_block_norms(h->band_ptr, m_max, k, h->d_offsets.get(), p, nullptr, h->norms.get(), s,
                       h->op_nonfinite.get(), nullptr, true);
    launch_copy_blocks_f32(h->band_ptr, k, h->d_offsets.get(), p, h->fst, h->lu_f.get(), want_ul ? h->ul_f.get() : nullptr,
                           s);
    const int njobs = want_ul ? 2 * p : p;
    std::vector<FactorJobF> jobs(njobs);
    const size_t w = 2 * (size_t)k + 1;
    for (int b = 0; b < p; ++b) {
        const int m = L.sizes[b];
        jobs[b] = FactorJobF{h->lu_f.get() + h->fst.block(b) + k, 1, 2LL * k, m, k, h->norms.get() + b,
                             h->boosts.get() + b};
        if (want_ul)
            jobs[p + b] = FactorJobF{h->ul_f.get() + h->fst.block(b) + (size_t)(m - 1) * w + k, -1, -2LL * k, m, k,
                                     h->norms.get() + b, h->boosts.get() + p + b};
    }
    h->fjobs.alloc(njobs);
    SAP_CUDA(cudaMemcpyAsync(h->fjobs.get(), jobs.data(), sizeof(FactorJobF) * njobs, cudaMemcpyHostToDevice, s));
    SAP_CUDA(cudaEventRecord(h->ev[8], s));
    launch_band_lu_f32(h->fjobs.get(), njobs, k, h->opt.boost_eps, s);
    SAP_CUDA(cudaEventRecord(h->ev[9], s));
    h->kappa_f.alloc(2);
    SAP_CUDA(cudaMemsetAsync(h->kappa_f.get(), 0, 2 * sizeof(unsigned long long), s));
    {
        SweepPlan<float>& lp = h->lplan_f;
        lp = SweepPlan<float>{};
        lp.f = h->lu_f.get();
        lp.st = h->fst;
        lp.offs = h->d_offsets.get();
        lp.p = p;
        lp.k = k;
        h->dinv_f.alloc(std::max<size_t>(sweep_dinv_elems(lp), 1));
        plan_sweeps(lp, h->dinv_f.get());
        lp.kappa = h->kappa_f.get();
        launch_chunk_inverses(lp, s);
    }
    SAP_CUDA(cudaEventRecord(h->ev[2], s));
    for (int b = 0; b < p; ++b) {
        const double m = L.sizes[b], kk = std::min<double>(k, m - 1 > 0 ? m - 1 : 0);
        const double f = (m - kk) * (2 * kk * kk + kk) + (kk - 1) * kk * (4 * kk + 1) / 6.0;
        h->rep.factor_flops += (want_ul ? 2.0 : 1.0) * f;
    }
    int ni = 0;
    if (h->coupled) {
        ni = p - 1;
        const size_t ww = (size_t)k * k * ni;
        h->rst = BandStore::make(k, k > 0 ? k - 1 : 0);
        h->bblk.alloc(std::max<size_t>(ww, 1));
        h->cblk.alloc(std::max<size_t>(ww, 1));
        h->bblk_f.alloc(std::max<size_t>(ww, 1));
        h->cblk_f.alloc(std::max<size_t>(ww, 1));
        h->vb_f.alloc(std::max<size_t>(ww, 1));
        h->wt_f.alloc(std::max<size_t>(ww, 1));
        h->rbar_f.alloc(std::max<size_t>(h->rst.total(ni), 1));
        SAP_CUDA(cudaMemsetAsync(h->rbar_f.get(), 0, sizeof(float) * h->rst.total(ni), s));
        h->rbar_boosts.alloc(ni);
        h->nonfinite.alloc(3 * (size_t)ni);
        SAP_CUDA(cudaMemsetAsync(h->nonfinite.get(), 0, sizeof(int) * 3 * ni, s));
        SAP_CUDA(cudaMemsetAsync(h->rbar_boosts.get(), 0, sizeof(int) * ni, s));
        h->xt_f.alloc(std::max<size_t>((size_t)ni * k, 1));
        h->xb_f.alloc(std::max<size_t>((size_t)ni * k, 1));
        std::vector<int> roffs(ni + 1);
        for (int t = 0; t <= ni; ++t) roffs[t] = t * k;
        h->d_roffsets.alloc(ni + 1);
        SAP_CUDA(cudaMemcpyAsync(h->d_roffsets.get(), roffs.data(), sizeof(int) * (ni + 1), cudaMemcpyHostToDevice, s));
        // T_BC: extract_coupling<float> = the FP64 corners rounded to float (the band is cast entrywise)
        launch_extract_coupling(h->band_ptr, n, k, h->d_offsets.get(), p, h->bblk.get(), h->cblk.get(), s);
        launch_cast_band<float>(h->bblk.get(), h->bblk_f.get(), ww, s);
        launch_cast_band<float>(h->cblk.get(), h->cblk_f.get(), ww, s);
        SAP_CUDA(cudaEventRecord(h->ev[3], s));
        // T_SPK: compute_spike_tips<float>
        std::vector<TipJobF> tj;
        for (int t = 0; t < ni; ++t) {
            const size_t o = (size_t)t * k * k;
            tj.push_back(TipJobF{h->lu_f.get() + h->fst.block(t), L.sizes[t] - k, 0, h->bblk_f.get() + o,
                                 h->vb_f.get() + o, 2 * t});
            tj.push_back(TipJobF{h->ul_f.get() + h->fst.block(t + 1), 0, 1, h->cblk_f.get() + o, h->wt_f.get() + o,
                                 2 * t + 1});
        }
        h->ftipjobs.alloc(std::max<size_t>(tj.size(), 1));
        SAP_CUDA(cudaMemcpyAsync(h->ftipjobs.get(), tj.data(), sizeof(TipJobF) * tj.size(), cudaMemcpyHostToDevice, s));
        launch_spike_tips_f32(h->ftipjobs.get(), (int)tj.size(), k, h->nonfinite.get(), s);
        SAP_CUDA(cudaEventRecord(h->ev[4], s));
        // T_LUrdcd: finish_reduced_blocks<float>
        if (k > 0) {
            launch_rbar_f32(h->wt_f.get(), h->vb_f.get(), k, ni, h->opt.boost_eps, h->rbar_f.get(), h->rst,
                            h->rbar_boosts.get(), h->nonfinite.get() + 2 * ni, s);
            SweepPlan<float>& rp = h->rplan_f;
            rp = SweepPlan<float>{};
            rp.f = h->rbar_f.get();
            rp.st = h->rst;
            rp.offs = h->d_roffsets.get();
            rp.p = ni;
            rp.k = k - 1;
            h->rdinv_f.alloc(std::max<size_t>(sweep_dinv_elems(rp), 1));
            plan_sweeps(rp, h->rdinv_f.get());
            rp.kappa = h->kappa_f.get() + 1;
            launch_chunk_inverses(rp, s);
        }
        SAP_CUDA(cudaEventRecord(h->ev[5], s));
    }
    h->g_f.alloc(std::max(n, 1));
    h->o_f.alloc(std::max(n, 1));
    h->scratch_in.alloc(std::max(n, 1));
    h->scratch_out.alloc(std::max(n, 1));
    SAP_CUDA(cudaStreamSynchronize(s));
    int opbad = 0;
    SAP_CUDA(cudaMemcpy(&opbad, h->op_nonfinite.get(), sizeof(int), cudaMemcpyDeviceToHost));
    h->op_finite = opbad == 0;
    {  // chunk triangles of the FP32 factors: the same substitution rule as the FP64 sweeps
        unsigned long long kb[2] = {0, 0};
        SAP_CUDA(cudaMemcpy(kb, h->kappa_f.get(), sizeof(kb), cudaMemcpyDeviceToHost));
        double kap[2];
        std::memcpy(kap, kb, sizeof(kap));
        const int force = h->opt.triangle_solve;
        h->lplan_f.subst = force ? force == 2 : kap[0] > kSubstKappa;
        h->rplan_f.subst = force ? force == 2 : kap[1] > kSubstKappa;
        h->rep.chunk_condition = kap[0];
        h->rep.sweep_substitution = h->lplan_f.subst ? 1 : 0;
    }
    h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
    h->rep.t_lu = ev_ms(h->ev[1], h->ev[2]) * 1e-3;
    h->rep.t_factor_kernel = ev_ms(h->ev[8], h->ev[9]) * 1e-3;
    std::vector<int> hb(2 * p);
    SAP_CUDA(cudaMemcpy(hb.data(), h->boosts.get(), sizeof(int) * 2 * p, cudaMemcpyDeviceToHost));
    for (int b = 0; b < p; ++b) {
        h->rep.total_boosts += hb[b];
        h->rep.total_boosts_ul += hb[p + b];
    }
    if (h->coupled) {
        h->rep.t_bc = ev_ms(h->ev[2], h->ev[3]) * 1e-3;
        h->rep.t_spk = ev_ms(h->ev[3], h->ev[4]) * 1e-3;
        h->rep.t_lurdcd = ev_ms(h->ev[4], h->ev[5]) * 1e-3;
        std::vector<int> nf(3 * ni), rb(ni);
        SAP_CUDA(cudaMemcpy(nf.data(), h->nonfinite.get(), sizeof(int) * 3 * ni, cudaMemcpyDeviceToHost));
        SAP_CUDA(cudaMemcpy(rb.data(), h->rbar_boosts.get(), sizeof(int) * ni, cudaMemcpyDeviceToHost));
        for (int t = 0; t < ni; ++t) h->rep.total_rbar_boosts += rb[t];
        for (int t = 0; t < ni; ++t) {
            if (nf[2 * t]) throw PreconditionerFailure("right spike tip at interface " + std::to_string(t) + " is not finite");
            if (nf[2 * t + 1]) throw PreconditionerFailure("left spike tip at interface " + std::to_string(t) + " is not finite");
        }
        for (int t = 0; t < ni; ++t)
            if (nf[2 * ni + t]) throw PreconditionerFailure("reduced interface block " + std::to_string(t) + " is not finite");
    }
    h->ready = true;
}

void setup_banded(sap_handle* h, int n, int k, const double* band, int on_device) {
    PrioScope prio_scope(h);
    h->op_finite = false;
    require(n >= 0 && k >= 0, "BandedMatrix: negative dimension");
    require(band != nullptr || n == 0, "sap_setup_banded: null band");
    const cudaStream_t s = h->stream;
    h->mixed = false;
    h->f32fac = false;
    h->ready = false;
    h->ul_tips = false;
    h->kind = h->opt.precond;
    require(h->kind >= 0 && h->kind <= 3, "sap_setup_banded: unknown preconditioner kind");
    const bool blocks = h->kind == SAP_PRECOND_COUPLED || h->kind == SAP_PRECOND_DECOUPLED;
    Layout L;
    if (blocks) L = make_layout(n, h->opt.p, k);
    h->n = n;
    h->k = k;
    h->layout = L;
    const int p = L.p;
    h->coupled = h->kind == SAP_PRECOND_COUPLED && p > 1;
    // third stage (pipeline.hpp:312-319): only for the block preconditioners
    h->ts = h->ts_armed && blocks && n > 0;
    if (h->ts) {
        require((int)h->ts_k.size() == p, "third stage: block count does not match the partition layout");
        bool any_perm = false;
        for (int b = 0; b < p; ++b) any_perm = any_perm || h->ts_has[b];
        require(!any_perm || (int)h->ts_perm.size() == n, "third stage: permutation length does not match n");
        for (int b = 0; b < p; ++b) {
            require(h->ts_k[b] >= 0 && h->ts_k[b] <= k,
                    "third stage: per-partition half-bandwidth outside [0, k]");
            if (!h->ts_has[b]) continue;
            std::vector<char> seen(L.sizes[b], 0);
            for (int r = 0; r < L.sizes[b]; ++r) {
                const int v = h->ts_perm[L.offsets[b] + r];
                require(v >= 0 && v < L.sizes[b] && !seen[v], "third stage: block permutation is not a permutation");
                seen[v] = 1;
            }
        }
    }
    const bool want_ul = h->coupled && !h->ts;  // build_precond_op: UL only without the third stage (:163-164)
    h->rep = sap_report{};
    h->rep.n = n;
    h->rep.k = k;
    h->rep.partitions = p;

    const size_t total = (size_t)n * (2 * (size_t)k + 1);
    // host band + block preconditioner on the default LU kernel: the upload streams in rounds while the
    // LU / UL jobs factor the columns that have arrived (k_band_lu_res wait_cols)
    // FP32 factorization (mixed precision without the third stage): setup_mixed, after a plain upload
    const bool f32fac = blocks && !h->ts && h->opt.mixed_precision && n > 0;
    const bool streamed = on_device == 0 && blocks && !h->ts && !f32fac && n > 0 && k >= 1 && L.p >= 1 &&
                          band_lu_reads_source(k) && write_value_fn() != nullptr;
    SAP_CUDA(cudaEventRecord(h->ev[0], s));
    if (on_device == 2) {
        h->band.release();
        h->band_ptr = band;
    } else {
        h->band.alloc(total);
        if (n > 0 && !streamed)
            SAP_CUDA(cudaMemcpyAsync(h->band.get(), band, sizeof(double) * total,
                                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        h->band_ptr = h->band.get();
    }
    if (!streamed) SAP_CUDA(cudaEventRecord(h->ev[1], s));
    // resident band on the same kernel: the LU starts at once in the no-boost mode while the block norms
    // run beside it on the side stream (the check and gated refactor below keep it exact)
    const bool early = !streamed && on_device != 0 && blocks && !h->ts && !f32fac && n > 0 && k >= 1 && L.p >= 1 &&
                       band_lu_reads_source(k);
    h->scratch_in.alloc(std::max(n, 1));
    h->scratch_out.alloc(std::max(n, 1));
    h->dscal.alloc(4);

    if (h->kind == SAP_PRECOND_NONE || n == 0) {
        SAP_CUDA(cudaStreamSynchronize(s));
        h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
        h->ready = true;
        return;
    }
    if (h->kind == SAP_PRECOND_DIAGONAL) {
        // scale = banded.inf_norm() (pipeline.hpp:153) = the 1-block norm over all rows
        DevBuf<int> offs1;
        offs1.alloc(2);
        const int ho[2] = {0, n};
        SAP_CUDA(cudaMemcpyAsync(offs1.get(), ho, sizeof(ho), cudaMemcpyHostToDevice, s));
        h->diag.alloc(n);
        h->diag_f32 = h->opt.mixed_precision != 0;  // build_precond_op<float> (pipeline.hpp:325-327)
        launch_block_norms(h->band_ptr, n, k, offs1.get(), 1, nullptr, h->dscal.get(), s, nullptr, nullptr,
                           h->diag_f32);
        launch_boosted_diag(h->band_ptr, n, k, h->dscal.get(), h->opt.boost_eps, h->diag.get(), s, h->diag_f32);
        SAP_CUDA(cudaEventRecord(h->ev[2], s));
        SAP_CUDA(cudaStreamSynchronize(s));
        h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
        h->rep.t_lu = ev_ms(h->ev[1], h->ev[2]) * 1e-3;
        h->ready = true;
        return;
    }

    if (f32fac) return setup_mixed(h, L, want_ul);
    // ---- factor_blocks: norms, block band copies, LU (+ UL) ----
    h->d_offsets.alloc(p + 1);
    SAP_CUDA(cudaMemcpyAsync(h->d_offsets.get(), L.offsets.data(), sizeof(int) * (p + 1), cudaMemcpyHostToDevice, s));
    h->norms.alloc(p);
    h->boosts.alloc(2 * (size_t)p);
    SAP_CUDA(cudaMemsetAsync(h->boosts.get(), 0, sizeof(int) * 2 * p, s));
    const int m_max = L.sizes[0];
    h->fst = BandStore::make(m_max, k);
    h->lu.alloc(h->fst.total(p));
    if (want_ul)
        h->ul.alloc(h->fst.total(p));
    else
        h->ul.release();
    const int njobs = want_ul ? 2 * p : p;
    std::vector<FactorJob> jobs(njobs);
    // the default LU kernel reads the unfactored blocks straight from the band (no block copies);
    // the third stage factors the permuted blocks assembled in the store
    const bool from_src = band_lu_reads_source(k) && !h->ts;
    const size_t w = 2 * (size_t)k + 1;
    for (int b = 0; b < p; ++b) {
        const int m = L.sizes[b];
        double* f = h->lu.get() + h->fst.block(b);
        const double* a = h->band_ptr + (size_t)L.offsets[b] * w;
        // third stage: block b is factored at its own K_b inside the k-wide store (block_factors.hpp:155-180;
        // the entries beyond K_b are zero and stay zero), so its cost scales with K_b^2
        const int kj = h->ts ? std::max(h->ts_k[b], 1) : k;
        jobs[b] = FactorJob{f + k, 1, 2LL * k, m, kj, h->norms.get() + b, h->boosts.get() + b, from_src ? a + k : nullptr};
        if (want_ul) {
            double* g = h->ul.get() + h->fst.block(b);
            const size_t last = (size_t)(m - 1) * w + k;
            jobs[p + b] = FactorJob{g + last, -1, -2LL * k, m, k, h->norms.get() + b, h->boosts.get() + p + b,
                                    from_src ? a + last : nullptr};
        }
    }
    h->jobs.alloc(njobs);
    lu_df_clear_error(lu_scratch(h, njobs, m_max), s);
    SAP_CUDA(cudaMemcpyAsync(h->jobs.get(), jobs.data(), sizeof(FactorJob) * njobs, cudaMemcpyHostToDevice, s));
    h->kappa.alloc(3);
    SAP_CUDA(cudaMemsetAsync(h->kappa.get(), 0, 3 * sizeof(unsigned long long), s));
    h->op_nonfinite.alloc(1);
    SAP_CUDA(cudaMemsetAsync(h->op_nonfinite.get(), 0, sizeof(int), s));
    if (h->ts) {
        // P_b A_b P_b^T at K_b into the zeroed store (block_factors.hpp:155-180), norms over it (:187-195)
        std::vector<int> gperm(n);
        for (int b = 0; b < p; ++b)
            for (int r = 0; r < L.sizes[b]; ++r)
                gperm[L.offsets[b] + r] = L.offsets[b] + (h->ts_has[b] ? h->ts_perm[L.offsets[b] + r] : r);
        h->d_gperm.alloc(n);
        h->d_has.alloc(p);
        h->d_kb.alloc(p);
        h->d_bad.alloc(1);
        SAP_CUDA(cudaMemcpyAsync(h->d_gperm.get(), gperm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemcpyAsync(h->d_has.get(), h->ts_has.data(), sizeof(int) * p, cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemcpyAsync(h->d_kb.get(), h->ts_k.data(), sizeof(int) * p, cudaMemcpyHostToDevice, s));
        static const int big = 0x7fffffff;
        SAP_CUDA(cudaMemcpyAsync(h->d_bad.get(), &big, sizeof(int), cudaMemcpyHostToDevice, s));
        h->norms_op.alloc(p);
        launch_block_norms(h->band_ptr, m_max, k, h->d_offsets.get(), p, nullptr, h->norms_op.get(), s,
                           h->op_nonfinite.get());
        SAP_CUDA(cudaMemsetAsync(h->lu.get(), 0, sizeof(double) * h->fst.total(p), s));
        launch_assemble_blocks(h->band_ptr, n, k, h->d_offsets.get(), p, h->d_gperm.get(), h->d_has.get(),
                               h->d_kb.get(), h->fst, h->lu.get(), h->d_bad.get(), s);
        launch_block_norms(h->lu.get(), m_max, k, h->d_offsets.get(), p, &h->fst, h->norms.get(), s);
        h->scratch_p.alloc(n);
    } else if (!streamed && !early) {
        launch_block_norms(h->band_ptr, m_max, k, h->d_offsets.get(), p, nullptr, h->norms.get(), s,
                           h->op_nonfinite.get());
        if (from_src)
            launch_zero_pad(k, h->d_offsets.get(), p, h->fst, h->lu.get(), want_ul ? h->ul.get() : nullptr, s);
        else
            launch_copy_blocks(h->band_ptr, k, h->d_offsets.get(), p, h->fst, h->lu.get(),
                               want_ul ? h->ul.get() : nullptr, s);
    }
    if (streamed || early) {
        // 1. (streamed) every upload round and its counter write, enqueued on the side stream BEFORE the
        //    kernel that polls the counter is launched (nothing the host does afterwards can hold the
        //    copies back); round r brings `piece` more columns of every block from its top (LU) and, for
        //    SaP-C, its bottom (UL). The counter is reset on s, ahead of the kernel in stream order (a
        //    previous setup left it at its final value). (early) the counter says "all arrived".
        const cudaStream_t cs = h->side;
        const int ends = want_ul ? 2 : 1;
        h->d_ready.alloc(1);
        h->d_minpiv.alloc(njobs);
        h->d_sbad.alloc(1);
        if (!h->sev_norm) SAP_CUDA(cudaEventCreateWithFlags(&h->sev_norm, cudaEventDisableTiming));
        SAP_CUDA(cudaMemsetAsync(h->d_ready.get(), early ? 0x7f : 0, sizeof(unsigned), s));
        SAP_CUDA(cudaEventRecord(h->sev[0], s));  // earlier work on s may still read the old band
        SAP_CUDA(cudaStreamWaitEvent(cs, h->sev[0], 0));
        SAP_CUDA(cudaMemsetAsync(h->op_nonfinite.get(), 0, sizeof(int), cs));
        std::vector<int> piece(p);
        for (int b = 0; b < p; ++b)
            piece[b] = early ? 1 : (L.sizes[b] + ends * kUploadRounds - 1) / (ends * kUploadRounds);
        const size_t cb = w * sizeof(double);
        bool uniform = streamed;  // equal blocks: one 2-D copy per round and end (block pitch), not one per block
        for (int b = 1; b < p; ++b) uniform = uniform && L.sizes[b] == L.sizes[0];
        for (int r = 0; r < kUploadRounds && uniform; ++r) {
            const int m = L.sizes[0], pc = piece[0];
            const size_t pitch = (size_t)m * cb;
            const int t0 = std::min(m, r * pc), t1 = std::min(m, (r + 1) * pc);
            if (t1 > t0)
                SAP_CUDA(cudaMemcpy2DAsync(h->band.get() + (size_t)t0 * w, pitch, band + (size_t)t0 * w, pitch,
                                           cb * (t1 - t0), p, cudaMemcpyHostToDevice, cs));
            if (ends == 2) {
                const int b1 = std::max(0, m - r * pc), b0 = std::max(0, m - (r + 1) * pc);
                if (b1 > b0)
                    SAP_CUDA(cudaMemcpy2DAsync(h->band.get() + (size_t)b0 * w, pitch, band + (size_t)b0 * w, pitch,
                                               cb * (b1 - b0), p, cudaMemcpyHostToDevice, cs));
            }
            const CUresult wr = write_value_fn()(cs, (CUdeviceptr)h->d_ready.get(), (cuuint32_t)(r + 1), 0);
            if (wr != CUDA_SUCCESS) throw CudaFailure("cuStreamWriteValue32 failed");
        }
        for (int r = 0; r < kUploadRounds && streamed && !uniform; ++r) {
            for (int b = 0; b < p; ++b) {
                const int m = L.sizes[b], off = L.offsets[b], pc = piece[b];
                const int t0 = std::min(m, r * pc), t1 = std::min(m, (r + 1) * pc);
                if (t1 > t0)
                    SAP_CUDA(cudaMemcpyAsync(h->band.get() + (size_t)(off + t0) * w, band + (size_t)(off + t0) * w,
                                             cb * (t1 - t0), cudaMemcpyHostToDevice, cs));
                if (ends == 2) {
                    const int b1 = std::max(0, m - r * pc), b0 = std::max(0, m - (r + 1) * pc);
                    if (b1 > b0)
                        SAP_CUDA(cudaMemcpyAsync(h->band.get() + (size_t)(off + b0) * w,
                                                 band + (size_t)(off + b0) * w, cb * (b1 - b0),
                                                 cudaMemcpyHostToDevice, cs));
                }
            }
            const CUresult wr = write_value_fn()(cs, (CUdeviceptr)h->d_ready.get(), (cuuint32_t)(r + 1), 0);
            if (wr != CUDA_SUCCESS) throw CudaFailure("cuStreamWriteValue32 failed");
        }
        if (streamed) SAP_CUDA(cudaEventRecord(h->ev[1], cs));
        // the stores' out-of-matrix slots (disjoint from everything the LU writes), beside the LU; the
        // sweeps and chunk inverses that read them come after sev_norm / the side stream's later work
        launch_zero_pad(k, h->d_offsets.get(), p, h->fst, h->lu.get(), want_ul ? h->ul.get() : nullptr, cs);
        launch_block_norms(h->band_ptr, m_max, k, h->d_offsets.get(), p, nullptr, h->norms.get(), cs,
                           h->op_nonfinite.get());
        SAP_CUDA(cudaEventRecord(h->sev_norm, cs));
        // 2. the LU / UL kernel in streamed mode (no boosting; min |pivot| per job)
        std::vector<FactorJob> sj = jobs;
        for (int j = 0; j < njobs; ++j) {
            sj[j].ready = h->d_ready.get();
            sj[j].piece = piece[j % p];
            sj[j].ends = ends;
            sj[j].minpiv = h->d_minpiv.get() + j;
        }
        std::vector<FactorJob> gj = jobs;
        for (int j = 0; j < njobs; ++j) gj[j].gate = h->d_sbad.get();
        h->sjobs.alloc(njobs);
        h->gjobs.alloc(njobs);
        SAP_CUDA(cudaMemcpyAsync(h->sjobs.get(), sj.data(), sizeof(FactorJob) * njobs, cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemcpyAsync(h->gjobs.get(), gj.data(), sizeof(FactorJob) * njobs, cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemsetAsync(h->d_minpiv.get(), 0, sizeof(double) * njobs, s));  // -1 = stalled upload
        SAP_CUDA(cudaEventRecord(h->ev[8], s));
        launch_band_lu(h->sjobs.get(), njobs, k, h->opt.boost_eps, s, true, m_max, lu_scratch(h, njobs, m_max), h->opt.lu_kernel);
        SAP_CUDA(cudaEventRecord(h->ev[9], s));
        // 3. once the norms exist: any pivot below the boost threshold means the reference would have
        //    boosted -> refactor with boosting (rare; exact either way)
        SAP_CUDA(cudaStreamWaitEvent(s, h->sev_norm, 0));
        launch_stream_check(h->sjobs.get(), h->d_minpiv.get(), h->norms.get(), njobs, p, h->opt.boost_eps,
                            h->d_sbad.get(), s);
        // the refactor with boosting is always launched; its CTAs exit at once unless the check asked for it
        launch_band_lu(h->gjobs.get(), njobs, k, h->opt.boost_eps, s, false, m_max, lu_scratch(h, njobs, m_max), h->opt.lu_kernel);
    } else {
        SAP_CUDA(cudaEventRecord(h->ev[8], s));
        launch_band_lu(h->jobs.get(), njobs, k, h->opt.boost_eps, s, false, m_max, lu_scratch(h, njobs, m_max), h->opt.lu_kernel);
        SAP_CUDA(cudaEventRecord(h->ev[9], s));
    }
    {
        SweepPlan<double>& lp = h->lplan;
        lp = SweepPlan<double>{};
        lp.f = h->lu.get();
        lp.st = h->fst;
        lp.offs = h->d_offsets.get();
        lp.p = p;
        lp.k = k;
        h->dinv.alloc(std::max<size_t>(sweep_dinv_elems(lp), 1));
        plan_sweeps(lp, h->dinv.get());
        lp.kappa = h->kappa.get();
        lp.kb = h->ts ? h->d_kb.get() : nullptr;  // third stage: sweeps read each block's K_b columns only
        if (want_ul) {  // only the solve needs them: overlap with coupling / tips / reduced blocks
            SAP_CUDA(cudaEventRecord(h->sev[0], s));
            SAP_CUDA(cudaStreamWaitEvent(h->side, h->sev[0], 0));
            launch_chunk_inverses(lp, h->side);
            SweepPlan<double>& up = h->uplan;
            up = SweepPlan<double>{};
            if (!h->ts && !h->opt.mixed_precision && h->opt.tip_solve != 1 && lp.tma && lp.tr == 32 &&
                tip_sweeps_fit(p)) {
                up.f = h->ul.get();
                up.st = h->fst;
                up.offs = h->d_offsets.get();
                up.p = p;
                up.k = k;
                up.ul = true;
                h->udinv.alloc(std::max<size_t>(sweep_dinv_elems(up), 1));
                plan_sweeps(up, h->udinv.get());
                up.kappa = h->kappa.get() + 2;
                if (up.tma && up.tr == 32) launch_chunk_inverses(up, h->side);
            }
            SAP_CUDA(cudaEventRecord(h->sev[1], h->side));
        } else {
            launch_chunk_inverses(lp, s);
        }
    }
    SAP_CUDA(cudaEventRecord(h->ev[2], s));
    for (int b = 0; b < p; ++b) {
        // band_lu_inplace op count: sum over columns of d + 2 d^2, d = min(k, m-1-j)
        const double m = L.sizes[b], kk = std::min<double>(k, m - 1 > 0 ? m - 1 : 0);
        const double f = (m - kk) * (2 * kk * kk + kk) + (kk - 1) * kk * (4 * kk + 1) / 6.0;
        h->rep.factor_flops += (want_ul ? 2.0 : 1.0) * f;
    }

    int ni = 0;
    if (h->coupled) {
        ni = p - 1;
        const size_t ww = (size_t)k * k * ni;
        h->rst = BandStore::make(k, k > 0 ? k - 1 : 0);  // reduced blocks in band layout, k' = w-1
        h->bblk.alloc(std::max<size_t>(ww, 1));
        h->cblk.alloc(std::max<size_t>(ww, 1));
        h->vb.alloc(std::max<size_t>(ww, 1));
        h->wt.alloc(std::max<size_t>(ww, 1));
        h->rbar.alloc(std::max<size_t>(h->rst.total(ni), 1));
        SAP_CUDA(cudaMemsetAsync(h->rbar.get(), 0, sizeof(double) * h->rst.total(ni), s));
        h->rbar_norms.alloc(ni);
        h->rbar_boosts.alloc(ni);
        h->nonfinite.alloc(3 * (size_t)ni);
        h->scratch_g.alloc(n);
        h->xt.alloc(std::max<size_t>((size_t)ni * k, 1));
        h->xb.alloc(std::max<size_t>((size_t)ni * k, 1));
        std::vector<int> roffs(ni + 1);
        for (int t = 0; t <= ni; ++t) roffs[t] = t * k;
        h->d_roffsets.alloc(ni + 1);
        SAP_CUDA(cudaMemcpyAsync(h->d_roffsets.get(), roffs.data(), sizeof(int) * (ni + 1), cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemsetAsync(h->nonfinite.get(), 0, sizeof(int) * 3 * ni, s));
        SAP_CUDA(cudaMemsetAsync(h->rbar_boosts.get(), 0, sizeof(int) * ni, s));
        // ---- T_BC: extract_coupling ----
        if (h->ts) {
            h->widths.assign(ni, 0);
            for (int t = 0; t < ni; ++t) h->widths[t] = std::max(h->ts_k[t], h->ts_k[t + 1]);  // spike.hpp:102
            h->d_wid.alloc(ni);
            SAP_CUDA(cudaMemcpyAsync(h->d_wid.get(), h->widths.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, s));
        }
        launch_extract_coupling(h->band_ptr, n, k, h->d_offsets.get(), p, h->bblk.get(), h->cblk.get(), s,
                                h->ts ? h->d_wid.get() : nullptr);
        SAP_CUDA(cudaEventRecord(h->ev[3], s));
        // ---- T_SPK: spike tips (third stage: full spikes, spike.hpp:258-296) ----
        if (h->ts) {
            const size_t nk = (size_t)n * k;
            h->vfull.alloc(std::max<size_t>(nk, 1));
            h->wfull.alloc(std::max<size_t>(nk, 1));
            SAP_CUDA(cudaMemsetAsync(h->vfull.get(), 0, sizeof(double) * nk, s));
            SAP_CUDA(cudaMemsetAsync(h->wfull.get(), 0, sizeof(double) * nk, s));
            launch_full_rhs(h->bblk.get(), h->cblk.get(), k, h->d_offsets.get(), ni, h->d_gperm.get(),
                            h->vfull.get(), h->wfull.get(), s);
            std::vector<FullSpikeJob> fj;
            for (int t = 0; t < ni; ++t) {
                // forward sweeps start at the first permuted row carrying a right-hand side
                const int e = L.offsets[t + 1];
                int fv = L.sizes[t], fw = L.sizes[t + 1];
                for (int r = 0; r < k; ++r) {
                    const int ov = e - k + r - L.offsets[t], ow = r;
                    fv = std::min(fv, h->ts_has[t] ? h->ts_perm[L.offsets[t] + ov] : ov);
                    fw = std::min(fw, h->ts_has[t + 1] ? h->ts_perm[e + ow] : ow);
                }
                // V' lives in columns [0, w_t), W' in [k - w_t, k) (third.cu header)
                const int w = h->widths[t];
                fj.push_back(FullSpikeJob{h->lu.get() + h->fst.block(t) + k, h->vfull.get() + (size_t)L.offsets[t] * k,
                                          L.sizes[t], fv, 2 * t, 0, w, h->ts_k[t], t});
                fj.push_back(FullSpikeJob{h->lu.get() + h->fst.block(t + 1) + k, h->wfull.get() + (size_t)e * k,
                                          L.sizes[t + 1], fw, 2 * t + 1, k - w, k, h->ts_k[t + 1], t + 1});
            }
            h->fsjobs.alloc(fj.size());
            SAP_CUDA(cudaMemcpyAsync(h->fsjobs.get(), fj.data(), sizeof(FullSpikeJob) * fj.size(),
                                     cudaMemcpyHostToDevice, s));
            const bool inv = h->lplan.tma && h->lplan.tr == 32 && h->opt.triangle_solve != 2;
            launch_full_spikes(h->fsjobs.get(), (int)fj.size(), k, h->nonfinite.get(), inv ? h->lplan.dinv : nullptr,
                               h->lplan.nch_max, h->kappa.get(), h->opt.triangle_solve == 1 ? HUGE_VAL : kSubstKappa,
                               s);
            launch_full_tips(h->vfull.get(), h->wfull.get(), k, h->d_offsets.get(), ni, h->d_gperm.get(),
                             h->d_wid.get(), h->vb.get(), h->wt.get(), s);
        } else {
            std::vector<TipJob> tj;
            for (int t = 0; t < ni; ++t) {
                const size_t o = (size_t)t * k * k;
                tj.push_back(TipJob{h->lu.get() + h->fst.block(t), L.sizes[t] - k, 0, h->bblk.get() + o,
                                    h->vb.get() + o, 2 * t});
                tj.push_back(TipJob{h->ul.get() + h->fst.block(t + 1), 0, 1, h->cblk.get() + o,
                                    h->wt.get() + o, 2 * t + 1});
            }
            h->tipjobs.alloc(std::max<size_t>(tj.size(), 1));
            SAP_CUDA(cudaMemcpyAsync(h->tipjobs.get(), tj.data(), sizeof(TipJob) * tj.size(), cudaMemcpyHostToDevice, s));
            launch_spike_tips(h->tipjobs.get(), (int)tj.size(), k, h->nonfinite.get(), s);
        }
        SAP_CUDA(cudaEventRecord(h->ev[4], s));
        // ---- T_LUrdcd: rbar = I - W V (band layout, k' = w-1) and its boosted no-pivot LU ----
        if (k > 0) {
            launch_rbar(h->wt.get(), h->vb.get(), k, ni, h->rbar.get(), h->rst, h->nonfinite.get() + 2 * ni, s);
            // third stage: R' = diag(R_t, I); the boost scale is R_t's norm (rows < w_t)
            launch_block_norms(h->rbar.get(), k, k - 1, h->d_roffsets.get(), ni, &h->rst, h->rbar_norms.get(), s,
                               nullptr, h->ts ? h->d_wid.get() : nullptr);
            std::vector<FactorJob> rj(ni);
            for (int t = 0; t < ni; ++t)
                rj[t] = FactorJob{h->rbar.get() + h->rst.block(t) + (k - 1), 1, 2LL * (k - 1), k, k - 1,
                                  h->rbar_norms.get() + t, h->rbar_boosts.get() + t};
            h->rjobs.alloc(ni);
            SAP_CUDA(cudaMemcpyAsync(h->rjobs.get(), rj.data(), sizeof(FactorJob) * ni, cudaMemcpyHostToDevice, s));
            launch_band_lu(h->rjobs.get(), ni, k - 1, h->opt.boost_eps, s, false, k, lu_scratch(h, ni, k), h->opt.lu_kernel);
            SweepPlan<double>& rp = h->rplan;
            rp = SweepPlan<double>{};
            rp.f = h->rbar.get();
            rp.st = h->rst;
            rp.offs = h->d_roffsets.get();
            rp.p = ni;
            rp.k = k - 1;
            h->rdinv.alloc(std::max<size_t>(sweep_dinv_elems(rp), 1));
            plan_sweeps(rp, h->rdinv.get());
            rp.kappa = h->kappa.get() + 1;
            launch_chunk_inverses(rp, s);
        }
        SAP_CUDA(cudaEventRecord(h->ev[5], s));
        if (want_ul) SAP_CUDA(cudaStreamWaitEvent(s, h->sev[1], 0));  // the LU chunk inverses (side stream)
    }
    if (h->opt.mixed_precision) {
        build_fp32_preconditioner(h, s);
        if (h->ts) h->scratch_pf.alloc(n);
    }
    SAP_CUDA(cudaStreamSynchronize(s));
    lu_check(h);
    if (streamed || early) {
        int bad = 0;
        SAP_CUDA(cudaMemcpy(&bad, h->d_sbad.get(), sizeof(int), cudaMemcpyDeviceToHost));
        if (bad & 2) throw CudaFailure("streamed band upload stalled");
    }
    if (h->ts) {
        int bad = 0;
        SAP_CUDA(cudaMemcpy(&bad, h->d_bad.get(), sizeof(int), cudaMemcpyDeviceToHost));
        if (bad != 0x7fffffff)
            throw InvalidArgument("factor_blocks: block permutation exceeds bandwidth " + std::to_string(h->ts_k[bad]));
    }
    choose_triangle_solve(h);
    h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
    h->rep.t_lu = ev_ms(h->ev[1], h->ev[2]) * 1e-3;
    h->rep.t_factor_kernel = ev_ms(h->ev[8], h->ev[9]) * 1e-3;
    std::vector<int> hb(2 * p);
    SAP_CUDA(cudaMemcpy(hb.data(), h->boosts.get(), sizeof(int) * 2 * p, cudaMemcpyDeviceToHost));
    for (int b = 0; b < p; ++b) {
        h->rep.total_boosts += hb[b];
        h->rep.total_boosts_ul += hb[p + b];
    }
    if (h->coupled) {
        h->rep.t_bc = ev_ms(h->ev[2], h->ev[3]) * 1e-3;
        h->rep.t_spk = ev_ms(h->ev[3], h->ev[4]) * 1e-3;
        h->rep.t_lurdcd = ev_ms(h->ev[4], h->ev[5]) * 1e-3;
        std::vector<int> nf(3 * ni), rb(ni);
        SAP_CUDA(cudaMemcpy(nf.data(), h->nonfinite.get(), sizeof(int) * 3 * ni, cudaMemcpyDeviceToHost));
        SAP_CUDA(cudaMemcpy(rb.data(), h->rbar_boosts.get(), sizeof(int) * ni, cudaMemcpyDeviceToHost));
        for (int t = 0; t < ni; ++t) h->rep.total_rbar_boosts += rb[t];
        // the reference throws at the first failure in interface order (spike.hpp:217-219, :246-248),
        // then at the first non-finite reduced block (:162-164)
        for (int t = 0; t < ni && h->ts; ++t)  // compute_full_spikes, spike.hpp:279-280
            if (nf[2 * t] || nf[2 * t + 1])
                throw PreconditionerFailure("spike at interface " + std::to_string(t) + " is not finite");
        for (int t = 0; t < ni; ++t) {
            if (nf[2 * t]) throw PreconditionerFailure("right spike tip at interface " + std::to_string(t) + " is not finite");
            if (nf[2 * t + 1]) throw PreconditionerFailure("left spike tip at interface " + std::to_string(t) + " is not finite");
        }
        for (int t = 0; t < ni; ++t)
            if (nf[2 * ni + t]) throw PreconditionerFailure("reduced interface block " + std::to_string(t) + " is not finite");
        // first block solve of the apply from the LU (last rows) and UL (first rows) sweeps: equal to the LU
        // solve's rows up to rounding when neither factorization boosted a pivot (a boosted LU and UL are
        // different perturbations of A_b) and both stores' chunk triangles are well conditioned
        const SweepPlan<double>& up = h->uplan;
        if (up.ul && up.tma && up.tr == 32 && !h->lplan.subst && !h->ts && !h->mixed && h->rep.total_boosts == 0 &&
            h->rep.total_boosts_ul == 0 && h->opt.tip_solve != 1 && h->opt.triangle_solve != 2) {
            unsigned long long kb = 0;
            SAP_CUDA(cudaMemcpy(&kb, h->kappa.get() + 2, sizeof(kb), cudaMemcpyDeviceToHost));
            double kap;
            std::memcpy(&kap, &kb, sizeof(kap));
            h->ul_tips = kap <= kSubstKappa;
            if (h->ul_tips) h->scratch_gu.alloc(n);
        }
    }
    h->rep.ul_tip_sweeps = h->ul_tips ? 1 : 0;
    h->ready = true;
}

// ---------------------------------------------------------------------------
// Multi-GPU: the partitions are sharded across ranks in order (rank r owns a contiguous run of
// whole partitions). A rank factors its own blocks and the spike tips it can compute from them;
// the neighbours swap the one tip each needs (V^b of the left rank's last block, W^t of the right
// rank's first block) once at setup. Each cross interface's reduced block R̄ is then built and
// factored on BOTH ranks (bitwise identical), so an apply needs one neighbour exchange of w rows of
// g = D^{-1} in each way and no second round. The operator exchanges a k-row halo each way;
// Krylov dots are summed over ranks.

// Neighbour exchange of device buffers (counts may be 0). NCCL: grouped send / recv on the handle's stream,
// stream-ordered with the kernels around it (no host synchronisation). Callbacks: the stream is synchronised
// first and the callback completes the transfer before returning.
void comm_exchange_raw(sap_handle* h, const double* sl, int n_sl, const double* sr, int n_sr, double* rl, int n_rl,
                       double* rr, int n_rr) {
    if (h->comm.world <= 1) return;
    if (h->nccl) return nccl_exchange(h->nccl, sl, n_sl, sr, n_sr, rl, n_rl, rr, n_rr, h->stream);
    SAP_CUDA(cudaStreamSynchronize(h->stream));
    const int rc = h->comm.exchange(h->comm.ctx, sl, n_sl, sr, n_sr, rl, n_rl, rr, n_rr);
    if (rc != 0) throw CommFailure("sap: neighbour exchange failed (" + std::to_string(rc) + ")");
}

void comm_exchange(sap_handle* h, const double* sl, const double* sr, double* rl, double* rr, int count) {
    if (count == 0) return;
    comm_exchange_raw(h, h->has_left ? sl : nullptr, h->has_left ? count : 0, h->has_right ? sr : nullptr,
                      h->has_right ? count : 0, h->has_left ? rl : nullptr, h->has_left ? count : 0,
                      h->has_right ? rr : nullptr, h->has_right ? count : 0);
}

// In-place sum over ranks of `count` HOST doubles (setup flags, Krylov failure flags).
void comm_allreduce(sap_handle* h, double* v, int count) {
    if (h->comm.world <= 1 || count == 0) return;
    if (h->nccl) {
        h->dred.alloc(std::max(count, 16));
        SAP_CUDA(cudaMemcpyAsync(h->dred.get(), v, sizeof(double) * count, cudaMemcpyHostToDevice, h->stream));
        nccl_allreduce(h->nccl, h->dred.get(), count, h->stream);
        SAP_CUDA(cudaMemcpyAsync(v, h->dred.get(), sizeof(double) * count, cudaMemcpyDeviceToHost, h->stream));
        SAP_CUDA(cudaStreamSynchronize(h->stream));
        return;
    }
    const int rc = h->comm.allreduce_sum(h->comm.ctx, v, count);
    if (rc != 0) throw CommFailure("sap: allreduce failed (" + std::to_string(rc) + ")");
}

void apply_m_dist(sap_handle* h, const double* in, double* out) {
    const cudaStream_t s = h->stream;
    const int n = h->n, k = h->k;
    const size_t bytes = sizeof(double) * (size_t)n;
    if (h->kind == SAP_PRECOND_NONE) {
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (!h->coupled) {
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        launch_block_solve<double>(h->lplan, out, s);
        return;
    }
    double* g = h->scratch_g.get() + k;  // [left halo w | own n | right halo w]
    SAP_CUDA(cudaMemcpyAsync(g, in, bytes, cudaMemcpyDeviceToDevice, s));
    if (h->ul_tips) {
        // g's last rows of every block from the LU tip sweeps, the first rows from the UL ones (gu, same
        // halo layout); this rank's first w rows go left from gu, its last w rows right from g, and the halos
        // land where the interfaces read them (left: bottom rows in g, right: top rows in gu)
        double* gu = h->scratch_gu.get() + k;
        SAP_CUDA(cudaMemcpyAsync(gu, in, bytes, cudaMemcpyDeviceToDevice, s));
        SAP_CUDA(cudaEventRecord(h->tev[0], s));
        SAP_CUDA(cudaStreamWaitEvent(h->tside, h->tev[0], 0));
        launch_block_solve<double>(h->uplan, gu, h->tside, k);
        SAP_CUDA(cudaEventRecord(h->tev[1], h->tside));
        if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
        launch_block_solve<double>(h->lplan, g, s, k);
        SAP_CUDA(cudaStreamWaitEvent(s, h->tev[1], 0));
        comm_exchange(h, gu, g + n - k, g - k, gu + n, k);
        launch_interfaces<double>(g, h->d_ioffs.get(), h->rplan, h->ni_tot, k, h->wt.get(), h->vb.get(),
                                  h->bblk.get(), h->cblk.get(), h->xt.get(), h->xb.get(), out, h->has_left,
                                  h->has_right, s, gu);
        launch_block_solve<double>(h->lplan, out, s);
        return;
    }
    if (out != in) SAP_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, s));
    launch_block_solve<double>(h->lplan, g, s);
    comm_exchange(h, g, g + n - k, g - k, g + n, k);
    launch_interfaces<double>(g, h->d_ioffs.get(), h->rplan, h->ni_tot, k, h->wt.get(), h->vb.get(), h->bblk.get(),
                              h->cblk.get(), h->xt.get(), h->xb.get(), out, h->has_left, h->has_right, s);
    launch_block_solve<double>(h->lplan, out, s);
}

void apply_a_dist(sap_handle* h, const double* in, double* out) {
    const cudaStream_t s = h->stream;
    const int n = h->n, k = h->k;
    const int band_n = h->c_hi - h->c_lo, own = h->row_lo - h->c_lo;
    double* x = h->xext.get();
    SAP_CUDA(cudaMemcpyAsync(x + own, in, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s));
    comm_exchange(h, in, in + n - k, x, x + own + n, k);
    launch_band_spmv_rows(h->band_ptr, band_n, k, own, own + n, x, out, s);
}

void setup_banded_dist(sap_handle* h, int n, int k, int row_lo, int row_hi, const double* slice, int on_device) {
    h->op_finite = false;
    require(n >= 0 && k >= 0, "BandedMatrix: negative dimension");
    if (h->opt.mixed_precision)
        throw InvalidArgument("sap_setup_banded_dist: mixed_precision is not supported by this build");
    const cudaStream_t s = h->stream;
    h->ready = false;
    h->ul_tips = false;
    h->kind = h->opt.precond;
    require(h->kind == SAP_PRECOND_COUPLED || h->kind == SAP_PRECOND_DECOUPLED || h->kind == SAP_PRECOND_NONE,
            "sap_setup_banded_dist: only the coupled, decoupled and none preconditioners are distributed");
    const Layout G = make_layout(n, h->opt.p, k);
    require(G.p >= h->comm.world, "sap_setup_banded_dist: fewer partitions than ranks");
    int pb = -1, pe = -1;
    for (int b = 0; b <= G.p; ++b) {
        if (G.offsets[b] == row_lo) pb = b;
        if (G.offsets[b] == row_hi) pe = b;
    }
    require(pb >= 0 && pe > pb, "sap_setup_banded_dist: row range does not align with partition boundaries");
    require(slice != nullptr, "sap_setup_banded_dist: null band slice");
    const int pl = pe - pb, nl = row_hi - row_lo;
    Layout L;
    L.n = nl;
    L.p = pl;
    L.k = k;
    L.sizes.assign(G.sizes.begin() + pb, G.sizes.begin() + pe);
    L.offsets.resize(pl + 1);
    for (int b = 0; b <= pl; ++b) L.offsets[b] = G.offsets[pb + b] - row_lo;
    h->glayout = G;
    h->layout = L;
    h->n_glob = n;
    h->n = nl;
    h->k = k;
    h->row_lo = row_lo;
    h->row_hi = row_hi;
    h->pb = pb;
    h->pe = pe;
    h->c_lo = std::max(0, row_lo - k);
    h->c_hi = std::min(n, row_hi + k);
    h->has_left = row_lo > 0;
    h->has_right = row_hi < n;
    h->coupled = h->kind == SAP_PRECOND_COUPLED && G.p > 1 && k > 0;
    const int band_n = h->c_hi - h->c_lo, own = row_lo - h->c_lo;
    h->rep = sap_report{};
    h->rep.n = n;
    h->rep.k = k;
    h->rep.partitions = G.p;

    const size_t total = (size_t)band_n * (2 * (size_t)k + 1);
    SAP_CUDA(cudaEventRecord(h->ev[0], s));
    if (on_device == 2) {
        h->band.release();
        h->band_ptr = slice;
    } else {
        h->band.alloc(total);
        SAP_CUDA(cudaMemcpyAsync(h->band.get(), slice, sizeof(double) * total,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        h->band_ptr = h->band.get();
    }
    SAP_CUDA(cudaEventRecord(h->ev[1], s));
    h->scratch_in.alloc(nl);
    h->scratch_out.alloc(nl);
    h->xext.alloc(band_n);
    SAP_CUDA(cudaMemsetAsync(h->xext.get(), 0, sizeof(double) * band_n, s));
    if (h->kind == SAP_PRECOND_NONE) {
        SAP_CUDA(cudaStreamSynchronize(s));
        h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
        h->ready = true;
        return;
    }

    // ---- factor the local blocks (as setup_banded) ----
    std::vector<int> boffs(pl + 1);
    for (int b = 0; b <= pl; ++b) boffs[b] = L.offsets[b] + own;
    h->d_offsets.alloc(pl + 1);
    h->d_boffs.alloc(pl + 1);
    SAP_CUDA(cudaMemcpyAsync(h->d_offsets.get(), L.offsets.data(), sizeof(int) * (pl + 1), cudaMemcpyHostToDevice, s));
    SAP_CUDA(cudaMemcpyAsync(h->d_boffs.get(), boffs.data(), sizeof(int) * (pl + 1), cudaMemcpyHostToDevice, s));
    h->norms.alloc(pl);
    h->boosts.alloc(2 * (size_t)pl);
    SAP_CUDA(cudaMemsetAsync(h->boosts.get(), 0, sizeof(int) * 2 * pl, s));
    const int m_max = *std::max_element(L.sizes.begin(), L.sizes.end());
    h->fst = BandStore::make(m_max, k);
    h->lu.alloc(h->fst.total(pl));
    if (h->coupled)
        h->ul.alloc(h->fst.total(pl));
    else
        h->ul.release();
    const int njobs = h->coupled ? 2 * pl : pl;
    std::vector<FactorJob> jobs(njobs);
    const bool from_src = band_lu_reads_source(k);
    const size_t w = 2 * (size_t)k + 1;
    for (int b = 0; b < pl; ++b) {
        const int m = L.sizes[b];
        const double* a = h->band_ptr + (size_t)boffs[b] * w;
        jobs[b] = FactorJob{h->lu.get() + h->fst.block(b) + k, 1, 2LL * k, m, k, h->norms.get() + b,
                            h->boosts.get() + b, from_src ? a + k : nullptr};
        if (h->coupled) {
            const size_t last = (size_t)(m - 1) * w + k;
            jobs[pl + b] = FactorJob{h->ul.get() + h->fst.block(b) + last, -1, -2LL * k, m, k, h->norms.get() + b,
                                     h->boosts.get() + pl + b, from_src ? a + last : nullptr};
        }
    }
    h->jobs.alloc(njobs);
    lu_df_clear_error(lu_scratch(h, njobs, m_max), s);
    SAP_CUDA(cudaMemcpyAsync(h->jobs.get(), jobs.data(), sizeof(FactorJob) * njobs, cudaMemcpyHostToDevice, s));
    h->kappa.alloc(3);
    SAP_CUDA(cudaMemsetAsync(h->kappa.get(), 0, 3 * sizeof(unsigned long long), s));
    launch_block_norms(h->band_ptr, m_max, k, h->d_boffs.get(), pl, nullptr, h->norms.get(), s);
    if (from_src)
        launch_zero_pad(k, h->d_boffs.get(), pl, h->fst, h->lu.get(), h->coupled ? h->ul.get() : nullptr, s);
    else
        launch_copy_blocks(h->band_ptr, k, h->d_boffs.get(), pl, h->fst, h->lu.get(),
                           h->coupled ? h->ul.get() : nullptr, s);
    SAP_CUDA(cudaEventRecord(h->ev[8], s));
    launch_band_lu(h->jobs.get(), njobs, k, h->opt.boost_eps, s, false, m_max, lu_scratch(h, njobs, m_max), h->opt.lu_kernel);
    SAP_CUDA(cudaEventRecord(h->ev[9], s));
    {
        SweepPlan<double>& lp = h->lplan;
        lp = SweepPlan<double>{};
        lp.f = h->lu.get();
        lp.st = h->fst;
        lp.offs = h->d_offsets.get();
        lp.p = pl;
        lp.k = k;
        h->dinv.alloc(std::max<size_t>(sweep_dinv_elems(lp), 1));
        plan_sweeps(lp, h->dinv.get());
        lp.kappa = h->kappa.get();
        launch_chunk_inverses(lp, s);
        // UL tip sweeps (sap_options::tip_solve), as in setup_banded; the choice is made over all ranks below
        SweepPlan<double>& up = h->uplan;
        up = SweepPlan<double>{};
        if (h->coupled && h->opt.tip_solve != 1 && lp.tma && lp.tr == 32 && tip_sweeps_fit(G.p)) {
            up.f = h->ul.get();
            up.st = h->fst;
            up.offs = h->d_offsets.get();
            up.p = pl;
            up.k = k;
            up.ul = true;
            h->udinv.alloc(std::max<size_t>(sweep_dinv_elems(up), 1));
            plan_sweeps(up, h->udinv.get());
            up.kappa = h->kappa.get() + 2;
            if (up.tma && up.tr == 32) launch_chunk_inverses(up, s);
        }
    }
    SAP_CUDA(cudaEventRecord(h->ev[2], s));
    for (int b = 0; b < pl; ++b) {
        const double m = L.sizes[b], kk = std::min<double>(k, m - 1 > 0 ? m - 1 : 0);
        const double f = (m - kk) * (2 * kk * kk + kk) + (kk - 1) * kk * (4 * kk + 1) / 6.0;
        h->rep.factor_flops += (h->coupled ? 2.0 : 1.0) * f;
    }

    // ---- interfaces: [left cross?] [local 0..pl-2] [right cross?] ----
    const int lc = h->coupled && h->has_left ? 1 : 0, rc = h->coupled && h->has_right ? 1 : 0;
    const int ni = h->coupled ? lc + (pl - 1) + rc : 0;
    h->ni_tot = ni;
    const int gi0 = pb - lc;  // global index of interface slot 0
    const int P = G.p;
    if (ni > 0) {
        const int w = k;
        const size_t ww = (size_t)w * w;
        std::vector<int> ioffs(ni + 1, 0);
        for (int t = 0; t < ni; ++t) {
            const int li = t - lc;  // local interface index (-1: left cross, pl-1: right cross)
            ioffs[t + 1] = li < 0 ? 0 : (li >= pl - 1 ? nl : L.offsets[li + 1]);
        }
        h->d_ioffs.alloc(ni + 1);
        SAP_CUDA(cudaMemcpyAsync(h->d_ioffs.get(), ioffs.data(), sizeof(int) * (ni + 1), cudaMemcpyHostToDevice, s));
        h->rst = BandStore::make(w, w - 1);
        for (auto* b : {&h->bblk, &h->cblk, &h->vb, &h->wt}) b->alloc(ww * ni);
        h->rbar.alloc(h->rst.total(ni));
        SAP_CUDA(cudaMemsetAsync(h->rbar.get(), 0, sizeof(double) * h->rst.total(ni), s));
        h->rbar_norms.alloc(ni);
        h->rbar_boosts.alloc(ni);
        h->nonfinite.alloc(3 * (size_t)ni);
        SAP_CUDA(cudaMemsetAsync(h->nonfinite.get(), 0, sizeof(int) * 3 * ni, s));
        SAP_CUDA(cudaMemsetAsync(h->rbar_boosts.get(), 0, sizeof(int) * ni, s));
        h->scratch_g.alloc((size_t)nl + 2 * w);
        SAP_CUDA(cudaMemsetAsync(h->scratch_g.get(), 0, sizeof(double) * ((size_t)nl + 2 * w), s));
        h->xt.alloc((size_t)ni * w);
        h->xb.alloc((size_t)ni * w);
        std::vector<int> roffs(ni + 1);
        for (int t = 0; t <= ni; ++t) roffs[t] = t * w;
        h->d_roffsets.alloc(ni + 1);
        SAP_CUDA(cudaMemcpyAsync(h->d_roffsets.get(), roffs.data(), sizeof(int) * (ni + 1), cudaMemcpyHostToDevice, s));
        // T_BC: every corner lies in this rank's column slice
        if (pl > 1)
            launch_extract_coupling(h->band_ptr, band_n, k, h->d_boffs.get(), pl, h->bblk.get() + lc * ww,
                                    h->cblk.get() + lc * ww, s);
        if (lc) {
            launch_extract_one(h->band_ptr, band_n, k, own, 0, h->bblk.get(), s);
            launch_extract_one(h->band_ptr, band_n, k, own, 1, h->cblk.get(), s);
        }
        if (rc) {
            launch_extract_one(h->band_ptr, band_n, k, own + nl, 0, h->bblk.get() + (ni - 1) * ww, s);
            launch_extract_one(h->band_ptr, band_n, k, own + nl, 1, h->cblk.get() + (ni - 1) * ww, s);
        }
        SAP_CUDA(cudaEventRecord(h->ev[3], s));
        // T_SPK: the tips this rank's factors give; V of the left cross / W of the right cross come
        // from the neighbours
        std::vector<TipJob> tj;
        for (int t = 0; t < ni; ++t) {
            const int li = t - lc;
            const size_t o = (size_t)t * ww;
            if (li >= 0)  // V^b from this rank's block li
                tj.push_back(TipJob{h->lu.get() + h->fst.block(li), L.sizes[li] - w, 0, h->bblk.get() + o,
                                    h->vb.get() + o, 2 * t});
            if (li + 1 < pl)  // W^t from this rank's block li+1
                tj.push_back(TipJob{h->ul.get() + h->fst.block(li + 1), 0, 1, h->cblk.get() + o, h->wt.get() + o,
                                    2 * t + 1});
        }
        h->tipjobs.alloc(tj.size());
        SAP_CUDA(cudaMemcpyAsync(h->tipjobs.get(), tj.data(), sizeof(TipJob) * tj.size(), cudaMemcpyHostToDevice, s));
        launch_spike_tips(h->tipjobs.get(), (int)tj.size(), k, h->nonfinite.get(), s);
        if (h->comm.world > 1) {
            const int cnt = (int)ww;
            comm_exchange_raw(h, lc ? h->wt.get() : nullptr, lc ? cnt : 0, rc ? h->vb.get() + (ni - 1) * ww : nullptr,
                              rc ? cnt : 0, lc ? h->vb.get() : nullptr, lc ? cnt : 0,
                              rc ? h->wt.get() + (ni - 1) * ww : nullptr, rc ? cnt : 0);
        }
        SAP_CUDA(cudaEventRecord(h->ev[4], s));
        // T_LUrdcd: every slot's R̄ (cross ones on both ranks)
        launch_rbar(h->wt.get(), h->vb.get(), w, ni, h->rbar.get(), h->rst, h->nonfinite.get() + 2 * ni, s);
        launch_block_norms(h->rbar.get(), w, w - 1, h->d_roffsets.get(), ni, &h->rst, h->rbar_norms.get(), s);
        std::vector<FactorJob> rj(ni);
        for (int t = 0; t < ni; ++t)
            rj[t] = FactorJob{h->rbar.get() + h->rst.block(t) + (w - 1), 1, 2LL * (w - 1), w, w - 1,
                              h->rbar_norms.get() + t, h->rbar_boosts.get() + t};
        h->rjobs.alloc(ni);
        SAP_CUDA(cudaMemcpyAsync(h->rjobs.get(), rj.data(), sizeof(FactorJob) * ni, cudaMemcpyHostToDevice, s));
        launch_band_lu(h->rjobs.get(), ni, w - 1, h->opt.boost_eps, s, false, w, lu_scratch(h, ni, w), h->opt.lu_kernel);
        SweepPlan<double>& rp = h->rplan;
        rp = SweepPlan<double>{};
        rp.f = h->rbar.get();
        rp.st = h->rst;
        rp.offs = h->d_roffsets.get();
        rp.p = ni;
        rp.k = w - 1;
        h->rdinv.alloc(std::max<size_t>(sweep_dinv_elems(rp), 1));
        plan_sweeps(rp, h->rdinv.get());
        rp.kappa = h->kappa.get() + 1;
        launch_chunk_inverses(rp, s);
        SAP_CUDA(cudaEventRecord(h->ev[5], s));
    }
    SAP_CUDA(cudaStreamSynchronize(s));
    lu_check(h);
    choose_triangle_solve(h);
    h->rep.t_dtransf = ev_ms(h->ev[0], h->ev[1]) * 1e-3;
    h->rep.t_lu = ev_ms(h->ev[1], h->ev[2]) * 1e-3;
    h->rep.t_factor_kernel = ev_ms(h->ev[8], h->ev[9]) * 1e-3;
    if (ni > 0) {
        h->rep.t_bc = ev_ms(h->ev[2], h->ev[3]) * 1e-3;
        h->rep.t_spk = ev_ms(h->ev[3], h->ev[4]) * 1e-3;
        h->rep.t_lurdcd = ev_ms(h->ev[4], h->ev[5]) * 1e-3;
    }
    // global failure flags and boost counts, summed over ranks so every rank raises the same error
    const int nig = P - 1;
    std::vector<double> gl(3 * (size_t)nig + 4, 0.0);
    {  // UL tip sweeps: vetoed on every rank if any rank cannot use them (the single-GPU choice, made globally)
        bool ok = h->uplan.ul && h->uplan.tma && h->uplan.tr == 32 && !h->lplan.subst &&
                  h->opt.triangle_solve != 2;
        if (ok) {
            unsigned long long kb = 0;
            SAP_CUDA(cudaStreamSynchronize(s));
            SAP_CUDA(cudaMemcpy(&kb, h->kappa.get() + 2, sizeof(kb), cudaMemcpyDeviceToHost));
            double kap;
            std::memcpy(&kap, &kb, sizeof(kap));
            ok = kap <= kSubstKappa;
        }
        gl[3 * (size_t)nig + 3] = (h->coupled && !ok) ? 1.0 : 0.0;
    }
    std::vector<int> hb(2 * pl);
    SAP_CUDA(cudaMemcpy(hb.data(), h->boosts.get(), sizeof(int) * 2 * pl, cudaMemcpyDeviceToHost));
    for (int b = 0; b < pl; ++b) {
        gl[3 * nig] += hb[b];
        gl[3 * nig + 1] += hb[pl + b];
    }
    if (ni > 0) {
        std::vector<int> nf(3 * ni), rb(ni);
        SAP_CUDA(cudaMemcpy(nf.data(), h->nonfinite.get(), sizeof(int) * 3 * ni, cudaMemcpyDeviceToHost));
        SAP_CUDA(cudaMemcpy(rb.data(), h->rbar_boosts.get(), sizeof(int) * ni, cudaMemcpyDeviceToHost));
        for (int t = 0; t < ni; ++t) {
            const int gi = gi0 + t;
            gl[2 * gi] += nf[2 * t];
            gl[2 * gi + 1] += nf[2 * t + 1];
            if (t >= lc) {  // a cross R̄ is counted by the rank on its left
                gl[2 * nig + gi] += nf[2 * ni + t];
                gl[3 * nig + 2] += rb[t];
            }
        }
    }
    comm_allreduce(h, gl.data(), (int)gl.size());
    h->rep.total_boosts = (int)gl[3 * nig];
    h->rep.total_boosts_ul = (int)gl[3 * nig + 1];
    h->rep.total_rbar_boosts = (int)gl[3 * nig + 2];
    h->ul_tips = h->coupled && gl[3 * (size_t)nig + 3] == 0.0 && h->rep.total_boosts == 0 && h->rep.total_boosts_ul == 0;
    if (h->ul_tips) {
        h->scratch_gu.alloc((size_t)h->n + 2 * k);
        SAP_CUDA(cudaMemsetAsync(h->scratch_gu.get(), 0, sizeof(double) * ((size_t)h->n + 2 * k), s));
    }
    h->rep.ul_tip_sweeps = h->ul_tips ? 1 : 0;
    for (int t = 0; t < nig; ++t) {
        if (gl[2 * t] != 0.0) throw PreconditionerFailure("right spike tip at interface " + std::to_string(t) + " is not finite");
        if (gl[2 * t + 1] != 0.0) throw PreconditionerFailure("left spike tip at interface " + std::to_string(t) + " is not finite");
    }
    for (int t = 0; t < nig; ++t)
        if (gl[2 * nig + t] != 0.0)
            throw PreconditionerFailure("reduced interface block " + std::to_string(t) + " is not finite");
    h->ready = true;
}

}  // namespace

extern "C" {

void sap_options_default(sap_options* o) {
    if (!o) return;
    o->p = 1;
    o->precond = SAP_PRECOND_COUPLED;
    o->boost_eps = 1e-10;
    o->method = SAP_KRYLOV_BICGSTAB_L;
    o->ell = 2;
    o->rel_tol = 1e-10;
    o->abs_tol = 0.0;
    o->max_iterations = 500;
    o->mixed_precision = 0;
    o->caller_asserts_spd = 0;
    o->device = 0;
    o->triangle_solve = 0;
    o->lu_kernel = 0;
    o->tip_solve = 0;
}

int sap_max_feasible_partitions(int n, int k) {
    if (n <= 0) return 0;
    return k == 0 ? n : n / (2 * k);
}

sap_status sap_partition_layout(int n, int p, int k, int* sizes, int* offsets) {
    return guard([&] {
        const Layout L = make_layout(n, p, k);
        if (sizes) std::copy(L.sizes.begin(), L.sizes.end(), sizes);
        if (offsets) std::copy(L.offsets.begin(), L.offsets.end(), offsets);
    });
}

const char* sap_last_error(void) { return g_last_error.c_str(); }

const char* sap_status_string(sap_status s) {
    switch (s) {
        case SAP_OK: return "ok";
        case SAP_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SAP_ERR_PRECONDITIONER: return "preconditioner error";
        case SAP_ERR_CUDA: return "cuda error";
        case SAP_ERR_COMM: return "communication error";
        case SAP_ERR_STATE: return "invalid call order";
    }
    return "unknown";
}

const char* sap_version(void) { return "sap_gpu 0.1 (sm_100a)"; }

sap_status sap_random_banded(int n, int k, double d, unsigned seed, double* band, double* rhs) {
    return guard([&] {
        require(n >= 0 && k >= 0, "BandedMatrix: negative dimension");
        require(band != nullptr || n == 0, "sap_random_banded: null band");
        // testsup::random_banded (proj/tests/test_support.hpp:133-150), same generator stream
        std::mt19937 rng(seed);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        const size_t w = 2 * (size_t)k + 1;
        std::memset(band, 0, sizeof(double) * (size_t)n * w);
        for (int i = 0; i < n; ++i) {
            double off = 0.0;
            const int lo = i - k > 0 ? i - k : 0;
            const int hi = i + k < n - 1 ? i + k : n - 1;
            for (int j = lo; j <= hi; ++j) {
                if (j == i) continue;
                double v = u(rng);
                if (v == 0.0) v = 0.5;
                band[(size_t)j * w + (size_t)(i - j + k)] = v;
                off += std::abs(v);
            }
            band[(size_t)i * w + (size_t)k] = off > 0.0 ? d * off : d;
        }
        if (rhs)
            for (int i = 0; i < n; ++i) rhs[i] = u(rng);
    });
}

sap_status sap_create(const sap_options* opts, sap_handle** out) {
    return guard([&] {
        require(out != nullptr, "sap_create: null output");
        *out = nullptr;
        auto* h = new sap_handle();
        if (opts)
            h->opt = *opts;
        else
            sap_options_default(&h->opt);
        try {
            SAP_CUDA(cudaSetDevice(h->opt.device));
            SAP_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
            h->stream = h->own_stream;
            for (auto& e : h->ev) SAP_CUDA(cudaEventCreate(&e));
            int least = 0, greatest = 0;
            SAP_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            SAP_CUDA(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, least));
            SAP_CUDA(cudaStreamCreateWithPriority(&h->prio, cudaStreamNonBlocking, greatest));
            SAP_CUDA(cudaEventCreateWithFlags(&h->pev, cudaEventDisableTiming));
            for (auto& e : h->sev) SAP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            SAP_CUDA(cudaStreamCreateWithFlags(&h->tside, cudaStreamNonBlocking));
            for (auto& e : h->tev) SAP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void sap_destroy(sap_handle* h) {
    if (!h) return;
    cudaSetDevice(h->opt.device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : h->sev)
        if (e) cudaEventDestroy(e);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->prio) cudaStreamDestroy(h->prio);
    for (auto& e : h->tev)
        if (e) cudaEventDestroy(e);
    if (h->tside) cudaStreamDestroy(h->tside);
    if (h->pev) cudaEventDestroy(h->pev);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    for (auto& e : h->cev)
        if (e) cudaEventDestroy(e);
    nccl_destroy(h->nccl);
    delete h;
}

sap_status sap_set_stream(sap_handle* h, void* stream) {
    return guard([&] {
        require(h != nullptr, "null handle");
        h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
    });
}

sap_status sap_synchronize(sap_handle* h) {
    return guard([&] {
        require(h != nullptr, "null handle");
        SAP_CUDA(cudaStreamSynchronize(h->stream));
    });
}

sap_status sap_setup_banded(sap_handle* h, int n, int k, const double* band, int band_on_device) {
    return guard([&] {
        require(h != nullptr, "null handle");
        require(!h->dist, "sap_setup_banded: use sap_setup_banded_dist on a distributed handle");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        h->csr = false;  // a dense setup's Krylov operator is its band (acceptance.cpp:114-132)
        setup_banded(h, n, k, band, band_on_device);
    });
}

sap_status sap_rank_rows(int n, int p, int k, int rank, int world, int* row_lo, int* row_hi) {
    return guard([&] {
        require(world >= 1 && rank >= 0 && rank < world, "sap_rank_rows: rank out of range");
        const Layout L = make_layout(n, p, k);
        require(p >= world, "sap_rank_rows: fewer partitions than ranks");
        const int b0 = (int)((long long)rank * p / world), b1 = (int)((long long)(rank + 1) * p / world);
        if (row_lo) *row_lo = L.offsets[b0];
        if (row_hi) *row_hi = L.offsets[b1];
    });
}

sap_status sap_create_distributed(const sap_options* opts, const sap_comm* comm, sap_handle** out) {
    return guard([&] {
        require(comm != nullptr && out != nullptr, "sap_create_distributed: null argument");
        require(comm->world >= 1 && comm->rank >= 0 && comm->rank < comm->world,
                "sap_create_distributed: rank out of range");
        require(comm->world == 1 || (comm->allreduce_sum && comm->exchange),
                "sap_create_distributed: missing communication callbacks");
        const sap_status st = sap_create(opts, out);
        if (st != SAP_OK) throw InvalidArgument(g_last_error);
        (*out)->dist = true;
        (*out)->comm = *comm;
    });
}

sap_status sap_nccl_get_unique_id(unsigned char* id) {
    return guard([&] {
        require(id != nullptr, "sap_nccl_get_unique_id: null argument");
        nccl_unique_id(id);
    });
}

sap_status sap_create_distributed_nccl(const sap_options* opts, const unsigned char* id, int rank, int world,
                                       sap_handle** out) {
    return guard([&] {
        require(id != nullptr && out != nullptr, "sap_create_distributed_nccl: null argument");
        require(world >= 1 && rank >= 0 && rank < world, "sap_create_distributed_nccl: rank out of range");
        const sap_status st = sap_create(opts, out);
        if (st != SAP_OK) throw InvalidArgument(g_last_error);
        sap_handle* h = *out;
        h->dist = true;
        h->comm = sap_comm{};
        h->comm.rank = rank;
        h->comm.world = world;
        try {
            SAP_CUDA(cudaSetDevice(h->opt.device));
            h->nccl = nccl_create(id, rank, world);
        } catch (...) {
            sap_destroy(h);
            *out = nullptr;
            throw;
        }
    });
}

sap_status sap_setup_banded_dist(sap_handle* h, int n, int k, int row_lo, int row_hi, const double* band_slice,
                                 int on_device) {
    return guard([&] {
        require(h != nullptr, "null handle");
        require(h->dist, "sap_setup_banded_dist: handle was not created by sap_create_distributed");
        require(!h->ts_armed, "sap_setup_banded_dist: the third stage is not distributed");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        setup_banded_dist(h, n, k, row_lo, row_hi, band_slice, on_device);
    });
}

namespace {
// CSR (host or device) -> device pointers held by the handle
void csr_to_device(sap_handle* h, int n, int nnz, const int*& rp, const int*& ci, const double*& v, int on_device) {
    if (on_device) return;
    const cudaStream_t s = h->stream;
    h->asm_rp.alloc(n + 1);
    h->asm_ci.alloc(std::max(nnz, 1));
    h->asm_v.alloc(std::max(nnz, 1));
    SAP_CUDA(cudaMemcpyAsync(h->asm_rp.get(), rp, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
        SAP_CUDA(cudaMemcpyAsync(h->asm_ci.get(), ci, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
        SAP_CUDA(cudaMemcpyAsync(h->asm_v.get(), v, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    rp = h->asm_rp.get();
    ci = h->asm_ci.get();
    v = h->asm_v.get();
}

void csr_event(sap_handle* h, int i) {
    if (!h->cev[i]) SAP_CUDA(cudaEventCreate(&h->cev[i]));
    SAP_CUDA(cudaEventRecord(h->cev[i], h->stream));
}

// assemble_banded on the device; drop = true filters |i - j| > k (drop_off) instead of failing. The report's
// t_drop (cev[0] -> cev[1], recorded by the caller around drop_off) and t_asmbl (cev[1] -> cev[2]) are
// filled in after the setup (which resets the report).
void assemble_and_setup(sap_handle* h, int n, int k, const int* rp, const int* ci, const double* v, bool drop,
                        bool timed_drop) {
    const cudaStream_t s = h->stream;
    if (!timed_drop) {
        csr_event(h, 0);
        csr_event(h, 1);
    }
    const size_t total = (size_t)n * (2 * (size_t)k + 1);
    h->asm_band.alloc(std::max<size_t>(total, 1));
    SAP_CUDA(cudaMemsetAsync(h->asm_band.get(), 0, sizeof(double) * total, s));
    h->asm_bad.alloc(1);
    SAP_CUDA(cudaMemsetAsync(h->asm_bad.get(), 0xff, sizeof(unsigned long long), s));
    launch_assemble_band(rp, ci, v, n, k, h->asm_band.get(), drop ? nullptr : h->asm_bad.get(), s);
    unsigned long long bad = 0;
    SAP_CUDA(cudaMemcpyAsync(&bad, h->asm_bad.get(), sizeof(bad), cudaMemcpyDeviceToHost, s));
    SAP_CUDA(cudaStreamSynchronize(s));
    if (bad != ~0ULL)
        throw InvalidArgument("assemble_banded: entry (" + std::to_string(bad / (unsigned long long)n) + ", " +
                              std::to_string(bad % (unsigned long long)n) + ") outside half-bandwidth " +
                              std::to_string(k));
    csr_event(h, 2);
    // solve_sparse's partition count (pipeline.hpp:291-301): reduced to max_feasible_partitions(n, k) when
    // the requested p would leave a block below 2k rows
    const int p_req = h->opt.p;
    const int p_max = sap_max_feasible_partitions(n, k);
    if (p_max >= 1 && p_req > p_max) h->opt.p = p_max;
    try {
        setup_banded(h, n, k, h->asm_band.get(), 2);
    } catch (...) {
        h->opt.p = p_req;
        throw;
    }
    h->opt.p = p_req;
    h->rep.t_drop = timed_drop ? ev_ms(h->cev[0], h->cev[1]) * 1e-3 : 0.0;
    h->rep.t_asmbl = ev_ms(h->cev[1], h->cev[2]) * 1e-3;
}
}  // namespace

sap_status sap_setup_banded_from_csr(sap_handle* h, int n, int k, int nnz, const int* row_ptr, const int* col_idx,
                                     const double* values, int csr_on_device) {
    return guard([&] {
        require(h != nullptr, "null handle");
        require(!h->dist, "sap_setup_banded_from_csr: not available on a distributed handle");
        require(n >= 0 && k >= 0 && nnz >= 0, "BandedMatrix: negative dimension");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const int* rp = row_ptr;
        const int* ci = col_idx;
        const double* v = values;
        h->csr = false;  // cleared by every setup; sap_set_operator_csr after it re-arms the CSR operator
        csr_to_device(h, n, nnz, rp, ci, v, csr_on_device);
        assemble_and_setup(h, n, k, rp, ci, v, false, false);
    });
}

sap_status sap_setup_from_csr_drop(sap_handle* h, int n, int nnz, const int* row_ptr, const int* col_idx,
                                   const double* values, double drop_tol, int csr_on_device, int* k_after) {
    return guard([&] {
        require(h != nullptr, "null handle");
        require(!h->dist, "sap_setup_from_csr_drop: not available on a distributed handle");
        require(n >= 0 && nnz >= 0, "sap_setup_from_csr_drop: negative size");
        if (!(drop_tol >= 0.0 && drop_tol <= 1.0)) throw InvalidArgument("drop_off: tolerance must lie in [0, 1]");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const int* rp = row_ptr;
        const int* ci = col_idx;
        const double* v = values;
        h->csr = false;
        csr_to_device(h, n, nnz, rp, ci, v, csr_on_device);
        csr_event(h, 0);
        const int k = drop_off_k(rp, ci, v, n, nnz, drop_tol, h->stream);
        csr_event(h, 1);
        if (k_after) *k_after = k;
        assemble_and_setup(h, n, k, rp, ci, v, drop_tol > 0.0, true);
    });
}

sap_status sap_set_operator_csr(sap_handle* h, int n, int nnz, const int* row_ptr, const int* col_idx,
                                const double* values, int on_device) {
    return guard([&] {
        require(h != nullptr, "null handle");
        require(n >= 0 && nnz >= 0, "sap_set_operator_csr: negative size");
        require(!h->dist, "sap_set_operator_csr: not available on a distributed handle");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        h->rp.alloc(n + 1);
        h->ci.alloc(std::max(nnz, 1));
        h->vals.alloc(std::max(nnz, 1));
        SAP_CUDA(cudaMemcpyAsync(h->rp.get(), row_ptr, sizeof(int) * (n + 1), kind, h->stream));
        if (nnz > 0) {
            SAP_CUDA(cudaMemcpyAsync(h->ci.get(), col_idx, sizeof(int) * nnz, kind, h->stream));
            SAP_CUDA(cudaMemcpyAsync(h->vals.get(), values, sizeof(double) * nnz, kind, h->stream));
        }
        SAP_CUDA(cudaStreamSynchronize(h->stream));
        h->csr = true;
        h->csr_n = n;
    });
}

static void io_apply(sap_handle* h, const double* in, double* out, int on_device, bool precond) {
    require(h != nullptr, "null handle");
    SAP_CUDA(cudaSetDevice(h->opt.device));
    if (precond && !h->ready) throw StateError("preconditioner applied before setup");
    if (!precond && !h->csr && !h->ready) throw StateError("operator applied before setup");
    const int n = precond ? h->n : op_n(h);
    if (n == 0) return;
    const size_t bytes = sizeof(double) * (size_t)n;
    const double* din = in;
    double* dout = out;
    if (!on_device) {
        h->scratch_in.alloc(n);
        h->scratch_out.alloc(n);
        SAP_CUDA(cudaMemcpyAsync(h->scratch_in.get(), in, bytes, cudaMemcpyHostToDevice, h->stream));
        din = h->scratch_in.get();
        dout = h->scratch_out.get();
    }
    if (precond)
        apply_m(h, din, dout);
    else
        apply_a(h, din, dout);
    if (!on_device) SAP_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, h->stream));
    SAP_CUDA(cudaStreamSynchronize(h->stream));
}

sap_status sap_apply_preconditioner(sap_handle* h, const double* in, double* out, int on_device) {
    return guard([&] { io_apply(h, in, out, on_device, true); });
}

sap_status sap_apply_operator(sap_handle* h, const double* in, double* out, int on_device) {
    return guard([&] { io_apply(h, in, out, on_device, false); });
}

sap_status sap_solve(sap_handle* h, const double* b, double* x, int on_device, sap_solve_stats* stats) {
    return guard([&] {
        require(h != nullptr, "null handle");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const bool m_ok = h->ready;
        const bool a_ok = h->csr || h->ready;
        if (!a_ok) throw StateError("sap_solve before setup");
        const int n = op_n(h);
        if (!m_ok && h->opt.precond != SAP_PRECOND_NONE) throw StateError("sap_solve before preconditioner setup");
        if (m_ok && h->n != n) throw InvalidArgument("sap_solve: operator and preconditioner sizes differ");
        const cudaStream_t s = h->stream;
        const size_t bytes = sizeof(double) * (size_t)n;
        const double* db = b;
        double* dx = x;
        if (!on_device) {
            h->kb.alloc(std::max(n, 1));
            h->kx.alloc(std::max(n, 1));
            if (n) SAP_CUDA(cudaMemcpyAsync(h->kb.get(), b, bytes, cudaMemcpyHostToDevice, s));
            db = h->kb.get();
            dx = h->kx.get();
        }
        KrylovConfig kc;
        kc.method = h->opt.method;
        kc.ell = h->opt.ell;
        kc.rel_tol = h->opt.rel_tol;
        kc.abs_tol = h->opt.abs_tol;
        kc.max_iterations = h->opt.max_iterations;
        kc.caller_asserts_spd = h->opt.caller_asserts_spd != 0;
        kc.zero_guess_exact = h->op_finite && !h->csr && !h->dist;
        if (h->dist && h->comm.world > 1) {
            kc.reduce = [h](double* v, int c) { comm_allreduce(h, v, c); };
            if (h->nccl)  // dot products reduced on the device before their one copy to the host
                kc.dreduce = [h](double* d, int c, cudaStream_t st) { nccl_allreduce(h->nccl, d, c, st); };
            kc.row_offset = h->row_lo;
        }
        DeviceOp A = [h](const double* in, double* out) { apply_a(h, in, out); };
        DeviceOp M = [h](const double* in, double* out) {
            if (h->ready)
                apply_m(h, in, out);
            else if (out != in)
                SAP_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * (size_t)op_n(h), cudaMemcpyDeviceToDevice,
                                         h->stream));
        };
        DeviceOp2 A2;  // banded operator on one GPU: A r_j and the true residual's A x in one band read
        if (!h->dist && !h->csr)
            A2 = [h](const double* i0, double* o0, const double* i1, double* o1) {
                launch_band_spmv2(h->band_ptr, h->n, h->k, i0, o0, i1, o1, h->stream);
            };
        SAP_CUDA(cudaEventRecord(h->ev[6], s));
        const KrylovResult r = h->krylov.run(A, M, db, dx, n, kc, s, A2);
        SAP_CUDA(cudaEventRecord(h->ev[7], s));
        if (!on_device && n) SAP_CUDA(cudaMemcpyAsync(x, dx, bytes, cudaMemcpyDeviceToHost, s));
        SAP_CUDA(cudaStreamSynchronize(s));
        h->rep.t_kry = ev_ms(h->ev[6], h->ev[7]) * 1e-3;
        h->rep.krylov_host_syncs = h->krylov.host_syncs();
        if (stats) {
            stats->iterations = r.iterations;
            stats->converged = r.converged ? 1 : 0;
            stats->final_relative_residual = r.final_relative_residual;
            stats->failure = r.failure;
            stats->history_len = (int)r.residual_history.size();
            if (stats->history && stats->history_capacity > 0) {
                const int c = std::min(stats->history_capacity, stats->history_len);
                std::copy(r.residual_history.begin(), r.residual_history.begin() + c, stats->history);
            }
        }
    });
}

sap_status sap_get_report(const sap_handle* h, sap_report* rep) {
    return guard([&] {
        require(h != nullptr && rep != nullptr, "null argument");
        *rep = h->rep;
        rep->kernel_launches = g_launch_count;
    });
}

sap_status sap_get_factor(sap_handle* h, int part, int which, double* out, int* boosts, double* block_norm) {
    return guard([&] {
        require(h != nullptr, "null handle");
        if (!h->ready) throw StateError("sap_get_factor before setup");
        require(h->kind == SAP_PRECOND_COUPLED || h->kind == SAP_PRECOND_DECOUPLED,
                "sap_get_factor: no block factors for this preconditioner kind");
        if (h->dist) {
            require(part >= h->pb && part < h->pe, "sap_get_factor: partition not on this rank");
            part -= h->pb;
        }
        require(part >= 0 && part < h->layout.p, "sap_get_factor: partition out of range");
        require(which == 0 || which == 1, "sap_get_factor: which must be 0 (LU) or 1 (UL)");
        if (which == 1 && (!h->coupled || (h->f32fac ? h->ul_f.get() == nullptr : h->ul.get() == nullptr)))
            throw InvalidArgument("block_solve: UL factors not available");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const size_t w = 2 * (size_t)h->k + 1;
        if (h->f32fac) {  // factor_blocks<float>'s factors, widened
            const int m = h->layout.sizes[part];
            if (out) {
                std::vector<float> f((size_t)m * w);
                SAP_CUDA(cudaMemcpy(f.data(), (which == 0 ? h->lu_f.get() : h->ul_f.get()) + h->fst.block(part),
                                    sizeof(float) * f.size(), cudaMemcpyDeviceToHost));
                for (size_t i = 0; i < f.size(); ++i) out[i] = f[i];
            }
            if (boosts)
                SAP_CUDA(cudaMemcpy(boosts, h->boosts.get() + (which == 0 ? 0 : h->layout.p) + part, sizeof(int),
                                    cudaMemcpyDeviceToHost));
            if (block_norm)
                SAP_CUDA(cudaMemcpy(block_norm, h->norms.get() + part, sizeof(double), cudaMemcpyDeviceToHost));
            return;
        }
        const double* src = (which == 0 ? h->lu.get() : h->ul.get()) + h->fst.block(part);
        const int m = h->layout.sizes[part];
        if (out && h->ts && h->ts_k[part] != h->k) {
            // third stage: the reference stores block b at its own bandwidth K_b (block_factors.hpp:158-160)
            std::vector<double> band((size_t)m * w);
            SAP_CUDA(cudaMemcpy(band.data(), src, sizeof(double) * band.size(), cudaMemcpyDeviceToHost));
            const int k = h->k, kb = h->ts_k[part];
            const size_t wb = 2 * (size_t)kb + 1;
            for (int j = 0; j < m; ++j)
                for (int d = -kb; d <= kb; ++d) out[(size_t)j * wb + d + kb] = band[(size_t)j * w + d + k];
        } else if (out) {
            SAP_CUDA(cudaMemcpy(out, src, sizeof(double) * (size_t)m * w, cudaMemcpyDeviceToHost));
        }
        if (boosts)
            SAP_CUDA(cudaMemcpy(boosts, h->boosts.get() + (which == 0 ? 0 : h->layout.p) + part, sizeof(int),
                                cudaMemcpyDeviceToHost));
        if (block_norm) SAP_CUDA(cudaMemcpy(block_norm, h->norms.get() + part, sizeof(double), cudaMemcpyDeviceToHost));
    });
}

sap_status sap_set_third_stage(sap_handle* h, int p, const int* block_k, const int* has_perm, const int* perm,
                               int n) {
    return guard([&] {
        require(h != nullptr, "null handle");
        if (!block_k) {
            h->ts_armed = false;
            return;
        }
        require(p >= 1 && n >= 0, "sap_set_third_stage: bad sizes");
        require(perm != nullptr || has_perm == nullptr, "sap_set_third_stage: has_perm without perm");
        h->ts_k.assign(block_k, block_k + p);
        h->ts_has.assign(p, 0);
        if (has_perm) h->ts_has.assign(has_perm, has_perm + p);
        h->ts_perm.assign(n, 0);
        if (perm) h->ts_perm.assign(perm, perm + n);
        h->ts_armed = true;
    });
}

sap_status sap_get_full_spike(sap_handle* h, int iface, double* v_full, double* w_full) {
    return guard([&] {
        require(h != nullptr, "null handle");
        if (!h->ready) throw StateError("sap_get_full_spike before setup");
        require(h->ts && h->coupled, "sap_get_full_spike: full spikes exist only for the coupled third stage");
        require(iface >= 0 && iface < h->layout.p - 1, "sap_get_full_spike: interface out of range");
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const int k = h->k, w = h->widths[iface], o = k - w;
        for (int side = 0; side < 2; ++side) {
            double* out = side == 0 ? v_full : w_full;
            if (!out) continue;
            const int b = iface + side, off = h->layout.offsets[b], m = h->layout.sizes[b];
            std::vector<double> X((size_t)m * k);
            SAP_CUDA(cudaMemcpy(X.data(), (side == 0 ? h->vfull.get() : h->wfull.get()) + (size_t)off * k,
                                sizeof(double) * X.size(), cudaMemcpyDeviceToHost));
            // reference layout: m x w column-major in original row order (spike.hpp:266-276)
            for (int r = 0; r < m; ++r) {
                const int pr = h->ts_has[b] ? h->ts_perm[off + r] : r;
                for (int c = 0; c < w; ++c) out[(size_t)c * m + r] = X[(size_t)pr * k + (side == 0 ? c : o + c)];
            }
        }
    });
}

sap_status sap_get_spike(sap_handle* h, int iface, double* b_block, double* c_block, double* v_bottom, double* w_top,
                         double* rbar, int* rbar_boosts) {
    return guard([&] {
        require(h != nullptr, "null handle");
        if (!h->ready) throw StateError("sap_get_spike before setup");
        require(h->coupled, "sap_get_spike: no spikes (not a coupled preconditioner with p > 1)");
        if (h->dist) {
            const int slot = iface - (h->pb - (h->has_left ? 1 : 0));
            require(slot >= 0 && slot < h->ni_tot, "sap_get_spike: interface not on this rank");
            iface = slot;
        } else {
            require(iface >= 0 && iface < h->layout.p - 1, "sap_get_spike: interface out of range");
        }
        SAP_CUDA(cudaSetDevice(h->opt.device));
        const size_t ww = (size_t)h->k * h->k, off = ww * iface, bytes = sizeof(double) * ww;
        if (h->f32fac) {  // compute_spike_tips<float> / finish_reduced_blocks<float>, widened
            auto get = [&](double* dst, const float* src) {
                if (!dst) return;
                std::vector<float> f(ww);
                SAP_CUDA(cudaMemcpy(f.data(), src + off, sizeof(float) * ww, cudaMemcpyDeviceToHost));
                for (size_t i = 0; i < ww; ++i) dst[i] = f[i];
            };
            get(b_block, h->bblk_f.get());
            get(c_block, h->cblk_f.get());
            get(v_bottom, h->vb_f.get());
            get(w_top, h->wt_f.get());
            if (rbar && h->k > 0) {
                const int w = h->k;
                std::vector<float> band((size_t)w * (2 * (size_t)w - 1));
                SAP_CUDA(cudaMemcpy(band.data(), h->rbar_f.get() + h->rst.block(iface), sizeof(float) * band.size(),
                                    cudaMemcpyDeviceToHost));
                for (int i = 0; i < w; ++i)
                    for (int j = 0; j < w; ++j) rbar[(size_t)i * w + j] = band[(size_t)j * (2 * w - 1) + (i - j + w - 1)];
            }
            if (rbar_boosts)
                SAP_CUDA(cudaMemcpy(rbar_boosts, h->rbar_boosts.get() + iface, sizeof(int), cudaMemcpyDeviceToHost));
            return;
        }
        if (h->ts) {
            // third stage: interface width w_t <= k, embedded in the k x k corners (third.cu header)
            const int k = h->k, w = h->widths[iface], o = k - w;
            std::vector<double> B(ww), Cc(ww), V(ww), W(ww);
            SAP_CUDA(cudaMemcpy(B.data(), h->bblk.get() + off, bytes, cudaMemcpyDeviceToHost));
            SAP_CUDA(cudaMemcpy(Cc.data(), h->cblk.get() + off, bytes, cudaMemcpyDeviceToHost));
            SAP_CUDA(cudaMemcpy(V.data(), h->vb.get() + off, bytes, cudaMemcpyDeviceToHost));
            SAP_CUDA(cudaMemcpy(W.data(), h->wt.get() + off, bytes, cudaMemcpyDeviceToHost));
            std::vector<double> band((size_t)k * (2 * (size_t)k - 1));
            if (rbar && k > 0)
                SAP_CUDA(cudaMemcpy(band.data(), h->rbar.get() + h->rst.block(iface), sizeof(double) * band.size(),
                                    cudaMemcpyDeviceToHost));
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j) {
                    const size_t d = (size_t)i * w + j;
                    if (b_block) b_block[d] = B[(size_t)(o + i) * k + j];
                    if (c_block) c_block[d] = Cc[(size_t)i * k + o + j];
                    if (v_bottom) v_bottom[d] = V[(size_t)(o + i) * k + j];
                    if (w_top) w_top[d] = W[(size_t)i * k + o + j];
                    if (rbar) rbar[d] = band[(size_t)j * (2 * k - 1) + (i - j + k - 1)];
                }
            if (rbar_boosts)
                SAP_CUDA(cudaMemcpy(rbar_boosts, h->rbar_boosts.get() + iface, sizeof(int), cudaMemcpyDeviceToHost));
            return;
        }
        if (b_block) SAP_CUDA(cudaMemcpy(b_block, h->bblk.get() + off, bytes, cudaMemcpyDeviceToHost));
        if (c_block) SAP_CUDA(cudaMemcpy(c_block, h->cblk.get() + off, bytes, cudaMemcpyDeviceToHost));
        if (v_bottom) SAP_CUDA(cudaMemcpy(v_bottom, h->vb.get() + off, bytes, cudaMemcpyDeviceToHost));
        if (w_top) SAP_CUDA(cudaMemcpy(w_top, h->wt.get() + off, bytes, cudaMemcpyDeviceToHost));
        if (rbar && h->k > 0) {
            const int w = h->k;
            const size_t rb = (size_t)w * (2 * (size_t)w - 1);
            std::vector<double> band(rb);
            SAP_CUDA(cudaMemcpy(band.data(), h->rbar.get() + h->rst.block(iface), sizeof(double) * rb,
                                cudaMemcpyDeviceToHost));
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j) rbar[(size_t)i * w + j] = band[(size_t)j * (2 * w - 1) + (i - j + w - 1)];
        }
        if (rbar_boosts)
            SAP_CUDA(cudaMemcpy(rbar_boosts, h->rbar_boosts.get() + iface, sizeof(int), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
