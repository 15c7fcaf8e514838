/*
 * sap_gpu.h — C ABI of the B200-native SaP (split-and-parallelize) banded
 * solver hot path (arXiv 1509.07919). Implemented by libsap_gpu.so
 * (paper_1509_07919_b200/csrc/). Plain C types only: no CUDA, no torch and no
 * C++ types cross this boundary; every call returns a sap_status and never
 * throws.
 *
 * The reference (/root/reference/proj, header-only C++20) has no FFI; its
 * hot-path boundary is the in-process C++ interface below, and each entry
 * point names the reference function it replaces:
 *
 *   setup  ≙ sap::detail::build_precond_op<T>      proj/include/sap/pipeline.hpp:140-202
 *            (factor_blocks block_factors.hpp:138-206, extract_coupling spike.hpp:95-116,
 *             compute_spike_tips spike.hpp:178-254, finish_reduced_blocks spike.hpp:143-170)
 *   M op   ≙ the returned LinearOp / apply_preconditioner   spike.hpp:304-351, krylov.hpp:14
 *   A op   ≙ BandedMatrix::matvec banded_matrix.hpp:72-80 / SparseMatrix::matvec sparse_matrix.hpp:24-31
 *   solve  ≙ sap::run_krylov (BiCGStab(l) solve_krylov)   krylov.hpp:434-442, :110-350
 *
 * Error mapping (status -> the reference's exception / failure channel):
 *   SAP_ERR_INVALID_ARGUMENT  std::invalid_argument   (partition.hpp:52-63, block_factors.hpp:142-143,
 *                                                      spike.hpp:180-184, :311-318, krylov.hpp:115)
 *   SAP_ERR_PRECONDITIONER    sap::PreconditionerError (errors.hpp:17-20; spike.hpp:162-164, :217-219, :246-248)
 *   Krylov numerical failures are NOT errors: sap_solve returns SAP_OK with
 *   sap_solve_stats.failure set, exactly like SolveStats.failure (krylov.hpp:18, :35-41).
 *   SAP_ERR_CUDA / SAP_ERR_COMM / SAP_ERR_STATE have no reference analogue
 *   (device, communicator, call-order errors).
 *
 * Storage conventions (identical to the reference):
 *   band   : "tall and thin" column-major, n*(2k+1) doubles, entry (i, j) at
 *            j*(2k+1) + (i-j+k); out-of-matrix slots are zero (banded_matrix.hpp:22-51).
 *   blocks : coupling corners, spike tips and reduced blocks are dense
 *            row-major w x w (spike.hpp:80-138).
 * Pointers flagged *_on_device are CUDA device pointers on the handle's
 * device; otherwise host pointers (pageable or pinned).
 *
 * Threading: a handle is single-threaded and owns one CUDA stream; separate
 * handles may run concurrently.
 */
#ifndef SAP_GPU_H
#define SAP_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sap_status {
    SAP_OK = 0,
    SAP_ERR_INVALID_ARGUMENT = 1,
    SAP_ERR_PRECONDITIONER = 2,
    SAP_ERR_CUDA = 3,
    SAP_ERR_COMM = 4,
    SAP_ERR_STATE = 5
} sap_status;

/* sap::PrecondKind, proj/include/sap/spike.hpp:14 (same order). */
typedef enum sap_precond_kind {
    SAP_PRECOND_COUPLED = 0,   /* SaP-C: truncated SPIKE */
    SAP_PRECOND_DECOUPLED = 1, /* SaP-D: block Jacobi */
    SAP_PRECOND_DIAGONAL = 2,
    SAP_PRECOND_NONE = 3
} sap_precond_kind;

/* sap::KrylovMethod, proj/include/sap/krylov.hpp:16. */
typedef enum sap_krylov_method {
    SAP_KRYLOV_BICGSTAB_L = 0,
    SAP_KRYLOV_CG = 1,
    SAP_KRYLOV_AUTOMATIC = 2
} sap_krylov_method;

/* sap::KrylovFailure, proj/include/sap/krylov.hpp:18. */
typedef enum sap_krylov_failure {
    SAP_FAILURE_NONE = 0,
    SAP_FAILURE_MAX_ITERATIONS = 1,
    SAP_FAILURE_BREAKDOWN = 2,
    SAP_FAILURE_NON_FINITE = 3,
    SAP_FAILURE_INDEFINITE_OPERATOR = 4
} sap_krylov_failure;

/* PipelineConfig (pipeline.hpp:21-32) fields that reach the hot path, plus
 * KrylovOptions (krylov.hpp:20-28). Defaults from sap_options_default() equal
 * the reference's member initialisers. */
typedef struct sap_options {
    int p;                   /* partition count (PipelineConfig::p), default 1 */
    int precond;             /* sap_precond_kind, default SAP_PRECOND_COUPLED */
    double boost_eps;        /* pivot boosting threshold factor, default 1e-10 */
    int method;              /* sap_krylov_method, default SAP_KRYLOV_BICGSTAB_L */
    int ell;                 /* BiCGStab(l) degree, default 2 */
    double rel_tol;          /* default 1e-10 */
    double abs_tol;          /* default 0 */
    int max_iterations;      /* default 500 */
    int mixed_precision;     /* FP32 preconditioner (build_precond_op<float>), default 0 */
    int caller_asserts_spd;  /* lets AUTOMATIC pick CG, default 0 */
    int device;              /* CUDA device ordinal, default 0 */
    /* 32-row chunk triangles of the block solves (sweeps, third-stage full spikes): 0 = automatic (explicit
     * chunk inverses unless their condition estimate exceeds 1e4, then substitution),
     * 1 = always the inverse products, 2 = always substitution (the reference's band_lu_solve order).
     * Not a reference option: it selects between two implementations of block_solve. Default 0. */
    int triangle_solve;
    /* Band LU kernel (not a reference option: two implementations of band_lu_inplace / band_ul_inplace with
     * bitwise-equal factors): 0 = automatic (the dataflow kernel for K in [192, 224] with at
     * most 0.7 x SMs jobs of at least 512 rows and for K in (224, 512], else one CTA per job), 1 = one CTA per job,
     * 2 = the dataflow kernel wherever it supports the bandwidth (K in [64, 512]). Default 0. */
    int lu_kernel;
    /* SaP-C apply, first block solve g = D^{-1} r (not a reference option: the interfaces read only g's first
     * and last w rows of every block): 0 = automatic (the last rows from the LU sweeps with the backward sweep
     * stopped there, the first rows from UL sweeps over the UL factors with the top-down sweep stopped there,
     * both at once -- when no LU or UL pivot was boosted and both stores' chunk triangles are well
     * conditioned; equal to the LU solve's rows up to rounding), 1 = the full LU block solve
     * (spike.hpp:323-329). Default 0. */
    int tip_solve;
} sap_options;

/* PipelineReport T_* stage timings (pipeline.hpp:37-52), in seconds,
 * measured with CUDA events on the handle's stream. */
typedef struct sap_report {
    double t_lu;      /* factor_blocks: block norms, band copies, LU (+UL) */
    double t_bc;      /* extract_coupling */
    double t_spk;     /* spike tips */
    double t_lurdcd;  /* reduced blocks: R = I - W V and its LU */
    double t_kry;     /* last sap_solve (Krylov), device-resident */
    double t_dtransf; /* host->device upload of the band in the last setup */
    int n, k, partitions;
    int total_boosts;     /* LU boosts summed over blocks */
    int total_boosts_ul;  /* UL boosts summed over blocks */
    int total_rbar_boosts;
    long long kernel_launches; /* sm_100a kernels launched by this process so far */
    double t_factor_kernel;    /* device time of the block LU/UL factorization launch alone */
    double factor_flops;       /* algorithmic flops of that launch (band_lu_inplace op count) */
    /* sweeps: max over 32-row chunks of ||T|| ||T^-1|| of the LU chunk triangles (T^-1 explicit); above 1e4
     * the block solves use substitution instead of the inverse products (1 = substitution) */
    double chunk_condition;
    int sweep_substitution;
    /* CSR setups (sap_setup_banded_from_csr, sap_setup_from_csr_drop): drop_off on the device (T_Drop) and
     * the band assembly (T_Asmbl), CUDA events; 0 for the other setups */
    double t_drop;
    double t_asmbl;
    /* host synchronisations of the last sap_solve (each scalar the host recurrences need costs one; the dot
     * products a step needs next ride with its true residual, MGS runs on device scalars) */
    long long krylov_host_syncs;
    /* 1 if the last setup's SaP-C applies form g's interface rows from LU + UL tip sweeps (tip_solve) */
    int ul_tip_sweeps;
} sap_report;

/* SolveStats (krylov.hpp:35-41). history: caller-owned buffer of
 * history_capacity doubles (may be NULL); history_len is the full count. */
typedef struct sap_solve_stats {
    double iterations;
    int converged;
    double final_relative_residual;
    int failure; /* sap_krylov_failure */
    int history_len;
    double* history;
    int history_capacity;
} sap_solve_stats;

typedef struct sap_handle sap_handle;

/* ---- options / layout (host logic; no device work) ---- */
void sap_options_default(sap_options* opts);
/* max_feasible_partitions, partition.hpp:34-37 */
int sap_max_feasible_partitions(int n, int k);
/* make_partition_layout, partition.hpp:42-69: sizes[p], offsets[p+1].
 * SAP_ERR_INVALID_ARGUMENT with the reference's message on infeasible input. */
sap_status sap_partition_layout(int n, int p, int k, int* sizes, int* offsets);
/* Message of the last failed call on this thread (handle-independent). */
const char* sap_last_error(void);
const char* sap_status_string(sap_status s);
/* libsap_gpu version / build string. */
const char* sap_version(void);

/* ---- synthetic input: testsup::random_banded (proj/tests/test_support.hpp:133-150)
 * followed, if rhs != NULL, by random_rhs (proj/tests/acceptance.cpp:48-53). ---- */
sap_status sap_random_banded(int n, int k, double d, unsigned seed, double* band, double* rhs);

/* ---- handle ---- */
sap_status sap_create(const sap_options* opts, sap_handle** out);
void sap_destroy(sap_handle* h);
/* Use an external CUDA stream (cudaStream_t passed as void*); NULL = the handle's own. */
sap_status sap_set_stream(sap_handle* h, void* stream);
sap_status sap_synchronize(sap_handle* h);

/* ---- setup ≙ build_precond_op<double|float> over make_partition_layout(n, opts.p, k).
 * Installs the band as the Krylov A operator too (the dense wiring of
 * proj/tests/acceptance.cpp:114-132). band_on_device: 0 = host pointer, copied (for the block
 * preconditioners the copy is streamed in rounds under the factorization; pinned memory overlaps best);
 * 1 = device pointer, copied; 2 = device pointer BORROWED for the A operator
 * (no copy; it must stay valid while the handle applies A, like the
 * reference's LinearOp capturing the BandedMatrix by reference). */
sap_status sap_setup_banded(sap_handle* h, int n, int k, const double* band, int band_on_device);

/* setup from a sparse matrix (pipeline.hpp:103-115 assemble_banded + build_precond_op): the CSR matrix
 * (already reordered / dropped by the host stage, every entry within half-bandwidth k) is assembled into
 * band storage ON THE DEVICE and set up like sap_setup_banded; entries outside the band are the
 * reference's std::invalid_argument ("assemble_banded: entry (i, j) outside half-bandwidth k").
 * csr_on_device: 0 host pointers, 1 device pointers. Replaces solve_sparse's assemble + setup
 * (pipeline.hpp:286-330); the Krylov operator stays the banded one until sap_set_operator_csr. */
sap_status sap_setup_banded_from_csr(sap_handle* h, int n, int k, int nnz, const int* row_ptr, const int* col_idx,
                                     const double* values, int csr_on_device);
/* drop_off (pipeline.hpp:59-99) + assemble_banded + setup, on the device (solve_sparse's
 * pipeline.hpp:265-330 after the host reorderings): k_after = the smallest half-bandwidth whose
 * dropped outside-band mass satisfies ||dropped||_F <= drop_tol ||A||_F (drop_tol = 0: half_bandwidth(A),
 * nothing dropped), entries beyond it dropped, the band assembled at k_after and set up. The squared
 * masses are summed in the reference's order, so k_after is the reference's. drop_tol outside [0, 1]
 * -> SAP_ERR_INVALID_ARGUMENT ("drop_off: tolerance must lie in [0, 1]"). k_after may be NULL. */
sap_status sap_setup_from_csr_drop(sap_handle* h, int n, int nnz, const int* row_ptr, const int* col_idx,
                                   const double* values, double drop_tol, int csr_on_device, int* k_after);
/* ---- A operator override: CSR matrix (solve_sparse's apply_a, pipeline.hpp:336-338).
 * row_ptr[n+1], col_idx[nnz], values[nnz]; copied. Which call wins: every setup (sap_setup_banded,
 * sap_setup_banded_from_csr, sap_setup_from_csr_drop) resets the operator to the band it set up; a
 * sap_set_operator_csr AFTER the setup makes the CSR matrix the operator until the next setup
 * (solve_sparse's order: setup, then the solve over the unreduced CSR matrix). */
sap_status sap_set_operator_csr(sap_handle* h, int n, int nnz, const int* row_ptr, const int* col_idx,
                                const double* values, int on_device);

/* ---- the two LinearOps (krylov.hpp:14): out = M^{-1} in, out = A in. length n. ---- */
sap_status sap_apply_preconditioner(sap_handle* h, const double* in, double* out, int on_device);
sap_status sap_apply_operator(sap_handle* h, const double* in, double* out, int on_device);

/* ---- solve ≙ run_krylov(A, M, b, x, KrylovOptions): x0 = 0, true-residual
 * convergence ||b - A x|| <= rel_tol ||b|| + abs_tol, quarter-iteration accounting. */
sap_status sap_solve(sap_handle* h, const double* b, double* x, int on_device, sap_solve_stats* stats);

sap_status sap_get_report(const sap_handle* h, sap_report* rep);

/* ---- parity accessors (BlockFactors / SpikeSet contents) ----
 * which = 0: LU, 1: UL (SaP-C only). out: sizes[part]*(2k+1) doubles in the
 * reference's per-block band layout. boosts / block_norm may be NULL. */
sap_status sap_get_factor(sap_handle* h, int part, int which, double* out, int* boosts, double* block_norm);
/* Interface t in [0, p-1): w = k (third stage: w_t). Any output pointer may be NULL. */
sap_status sap_get_spike(sap_handle* h, int iface, double* b_block, double* c_block, double* v_bottom,
                         double* w_top, double* rbar, int* rbar_boosts);

/* ---- third stage: per-block reordering (PipelineConfig::third_stage, pipeline.hpp:312-319) ----
 * Arms every following sap_setup_banded / sap_setup_banded_from_csr of a coupled or decoupled
 * preconditioner with sap::third_stage's result (ThirdStageResult, reorder_cm.hpp:227-231), computed
 * on the host by the caller: block_k[p] the per-partition half-bandwidths (each in [0, k]; p must equal
 * the setup's partition count), has_perm[p] (NULL = no permutations) and perm[n]: for a block b with
 * has_perm[b], perm[offsets[b] + r] is the position of block row r in the reordered block. The setup
 * then factors P_b A_b P_b^T at K_b (LU only; block_factors.hpp:138-206), extracts the couplings at
 * w_t = max(K_t, K_{t+1}) (spike.hpp:95-116) and solves full spikes (compute_full_spikes,
 * spike.hpp:258-296); every block solve permutes (block_solve, block_factors.hpp:210-236).
 * Errors: a nonzero entry pushed outside K_b -> SAP_ERR_INVALID_ARGUMENT ("factor_blocks: block
 * permutation exceeds bandwidth K_b"); a non-finite spike -> SAP_ERR_PRECONDITIONER.
 * block_k == NULL disarms. Single-GPU handles only. sap_get_factor then returns block b at its own
 * bandwidth (m_b*(2K_b+1) doubles) and sap_get_spike w_t x w_t blocks. */
sap_status sap_set_third_stage(sap_handle* h, int p, const int* block_k, const int* has_perm, const int* perm, int n);
/* SpikeSet::v_full / w_full of interface t (third stage, coupled): V_t (sizes[t] x w_t) and W_t
 * (sizes[t+1] x w_t), column-major in the original row order, as compute_full_spikes stores them.
 * Either pointer may be NULL. */
sap_status sap_get_full_spike(sap_handle* h, int iface, double* v_full, double* w_full);

/* ---- multi-GPU (one process per GPU) ----
 * Communication is supplied by the caller (NCCL through torch.distributed on a
 * node, or any other transport). Each rank owns a contiguous range of whole
 * partitions, [offsets[pb], offsets[pe]) of make_partition_layout(n, opts.p, k).
 * Factorization is rank-local. At setup the neighbours swap the one spike tip
 * of each rank-crossing interface they cannot compute (V^b of the left rank's
 * last block, W^t of the right rank's first block; w*w doubles each way), and
 * both ranks build and factor that interface's reduced block. Every
 * preconditioner apply then makes ONE neighbour exchange of w = k rows of
 * D^{-1} r each way, every operator apply one exchange of the k-row x halo, and
 * every Krylov reduction is a host allreduce. Callbacks are invoked with the
 * handle's stream synchronized and must complete the transfer before returning.
 * The preconditioner kinds distributed are coupled, decoupled and none. */
typedef struct sap_comm {
    void* ctx;
    int rank, world;
    /* in-place sum over all ranks of `count` doubles in HOST memory; 0 = ok */
    int (*allreduce_sum)(void* ctx, double* host, int count);
    /* neighbour exchange of DEVICE buffers: send_left[n_sl] -> rank-1, send_right[n_sr] -> rank+1,
     * recv_left[n_rl] <- rank-1, recv_right[n_rr] <- rank+1 (any count may be 0); 0 = ok */
    int (*exchange)(void* ctx, const double* send_left, int n_sl, const double* send_right, int n_sr,
                    double* recv_left, int n_rl, double* recv_right, int n_rr);
} sap_comm;

/* Native NCCL data plane (one process per GPU): the library opens libnccl.so.2 itself and runs every
 * neighbour exchange (spike tips at setup, interface rows per preconditioner apply, the k-row operator
 * halo) as grouped ncclSend / ncclRecv on the handle's stream and every Krylov dot as an ncclAllReduce on
 * the device scalar -- no callbacks, no host staging, no stream synchronisation per exchange.
 * Rank 0 calls sap_nccl_get_unique_id; the 128 id bytes reach every rank out of band (torch.distributed,
 * MPI, a file); then every rank calls sap_create_distributed_nccl (collective) with its CUDA device in
 * opts->device. Setup / apply / solve are the same calls as for sap_create_distributed. */
sap_status sap_nccl_get_unique_id(unsigned char id[128]);
sap_status sap_create_distributed_nccl(const sap_options* opts, const unsigned char id[128], int rank, int world,
                                       sap_handle** out);

/* Rank r's row range under the SURVEY §8e assignment: partitions
 * [r*p/world, (r+1)*p/world) of make_partition_layout(n, p, k). */
sap_status sap_rank_rows(int n, int p, int k, int rank, int world, int* row_lo, int* row_hi);
sap_status sap_create_distributed(const sap_options* opts, const sap_comm* comm, sap_handle** out);
/* band_slice: the GLOBAL band's columns [max(0, row_lo-k), min(n, row_hi+k)) (tall-thin layout,
 * (2k+1) doubles per column). Afterwards apply / operator / solve take the rank's local vectors
 * (length row_hi - row_lo). Collective: every rank must call it. */
sap_status sap_setup_banded_dist(sap_handle* h, int n, int k, int row_lo, int row_hi, const double* band_slice,
                                 int on_device);

#ifdef __cplusplus
}
#endif
#endif /* SAP_GPU_H */
