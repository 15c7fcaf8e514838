// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference headers (compiled in place from
// /root/reference/proj/include by oracle/Makefile; no reference source is
// copied into this repository). The product library (libsap_gpu.so) never
// loads this; tests/, __graft_entry__.smoke() and bench.py's reference /
// cpu_baseline legs do, as the checker and as the CPU baseline.
//
// Every entry point wires the reference's own public functions exactly as
// the reference does:
//   * sapref_random_banded  : testsup::random_banded (proj/tests/test_support.hpp:133-150)
//                             followed by random_rhs (proj/tests/acceptance.cpp:48-53)
//   * sapref_factor_blocks  : sap::factor_blocks (proj/include/sap/block_factors.hpp:138-206)
//   * sapref_spikes         : extract_coupling + compute_spike_tips
//                             (proj/include/sap/spike.hpp:95-116, :178-254)
//   * sapref_apply          : apply_preconditioner (proj/include/sap/spike.hpp:304-351)
//   * sapref_solve_banded   : detail::build_precond_op + run_krylov with the banded
//                             operator (proj/include/sap/pipeline.hpp:140-202,
//                             proj/include/sap/krylov.hpp:434-442), the dense wiring of
//                             proj/tests/acceptance.cpp:114-132.
//   * sapref_solve_sparse   : sap::solve_sparse (proj/include/sap/pipeline.hpp:213-369).
//   * sapref_*_f32          : the same factor_blocks / extract_coupling + compute_spike_tips /
//                             apply_preconditioner at T = float on banded_cast<float> of the band:
//                             build_precond_op<float>'s preconditioner (proj/include/sap/pipeline.hpp:140-202,
//                             banded_matrix.hpp:129-136), outputs widened to double.
//   * sapref_third_*        : the third stage - sap::third_stage (proj/include/sap/reorder_cm.hpp:233-274),
//                             factor_blocks with block permutations and per-partition bandwidths,
//                             compute_full_spikes (spike.hpp:258-296), apply_preconditioner and
//                             build_precond_op(third_active = true) + run_krylov.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "sap/sap.hpp"
#include "test_support.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

// 1 = std::invalid_argument, 2 = PreconditionerError, 3 = StructuralSingularityError, 9 = other
#define SAPREF_TRY try {
#define SAPREF_CATCH                                                           \
    }                                                                          \
    catch (const std::invalid_argument& e) { return fail(1, e.what()); }       \
    catch (const sap::PreconditionerError& e) { return fail(2, e.what()); }    \
    catch (const sap::StructuralSingularityError& e) { return fail(3, e.what()); } \
    catch (const std::exception& e) { return fail(9, e.what()); }              \
    return 0;

sap::BandedMatrix<double> wrap_band(int n, int k, const double* band) {
    sap::BandedMatrix<double> a(n, k);
    std::memcpy(a.storage().data(), band, sizeof(double) * static_cast<std::size_t>(n) * (2 * k + 1));
    return a;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

sap::PartitionLayout ts_layout(int n, int p, int k, const int* block_k) {
    sap::PartitionLayout l = sap::make_partition_layout(n, p, k);
    l.per_partition_k.assign(block_k, block_k + p);
    return l;
}

// block_perms as sap::third_stage returns them: empty vector = identity
std::vector<std::vector<int>> ts_perms(const sap::PartitionLayout& l, const int* has_perm, const int* perm) {
    std::vector<std::vector<int>> out(static_cast<std::size_t>(l.p));
    for (int b = 0; b < l.p; ++b)
        if (has_perm && has_perm[b]) out[static_cast<std::size_t>(b)].assign(perm + l.offset(b), perm + l.offset(b) + l.size(b));
    return out;
}

}  // namespace

extern "C" {

const char* sapref_last_error() { return g_err.c_str(); }

int sapref_random_banded(int n, int k, double d, unsigned seed, double* band_out, double* rhs_out) {
    SAPREF_TRY
    std::mt19937 rng(seed);
    const sap::BandedMatrix<double> a = testsup::random_banded(n, k, d, rng);
    std::memcpy(band_out, a.storage().data(), sizeof(double) * a.storage().size());
    if (rhs_out) {
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (int i = 0; i < n; ++i) rhs_out[i] = u(rng);
    }
    SAPREF_CATCH
}

int sapref_partition_layout(int n, int p, int k, int* sizes, int* offsets) {
    SAPREF_TRY
    const sap::PartitionLayout l = sap::make_partition_layout(n, p, k);
    for (int i = 0; i < p; ++i) sizes[i] = l.sizes[static_cast<std::size_t>(i)];
    for (int i = 0; i <= p; ++i) offsets[i] = l.offsets[static_cast<std::size_t>(i)];
    SAPREF_CATCH
}

int sapref_band_matvec(int n, int k, const double* band, const double* x, double* y) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    a.matvec(std::span<const double>(x, static_cast<std::size_t>(n)), std::span<double>(y, static_cast<std::size_t>(n)));
    SAPREF_CATCH
}

// lu_out / ul_out: per-block bands concatenated in partition order
// (block b occupies sizes[b]*(2k+1) doubles). ul_out may be null for lu_only.
int sapref_factor_blocks(int n, int k, const double* band, int p, int lu_and_ul, double boost_eps,
                         double* lu_out, double* ul_out, int* boosts, int* boosts_ul, double* norms) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    const auto f = sap::factor_blocks<double>(
        a, layout, lu_and_ul ? sap::FactorMode::lu_and_ul : sap::FactorMode::lu_only, boost_eps);
    std::size_t off = 0;
    for (int b = 0; b < p; ++b) {
        const auto& lu = f.lu[static_cast<std::size_t>(b)];
        std::memcpy(lu_out + off, lu.data(), sizeof(double) * lu.size());
        if (lu_and_ul && ul_out) std::memcpy(ul_out + off, f.ul[static_cast<std::size_t>(b)].data(), sizeof(double) * lu.size());
        off += lu.size();
        boosts[b] = f.boost_count[static_cast<std::size_t>(b)];
        if (boosts_ul) boosts_ul[b] = f.boost_count_ul[static_cast<std::size_t>(b)];
        if (norms) norms[b] = f.block_norm[static_cast<std::size_t>(b)];
    }
    SAPREF_CATCH
}

// Coupling corners and spike tips for every interface (uniform width w = k).
// Each output holds (p-1) row-major w x w blocks back to back.
int sapref_spikes(int n, int k, const double* band, int p, double boost_eps, double* b_out, double* c_out,
                  double* vb_out, double* wt_out, double* rbar_out, int* rbar_boosts) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    const auto f = sap::factor_blocks<double>(a, layout, sap::FactorMode::lu_and_ul, boost_eps);
    const auto cb = sap::extract_coupling<double>(a, layout);
    const auto s = sap::compute_spike_tips<double>(f, cb);
    std::size_t off = 0;
    for (int t = 0; t < s.interfaces(); ++t) {
        const std::size_t ww = s.v_bottom[static_cast<std::size_t>(t)].size();
        std::memcpy(b_out + off, cb.b_blocks[static_cast<std::size_t>(t)].data(), sizeof(double) * ww);
        std::memcpy(c_out + off, cb.c_blocks[static_cast<std::size_t>(t)].data(), sizeof(double) * ww);
        std::memcpy(vb_out + off, s.v_bottom[static_cast<std::size_t>(t)].data(), sizeof(double) * ww);
        std::memcpy(wt_out + off, s.w_top[static_cast<std::size_t>(t)].data(), sizeof(double) * ww);
        std::memcpy(rbar_out + off, s.rbar[static_cast<std::size_t>(t)].data(), sizeof(double) * ww);
        rbar_boosts[t] = s.rbar_boosts[static_cast<std::size_t>(t)];
        off += ww;
    }
    SAPREF_CATCH
}

// kind: 0 coupled, 1 decoupled (sap::PrecondKind order).
int sapref_apply(int n, int k, const double* band, int p, int kind, double boost_eps, const double* in,
                 double* out) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    const bool coupled = kind == 0 && p > 1;
    const auto f = sap::factor_blocks<double>(
        a, layout, coupled ? sap::FactorMode::lu_and_ul : sap::FactorMode::lu_only, boost_eps);
    sap::SpikeSet<double> s;
    if (coupled) s = sap::compute_spike_tips<double>(f, sap::extract_coupling<double>(a, layout));
    const auto r = sap::apply_preconditioner<double>(static_cast<sap::PrecondKind>(kind), f, s,
                                                     std::span<const double>(in, static_cast<std::size_t>(n)));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    SAPREF_CATCH
}

// ---- T = float (mixed_precision): build_precond_op<float>'s pieces on banded_cast<float>(band) ----
int sapref_factor_blocks_f32(int n, int k, const double* band, int p, int lu_and_ul, double boost_eps,
                             double* lu_out, double* ul_out, int* boosts, int* boosts_ul, double* norms) {
    SAPREF_TRY
    const auto a = sap::banded_cast<float>(wrap_band(n, k, band));
    const auto layout = sap::make_partition_layout(n, p, k);
    const auto f = sap::factor_blocks<float>(
        a, layout, lu_and_ul ? sap::FactorMode::lu_and_ul : sap::FactorMode::lu_only, boost_eps);
    std::size_t off = 0;
    for (int b = 0; b < p; ++b) {
        const auto& lu = f.lu[static_cast<std::size_t>(b)];
        for (std::size_t i = 0; i < lu.size(); ++i) lu_out[off + i] = lu[i];
        if (lu_and_ul && ul_out)
            for (std::size_t i = 0; i < lu.size(); ++i) ul_out[off + i] = f.ul[static_cast<std::size_t>(b)][i];
        off += lu.size();
        boosts[b] = f.boost_count[static_cast<std::size_t>(b)];
        if (boosts_ul) boosts_ul[b] = f.boost_count_ul[static_cast<std::size_t>(b)];
        if (norms) norms[b] = f.block_norm[static_cast<std::size_t>(b)];
    }
    SAPREF_CATCH
}

int sapref_spikes_f32(int n, int k, const double* band, int p, double boost_eps, double* b_out, double* c_out,
                      double* vb_out, double* wt_out, double* rbar_out, int* rbar_boosts) {
    SAPREF_TRY
    const auto a = sap::banded_cast<float>(wrap_band(n, k, band));
    const auto layout = sap::make_partition_layout(n, p, k);
    const auto f = sap::factor_blocks<float>(a, layout, sap::FactorMode::lu_and_ul, boost_eps);
    const auto cb = sap::extract_coupling<float>(a, layout);
    const auto s = sap::compute_spike_tips<float>(f, cb);
    std::size_t off = 0;
    auto widen = [](double* dst, const std::vector<float>& v) {
        for (std::size_t i = 0; i < v.size(); ++i) dst[i] = v[i];
    };
    for (int t = 0; t < s.interfaces(); ++t) {
        const std::size_t ww = s.v_bottom[static_cast<std::size_t>(t)].size();
        widen(b_out + off, cb.b_blocks[static_cast<std::size_t>(t)]);
        widen(c_out + off, cb.c_blocks[static_cast<std::size_t>(t)]);
        widen(vb_out + off, s.v_bottom[static_cast<std::size_t>(t)]);
        widen(wt_out + off, s.w_top[static_cast<std::size_t>(t)]);
        widen(rbar_out + off, s.rbar[static_cast<std::size_t>(t)]);
        rbar_boosts[t] = s.rbar_boosts[static_cast<std::size_t>(t)];
        off += ww;
    }
    SAPREF_CATCH
}

// M r through build_precond_op<float>'s closure: r cast to float, apply_preconditioner<float>, widened back
int sapref_apply_f32(int n, int k, const double* band, int p, int kind, double boost_eps, const double* in,
                     double* out) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    sap::PipelineConfig cfg;
    cfg.precond = static_cast<sap::PrecondKind>(kind);
    cfg.boost_eps = boost_eps;
    sap::PipelineReport rep;
    const sap::LinearOp op = sap::detail::build_precond_op<float>(a, layout, cfg, false, nullptr, rep);
    op(std::span<const double>(in, static_cast<std::size_t>(n)), std::span<double>(out, static_cast<std::size_t>(n)));
    SAPREF_CATCH
}

// Dense-banded SaP solve through the reference's own setup (build_precond_op)
// and solve (run_krylov) entry points, A = BandedMatrix::matvec.
// timings[0..4] = t_lu, t_bc, t_spk, t_lurdcd, t_kry (seconds).
int sapref_solve_banded(int n, int k, const double* band, const double* rhs, int p, int kind,
                        double boost_eps, int ell, double rel_tol, double abs_tol, int max_iterations,
                        int mixed_precision, double* x_out, double* iterations, int* converged,
                        double* final_res, int* failure, double* history, int hist_cap, int* hist_len,
                        double* timings) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    sap::PipelineConfig cfg;
    cfg.p = p;
    cfg.precond = static_cast<sap::PrecondKind>(kind);
    cfg.boost_eps = boost_eps;
    cfg.krylov.ell = ell;
    cfg.krylov.rel_tol = rel_tol;
    cfg.krylov.abs_tol = abs_tol;
    cfg.krylov.max_iterations = max_iterations;
    cfg.krylov.mixed_precision = mixed_precision != 0;
    sap::PipelineReport rep;
    sap::LinearOp op_m;
    try {
        op_m = mixed_precision ? sap::detail::build_precond_op<float>(a, layout, cfg, false, nullptr, rep)
                               : sap::detail::build_precond_op<double>(a, layout, cfg, false, nullptr, rep);
    } catch (...) {
        if (timings) {
            timings[0] = rep.t_lu; timings[1] = rep.t_bc; timings[2] = rep.t_spk; timings[3] = rep.t_lurdcd; timings[4] = 0;
        }
        throw;
    }
    sap::LinearOp op_a = [&a](std::span<const double> in, std::span<double> out) { a.matvec(in, out); };
    std::vector<double> x(static_cast<std::size_t>(n), 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    const sap::SolveStats st = sap::run_krylov(op_a, op_m, std::span<const double>(rhs, static_cast<std::size_t>(n)), x, cfg.krylov);
    const double t_kry = seconds_since(t0);
    std::memcpy(x_out, x.data(), sizeof(double) * x.size());
    *iterations = st.iterations;
    *converged = st.converged ? 1 : 0;
    *final_res = st.final_relative_residual;
    *failure = static_cast<int>(st.failure);
    const int hl = static_cast<int>(st.residual_history.size());
    *hist_len = hl;
    for (int i = 0; i < hl && i < hist_cap; ++i) history[i] = st.residual_history[static_cast<std::size_t>(i)];
    if (timings) {
        timings[0] = rep.t_lu; timings[1] = rep.t_bc; timings[2] = rep.t_spk; timings[3] = rep.t_lurdcd; timings[4] = t_kry;
    }
    SAPREF_CATCH
}

// Krylov on an explicit CSR operator with the identity preconditioner
// (proj/tests/test_krylov.cpp style): exercises solve_krylov alone.
int sapref_krylov_csr_identity(int n, const int* row_ptr, const int* col_idx, const double* vals,
                               const double* rhs, int ell, double rel_tol, int max_iterations,
                               double* x_out, double* iterations, int* converged, double* final_res,
                               int* failure, double* history, int hist_cap, int* hist_len) {
    SAPREF_TRY
    sap::SparseMatrix m;
    m.n = n;
    m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    m.col_idx.assign(col_idx, col_idx + row_ptr[n]);
    m.values.assign(vals, vals + row_ptr[n]);
    sap::LinearOp op_a = [&m](std::span<const double> in, std::span<double> out) { m.matvec(in, out); };
    sap::LinearOp op_m = [](std::span<const double> in, std::span<double> out) {
        std::copy(in.begin(), in.end(), out.begin());
    };
    sap::KrylovOptions ko;
    ko.ell = ell;
    ko.rel_tol = rel_tol;
    ko.max_iterations = max_iterations;
    std::vector<double> x(static_cast<std::size_t>(n), 0.0);
    const auto st = sap::solve_krylov(op_a, op_m, std::span<const double>(rhs, static_cast<std::size_t>(n)), x, ko);
    std::memcpy(x_out, x.data(), sizeof(double) * x.size());
    *iterations = st.iterations;
    *converged = st.converged ? 1 : 0;
    *final_res = st.final_relative_residual;
    *failure = static_cast<int>(st.failure);
    const int hl = static_cast<int>(st.residual_history.size());
    *hist_len = hl;
    for (int i = 0; i < hl && i < hist_cap; ++i) history[i] = st.residual_history[static_cast<std::size_t>(i)];
    SAPREF_CATCH
}

// End-to-end sparse pipeline (config 4). report[0..9] = t_db, t_cm, t_drop,
// t_asmbl, t_bc, t_lu, t_spk, t_lurdcd, t_kry, k_after; stats as above.
int sapref_solve_sparse(int n, const int* row_ptr, const int* col_idx, const double* vals, const double* rhs,
                        int use_db, int db_scaling, int use_cm, int third_stage, int p, double drop_tol,
                        int kind, double boost_eps, unsigned seed, int ell, double rel_tol, int max_iterations,
                        int mixed_precision, double* x_out, double* report, double* iterations,
                        int* converged, double* final_res, int* failure) {
    SAPREF_TRY
    sap::SparseMatrix m;
    m.n = n;
    m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    m.col_idx.assign(col_idx, col_idx + row_ptr[n]);
    m.values.assign(vals, vals + row_ptr[n]);
    sap::PipelineConfig cfg;
    cfg.use_db = use_db != 0;
    cfg.db_scaling = db_scaling != 0;
    cfg.use_cm = use_cm != 0;
    cfg.third_stage = third_stage != 0;
    cfg.p = p;
    cfg.drop_tol = drop_tol;
    cfg.precond = static_cast<sap::PrecondKind>(kind);
    cfg.boost_eps = boost_eps;
    cfg.seed = seed;
    cfg.krylov.ell = ell;
    cfg.krylov.rel_tol = rel_tol;
    cfg.krylov.max_iterations = max_iterations;
    cfg.krylov.mixed_precision = mixed_precision != 0;
    sap::PipelineReport rep;
    const auto x = sap::solve_sparse(m, std::span<const double>(rhs, static_cast<std::size_t>(n)), cfg, rep);
    std::memcpy(x_out, x.data(), sizeof(double) * x.size());
    report[0] = rep.t_db; report[1] = rep.t_cm; report[2] = rep.t_drop; report[3] = rep.t_asmbl;
    report[4] = rep.t_bc; report[5] = rep.t_lu; report[6] = rep.t_spk; report[7] = rep.t_lurdcd;
    report[8] = rep.t_kry; report[9] = rep.k;
    *iterations = rep.stats.iterations;
    *converged = rep.stats.converged ? 1 : 0;
    *final_res = rep.stats.final_relative_residual;
    *failure = static_cast<int>(rep.stats.failure);
    if (!rep.success && !rep.failure_stage.empty()) g_err = rep.failure_stage + ": " + rep.failure_message;
    SAPREF_CATCH
}

// solve_sparse's host stage (pipeline.hpp:228-266): db_reorder (+ row/column scaling) and cm_reorder with the
// matching right-hand-side permutations, exactly as solve_sparse runs them. Outputs the reordered matrix
// (same nnz: row_ptr[n+1], col_idx, values), the reordered rhs, the CM permutation (identity when off) and
// the column scaling (ones when off) that map the solution back, and the stage times.
// timings[0] = t_db, [1] = t_cm (seconds).
int sapref_host_stage(int n, const int* row_ptr, const int* col_idx, const double* vals, const double* rhs,
                      int use_db, int db_scaling, int use_cm, unsigned seed, int* out_rp, int* out_ci,
                      double* out_v, double* out_rhs, int* cm_perm, double* col_scale, double* timings) {
    SAPREF_TRY
    sap::SparseMatrix work;
    work.n = n;
    work.row_ptr.assign(row_ptr, row_ptr + n + 1);
    work.col_idx.assign(col_idx, col_idx + row_ptr[n]);
    work.values.assign(vals, vals + row_ptr[n]);
    std::vector<double> r(rhs, rhs + n);
    for (int i = 0; i < n; ++i) {
        cm_perm[i] = i;
        col_scale[i] = 1.0;
    }
    timings[0] = timings[1] = 0.0;
    if (use_db) {
        const auto t0 = std::chrono::steady_clock::now();
        sap::DbResult db = sap::db_reorder(work, db_scaling != 0);
        if (db.scaled) {
            work = sap::scale_rows_cols(work, db.row_scale, db.col_scale);
            for (int i = 0; i < n; ++i) r[static_cast<std::size_t>(i)] *= db.row_scale[static_cast<std::size_t>(i)];
            for (int i = 0; i < n; ++i) col_scale[i] = db.col_scale[static_cast<std::size_t>(i)];
        }
        work = sap::permute_rows(work, db.perm);
        std::vector<double> pr(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) pr[static_cast<std::size_t>(db.perm[static_cast<std::size_t>(i)])] = r[static_cast<std::size_t>(i)];
        r = std::move(pr);
        timings[0] = seconds_since(t0);
    }
    if (use_cm) {
        const auto t0 = std::chrono::steady_clock::now();
        const sap::AdjGraph g = sap::build_graph(work);
        sap::CmResult cm = sap::cm_reorder(g, seed);
        work = sap::permute_symmetric(work, cm.perm);
        std::vector<double> pr(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) pr[static_cast<std::size_t>(cm.perm[static_cast<std::size_t>(i)])] = r[static_cast<std::size_t>(i)];
        r = std::move(pr);
        for (int i = 0; i < n; ++i) cm_perm[i] = cm.perm[static_cast<std::size_t>(i)];
        timings[1] = seconds_since(t0);
    }
    std::memcpy(out_rp, work.row_ptr.data(), sizeof(int) * (n + 1));
    std::memcpy(out_ci, work.col_idx.data(), sizeof(int) * work.col_idx.size());
    std::memcpy(out_v, work.values.data(), sizeof(double) * work.values.size());
    std::memcpy(out_rhs, r.data(), sizeof(double) * n);
    SAPREF_CATCH
}

// sap::drop_off (pipeline.hpp:59-99): the kept half-bandwidth and the kept entry count.
int sapref_drop_off(int n, const int* row_ptr, const int* col_idx, const double* vals, double tol, int* k_after,
                    int* nnz_after) {
    SAPREF_TRY
    sap::SparseMatrix m;
    m.n = n;
    m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    m.col_idx.assign(col_idx, col_idx + row_ptr[n]);
    m.values.assign(vals, vals + row_ptr[n]);
    const sap::DropResult r = sap::drop_off(m, tol);
    *k_after = r.k_after;
    *nnz_after = static_cast<int>(r.matrix.values.size());
    SAPREF_CATCH
}

// sap::third_stage: block_k[p], has_perm[p], perm[n] (perm[offset(b) + r] = new position of block row r).
int sapref_third_stage(int n, int k, const double* band, int p, unsigned seed, int* block_k, int* has_perm,
                       int* perm) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = sap::make_partition_layout(n, p, k);
    const sap::ThirdStageResult ts = sap::third_stage(a, layout, seed);
    for (int b = 0; b < p; ++b) {
        block_k[b] = ts.block_k[static_cast<std::size_t>(b)];
        const auto& pm = ts.block_perms[static_cast<std::size_t>(b)];
        has_perm[b] = pm.empty() ? 0 : 1;
        for (int r = 0; r < layout.size(b); ++r) perm[layout.offset(b) + r] = pm.empty() ? r : pm[static_cast<std::size_t>(r)];
    }
    SAPREF_CATCH
}

// Third-stage setup: factor_blocks (LU only, perms, K_b) + extract_coupling + compute_full_spikes.
// lu_out: blocks at their own bandwidth back to back (m_b*(2K_b+1)); b/c/vb/wt/rbar: w_t x w_t per
// interface back to back; vfull/wfull: m_t x w_t and m_{t+1} x w_t column-major back to back. Any
// spike output may be null (coupled = 0 skips the spikes).
int sapref_third_setup(int n, int k, const double* band, int p, const int* block_k, const int* has_perm,
                       const int* perm, double boost_eps, int coupled, double* lu_out, int* boosts, double* norms,
                       double* b_out, double* c_out, double* vb_out, double* wt_out, double* rbar_out,
                       int* rbar_boosts, double* vfull_out, double* wfull_out) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = ts_layout(n, p, k, block_k);
    const auto perms = ts_perms(layout, has_perm, perm);
    const auto f = sap::factor_blocks<double>(a, layout, sap::FactorMode::lu_only, boost_eps, &perms);
    std::size_t off = 0;
    for (int b = 0; b < p; ++b) {
        const auto& lu = f.lu[static_cast<std::size_t>(b)];
        if (lu_out) std::memcpy(lu_out + off, lu.data(), sizeof(double) * lu.size());
        off += lu.size();
        if (boosts) boosts[b] = f.boost_count[static_cast<std::size_t>(b)];
        if (norms) norms[b] = f.block_norm[static_cast<std::size_t>(b)];
    }
    if (!coupled || p < 2) return 0;
    const auto cb = sap::extract_coupling<double>(a, layout);
    const auto s = sap::compute_full_spikes<double>(f, cb);
    std::size_t o2 = 0, ov = 0, ow = 0;
    for (int t = 0; t < s.interfaces(); ++t) {
        const auto T = static_cast<std::size_t>(t);
        const std::size_t ww = s.v_bottom[T].size();
        if (b_out) std::memcpy(b_out + o2, cb.b_blocks[T].data(), sizeof(double) * ww);
        if (c_out) std::memcpy(c_out + o2, cb.c_blocks[T].data(), sizeof(double) * ww);
        if (vb_out) std::memcpy(vb_out + o2, s.v_bottom[T].data(), sizeof(double) * ww);
        if (wt_out) std::memcpy(wt_out + o2, s.w_top[T].data(), sizeof(double) * ww);
        if (rbar_out) std::memcpy(rbar_out + o2, s.rbar[T].data(), sizeof(double) * ww);
        if (rbar_boosts) rbar_boosts[t] = s.rbar_boosts[T];
        if (vfull_out) std::memcpy(vfull_out + ov, s.v_full[T].data(), sizeof(double) * s.v_full[T].size());
        if (wfull_out) std::memcpy(wfull_out + ow, s.w_full[T].data(), sizeof(double) * s.w_full[T].size());
        o2 += ww;
        ov += s.v_full[T].size();
        ow += s.w_full[T].size();
    }
    SAPREF_CATCH
}

// apply_preconditioner over third-stage factors; kind 0 coupled, 1 decoupled.
int sapref_third_apply(int n, int k, const double* band, int p, const int* block_k, const int* has_perm,
                       const int* perm, int kind, double boost_eps, const double* in, double* out) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = ts_layout(n, p, k, block_k);
    const auto perms = ts_perms(layout, has_perm, perm);
    const auto f = sap::factor_blocks<double>(a, layout, sap::FactorMode::lu_only, boost_eps, &perms);
    sap::SpikeSet<double> s;
    if (kind == 0 && p > 1) s = sap::compute_full_spikes<double>(f, sap::extract_coupling<double>(a, layout));
    const auto r = sap::apply_preconditioner<double>(static_cast<sap::PrecondKind>(kind), f, s,
                                                     std::span<const double>(in, static_cast<std::size_t>(n)));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    SAPREF_CATCH
}

// build_precond_op(third_active = true, block_perms) + run_krylov, A = BandedMatrix::matvec.
int sapref_third_solve_banded(int n, int k, const double* band, const double* rhs, int p, const int* block_k,
                              const int* has_perm, const int* perm, int kind, double boost_eps, int ell,
                              double rel_tol, int max_iterations, int mixed_precision, double* x_out,
                              double* iterations, int* converged, double* final_res, int* failure) {
    SAPREF_TRY
    const auto a = wrap_band(n, k, band);
    const auto layout = ts_layout(n, p, k, block_k);
    const auto perms = ts_perms(layout, has_perm, perm);
    sap::PipelineConfig cfg;
    cfg.p = p;
    cfg.precond = static_cast<sap::PrecondKind>(kind);
    cfg.boost_eps = boost_eps;
    cfg.krylov.ell = ell;
    cfg.krylov.rel_tol = rel_tol;
    cfg.krylov.max_iterations = max_iterations;
    cfg.krylov.mixed_precision = mixed_precision != 0;
    sap::PipelineReport rep;
    const sap::LinearOp op_m = mixed_precision
                                   ? sap::detail::build_precond_op<float>(a, layout, cfg, true, &perms, rep)
                                   : sap::detail::build_precond_op<double>(a, layout, cfg, true, &perms, rep);
    sap::LinearOp op_a = [&a](std::span<const double> in, std::span<double> out) { a.matvec(in, out); };
    std::vector<double> x(static_cast<std::size_t>(n), 0.0);
    const sap::SolveStats st = sap::run_krylov(op_a, op_m, std::span<const double>(rhs, static_cast<std::size_t>(n)), x, cfg.krylov);
    std::memcpy(x_out, x.data(), sizeof(double) * x.size());
    *iterations = st.iterations;
    *converged = st.converged ? 1 : 0;
    *final_res = st.final_relative_residual;
    *failure = static_cast<int>(st.failure);
    SAPREF_CATCH
}

}  // extern "C"
