// sap_gpu.hpp — header-only C++ adaptor over the C ABI (sap_gpu.h) that drops
// the GPU path into the reference's own C++ interfaces:
//
//   sap::LinearOp          proj/include/sap/krylov.hpp:14
//   sap::detail::build_precond_op<T>  proj/include/sap/pipeline.hpp:140-202
//   sap::run_krylov        proj/include/sap/krylov.hpp:434-442
//
// It depends only on <functional>/<span>/<stdexcept> and sap_gpu.h; the
// reference's headers are NOT required. Errors are rethrown as the
// reference's exception types when the including translation unit defines
// SAP_GPU_REFERENCE_ERRORS after including "sap/errors.hpp".
#pragma once

#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sap_gpu.h"

namespace sap::gpu {

// Same signature as sap::LinearOp.
using LinearOp = std::function<void(std::span<const double>, std::span<double>)>;

[[noreturn]] inline void throw_status(sap_status s) {
    const std::string msg = sap_last_error();
#ifdef SAP_GPU_REFERENCE_ERRORS
    if (s == SAP_ERR_PRECONDITIONER) throw sap::PreconditionerError(msg);
#endif
    if (s == SAP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(std::string(sap_status_string(s)) + ": " + msg);
}

inline void check(sap_status s) {
    if (s != SAP_OK) throw_status(s);
}

// One handle = one factorization (the reference's PrecondState) + operators.
class Solver {
public:
    explicit Solver(const sap_options& o) { check(sap_create(&o, &h_)); }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;
    ~Solver() { sap_destroy(h_); }

    // setup ≙ build_precond_op over make_partition_layout(n, opts.p, k); band is
    // the reference BandedMatrix<double>::storage() (host memory).
    void setup(int n, int k, std::span<const double> band) { check(sap_setup_banded(h_, n, k, band.data(), 0)); n_ = n; }
    void set_operator_csr(int n, std::span<const int> rp, std::span<const int> ci, std::span<const double> v) {
        check(sap_set_operator_csr(h_, n, static_cast<int>(ci.size()), rp.data(), ci.data(), v.data(), 0));
    }

    // The two LinearOps; capture the handle by pointer (the Solver must outlive them).
    LinearOp precond_op() {
        return [h = h_](std::span<const double> in, std::span<double> out) {
            check(sap_apply_preconditioner(h, in.data(), out.data(), 0));
        };
    }
    LinearOp operator_op() {
        return [h = h_](std::span<const double> in, std::span<double> out) {
            check(sap_apply_operator(h, in.data(), out.data(), 0));
        };
    }

    // solve ≙ run_krylov(A, M, b, x, KrylovOptions) entirely on the device.
    sap_solve_stats solve(std::span<const double> b, std::span<double> x, std::vector<double>* history = nullptr) {
        sap_solve_stats st{};
        std::vector<double> hist(8 * 1024);
        st.history = hist.data();
        st.history_capacity = static_cast<int>(hist.size());
        check(sap_solve(h_, b.data(), x.data(), 0, &st));
        if (history) history->assign(hist.begin(), hist.begin() + std::min<int>(st.history_len, st.history_capacity));
        st.history = nullptr;
        return st;
    }

    sap_report report() const {
        sap_report r{};
        check(sap_get_report(h_, &r));
        return r;
    }
    sap_handle* handle() const { return h_; }

private:
    sap_handle* h_ = nullptr;
    int n_ = 0;
};

}  // namespace sap::gpu
