// Device-resident BiCGStab(l) and CG (the reference's solve_krylov / solve_cg /
// run_krylov, proj/include/sap/krylov.hpp:110-442). Vectors live in HBM; the
// scalar recurrences run on the host exactly as the reference writes them,
// fed by deterministic device reductions.
#pragma once

#include <functional>
#include <initializer_list>
#include <vector>

#include "common.cuh"

namespace sapgpu {

// Device LinearOp: out = Op(in), both device pointers of length n.
using DeviceOp = std::function<void(const double* in, double* out)>;
// Optional fused pair: out0 = Op(in0), out1 = Op(in1) in one pass over the operator (empty = two Op calls).
using DeviceOp2 = std::function<void(const double* in0, double* out0, const double* in1, double* out1)>;

struct KrylovResult {
    double iterations = 0.0;
    std::vector<double> residual_history;
    bool converged = false;
    double final_relative_residual = 0.0;
    int failure = 0;  // sap_krylov_failure
};

struct KrylovConfig {
    int method = 0;  // 0 bicgstab_l, 1 cg, 2 automatic
    int ell = 2;
    double rel_tol = 1e-10;
    double abs_tol = 0.0;
    int max_iterations = 500;
    bool caller_asserts_spd = false;
    // multi-GPU: in-place sum over ranks of host doubles (null = single rank), and the
    // global index of this rank's first row (for the restart perturbation stream)
    std::function<void(double*, int)> reduce;
    // multi-GPU over NCCL: in-place sum over ranks of device doubles on the solver's stream; when set, dot
    // products are reduced on the device before their single device->host copy
    std::function<void(double*, int, cudaStream_t)> dreduce;
    long long row_offset = 0;
    // the operator has only finite entries (checked at setup): with the zero initial guess the first
    // residual b - A*0 is b exactly (every row sum of a*(+0) terms is +0), so the first A apply is skipped
    bool zero_guess_exact = false;
};

class KrylovSolver {
public:
    KrylovSolver() = default;
    ~KrylovSolver();
    KrylovSolver(const KrylovSolver&) = delete;
    KrylovSolver& operator=(const KrylovSolver&) = delete;

    // run_krylov: b, x device pointers; x is overwritten (x0 = 0).
    KrylovResult run(const DeviceOp& A, const DeviceOp& M, const double* b, double* x, int n,
                     const KrylovConfig& cfg, cudaStream_t s, const DeviceOp2& A2 = nullptr);
    long long host_syncs() const { return syncs_; }  // stream synchronisations of the last run

private:
    struct DotReq {
        const double* a;
        const double* b;
        int kind;  // 0: dot(a, b); 1: ||a - b||^2
    };
    void ensure(int n, int ell);
    void sync_host();
    double dot(const double* a, const double* b);
    std::vector<double> dots(const std::vector<DotReq>& reqs, bool flag_too = false);
    bool any_flag(int local);
    bool nonfinite(const double* v);
    KrylovResult bicgstab(const DeviceOp& A, const DeviceOp& M, const double* b, double* x, const KrylovConfig& cfg,
                          const DeviceOp2& A2);
    KrylovResult cg(const DeviceOp& A, const DeviceOp& M, const double* b, double* x, const KrylovConfig& cfg);

    int n_ = 0, ell_ = 0;
    long long syncs_ = 0;
    std::function<void(double*, int)> reduce_;
    std::function<void(double*, int, cudaStream_t)> dreduce_;
    cudaStream_t s_ = nullptr;
    double* buf_ = nullptr;       // all vectors
    double* partials_ = nullptr;  // reduction partials
    double* dscal_ = nullptr;     // device scalar outputs
    unsigned* counter_ = nullptr;
    int* dflag_ = nullptr;
    double* hpinned_ = nullptr;   // pinned host scalars (mapped: k_dots writes its results here directly)
    int* hflag_ = nullptr;
    double* dhpinned_ = nullptr;  // their device aliases
    int* dhflag_ = nullptr;
    std::vector<double*> r_, u_;
    double *tmp_ = nullptr, *rtilde_ = nullptr, *scratch_ = nullptr, *xc_ = nullptr, *noise_ = nullptr;
};

}  // namespace sapgpu
