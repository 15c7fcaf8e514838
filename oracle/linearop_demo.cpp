// TEST INFRASTRUCTURE — the INTEGRATION.md drop-in, compiled against the
// UNMODIFIED reference headers: the GPU preconditioner / operator / solve
// (libsap_gpu.so through include/sap_gpu.hpp) plugged into the reference's own
// sap::solve_krylov via sap::LinearOp (proj/include/sap/krylov.hpp:14, :110).
// Wiring follows proj/tests/acceptance.cpp:114-132.
//   usage: linearop_demo n k d seed p kind(0 coupled, 1 decoupled)
#include <cstdio>
#include <cstdlib>
#include <random>

#include "sap/sap.hpp"
#include "test_support.hpp"
#define SAP_GPU_REFERENCE_ERRORS
#include "sap_gpu.hpp"

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 10000, k = argc > 2 ? atoi(argv[2]) : 50;
    const double d = argc > 3 ? atof(argv[3]) : 1.0;
    const unsigned seed = argc > 4 ? (unsigned)atoi(argv[4]) : 3000;
    const int p = argc > 5 ? atoi(argv[5]) : 8, kind = argc > 6 ? atoi(argv[6]) : 0;
    std::mt19937 rng(seed);
    const sap::BandedMatrix<double> a = testsup::random_banded(n, k, d, rng);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<double> b(n);
    for (double& v : b) v = u(rng);

    // reference setup + solve (acceptance.cpp:114-132)
    const auto layout = sap::make_partition_layout(n, p, k);
    const auto f = sap::factor_blocks<double>(a, layout, kind == 0 ? sap::FactorMode::lu_and_ul : sap::FactorMode::lu_only);
    sap::SpikeSet<double> sp;
    if (kind == 0 && p > 1) sp = sap::compute_spike_tips<double>(f, sap::extract_coupling<double>(a, layout));
    sap::LinearOp op_a = [&a](std::span<const double> in, std::span<double> out) { a.matvec(in, out); };
    sap::LinearOp op_m = [&](std::span<const double> in, std::span<double> out) {
        const auto r = sap::apply_preconditioner(static_cast<sap::PrecondKind>(kind), f, sp, in);
        std::copy(r.begin(), r.end(), out.begin());
    };
    sap::KrylovOptions ko;
    std::vector<double> x_ref(n);
    const auto st_ref = sap::solve_krylov(op_a, op_m, b, x_ref, ko);

    // GPU setup; the GPU M (and A) dropped into the reference's own solve_krylov
    sap_options o;
    sap_options_default(&o);
    o.p = p;
    o.precond = kind;
    sap::gpu::Solver g(o);
    g.setup(n, k, a.storage());
    std::vector<double> x_mix(n);
    const auto st_mix = sap::solve_krylov(g.operator_op(), g.precond_op(), b, x_mix, ko);
    // fully device-resident solve through the C ABI
    std::vector<double> x_gpu(n);
    const auto st_gpu = g.solve(b, x_gpu);

    printf("reference solve_krylov: iterations %.2f residual %.3e\n", st_ref.iterations, st_ref.final_relative_residual);
    printf("reference solve_krylov + GPU LinearOps: iterations %.2f residual %.3e\n", st_mix.iterations,
           st_mix.final_relative_residual);
    printf("sap_solve (device BiCGStab): iterations %.2f residual %.3e\n", st_gpu.iterations,
           st_gpu.final_relative_residual);
    const bool ok = st_mix.converged && st_gpu.converged && std::abs(st_mix.iterations - st_ref.iterations) <= 1.0 &&
                    std::abs(st_gpu.iterations - st_ref.iterations) <= 1.0;
    printf(ok ? "OK\n" : "MISMATCH\n");
    return ok ? 0 : 1;
}
