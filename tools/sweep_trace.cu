// Driver: config-2 SaP-D setup + preconditioner applies with the traced k_sweep_tma; prints, for block 0's
// forward sweep, cycles per chunk spent waiting on the slab mbarrier, at barrier A, in phase 1 and phase 2
// (thread 0 = warp 0, thread 32 = warp 1).
#include <cstdio>
#include <vector>
#include "../include/sap_gpu.h"
namespace sapgpu { void read_sweep_trace(long long* out); }
int main() {
    const int n = 200000, k = 200, p = 50;
    std::vector<double> band((size_t)n * (2 * k + 1)), rhs(n), out(n);
    sap_random_banded(n, k, 1.0, 1, band.data(), rhs.data());
    sap_options o; sap_options_default(&o); o.p = p; o.precond = SAP_PRECOND_DECOUPLED;
    sap_handle* h; sap_create(&o, &h);
    sap_setup_banded(h, n, k, band.data(), 0);
    sap_apply_preconditioner(h, rhs.data(), out.data(), 0);
    sap_apply_preconditioner(h, rhs.data(), out.data(), 0);
    long long t[24];
    sapgpu::read_sweep_trace(t);
    for (int w = 0; w < 3; ++w) {
        const long long* r = t + 6 * w;
        const double c = (double)r[5];
        printf("%s: %lld chunks, per chunk: total %.0f | mbar wait %.0f | barrier A %.0f | phase 1 %.0f | "
               "phase 2 (+B) %.0f cycles\n", w == 0 ? "warp 0 (finisher)" : w == 1 ? "warp 1 (helper)" : "warp 15 (producer)", r[5], r[0] / c, r[1] / c, r[2] / c, r[3] / c, r[4] / c);
    }
    sap_destroy(h);
}
