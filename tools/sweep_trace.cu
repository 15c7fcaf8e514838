// Driver: config-2 SaP-D setup + one preconditioner apply with the traced pair sweep (forward chunks 8..39 of
// block 0); prints per-chunk clock64 deltas, finisher CTA and helper CTA separately (different SMs).
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
    long long t[32 * 12];
    sapgpu::read_sweep_trace(t);
    printf("F (relative to w0 X-sync of the chunk): w0 Y-arrive | w1: start slab bar5 hpart wbuf || H (rel. to start): slab+sync sent | H period\n");
    for (int c = 0; c < 31; ++c) {
        const long long* r = t + c * 12;
        long long b = r[0];
        printf("%2d: %6lld | %6lld %6lld %6lld %6lld %6lld | F period %6lld || %6lld %6lld | %6lld\n", c + 8, r[1] - b, r[2] - b, r[3] - b,
               r[4] - b, r[5] - b, r[6] - b, r[12] - b, r[8] - r[7], r[9] - r[7], r[12 + 7] - r[7]);
    }
    sap_destroy(h);
}
