// Driver: config-2 SaP-D setup + one preconditioner apply with the traced sweep; prints the per-chunk timeline.
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
    long long t[24 * 8];
    sapgpu::read_sweep_trace(t);
    printf("chunk: wait_done barA phase1(w0) phase1(w1) phase1(w15) barB | next\n");
    for (int c = 1; c < 23; ++c) {
        long long b = t[c * 8];
        printf("%2d: %6lld %6lld %6lld %6lld %6lld %6lld | %6lld\n", c, t[c*8+1]-b, t[c*8+2]-b, t[c*8+3]-b, t[c*8+4]-b, t[c*8+5]-b, t[c*8+6]-b, t[(c+1)*8]-b);
    }
    sap_destroy(h);
}
