// Standalone driver: factor config-2 blocks once with the traced LU and print the per-phase timeline.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../include/sap_gpu.h"
namespace sapgpu { void read_lu_trace(long long* out); void read_lu_wtrace(long long* out); }
// usage: lu_trace [D] [k]   (SaP-C by default; the one-CTA-per-job kernel, sap_options::lu_kernel = 1)
int main(int argc, char** argv) {
    const int n = 200000, p = 50;
    const int k = argc > 2 ? atoi(argv[2]) : 200;
    std::vector<double> band((size_t)n * (2 * k + 1)), rhs(n);
    sap_random_banded(n, k, 1.0, 1, band.data(), rhs.data());
    sap_options o; sap_options_default(&o); o.p = p;
    o.precond = (argc > 1 && argv[1][0] == 'D') ? SAP_PRECOND_DECOUPLED : SAP_PRECOND_COUPLED;
    o.lu_kernel = 1;
    sap_handle* h; sap_create(&o, &h);
    sap_setup_banded(h, n, k, band.data(), 0);
    sap_setup_banded(h, n, k, band.data(), 0);
    sap_report r; sap_get_report(h, &r);
    printf("t_factor_kernel %.3f ms\n", r.t_factor_kernel * 1e3);
    long long t[16 * 12];
    sapgpu::read_lu_trace(t);
    const char* names[] = {"S0", "S1", "s2", "rowscols", "s4", "s5", "s6", "bulk", "diag+stores", "s9"};
    for (int s = 0; s < 15; ++s) {
        long long b = t[s * 12];
        printf("step %2d:", s);
        for (int q = 1; q < 10; ++q) printf(" %s=%6lld", names[q], t[s * 12 + q] ? t[s * 12 + q] - b : -1);
        printf(" | next S0 %6lld\n", t[(s + 1) * 12] - b);
    }
    long long wt[64];
    sapgpu::read_lu_wtrace(wt);
    printf("step 8 per-warp trailing-update time (tile loop, cycles):");
    for (int w = 0; w < 16; ++w) printf(" %lld", wt[16 + w] - wt[w]);
    printf("\nstep 8 per-warp start offset (vs warp 0):");
    for (int w = 0; w < 16; ++w) printf(" %lld", wt[w] - wt[0]);
    printf("\n");
    sap_destroy(h);
}
