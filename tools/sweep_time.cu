// Driver: config-2 SaP-D setup, then 20 preconditioner applies on device vectors; prints ms per apply.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../include/sap_gpu.h"
int main() {
    const int n = 200000, k = 200, p = 50;
    std::vector<double> band((size_t)n * (2 * k + 1)), rhs(n);
    sap_random_banded(n, k, 1.0, 1, band.data(), rhs.data());
    sap_options o; sap_options_default(&o); o.p = p; o.precond = SAP_PRECOND_DECOUPLED;
    sap_handle* h; sap_create(&o, &h);
    sap_setup_banded(h, n, k, band.data(), 0);
    double *din, *dout;
    cudaMalloc(&din, n * 8); cudaMalloc(&dout, n * 8);
    cudaMemcpy(din, rhs.data(), n * 8, cudaMemcpyHostToDevice);
    for (int i = 0; i < 3; ++i) sap_apply_preconditioner(h, din, dout, 1);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) sap_apply_preconditioner(h, din, dout, 1);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("SaP-D apply (one block solve): %.1f us\n", ms * 1e3 / 20);
    sap_destroy(h);
}
