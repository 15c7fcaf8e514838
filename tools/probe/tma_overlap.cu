// Probe: does a TMA tiled tensor map accept an overlapping 2D view of the
// tall-thin band (dim0 = rows, stride1 = 2k doubles < dim0 extent)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k_load(const __grid_constant__ CUtensorMap tm, double* out, int x0, int x1, int ncol) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long mbar;
    unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned bytes = 32 * ncol * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes));
        unsigned dst = (unsigned)__cvta_generic_to_shared(sm);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"(&tm), "r"(x0), "r"(x1), "r"(mb) : "memory");
    }
    unsigned done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mb));
    }
    for (int i = threadIdx.x; i < 32 * ncol; i += blockDim.x) out[i] = sm[i];
}

int main() {
    const int n = 4000, k = 200;
    const size_t total = (size_t)n * (2 * k + 1) + 64;
    std::vector<double> h(total);
    for (size_t i = 0; i < total; ++i) h[i] = (double)i;
    double* d;
    cudaMalloc(&d, total * 8);
    cudaMemcpy(d, h.data(), total * 8, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    printf("entry point %p\n", (void*)enc);
    CUtensorMap tm;
    // element (i, c) at base + c*2k + i, base = d + k  (i = row 0..n-1, c = column)
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)2 * k * 8};
    int ncol = 232;
    cuuint32_t box[2] = {32, 232};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d + k, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode overlapping: %d\n", (int)r);
    if (r != 0) return 1;
    double* out;
    cudaMalloc(&out, 32 * ncol * 8);
    cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * ncol * 8);
    for (int trial = 0; trial < 2; ++trial) {
        int i0 = trial == 0 ? 640 : 3968, c0 = i0 - k;
        k_load<<<1, 256, 32 * ncol * 8>>>(tm, out, i0, c0, ncol);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(32 * ncol);
        cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0, oob = 0;
        for (int cc = 0; cc < ncol; ++cc)
            for (int rr = 0; rr < 32; ++rr) {
                int i = i0 + rr, c = c0 + cc;
                double want = (i < n && c >= 0 && c < n) ? (double)((size_t)c * 2 * k + i + k) : 0.0;
                if (o[cc * 32 + rr] != want) ++bad;
                if (!(i < n && c >= 0 && c < n)) ++oob;
            }
        printf("trial %d err=%s mismatches=%d (oob elems %d)\n", trial, cudaGetErrorString(e), bad, oob);
    }
    return 0;
}
