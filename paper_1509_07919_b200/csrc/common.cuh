// Shared definitions for the SaP B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sapgpu {

// ---------------------------------------------------------------------------
// Errors crossing from kernels/host helpers to the C ABI.

struct InvalidArgument : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct PreconditionerFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CommFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
#define SAP_CUDA(call) ::sapgpu::cuda_check((call), #call)

// Launch counter (read back through sap_report.kernel_launches).
extern long long g_launch_count;
inline void count_launch(int n = 1) { g_launch_count += n; }
#define SAP_LAUNCHED() do { ::sapgpu::count_launch(); SAP_CUDA(cudaGetLastError()); } while (0)

// ---------------------------------------------------------------------------
// Strided matrix view: element (i, c) lives at base[i*rs + c*cs].
//   band LU  : base = f + k,                     rs = 1,  cs = 2k
//   band UL  : base = f + (m-1)(2k+1) + k,       rs = -1, cs = -2k   (flipped system J A J)
//   dense row-major w x w : base = a,            rs = w,  cs = 1
// With slot(i, j) = j*(2k+1) + (i-j+k) = j*2k + i + k the tall-thin band is a
// column-major matrix of leading dimension 2k, which is what makes one
// factorization kernel serve all three.
struct FactorJob {
    double* base;
    long long rs;
    long long cs;
    int m;            // order of the block
    int k;            // half-bandwidth (dense: w-1)
    const double* scale;  // boost scale (block infinity norm), device pointer
    int* boosts;      // device counter (written, not accumulated)
    const double* src = nullptr;  // unfactored block in the same strided view (nullptr: in place, base)
    // streamed upload (k_band_lu_res only): the band arrives while the kernel runs. *ready counts the
    // finished upload rounds; each brings `piece` more columns of this job's view from its own end
    // (`ends` = 2: the other end too, for the UL job of the same block). No boosting in this mode:
    // the kernel records min |pivot| in *minpiv and the caller checks it against the final scale.
    const unsigned* ready = nullptr;
    int piece = 0;
    int ends = 1;
    double* minpiv = nullptr;
    const int* gate = nullptr;  // k_band_lu_res<B, false>: run only if (*gate & 1) (the streamed refactor)
};

// Per-block strided band store used for every factor buffer (LU, UL, reduced
// blocks): block b's tall-thin band (m_b*(2k+1) doubles in the reference's slot
// layout) starts at base + b*pstride + pad. pad = k & 1 makes (block start + k)
// 16-byte aligned, so every 32-row column segment (slot c*2k + i0 + k, i0 % 32 == 0)
// is 16-byte aligned for TMA. Padding slots are zero.
struct BandStore {
    long long pstride = 0;
    int pad = 0;
    int m_max = 0;
    int k = 0;
    static BandStore make(int m_max, int k) {
        BandStore b;
        b.m_max = m_max;
        b.k = k;
        b.pad = k & 1;
        long long need = (long long)m_max * (2LL * k + 1) + 64 + 2;
        b.pstride = (need + 15) & ~15LL;
        return b;
    }
    size_t total(int blocks) const { return (size_t)pstride * blocks; }
    long long block(int b) const { return (long long)b * pstride + pad; }
};

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b, double c0, double c1) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace sapgpu
