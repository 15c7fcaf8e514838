// Banded SpMV variants at config 2 (N = 200000, K = 200), same per-row summation order (ascending columns, one
// FMA chain from zero): V0 = k_band_spmv (spmv.cu), V1 = 16 loads batched ahead of their FMAs, V2 = two row
// groups per warp (rows r0 + lane and r0 + 32 + lane: two independent chains). Prints us / GB/s and bitwise checks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe/spmv_probe.cu -o tools/probe/spmv_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__global__ void __launch_bounds__(256) v0(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
#pragma unroll 8
        for (int j = clo; j <= chi; ++j, col += ld) {
            const double xv = __ldg(x + j);
            if (i < n && i - j <= k && j - i <= k) acc = fma(*col, xv, acc);
        }
        if (i < n) y[i] = acc;
    }
}

template <int NB>
__global__ void __launch_bounds__(256) v1(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 32; r0 < n; r0 += nw * 32) {
        const int i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        double acc = 0.0;
        const double* col = a + (long long)clo * ld + i + k;
        for (int j0 = clo; j0 <= chi; j0 += NB) {
            double v[NB], xv[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int j = j0 + u;
                const bool ok = j <= chi && i < n && i - j <= k && j - i <= k;
                v[u] = ok ? __ldcs(col + (long long)u * ld) : 0.0;
                xv[u] = j <= chi ? __ldg(x + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int j = j0 + u;
                if (j <= chi && i < n && i - j <= k && j - i <= k) acc = fma(v[u], xv[u], acc);
            }
            col += NB * ld;
        }
        if (i < n) y[i] = acc;
    }
}

__global__ void __launch_bounds__(256) v2(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const long long ld = 2LL * k;
    for (int r0 = wg * 64; r0 < n; r0 += nw * 64) {
        const int i0 = r0 + lane, i1 = r0 + 32 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 63 + k, n - 1);
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = a + (long long)clo * ld + i0 + k;
#pragma unroll 8
        for (int j = clo; j <= chi; ++j, col += ld) {
            const double xv = __ldg(x + j);
            if (i0 < n && i0 - j <= k && j - i0 <= k) acc0 = fma(col[0], xv, acc0);
            if (i1 < n && i1 - j <= k && j - i1 <= k) acc1 = fma(col[32], xv, acc1);
        }
        if (i0 < n) y[i0] = acc0;
        if (i1 < n) y[i1] = acc1;
    }
}

// V3: the CTA's 8 warps (rows rb .. rb + 255) walk one common column range in lock-step (a barrier every SYNC
// columns), each warp active on its own window, so at any time the CTA reads ~2 KB contiguous of one column
// block instead of 8 scattered 256-byte pieces (same per-row order)
template <int SYNC>
__global__ void __launch_bounds__(256) v3(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long ld = 2LL * k;
    for (int rb = blockIdx.x * 256; rb < n; rb += gridDim.x * 256) {
        const int r0 = rb + 32 * warp, i = r0 + lane;
        const int clo = max(r0 - k, 0), chi = min(r0 + 31 + k, n - 1);
        const int blo = max(rb - k, 0), bhi = min(rb + 255 + k, n - 1);
        double acc = 0.0;
        for (int j0 = blo; j0 <= bhi; j0 += SYNC) {
            const int ja = max(j0, clo), jb = min(j0 + SYNC - 1, chi);
            const double* col = a + (long long)ja * ld + i + k;
#pragma unroll 8
            for (int j = ja; j <= jb; ++j, col += ld) {
                const double xv = __ldg(x + j);
                if (i < n && i - j <= k && j - i <= k) acc = fma(*col, xv, acc);
            }
            __syncthreads();
        }
        if (i < n) y[i] = acc;
    }
}

// V5: bulk-copy pipeline. A CTA (128 threads, a row each) takes 128-row tiles; per 32-column chunk one thread
// issues, per column, one cp.async.bulk of that column's in-band run for the tile's rows (~1 KB contiguous,
// 16-byte aligned), three chunks in flight under mbarriers; every row's FMA chain runs over ascending columns
// as in V0 (bitwise equal).
namespace v5ns {
constexpr int R = 128, C = 32, ST = 3, LD = R + 4;
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(su32(bar)), "r"(parity)
                     : "memory");
}
}  // namespace v5ns

__global__ void __launch_bounds__(128) v5(const double* __restrict__ a, int n, int k, const double* __restrict__ x,
                                          double* __restrict__ y) {
    using namespace v5ns;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    __shared__ int cb[ST][C];  // smem index of (row 0, column j0 + u) = cb + i; -1: column empty
    __shared__ int ce[ST][C];  // rows i with cb + i < ce came in the copy (the array's odd last element: direct)
    const int tid = threadIdx.x, lane = tid & 31;
    const int W = 2 * k + 1;
    const long long total = (long long)n * W;
    const int ntiles = (n + R - 1) / R;
    if (tid == 0) {
        for (int q = 0; q < ST; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[q])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int pt = blockIdx.x, pc = 0, issued = 0;  // producer cursor (warp 0, uniform)
    auto tile_cols = [&](int t, int& jlo, int& nch) {
        const int r0 = t * R;
        jlo = max(r0 - k, 0);
        const int jhi = min(r0 + R - 1 + k, n - 1);
        nch = (jhi - jlo + C) / C;
    };
    auto issue = [&]() {  // warp 0: lane u issues column u of the next chunk
        if (pt >= ntiles) return;
        int jlo, nch;
        tile_cols(pt, jlo, nch);
        const int r0 = pt * R, st = issued % ST, j = jlo + pc * C + lane;
        const int rhi = min(r0 + R, n) - 1;
        int len = 0;
        long long g0 = 0;
        if (j < n && j <= r0 + R - 1 + k) {
            const int slo = max(r0 - j + k, 0), shi = min(rhi - j + k, 2 * k);
            if (slo <= shi) {
                g0 = ((long long)j * W + slo) & ~1LL;
                long long g1 = ((long long)j * W + shi + 2) & ~1LL;
                if (g1 > total) g1 = total & ~1LL;
                len = g1 > g0 ? (int)(g1 - g0) : 0;
            }
        }
        const int sbase = (st * C + lane) * LD;
        cb[st][lane] = len > 0 ? sbase + (int)((long long)j * W + k - j - g0) : -1;
        ce[st][lane] = sbase + len;
        unsigned bytes = 8u * (unsigned)len;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[st])), "r"(bytes)
                         : "memory");
        __syncwarp();
        if (len > 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm + sbase)),
                         "l"(a + g0), "r"(8u * (unsigned)len), "r"(su32(&bar[st]))
                         : "memory");
        ++issued;
        if (++pc == nch) {
            pc = 0;
            pt += gridDim.x;
        }
    };
    if (tid < 32)
        for (int q = 0; q < ST; ++q) issue();
    int consumed = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int jlo, nch;
        tile_cols(t, jlo, nch);
        const int i = t * R + tid;
        double acc = 0.0;
        for (int c = 0; c < nch; ++c, ++consumed) {
            const int st = consumed % ST;
            v5ns::wait(&bar[st], (consumed / ST) & 1);
            const int j0 = jlo + c * C;
#pragma unroll 8
            for (int u = 0; u < C; ++u) {
                const int j = j0 + u;
                if (i < n && j < n && i - j <= k && j - i <= k) {
                    const int e = cb[st][u] + i;
                    const double v = e < ce[st][u] ? sm[e] : a[(long long)j * W + (i - j + k)];
                    acc = fma(v, __ldg(x + j), acc);
                }
            }
            __syncthreads();  // every thread is done with this stage
            if (tid < 32) issue();
        }
        if (i < n) y[i] = acc;
    }
}

int main() {
    const int n = 200000, k = 200;
    const size_t w = 2 * k + 1, total = (size_t)n * w;
    std::vector<double> ha(total, 0.0), hx(n);
    srand(3);
    for (size_t j = 0; j < (size_t)n; ++j)
        for (int s = 0; s < (int)w; ++s) {
            const long long i = (long long)j - k + s;
            if (i >= 0 && i < n) ha[j * w + s] = rand() / (double)RAND_MAX - 0.5;
        }
    for (int i = 0; i < n; ++i) hx[i] = rand() / (double)RAND_MAX - 0.5;
    double *a, *x, *y0, *y1;
    cudaMalloc(&a, total * 8);
    cudaMalloc(&x, n * 8);
    cudaMalloc(&y0, n * 8);
    cudaMalloc(&y1, n * 8);
    cudaMemcpy(a, ha.data(), total * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice);
    const double bytes = 8.0 * total + 16.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 5; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 50; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 50;
        std::vector<double> h0(n), h1(n);
        cudaMemcpy(h0.data(), y0, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(h1.data(), y1, n * 8, cudaMemcpyDeviceToHost);
        printf("%-28s %7.1f us  %6.0f GB/s  bitwise vs v0: %s\n", name, us, bytes / (us * 1e-6) / 1e9,
               memcmp(h0.data(), h1.data(), n * 8) == 0 ? "yes" : "NO");
    };
    const int warps = (n + 31) / 32;
    auto g = [](int warps_, int per) { return std::min((warps_ + per - 1) / per, 148 * 64); };
    v0<<<g(warps, 8), 256>>>(a, n, k, x, y0);
    timeit("v0 (current)", [&] { v0<<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v1 batch 16", [&] { v1<16><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v1 batch 32", [&] { v1<32><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v2 two row groups", [&] { v2<<<g((n + 63) / 64, 8), 256>>>(a, n, k, x, y1); });
    timeit("v0 128-thread blocks", [&] { v0<<<g(warps, 4), 128>>>(a, n, k, x, y1); });
    {
        const int sm5 = v5ns::ST * v5ns::C * v5ns::LD * 8;
        cudaFuncSetAttribute(v5, cudaFuncAttributeMaxDynamicSharedMemorySize, sm5);
        int nsm = 148, per = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, v5, 128, sm5);
        printf("v5: %d CTAs per SM, %d bytes smem\n", per, sm5);
        timeit("v5 bulk-copy pipeline", [&] { v5<<<nsm * per, 128, sm5>>>(a, n, k, x, y1); });
    }
    timeit("v3 lock-step, sync 16", [&] { v3<16><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v3 lock-step, sync 32", [&] { v3<32><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    timeit("v3 lock-step, sync 64", [&] { v3<64><<<g(warps, 8), 256>>>(a, n, k, x, y1); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
