// Deterministic reductions and small vector kernels.
//
// Dot products (krylov.hpp:45-49 sums sequentially) are formed over a fixed
// partition of [0, n) into kRedChunk-element chunks, each reduced by a fixed
// tree; the chunk partials are summed in index order by the last CTA to
// finish. The result therefore depends only on n and the data - never on
// scheduling - which keeps solves bitwise repeatable (acceptance criterion
// 10, proj/tests/acceptance.cpp:592-606).
#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

constexpr int kRedThreads = 256;
constexpr int kRedChunk = 4096;

int reduce_blocks(int n) { return std::max(1, ceil_div(n, kRedChunk)); }

__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    return t;  // valid on thread 0
}

// The last CTA's sum of the per-CTA partials of m reductions (partials[q * G + b]): thread q < m adds them in
// block order b = 0, 1, ... (the order the result is defined by); the loads are staged through shared memory by
// every thread at once (a serial ld.cg per partial was ~15 us of L2 latency per dot at n = 200 000).
__device__ double sum_partials(const double* __restrict__ partials, int G, int m, int q) {
    constexpr int kStage = 1024;
    __shared__ double stage[kStage];
    const int T = kStage / max(m, 1);
    double tot = 0.0;
    for (int b0 = 0; b0 < G; b0 += T) {
        const int nb = min(T, G - b0);
        for (int e = threadIdx.x; e < m * nb; e += blockDim.x) {
            const int qq = e / nb, b = e - qq * nb;
            stage[qq * T + b] = __ldcg(partials + (size_t)qq * G + b0 + b);
        }
        __syncthreads();
        if (q < m)
            for (int b = 0; b < nb; ++b) tot += stage[q * T + b];
        __syncthreads();
    }
    return tot;
}

__global__ void __launch_bounds__(kRedThreads)
    k_dot(const double* __restrict__ a, const double* __restrict__ b, int n, double* __restrict__ partials,
          unsigned* __restrict__ counter, double* __restrict__ out) {
    __shared__ double sh[32];
    __shared__ bool last;
    const int base = blockIdx.x * kRedChunk;
    const int end = min(base + kRedChunk, n);
    constexpr int kPer = kRedChunk / kRedThreads;  // all the thread's loads in flight, then its chain in order
    double va[kPer], vb[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int i = base + threadIdx.x + u * kRedThreads;
        va[u] = i < end ? __ldcg(a + i) : 0.0;
        vb[u] = i < end ? __ldcg(b + i) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        if (base + (int)threadIdx.x + u * kRedThreads >= end) break;
        s = fma(va[u], vb[u], s);
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = t;
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        const double tot = sum_partials(partials, gridDim.x, 1, 0);
        if (threadIdx.x == 0) {
            *out = tot;
            *counter = 0u;
        }
    }
}

void launch_dot(const double* a, const double* b, int n, double* partials, unsigned* counter, double* out,
                cudaStream_t s) {
    k_dot<<<reduce_blocks(n), kRedThreads, 0, s>>>(a, b, n, partials, counter, out);
    SAP_LAUNCHED();
}

// Several dot products in one pass over the same fixed partition and trees as k_dot: pair q is bitwise
// k_dot(a[q], b[q]). kind[q] = 1: the squared norm of the residual a[q] - b[q] (each element fma(-1, b, a),
// exactly k_xpay's scratch = b - A x, then fma(r, r, acc) as k_dot(scratch, scratch)) without storing it.
__global__ void __launch_bounds__(kRedThreads)
    k_dots(DotBatch d, int n, double* __restrict__ partials, unsigned* __restrict__ counter, double* __restrict__ out) {
    __shared__ double sh[32];
    __shared__ bool last;
    const int base = blockIdx.x * kRedChunk;
    const int end = min(base + kRedChunk, n);
    // per pair: the thread's 16 element pairs loaded at once, then its FMA chain in element order (the same
    // chain and tree as before; 49 CTAs at n = 200 000 need the loads in flight together)
    constexpr int kPer = kRedChunk / kRedThreads;
    double s[kMaxDots];
#pragma unroll
    for (int q = 0; q < kMaxDots; ++q) {
        s[q] = 0.0;
        if (q >= d.m) continue;
        double va[kPer], vb[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int i = base + threadIdx.x + u * kRedThreads;
            va[u] = i < end ? __ldcg(d.a[q] + i) : 0.0;
            vb[u] = i < end ? __ldcg(d.b[q] + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            if (base + (int)threadIdx.x + u * kRedThreads >= end) break;
            if (d.kind[q]) {
                const double r = fma(-1.0, vb[u], va[u]);
                s[q] = fma(r, r, s[q]);
            } else {
                s[q] = fma(va[u], vb[u], s[q]);
            }
        }
    }
    for (int q = 0; q < d.m; ++q) {
        const double t = block_sum(s[q], sh);
        if (threadIdx.x == 0) partials[q * gridDim.x + blockIdx.x] = t;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        const double tot = sum_partials(partials, gridDim.x, d.m, threadIdx.x);
        if (threadIdx.x < d.m) {
            out[threadIdx.x] = tot;
            if (d.hout) d.hout[threadIdx.x] = tot;
        }
        if (threadIdx.x == 0 && d.flag_dst) *d.flag_dst = __ldcg(d.flag_src);
        __syncthreads();
        if (threadIdx.x == 0) *counter = 0u;
    }
}

void launch_dots(const DotBatch& d, int n, double* partials, unsigned* counter, double* out, cudaStream_t s) {
    if (d.m <= 0) return;
    k_dots<<<reduce_blocks(n), kRedThreads, 0, s>>>(d, n, partials, counter, out);
    SAP_LAUNCHED();
}

// y -= (num / den) x with num, den device scalars (the quotient on the device, IEEE division like the host's
// dot / sigma): the MGS step of krylov.hpp:323-329 without a host round trip.
__global__ void k_axpy_quot(double* __restrict__ y, const double* __restrict__ num, const double* __restrict__ den,
                            const double* __restrict__ x, int n) {
    const double a = -(*num / *den);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) y[t] = fma(a, x[t], y[t]);
}

void launch_axpy_quot(double* y, const double* num, const double* den, const double* x, int n, cudaStream_t s) {
    k_axpy_quot<<<std::max(1, std::min(ceil_div(n, 256), 148 * 8)), 256, 0, s>>>(y, num, den, x, n);
    SAP_LAUNCHED();
}

__global__ void k_nonfinite(const double* __restrict__ a, int n, int* flag) {
    int bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (!isfinite(a[i])) bad = 1;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

void launch_nonfinite(const double* a, int n, int* flag, cudaStream_t s) {
    k_nonfinite<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(a, n, flag);
    SAP_LAUNCHED();
}

__global__ void k_cast_d2f(const double* __restrict__ in, float* __restrict__ out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (float)in[i];
}
__global__ void k_cast_f2d(const float* __restrict__ in, double* __restrict__ out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (double)in[i];
}
void launch_cast_d2f(const double* in, float* out, int n, cudaStream_t s) {
    k_cast_d2f<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(in, out, n);
    SAP_LAUNCHED();
}
void launch_cast_f2d(const float* in, double* out, int n, cudaStream_t s) {
    k_cast_f2d<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(in, out, n);
    SAP_LAUNCHED();
}

template <class T>
__global__ void k_cast_band(const double* __restrict__ in, T* __restrict__ out, size_t count) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        out[i] = static_cast<T>(in[i]);
}
template <class T>
void launch_cast_band(const double* in, T* out, size_t count, cudaStream_t s) {
    k_cast_band<T><<<(int)std::min<size_t>((count + 255) / 256, 148 * 16), 256, 0, s>>>(in, out, count);
    SAP_LAUNCHED();
}
template void launch_cast_band<float>(const double*, float*, size_t, cudaStream_t);
template void launch_cast_band<double>(const double*, double*, size_t, cudaStream_t);

}  // namespace sapgpu
