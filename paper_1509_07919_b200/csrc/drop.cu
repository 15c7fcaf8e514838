// drop_off on the device (proj/include/sap/pipeline.hpp:59-99): the smallest half-bandwidth k whose
// dropped outside-band mass satisfies ||dropped||_F <= tol ||A||_F, for a CSR matrix.
//
// The decision compares floating-point sums, so they are formed in the reference's order: sums[d]
// accumulates v*v of the entries at distance d = |i - j| in CSR order (pipeline.hpp:67-71), and the
// suffix sums run from the largest distance down (:74-76). The entries are stably radix-sorted by
// distance (CUB; stable, so CSR order survives inside each distance), each distance's run is summed
// sequentially by one thread, and one thread forms the suffix chain and picks k. The
// half-bandwidth max|i - j| (half_bandwidth, the tol = 0 case) is an integer max reduction.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace sapgpu {

__global__ void k_half_bw(const int* __restrict__ rp, const int* __restrict__ ci, int n, int* __restrict__ kmax) {
    int best = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int s = rp[i]; s < rp[i + 1]; ++s) best = max(best, abs(i - ci[s]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best > 0) atomicMax(kmax, best);
}

// key = |i - j|, val = v * v (the reference's product), entry s of row i
__global__ void k_drop_terms(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                             int n, int* __restrict__ key, double* __restrict__ val) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int s = rp[i]; s < rp[i + 1]; ++s) {
            key[s] = abs(i - ci[s]);
            val[s] = v[s] * v[s];
        }
}

// run boundaries of the sorted keys: start[d] / end[d] (end exclusive; empty runs stay 0 / 0)
__global__ void k_runs(const int* __restrict__ key, int nnz, int* __restrict__ start, int* __restrict__ end) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nnz; s += gridDim.x * blockDim.x) {
        const int d = key[s];
        if (s == 0 || key[s - 1] != d) start[d] = s;
        if (s == nnz - 1 || key[s + 1] != d) end[d] = s + 1;
    }
}

// sums[d] = sequential sum of the run (pipeline.hpp:70: sums[d] += v * v in CSR order)
__global__ void k_run_sums(const double* __restrict__ val, const int* __restrict__ start, const int* __restrict__ end,
                           int kmax, double* __restrict__ sums) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d > kmax) return;
    double acc = 0.0;
    for (int s = start[d]; s < end[d]; ++s) acc += val[s];
    sums[d] = acc;
}

// suffix chain and the choice of k (pipeline.hpp:74-83), in place over sums[0 .. kmax + 1]:
// suf[d] = suf[d + 1] + sums[d] from the top (distances beyond kmax carry zero mass, so the chain
// from n - 1 down reaches kmax + 1 as +0.0), thr = tol * tol * suf[0], k = the first c with
// suf[c + 1] <= thr
__global__ void k_drop_pick(double* __restrict__ sums, int kmax, int n, double tol, int* __restrict__ k_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    sums[kmax + 1] = 0.0;
    for (int d = kmax; d >= 0; --d) sums[d] = sums[d + 1] + sums[d];
    const double thr = tol * tol * sums[0];
    int k = n > 0 ? n - 1 : 0;
    for (int c = 0; c < n; ++c)
        if ((c + 1 <= kmax + 1 ? sums[c + 1] : 0.0) <= thr) {
            k = c;
            break;
        }
    *k_out = k;
}

namespace {
template <class T>
struct Scratch {  // stream-ordered scratch for one drop_off_k call
    T* p = nullptr;
    cudaStream_t s;
    Scratch(size_t count, cudaStream_t st) : s(st) { SAP_CUDA(cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(count, 1), s)); }
    ~Scratch() { cudaFreeAsync(p, s); }
    T* get() const { return p; }
};
}  // namespace

int drop_off_k(const int* rp, const int* ci, const double* v, int n, int nnz, double tol, cudaStream_t s) {
    Scratch<int> kmax(1, s);
    SAP_CUDA(cudaMemsetAsync(kmax.get(), 0, sizeof(int), s));
    if (n > 0) {
        k_half_bw<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(rp, ci, n, kmax.get());
        SAP_LAUNCHED();
    }
    int hk = 0;
    SAP_CUDA(cudaMemcpyAsync(&hk, kmax.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    SAP_CUDA(cudaStreamSynchronize(s));
    if (tol == 0.0 || nnz == 0) return hk;
    Scratch<int> key(nnz, s), key2(nnz, s), start(hk + 1, s), end(hk + 1, s), kout(1, s);
    Scratch<double> val(nnz, s), val2(nnz, s), sums(hk + 2, s);
    k_drop_terms<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(rp, ci, v, n, key.get(), val.get());
    SAP_LAUNCHED();
    int bits = 1;
    while (bits < 31 && (1 << bits) <= hk) ++bits;
    size_t tmp_bytes = 0;
    SAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.get(), key2.get(), val.get(), val2.get(), nnz, 0,
                                             bits, s));
    Scratch<unsigned char> tmp(tmp_bytes, s);
    SAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, key.get(), key2.get(), val.get(), val2.get(), nnz,
                                             0, bits, s));
    count_launch();
    SAP_CUDA(cudaMemsetAsync(start.get(), 0, sizeof(int) * (hk + 1), s));
    SAP_CUDA(cudaMemsetAsync(end.get(), 0, sizeof(int) * (hk + 1), s));
    k_runs<<<std::min(ceil_div(nnz, 256), 148 * 8), 256, 0, s>>>(key2.get(), nnz, start.get(), end.get());
    SAP_LAUNCHED();
    k_run_sums<<<ceil_div(hk + 1, 128), 128, 0, s>>>(val2.get(), start.get(), end.get(), hk, sums.get());
    SAP_LAUNCHED();
    k_drop_pick<<<1, 32, 0, s>>>(sums.get(), hk, n, tol, kout.get());
    SAP_LAUNCHED();
    int k = 0;
    SAP_CUDA(cudaMemcpyAsync(&k, kout.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    SAP_CUDA(cudaStreamSynchronize(s));
    return k;
}

}  // namespace sapgpu
