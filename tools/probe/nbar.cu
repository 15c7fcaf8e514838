// Named-barrier producer/consumer handoff cost: warp 0 <-> 15 helper warps, alternating barrier ids (as in
// k_sweep_pair), trivial work; also __syncthreads ping-pong for reference. Cycles per iteration.
#include <cstdio>
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__global__ void k(long long* out, int iters, int mode, double* g) {
    __shared__ double buf[64];
    __shared__ __align__(16) double dst[64];
    __shared__ unsigned long long mb;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb)));
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    double acc = 0;
    if (mode == 0) {
        if (warp == 0) {
            for (int t = 0; t < iters; ++t) {
                nbar_sync(1 + (t & 1), 512);
                buf[lane] = acc + t;
                nbar_arrive(3 + (t & 1), 512);
            }
        } else {
            for (int t = 0; t < iters; ++t) {
                if (t >= 2) nbar_sync(3 + (t & 1), 512);
                acc += buf[lane];
                nbar_arrive(1 + (t & 1), 512);
            }
            for (int t = iters; t < iters + 2; ++t) nbar_sync(3 + (t & 1), 512);
        }
    } else if (mode == 1) {
        for (int t = 0; t < iters; ++t) {
            if (warp == 0) buf[lane] = acc + t;
            __syncthreads();
            acc += buf[lane];
            __syncthreads();
        }
    } else if (mode >= 3) {
        if (warp == 0) {
            for (int t = 0; t < iters; ++t) {
                nbar_sync(1 + (t & 1), 512);
                buf[lane] = acc + t;
                if (mode == 3) g[lane] = acc + t;
                if (mode == 4 || mode == 5) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (mode == 5) {
                    __syncwarp();
                    if (lane == 0) {
                        const unsigned a = (unsigned)__cvta_generic_to_shared(&mb);
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 256;" ::"r"(a) : "memory");
                        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                                     ::"r"((unsigned)__cvta_generic_to_shared(dst)), "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(a) : "memory");
                    }
                }
                nbar_arrive(3 + (t & 1), 512);
            }
        } else {
            for (int t = 0; t < iters; ++t) {
                if (t >= 2) nbar_sync(3 + (t & 1), 512);
                acc += buf[lane];
                nbar_arrive(1 + (t & 1), 512);
            }
            for (int t = iters; t < iters + 2; ++t) nbar_sync(3 + (t & 1), 512);
        }
    } else {
        // helpers-only barrier (480) + handoff
        if (warp == 0) {
            for (int t = 0; t < iters; ++t) {
                nbar_sync(1 + (t & 1), 512);
                buf[lane] = acc + t;
                nbar_arrive(3 + (t & 1), 512);
            }
        } else {
            for (int t = 0; t < iters; ++t) {
                if (t >= 2) nbar_sync(3 + (t & 1), 512);
                acc += buf[lane];
                nbar_sync(5, 480);
                nbar_arrive(1 + (t & 1), 512);
            }
            for (int t = iters; t < iters + 2; ++t) nbar_sync(3 + (t & 1), 512);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (acc == 12345) out[1] = 1;
}
int main() {
    long long* o; cudaMallocManaged(&o, 16);
    double* g; cudaMalloc(&g, 4096);
    const char* nm[] = {"named-barrier handoff", "syncthreads x2", "handoff + helper barrier", "handoff + STG", "handoff + fence.proxy.async", "handoff + fence + bulk s2s"};
    for (int mode = 0; mode < 6; ++mode) {
        k<<<1, 512>>>(o, 100, mode, g); cudaDeviceSynchronize();
        k<<<1, 512>>>(o, 1000, mode, g); cudaDeviceSynchronize();
        printf("%-28s %lld cycles/iter  %s\n", nm[mode], o[0], cudaGetErrorString(cudaGetLastError()));
    }
}
