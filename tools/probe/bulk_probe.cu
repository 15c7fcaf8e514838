// Isolated trailing-update (bulk) timing: 100 CTAs x 512 threads, each CTA repeatedly updates its own
// 200 x 200 window of a tall-thin band (L2 resident) with 16 x 32 DMMA tiles, operands in smem.
// mode 0: as in k_band_lu_res (C from/to global); 1: C kept in registers (no global traffic);
// 2: global load/store only (no DMMA).
#include "../../paper_1509_07919_b200/csrc/lu.cu"
namespace sapgpu { long long g_launch_count = 0; }
using namespace sapgpu;

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_bulk(double* band, int K, int pld, int uld, int steps, int mode,
                                                 long long* cyc) {
    extern __shared__ __align__(16) double smem[];
    double* P = smem;
    double* U = smem + 32 * pld;
    for (int i = threadIdx.x; i < 32 * pld + 32 * uld; i += NT) smem[i] = 1e-3 * ((i * 37) % 101);
    __syncthreads();
    const long long ld = 2LL * K;
    const int m = 4000;
    double* base = band + (long long)blockIdx.x * m * (2 * K + 1) + K;
    Lu L{base, 1, ld, m, K, 32, pld, uld, 1e-10};
    const int R = K, nb = 32, ja = 64;
    const TileCtx T = make_tiles(0, R, 0, R, ja, ja, nb, 0, 0, 0);
    const int ntiles = ((R + kTileR - 1) / kTileR) * T.tcols;
    const int warp = threadIdx.x >> 5, nw = NT / 32, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    double keep[6][2][kTQ][2];
    for (int i = 0; i < 6; ++i) for (int a = 0; a < 2; ++a) for (int q = 0; q < kTQ; ++q) keep[i][a][q][0] = keep[i][a][q][1] = 0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        int it = 0;
        for (int t = warp; t < ntiles; t += nw, ++it) {
            double acc[2][kTQ][2];
            if (mode == 1) {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int q = 0; q < kTQ; ++q) { acc[a][q][0] = keep[it % 6][a][q][0]; acc[a][q][1] = keep[it % 6][a][q][1]; }
            } else {
                tile_load(L, T, t, acc);
            }
            if (mode != 2 && mode != 4) {
                const int row0 = (t / T.tcols) * kTileR, col0 = (t % T.tcols) * kTileC;
                const double* pk = P + nb + row0 + lr;
                const double* uk = U + col0 + lr;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const int kk = ks * 4 + lc;
                    const double b0 = -pk[kk * pld], b1 = -pk[kk * pld + 8];
#pragma unroll
                    for (int q = 0; q < kTQ; ++q) {
                        if (col0 + q * 8 >= R) continue;
                        const double aq = uk[kk * uld + q * 8];
                        dmma_m8n8k4(acc[0][q][0], acc[0][q][1], aq, b0, acc[0][q][0], acc[0][q][1]);
                        dmma_m8n8k4(acc[1][q][0], acc[1][q][1], aq, b1, acc[1][q][0], acc[1][q][1]);
                    }
                }
            }
            if (mode == 1) {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int q = 0; q < kTQ; ++q) { keep[it % 6][a][q][0] = acc[a][q][0]; keep[it % 6][a][q][1] = acc[a][q][1]; }
            } else if (mode >= 3) {
                const long long ra8 = 8, cq8 = 8 * ld;
                const int row0 = (t / T.tcols) * kTileR, col0 = (t % T.tcols) * kTileC;
                const int ib = row0 + 2 * lc, cb = col0 + lr;
                double* p00 = L.at(ja + ib, ja + cb);
                const bool full = row0 + kTileR <= R && col0 + kTileC <= R;
                if (full && ((reinterpret_cast<uintptr_t>(p00) & 15) == 0)) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q) __stcg(reinterpret_cast<double2*>(p00 + a * ra8 + q * cq8), make_double2(acc[a][q][0], acc[a][q][1]));
                } else {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int q = 0; q < kTQ; ++q)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int i = ib + a * 8 + e, c = cb + q * 8;
                                if (i < R && c < R) __stcg(p00 + a * ra8 + e + q * cq8, acc[a][q][e]);
                            }
                }
            } else {
                const long long ra8 = 8, cq8 = 8 * ld;
                const int row0 = (t / T.tcols) * kTileR, col0 = (t % T.tcols) * kTileC;
                const int ib = row0 + 2 * lc, cb = col0 + lr;
                double* p00 = L.at(ja + ib, ja + cb);
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int q = 0; q < kTQ; ++q)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int i = ib + a * 8 + e, c = cb + q * 8;
                            if (i < R && c < R) __stcg(p00 + a * ra8 + e + q * cq8, acc[a][q][e]);
                        }
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (mode == 1 && keep[0][0][0][0] == 12345.0) band[0] = keep[1][1][1][1];
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / steps;
}

// 32 x 32 warp tiles (4 x 4 DMMA tiles): half the operand loads per DMMA, half the tiles.
template <bool GLOBAL_C, bool DO_MMA>
__global__ void __launch_bounds__(512, 1) k_bulk32(double* band, int K, int pld, int uld, int steps, long long* cyc) {
    extern __shared__ __align__(16) double smem[];
    double* P = smem;
    double* U = smem + 32 * pld;
    for (int i = threadIdx.x; i < 32 * pld + 32 * uld; i += 512) smem[i] = 1e-3 * ((i * 37) % 101);
    __syncthreads();
    const long long ld = 2LL * K;
    const int m = 4000;
    double* base = band + (long long)blockIdx.x * m * (2 * K + 1) + K;
    const int R = K, nb = 32, ja = 64;
    const int tr = (R + 31) / 32, ntiles = tr * tr;
    const int warp = threadIdx.x >> 5, nw = 16, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    double sink = 0.0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        for (int t = warp; t < ntiles; t += nw) {
            const int row0 = (t / tr) * 32, col0 = (t % tr) * 32;
            double acc[4][4][2];
            double* p00 = base + (long long)(ja + col0 + lr) * ld + ja + row0 + 2 * lc;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool ok = row0 + a * 8 < R && col0 + q * 8 < R;
                    if (GLOBAL_C && ok) {
                        const double2 v = __ldcg(reinterpret_cast<const double2*>(p00 + a * 8 + q * 8 * ld));
                        acc[a][q][0] = v.x; acc[a][q][1] = v.y;
                    } else { acc[a][q][0] = 0.0; acc[a][q][1] = 0.0; }
                }
            if (DO_MMA) {
                const double* pk = P + nb + row0 + lr;
                const double* uk = U + col0 + lr;
#pragma unroll 2
                for (int ks = 0; ks < 8; ++ks) {
                    const int kk = ks * 4 + lc;
                    double b[4], a4[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) b[a] = (row0 + a * 8 < R) ? -pk[kk * pld + a * 8] : 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) a4[q] = (col0 + q * 8 < R) ? uk[kk * uld + q * 8] : 0.0;
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int q = 0; q < 4; ++q) dmma_m8n8k4(acc[a][q][0], acc[a][q][1], a4[q], b[a], acc[a][q][0], acc[a][q][1]);
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool ok = row0 + a * 8 < R && col0 + q * 8 < R;
                    if (GLOBAL_C) {
                        if (ok) __stcg(reinterpret_cast<double2*>(p00 + a * 8 + q * 8 * ld), make_double2(acc[a][q][0], acc[a][q][1]));
                    } else sink += acc[a][q][0] + acc[a][q][1];
                }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (sink == 12345.0) band[0] = sink;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / steps;
}

int main() {
    const int K = 200, m = 4000, ctas = 100, pld = 236, uld = 204;
    double* band;
    cudaMalloc(&band, sizeof(double) * (size_t)ctas * m * (2 * K + 1));
    cudaMemset(band, 0, sizeof(double) * (size_t)ctas * m * (2 * K + 1));
    long long* cyc;
    cudaMallocManaged(&cyc, sizeof(long long) * ctas);
    const size_t bytes = sizeof(double) * (32 * pld + 32 * uld);
    cudaFuncSetAttribute(k_bulk<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_bulk<768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_bulk<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    for (int nt : {768, 1024}) {
        auto k = nt == 768 ? k_bulk<768> : k_bulk<1024>;
        for (int mode : {3, 4}) {
            k<<<ctas, nt, bytes>>>(band, K, pld, uld, 50, mode, cyc);
            cudaDeviceSynchronize();
            long long mx = 0;
            for (int i = 0; i < ctas; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
            printf("threads %d mode %d: %lld cycles/step  %s\n", nt, mode, mx, cudaGetErrorString(cudaGetLastError()));
        }
    }
    const char* names[] = {"global C scalar st", "C in registers", "global only scalar st", "global C double2 st", "global only double2 st"};
    for (int mode = 0; mode < 5; ++mode)
        for (int nc : {1, ctas}) {
            k_bulk<512><<<nc, 512, bytes>>>(band, K, pld, uld, 50, mode, cyc);
            cudaDeviceSynchronize();
            long long mx = 0;
            for (int i = 0; i < nc; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
            printf("%-24s ctas=%3d: %lld cycles/step (DMMA-peak bound ~20000)\n", names[mode], nc, mx);
        }
    auto run32 = [&](auto kern, const char* nm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<ctas, 512, bytes>>>(band, K, pld, uld, 50, cyc);
        cudaDeviceSynchronize();
        long long mx = 0;
        for (int i = 0; i < ctas; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
        printf("%-24s ctas=%3d: %lld cycles/step\n", nm, ctas, mx);
    };
    run32(k_bulk32<true, true>, "32x32 global C + DMMA");
    run32(k_bulk32<false, true>, "32x32 DMMA only");
    run32(k_bulk32<true, false>, "32x32 global only");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
