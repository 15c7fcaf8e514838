// Instruction-cache probe: one warp runs a straight-line block of N dependent-free DADDs (16-byte
// instructions), repeated REPS times; cycles per instruction vs code size show the i-cache capacity and
// the miss cost for code executed once per loop trip.
#include <cstdio>
template <int N>
__global__ void k(double* out, long long* cyc, int reps) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = a0 + a1 + a2 + a3;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int N>
void run(double* o, long long* c) {
    for (int reps : {1, 8}) {
        k<N><<<1, 32>>>(o, c, reps);
        cudaDeviceSynchronize();
        k<N><<<1, 32>>>(o, c, reps);
        cudaDeviceSynchronize();
        printf("N=%6d instrs (%7d bytes) reps=%d: %.2f cycles/instr\n", N, N * 16, reps, (double)*c / (N * (double)reps));
    }
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 32); cudaMallocManaged(&c, 8);
    run<256>(o, c); run<512>(o, c); run<1024>(o, c); run<2048>(o, c); run<4096>(o, c); run<8192>(o, c); run<16384>(o, c);
}
