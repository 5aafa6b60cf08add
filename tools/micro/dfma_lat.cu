// DFMA dependent-chain latency / ILP probe: one CTA per SM, W warps, C chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void chains(double* out, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(int warps, double* out) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<C><<<148, warps * 32>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e0);
    chains<C><<<148, warps * 32>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double wi = 148.0 * warps * (double)iters * C;  // warp DFMA instructions
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("warps/SM %2d chains %2d: %.3f ms  warp-DFMA per SMSP-cycle %.3f  cycles per dependent DFMA per warp %.1f\n",
           warps, C, ms, wi / 148 / 4 / cyc, cyc * (warps < 4 ? 1 : warps / 4.0) / iters / (warps < 4 ? 1 : 1) / 1.0 / (warps >= 4 ? warps / 4.0 : 1));
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    for (int w : {4, 8, 16}) {
        run<1>(w, out);
        run<2>(w, out);
        run<4>(w, out);
        run<8>(w, out);
        run<16>(w, out);
    }
    return 0;
}
