// Do DMMA (fp64 mma.sync m8n8k4) and DFMA share the fp64 pipe on B200?
// Each warp runs a DMMA chain set and/or a DFMA chain set; report FLOP rates.
#include <cstdio>
#include <cuda_runtime.h>
template <bool MMA, bool FMA>
__global__ void mix(long iters, double* out) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double c[4][2] = {};
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (long it = 0; it < iters; ++it) {
        if (MMA) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
        if (FMA) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, 1e-12);
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, 1e-12);
        }
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}
template <bool MMA, bool FMA>
void run(const char* name) {
    double* out;
    cudaMalloc(&out, 8);
    const long iters = 20000;
    const int blocks = 148 * 4, threads = 256;
    mix<MMA, FMA><<<blocks, threads>>>(iters, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<MMA, FMA><<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    const double mma_fl = MMA ? warps * iters * 4 * 512.0 : 0;   // 8x8x4 x2 flops per mma
    const double fma_fl = FMA ? warps * 32 * iters * 16 * 2.0 : 0;
    printf("%-10s %.3f ms  DMMA %.1f TF/s  DFMA %.1f TF/s  total %.1f TF/s\n", name, ms, mma_fl / ms / 1e9,
           fma_fl / ms / 1e9, (mma_fl + fma_fl) / ms / 1e9);
}
int main() {
    run<true, false>("dmma");
    run<false, true>("dfma");
    run<true, true>("both");
    return 0;
}
