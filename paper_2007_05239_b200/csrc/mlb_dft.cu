// Pruned separable DFT convolution (replaces rfftn * fused * irfftn,
// fastsum.py:492-495) as a chain of batched complex GEMMs.
//
// The spread grid is nonzero only on the active sub-box of L cells per axis,
// and the fused weights only on the band |k| <= N/2 (K = N+1 frequencies; the
// last axis keeps k >= 0, Kh = N/2+1, by Hermitian symmetry).  Each stage
// contracts one axis with the L x K twiddle table
//     E[u][k] = exp(-2 pi i k u / ng)        (u = ulo + cell, k = -N/2..N/2),
// forward (cells -> band) then inverse (band -> cells, conj(E), last axis
// real with weights 1,2,2,...,2 = the Hermitian pairing of +-k).
//
// Every stage is C[m][n] = sum_k A[m][k] B[k][n] (complex, batched) on
// 32x32 output tiles with the full reduction extent staged in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "mlb_internal.cuh"
#include "mlb_tma.cuh"

namespace mlb {

// operand kinds
enum : int {
    OP_DATA_C = 0,   // complex data: ptr[batch*bstride + row*ld + col]
    OP_DATA_R = 1,   // real data, same indexing (imag = 0)
    OP_TW = 2,       // twiddle E[u][k]: element (r, c) = tw[r*K + c + koff]
    OP_TW_T = 3,     // twiddle transposed: element (r, c) = tw[c*K + r + koff]
    OP_TWC = 4,      // conj twiddle E[u][k]:           (r, c) = conj(tw[r*K + c + koff])
    OP_TWC_T = 5,    // conj twiddle transposed:        (r, c) = conj(tw[c*K + r + koff])
    OP_DATA_HW = 6,  // complex data * Hermitian weight of its column (1 for col 0, else 2)
};
// epilogue kinds
enum : int { EP_C = 0, EP_C_MUL = 1, EP_REAL = 2 };

struct Operand {
    const void* p;
    int64_t bstride;
    int ld;
    int koff;
};

struct GemmArgs {
    Operand A, B;
    void* C;
    int64_t c_bstride;
    int ldc;
    int M, N, Kd;
    const double2* tw;
    int K;  // twiddle row stride
    const double* fused;
};

template <int KIND>
__device__ __forceinline__ double2 load_op(const Operand& o, const double2* tw, int K, int64_t batch, int r, int c) {
    if (KIND == OP_DATA_C) {
        return reinterpret_cast<const double2*>(o.p)[batch * o.bstride + (int64_t)r * o.ld + c];
    } else if (KIND == OP_DATA_R) {
        return make_double2(reinterpret_cast<const double*>(o.p)[batch * o.bstride + (int64_t)r * o.ld + c], 0.0);
    } else if (KIND == OP_DATA_HW) {
        double2 v = reinterpret_cast<const double2*>(o.p)[batch * o.bstride + (int64_t)r * o.ld + c];
        const double w = (c == 0) ? 1.0 : 2.0;
        return make_double2(v.x * w, v.y * w);
    } else if (KIND == OP_TW) {
        return tw[r * K + c + o.koff];
    } else if (KIND == OP_TW_T) {
        return tw[c * K + r + o.koff];
    } else if (KIND == OP_TWC) {
        double2 t = tw[r * K + c + o.koff];
        return make_double2(t.x, -t.y);
    } else {
        double2 t = tw[c * K + r + o.koff];
        return make_double2(t.x, -t.y);
    }
}

constexpr int TM = 32, TN = 32;

// One 32x32 output tile per CTA; the whole reduction extent (Kd <= ~130: the
// active cells L or the band K) is staged in shared memory at once, so every
// operand load is issued up front (no K-loop barriers); 2x2 outputs per
// thread (16 DFMA per 2 broadcast + 2 two-wavefront 16-byte loads).
template <int KA, int KB, int EP>
__global__ void __launch_bounds__(256) cgemm_kernel(GemmArgs g) {
    extern __shared__ double2 sm2[];
    const int KD = g.Kd;
    double2* As = sm2;               // [KD][TM+1]
    double2* Bs = sm2 + KD * (TM + 1);  // [KD][TN+1]
    const int64_t batch = blockIdx.z;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    for (int e = threadIdx.x; e < KD * TM; e += 256) {
        const int kk = e / TM, mm = e % TM;
        const int r = m0 + mm;
        As[kk * (TM + 1) + mm] = (r < g.M) ? load_op<KA>(g.A, g.tw, g.K, batch, r, kk) : make_double2(0.0, 0.0);
    }
    for (int e = threadIdx.x; e < KD * TN; e += 256) {
        const int kk = e / TN, nn = e % TN;
        const int c = n0 + nn;
        Bs[kk * (TN + 1) + nn] = (c < g.N) ? load_op<KB>(g.B, g.tw, g.K, batch, kk, c) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double2 acc[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j] = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int kk = 0; kk < KD; ++kk) {
        double2 a[2], b[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) a[i] = As[kk * (TM + 1) + ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = Bs[kk * (TN + 1) + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                acc[i][j].x = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, acc[i][j].x));
                acc[i][j].y = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, acc[i][j].y));
            }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = m0 + ty + 16 * i, c = n0 + tx + 16 * j;
            if (r >= g.M || c >= g.N) continue;
            const int64_t off = batch * g.c_bstride + (int64_t)r * g.ldc + c;
            double2 v = acc[i][j];
            if (EP == EP_C_MUL) {
                const double f = __ldg(g.fused + (int64_t)r * g.N + c);
                v.x *= f;
                v.y *= f;
            }
            if (EP == EP_REAL) reinterpret_cast<double*>(g.C)[off] = v.x;
            else reinterpret_cast<double2*>(g.C)[off] = v;
        }
}

template <int KA, int KB, int EP>
static void run_gemm(const GemmArgs& g, int batches, cudaStream_t st) {
    dim3 grid((g.N + TN - 1) / TN, (g.M + TM - 1) / TM, batches);
    const size_t smem = (size_t)g.Kd * (TM + 1 + TN + 1) * sizeof(double2);
    auto kern = cgemm_kernel<KA, KB, EP>;
    if (smem > 48 * 1024) ensure_max_smem((const void*)kern, smem);
    kern<<<grid, 256, smem, st>>>(g);
    note_launches(1);
}

static Operand op(const void* p, int64_t bstride, int ld, int koff = 0) {
    Operand o;
    o.p = p;
    o.bstride = bstride;
    o.ld = ld;
    o.koff = koff;
    return o;
}

// d <= 2: direct sub-box convolution out[u] = sum_u' Kc[u - u'] g[u'] with the
// host-computed real kernel (exactly the band-limited rfftn * fused * irfftn
// restricted to the active cells).  d = 2: one block per output row u0,
// threads = (u1, group of input rows); the groups combine in fixed order.
__global__ void conv2d_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                              const double* __restrict__ Kc, int L) {
    // one warp per output cell; lanes stride the input columns, the 32 lane
    // sums combine by a fixed shuffle tree -> deterministic.  The grid and the
    // kernel table arrive by TMA bulk copies.
    extern __shared__ __align__(16) double sm[];
    __shared__ uint64_t bar;
    const int KL = 2 * L - 1;
    const int gsz = (L * L + 1) & ~1;
    double* sg = sm;            // L*L input grid (padded to even)
    double* sk = sm + gsz;      // KL*KL kernel
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // the grid may be a caller buffer: bulk-copy whole 16-byte units, the
        // odd tail element separately; the kernel table is padded by the plan
        const uint32_t b1 = (uint32_t)((L * L * 8) & ~15), b2 = (uint32_t)(((KL * KL * 8) + 15) & ~15);
        mbar_arrive_expect_tx(&bar, b1 + b2);
        if (b1) tma_load_1d(sg, gin, b1, &bar);
        tma_load_1d(sk, Kc, b2, &bar);
        if ((L * L) & 1) sg[L * L - 1] = __ldg(gin + L * L - 1);
    }
    mbar_wait(&bar, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (o >= L * L) return;
    const int u0 = o / L, u1 = o % L;
    double s = 0.0;
    for (int v0 = 0; v0 < L; ++v0) {
        const double* kr = sk + (u0 - v0 + L - 1) * KL + (u1 + L - 1);
        const double* gr = sg + v0 * L;
        for (int v1 = lane; v1 < L; v1 += 32) s = fma(kr[-v1], gr[v1], s);
    }
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) gout[o] = s;
}

__global__ void conv1d_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                              const double* __restrict__ Kc, int L) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= L) return;
    double s = 0.0;
    for (int v = 0; v < L; ++v) s = fma(Kc[u - v + L - 1], gin[v], s);
    gout[u] = s;
}

// ---------------------------------------------------------------- d = 3 ----
// The six GEMM stages fused pairwise into three kernels; each stages the L x K
// twiddle table in shared memory:
//   F12 (u0, k2-tile):  slab g[u0] -> A1[u1][k2] (axis 2) -> A2[k1][k2] (axis 1)
//   F34 (column tile):  A2[u0][c] -> X[k0][c] * F -> Y[u0][c]   (axis 0 there and back)
//   F56 (u0, u1-tile):  Y[u0][k1][k2] -> w * A5[u1][k2] -> out[u0][u1][u2] (real)
struct F3Args {
    const double* grid;    // L^3 real
    double2* A2;           // [u0][K][Kh]
    double2* Y;            // [u0][K][Kh]
    double* out;           // L^3 real
    const double2* tw;     // L x K
    const double* fused;   // [K][K][Kh]
    int L, K, Kh, half;
};

constexpr int F12_T2 = 8;   // k2 columns per CTA
constexpr int F34_T = 16;   // (k1,k2) columns per CTA
constexpr int F56_T1 = 8;   // u1 rows per CTA

__device__ __forceinline__ void load_tw(double2* sE, const double2* tw, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) sE[i] = __ldg(reinterpret_cast<const double2*>(tw) + i);
}

__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
    return acc;
}
__device__ __forceinline__ double2 cmac_conj_a(double2 acc, double2 a, double2 b) {  // conj(a) * b
    acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
    return acc;
}

__global__ void __launch_bounds__(256) f12_kernel(F3Args p) {
    extern __shared__ double2 sm3[];
    const int L = p.L, K = p.K, Kh = p.Kh;
    double2* sE = sm3;                          // L*K
    double2* sA1 = sE + L * K;                  // L*T2
    double* sg = reinterpret_cast<double*>(sA1 + L * F12_T2);  // L*L
    __shared__ uint64_t bar;
    const int u0 = blockIdx.y;
    const int k2_0 = blockIdx.x * F12_T2;
    const int nt = min(F12_T2, Kh - k2_0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const double* slab = p.grid + (int64_t)u0 * L * L;
    for (int i = threadIdx.x; i < L * L; i += blockDim.x) cp_async8(sg + i, slab + i);
    tma_stage(sE, p.tw, (uint32_t)(L * K * 16), &bar, 0);
    cp_async_wait_all();
    __syncthreads();
    // A1[u1][j] = sum_u2 g[u1][u2] E[u2][k2_0 + j + half]
    for (int o = threadIdx.x; o < L * F12_T2; o += blockDim.x) {
        const int u1 = o / F12_T2, j = o % F12_T2;
        double2 acc = make_double2(0.0, 0.0);
        if (j < nt) {
            const int kc = k2_0 + j + p.half;
            double2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
            int u2 = 0;
            for (; u2 + 3 < L; u2 += 4) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const double gv = sg[u1 * L + u2 + r];
                    const double2 e = sE[(u2 + r) * K + kc];
                    q[r].x = fma(gv, e.x, q[r].x);
                    q[r].y = fma(gv, e.y, q[r].y);
                }
            }
            for (; u2 < L; ++u2) {
                const double gv = sg[u1 * L + u2];
                const double2 e = sE[u2 * K + kc];
                q[0].x = fma(gv, e.x, q[0].x);
                q[0].y = fma(gv, e.y, q[0].y);
            }
            acc.x = (q[0].x + q[1].x) + (q[2].x + q[3].x);
            acc.y = (q[0].y + q[1].y) + (q[2].y + q[3].y);
        }
        sA1[u1 * F12_T2 + j] = acc;
    }
    __syncthreads();
    // A2[k1][j] = sum_u1 E[u1][k1] A1[u1][j]
    double2* dst = p.A2 + (int64_t)u0 * K * Kh;
    for (int o = threadIdx.x; o < K * F12_T2; o += blockDim.x) {
        const int k1 = o / F12_T2, j = o % F12_T2;
        if (j >= nt) continue;
        double2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        int u1 = 0;
        for (; u1 + 3 < L; u1 += 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r) q[r] = cmac(q[r], sE[(u1 + r) * K + k1], sA1[(u1 + r) * F12_T2 + j]);
        }
        for (; u1 < L; ++u1) q[0] = cmac(q[0], sE[u1 * K + k1], sA1[u1 * F12_T2 + j]);
        dst[(int64_t)k1 * Kh + k2_0 + j] = make_double2((q[0].x + q[1].x) + (q[2].x + q[3].x),
                                                        (q[0].y + q[1].y) + (q[2].y + q[3].y));
    }
}

__global__ void __launch_bounds__(256) f34_kernel(F3Args p) {
    extern __shared__ double2 sm3[];
    const int L = p.L, K = p.K, Kh = p.Kh;
    const int ncol = K * Kh;
    double2* sE = sm3;               // L*K
    double2* sX = sE + L * K;        // L*T  input columns
    double2* sF = sX + L * F34_T;    // K*T  band columns
    __shared__ uint64_t bar;
    const int c0 = blockIdx.x * F34_T;
    const int nt = min(F34_T, ncol - c0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < L * F34_T; i += blockDim.x) {
        const int u0 = i / F34_T, t = i % F34_T;
        if (t < nt) cp_async16(sX + i, p.A2 + (int64_t)u0 * ncol + c0 + t);
        else sX[i] = make_double2(0.0, 0.0);
    }
    tma_stage(sE, p.tw, (uint32_t)(L * K * 16), &bar, 0);
    cp_async_wait_all();
    __syncthreads();
    // sF[k0][t] = F[k0][c] * sum_u0 E[u0][k0] X[u0][t]
    for (int o = threadIdx.x; o < K * F34_T; o += blockDim.x) {
        const int k0 = o / F34_T, t = o % F34_T;
        double2 acc = make_double2(0.0, 0.0);
        if (t < nt) {
            double2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
            int u0 = 0;
            for (; u0 + 3 < L; u0 += 4) {
#pragma unroll
                for (int r = 0; r < 4; ++r) q[r] = cmac(q[r], sE[(u0 + r) * K + k0], sX[(u0 + r) * F34_T + t]);
            }
            for (; u0 < L; ++u0) q[0] = cmac(q[0], sE[u0 * K + k0], sX[u0 * F34_T + t]);
            const double f = __ldg(p.fused + (int64_t)k0 * ncol + c0 + t);
            acc.x = ((q[0].x + q[1].x) + (q[2].x + q[3].x)) * f;
            acc.y = ((q[0].y + q[1].y) + (q[2].y + q[3].y)) * f;
        }
        sF[o] = acc;
    }
    __syncthreads();
    // Y[u0][t] = sum_k0 conj(E[u0][k0]) sF[k0][t]
    for (int o = threadIdx.x; o < L * F34_T; o += blockDim.x) {
        const int u0 = o / F34_T, t = o % F34_T;
        if (t >= nt) continue;
        double2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        int k0 = 0;
        for (; k0 + 3 < K; k0 += 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r) q[r] = cmac_conj_a(q[r], sE[u0 * K + k0 + r], sF[(k0 + r) * F34_T + t]);
        }
        for (; k0 < K; ++k0) q[0] = cmac_conj_a(q[0], sE[u0 * K + k0], sF[k0 * F34_T + t]);
        p.Y[(int64_t)u0 * ncol + c0 + t] = make_double2((q[0].x + q[1].x) + (q[2].x + q[3].x),
                                                        (q[0].y + q[1].y) + (q[2].y + q[3].y));
    }
}

__global__ void __launch_bounds__(256) f56_kernel(F3Args p) {
    extern __shared__ double2 sm3[];
    const int L = p.L, K = p.K, Kh = p.Kh;
    double2* sE = sm3;               // L*K
    double2* sB = sE + L * K;        // K*Kh slab
    double2* sA = sB + K * Kh;       // T1*Kh
    __shared__ uint64_t bar;
    const int u0 = blockIdx.y;
    const int u1_0 = blockIdx.x * F56_T1;
    const int nr = min(F56_T1, L - u1_0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const double2* slab = p.Y + (int64_t)u0 * K * Kh;
    if (threadIdx.x == 0) {
        const uint32_t b1 = (uint32_t)(L * K * 16), b2 = (uint32_t)(K * Kh * 16);
        mbar_arrive_expect_tx(&bar, b1 + b2);
        tma_load_1d(sE, p.tw, b1, &bar);
        tma_load_1d(sB, slab, b2, &bar);
    }
    mbar_wait(&bar, 0);
    // A5[i][k2] = w(k2) * sum_k1 conj(E[u1][k1]) B[k1][k2]
    for (int o = threadIdx.x; o < F56_T1 * Kh; o += blockDim.x) {
        const int i = o / Kh, k2 = o % Kh;
        double2 acc = make_double2(0.0, 0.0);
        if (i < nr) {
            const int u1 = u1_0 + i;
            double2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
            int k1 = 0;
            for (; k1 + 3 < K; k1 += 4) {
#pragma unroll
                for (int r = 0; r < 4; ++r) q[r] = cmac_conj_a(q[r], sE[u1 * K + k1 + r], sB[(k1 + r) * Kh + k2]);
            }
            for (; k1 < K; ++k1) q[0] = cmac_conj_a(q[0], sE[u1 * K + k1], sB[k1 * Kh + k2]);
            const double w = (k2 == 0) ? 1.0 : 2.0;
            acc.x = ((q[0].x + q[1].x) + (q[2].x + q[3].x)) * w;
            acc.y = ((q[0].y + q[1].y) + (q[2].y + q[3].y)) * w;
        }
        sA[o] = acc;
    }
    __syncthreads();
    // out[u0][u1][u2] = Re sum_k2 A5[i][k2] conj(E[u2][k2 + half])
    for (int o = threadIdx.x; o < F56_T1 * L; o += blockDim.x) {
        const int i = o / L, u2 = o % L;
        if (i >= nr) continue;
        double q[4] = {0, 0, 0, 0};
        int k2 = 0;
        for (; k2 + 3 < Kh; k2 += 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double2 a = sA[i * Kh + k2 + r];
                const double2 e = sE[u2 * K + k2 + r + p.half];
                q[r] = fma(a.x, e.x, fma(a.y, e.y, q[r]));
            }
        }
        for (; k2 < Kh; ++k2) {
            const double2 a = sA[i * Kh + k2];
            const double2 e = sE[u2 * K + k2 + p.half];
            q[0] = fma(a.x, e.x, fma(a.y, e.y, q[0]));
        }
        p.out[((int64_t)u0 * L + u1_0 + i) * L + u2] = (q[0] + q[1]) + (q[2] + q[3]);
    }
}

static size_t f12_smem(int L, int K) { return (size_t)(L * K + L * F12_T2) * 16 + (size_t)L * L * 8; }
static size_t f34_smem(int L, int K) { return (size_t)(L * K + L * F34_T + K * F34_T) * 16; }
static size_t f56_smem(int L, int K, int Kh) { return (size_t)(L * K + K * Kh + F56_T1 * Kh) * 16; }

static int convolve3_fused(mlb_binding* b, const double* gin, double* gout, cudaStream_t st) {
    const Geom& G = b->plan->g;
    F3Args p;
    p.grid = gin;
    p.A2 = reinterpret_cast<double2*>(b->stage_a);
    p.Y = reinterpret_cast<double2*>(b->stage_b);
    p.out = gout;
    p.tw = b->plan->twid;
    p.fused = b->plan->fused;
    p.L = G.L;
    p.K = G.K;
    p.Kh = G.Kh;
    p.half = G.N / 2;
    const size_t s12 = f12_smem(G.L, G.K), s34 = f34_smem(G.L, G.K), s56 = f56_smem(G.L, G.K, G.Kh);
    MLB_CUDA_TRY(cudaFuncSetAttribute(f12_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s12));
    MLB_CUDA_TRY(cudaFuncSetAttribute(f34_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s34));
    MLB_CUDA_TRY(cudaFuncSetAttribute(f56_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s56));
    f12_kernel<<<dim3((G.Kh + F12_T2 - 1) / F12_T2, G.L), 256, s12, st>>>(p);
    f34_kernel<<<(G.K * G.Kh + F34_T - 1) / F34_T, 256, s34, st>>>(p);
    f56_kernel<<<dim3((G.L + F56_T1 - 1) / F56_T1, G.L), 256, s56, st>>>(p);
    note_launches(3);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

// ------------------------------------------------------------ separable ----
// When the band weights are a rank-1 tensor F(k) = prod_a f(k_a) (Gaussian
// kernels whose regularised profile equals the Gaussian to rounding on the
// sampling cube; the host checks F against the product to 1e-13), the
// convolution is d one-dimensional passes out[..u..] = sum_v c[u-v] in[..v..]
// with the real kernel c[D] = sum_k f(k) cos(2 pi k D / ng).

// 4 consecutive outputs u0..u0+3 of one line: out[u] = sum_v c[u - v] x[v];
// the kernel taps slide through registers (2 shared loads per 4 FMAs)
__device__ __forceinline__ void sep_line4(const double* __restrict__ sc, int u0, const double* __restrict__ x,
                                          int L, int stride, double* o) {
    const double* cc = sc + L - 1 + u0;  // cc[j - v] = c[u0 + j - v]
    double w0 = cc[0], w1 = cc[1], w2 = cc[2], w3 = cc[3];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int v = 0; v < L; ++v) {
        const double xv = x[v * stride];
        s0 = fma(w0, xv, s0);
        s1 = fma(w1, xv, s1);
        s2 = fma(w2, xv, s2);
        s3 = fma(w3, xv, s3);
        w3 = w2;
        w2 = w1;
        w1 = w0;
        w0 = cc[-v - 1];
    }
    o[0] = s0;
    o[1] = s1;
    o[2] = s2;
    o[3] = s3;
}

// whole sub-box in smem, one CTA, all passes (d <= 2 and small grids)
__device__ __forceinline__ void sep_small_body(const double* __restrict__ gin, double* __restrict__ gout,
                                               const double* __restrict__ c, int L, int d) {
    extern __shared__ double sm[];
    const int cells = (d == 1) ? L : L * L;
    const int rows = cells / L;
    const int LQ = (L + 3) / 4;  // 4-output groups per line
    double* a = sm;
    double* b = sm + cells;
    double* sc = sm + 2 * cells;  // 2L-1 taps padded by 4 zeros on both sides
    for (int i = threadIdx.x; i < 2 * L + 7; i += blockDim.x) {
        const int k = i - 4;
        sc[i] = (k >= 0 && k < 2 * L - 1) ? __ldg(c + k) : 0.0;
    }
    pdl_wait();  // the grid comes from the reduction
    for (int i = threadIdx.x; i < cells; i += blockDim.x) a[i] = __ldg(gin + i);
    __syncthreads();
    const double* scp = sc + 4;
    // last axis
    for (int w = threadIdx.x; w < rows * LQ; w += blockDim.x) {
        const int r = w / LQ, q = w % LQ;
        double o[4];
        sep_line4(scp, 4 * q, a + r * L, L, 1, o);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * q + j < L) b[r * L + 4 * q + j] = o[j];
    }
    __syncthreads();
    if (d == 1) {
        for (int o = threadIdx.x; o < cells; o += blockDim.x) gout[o] = b[o];
        pdl_launch();
        return;
    }
    // first axis (d = 2)
    for (int w = threadIdx.x; w < L * LQ; w += blockDim.x) {
        const int col = w % L, q = w / L;
        double o[4];
        sep_line4(scp, 4 * q, b + col, L, L, o);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * q + j < L) gout[(4 * q + j) * L + col] = o[j];
    }
    pdl_launch();
}

__global__ void sep_small_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                                 const double* __restrict__ c, int L, int d) {
    sep_small_body(gin, gout, c, L, d);
}

// one CTA per layer of mlb_apply_multi (same L and d for every layer)
__global__ void sep_small_multi_kernel(const ConvJob* __restrict__ jobs, int L, int d) {
    const ConvJob& J = jobs[blockIdx.x];
    sep_small_body(J.gin, J.gout, J.c, L, d);
}

// one pass over a contiguous axis (rows of length L): CTA = 8 rows
__global__ void sep_rows_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                                const double* __restrict__ c, int L, int64_t rows) {
    extern __shared__ double sm[];
    constexpr int RB = 8;
    double* sr = sm;              // RB x L
    double* sc = sm + RB * L;     // 2L-1
    const int64_t r0 = (int64_t)blockIdx.x * RB;
    const int nr = (int)min((int64_t)RB, rows - r0);
    for (int i = threadIdx.x; i < nr * L; i += blockDim.x) cp_async8(sr + i, gin + r0 * L + i);
    for (int i = threadIdx.x; i < 2 * L - 1; i += blockDim.x) sc[i] = __ldg(c + i);
    cp_async_wait_all();
    __syncthreads();
    for (int o = threadIdx.x; o < nr * L; o += blockDim.x) {
        const int r = o / L, u = o % L;
        const double* cc = sc + u + L - 1;
        const double* x = sr + r * L;
        double q0 = 0.0, q1 = 0.0;
        int v = 0;
        for (; v + 1 < L; v += 2) {
            q0 = fma(cc[-v], x[v], q0);
            q1 = fma(cc[-v - 1], x[v + 1], q1);
        }
        if (v < L) q0 = fma(cc[-v], x[v], q0);
        gout[r0 * L + o] = q0 + q1;
    }
}

// one pass over a strided axis: data [A][L][B]; CTA = (a, 32 columns of B)
__global__ void sep_cols_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                                const double* __restrict__ c, int L, int B) {
    extern __shared__ double sm[];
    constexpr int BT = 32;
    double* st = sm;              // L x BT
    double* sc = sm + L * BT;     // 2L-1
    const int a = blockIdx.y;
    const int b0 = blockIdx.x * BT;
    const int nb = min(BT, B - b0);
    const double* base = gin + (int64_t)a * L * B + b0;
    for (int i = threadIdx.x; i < L * BT; i += blockDim.x) {
        const int v = i / BT, t = i % BT;
        if (t < nb) cp_async8(st + i, base + (int64_t)v * B + t);
    }
    for (int i = threadIdx.x; i < 2 * L - 1; i += blockDim.x) sc[i] = __ldg(c + i);
    cp_async_wait_all();
    __syncthreads();
    double* obase = gout + (int64_t)a * L * B + b0;
    for (int o = threadIdx.x; o < L * BT; o += blockDim.x) {
        const int u = o / BT, t = o % BT;
        if (t >= nb) continue;
        const double* cc = sc + u + L - 1;
        double q0 = 0.0, q1 = 0.0;
        int v = 0;
        for (; v + 1 < L; v += 2) {
            q0 = fma(cc[-v], st[v * BT + t], q0);
            q1 = fma(cc[-v - 1], st[(v + 1) * BT + t], q1);
        }
        if (v < L) q0 = fma(cc[-v], st[v * BT + t], q0);
        obase[(int64_t)u * B + t] = q0 + q1;
    }
}

// d = 3 in two launches: (a) one CTA per axis-0 slab: the L x L plane is
// convolved along axis 2 then axis 1 in shared memory; (b) one CTA per
// axis-1 index: the (axis 0, axis 2) plane is convolved along axis 0.
__device__ __forceinline__ double sep_line(const double* __restrict__ cc, const double* __restrict__ x, int L,
                                           int stride) {
    // sum_v cc[-v] x[v * stride], two chains
    double q0 = 0.0, q1 = 0.0;
    int v = 0;
    for (; v + 1 < L; v += 2) {
        q0 = fma(cc[-v], x[v * stride], q0);
        q1 = fma(cc[-v - 1], x[(v + 1) * stride], q1);
    }
    if (v < L) q0 = fma(cc[-v], x[v * stride], q0);
    return q0 + q1;
}

__global__ void __launch_bounds__(512) sep3_p21_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                                                       const double* __restrict__ c, int L) {
    extern __shared__ double sm[];
    const int LL = L * L;
    const int LQ = (L + 3) / 4;  // 4-output groups per line
    double* a = sm;                  // plane [u1][u2]
    double* b = sm + LL + 4 * L;     // after the axis-2 pass (padded rows)
    double* sc = b + LL + 4 * L;     // 2L-1 taps, padded by 4 on both sides with zeros
    const int64_t base = (int64_t)blockIdx.x * LL;
    for (int i = threadIdx.x; i < 2 * L + 7; i += blockDim.x) {
        const int k = i - 4;  // tap index
        sc[i] = (k >= 0 && k < 2 * L - 1) ? __ldg(c + k) : 0.0;
    }
    pdl_wait();  // the grid comes from the reduction
    for (int i = threadIdx.x; i < LL; i += blockDim.x) cp_async8(a + i, gin + base + i);
    cp_async_wait_all();
    __syncthreads();
    const double* scp = sc + 4;
    for (int w = threadIdx.x; w < L * LQ; w += blockDim.x) {  // axis 2: line u1, outputs 4q..4q+3
        const int u1 = w / LQ, q = w % LQ;
        double o[4];
        sep_line4(scp, 4 * q, a + u1 * L, L, 1, o);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * q + j < L) b[u1 * L + 4 * q + j] = o[j];
    }
    __syncthreads();
    for (int w = threadIdx.x; w < L * LQ; w += blockDim.x) {  // axis 1: column u2, outputs 4q..4q+3
        const int u2 = w % L, q = w / L;
        double o[4];
        sep_line4(scp, 4 * q, b + u2, L, L, o);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * q + j < L) gout[base + (4 * q + j) * L + u2] = o[j];
    }
    pdl_launch();
}

__global__ void __launch_bounds__(512) sep3_p0_kernel(const double* __restrict__ gin, double* __restrict__ gout,
                                                      const double* __restrict__ c, int L) {
    extern __shared__ double sm[];
    const int LL = L * L;
    const int LQ = (L + 3) / 4;
    double* a = sm;              // plane [u0][u2] at fixed u1
    double* sc = sm + LL + 4 * L;
    const int u1 = blockIdx.x;
    for (int i = threadIdx.x; i < 2 * L + 7; i += blockDim.x) {
        const int k = i - 4;
        sc[i] = (k >= 0 && k < 2 * L - 1) ? __ldg(c + k) : 0.0;
    }
    pdl_wait();  // the first pass
    for (int i = threadIdx.x; i < LL; i += blockDim.x) {
        const int u0 = i / L, u2 = i % L;
        cp_async8(a + i, gin + ((int64_t)u0 * L + u1) * L + u2);
    }
    cp_async_wait_all();
    __syncthreads();
    const double* scp = sc + 4;
    for (int w = threadIdx.x; w < L * LQ; w += blockDim.x) {  // axis 0: column u2, outputs 4q..4q+3
        const int u2 = w % L, q = w / L;
        double o[4];
        sep_line4(scp, 4 * q, a + u2, L, L, o);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * q + j < L) gout[((int64_t)(4 * q + j) * L + u1) * L + u2] = o[j];
    }
    pdl_launch();
}

static int convolve_separable(mlb_binding* b, const double* gin, double* gout, cudaStream_t st) {
    const Geom& G = b->plan->g;
    const int L = G.L, d = G.d;
    const double* c = b->plan->sep;
    const int64_t cells = b->grid_cells;
    if (d <= 2 && (2 * cells + 2 * L + 8) * 8 <= 96 * 1024) {
        const size_t smem = (size_t)(2 * cells + 2 * L + 8) * sizeof(double);
        MLB_CUDA_TRY(cudaFuncSetAttribute(sep_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        MLB_CUDA_TRY(launch_k(sep_small_kernel, dim3(1), dim3(512), smem, st, gin, gout, c, L, d));
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    if (d == 3 && (2 * (size_t)L * L + 16 * L) * 8 <= 200 * 1024) {
        const size_t s21 = (2 * (size_t)L * L + 8 * L + 2 * L + 8) * sizeof(double);
        const size_t s0 = ((size_t)L * L + 4 * L + 2 * L + 8) * sizeof(double);
        int rc = ensure_max_smem((const void*)sep3_p21_kernel, s21);  // per (kernel, device)
        if (rc == MLB_OK) rc = ensure_max_smem((const void*)sep3_p0_kernel, s0);
        if (rc != MLB_OK) return rc;
        MLB_CUDA_TRY(launch_k(sep3_p21_kernel, dim3(L), dim3(512), s21, st, gin, b->stage_a, c, L));
        MLB_CUDA_TRY(launch_k(sep3_p0_kernel, dim3(L), dim3(512), s0, st, (const double*)b->stage_a, gout, c, L));
        note_launches(2);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    // d passes: last axis (rows), then the strided axes; ping-pong via stage_a
    double* tmp = b->stage_a;
    const size_t srow = (size_t)(8 * L + 2 * L) * sizeof(double);
    const size_t scol = (size_t)(32 * L + 2 * L) * sizeof(double);
    const int64_t rows = cells / L;
    const double* src = gin;
    double* dst = (d == 1) ? gout : tmp;
    sep_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, srow, st>>>(src, dst, c, L, rows);
    note_launches(1);
    for (int ax = d - 2; ax >= 0; --ax) {
        int64_t A = 1, B = 1;
        for (int i = 0; i < ax; ++i) A *= L;
        for (int i = ax + 1; i < d; ++i) B *= L;
        src = dst;
        dst = (ax == 0) ? gout : (src == tmp ? b->stage_b : tmp);
        sep_cols_kernel<<<dim3((unsigned)((B + 31) / 32), (unsigned)A), 256, scol, st>>>(src, dst, c, L, (int)B);
        note_launches(1);
    }
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_sep_small_multi(const ConvJob* jobs_dev, int T, int L, int d, cudaStream_t st) {
    const int cells = (d == 1) ? L : L * L;
    const size_t smem = (size_t)(2 * cells + 2 * L + 8) * sizeof(double);
    if (int rc = ensure_max_smem((const void*)sep_small_multi_kernel, smem)) return rc;
    MLB_CUDA_TRY(launch_k(sep_small_multi_kernel, dim3(T), dim3(512), smem, st, jobs_dev, L, d));
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_convolve(mlb_binding* b, const double* gin, double* gout, cudaStream_t st) {
    const Geom& G = b->plan->g;
    if (b->plan->sep) return convolve_separable(b, gin, gout, st);
    if (b->plan->conv && G.d == 1) {
        conv1d_kernel<<<(G.L + 127) / 128, 128, 0, st>>>(gin, gout, b->plan->conv, G.L);
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    if (b->plan->conv && G.d == 2) {
        const size_t smem = ((size_t)((G.L * G.L + 1) & ~1) + (size_t)(2 * G.L - 1) * (2 * G.L - 1) + 2) *
                            sizeof(double);
        if (smem <= 200 * 1024) {
            MLB_CUDA_TRY(cudaFuncSetAttribute(conv2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem));
            const int outs = G.L * G.L;
            conv2d_kernel<<<(outs + 7) / 8, 256, smem, st>>>(gin, gout, b->plan->conv, G.L);
            note_launches(1);
            MLB_CUDA_TRY(cudaGetLastError());
            return MLB_OK;
        }
    }
    const int L = G.L, K = G.K, Kh = G.Kh, half = G.N / 2;
    const double2* tw = b->plan->twid;
    double* SA = b->stage_a;
    double* SB = b->stage_b;
    GemmArgs g;
    g.tw = tw;
    g.K = K;
    g.fused = b->plan->fused;
    if (G.d == 1) {
        // [u] -> [k] (k = 0..N/2) * F -> [u]
        g.A = op(gin, 0, L);
        g.B = op(nullptr, 0, 0, half);
        g.C = SA;
        g.c_bstride = 0;
        g.ldc = Kh;
        g.M = 1;
        g.N = Kh;
        g.Kd = L;
        run_gemm<OP_DATA_R, OP_TW, EP_C_MUL>(g, 1, st);
        g.A = op(SA, 0, Kh);
        g.B = op(nullptr, 0, 0, half);  // (k, u) = conj(E[u][k+half])
        g.C = gout;
        g.ldc = L;
        g.M = 1;
        g.N = L;
        g.Kd = Kh;
        run_gemm<OP_DATA_HW, OP_TWC_T, EP_REAL>(g, 1, st);
    } else if (G.d == 2) {
        // S1: [u0][u1] -> [u0][k1]          C = grid (L x L) . E (L x Kh)
        g.A = op(gin, 0, L);
        g.B = op(nullptr, 0, 0, half);
        g.C = SA;
        g.c_bstride = 0;
        g.ldc = Kh;
        g.M = L;
        g.N = Kh;
        g.Kd = L;
        run_gemm<OP_DATA_R, OP_TW, EP_C>(g, 1, st);
        // S2: [u0][k1] -> [k0][k1] * F      C = E^T (K x L) . S1 (L x Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SA, 0, Kh);
        g.C = SB;
        g.ldc = Kh;
        g.M = K;
        g.N = Kh;
        g.Kd = L;
        run_gemm<OP_TW_T, OP_DATA_C, EP_C_MUL>(g, 1, st);
        // S3: [k0][k1] -> [u0][k1]          C = conj(E) (L x K) . S2 (K x Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SB, 0, Kh);
        g.C = SA;
        g.ldc = Kh;
        g.M = L;
        g.N = Kh;
        g.Kd = K;
        run_gemm<OP_TWC, OP_DATA_C, EP_C>(g, 1, st);
        // S4: [u0][k1] -> [u0][u1] real     C = (S3 * w) (L x Kh) . conj(E)^T (Kh x L)
        g.A = op(SA, 0, Kh);
        g.B = op(nullptr, 0, 0, half);
        g.C = gout;
        g.ldc = L;
        g.M = L;
        g.N = L;
        g.Kd = Kh;
        run_gemm<OP_DATA_HW, OP_TWC_T, EP_REAL>(g, 1, st);
    } else {
        const size_t smax = std::max(f12_smem(L, K), std::max(f34_smem(L, K), f56_smem(L, K, Kh)));
        if (smax <= 200 * 1024) return convolve3_fused(b, gin, gout, st);
        const int64_t LL = (int64_t)L * L;
        // S1: [u0 u1][u2] -> [u0 u1][k2]
        g.A = op(gin, 0, L);
        g.B = op(nullptr, 0, 0, half);
        g.C = SA;
        g.c_bstride = 0;
        g.ldc = Kh;
        g.M = (int)LL;
        g.N = Kh;
        g.Kd = L;
        run_gemm<OP_DATA_R, OP_TW, EP_C>(g, 1, st);
        // S2: per u0: [u1][k2] -> [k1][k2]  C_b = E^T (K x L) . S1_b (L x Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SA, (int64_t)L * Kh, Kh);
        g.C = SB;
        g.c_bstride = (int64_t)K * Kh;
        g.ldc = Kh;
        g.M = K;
        g.N = Kh;
        g.Kd = L;
        run_gemm<OP_TW_T, OP_DATA_C, EP_C>(g, L, st);
        // S3: [u0][k1 k2] -> [k0][k1 k2] * F   C = E^T (K x L) . S2 (L x K*Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SB, 0, K * Kh);
        g.C = SA;
        g.c_bstride = 0;
        g.ldc = K * Kh;
        g.M = K;
        g.N = K * Kh;
        g.Kd = L;
        run_gemm<OP_TW_T, OP_DATA_C, EP_C_MUL>(g, 1, st);
        // S4: [k0][k1 k2] -> [u0][k1 k2]       C = conj(E) (L x K) . S3 (K x K*Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SA, 0, K * Kh);
        g.C = SB;
        g.ldc = K * Kh;
        g.M = L;
        g.N = K * Kh;
        g.Kd = K;
        run_gemm<OP_TWC, OP_DATA_C, EP_C>(g, 1, st);
        // S5: per u0: [k1][k2] -> [u1][k2]     C_b = conj(E) (L x K) . S4_b (K x Kh)
        g.A = op(nullptr, 0, 0, 0);
        g.B = op(SB, (int64_t)K * Kh, Kh);
        g.C = SA;
        g.c_bstride = (int64_t)L * Kh;
        g.ldc = Kh;
        g.M = L;
        g.N = Kh;
        g.Kd = K;
        run_gemm<OP_TWC, OP_DATA_C, EP_C>(g, L, st);
        // S6: [u0 u1][k2] -> [u0 u1][u2] real  C = (S5 * w) (L^2 x Kh) . conj(E)^T (Kh x L)
        g.A = op(SA, 0, Kh);
        g.B = op(nullptr, 0, 0, half);
        g.C = gout;
        g.c_bstride = 0;
        g.ldc = L;
        g.M = (int)LL;
        g.N = L;
        g.Kd = Kh;
        run_gemm<OP_DATA_HW, OP_TWC_T, EP_REAL>(g, 1, st);
    }
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

// Complex band DFT between the active sub-box (L^d cells) and the full band
// (K^d frequencies k = -N/2..N/2): the bare NFFT test hooks of the reference
// (nfft_adjoint / nfft_forward, fastsum.py:418-468) use it.
//   forward: out[k] = sum_u in[u] exp(-2 pi i k.u/ng)
//   inverse: out[u] = sum_k in[k] exp(+2 pi i k.u/ng)   (unnormalised)
int band_dft(mlb_binding* b, const double* in, double* out, int inverse, cudaStream_t st) {
    const Geom& G = b->plan->g;
    const int L = G.L, K = G.K, d = G.d;
    const int nin = inverse ? K : L, nout = inverse ? L : K;
    // ping-pong through the stage buffers (grown on demand: max(L,K)^d complex)
    const int64_t need = 2 * (int64_t)std::llround(std::pow((double)std::max(L, K), d));
    if (need > b->stage_elems) {
        cudaFree(b->stage_a);
        cudaFree(b->stage_b);
        b->stage_a = b->stage_b = nullptr;
        MLB_CUDA_TRY(cudaMalloc((void**)&b->stage_a, need * sizeof(double)));
        MLB_CUDA_TRY(cudaMalloc((void**)&b->stage_b, need * sizeof(double)));
        b->stage_elems = need;
    }
    GemmArgs g;
    g.tw = b->plan->twid;
    g.K = K;
    g.fused = nullptr;
    const double* cur = in;
    // row-major [n0]..[n_{d-1}]: transform the last axis first; the data is
    // viewed as [before][nin][after] -> [before][nout][after]
    int64_t before = 1, after = 1;
    for (int i = 1; i < d; ++i) before *= nin;
    double* bufs[2] = {b->stage_a, b->stage_b};
    for (int step = 0; step < d; ++step) {
        double* dst = (step == d - 1) ? out : bufs[step & 1];
        if (after == 1) {
            g.A = op(cur, 0, nin);
            g.B = op(nullptr, 0, 0, 0);
            g.C = dst;
            g.c_bstride = 0;
            g.ldc = nout;
            g.M = (int)before;
            g.N = nout;
            g.Kd = nin;
            if (inverse) run_gemm<OP_DATA_C, OP_TWC_T, EP_C>(g, 1, st);   // (k,u) = conj(E[u][k])
            else run_gemm<OP_DATA_C, OP_TW, EP_C>(g, 1, st);              // (u,k) = E[u][k]
        } else {
            g.A = op(nullptr, 0, 0, 0);
            g.B = op(cur, (int64_t)nin * after, (int)after);
            g.C = dst;
            g.c_bstride = (int64_t)nout * after;
            g.ldc = (int)after;
            g.M = nout;
            g.N = (int)after;
            g.Kd = nin;
            if (inverse) run_gemm<OP_TWC, OP_DATA_C, EP_C>(g, (int)before, st);   // (u,k) = conj(E[u][k])
            else run_gemm<OP_TW_T, OP_DATA_C, EP_C>(g, (int)before, st);          // (k,u) = E[u][k]
        }
        cur = dst;
        after *= nout;
        if (step < d - 1) before /= nin;
    }
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

}  // namespace mlb

extern "C" int mlb_band_dft(mlb_binding* b, const double* in_dev, double* out_dev, int inverse, void* stream) {
    if (!b || !in_dev || !out_dev) return mlb::fail(MLB_ERR_ARG, "null argument");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != b->plan->device) cudaSetDevice(b->plan->device);
    const int rc = mlb::band_dft(b, in_dev, out_dev, inverse, (cudaStream_t)stream);
    if (dev != b->plan->device) cudaSetDevice(dev);
    return rc;
}
