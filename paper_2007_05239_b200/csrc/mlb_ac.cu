// Multiclass Allen-Cahn convexity-splitting step in the eigenbasis
// (allencahn.py:172-223), plus argmax labels (allencahn.py:226-229) and the
// exact O(n^2) kernel sum (direct_apply, fastsum.py:500-553).
//
// One iteration = 3 kernels:
//   ac_rhs_project : per row, the well force T(U) (allencahn.py:127-154), R,
//                    and this block's fixed-order partial of Phi^T R (k x m);
//   ac_finish      : Vc = (sum of block partials in order) / denom;
//   ac_update      : per row U_next = proj_simplex(Phi Vc) (allencahn.py:105-124)
//                    and per-block maxima of |dU_i|^2 and |U_next_i|^2.
#include <cuda_runtime.h>

#include <algorithm>

#include "mlb_internal.cuh"
#include "mlb_tma.cuh"

namespace mlb {

constexpr int kAcMaxM = 32;     // classes
constexpr int kAcRows = 128;    // rows per tile
constexpr int kAcBlocks = 148 * 6;  // partition capacity (6 CTAs per B200 SM); launches use <= this

// well force for one row (m <= kAcMaxM), leave-one-out products as the reference
__device__ void well_force_row(const double* u, int m, double* t) {
    double asum = 0.0;
    for (int q = 0; q < m; ++q) asum += fabs(u[q]);
    double A[kAcMaxM], B[kAcMaxM];
    for (int q = 0; q < m; ++q) {
        A[q] = asum - fabs(u[q]) + fabs(u[q] - 1.0);
        B[q] = 0.25 * A[q] * A[q];
    }
    // left[q] = prod_{l<q} B[l] ; right[q] = prod_{l>q} B[l]
    double left[kAcMaxM];
    double acc = 1.0;
    for (int q = 0; q < m; ++q) {
        left[q] = acc;
        acc *= B[q];
    }
    double wsum = 0.0;
    double right = 1.0;
    double wt[kAcMaxM];
    for (int q = m - 1; q >= 0; --q) {
        wt[q] = A[q] * (left[q] * right);
        right *= B[q];
    }
    for (int q = 0; q < m; ++q) wsum += wt[q];
    for (int q = 0; q < m; ++q) t[q] = 0.5 * wsum - wt[q];
}

// block b owns rows [b*per, (b+1)*per); partial[b][a*m + c] = sum_i Phi[i][a] R[i][c]
__global__ void ac_rhs_kernel(const double* __restrict__ Phi, int64_t n, int k, int m, const double* __restrict__ U,
                              const double* __restrict__ F, const double* __restrict__ fid, double c_dt,
                              double dt_2eps, double dt, double* __restrict__ partial) {
    extern __shared__ double sm[];
    double* Rt = sm;                       // kAcRows x m
    double* Pt = sm + kAcRows * m;         // kAcRows x k
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int nout = k * m;
    // each thread owns outputs o = threadIdx.x + j*blockDim.x
    constexpr int kMaxOut = 16;
    double acc[kMaxOut];
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) acc[j] = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kAcRows) {
        const int rows = (int)min((int64_t)kAcRows, r1 - t0);
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            const int64_t i = t0 + r;
            double u[kAcMaxM], t[kAcMaxM];
            for (int q = 0; q < m; ++q) u[q] = U[i * m + q];
            well_force_row(u, m, t);
            const double fi = fid[i];
            for (int q = 0; q < m; ++q)
                Rt[r * m + q] = c_dt * u[q] - dt_2eps * t[q] - dt * fi * (u[q] - F[i * m + q]);
        }
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = Phi[t0 * k + e];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kMaxOut; ++j) {
            const int o = threadIdx.x + j * blockDim.x;
            if (o < nout) {
                const int a = o / m, c = o % m;
                double s = acc[j];
                for (int r = 0; r < rows; ++r) s = fma(Pt[r * k + a], Rt[r * m + c], s);
                acc[j] = s;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) {
        const int o = threadIdx.x + j * blockDim.x;
        if (o < nout) partial[(int64_t)blockIdx.x * nout + o] = acc[j];
    }
}

// ---- register-resident row kernels (m <= MM, MM in {4, 8, 16, 32}) -------
template <int MM>
__device__ __forceinline__ void well_force_t(const double* u, int m, double* t) {
    double asum = 0.0;
#pragma unroll
    for (int q = 0; q < MM; ++q)
        if (q < m) asum += fabs(u[q]);
    double A[MM], B[MM];
#pragma unroll
    for (int q = 0; q < MM; ++q) {
        A[q] = (q < m) ? asum - fabs(u[q]) + fabs(u[q] - 1.0) : 0.0;
        B[q] = (q < m) ? 0.25 * A[q] * A[q] : 1.0;
    }
    double left[MM];
    double acc = 1.0;
#pragma unroll
    for (int q = 0; q < MM; ++q) {
        left[q] = acc;
        if (q < m) acc *= B[q];
    }
    double wt[MM];
    double right = 1.0;
#pragma unroll
    for (int q = MM - 1; q >= 0; --q) {
        if (q < m) {
            wt[q] = A[q] * (left[q] * right);
            right *= B[q];
        } else {
            wt[q] = 0.0;
        }
    }
    double wsum = 0.0;
#pragma unroll
    for (int q = 0; q < MM; ++q)
        if (q < m) wsum += wt[q];
#pragma unroll
    for (int q = 0; q < MM; ++q) t[q] = 0.5 * wsum - wt[q];
}

// descending bitonic sort of MM register values (padding = -inf sorts last)
template <int MM>
__device__ __forceinline__ void sort_desc(double* s) {
#pragma unroll
    for (int size = 2; size <= MM; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
            for (int i = 0; i < MM; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = ((i & size) == 0);
                    const double x = s[i], y = s[j];
                    const bool sw = desc ? (x < y) : (x > y);
                    s[i] = sw ? y : x;
                    s[j] = sw ? x : y;
                }
            }
}

// rhs: R rows from staged U / F tiles, then Phi^T R with every thread busy
// (4 x 8 output tiles x row groups, fixed-order group reduction)
template <int MM>
__global__ void __launch_bounds__(256, 2) ac_rhs3_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                                      const double* __restrict__ U, const double* __restrict__ F,
                                                      const double* __restrict__ fid, double c_dt, double dt_2eps,
                                                      double dt, double* __restrict__ partial) {
    extern __shared__ double sm[];
    constexpr int T = 256;
    double* Pt = sm;              // T x k
    double* Ut = Pt + T * k;      // T x m (U, then R in place)
    double* Ft = Ut + T * m;      // T x m
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    constexpr int TC = MM < 8 ? MM : 8;  // output tile: 4 rows of Phi^T x TC classes
    const int ta = (k + 3) / 4, tc = (m + TC - 1) / TC;
    const int NO = ta * tc, NG = blockDim.x / NO;
    const int o = threadIdx.x % NO, g = threadIdx.x / NO;
    const bool live = g < NG;
    const int a0 = (o / tc) * 4, c0 = (o % tc) * TC;
    double acc[4][TC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) acc[i][j] = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += T) {
        const int rows = (int)min((int64_t)T, r1 - t0);
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = __ldg(Phi + t0 * k + e);
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) {
            Ut[e] = __ldg(U + t0 * m + e);
            Ft[e] = __ldg(F + t0 * m + e);
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            const int r = threadIdx.x;
            double u[MM], t[MM];
#pragma unroll
            for (int q = 0; q < MM; ++q) u[q] = (q < m) ? Ut[r * m + q] : 0.0;
            well_force_t<MM>(u, m, t);
            const double fi = __ldg(fid + t0 + r);
#pragma unroll
            for (int q = 0; q < MM; ++q)
                if (q < m) Ut[r * m + q] = c_dt * u[q] - dt_2eps * t[q] - dt * fi * (u[q] - Ft[r * m + q]);
        }
        __syncthreads();
        if (live) {
            for (int r = g; r < rows; r += NG) {
                double pa[4], rc[TC];
#pragma unroll
                for (int i = 0; i < 4; ++i) pa[i] = (a0 + i < k) ? Pt[r * k + a0 + i] : 0.0;
#pragma unroll
                for (int j = 0; j < TC; ++j) rc[j] = (c0 + j < m) ? Ut[r * m + c0 + j] : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < TC; ++j) acc[i][j] = fma(pa[i], rc[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
    double* red = sm;  // NG * NO * 4 * TC <= 256 * 32 doubles
    if (live)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < TC; ++j) red[((size_t)g * NO + o) * (4 * TC) + i * TC + j] = acc[i][j];
    __syncthreads();
    const int nout = k * m;
    for (int e = threadIdx.x; e < nout; e += blockDim.x) {
        const int a = e / m, c = e % m;
        const int oo = (a / 4) * tc + c / TC, slot = (a % 4) * TC + (c % TC);
        double sum = 0.0;
        for (int gg = 0; gg < NG; ++gg) sum += red[((size_t)gg * NO + oo) * (4 * TC) + slot];
        partial[(int64_t)blockIdx.x * nout + e] = sum;
    }
}

// update: U_next = proj_simplex(Phi Vc) per row from staged Phi / U tiles,
// written back through shared memory (coalesced), plus the stopping maxima
template <int MM>
__global__ void __launch_bounds__(256) ac_update3_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                                         const double* __restrict__ Vc,
                                                         const double* __restrict__ U, double* __restrict__ Un,
                                                         double* __restrict__ mx_partial) {
    extern __shared__ double sm[];
    constexpr int T = 256;
    double* vsh = sm;                 // k x m
    double* Pt = vsh + ((k * m + 1) & ~1);  // T x k
    double* Ut = Pt + T * k;          // T x m (U, then U_next in place)
    __shared__ double sh_d[8], sh_u[8];
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) vsh[e] = Vc[e];
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double md = 0.0, mu = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += T) {
        const int rows = (int)min((int64_t)T, r1 - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = __ldg(Phi + t0 * k + e);
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) Ut[e] = __ldg(U + t0 * m + e);
        __syncthreads();
        if (threadIdx.x < rows) {
            const int r = threadIdx.x;
            double y[MM];
#pragma unroll
            for (int c = 0; c < MM; ++c) y[c] = 0.0;
            for (int a = 0; a < k; ++a) {
                const double p = Pt[r * k + a];
#pragma unroll
                for (int c = 0; c < MM; ++c)
                    if (c < m) y[c] = fma(p, vsh[a * m + c], y[c]);
            }
            double s[MM];
#pragma unroll
            for (int c = 0; c < MM; ++c) s[c] = (c < m) ? y[c] : -INFINITY;
            sort_desc<MM>(s);
            double cs = 0.0, cs_rho = 0.0;
            int rho = 0;
#pragma unroll
            for (int j = 0; j < MM; ++j) {
                if (j < m) {
                    cs += s[j];
                    if (s[j] + (1.0 - cs) / (j + 1) > 0) {
                        rho = j;
                        cs_rho = cs;
                    }
                }
            }
            const double tau = (1.0 - cs_rho) / (rho + 1);
            double dd = 0.0, uu = 0.0;
#pragma unroll
            for (int c = 0; c < MM; ++c) {
                if (c < m) {
                    const double v = fmax(y[c] + tau, 0.0);
                    const double df = v - Ut[r * m + c];
                    dd = fma(df, df, dd);
                    uu = fma(v, v, uu);
                    Ut[r * m + c] = v;
                }
            }
            md = fmax(md, dd);
            mu = fmax(mu, uu);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) Un[t0 * m + e] = Ut[e];
    }
    for (int o = 16; o > 0; o >>= 1) {
        md = fmax(md, __shfl_down_sync(0xffffffffu, md, o));
        mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh_d[w] = md;
        sh_u[w] = mu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            md = fmax(md, sh_d[i]);
            mu = fmax(mu, sh_u[i]);
        }
        mx_partial[2 * blockIdx.x] = md;
        mx_partial[2 * blockIdx.x + 1] = mu;
    }
}

// One pass over Phi per iteration: the update of iteration t (U -> U_next)
// and the right-hand side of iteration t+1 (R(U_next), Phi^T R) share the
// staged Phi tile.  Per tile: stage Phi, U, F; per row: y = Phi_i Vc,
// simplex projection, the stopping maxima, then R(U_next); write U_next;
// accumulate Phi^T R in register tiles (the same partition and order as
// ac_rhs3, so the iterates are those of the two-pass step).
template <int MM>
__global__ void __launch_bounds__(256, 2) ac_fused_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                                          const double* __restrict__ Vc,
                                                          const double* __restrict__ U,
                                                          const double* __restrict__ F,
                                                          const double* __restrict__ fid, double c_dt,
                                                          double dt_2eps, double dt, double* __restrict__ Un,
                                                          double* __restrict__ mx_partial,
                                                          double* __restrict__ partial) {
    extern __shared__ double sm[];
    constexpr int T = 256;
    constexpr int TC = MM < 8 ? MM : 8;
    // two stage buffers (tile t computes while tile t+1 loads by cp.async)
    double* vsh = sm;                               // k x m
    double* Rt = vsh + ((k * m + 1) & ~1);          // T x m
    double* buf0 = Rt + T * m;                      // [Pt T x k | Ut T x m | Ft T x m]
    const int bstride = T * (k + 2 * m);
    __shared__ double sh_d[8], sh_u[8];
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) vsh[e] = Vc[e];
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int ta = (k + 3) / 4, tc = (m + TC - 1) / TC;
    const int NO = ta * tc, NG = blockDim.x / NO;
    const int o = threadIdx.x % NO, g = threadIdx.x / NO;
    const bool live = g < NG;
    const int a0 = (o / tc) * 4, c0 = (o % tc) * TC;
    double acc[4][TC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) acc[i][j] = 0.0;
    double md = 0.0, mu = 0.0;
    auto stage = [&](int64_t ts, double* bf) {
        const int rows = (int)min((int64_t)T, r1 - ts);
        double* P = bf;
        double* Uu = bf + T * k;
        double* Ff = Uu + T * m;
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) cp_async8(P + e, Phi + ts * k + e);
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) {
            cp_async8(Uu + e, U + ts * m + e);
            cp_async8(Ff + e, F + ts * m + e);
        }
        cp_async_commit();
    };
    if (r0 < r1) stage(r0, buf0);
    int bsel = 0;
    for (int64_t t0 = r0; t0 < r1; t0 += T) {
        const int rows = (int)min((int64_t)T, r1 - t0);
        double* Pt = buf0 + bsel * bstride;
        double* Ut = Pt + T * k;
        double* Ft = Ut + T * m;
        cp_async_wait_all();
        __syncthreads();  // tile t landed; the previous tile's readers are done
        if (t0 + T < r1) stage(t0 + T, buf0 + (bsel ^ 1) * bstride);
        if (threadIdx.x < rows) {
            const int r = threadIdx.x;
            double y[MM];
#pragma unroll
            for (int c = 0; c < MM; ++c) y[c] = 0.0;
            for (int a = 0; a < k; ++a) {
                const double p = Pt[r * k + a];
#pragma unroll
                for (int c = 0; c < MM; ++c)
                    if (c < m) y[c] = fma(p, vsh[a * m + c], y[c]);
            }
            double s[MM];
#pragma unroll
            for (int c = 0; c < MM; ++c) s[c] = (c < m) ? y[c] : -INFINITY;
            sort_desc<MM>(s);
            double cs = 0.0, cs_rho = 0.0;
            int rho = 0;
#pragma unroll
            for (int j = 0; j < MM; ++j) {
                if (j < m) {
                    cs += s[j];
                    if (s[j] + (1.0 - cs) / (j + 1) > 0) {
                        rho = j;
                        cs_rho = cs;
                    }
                }
            }
            const double tau = (1.0 - cs_rho) / (rho + 1);
            double un[MM];
            double dd = 0.0, uu = 0.0;
#pragma unroll
            for (int c = 0; c < MM; ++c) {
                un[c] = (c < m) ? fmax(y[c] + tau, 0.0) : 0.0;
                if (c < m) {
                    const double df = un[c] - Ut[r * m + c];
                    dd = fma(df, df, dd);
                    uu = fma(un[c], un[c], uu);
                    Ut[r * m + c] = un[c];
                }
            }
            md = fmax(md, dd);
            mu = fmax(mu, uu);
            // next iteration's right-hand side row
            double t[MM];
            well_force_t<MM>(un, m, t);
            const double fi = __ldg(fid + t0 + r);
#pragma unroll
            for (int q = 0; q < MM; ++q)
                if (q < m) Rt[r * m + q] = c_dt * un[q] - dt_2eps * t[q] - dt * fi * (un[q] - Ft[r * m + q]);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) Un[t0 * m + e] = Ut[e];
        if (live) {
            for (int r = g; r < rows; r += NG) {
                double pa[4], rc[TC];
#pragma unroll
                for (int i = 0; i < 4; ++i) pa[i] = (a0 + i < k) ? Pt[r * k + a0 + i] : 0.0;
#pragma unroll
                for (int j = 0; j < TC; ++j) rc[j] = (c0 + j < m) ? Rt[r * m + c0 + j] : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < TC; ++j) acc[i][j] = fma(pa[i], rc[j], acc[i][j]);
            }
        }
        bsel ^= 1;
    }
    cp_async_wait_all();
    __syncthreads();
    double* red = sm;
    if (live)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < TC; ++j) red[((size_t)g * NO + o) * (4 * TC) + i * TC + j] = acc[i][j];
    for (int off = 16; off > 0; off >>= 1) {
        md = fmax(md, __shfl_down_sync(0xffffffffu, md, off));
        mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, off));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh_d[w] = md;
        sh_u[w] = mu;
    }
    __syncthreads();
    const int nout = k * m;
    for (int e = threadIdx.x; e < nout; e += blockDim.x) {
        const int a = e / m, c = e % m;
        const int oo = (a / 4) * tc + c / TC, slot = (a % 4) * TC + (c % TC);
        double sum = 0.0;
        for (int gg = 0; gg < NG; ++gg) sum += red[((size_t)gg * NO + oo) * (4 * TC) + slot];
        partial[(int64_t)blockIdx.x * nout + e] = sum;
    }
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            md = fmax(md, sh_d[i]);
            mu = fmax(mu, sh_u[i]);
        }
        mx_partial[2 * blockIdx.x] = md;
        mx_partial[2 * blockIdx.x + 1] = mu;
    }
}

// Phi^T R with every thread busy: per tile of kTile rows the CTA stages Phi
// (a linear, coalesced copy: Phi is row-major) and R (one row per thread) in
// shared memory; thread t then owns a 4 x 8 output tile o = t % NO and a row
// group g = t / NO, accumulating its rows in registers; the NG group partials
// of each output meet in a fixed order at the end (deterministic).
constexpr int kTile = 256;
__global__ void __launch_bounds__(256) ac_rhs2_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                                      const double* __restrict__ U, const double* __restrict__ F,
                                                      const double* __restrict__ fid, double c_dt, double dt_2eps,
                                                      double dt, double* __restrict__ partial) {
    extern __shared__ double sm[];
    double* Pt = sm;                  // kTile x k
    double* Rt = sm + kTile * k;      // kTile x m (reused for the group reduction)
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int ta = (k + 3) / 4, tc = (m + 7) / 8;
    const int NO = ta * tc, NG = blockDim.x / NO;
    const int o = threadIdx.x % NO, g = threadIdx.x / NO;
    const bool live = g < NG;
    const int a0 = (o / tc) * 4, c0 = (o % tc) * 8;
    double acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kTile) {
        const int rows = (int)min((int64_t)kTile, r1 - t0);
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = __ldg(Phi + t0 * k + e);
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            const int64_t i = t0 + r;
            double u[kAcMaxM], t[kAcMaxM];
            for (int q = 0; q < m; ++q) u[q] = U[i * m + q];
            well_force_row(u, m, t);
            const double fi = fid[i];
            for (int q = 0; q < m; ++q) Rt[r * m + q] = c_dt * u[q] - dt_2eps * t[q] - dt * fi * (u[q] - F[i * m + q]);
        }
        __syncthreads();
        if (live) {
            for (int r = g; r < rows; r += NG) {
                double pa[4], rc[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) pa[i] = (a0 + i < k) ? Pt[r * k + a0 + i] : 0.0;
#pragma unroll
                for (int j = 0; j < 8; ++j) rc[j] = (c0 + j < m) ? Rt[r * m + c0 + j] : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fma(pa[i], rc[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
    // group reduction in fixed order: red[g][o][32]
    double* red = sm;  // NG * NO * 32 <= 256 * 32 doubles
    if (live)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) red[((size_t)g * NO + o) * 32 + i * 8 + j] = acc[i][j];
    __syncthreads();
    const int nout = k * m;
    for (int e = threadIdx.x; e < nout; e += blockDim.x) {
        const int a = e / m, c = e % m;
        const int oo = (a / 4) * tc + c / 8, slot = (a % 4) * 8 + (c % 8);
        double sum = 0.0;
        for (int gg = 0; gg < NG; ++gg) sum += red[((size_t)gg * NO + oo) * 32 + slot];
        partial[(int64_t)blockIdx.x * nout + e] = sum;
    }
}

// one warp per output: lanes sum strided block partials, then a fixed
// shuffle tree (deterministic; no serial 296-long chain)
__global__ void ac_finish_kernel(const double* __restrict__ partial, int nb, int k, int m,
                                 const double* __restrict__ denom, double* __restrict__ Vc) {
    const int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (o >= k * m) return;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += partial[(int64_t)b * k * m + o];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) Vc[o] = denom ? s / denom[o / m] : s;  // (no denom: the plain sum, sharded partials)
}

__global__ void ac_update_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                 const double* __restrict__ Vc, const double* __restrict__ U,
                                 double* __restrict__ Un, double* __restrict__ mx_partial) {
    extern __shared__ double vsh[];
    __shared__ double sh_d[32], sh_u[32];
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) vsh[e] = Vc[e];
    __syncthreads();
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double md = 0.0, mu = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        double y[kAcMaxM];
        for (int c = 0; c < m; ++c) y[c] = 0.0;
        for (int a = 0; a < k; ++a) {
            const double p = Phi[i * k + a];
            for (int c = 0; c < m; ++c) y[c] = fma(p, vsh[a * m + c], y[c]);
        }
        // simplex projection: sort descending, largest prefix with s_j + (1-cs_j)/(j+1) > 0
        double s[kAcMaxM];
        for (int c = 0; c < m; ++c) s[c] = y[c];
        for (int a = 1; a < m; ++a) {
            const double x = s[a];
            int b = a - 1;
            while (b >= 0 && s[b] < x) {
                s[b + 1] = s[b];
                --b;
            }
            s[b + 1] = x;
        }
        double cs = 0.0, cs_rho = 0.0;
        int rho = 0;
        for (int j = 0; j < m; ++j) {
            cs += s[j];
            if (s[j] + (1.0 - cs) / (j + 1) > 0) {
                rho = j;
                cs_rho = cs;
            }
        }
        const double tau = (1.0 - cs_rho) / (rho + 1);
        double dd = 0.0, uu = 0.0;
        for (int c = 0; c < m; ++c) {
            const double v = fmax(y[c] + tau, 0.0);
            const double df = v - U[i * m + c];
            dd = fma(df, df, dd);
            uu = fma(v, v, uu);
            Un[i * m + c] = v;
        }
        md = fmax(md, dd);
        mu = fmax(mu, uu);
    }
    for (int o = 16; o > 0; o >>= 1) {
        md = fmax(md, __shfl_down_sync(0xffffffffu, md, o));
        mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh_d[w] = md;
        sh_u[w] = mu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            md = fmax(md, sh_d[i]);
            mu = fmax(mu, sh_u[i]);
        }
        mx_partial[2 * blockIdx.x] = md;
        mx_partial[2 * blockIdx.x + 1] = mu;
    }
}

__global__ void ac_max_finish(const double* __restrict__ mx_partial, int nb, double* __restrict__ stats) {
    // one warp: strided maxima then a shuffle tree (max is order-independent)
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    double md = 0.0, mu = 0.0;
    for (int b = lane; b < nb; b += 32) {
        md = fmax(md, mx_partial[2 * b]);
        mu = fmax(mu, mx_partial[2 * b + 1]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        md = fmax(md, __shfl_down_sync(0xffffffffu, md, off));
        mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, off));
    }
    if (lane == 0) {
        stats[0] = md;
        stats[1] = mu;
    }
}

// ---- binary scheme (allencahn.py:261-309): scalar scores u = Phi v ------
// partial[b][a] = sum_i Phi[i][a] u_i^3, partial[b][k + a] = sum_i Phi[i][a] fid_i (u_i - f_i)
__global__ void bac_rhs_kernel(const double* __restrict__ Phi, int64_t n, int k, const double* __restrict__ u,
                               const double* __restrict__ f, const double* __restrict__ fid,
                               double* __restrict__ partial) {
    extern __shared__ double sm[];
    double* X = sm;                  // kAcRows x 2
    double* Pt = sm + 2 * kAcRows;   // kAcRows x k
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int o = threadIdx.x;  // output: a = o % k, which = o / k
    const bool live = o < 2 * k;
    const int a = o % k, which = o / k;
    double acc = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kAcRows) {
        const int rows = (int)min((int64_t)kAcRows, r1 - t0);
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            const double ui = u[t0 + r];
            X[2 * r] = ui * ui * ui;
            X[2 * r + 1] = fid[t0 + r] * (ui - f[t0 + r]);
        }
        for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = Phi[t0 * k + e];
        __syncthreads();
        if (live)
            for (int r = 0; r < rows; ++r) acc = fma(Pt[r * k + a], X[2 * r + which], acc);
        __syncthreads();
    }
    if (live) partial[(int64_t)blockIdx.x * 2 * k + o] = acc;
}

__global__ void bac_finish_kernel(const double* __restrict__ partial, int nb, int k, const double* __restrict__ v,
                                  const double* __restrict__ denom, double lead, double dt_eps, double dt,
                                  double* __restrict__ v_next) {
    // one warp per coefficient: strided block partials + a fixed shuffle tree
    const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (a >= k) return;
    double g1 = 0.0, g2 = 0.0;
    for (int b = lane; b < nb; b += 32) {
        g1 += partial[(int64_t)b * 2 * k + a];
        g2 += partial[(int64_t)b * 2 * k + k + a];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        g1 += __shfl_down_sync(0xffffffffu, g1, off);
        g2 += __shfl_down_sync(0xffffffffu, g2, off);
    }
    if (lane == 0) {
        double rhs = lead * v[a];
        rhs -= dt_eps * g1;
        rhs -= dt * g2;
        v_next[a] = rhs / denom[a];
    }
}

__global__ void bac_update_kernel(const double* __restrict__ Phi, int64_t n, int k, const double* __restrict__ v,
                                  const double* __restrict__ u, double* __restrict__ un,
                                  double* __restrict__ mx_partial) {
    extern __shared__ double vsh[];
    __shared__ double sh_d[32], sh_u[32];
    for (int e = threadIdx.x; e < k; e += blockDim.x) vsh[e] = v[e];
    __syncthreads();
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double md = 0.0, mu = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        double y = 0.0;
        for (int a = 0; a < k; ++a) y = fma(Phi[i * k + a], vsh[a], y);
        const double df = y - u[i];
        md = fmax(md, df * df);
        mu = fmax(mu, y * y);
        un[i] = y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        md = fmax(md, __shfl_down_sync(0xffffffffu, md, o));
        mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh_d[w] = md;
        sh_u[w] = mu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            md = fmax(md, sh_d[i]);
            mu = fmax(mu, sh_u[i]);
        }
        mx_partial[2 * blockIdx.x] = md;
        mx_partial[2 * blockIdx.x + 1] = mu;
    }
}

// ---- Ginzburg-Landau energy partials (allencahn.py:232-252) -------------
// partial[b] = [ C_b (k x m: sum_i Phi[i][a] U[i][c]) | well_b | fid_b ] with
// well = sum_i prod_q (0.25 A_iq^2), fid = sum_i fid_i |F_i - U_i|^2
__global__ void gl_energy_kernel(const double* __restrict__ Phi, int64_t n, int k, int m,
                                 const double* __restrict__ U, const double* __restrict__ F,
                                 const double* __restrict__ fid, double* __restrict__ partial) {
    extern __shared__ double sm[];
    double* Ut = sm;                 // kAcRows x m
    double* Pt = sm + kAcRows * m;   // kAcRows x k
    __shared__ double red[2][256];
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int nout = k * m;
    constexpr int kMaxOut = 16;
    double acc[kMaxOut];
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) acc[j] = 0.0;
    double well = 0.0, fsum = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kAcRows) {
        const int rows = (int)min((int64_t)kAcRows, r1 - t0);
        for (int e = threadIdx.x; e < rows * m; e += blockDim.x) Ut[e] = U[t0 * m + e];
        if (Phi)
            for (int e = threadIdx.x; e < rows * k; e += blockDim.x) Pt[e] = Phi[t0 * k + e];
        __syncthreads();
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            const int64_t i = t0 + r;
            double asum = 0.0;
            for (int q = 0; q < m; ++q) asum += fabs(Ut[r * m + q]);
            double prod = 1.0, dd = 0.0;
            for (int q = 0; q < m; ++q) {
                const double uq = Ut[r * m + q];
                const double A = asum - fabs(uq) + fabs(uq - 1.0);
                prod *= 0.25 * A * A;
                const double df = F[i * m + q] - uq;
                dd = fma(df, df, dd);
            }
            well += prod;
            fsum += fid[i] * dd;
        }
        if (Phi) {
#pragma unroll
            for (int j = 0; j < kMaxOut; ++j) {
                const int o = threadIdx.x + j * blockDim.x;
                if (o < nout) {
                    const int a = o / m, c = o % m;
                    double s = acc[j];
                    for (int r = 0; r < rows; ++r) s = fma(Pt[r * k + a], Ut[r * m + c], s);
                    acc[j] = s;
                }
            }
        }
        __syncthreads();
    }
    double* out = partial + (int64_t)blockIdx.x * (nout + 2);
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) {
        const int o = threadIdx.x + j * blockDim.x;
        if (o < nout) out[o] = acc[j];
    }
    // fixed-order block sums of the per-thread well / fidelity terms
    red[0][threadIdx.x] = well;
    red[1][threadIdx.x] = fsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double w = 0.0, fs = 0.0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            w += red[0][t];
            fs += red[1][t];
        }
        out[nout] = w;
        out[nout + 1] = fs;
    }
}

__global__ void argmax_kernel(const double* __restrict__ U, int64_t n, int m, int32_t* __restrict__ lab) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int best = 0;
        double bv = U[i * m];
        for (int c = 1; c < m; ++c) {
            const double x = U[i * m + c];
            if (x > bv) {
                bv = x;
                best = c;
            }
        }
        lab[i] = best;
    }
}

// exact kernel sums: y_i = alpha v_i + s_i (beta sum_j K(|x_i-x_j|) s_j v_j + gamma s_i v_i)
// (the j = i term K(0) s_i v_i is inside the sum, as in direct_apply before its
// final "- K0 v"); points row-major n x d in device memory.
__global__ void direct_kernel(const double* __restrict__ X, int64_t n, int d, int family, double inv_sigma,
                              const double* __restrict__ v, const double* __restrict__ s, double* __restrict__ y,
                              double alpha, double beta, double gamma, int accumulate) {
    extern __shared__ double tile[];  // 128 x (d + 1)
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double xi[16];
    const bool live = i < n;
    const int dd = d < 16 ? d : 16;
    for (int a = 0; a < dd; ++a) xi[a] = live ? X[i * d + a] : 0.0;
    double acc = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += 128) {
        const int cnt = (int)min((int64_t)128, n - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const int64_t j = j0 + e;
            for (int a = 0; a < d; ++a) tile[e * (d + 1) + a] = X[j * d + a];
            tile[e * (d + 1) + d] = v[j] * (s ? s[j] : 1.0);
        }
        __syncthreads();
        if (live) {
            for (int e = 0; e < cnt; ++e) {
                double r2 = 0.0;
                for (int a = 0; a < d; ++a) {
                    const double xa = (a < 16) ? xi[a] : X[i * d + a];
                    const double df = (xa - tile[e * (d + 1) + a]) * inv_sigma;
                    r2 = fma(df, df, r2);
                }
                const double kv = (family == 0) ? exp(-r2) : exp(-sqrt(r2));
                acc = fma(kv, tile[e * (d + 1) + d], acc);
            }
        }
    }
    if (live) {
        const double si = s ? s[i] : 1.0;
        double r = alpha * v[i] + si * (beta * acc + gamma * si * v[i]);
        if (accumulate) r += y[i];
        y[i] = r;
    }
}

// exact sums at a target subset (the accuracy check of run_fastsum_bench,
// runner.py:496-512, on a 2,000-target sample of up to 10^7 sources): block
// (bx, sy) sums sources [sy*chunk, (sy+1)*chunk) for targets bx*128.. into
// partial[sy * nt + t]; direct_targets_finish sums the slices in slice order
__global__ void direct_targets_kernel(const double* __restrict__ X, int64_t n, int d, int family, double inv_sigma,
                                      const double* __restrict__ v, const double* __restrict__ Xt, int64_t nt,
                                      int64_t chunk, double* __restrict__ partial) {
    extern __shared__ double tile[];  // 128 x (d + 1)
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = t < nt;
    double xt[16];
    const int dd = d < 16 ? d : 16;
    for (int a = 0; a < dd; ++a) xt[a] = live ? Xt[t * d + a] : 0.0;
    const int64_t s0 = blockIdx.y * chunk, s1 = min(n, s0 + chunk);
    double acc = 0.0;
    for (int64_t j0 = s0; j0 < s1; j0 += 128) {
        const int cnt = (int)min((int64_t)128, s1 - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            for (int a = 0; a < d; ++a) tile[e * (d + 1) + a] = X[(j0 + e) * d + a];
            tile[e * (d + 1) + d] = v[j0 + e];
        }
        __syncthreads();
        if (live)
            for (int e = 0; e < cnt; ++e) {
                double r2 = 0.0;
                for (int a = 0; a < d; ++a) {
                    const double xa = (a < 16) ? xt[a] : Xt[t * d + a];
                    const double df = (xa - tile[e * (d + 1) + a]) * inv_sigma;
                    r2 = fma(df, df, r2);
                }
                acc = fma((family == 0) ? exp(-r2) : exp(-sqrt(r2)), tile[e * (d + 1) + d], acc);
            }
    }
    if (live) partial[(int64_t)blockIdx.y * nt + t] = acc;
}

__global__ void direct_targets_finish(const double* __restrict__ partial, int slices, int64_t nt,
                                      double* __restrict__ yt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    double acc = 0.0;
    for (int sl = 0; sl < slices; ++sl) acc += partial[(int64_t)sl * nt + t];
    yt[t] = acc;
}

}  // namespace mlb

using namespace mlb;

extern "C" {

int64_t mlb_direct_targets_work_size(int64_t nt) { return 1024 * nt; }

int mlb_direct_targets(const double* X, int64_t n, int d, int family, double sigma, const double* v, const double* Xt,
                       int64_t nt, double* yt, double* work, void* stream) {
    if (nt <= 0) return MLB_OK;
    if (d < 1 || d > 4096) return fail(MLB_ERR_CONFIG, "direct kernel needs 1 <= d <= 4096");
    const size_t smem = (size_t)128 * (d + 1) * sizeof(double);
    if (smem > 200 * 1024) return fail(MLB_ERR_CONFIG, "direct kernel: d too large for the smem tile");
    if (int rc = ensure_max_smem((const void*)direct_targets_kernel, smem)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t tx = (nt + 127) / 128;
    // enough source slices to fill the GPU several times over (<= 1024 slices)
    int64_t slices = std::max<int64_t>(1, std::min<int64_t>(1024, (int64_t)device_sms() * 8 / std::max<int64_t>(tx, 1)));
    slices = std::min<int64_t>(slices, std::max<int64_t>(1, (n + 127) / 128));
    const int64_t chunk = (n + slices - 1) / slices;
    direct_targets_kernel<<<dim3((unsigned)tx, (unsigned)slices), 128, smem, st>>>(X, n, d, family, 1.0 / sigma, v, Xt,
                                                                                    nt, chunk, work);
    direct_targets_finish<<<(unsigned)tx, 128, 0, st>>>(work, (int)slices, nt, yt);
    note_launches(2);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int64_t mlb_ac_work_size(int64_t n, int k, int m) {
    (void)n;  // (m = 1: the binary scheme's 2k partials + maxima fit as well)
    return (int64_t)kAcBlocks * k * std::max(m, 2) + 2 * kAcBlocks + (int64_t)k * std::max(m, 2);
}

int mlb_ac_step(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                const double* denom, double c_dt, double dt_2eps, double dt, double* U_next, double* stats,
                double* work, void* stream) {
    if (m < 2 || m > kAcMaxM) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels support 2 <= m <= 32 classes");
    if (k < 1 || k * m > 16 * 256) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels need k*m <= 4096");
    cudaStream_t st = (cudaStream_t)stream;
    // row partition: ~1k rows per CTA, between one and six CTAs per SM
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(
        (n + kAcRows - 1) / kAcRows, std::min<int64_t>(kAcBlocks, std::max<int64_t>(device_sms(), n / 1024))));
    double* partial = work;
    double* mx = work + (int64_t)kAcBlocks * k * m;
    double* Vc = mx + 2 * kAcBlocks;
    const size_t sm1 = std::max((size_t)256 * (k + 2 * m), (size_t)256 * 32) * sizeof(double);
    const size_t sm3 = ((size_t)((k * m + 1) & ~1) + (size_t)256 * (k + m)) * sizeof(double);
    if (std::max(sm1, sm3) > 200 * 1024) return fail(MLB_ERR_CONFIG, "Allen-Cahn tiles too large (k, m)");
    auto run = [&](auto rhs, auto upd) -> int {
        MLB_CUDA_TRY(cudaFuncSetAttribute(rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
        MLB_CUDA_TRY(cudaFuncSetAttribute(upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
        rhs<<<nb, 256, sm1, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
        ac_finish_kernel<<<(k * m * 32 + 255) / 256, 256, 0, st>>>(partial, nb, k, m, denom, Vc);
        upd<<<nb, 256, sm3, st>>>(Phi, n, k, m, Vc, U, U_next, mx);
        return MLB_OK;
    };
    int rc;
    if (m <= 4) {
        rc = run(ac_rhs3_kernel<4>, ac_update3_kernel<4>);
    } else if (m <= 8) {
        rc = run(ac_rhs3_kernel<8>, ac_update3_kernel<8>);
    } else {
        // many classes: the register-resident row kernels would spill; generic kernels
        const size_t sm2 = std::max((size_t)kTile * (m + k), (size_t)256 * 32) * sizeof(double);
        MLB_CUDA_TRY(cudaFuncSetAttribute(ac_rhs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
        ac_rhs2_kernel<<<nb, 256, sm2, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
        ac_finish_kernel<<<(k * m * 32 + 255) / 256, 256, 0, st>>>(partial, nb, k, m, denom, Vc);
        ac_update_kernel<<<nb, 256, (size_t)k * m * sizeof(double), st>>>(Phi, n, k, m, Vc, U, U_next, mx);
        rc = MLB_OK;
    }
    if (rc != MLB_OK) return rc;
    note_launches(3);
    ac_max_finish<<<1, 32, 0, st>>>(mx, nb, stats);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_ac_rhs_partial(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                       double c_dt, double dt_2eps, double dt, double* PtR, double* work, void* stream) {
    if (m < 2 || m > kAcMaxM) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels support 2 <= m <= 32 classes");
    if (k < 1 || k * m > 16 * 256) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels need k*m <= 4096");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        MLB_CUDA_TRY(cudaMemsetAsync(PtR, 0, (size_t)k * m * sizeof(double), st));
        return MLB_OK;
    }
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(
        (n + kAcRows - 1) / kAcRows, std::min<int64_t>(kAcBlocks, std::max<int64_t>(device_sms(), n / 1024))));
    double* partial = work;
    const size_t sm1 = std::max((size_t)256 * (k + 2 * m), (size_t)256 * 32) * sizeof(double);
    const size_t sm2 = std::max((size_t)kTile * (m + k), (size_t)256 * 32) * sizeof(double);
    if (sm1 > 200 * 1024 || sm2 > 200 * 1024) return fail(MLB_ERR_CONFIG, "Allen-Cahn tiles too large (k, m)");
    if (m <= 8) {
        auto rhs = m <= 4 ? ac_rhs3_kernel<4> : ac_rhs3_kernel<8>;
        if (int rc = ensure_max_smem((const void*)rhs, sm1)) return rc;
        rhs<<<nb, 256, sm1, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
    } else {
        if (int rc = ensure_max_smem((const void*)ac_rhs2_kernel, sm2)) return rc;
        ac_rhs2_kernel<<<nb, 256, sm2, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
    }
    ac_finish_kernel<<<(k * m * 32 + 255) / 256, 256, 0, st>>>(partial, nb, k, m, nullptr, PtR);
    note_launches(2);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_ac_update_from(const double* Phi, int64_t n, int k, int m, const double* PtR, const double* denom,
                       const double* U, double* U_next, double* stats, double* work, void* stream) {
    if (m < 2 || m > kAcMaxM) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels support 2 <= m <= 32 classes");
    if (k < 1 || k * m > 16 * 256) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels need k*m <= 4096");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(
        (n + kAcRows - 1) / kAcRows, std::min<int64_t>(kAcBlocks, std::max<int64_t>(device_sms(), n / 1024))));
    double* mx = work + (int64_t)kAcBlocks * k * m;
    double* Vc = mx + 2 * kAcBlocks;
    ac_finish_kernel<<<(k * m * 32 + 255) / 256, 256, 0, st>>>(PtR, 1, k, m, denom, Vc);
    note_launches(1);
    if (n == 0) {
        MLB_CUDA_TRY(cudaMemsetAsync(stats, 0, 2 * sizeof(double), st));
        return MLB_OK;
    }
    const size_t sm3 = ((size_t)((k * m + 1) & ~1) + (size_t)256 * (k + m)) * sizeof(double);
    if (m <= 8) {
        auto upd = m <= 4 ? ac_update3_kernel<4> : ac_update3_kernel<8>;
        if (sm3 > 200 * 1024) return fail(MLB_ERR_CONFIG, "Allen-Cahn tiles too large (k, m)");
        if (int rc = ensure_max_smem((const void*)upd, sm3)) return rc;
        upd<<<nb, 256, sm3, st>>>(Phi, n, k, m, Vc, U, U_next, mx);
    } else {
        ac_update_kernel<<<nb, 256, (size_t)k * m * sizeof(double), st>>>(Phi, n, k, m, Vc, U, U_next, mx);
    }
    ac_max_finish<<<1, 32, 0, st>>>(mx, nb, stats);
    note_launches(2);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_ac_step2(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                 const double* denom, double c_dt, double dt_2eps, double dt, int first, double* U_next,
                 double* stats, double* work, void* stream) {
    if (m > 8) {  // many classes: the two-pass step
        return mlb_ac_step(Phi, n, k, m, U, F, fid, denom, c_dt, dt_2eps, dt, U_next, stats, work, stream);
    }
    if (m < 2) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels support 2 <= m <= 32 classes");
    if (k < 1 || k * m > 16 * 256) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels need k*m <= 4096");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(
        (n + kAcRows - 1) / kAcRows, std::min<int64_t>(kAcBlocks, std::max<int64_t>(device_sms(), n / 1024))));
    double* partial = work;
    double* mx = work + (int64_t)kAcBlocks * k * m;
    double* Vc = mx + 2 * kAcBlocks;
    const size_t sm1 = std::max((size_t)256 * (k + 2 * m), (size_t)256 * 32) * sizeof(double);
    const size_t smf = std::max((size_t)((k * m + 1) & ~1) + (size_t)256 * (2 * k + 5 * m), (size_t)256 * 32) *
                       sizeof(double);
    if (std::max(sm1, smf) > 200 * 1024) return fail(MLB_ERR_CONFIG, "Allen-Cahn tiles too large (k, m)");
    auto run = [&](auto rhs, auto fused) -> int {
        if (first) {  // R(U_0) and Phi^T R once; afterwards the fused kernel provides them
            MLB_CUDA_TRY(cudaFuncSetAttribute(rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
            rhs<<<nb, 256, sm1, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
            note_launches(1);
        }
        MLB_CUDA_TRY(cudaFuncSetAttribute(fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf));
        ac_finish_kernel<<<(k * m * 32 + 255) / 256, 256, 0, st>>>(partial, nb, k, m, denom, Vc);
        fused<<<nb, 256, smf, st>>>(Phi, n, k, m, Vc, U, F, fid, c_dt, dt_2eps, dt, U_next, mx, partial);
        ac_max_finish<<<1, 32, 0, st>>>(mx, nb, stats);
        note_launches(3);
        return MLB_OK;
    };
    const int rc = (m <= 4) ? run(ac_rhs3_kernel<4>, ac_fused_kernel<4>) : run(ac_rhs3_kernel<8>, ac_fused_kernel<8>);
    if (rc != MLB_OK) return rc;
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_bac_step(const double* Phi, int64_t n, int k, const double* u, const double* f, const double* fid,
                 const double* v, const double* denom, double lead, double dt_eps, double dt, double* v_next,
                 double* u_next, double* stats, double* work, void* stream) {
    if (k < 1 || 2 * k > 256) return fail(MLB_ERR_CONFIG, "binary Allen-Cahn kernels need 1 <= k <= 128");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kAcBlocks, (n + kAcRows - 1) / kAcRows));
    double* partial = work;                       // nb x 2k
    double* mx = work + (int64_t)kAcBlocks * 2 * k;  // 2 x nb
    const size_t sm1 = (size_t)kAcRows * (2 + k) * sizeof(double);
    MLB_CUDA_TRY(cudaFuncSetAttribute(bac_rhs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    bac_rhs_kernel<<<nb, 256, sm1, st>>>(Phi, n, k, u, f, fid, partial);
    bac_finish_kernel<<<(k * 32 + 255) / 256, 256, 0, st>>>(partial, nb, k, v, denom, lead, dt_eps, dt, v_next);
    bac_update_kernel<<<nb, 256, (size_t)k * sizeof(double), st>>>(Phi, n, k, v_next, u, u_next, mx);
    ac_max_finish<<<1, 32, 0, st>>>(mx, nb, stats);
    note_launches(4);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int64_t mlb_gl_energy_work_size(int k, int m) { return (int64_t)kAcBlocks * ((int64_t)k * m + 2); }

int mlb_gl_energy_partials(const double* Phi, int64_t n, int k, int m, const double* U, const double* F,
                           const double* fid, double* partial, int* nblocks, void* stream) {
    if (m < 1 || m > kAcMaxM) return fail(MLB_ERR_CONFIG, "energy kernels support m <= 32 classes");
    if (Phi && (k < 1 || k * m > 16 * 256)) return fail(MLB_ERR_CONFIG, "energy kernels need k*m <= 4096");
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kAcBlocks, (n + kAcRows - 1) / kAcRows));
    if (nblocks) *nblocks = nb;
    const size_t sm1 = (size_t)kAcRows * (m + (Phi ? k : 0)) * sizeof(double);
    MLB_CUDA_TRY(cudaFuncSetAttribute(gl_energy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    gl_energy_kernel<<<nb, 256, sm1, (cudaStream_t)stream>>>(Phi, n, Phi ? k : 0, m, U, F, fid, partial);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_argmax_rows(const double* U, int64_t n, int m, int32_t* labels, void* stream) {
    if (n <= 0) return MLB_OK;
    int64_t b = std::min<int64_t>((n + 255) / 256, (int64_t)device_sms() * 16);
    argmax_kernel<<<(int)b, 256, 0, (cudaStream_t)stream>>>(U, n, m, labels);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_direct(const double* X, int64_t n, int d, int family, double sigma, const double* v, const double* s,
               double* y, double alpha, double beta, double gamma, int accumulate, void* stream) {
    if (n <= 0) return MLB_OK;
    if (d < 1 || d > 4096) return fail(MLB_ERR_CONFIG, "direct kernel needs 1 <= d <= 4096");
    const size_t smem = (size_t)128 * (d + 1) * sizeof(double);
    if (smem > 200 * 1024) return fail(MLB_ERR_CONFIG, "direct kernel: d too large for the smem tile");
    MLB_CUDA_TRY(cudaFuncSetAttribute(direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    direct_kernel<<<(unsigned)((n + 127) / 128), 128, smem, (cudaStream_t)stream>>>(
        X, n, d, family, 1.0 / sigma, v, s, y, alpha, beta, gamma, accumulate);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

}  // extern "C"
