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

namespace mlb {

constexpr int kAcMaxM = 32;     // classes
constexpr int kAcRows = 128;    // rows per tile
constexpr int kAcBlocks = 296;  // fixed partition (2 x SMs)

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

__global__ void ac_finish_kernel(const double* __restrict__ partial, int nb, int k, int m,
                                 const double* __restrict__ denom, double* __restrict__ Vc) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= k * m) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[(int64_t)b * k * m + o];
    Vc[o] = s / denom[o / m];
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
    if (threadIdx.x != 0) return;
    double md = 0.0, mu = 0.0;
    for (int b = 0; b < nb; ++b) {
        md = fmax(md, mx_partial[2 * b]);
        mu = fmax(mu, mx_partial[2 * b + 1]);
    }
    stats[0] = md;
    stats[1] = mu;
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

}  // namespace mlb

using namespace mlb;

extern "C" {

int64_t mlb_ac_work_size(int64_t n, int k, int m) {
    (void)n;
    return (int64_t)kAcBlocks * k * m + 2 * kAcBlocks + (int64_t)k * m;
}

int mlb_ac_step(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                const double* denom, double c_dt, double dt_2eps, double dt, double* U_next, double* stats,
                double* work, void* stream) {
    if (m < 2 || m > kAcMaxM) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels support 2 <= m <= 32 classes");
    if (k < 1 || k * m > 16 * 256) return fail(MLB_ERR_CONFIG, "Allen-Cahn kernels need k*m <= 4096");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kAcBlocks, (n + kAcRows - 1) / kAcRows));
    double* partial = work;
    double* mx = work + (int64_t)kAcBlocks * k * m;
    double* Vc = mx + 2 * kAcBlocks;
    const size_t sm1 = (size_t)kAcRows * (m + k) * sizeof(double);
    MLB_CUDA_TRY(cudaFuncSetAttribute(ac_rhs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    ac_rhs_kernel<<<nb, 256, sm1, st>>>(Phi, n, k, m, U, F, fid, c_dt, dt_2eps, dt, partial);
    note_launches(1);
    ac_finish_kernel<<<(k * m + 127) / 128, 128, 0, st>>>(partial, nb, k, m, denom, Vc);
    note_launches(1);
    ac_update_kernel<<<nb, 256, (size_t)k * m * sizeof(double), st>>>(Phi, n, k, m, Vc, U, U_next, mx);
    note_launches(1);
    ac_max_finish<<<1, 32, 0, st>>>(mx, nb, stats);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_argmax_rows(const double* U, int64_t n, int m, int32_t* labels, void* stream) {
    if (n <= 0) return MLB_OK;
    int64_t b = std::min<int64_t>((n + 255) / 256, 148 * 16);
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
