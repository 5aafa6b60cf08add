// Krylov vector kernels: tall-skinny GEMV (V^T w, V c), CGS2, restart GEMM,
// dot products, axpby, elementwise.  Replaces the OpenBLAS calls of
// krylov.py:65-71 (CGS2), :147 / :160 (restart V S), :208 (y = V c).
//
// All reductions are two-level with a FIXED partition of rows into blocks and
// a fixed-order final sum, so repeated runs are bitwise identical (the
// reference pins seed determinism: test_krylov.py:62-71).  V is column-major:
// column j starts at V + j*ld (coalesced reads down each column).
#include <cuda_runtime.h>

#include <algorithm>

#include "mlb_internal.cuh"

namespace mlb {

constexpr int kRedThreads = 256;
constexpr int kMaxRowBlocks = 256;
constexpr int kFusedBlocks = 296;  // CGS2 row-block capacity (2 per B200 SM); launches use min(this, 2 x SMs)

static int row_blocks(int64_t n) {
    int64_t b = (n + 2047) / 2048;
    if (b > kMaxRowBlocks) b = kMaxRowBlocks;
    return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    return s;  // valid in thread 0
}

// partial[j * nb + blockIdx.x] = sum_{rows of block} V[j][i] w[i]; grid (nb, cols)
__global__ void gemv_t_partial(const double* __restrict__ V, int64_t ld, int64_t n, const double* __restrict__ w,
                               double* __restrict__ partial) {
    __shared__ double sh[32];
    const int nb = gridDim.x, j = blockIdx.y;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const double* col = V + (int64_t)j * ld;
    double s = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) s = fma(col[i], w[i], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[(int64_t)j * nb + blockIdx.x] = s;
}

// out[j] = sum_b partial[j*nb + b] (+ add[j])
__global__ void finish_partial(const double* __restrict__ partial, int nb, int cols, double* __restrict__ out,
                               const double* __restrict__ add) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[(int64_t)j * nb + b];
    if (add) s += add[j];
    out[j] = s;
}

// y[i] (=|+=) scale * sum_j V[j][i] c[j]; optional per-block partial of y_new^2
__global__ void gemv_n_kernel(const double* __restrict__ V, int64_t ld, int64_t n, int cols,
                              const double* __restrict__ c, double* __restrict__ y, double scale, int accumulate,
                              double* __restrict__ nrm_partial) {
    extern __shared__ double csh[];
    __shared__ double sh[32];
    for (int j = threadIdx.x; j < cols; j += blockDim.x) csh[j] = c[j];
    __syncthreads();
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double ss = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < cols; ++j) acc = fma(V[(int64_t)j * ld + i], csh[j], acc);
        const double r = accumulate ? fma(scale, acc, y[i]) : scale * acc;
        y[i] = r;
        ss = fma(r, r, ss);
    }
    if (nrm_partial) {
        ss = block_sum(ss, sh);
        if (threadIdx.x == 0) nrm_partial[blockIdx.x] = ss;
    }
}

__global__ void dot_partial(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            double* __restrict__ partial) {
    __shared__ double sh[32];
    const int nb = gridDim.x;
    const int64_t per = (n + nb - 1) / nb;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double s = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) s = fma(x[i], y[i], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (b == 0.0) ? a * x[i] : fma(a, x[i], b * y[i]);
}

__global__ void scale_by_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n,
                                const double* __restrict__ s, double pw) {
    const double f = (pw == -0.5) ? 1.0 / sqrt(s[0]) : pow(s[0], pw);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] * f;
}

__global__ void hadamard_kernel(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ z,
                                int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        z[i] = x[i] * y[i];
}

// Out[:, j] = sum_l V[:, l] S[l, j]: 64-row x 32-col tiles, K-steps of 16 via smem.
__global__ void gemm_vs_kernel(const double* __restrict__ V, int64_t ld, int64_t n, int s,
                               const double* __restrict__ S, int k, double* __restrict__ Out, int64_t ldo) {
    __shared__ double Vt[16][65];
    __shared__ double St[16][33];
    const int64_t row0 = blockIdx.x * 64;
    const int col0 = blockIdx.y * 32;
    const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;  // 16 x 16 threads, each 4 rows x 2 cols
    double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int l0 = 0; l0 < s; l0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += blockDim.x) {
            const int l = e / 64, r = e % 64;
            const int64_t gi = row0 + r;
            Vt[l][r] = (l0 + l < s && gi < n) ? V[(int64_t)(l0 + l) * ld + gi] : 0.0;
        }
        for (int e = threadIdx.x; e < 16 * 32; e += blockDim.x) {
            const int l = e / 32, c = e % 32;
            St[l][c] = (l0 + l < s && col0 + c < k) ? S[(int64_t)(col0 + c) * s + l0 + l] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int l = 0; l < 16; ++l) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) acc[a][b] = fma(Vt[l][tr + 16 * a], St[l][tc + 16 * b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int64_t gi = row0 + tr + 16 * a;
            const int c = col0 + tc + 16 * b;
            if (gi < n && c < k) Out[(int64_t)c * ldo + gi] = acc[a][b];
        }
}

// ---- CGS2 for cols <= 64: 4 bandwidth passes, 4 launches -----------------
// Row blocks are a FIXED partition of the rows (nb blocks of contiguous
// rows, multiples of 4); a thread owns 4 consecutive rows of a 1024-row tile
// and reads them as two 16-byte loads per column, a warp covering 1 KB of a
// column per load pair; 4 columns are in flight per step.  Every sum has a
// fixed order (4 rows, fixed shuffle tree, tiles in order, warps in order,
// blocks in order by warp-per-column finishes that every block repeats
// identically): bitwise reproducible.  Needs an even leading dimension and
// 16-byte aligned V / w (checked by the launcher).
constexpr int kTileRows = 1024;

__device__ __forceinline__ void ld4(const double* p, bool ok, double* v) {
    if (ok) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
        v[0] = v[1] = v[2] = v[3] = 0.0;
    }
}

// part[j * nb + b] = sum over block b's rows of V[j][i] w[i]
__device__ __forceinline__ void cgs_dot_block(const double* __restrict__ V, int64_t ld, int64_t n, int cols,
                                              const double* __restrict__ w, double* __restrict__ part) {
    __shared__ double acc[8][64];  // per warp, per column (tiles accumulate in order)
    const int nb = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = ((n + nb - 1) / nb + 3) & ~(int64_t)3;
    const int64_t r0 = min(n, blockIdx.x * per), r1 = min(n, r0 + per);
    for (int j = threadIdx.x; j < 8 * 64; j += blockDim.x) (&acc[0][0])[j] = 0.0;
    __syncthreads();
    for (int64_t t0 = r0; t0 < r1; t0 += kTileRows) {
        const int64_t i0 = t0 + 4 * threadIdx.x;
        const bool full = i0 + 3 < r1;
        double wr[4];
        if (full) {
            ld4(w + i0, true, wr);
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) wr[r] = (i0 + r < r1) ? w[i0 + r] : 0.0;
        }
        for (int j0 = 0; j0 < cols; j0 += 4) {
            double vr[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double* col = V + (int64_t)min(j0 + q, cols - 1) * ld + i0;
                if (full) {
                    ld4(col, true, vr[q]);
                } else {
#pragma unroll
                    for (int r = 0; r < 4; ++r) vr[q][r] = (i0 + r < r1) ? __ldg(col + r) : 0.0;
                }
            }
            double s[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                s[q] = 0.0;
#pragma unroll
                for (int r = 0; r < 4; ++r) s[q] = fma(vr[q][r], wr[r], s[q]);
            }
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int q = 0; q < 4; ++q) s[q] += __shfl_down_sync(0xffffffffu, s[q], o);
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (j0 + q < cols) acc[warp][j0 + q] += s[q];
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cols; j += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < 8; ++k) s += acc[k][j];
        part[(int64_t)j * nb + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(256) cgs_dot_kernel(const double* __restrict__ V, int64_t ld, int64_t n, int cols,
                                                      const double* __restrict__ w, double* __restrict__ part) {
    cgs_dot_block(V, ld, n, cols, w, part);
}

// The lockstep PKSM's CGS2 of T chains in ONE launch per phase: chain t =
// blockIdx.y, its pointers from device arrays (every chain has the same n and
// column count; the row partition and every sum order are those of the
// single-chain kernels, so each chain's result is bitwise the same).
struct CgsBatch {
    const double* const* V;
    double* const* w;
    double* const* h_out;    // h1 + h2 (nullable entries not allowed: give scratch)
    double* const* h1_out;   // first-pass projections (alpha at cols - 1)
    double* const* nrm2;     // ||w||^2 after
    double* const* vnext;    // nullable array: V[t] column `cols` = w / sqrt(nrm2)
    double* work;            // T x per-chain scratch
    int64_t work_stride;
};

__global__ void __launch_bounds__(256) cgs_dot_batched(CgsBatch B, int64_t ld, int64_t n, int cols) {
    const int t = blockIdx.y;
    cgs_dot_block(B.V[t], ld, n, cols, B.w[t], B.work + t * B.work_stride);
}

// h[j] = sum_b part_in[j * nb + b] (warp per column, same in every block);
// w -= V h on the block's rows; npart[b] = the block's partial of ||w||^2.
// Block 0 stores h into h_save and h_prev + h into h_sum.
__device__ __forceinline__ void cgs_update_block(const double* __restrict__ V, int64_t ld, int64_t n, int cols,
                                                 const double* __restrict__ part_in, double* __restrict__ w,
                                                 double* __restrict__ npart, double* __restrict__ h_save,
                                                 const double* __restrict__ h_prev, double* __restrict__ h_sum) {
    __shared__ double h[64];
    __shared__ double sh[8];
    const int nb = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < cols; j += 8) {
        double s = 0.0;
        for (int b = lane; b < nb; b += 32) s += __ldcg(part_in + (int64_t)j * nb + b);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
            h[j] = s;
            if (blockIdx.x == 0) {
                if (h_save) h_save[j] = s;
                if (h_sum) h_sum[j] = h_prev[j] + s;
            }
        }
    }
    __syncthreads();
    const int64_t per = ((n + nb - 1) / nb + 3) & ~(int64_t)3;
    const int64_t r0 = min(n, blockIdx.x * per), r1 = min(n, r0 + per);
    double ss = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kTileRows) {
        const int64_t i0 = t0 + 4 * threadIdx.x;
        const bool full = i0 + 3 < r1;
        double x[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int j = 0; j < cols; ++j) {
            const double* col = V + (int64_t)j * ld + i0;
            const double hj = h[j];
            double v[4];
            if (full) {
                ld4(col, true, v);
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) v[r] = (i0 + r < r1) ? __ldg(col + r) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) x[r] = fma(v[r], hj, x[r]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = i0 + r;
            if (i >= r1) continue;
            const double wn = w[i] - x[r];
            w[i] = wn;
            ss = fma(wn, wn, ss);
        }
    }
    if (npart) {
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
        if (lane == 0) sh[warp] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
            npart[blockIdx.x] = t;
        }
    }
}

__global__ void __launch_bounds__(256) cgs_update_kernel(const double* __restrict__ V, int64_t ld, int64_t n, int cols,
                                                         const double* __restrict__ part_in, double* __restrict__ w,
                                                         double* __restrict__ npart, double* __restrict__ h_save,
                                                         const double* __restrict__ h_prev, double* __restrict__ h_sum) {
    cgs_update_block(V, ld, n, cols, part_in, w, npart, h_save, h_prev, h_sum);
}

// pass = 0: w -= V h1, h1 -> h1_out[t];  pass = 1: w -= V h2, h_out = h1 + h2, ||w||^2 partials
__global__ void __launch_bounds__(256) cgs_update_batched(CgsBatch B, int64_t ld, int64_t n, int cols, int pass) {
    const int t = blockIdx.y;
    double* wk = B.work + t * B.work_stride;
    double* npart = wk + (int64_t)kFusedBlocks * 64;
    if (pass == 0)
        cgs_update_block(B.V[t], ld, n, cols, wk, B.w[t], nullptr, B.h1_out[t], nullptr, nullptr);
    else
        cgs_update_block(B.V[t], ld, n, cols, wk, B.w[t], npart, nullptr, B.h1_out[t], B.h_out[t]);
}

// ||w||^2 of every chain (fixed-order sum of its block partials), then
// V[cols] = w / sqrt(||w||^2): grid (blocks, T)
__global__ void cgs_norm_scale_batched(CgsBatch B, int64_t ld, int64_t n, int cols, int nb) {
    const int t = blockIdx.y;
    const double* npart = B.work + t * B.work_stride + (int64_t)kFusedBlocks * 64;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += npart[b];   // the order of finish_partial
    if (blockIdx.x == 0 && threadIdx.x == 0) B.nrm2[t][0] = s;
    if (!B.vnext) return;
    const double f = 1.0 / sqrt(s);               // scale_by_kernel's factor
    const double* w = B.w[t];
    double* y = B.vnext[t] + (int64_t)cols * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = w[i] * f;
}

static int cgs2_fused(const double* V, int64_t ld, int64_t n, int cols, double* w, double* h_out, double* h1_out,
                      double* nrm2_out, double* work, cudaStream_t st) {
    const int nb = std::max(1, std::min(std::min(kFusedBlocks, 2 * device_sms()), (int)((n + kTileRows - 1) / kTileRows)));
    double* part = work;                              // nb x cols
    double* npart = part + (int64_t)kFusedBlocks * 64;  // nb
    double* h1 = npart + kFusedBlocks;                 // cols
    cgs_dot_kernel<<<nb, 256, 0, st>>>(V, ld, n, cols, w, part);
    cgs_update_kernel<<<nb, 256, 0, st>>>(V, ld, n, cols, part, w, nullptr, h1, nullptr, nullptr);
    cgs_dot_kernel<<<nb, 256, 0, st>>>(V, ld, n, cols, w, part);
    cgs_update_kernel<<<nb, 256, 0, st>>>(V, ld, n, cols, part, w, npart, nullptr, h1, h_out);
    note_launches(4);
    if (nrm2_out) {
        finish_partial<<<1, 64, 0, st>>>(npart, nb, 1, nrm2_out, nullptr);
        note_launches(1);
    }
    if (h1_out) MLB_CUDA_TRY(cudaMemcpyAsync(h1_out, h1, cols * sizeof(double), cudaMemcpyDeviceToDevice, st));
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

static int ew_grid(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > device_sms() * 16) b = device_sms() * 16;
    return (int)(b < 1 ? 1 : b);
}


// ------------------------------------------------------ PKSM coefficients --
// The lockstep PKSM's per-step coefficients on the device (krylov.py:196-216:
// eigh(T_s), f(Lambda), y = ||v|| V_s Q f(Lambda) Q[0,:]), one warp per
// chain, so no host eigh sits between two graph replays.  Step j of chain t:
//   * record alpha_j = ab[j] and beta_j = sqrt(max(ab[dim + j], 0)) (the
//     CGS2 just wrote them) into the chain's history;
//   * T_s (s = j + 1) = tridiag(beta, alpha, beta) -> eigenvalues and
//     eigenvectors by implicit QL with shifts (the EISPACK tql2 scheme): the
//     scalar recurrence is evaluated redundantly by every lane, lane 0 writes
//     the diagonal / off-diagonal back, and each rotation updates the
//     eigenvector matrix in shared memory with one lane per row;
//   * c = nv Q f(max(Lambda, 0)) Q[0,:]^T into C[t][j][0..s);
//   * stats after the row's <v,v> entry: min eigenvalue (unclamped), ||c||^2,
//     ||c - [c_{j-1}; 0]||^2 (fixed-order warp sums), status (1 = QL did not
//     converge in 60 sweeps: the host recomputes that step).
constexpr int kTriMax = 64;
constexpr int kTriLd = kTriMax + 1;

__device__ __forceinline__ double tri_f(double lam, double p) {
    lam = fmax(lam, 0.0);
    if (p == -1.0) return 1.0 / lam;   // numpy's fast paths for these powers
    if (p == 1.0) return lam;
    if (p == 2.0) return lam * lam;
    if (p == 0.5) return sqrt(lam);
    return pow(lam, p);
}

__global__ void __launch_bounds__(32) tridiag_fn_kernel(double* __restrict__ AB, int ld, int dim, int j, double p,
                                                        double* __restrict__ hist, double* __restrict__ Cc) {
    __shared__ double Q[kTriMax * kTriLd];
    __shared__ double dg[kTriMax], of[kTriMax];
    const int t = blockIdx.x, lane = threadIdx.x;
    double* ab = AB + (size_t)t * ld;
    double* al = hist + (size_t)t * 2 * dim;
    double* be = al + dim;
    const int s = j + 1;
    if (lane == 0) {
        al[j] = ab[j];
        be[j] = sqrt(fmax(ab[dim + j], 0.0));
    }
    __syncwarp();
    if (p == -1.0) {
        // f(T) e1 = T^{-1} e1: one LDL^T (Thomas) solve, O(s), instead of the
        // eigendecomposition.  All pivots positive <=> T SPD (Sylvester
        // inertia), then lmin is reported as the smallest pivot (> 0: the
        // host only tests its sign); otherwise the QL path below yields the
        // real minimum eigenvalue for the host's error.
        int spd = 1;
        double pmin = 0.0;
        if (lane == 0) {
            double piv = al[0];
            pmin = piv;
            dg[0] = piv;   // pivots in dg, the forward-eliminated right-hand side in of
            spd = piv > 0.0;
            double z = 1.0;
            of[0] = z;
            for (int i = 1; i < s && spd; ++i) {
                const double l = be[i - 1] / piv;
                piv = al[i] - l * be[i - 1];
                z = -l * z;
                dg[i] = piv;
                of[i] = z;
                pmin = fmin(pmin, piv);
                spd = piv > 0.0;
            }
        }
        spd = __shfl_sync(0xffffffffu, spd, 0);
        if (spd) {
            const double nv = sqrt(ab[2 * dim]);
            double* c = Cc + ((size_t)t * dim + j) * dim;
            const double* cp = Cc + ((size_t)t * dim + (j > 0 ? j - 1 : 0)) * dim;
            if (lane == 0) {   // back substitution: x_i = (z_i - be_i x_{i+1}) / piv_i
                double x = of[s - 1] / dg[s - 1];
                c[s - 1] = nv * x;
                for (int i = s - 2; i >= 0; --i) {
                    x = (of[i] - be[i] * x) / dg[i];
                    c[i] = nv * x;
                }
            }
            __syncwarp();
            double c2 = 0.0, d2 = 0.0;
            for (int i = lane; i < s; i += 32) {
                const double ci = c[i];
                const double di = ci - ((j > 0 && i < s - 1) ? cp[i] : 0.0);
                c2 = fma(ci, ci, c2);
                d2 = fma(di, di, d2);
            }
            for (int o = 16; o > 0; o >>= 1) {
                c2 += __shfl_xor_sync(0xffffffffu, c2, o);
                d2 += __shfl_xor_sync(0xffffffffu, d2, o);
            }
            if (lane == 0) {
                ab[2 * dim + 1] = pmin;
                ab[2 * dim + 2] = c2;
                ab[2 * dim + 3] = d2;
                ab[2 * dim + 4] = 0.0;
            }
            return;
        }
        __syncwarp();
    }
    for (int i = lane; i < s; i += 32) {
        dg[i] = al[i];
        of[i] = (i + 1 < s) ? be[i] : 0.0;
        for (int k = 0; k < s; ++k) Q[i * kTriLd + k] = (i == k) ? 1.0 : 0.0;
    }
    __syncwarp();
    int status = 0;
    for (int l = 0; l < s && !status; ++l) {
        for (int iter = 0;; ++iter) {
            int m = l;
            for (; m < s - 1; ++m) {   // first negligible off-diagonal at or after l
                const double e = fabs(of[m]);
                if (e == 0.0 || e <= 2.220446049250313e-16 * (fabs(dg[m]) + fabs(dg[m + 1]))) break;
            }
            if (m == l) break;
            if (iter == 60) {
                status = 1;
                break;
            }
            double g = (dg[l + 1] - dg[l]) / (2.0 * of[l]);
            double r = hypot(g, 1.0);
            g = dg[m] - dg[l] + of[l] / (g + copysign(r, g));
            double sn = 1.0, cs = 1.0, pp = 0.0;
            bool split = false;
            for (int i = m - 1; i >= l; --i) {
                const double ei = of[i], di = dg[i], di1 = dg[i + 1];
                __syncwarp();
                const double f = sn * ei, b = cs * ei;
                r = hypot(f, g);
                if (lane == 0) of[i + 1] = r;
                if (r == 0.0) {   // the rotation underflowed: deflate and restart at l
                    if (lane == 0) {
                        dg[i + 1] = di1 - pp;
                        of[m] = 0.0;
                    }
                    split = true;
                    __syncwarp();
                    break;
                }
                sn = f / r;
                cs = g / r;
                g = di1 - pp;
                r = (di - g) * sn + 2.0 * cs * b;
                pp = sn * r;
                if (lane == 0) dg[i + 1] = g + pp;
                g = cs * r - b;
                for (int k = lane; k < s; k += 32) {   // columns i, i+1 of the eigenvector matrix
                    double* q = Q + k * kTriLd;
                    const double qi = q[i], qi1 = q[i + 1];
                    q[i + 1] = sn * qi + cs * qi1;
                    q[i] = cs * qi - sn * qi1;
                }
                __syncwarp();
            }
            if (split) continue;
            if (lane == 0) {
                dg[l] -= pp;
                of[l] = g;
                of[m] = 0.0;
            }
            __syncwarp();
        }
    }
    // f(Lambda) Q[0,:] into `of`, then c = nv Q (f Q[0,:]) with one lane per row
    double lmin = dg[0];
    for (int k = 1; k < s; ++k) lmin = fmin(lmin, dg[k]);
    __syncwarp();
    for (int k = lane; k < s; k += 32) of[k] = tri_f(dg[k], p) * Q[k];
    __syncwarp();
    const double nv = sqrt(ab[2 * dim]);
    double* c = Cc + ((size_t)t * dim + j) * dim;
    const double* cp = Cc + ((size_t)t * dim + (j > 0 ? j - 1 : 0)) * dim;
    double c2 = 0.0, d2 = 0.0;
    for (int i = lane; i < s; i += 32) {
        double acc = 0.0;
        for (int k = 0; k < s; ++k) acc = fma(Q[i * kTriLd + k], of[k], acc);
        const double ci = nv * acc;
        c[i] = ci;
        const double di = ci - ((j > 0 && i < s - 1) ? cp[i] : 0.0);
        c2 = fma(ci, ci, c2);
        d2 = fma(di, di, d2);
    }
    for (int o = 16; o > 0; o >>= 1) {
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    if (lane == 0) {
        ab[2 * dim + 1] = lmin;
        ab[2 * dim + 2] = c2;
        ab[2 * dim + 3] = d2;
        ab[2 * dim + 4] = (double)status;
    }
}

}  // namespace mlb

using namespace mlb;

extern "C" {

int64_t mlb_krylov_work_size(int64_t n, int maxcols) {
    (void)n;
    const int64_t unfused = (int64_t)kMaxRowBlocks * (maxcols + 2) + 2 * (maxcols + 2);
    const int64_t fused = (int64_t)kFusedBlocks * (64 + 1) + 64;
    return std::max(unfused, fused);
}

int mlb_gemv_t(const double* V, int64_t ld, int64_t n, int cols, const double* w, double* h, double* work,
               void* stream) {
    if (cols <= 0) return MLB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = row_blocks(n);
    gemv_t_partial<<<dim3(nb, cols), kRedThreads, 0, st>>>(V, ld, n, w, work);
    note_launches(1);
    finish_partial<<<(cols + 63) / 64, 64, 0, st>>>(work, nb, cols, h, nullptr);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_gemv_n(const double* V, int64_t ld, int64_t n, int cols, const double* c, double* y, double scale,
               int accumulate, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = std::max(1, std::min(device_sms() * 4, (int)((n + 255) / 256)));
    gemv_n_kernel<<<nb, 256, cols * sizeof(double), st>>>(V, ld, n, cols, c, y, scale, accumulate, nullptr);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_cgs2(const double* V, int64_t ld, int64_t n, int cols, double* w, double* h_out, double* h1_out,
             double* nrm2_out, double* work, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (cols <= 0 || n <= 0) return MLB_OK;
    const bool aligned = !(ld & 1) && !(reinterpret_cast<uintptr_t>(V) & 15) && !(reinterpret_cast<uintptr_t>(w) & 15);
    if (cols <= 64 && aligned) return cgs2_fused(V, ld, n, cols, w, h_out, h1_out, nrm2_out, work, st);
    const int nb = row_blocks(n);
    double* part = work;                                     // kMaxRowBlocks * cols
    double* h1 = work + (int64_t)kMaxRowBlocks * (cols + 2);  // cols
    const int nbn = std::max(1, std::min(kMaxRowBlocks, (int)((n + 255) / 256)));
    // pass 1: h1 = V^T w ; w -= V h1
    gemv_t_partial<<<dim3(nb, cols), kRedThreads, 0, st>>>(V, ld, n, w, part);
    note_launches(1);
    finish_partial<<<(cols + 63) / 64, 64, 0, st>>>(part, nb, cols, h1, nullptr);
    note_launches(1);
    gemv_n_kernel<<<nbn, 256, cols * sizeof(double), st>>>(V, ld, n, cols, h1, w, -1.0, 1, nullptr);
    note_launches(1);
    // pass 2: h2 = V^T w ; w -= V h2 ; h_out = h1 + h2 ; ||w||^2
    gemv_t_partial<<<dim3(nb, cols), kRedThreads, 0, st>>>(V, ld, n, w, part);
    note_launches(1);
    finish_partial<<<(cols + 63) / 64, 64, 0, st>>>(part, nb, cols, h_out, h1);
    note_launches(1);
    // h2 = h_out - h1 is needed for the update: recompute it into h1's slot
    double* h2 = h1 + cols + 1;
    finish_partial<<<(cols + 63) / 64, 64, 0, st>>>(part, nb, cols, h2, nullptr);
    note_launches(1);
    double* npart = part + (int64_t)nb * cols;
    gemv_n_kernel<<<nbn, 256, cols * sizeof(double), st>>>(V, ld, n, cols, h2, w, -1.0, 1, npart);
    note_launches(1);
    if (nrm2_out) {
        finish_partial<<<1, 64, 0, st>>>(npart, nbn, 1, nrm2_out, nullptr);
        note_launches(1);
    }
    if (h1_out) MLB_CUDA_TRY(cudaMemcpyAsync(h1_out, h1, cols * sizeof(double), cudaMemcpyDeviceToDevice, st));
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int64_t mlb_cgs2_batched_work_size(int T) { return (int64_t)T * ((int64_t)kFusedBlocks * (64 + 1) + 64); }

int mlb_cgs2_batched(int T, const double* const* V, int64_t ld, int64_t n, int cols, double* const* w,
                     double* const* h_out, double* const* h1_out, double* const* nrm2_out, double* const* vnext,
                     double* work, void* stream) {
    if (T <= 0 || cols <= 0 || n <= 0) return MLB_OK;
    if (cols > 64 || (ld & 1)) return fail(MLB_ERR_ARG, "batched CGS2 needs cols <= 64 and an even leading dimension");
    if (!V || !w || !h_out || !h1_out || !nrm2_out || !work) return fail(MLB_ERR_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = std::max(1, std::min(std::min(kFusedBlocks, 2 * device_sms()), (int)((n + kTileRows - 1) / kTileRows)));
    CgsBatch B{V, w, h_out, h1_out, nrm2_out, vnext, work, (int64_t)kFusedBlocks * (64 + 1) + 64};
    cgs_dot_batched<<<dim3(nb, T), 256, 0, st>>>(B, ld, n, cols);
    cgs_update_batched<<<dim3(nb, T), 256, 0, st>>>(B, ld, n, cols, 0);
    cgs_dot_batched<<<dim3(nb, T), 256, 0, st>>>(B, ld, n, cols);
    cgs_update_batched<<<dim3(nb, T), 256, 0, st>>>(B, ld, n, cols, 1);
    cgs_norm_scale_batched<<<dim3(ew_grid(n) / std::max(1, T / 8) + 1, T), 256, 0, st>>>(B, ld, n, cols, nb);
    note_launches(5);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_tridiag_fn_batched(int T, double* AB, int64_t ld, int dim, int j, double p, double* hist, double* C,
                           void* stream) {
    if (T <= 0) return MLB_OK;
    if (dim < 1 || dim > kTriMax || j < 0 || j >= dim) return fail(MLB_ERR_ARG, "tridiagonal step needs 0 <= j < dim <= 64");
    if (ld < 2 * (int64_t)dim + 5) return fail(MLB_ERR_ARG, "AB rows need 2 dim + 5 entries");
    if (!AB || !hist || !C) return fail(MLB_ERR_ARG, "null argument");
    tridiag_fn_kernel<<<T, 32, 0, (cudaStream_t)stream>>>(AB, (int)ld, dim, j, p, hist, C);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_gemm_vs(const double* V, int64_t ld, int64_t n, int s, const double* S, int k, double* Out, int64_t ldo,
                void* stream) {
    if (k <= 0 || n <= 0) return MLB_OK;
    dim3 grid((unsigned)((n + 63) / 64), (unsigned)((k + 31) / 32));
    gemm_vs_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(V, ld, n, s, S, k, Out, ldo);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_dot(const double* x, const double* y, int64_t n, double* out, double* work, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = row_blocks(n);
    dot_partial<<<nb, kRedThreads, 0, st>>>(x, y, n, work);
    note_launches(1);
    finish_partial<<<1, 64, 0, st>>>(work, nb, 1, out, nullptr);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream) {
    if (n <= 0) return MLB_OK;
    axpby_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(a, x, b, y, n);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_scale_by(const double* x, double* y, int64_t n, const double* s_dev, double pw, void* stream) {
    if (n <= 0) return MLB_OK;
    scale_by_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(x, y, n, s_dev, pw);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_hadamard(const double* x, const double* y, double* z, int64_t n, void* stream) {
    if (n <= 0) return MLB_OK;
    hadamard_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(x, y, z, n);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

}  // extern "C"
