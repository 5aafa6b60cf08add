// Lattice (separable-per-cell) spread / gather for d = 2 layers whose points
// form product lattices inside their cells -- every spatial layer of an image
// (pixel coordinates).  Reference chain unchanged (fastsum.py:389-406: the
// spread / gather of the NFFT fast summation); only the order of the sums
// inside one cell changes.
//
// Inside a cell the points are an R x C product set: run r (C consecutive
// cell-sorted points) shares the "slow" axis offset, column c the "fast"
// axis offset, so with Ws[r] / Wf[c] the windows (2m+1 values) of row r /
// column c and SV the cell's s v as an R x C matrix
//   spread block   B  = Ws^T (SV Wf)            (S x S, S = 2m+1)
//   gather values  Y  = (Ws G) Wf^T             (R x C)
// i.e. ~S + S^2/C multiply-adds per point instead of ~S^2 plus 2S window
// polynomials (~300 DFMA per point per pass at m = 5).  Cells that are not
// lattices (node-range shard cuts, stray points) run as "diagonal" items:
// the same two contractions with one row per point (Wf per row).
//
// Work items (bind time, build_lattice below; lat_detect_kernel checks the
// structure and splits a cell cut by a node range into partial run +
// lattice + partial run): <= kLatRowsMax rows / kLatPts points of one cell
// segment, one CTA each.  The spread forms both contractions on the fp64
// tensor cores (mma.sync m8n8k4) and writes one S x S block per item;
// lat_reduce_kernel sums, per grid cell, the blocks covering it in (bin,
// item) order -- no atomics, bitwise reproducible.  The gather fuses the
// L_sym epilogue like gather_kernel (y = alpha v + s (beta acc + gamma s v)).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "mlb_internal.cuh"
#include "mlb_window.cuh"

// A/B switches (tools/build_variant.sh), defaults = the measured best at
// config 4 (d = 2 spread / gather us): CTAs per SM of the spread (2: 143 /
// 3: 124 / 4: 116) and gather (2: 98 / 3: 83), window polynomials as
// per-thread tasks (spread 166 -> 124 at 3 CTAs; gather 98 -> 137: divergent
// constant-bank reads), gather epilogue loads hoisted (123 -> 98 at 2 CTAs),
// the spread's two contractions on the fp64 tensor cores (DMMA m8n8k4: 116 ->
// 112 us; the FMA path with column-group partials stays as MLB_LAT_DMMA=0),
// the spread's window coefficients copied to shared memory (112 -> 102 us),
// then 5 spread CTAs per SM (51 registers, no spill: 102 -> 97 us; 6: spills,
// 119 us; per-value windows at 5: spills, 124 us)
#ifndef MLB_LAT_SPREAD_MINB
#define MLB_LAT_SPREAD_MINB 5
#endif
#ifndef MLB_LAT_GATHER_MINB
#define MLB_LAT_GATHER_MINB 3
#endif
#ifndef MLB_LAT_WTASK_S
#define MLB_LAT_WTASK_S 1
#endif
#ifndef MLB_LAT_WTASK_G
#define MLB_LAT_WTASK_G 0
#endif
#ifndef MLB_LAT_DMMA
#define MLB_LAT_DMMA 1
#endif
#ifndef MLB_LAT_WSMEM
#define MLB_LAT_WSMEM 1
#endif
#ifndef MLB_LAT_GHOIST
#define MLB_LAT_GHOIST 1
#endif

namespace mlb {

// fp64 tensor-core MMA (one warp): D(8x8) += A(8x4, row) B(4x8, col); lane l
// holds A[l/4][l%4], B[l%4][l/4] and D[l/4][2(l%4) .. 2(l%4)+1]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}



// ------------------------------------------------------------- detection --
// First index in [i0, i1) (step dir = +1) or last index in [i1, i0] (dir =
// -1, scanning down from i0) where f differs from f[i0]; returns the run
// length of the constant value starting at i0 in that direction.
__device__ __forceinline__ int lat_run(const double* __restrict__ f, int i0, int len, int dir, int lane) {
    const double f0 = f[i0];
    for (int base = 0; base < len; base += 32) {
        const int i = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < len && f[i0 + dir * i] != f0);
        if (m) return base + __ffs(m) - 1;
    }
    return len;
}

// Is [q0, q0 + Q) an (Q / C) x C product set with `fast` varying along runs of C?
__device__ __forceinline__ bool lat_check(const double* __restrict__ frac, int64_t n, int q0, int Q, int C, int fast,
                                          int lane) {
    const double* ff = frac + fast * n + q0;
    const double* fs = frac + (1 - fast) * n + q0;
    bool bad = false;
    for (int i = lane; i < Q; i += 32) {
        const int r = i / C, c = i - r * C;
        bad |= (ff[i] != ff[c]) || (fs[i] != fs[r * C]);
    }
    return !__any_sync(0xffffffffu, bad);
}

// One warp per cell (key): is the cell's point list (cell-sorted = node
// order, i.e. row-major for an image) an R x C product set, or -- a node
// range cutting the image's rows (a shard) -- a partial run, an R x C
// product set and a partial run?  out[4k..4k+3] = {code, fast | C << 1, a, b}:
// code 0 empty cell, -1 not a lattice, 1 one R x C lattice (all P points),
// 3 segments [0, a) (one run), [a, b) (runs of C), [b, P) (one run).
__global__ void lat_detect_kernel(const double* __restrict__ frac, int64_t n, const int32_t* __restrict__ ks,
                                  int nkeys, int cmax, int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k >= nkeys) return;
    const int p0 = ks[k], P = ks[k + 1] - p0;
    int code = -1, fastC = 0, a = 0, b = 0;
    if (P == 0) {
        code = 0;
    } else {
        // whole cell: axis 0 fixed along the first run -> axis 1 is fast
        const int run0 = lat_run(frac + p0, 0, P, 1, lane);
        const int run1 = lat_run(frac + n + p0, 0, P, 1, lane);
        const int fast = run0 >= 2 ? 1 : (run1 >= 2 ? 0 : 1);
        const int C = run0 >= 2 ? run0 : (run1 >= 2 ? run1 : 1);
        if (P % C == 0 && C <= cmax && lat_check(frac, n, p0, P, C, fast, lane)) {
            code = 1;
            fastC = fast | (C << 1);
        } else {
            // a partial first / last run around a lattice (either axis slow)
            for (int fa = 1; fa >= 0 && code < 0; --fa) {
                const double* fs = frac + (1 - fa) * n + p0;
                const int ra = lat_run(fs, 0, P, 1, lane);               // first run
                if (ra >= P) continue;
                const int rb = lat_run(fs, P - 1, P - ra, -1, lane);     // last run
                const int A = ra, B = P - rb;
                if (A > cmax || rb > cmax) continue;
                int Cm = 1;
                bool ok = true;
                if (B > A) {
                    Cm = lat_run(fs, A, B - A, 1, lane);
                    ok = (B - A) % Cm == 0 && Cm <= cmax && lat_check(frac, n, p0 + A, B - A, Cm, fa, lane);
                }
                if (ok) {
                    code = 3;
                    fastC = fa | (Cm << 1);
                    a = A;
                    b = B;
                }
            }
        }
    }
    if (lane == 0) {
        out[4 * k] = code;
        out[4 * k + 1] = fastC;
        out[4 * k + 2] = a;
        out[4 * k + 3] = b;
    }
}

// ------------------------------------------------------------ the kernels --
// shared-memory layout of one item (sizes from the binding's widest item)
struct LatLayout {
    int nf_max;   // Wf rows (lattice: C; diagonal: R)
    int r_max;    // rows
    int sv_max;   // staged s v values (rows padded to an odd stride)
};

// one polynomial of a window set: q = 0 -> w[0] = P_{-m}, q >= 1 -> the pair
// w[q + m], w[1 - q + m] (kb_windows' arithmetic, bitwise the same values)
template <int M>
__device__ __forceinline__ void kb_window_task(double f, int q, const WinCoef& c, double* w) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    const double s = 2.0 * f - 1.0;
    if (q == 0) {
        double p = c.mm[DM];
#pragma unroll
        for (int j = DM - 1; j >= 0; --j) p = fma(p, s, c.mm[j]);
        w[0] = p;
    } else {
        const double s2 = s * s;
        double e = c.e[q - 1][NE - 1];
#pragma unroll
        for (int j = NE - 2; j >= 0; --j) e = fma(e, s2, c.e[q - 1][j]);
        double od = c.o[q - 1][NO - 1];
#pragma unroll
        for (int j = NO - 2; j >= 0; --j) od = fma(od, s2, c.o[q - 1][j]);
        od *= s;
        w[q + M] = e + od;
        w[1 - q + M] = e - od;
    }
}

// windows of the item's table rows [t0, t1) (Wf rows first, then Ws), one
// polynomial per thread task so every thread of the CTA takes part
template <int M, bool TASKS>
__device__ __forceinline__ void lat_windows_range(const int4 it, const double* __restrict__ frac, int64_t n,
                                                  const WinCoef& wc, double* Wf, double* Ws, int t0, int t1) {
    constexpr int S = 2 * M + 1;
    const int R = it.y, C = it.z & 0xffff, fast = (it.z >> 16) & 1, diag = (it.z >> 17) & 1;
    const int nf = diag ? R : C;
    const double* ff = frac + (int64_t)fast * n + it.x;
    const double* fs = frac + (int64_t)(1 - fast) * n + it.x;
    const int rs = diag ? 1 : C;
    if (TASKS) {
    for (int task = (int)threadIdx.x; task < (t1 - t0) * (M + 1); task += blockDim.x) {
        const int t = t0 + task / (M + 1), q = task % (M + 1);
        const bool isf = t < nf;
        const double f = isf ? __ldg(ff + t) : __ldg(fs + (int64_t)(t - nf) * rs);
        kb_window_task<M>(f, q, wc, isf ? Wf + t * S : Ws + (t - nf) * S);
    }
    } else {
    for (int t = t0 + (int)threadIdx.x; t < t1; t += blockDim.x) {
        const bool isf = t < nf;
        const double f = isf ? __ldg(ff + t) : __ldg(fs + (int64_t)(t - nf) * rs);
        double w[S];
        kb_windows<M>(f, wc, w);
        double* dst = isf ? Wf + t * S : Ws + (t - nf) * S;
#pragma unroll
        for (int q = 0; q < S; ++q) dst[q] = w[q];
    }
    }
}

// One CTA per item.  D^-1/2 and the sorted -> node indices are static
// tables (set_isd's kernel is a plain launch: it completes before any PDL
// successor starts), so they load before pdl_wait; v is loaded after it,
// while the row windows are evaluated.
template <int M>
__global__ void __launch_bounds__(kLatThreads, MLB_LAT_SPREAD_MINB)
    lat_spread_kernel(const int4* __restrict__ items, const double* __restrict__ frac, int64_t n,
                      const int32_t* __restrict__ perm, const double* __restrict__ isd, WinCoef wc,
                      const double* __restrict__ v, unsigned flags, LatLayout lay, double* __restrict__ blocks) {
    constexpr int S = 2 * M + 1;
    constexpr int KP = kLatPts / kLatThreads;   // points per thread
    extern __shared__ double sm[];
    const int4 it = __ldg(items + blockIdx.x);
    const int p0 = it.x, R = it.y, C = it.z & 0xffff, fast = (it.z >> 16) & 1, diag = (it.z >> 17) & 1;
    const int P = diag ? R : R * C;
    const int Cw = diag ? 1 : C;
    const int Cp = diag ? 1 : (C | 1);   // odd row stride of SV: conflict-free column reads
    double* SV = sm;
    double* Wf = SV + lay.sv_max;
    double* Ws = Wf + lay.nf_max * S;
    double* Tp = Ws + lay.r_max * S;                          // column-group partials (FMA path)
    double* T = Tp + (MLB_LAT_DMMA ? 0 : kLatThreads * S);
    const bool sorted = (flags & MLB_SORTED) != 0, use_isd = (flags & MLB_USE_ISD) != 0;
    const int tid = threadIdx.x;
    int nd[KP];
    double sc[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        const int idx = tid + k * kLatThreads;
        nd[k] = idx < P ? (sorted ? p0 + idx : __ldg(perm + p0 + idx)) : -1;
        sc[k] = (idx < P && use_isd) ? __ldg(isd + p0 + idx) : 1.0;
    }
    const int nf = diag ? R : C;
#if MLB_LAT_WSMEM
    // the window coefficients in shared memory: the per-thread polynomial
    // tasks read different rows (divergent constant-bank reads serialise)
    __shared__ WinCoef wcs;
    {
        const double* src = reinterpret_cast<const double*>(&wc);
        double* dst = reinterpret_cast<double*>(&wcs);
        for (int i = tid; i < (int)(sizeof(WinCoef) / sizeof(double)); i += kLatThreads) dst[i] = src[i];
        __syncthreads();
    }
    const WinCoef& wq = wcs;
#else
    const WinCoef& wq = wc;
#endif
    lat_windows_range<M, MLB_LAT_WTASK_S>(it, frac, n, wq, Wf, Ws, 0, nf);
    pdl_wait();   // v comes from stream predecessors
    double x[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) x[k] = nd[k] >= 0 ? __ldg(v + nd[k]) * sc[k] : 0.0;
    lat_windows_range<M, MLB_LAT_WTASK_S>(it, frac, n, wq, Wf, Ws, nf, nf + R);
    {   // point idx = tid + k * kLatThreads sits at (r, c) of the item: step by (dr, dc)
        int r = tid / Cw, c = tid - r * Cw;
        const int dr = kLatThreads / Cw, dc = kLatThreads - dr * Cw;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            if (nd[k] >= 0) SV[r * Cp + c] = x[k];
            c += dc;
            r += dr;
            if (c >= Cw) {
                c -= Cw;
                ++r;
            }
        }
    }
    __syncthreads();
#if MLB_LAT_DMMA
    const int lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;   // fragment row / column group of the lane
    constexpr int NT = (S + 7) / 8;            // 8-wide tiles over the S window offsets
    if (!diag) {
        // T = SV Wf on the fp64 tensor cores: warp w owns 8 x 8 tiles
        // (row tile, offset tile) w, w + 8, ...; K = C columns in steps of 4
        const int MT = (R + 7) / 8;
        for (int tile = warp; tile < MT * NT; tile += kLatThreads / 32) {
            const int r0 = (tile / NT) * 8, q0 = (tile % NT) * 8;
            double d0 = 0.0, d1 = 0.0;
            const int ra = r0 + gq, qb = q0 + gq;
            for (int c0 = 0; c0 < C; c0 += 4) {
                const int c = c0 + tq;
                const double av = (ra < R && c < C) ? SV[ra * Cp + c] : 0.0;
                const double bv = (c < C && qb < S) ? Wf[c * S + qb] : 0.0;
                dmma884(d0, d1, av, bv);
            }
            const int q = q0 + 2 * tq;
            if (ra < R) {
                if (q < S) T[ra * S + q] = d0;
                if (q + 1 < S) T[ra * S + q + 1] = d1;
            }
        }
    } else {
        for (int r = tid; r < R; r += kLatThreads) {
            const double xv = SV[r];
#pragma unroll
            for (int q = 0; q < S; ++q) T[r * S + q] = xv * Wf[r * S + q];
        }
    }
    __syncthreads();
    // B = Ws^T T (S x S) on the tensor cores: one warp per 8 x 8 tile, K = R
    double* out = blocks + (int64_t)blockIdx.x * S * S;
    for (int tile = warp; tile < NT * NT; tile += kLatThreads / 32) {
        const int ks0 = (tile / NT) * 8, kf0 = (tile % NT) * 8;
        double d0 = 0.0, d1 = 0.0;
        const int ksa = ks0 + gq, kfb = kf0 + gq;
        for (int r0 = 0; r0 < R; r0 += 4) {
            const int r = r0 + tq;
            const double av = (r < R && ksa < S) ? Ws[r * S + ksa] : 0.0;
            const double bv = (r < R && kfb < S) ? T[r * S + kfb] : 0.0;
            dmma884(d0, d1, av, bv);
        }
        const int kf = kf0 + 2 * tq;
        if (ksa < S) {
            if (kf < S) out[fast ? ksa * S + kf : kf * S + ksa] = d0;
            if (kf + 1 < S) out[fast ? ksa * S + kf + 1 : (kf + 1) * S + ksa] = d1;
        }
    }
    pdl_launch();
    (void)Tp;
#else
    if (!diag) {
        // Tp[cg][r] = sum over column group cg of SV[r][c] Wf[c]: thread
        // (r, cg), r fastest, so a warp reads one Wf row (broadcast) per step
        const int NCG = max(1, min(C, kLatThreads / R));
        if (tid < NCG * R) {
            const int cg = tid / R, r = tid - cg * R;
            const int c0 = cg * C / NCG, c1 = (cg + 1) * C / NCG;
            double acc[S];
#pragma unroll
            for (int q = 0; q < S; ++q) acc[q] = 0.0;
            for (int c = c0; c < c1; ++c) {
                const double xv = SV[r * Cp + c];
                const double* w = Wf + c * S;
#pragma unroll
                for (int q = 0; q < S; ++q) acc[q] = fma(xv, w[q], acc[q]);
            }
#pragma unroll
            for (int q = 0; q < S; ++q) Tp[tid * S + q] = acc[q];
        }
        __syncthreads();
        for (int q = tid; q < R * S; q += kLatThreads) {
            double s = 0.0;
            for (int cg = 0; cg < NCG; ++cg) s += Tp[cg * R * S + q];
            T[q] = s;
        }
    } else {
        for (int r = tid; r < R; r += kLatThreads) {
            const double xv = SV[r];
#pragma unroll
            for (int q = 0; q < S; ++q) T[r * S + q] = xv * Wf[r * S + q];
        }
    }
    __syncthreads();
    // B[ks][kf] = sum_r Ws[r][ks] T[r][kf]; stored with axis 0 first
    double* out = blocks + (int64_t)blockIdx.x * S * S;
    for (int q = tid; q < S * S; q += kLatThreads) {
        const int ks = q / S, kf = q - ks * S;
        double s = 0.0;
        for (int r = 0; r < R; ++r) s = fma(Ws[r * S + ks], T[r * S + kf], s);
        out[fast ? q : kf * S + ks] = s;
    }
    pdl_launch();
#endif
}

// grid cell (u0, u1) = sum over the bins (u0 - i, u1 - j), i, j < S, of their
// items' block entries (i, j); one warp per grid cell, fixed xor tree
template <int M>
__global__ void lat_reduce_kernel(const double* __restrict__ blocks, const int32_t* __restrict__ bin_off, int nb,
                                  int L, PeerOut grid) {
    constexpr int S = 2 * M + 1;
    const int lane = threadIdx.x & 31;
    const int cell = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    pdl_wait();
    if (cell >= L * L) return;
    const int u0 = cell / L, u1 = cell - u0 * L;
    double s = 0.0;
    for (int q = lane; q < S * S; q += 32) {
        const int i = q / S, j = q - i * S;
        const int b0 = u0 - i, b1 = u1 - j;
        if (b0 < 0 || b0 >= nb || b1 < 0 || b1 >= nb) continue;
        const int bin = b0 * nb + b1;
        for (int t = __ldg(bin_off + bin); t < __ldg(bin_off + bin + 1); ++t) s += blocks[(int64_t)t * S * S + q];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) po_store(grid, cell, s);
    pdl_launch();
}

// One CTA per item.  Lattice items give thread (rg, c) one column (its
// windows stay in registers) and rows rg, rg + NG, ... (<= kLatGatherSlots);
// the epilogue's node indices, D^-1/2 and v are loaded at the start and
// arrive while the windows and H are formed.
template <int M>
__global__ void __launch_bounds__(kLatThreads, MLB_LAT_GATHER_MINB)
    lat_gather_kernel(const int4* __restrict__ items, const double* __restrict__ frac, int64_t n,
                      const int32_t* __restrict__ perm, const double* __restrict__ isd, WinCoef wc, int L,
                      const double* __restrict__ grid, const double* __restrict__ v, double* __restrict__ y,
                      double alpha, double beta, double gamma, unsigned flags, LatLayout lay) {
    constexpr int S = 2 * M + 1;
    constexpr int KG = kLatGatherSlots;
    extern __shared__ double sm[];
    const int4 it = __ldg(items + blockIdx.x);
    const int p0 = it.x, R = it.y, C = it.z & 0xffff, fast = (it.z >> 16) & 1, diag = (it.z >> 17) & 1;
    double* Wf = sm;
    double* Ws = Wf + lay.nf_max * S;
    double* H = Ws + lay.r_max * S;
    double* Gm = H + lay.r_max * S;
    const bool sorted = (flags & MLB_SORTED) != 0, use_isd = (flags & MLB_USE_ISD) != 0;
    const int tid = threadIdx.x;
    // this thread's points: (rg, c) lattice slots, or one row of a diagonal item
    const int NG = diag ? kLatThreads : kLatThreads / C;
    const int cw = diag ? 1 : C;
    const bool act = diag ? tid < R : tid < NG * C;
    const int rg = diag ? tid : tid / C, c = diag ? 0 : tid - rg * C;
    constexpr int KH = MLB_LAT_GHOIST ? KG : 1;
    int nd[KH];
    double sc[KH], vv[KH];
    if (MLB_LAT_GHOIST) {
#pragma unroll
        for (int k = 0; k < KH; ++k) {
            const int r = rg + k * NG;
            const bool ok = act && r < R;
            const int p = p0 + r * cw + c;
            nd[k] = ok ? (sorted ? p : __ldg(perm + p)) : -1;
            sc[k] = (ok && use_isd) ? __ldg(isd + p) : 1.0;
        }
    }
#if MLB_LAT_WTASK_G && MLB_LAT_WSMEM
    __shared__ WinCoef wcs;
    {
        const double* src = reinterpret_cast<const double*>(&wc);
        double* dst = reinterpret_cast<double*>(&wcs);
        for (int i = tid; i < (int)(sizeof(WinCoef) / sizeof(double)); i += kLatThreads) dst[i] = src[i];
        __syncthreads();
    }
    const WinCoef& wq = wcs;
#else
    const WinCoef& wq = wc;
#endif
    lat_windows_range<M, MLB_LAT_WTASK_G>(it, frac, n, wq, Wf, Ws, 0, (diag ? R : C) + R);
    pdl_wait();   // the grid and v come from stream predecessors
    if (MLB_LAT_GHOIST) {
#pragma unroll
        for (int k = 0; k < KH; ++k) vv[k] = (nd[k] >= 0 && v) ? __ldg(v + nd[k]) : 0.0;
    }
    // Gm[ks][kf] = grid neighbourhood in (slow, fast) axis order
    for (int q = tid; q < S * S; q += kLatThreads) {
        const int a = q / S, b = q - a * S;
        Gm[q] = __ldg(grid + it.w + (fast ? a * L + b : b * L + a));
    }
    __syncthreads();
    // H[r][kf] = sum_ks Ws[r][ks] Gm[ks][kf]
    for (int q = tid; q < R * S; q += kLatThreads) {
        const int r = q / S, kf = q - r * S;
        double s = 0.0;
#pragma unroll
        for (int ks = 0; ks < S; ++ks) s = fma(Ws[r * S + ks], Gm[ks * S + kf], s);
        H[q] = s;
    }
    __syncthreads();
    if (act) {
        double wf[S];
#pragma unroll
        for (int q = 0; q < S; ++q) wf[q] = Wf[(diag ? tid : c) * S + q];
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            const int r = rg + k * NG;
            int node;
            double s, x;
            if (MLB_LAT_GHOIST) {
                node = nd[k < KH ? k : 0];
                s = sc[k < KH ? k : 0];
                x = vv[k < KH ? k : 0];
                if (node < 0) continue;
            } else {
                if (r >= R) continue;
                const int p = p0 + r * cw + c;
                node = sorted ? p : __ldg(perm + p);
                s = use_isd ? __ldg(isd + p) : 1.0;
                x = v ? __ldg(v + node) : 0.0;
            }
            const double* h = H + r * S;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < S; ++q) acc = fma(h[q], wf[q], acc);
            double res = alpha * x + s * (beta * acc + gamma * s * x);
            if (flags & MLB_ACCUMULATE) res += y[node];
            y[node] = res;
        }
    }
    pdl_launch();
}

// -------------------------------------------------------------- launchers --
static LatLayout lat_layout(const mlb_binding* b) {
    LatLayout l;
    l.nf_max = b->lat_nf_max;
    l.r_max = b->lat_r_max;
    l.sv_max = b->lat_sv_max;
    return l;
}

static size_t lat_smem(int M, const LatLayout& l, bool gather) {
    const int S = 2 * M + 1;
    if (gather) return ((size_t)(l.nf_max + 2 * l.r_max) * S + (size_t)S * S) * sizeof(double);
    return ((size_t)l.sv_max + (size_t)(l.nf_max + 2 * l.r_max + (MLB_LAT_DMMA ? 0 : kLatThreads)) * S) * sizeof(double);
}

template <int M>
static cudaError_t lat_spread_m(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st) {
    const LatLayout lay = lat_layout(b);
    const size_t smem = lat_smem(M, lay, false);
    if (ensure_max_smem((const void*)lat_spread_kernel<M>, smem)) return cudaErrorInvalidValue;
    return launch_k(lat_spread_kernel<M>, dim3(b->lat_nitems), dim3(kLatThreads), smem, st,
                    reinterpret_cast<const int4*>(b->lat_items), (const double*)b->frac, b->n,
                    (const int32_t*)b->perm, (const double*)b->isd, b->plan->wc, v, flags, lay,
                    b->lat_blocks);
}

template <int M>
static cudaError_t lat_reduce_m(mlb_binding* b, const PeerOut& grid, cudaStream_t st) {
    const int L = b->plan->g.L;
    const int cells = L * L;
    return launch_k(lat_reduce_kernel<M>, dim3((cells + 7) / 8), dim3(256), 0, st, (const double*)b->lat_blocks,
                    (const int32_t*)b->lat_bin_off, b->plan->g.nb, L, grid);
}

template <int M>
static cudaError_t lat_gather_m(mlb_binding* b, const double* grid, const double* v, double* y, double alpha,
                                double beta, double gamma, unsigned flags, cudaStream_t st) {
    const LatLayout lay = lat_layout(b);
    const size_t smem = lat_smem(M, lay, true);
    if (ensure_max_smem((const void*)lat_gather_kernel<M>, smem)) return cudaErrorInvalidValue;
    return launch_k(lat_gather_kernel<M>, dim3(b->lat_nitems), dim3(kLatThreads), smem, st,
                    reinterpret_cast<const int4*>(b->lat_items), (const double*)b->frac, b->n,
                    (const int32_t*)b->perm, (const double*)b->isd, b->plan->wc, b->plan->g.L, grid, v, y, alpha,
                    beta, gamma, flags, lay);
}

#define MLB_LAT_CALL(FN, M, ...)                                                   \
    do {                                                                           \
        cudaError_t _e = cudaSuccess;                                              \
        switch (M) {                                                               \
            case 2: _e = FN<2>(__VA_ARGS__); break;                                \
            case 3: _e = FN<3>(__VA_ARGS__); break;                                \
            case 4: _e = FN<4>(__VA_ARGS__); break;                                \
            case 5: _e = FN<5>(__VA_ARGS__); break;                                \
            case 6: _e = FN<6>(__VA_ARGS__); break;                                \
            default: return fail(MLB_ERR_CONFIG, "lattice kernels cover m = 2..6"); \
        }                                                                          \
        if (_e != cudaSuccess) return fail(MLB_ERR_CUDA, std::string(#FN ": ") + cudaGetErrorString(_e)); \
    } while (0)

int launch_lat_spread(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st) {
    if (!v) return fail(MLB_ERR_ARG, "spread: null vector");
    MLB_LAT_CALL(lat_spread_m, b->plan->g.m, b, v, flags, st);
    note_launches(1);
    return MLB_OK;
}

int launch_lat_reduce(mlb_binding* b, const PeerOut& grid, cudaStream_t st) {
    MLB_LAT_CALL(lat_reduce_m, b->plan->g.m, b, grid, st);
    note_launches(1);
    return MLB_OK;
}

int launch_lat_gather(mlb_binding* b, const double* grid, const double* v, double* y, double alpha, double beta,
                      double gamma, unsigned flags, cudaStream_t st) {
    MLB_LAT_CALL(lat_gather_m, b->plan->g.m, b, grid, v, y, alpha, beta, gamma, flags, st);
    note_launches(1);
    return MLB_OK;
}

// ------------------------------------------------------------ bind tables --
// Lattice items of a d = 2 binding.  mode: -1 auto (n >= 2^16 and at least
// half the points in lattice cells of >= 2 x 2), 0 off, 1 forced.
int build_lattice(mlb_binding* b, const std::vector<int64_t>& cnt, const std::vector<int32_t>& key_gcell,
                  int mode, cudaStream_t st) {
    const Geom& g = b->plan->g;
    if (g.d != 2 || mode == 0 || b->n == 0 || g.m < 2 || g.m > kMaxM) return MLB_OK;
    if (mode < 0 && b->n < kLatMinN) return MLB_OK;
    const int nkeys = (int)key_gcell.size();
    std::vector<int32_t> ks(cnt.begin(), cnt.end());
    int32_t *ks_d = nullptr, *out_d = nullptr;
    MLB_CUDA_TRY(cudaMalloc(&ks_d, ks.size() * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMalloc(&out_d, (size_t)nkeys * 4 * sizeof(int32_t)));
    struct Free {
        int32_t *a, *b;
        ~Free() {
            cudaFree(a);
            cudaFree(b);
        }
    } fr{ks_d, out_d};
    MLB_CUDA_TRY(cudaMemcpyAsync(ks_d, ks.data(), ks.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    lat_detect_kernel<<<(nkeys + 7) / 8, 256, 0, st>>>(b->frac, b->n, ks_d, nkeys, kLatCols, out_d);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    std::vector<int32_t> lat((size_t)nkeys * 4);
    MLB_CUDA_TRY(cudaMemcpyAsync(lat.data(), out_d, lat.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    MLB_CUDA_TRY(cudaStreamSynchronize(st));
    // segments of a cell: {first point, rows, C, fast}; lattice = runs of C
    struct Seg { int64_t p0, R; int C, fast, diag; };
    auto segments = [&](int k, std::vector<Seg>& out) {
        out.clear();
        const int64_t p0 = cnt[k], P = cnt[k + 1] - p0;
        const int code = lat[4 * k], fast = lat[4 * k + 1] & 1, C = lat[4 * k + 1] >> 1;
        if (P == 0) return;
        if (code == 1) {
            out.push_back({p0, P / C, C, fast, 0});
        } else if (code == 3) {
            const int64_t a = lat[4 * k + 2], bb = lat[4 * k + 3];
            if (a > 0) out.push_back({p0, 1, (int)a, fast, 0});
            if (bb > a) out.push_back({p0 + a, (bb - a) / C, C, fast, 0});
            if (P > bb) out.push_back({p0 + bb, 1, (int)(P - bb), fast, 0});
        } else {
            out.push_back({p0, P, 1, 1, 1});   // diagonal: one row per point
        }
    };
    std::vector<Seg> segs;
    int64_t lat_pts = 0;
    for (int k = 0; k < nkeys; ++k) {
        segments(k, segs);
        for (const Seg& sg : segs)
            if (!sg.diag && sg.C >= 2 && sg.R >= 2) lat_pts += sg.R * sg.C;
    }
    if (mode < 0 && 2 * lat_pts < b->n) return MLB_OK;
    // items: <= rows_cap rows of one segment (about a CTA's share of the points)
    const int nsm = b->plan->nsm;
    int64_t tgt = std::min<int64_t>(kLatPts, std::max<int64_t>(512, b->n / (nsm * 8)));
    if (const char* env = std::getenv("MLB_LAT_TGT")) tgt = std::max<int64_t>(64, std::min<int64_t>(kLatPts, std::atoll(env)));   // tuning
    std::vector<int32_t> items;
    std::vector<std::vector<int32_t>> bin_items((size_t)g.nb * g.nb);
    int nf_max = 1, r_max = 1, sv_max = 1;
    for (int k = 0; k < nkeys; ++k) {
        segments(k, segs);
        if (segs.empty()) continue;
        const int gc = key_gcell[k];
        const int bin = (gc / g.L) * g.nb + gc % g.L;
        for (const Seg& sg : segs) {
            const int C = sg.C, fast = sg.fast, diag = sg.diag;
            const int64_t R = sg.R;
            int64_t rows_cap = diag ? kLatRowsMax : std::max<int64_t>(1, std::min<int64_t>(kLatRowsMax, tgt / C));
            if (!diag) rows_cap = std::min<int64_t>(rows_cap, (int64_t)kLatGatherSlots * (kLatThreads / C));   // gather slots
            const int64_t nparts = (R + rows_cap - 1) / rows_cap;
            rows_cap = (R + nparts - 1) / nparts;   // even parts
            for (int64_t r0 = 0; r0 < R; r0 += rows_cap) {
                const int64_t rn = std::min(rows_cap, R - r0);
                bin_items[bin].push_back((int32_t)(items.size() / 4));
                items.push_back((int32_t)(sg.p0 + r0 * (diag ? 1 : C)));
                items.push_back((int32_t)rn);
                items.push_back(C | (fast << 16) | (diag << 17));
                items.push_back(gc);
                nf_max = std::max<int>(nf_max, diag ? (int)rn : C);
                r_max = std::max<int>(r_max, (int)rn);
                sv_max = std::max<int>(sv_max, diag ? (int)rn : (int)rn * (C | 1));
            }
        }
    }
    // items sorted by bin (CSR) so the reduction walks each bin's items in order
    std::vector<int32_t> items_sorted, bin_off((size_t)g.nb * g.nb + 1, 0);
    items_sorted.reserve(items.size());
    for (size_t bin = 0; bin < bin_items.size(); ++bin) {
        bin_off[bin + 1] = bin_off[bin] + (int32_t)bin_items[bin].size();
        for (int32_t t : bin_items[bin]) items_sorted.insert(items_sorted.end(), items.begin() + 4 * t, items.begin() + 4 * t + 4);
    }
    const int nitems = (int)(items_sorted.size() / 4);
    const int S = 2 * g.m + 1;
    b->lat_nitems = nitems;
    b->lat_points = lat_pts;
    b->lat_nf_max = nf_max;
    b->lat_r_max = r_max;
    b->lat_sv_max = sv_max;
    auto up = [&](int32_t** dst, const std::vector<int32_t>& h) -> int {
        MLB_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, h.size()) * sizeof(int32_t)));
        MLB_CUDA_TRY(cudaMemcpy(*dst, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        return MLB_OK;
    };
    if (int rc = up(&b->lat_items, items_sorted)) return rc;
    if (int rc = up(&b->lat_bin_off, bin_off)) return rc;
    MLB_CUDA_TRY(cudaMalloc(&b->lat_blocks, std::max<size_t>(1, (size_t)nitems * S * S) * sizeof(double)));
    if (std::getenv("MLB_DEBUG"))
        fprintf(stderr, "[mlb] d2 lattice: %d items, %lld of %lld points in lattice cells, widest %d\n", nitems,
                (long long)lat_pts, (long long)b->n, nf_max);
    return MLB_OK;
}

}  // namespace mlb
