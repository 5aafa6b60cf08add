// NFFT fast-summation kernels for sm_100a: spread, partial-tile reduce,
// pruned separable DFT convolution, gather with the fused D^-1/2 epilogue.
//
// Reference chain (fastsum.py:475-497): spread (bincount, :389-391) ->
// rfftn * fused_weights * irfftn (:492-495) -> gather (bincount, :400-406)
// -> minus K(0) v.  The graph wrapper (graphs.py:197-201) adds the D^-1/2
// scalings and the shift; here they are fused into spread and gather.
//
// Layout:
//   * points are counting-sorted by (brick, cell); chunks are <= 32 points of
//     one cell; segments are <= max_seg_chunks chunks of one brick;
//   * a brick is Tb^d cells whose stencils cover a (Tb+2m)^d tile;
//   * the grid is only the active sub-box of L^d cells (u = ulo..ulo+L-1 per
//     axis); the FFT stage is a pruned DFT between that sub-box and the
//     (N+1)^(d-1) x (N/2+1) band where the fused weights are nonzero.
#include <cuda_runtime.h>

#include <algorithm>

#include "mlb_internal.cuh"
#include "mlb_window.cuh"

namespace mlb {

// ---------------------------------------------------------------- configs --
// Lane ownership of the (2M+1)^D stencil in the spread: lanes split axis a
// into P_a blocks of B_a cells; NPASS splits axis D-1 into passes so the
// per-lane accumulator block (B0*B1*B2 doubles) stays in registers.
template <int D, int M>
struct SpreadCfg;

template <int M>
struct SpreadCfg<1, M> {
    static constexpr int S = 2 * M + 1;
    static constexpr int P0 = S, P1 = 1, P2 = 1;
    static constexpr int B0 = 1, B1 = 1, B2 = 1;
    static constexpr int NPASS = 1, SP = S;
};
template <int M>
struct SpreadCfg<2, M> {
    static constexpr int S = 2 * M + 1;
    static constexpr int P0 = S, P1 = 32 / S, P2 = 1;
    static constexpr int B0 = 1, B1 = (S + P1 - 1) / P1, B2 = 1;
    static constexpr int NPASS = 1, SP = S;
};
template <int M>
struct SpreadCfg<3, M> {
    static constexpr int S = 2 * M + 1;
    static constexpr bool small = (M <= 4);
    static constexpr int P0 = small ? 3 : 4, P1 = small ? 3 : 4, P2 = small ? 3 : 2;
    static constexpr int NPASS = (M >= 6) ? 2 : 1;
    static constexpr int SP = (S + NPASS - 1) / NPASS;  // cells of axis 2 per pass
    static constexpr int B0 = (S + P0 - 1) / P0, B1 = (S + P1 - 1) / P1, B2 = (SP + P2 - 1) / P2;
};

constexpr int kWinPad = 17;  // staged window row stride (>= every P*B reach; odd -> no bank conflicts)

struct FsArgs {
    Geom g;
    int64_t n;
    const int32_t* perm;
    const double* frac;
    const int32_t* chunk_start;
    const int32_t* chunk_cell;
    const int32_t* seg_chunk;
    const int32_t* seg_brick;
    const int32_t* brick_seg;
    const double* isd;
    double* partial;
    int tile_cells;
};

__device__ __forceinline__ int ipow(int b, int e) {
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

// ----------------------------------------------------------------- spread --
// One CTA per segment.  Each warp owns a private smem copy of the brick tile
// and a contiguous share of the segment's chunks.  Per chunk: lanes compute
// the d(2m+1) window values of one point each (v*s folded into axis 0) into
// smem staging; then every lane accumulates its stencil block over the
// chunk's points in registers (all points of a chunk share one cell, so the
// block is fixed) and flushes into its warp tile when the cell changes.
// No atomics: warp tiles are summed in a fixed order -> bitwise reproducible.
template <int D, int M>
__global__ void __launch_bounds__(256) spread_kernel(FsArgs a, WinCoef wc, const double* __restrict__ v,
                                                     unsigned flags) {
    using C = SpreadCfg<D, M>;
    constexpr int S = C::S;
    extern __shared__ double smem[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TL = a.g.TL;
    const int tile = a.tile_cells;
    double* tiles = smem;                                   // nw * tile
    double* stage = smem + (size_t)nw * tile;               // nw * 32 * D * kWinPad
    double* my_tile = tiles + (size_t)warp * tile;
    double* my_stage = stage + (size_t)warp * 32 * D * kWinPad;

    for (int i = threadIdx.x; i < nw * tile; i += blockDim.x) tiles[i] = 0.0;
    for (int i = lane; i < 32 * D * kWinPad; i += 32) my_stage[i] = 0.0;
    __syncthreads();

    const int seg = blockIdx.x;
    const int c0 = a.seg_chunk[seg], c1 = a.seg_chunk[seg + 1];
    const int nch = c1 - c0;
    const int my0 = c0 + (int)(((long long)nch * warp) / nw);
    const int my1 = c0 + (int)(((long long)nch * (warp + 1)) / nw);

    const int l0 = lane / (C::P1 * C::P2), l1 = (lane / C::P2) % C::P1, l2 = lane % C::P2;
    const bool active = lane < C::P0 * C::P1 * C::P2;
    const int TL2 = (D == 3) ? TL * TL : 1;
    const int TL1 = (D >= 2) ? TL : 1;

    for (int pass = 0; pass < C::NPASS; ++pass) {
        const int off2 = pass * C::SP;
        double acc[C::B0][C::B1][C::B2];
#pragma unroll
        for (int i = 0; i < C::B0; ++i)
#pragma unroll
            for (int j = 0; j < C::B1; ++j)
#pragma unroll
                for (int k = 0; k < C::B2; ++k) acc[i][j][k] = 0.0;
        int cur = -1;

        auto flush = [&](int cell) {
            if (!active || cell < 0) return;
#pragma unroll
            for (int i = 0; i < C::B0; ++i) {
                const int o0 = l0 * C::B0 + i;
#pragma unroll
                for (int j = 0; j < C::B1; ++j) {
                    const int o1 = l1 * C::B1 + j;
#pragma unroll
                    for (int k = 0; k < C::B2; ++k) {
                        const int o2 = off2 + l2 * C::B2 + k;
                        bool ok = (o0 < S);
                        if (D >= 2) ok = ok && (o1 < S);
                        if (D == 3) ok = ok && (o2 < S) && (l2 * C::B2 + k < C::SP);
                        if (ok) {
                            int t;
                            if (D == 1) t = cell + o0;
                            else if (D == 2) t = cell + o0 * TL1 + o1;
                            else t = cell + o0 * TL2 + o1 * TL1 + o2;
                            my_tile[t] += acc[i][j][k];
                        }
                        acc[i][j][k] = 0.0;
                    }
                }
            }
        };

        for (int ch = my0; ch < my1; ++ch) {
            const int cell = a.chunk_cell[ch];
            const int p0 = a.chunk_start[ch];
            const int np = a.chunk_start[ch + 1] - p0;
            if (cell != cur) {
                flush(cur);
                cur = cell;
            }
            __syncwarp();
            if (lane < np) {
                const int p = p0 + lane;
                const int node = (flags & MLB_SORTED) ? p : a.perm[p];
                double val = __ldg(v + node);
                if (flags & MLB_USE_ISD) val *= __ldg(a.isd + p);
                double w[S];
#pragma unroll
                for (int ax = 0; ax < D; ++ax) {
                    kb_windows<M>(__ldg(a.frac + (int64_t)ax * a.n + p), wc, w);
                    double* dst = my_stage + (lane * D + ax) * kWinPad;
#pragma unroll
                    for (int o = 0; o < S; ++o) dst[o] = (ax == 0) ? w[o] * val : w[o];
                }
            }
            __syncwarp();
            if (active) {
                for (int jp = 0; jp < np; ++jp) {
                    const double* ws = my_stage + jp * D * kWinPad;
                    double w0[C::B0], w1[C::B1], w2[C::B2];
#pragma unroll
                    for (int i = 0; i < C::B0; ++i) w0[i] = ws[l0 * C::B0 + i];
#pragma unroll
                    for (int j = 0; j < C::B1; ++j) w1[j] = (D >= 2) ? ws[kWinPad + l1 * C::B1 + j] : 1.0;
#pragma unroll
                    for (int k = 0; k < C::B2; ++k)
                        w2[k] = (D == 3) ? ws[2 * kWinPad + off2 + l2 * C::B2 + k] : 1.0;
#pragma unroll
                    for (int i = 0; i < C::B0; ++i)
#pragma unroll
                        for (int j = 0; j < C::B1; ++j) {
                            const double w01 = w0[i] * w1[j];
#pragma unroll
                            for (int k = 0; k < C::B2; ++k) acc[i][j][k] = fma(w01, w2[k], acc[i][j][k]);
                        }
                }
            }
        }
        flush(cur);
        __syncwarp();
    }
    __syncthreads();
    // fixed-order sum of the warp tiles -> this segment's partial tile
    double* out = a.partial + (size_t)seg * tile;
    for (int i = threadIdx.x; i < tile; i += blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += tiles[(size_t)w * tile + i];
        out[i] = s;
    }
}

// ------------------------------------------------------------------ reduce --
// grid[u] = sum over the bricks whose tile covers u, over their segments in
// order, of partial[seg][u - brick_origin].  One thread per active cell.
template <int D>
__global__ void reduce_kernel(FsArgs a, double* __restrict__ grid) {
    const Geom g = a.g;
    const int L = g.L, Tb = g.Tb, TL = g.TL, nbr = g.nbr;
    int64_t total = 1;
    for (int i = 0; i < D; ++i) total *= L;
    for (int64_t cidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cidx < total;
         cidx += (int64_t)gridDim.x * blockDim.x) {
        int u[3] = {0, 0, 0};
        int64_t r = cidx;
        for (int ax = D - 1; ax >= 0; --ax) {
            u[ax] = (int)(r % L);
            r /= L;
        }
        int blo[3] = {0, 0, 0}, bhi[3] = {0, 0, 0};
        for (int ax = 0; ax < D; ++ax) {
            int lo = u[ax] - TL + 1;
            lo = lo <= 0 ? 0 : (lo + Tb - 1) / Tb;
            int hi = u[ax] / Tb;
            if (hi > nbr - 1) hi = nbr - 1;
            blo[ax] = lo;
            bhi[ax] = hi;
        }
        double s = 0.0;
        for (int b0 = blo[0]; b0 <= bhi[0]; ++b0)
            for (int b1 = (D >= 2 ? blo[1] : 0); b1 <= (D >= 2 ? bhi[1] : 0); ++b1)
                for (int b2 = (D == 3 ? blo[2] : 0); b2 <= (D == 3 ? bhi[2] : 0); ++b2) {
                    int brick, t;
                    if (D == 1) {
                        brick = b0;
                        t = u[0] - b0 * Tb;
                    } else if (D == 2) {
                        brick = b0 * nbr + b1;
                        t = (u[0] - b0 * Tb) * TL + (u[1] - b1 * Tb);
                    } else {
                        brick = (b0 * nbr + b1) * nbr + b2;
                        t = ((u[0] - b0 * Tb) * TL + (u[1] - b1 * Tb)) * TL + (u[2] - b2 * Tb);
                    }
                    const int s0 = a.brick_seg[brick], s1 = a.brick_seg[brick + 1];
                    for (int sg = s0; sg < s1; ++sg) s += a.partial[(size_t)sg * a.tile_cells + t];
                }
        grid[cidx] = s;
    }
}

// ---------------------------------------------------------------- DFT stage --
// out[a][k][b] = sum_u in[a][u][b] T(u,k).  Modes:
//   0: forward real->complex on the last axis (k = 0..N/2), B = 1
//   1: forward complex->complex (k = -N/2..N/2)
//   2: mode 1, then multiply by the fused band weights (last forward stage)
//   3: inverse complex->complex (sum over k, output u)
//   4: inverse complex->real on the last axis, Hermitian weights 1,2,2,..
//   5: mode 0 then multiply (d = 1)
struct DftArgs {
    const double* in;
    double* out;
    int A, U, Kout, B;
    const double2* tw;
    int K;        // twiddle row stride
    int koff;     // column offset into twiddle rows
    const double* fused;
};

template <int MODE>
__global__ void dft_kernel(DftArgs p) {
    const int64_t total = (int64_t)p.A * p.Kout * p.B;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(idx % p.B);
        const int k = (int)((idx / p.B) % p.Kout);
        const int64_t aa = idx / ((int64_t)p.B * p.Kout);
        double re = 0.0, im = 0.0;
        if (MODE == 0 || MODE == 5) {
            const double* x = p.in + aa * p.U;
            for (int u = 0; u < p.U; ++u) {
                const double2 t = p.tw[u * p.K + k + p.koff];
                const double xv = x[u];
                re = fma(xv, t.x, re);
                im = fma(xv, t.y, im);
            }
        } else if (MODE == 1 || MODE == 2) {
            const double2* x = reinterpret_cast<const double2*>(p.in) + aa * (int64_t)p.U * p.B + b;
            for (int u = 0; u < p.U; ++u) {
                const double2 t = p.tw[u * p.K + k + p.koff];
                const double2 xv = x[(int64_t)u * p.B];
                re = fma(xv.x, t.x, fma(-xv.y, t.y, re));
                im = fma(xv.x, t.y, fma(xv.y, t.x, im));
            }
        } else if (MODE == 3) {
            // here U = number of frequencies summed, Kout = L output cells
            const double2* x = reinterpret_cast<const double2*>(p.in) + aa * (int64_t)p.U * p.B + b;
            for (int kk = 0; kk < p.U; ++kk) {
                const double2 t = p.tw[k * p.K + kk + p.koff];  // conj applied below
                const double2 xv = x[(int64_t)kk * p.B];
                re = fma(xv.x, t.x, fma(xv.y, t.y, re));
                im = fma(xv.y, t.x, fma(-xv.x, t.y, im));
            }
        } else {  // MODE == 4
            const double2* x = reinterpret_cast<const double2*>(p.in) + aa * p.U;
            for (int kk = 0; kk < p.U; ++kk) {
                const double2 t = p.tw[k * p.K + kk + p.koff];
                const double2 xv = x[kk];
                const double wgt = (kk == 0) ? 1.0 : 2.0;
                re = fma(wgt, fma(xv.x, t.x, xv.y * t.y), re);
            }
        }
        if (MODE == 2 || MODE == 5) {
            const double f = p.fused[(int64_t)k * p.B + b];
            re *= f;
            im *= f;
        }
        if (MODE == 4) {
            p.out[aa * p.Kout + k] = re;
        } else {
            reinterpret_cast<double2*>(p.out)[(aa * p.Kout + k) * (int64_t)p.B + b] = make_double2(re, im);
        }
    }
}

template <int MODE>
static void run_dft(const DftArgs& p, cudaStream_t st) {
    const int64_t total = (int64_t)p.A * p.Kout * p.B;
    int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    dft_kernel<MODE><<<(int)blocks, threads, 0, st>>>(p);
}

// ------------------------------------------------------------------ gather --
// One CTA per segment: stage the brick tile of the convolved grid in smem,
// then one point per lane: y = alpha v + s (beta acc + gamma s v).
template <int D, int M>
__global__ void __launch_bounds__(256) gather_kernel(FsArgs a, WinCoef wc, const double* __restrict__ grid,
                                                     const double* __restrict__ v, double* __restrict__ y,
                                                     double alpha, double beta, double gamma, unsigned flags) {
    constexpr int S = 2 * M + 1;
    extern __shared__ double smem[];
    const Geom g = a.g;
    const int L = g.L, TL = g.TL, Tb = g.Tb, nbr = g.nbr;
    const int seg = blockIdx.x;
    const int brick = a.seg_brick[seg];
    int bo[3] = {0, 0, 0};
    {
        int r = brick;
        for (int ax = D - 1; ax >= 0; --ax) {
            bo[ax] = (r % nbr) * Tb;
            r /= nbr;
        }
    }
    double* tile = smem;
    const int tile_cells = a.tile_cells;
    for (int i = threadIdx.x; i < tile_cells; i += blockDim.x) {
        int t[3] = {0, 0, 0};
        int r = i;
        for (int ax = D - 1; ax >= 0; --ax) {
            t[ax] = r % TL;
            r /= TL;
        }
        bool ok = true;
        int64_t gi = 0;
        for (int ax = 0; ax < D; ++ax) {
            const int u = bo[ax] + t[ax];
            ok = ok && (u < L);
            gi = gi * L + u;
        }
        tile[i] = ok ? grid[gi] : 0.0;
    }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = a.seg_chunk[seg], c1 = a.seg_chunk[seg + 1];
    const int TL1 = (D >= 2) ? TL : 1;
    const int TL2 = (D == 3) ? TL * TL : 1;
    for (int ch = c0 + warp; ch < c1; ch += nw) {
        const int cell = a.chunk_cell[ch];
        const int p0 = a.chunk_start[ch];
        const int np = a.chunk_start[ch + 1] - p0;
        if (lane >= np) continue;
        const int p = p0 + lane;
        double w0[S], w1[S], w2[S];
        kb_windows<M>(__ldg(a.frac + p), wc, w0);
        if (D >= 2) kb_windows<M>(__ldg(a.frac + a.n + p), wc, w1);
        if (D == 3) kb_windows<M>(__ldg(a.frac + 2 * a.n + p), wc, w2);
        double acc = 0.0;
        const double* tb = tile + cell;
        if (D == 1) {
#pragma unroll
            for (int i = 0; i < S; ++i) acc = fma(w0[i], tb[i], acc);
        } else if (D == 2) {
#pragma unroll
            for (int i = 0; i < S; ++i) {
                double r1 = 0.0;
#pragma unroll
                for (int j = 0; j < S; ++j) r1 = fma(w1[j], tb[i * TL1 + j], r1);
                acc = fma(w0[i], r1, acc);
            }
        } else {
#pragma unroll 1
            for (int i = 0; i < S; ++i) {
                const double* ti = tb + i * TL2;
                double r1 = 0.0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    double r2 = 0.0;
#pragma unroll
                    for (int k = 0; k < S; ++k) r2 = fma(w2[k], ti[j * TL1 + k], r2);
                    r1 = fma(w1[j], r2, r1);
                }
                // w0[i] with a runtime i: select through a small unrolled scan
                double wi = 0.0;
#pragma unroll
                for (int q = 0; q < S; ++q) wi = (q == i) ? w0[q] : wi;
                acc = fma(wi, r1, acc);
            }
        }
        const int node = (flags & MLB_SORTED) ? p : a.perm[p];
        const double vv = v ? __ldg(v + node) : 0.0;
        const double s = (flags & MLB_USE_ISD) ? __ldg(a.isd + p) : 1.0;
        double res = alpha * vv + s * (beta * acc + gamma * s * vv);
        if (flags & MLB_ACCUMULATE) res += y[node];
        y[node] = res;
    }
}

// --------------------------------------------------------------- launchers --
static FsArgs make_args(mlb_binding* b) {
    FsArgs a;
    a.g = b->plan->g;
    a.n = b->n;
    a.perm = b->perm;
    a.frac = b->frac;
    a.chunk_start = b->chunk_start;
    a.chunk_cell = b->chunk_cell;
    a.seg_chunk = b->seg_chunk;
    a.seg_brick = b->seg_brick;
    a.brick_seg = b->brick_seg;
    a.isd = b->isd;
    a.partial = b->partial;
    a.tile_cells = b->tile_cells;
    return a;
}

static int spread_warps(int D, int tile_cells) {
    // warp-private tiles + window staging must fit in ~200 KB of smem
    const size_t per_warp = (size_t)tile_cells * 8 + 32 * D * kWinPad * 8;
    int nw = (int)(200 * 1024 / per_warp);
    return std::max(1, std::min(8, nw));
}

template <int D, int M>
static int spread_dm(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st) {
    FsArgs a = make_args(b);
    const int nw = spread_warps(D, b->tile_cells);
    const size_t smem = (size_t)nw * b->tile_cells * 8 + (size_t)nw * 32 * D * kWinPad * 8;
    auto kern = spread_kernel<D, M>;
    MLB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<b->nseg, nw * 32, smem, st>>>(a, b->plan->wc, v, flags);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

template <int D, int M>
static int gather_dm(mlb_binding* b, const double* grid, const double* v, double* y, double alpha,
                     double beta, double gamma, unsigned flags, cudaStream_t st) {
    FsArgs a = make_args(b);
    const size_t smem = (size_t)b->tile_cells * 8;
    auto kern = gather_kernel<D, M>;
    MLB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<b->nseg, 256, smem, st>>>(a, b->plan->wc, grid, v, y, alpha, beta, gamma, flags);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

#define MLB_DISPATCH_DM(FN, D, M, ...)                                   \
    switch ((D) * 10 + (M)) {                                            \
        case 12: return FN<1, 2>(__VA_ARGS__);                           \
        case 13: return FN<1, 3>(__VA_ARGS__);                           \
        case 14: return FN<1, 4>(__VA_ARGS__);                           \
        case 15: return FN<1, 5>(__VA_ARGS__);                           \
        case 16: return FN<1, 6>(__VA_ARGS__);                           \
        case 22: return FN<2, 2>(__VA_ARGS__);                           \
        case 23: return FN<2, 3>(__VA_ARGS__);                           \
        case 24: return FN<2, 4>(__VA_ARGS__);                           \
        case 25: return FN<2, 5>(__VA_ARGS__);                           \
        case 26: return FN<2, 6>(__VA_ARGS__);                           \
        case 32: return FN<3, 2>(__VA_ARGS__);                           \
        case 33: return FN<3, 3>(__VA_ARGS__);                           \
        case 34: return FN<3, 4>(__VA_ARGS__);                           \
        case 35: return FN<3, 5>(__VA_ARGS__);                           \
        case 36: return FN<3, 6>(__VA_ARGS__);                           \
        default: return fail(MLB_ERR_CONFIG, "unsupported (d, m)");      \
    }

int launch_spread(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st) {
    if (b->nseg == 0) return MLB_OK;
    const Geom& g = b->plan->g;
    MLB_DISPATCH_DM(spread_dm, g.d, g.m, b, v, flags, st);
}

int launch_reduce(mlb_binding* b, double* grid, cudaStream_t st) {
    FsArgs a = make_args(b);
    const int64_t total = b->grid_cells;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    switch (b->plan->g.d) {
        case 1: reduce_kernel<1><<<(int)blocks, 256, 0, st>>>(a, grid); break;
        case 2: reduce_kernel<2><<<(int)blocks, 256, 0, st>>>(a, grid); break;
        default: reduce_kernel<3><<<(int)blocks, 256, 0, st>>>(a, grid); break;
    }
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_convolve(mlb_binding* b, const double* gin, double* gout, cudaStream_t st) {
    const Geom& g = b->plan->g;
    const int L = g.L, K = g.K, Kh = g.Kh, half = g.N / 2;
    DftArgs p;
    p.tw = b->plan->twid;
    p.K = K;
    p.fused = b->plan->fused;
    double* A = b->stage_a;
    double* B = b->stage_b;
    if (g.d == 1) {
        p = {gin, A, 1, L, Kh, 1, b->plan->twid, K, half, b->plan->fused};
        run_dft<5>(p, st);
        p = {A, gout, 1, Kh, L, 1, b->plan->twid, K, half, nullptr};
        run_dft<4>(p, st);
    } else if (g.d == 2) {
        p = {gin, A, L, L, Kh, 1, b->plan->twid, K, half, nullptr};  // [u0][k1]
        run_dft<0>(p, st);
        p = {A, B, 1, L, K, Kh, b->plan->twid, K, 0, b->plan->fused};  // [k0][k1] * F
        run_dft<2>(p, st);
        p = {B, A, 1, K, L, Kh, b->plan->twid, K, 0, nullptr};  // [u0][k1]
        run_dft<3>(p, st);
        p = {A, gout, L, Kh, L, 1, b->plan->twid, K, half, nullptr};  // [u0][u1]
        run_dft<4>(p, st);
    } else {
        p = {gin, A, L * L, L, Kh, 1, b->plan->twid, K, half, nullptr};  // [u0][u1][k2]
        run_dft<0>(p, st);
        p = {A, B, L, L, K, Kh, b->plan->twid, K, 0, nullptr};  // [u0][k1][k2]
        run_dft<1>(p, st);
        p = {B, A, 1, L, K, K * Kh, b->plan->twid, K, 0, b->plan->fused};  // [k0][k1][k2] * F
        run_dft<2>(p, st);
        p = {A, B, 1, K, L, K * Kh, b->plan->twid, K, 0, nullptr};  // [u0][k1][k2]
        run_dft<3>(p, st);
        p = {B, A, L, K, L, Kh, b->plan->twid, K, 0, nullptr};  // [u0][u1][k2]
        run_dft<3>(p, st);
        p = {A, gout, L * L, Kh, L, 1, b->plan->twid, K, half, nullptr};  // [u0][u1][u2]
        run_dft<4>(p, st);
    }
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_gather(mlb_binding* b, const double* grid, const double* v, double* y, double alpha, double beta,
                  double gamma, unsigned flags, cudaStream_t st) {
    if (b->nseg == 0) return MLB_OK;
    const Geom& g = b->plan->g;
    MLB_DISPATCH_DM(gather_dm, g.d, g.m, b, grid, v, y, alpha, beta, gamma, flags, st);
}

}  // namespace mlb
