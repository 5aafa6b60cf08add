// NFFT fast-summation kernels for sm_100a: spread, deterministic partial-tile
// reduce, gather with the fused D^-1/2 epilogue (the convolution between them
// is mlb_dft.cu).
//
// Reference chain (fastsum.py:475-497): spread (bincount, :389-391) ->
// rfftn * fused_weights * irfftn (:492-495) -> gather (bincount, :400-406)
// -> minus K(0) v.  The graph wrapper (graphs.py:197-201) adds the D^-1/2
// scalings and the shift; here they are fused into spread and gather.
//
// Layout:
//   * points are counting-sorted by (brick, cell); a chunk is <= 64 points
//     of one cell; a segment is <= max_seg_chunks chunks of one brick;
//   * a brick is Tb^d cells whose stencils cover a (Tb+2m)^d tile;
//   * the grid is only the active sub-box of L^d cells (u = ulo..ulo+L-1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>
#include <cstdlib>

#include "mlb_internal.cuh"
#include "mlb_window.cuh"
#include "mlb_tma.cuh"

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
// d = 3: lane (i, j-block) owns one axis-0 offset, B1 axis-1 offsets and a
// whole axis-2 row, so each product w0[i] w1[j] is formed by exactly one lane
// (no redundant DMULs) and w2 is a broadcast read; NPASS splits axis 2 so the
// B1 x SP accumulator block stays <= 36 doubles.
template <int M>
struct SpreadCfg<3, M> {
    static constexpr int S = 2 * M + 1;
    static constexpr int P0 = S, P1 = 32 / S, P2 = 1;
    static constexpr int B0 = 1, B1 = (S + P1 - 1) / P1;
    // m >= 5 runs one 8-warp CTA per SM (shared memory), so it can hold 72
    // accumulators per lane: fewer passes = fewer window evaluations
    static constexpr int ACC = (M >= 5) ? 72 : 36;
    static constexpr int NPASS = (B1 * S <= ACC) ? 1 : ((B1 * ((S + 1) / 2) <= ACC) ? 2 : 3);
    static constexpr int SP = (S + NPASS - 1) / NPASS;  // cells of axis 2 per pass
    static constexpr int B2 = SP;
};

// staged window row stride: covers every lane's reach (entries >= S stay 0)
// and is odd (conflict-free 8-byte rows across lanes)
template <int D, int M>
struct StageCfg {
    using C = SpreadCfg<D, M>;
    static constexpr int r0 = C::P0 * C::B0;
    static constexpr int r1 = C::P1 * C::B1;
    static constexpr int r2 = (C::NPASS - 1) * C::SP + C::P2 * C::B2;
    static constexpr int reach = (r0 > r1 ? (r0 > r2 ? r0 : r2) : (r1 > r2 ? r1 : r2));
    // d = 3: even stride so the broadcast axis-2 row is read as 16-byte pairs
    static constexpr bool vec2 = (D == 3) && (C::NPASS == 1 || C::SP % 2 == 0);
    // d = 2 (grouped lanes, see spread_kernel): stride = 1 mod 8 doubles, so
    // the 8 point rows x 2 interleaved offsets one load touches are 16
    // distinct 8-byte bank pairs
    static constexpr int pad2 = ((C::S + 6) / 8) * 8 + 1;
    static constexpr int pad = (D == 2) ? pad2 : (vec2 ? (reach + (reach & 1)) : ((reach % 2) ? reach : reach + 1));
};

struct FsArgs {
    Geom g;
    int64_t n;
    const int32_t* perm;
    const double* frac;
    const int32_t* chunk_start;
    const int32_t* chunk_cell;
    const int32_t* chunk_gcell;
    const int2* sub_desc;     // sub-chunks in segment order: {first point, (count << 24) | tile cell}
    const int32_t* seg_sub;   // nseg + 1: CSR of sub-chunks per segment
    const int32_t* seg_chunk;
    const int32_t* seg_brick;
    const int32_t* brick_seg;
    const int32_t* brick_first;
    const double* isd;
    double* partial;
    // d = 3 cell blocks
    const int4* cblk;
    const int2* wstream;
    const int32_t* wstream_off;
    const int32_t* citem;
    const int32_t* citem_off;
    const int32_t* brick_blk;
    const int32_t* active_brick;
    const int32_t* merge_off;
    const int32_t* merge_pairs;
    double* blocks;
    const int2* ggrp;
    const int32_t* gslot;
    int ngrp;
    int tile_cells;
    int nchunks;
    int nseg;
    // d = 3 atomic mode (MLB_SPREAD_ATOMIC=1, A/B only): cell blocks are added
    // into this zeroed sub-box grid with red.global.add.f64 (no merge / R2;
    // not bitwise reproducible); nullptr: the deterministic blocks
    double* agrid;
    // d = 2 banded spread: CTA c owns segments [cta_seg[c], cta_seg[c+1])
    // (nullptr: warps take segments gw, gw + W, ... over the whole list)
    const int32_t* cta_seg;
    // d = 1 streaming spread / gather: first sorted point of every cell (nkeys + 1)
    const int32_t* key_start;
    int nkeys;
};

// sub-box index of element (o01 = o0*S + o1, o2) of d = 3 cell block `blk`
__device__ __forceinline__ int64_t block_grid_index(const FsArgs& a, int blk, int o01, int o2) {
    const int4 cb = __ldg(a.cblk + blk);
    const int S = a.g.S, TL = a.g.TL, Tb = a.g.Tb, nbr = a.g.nbr, L = a.g.L;
    const int c0 = cb.z / (TL * TL), c1 = (cb.z / TL) % TL, c2 = cb.z % TL;
    const int B0 = cb.w / (nbr * nbr), B1 = (cb.w / nbr) % nbr, B2 = cb.w % nbr;
    const int u0 = B0 * Tb + c0 + o01 / S, u1 = B1 * Tb + c1 + o01 % S, u2 = B2 * Tb + c2 + o2;
    return ((int64_t)u0 * L + u1) * L + u2;
}

// ----------------------------------------------------------------- spread --
// Warps own segments statically (gw, gw + W, ...).  A segment is a list of
// sub-chunks (<= 32 cell-sorted points of ONE cell; descriptor table built at
// bind time), walked through a 3-deep software pipeline so that no load waits
// on another in the steady state: descriptors 3 sub-chunks ahead, point
// indices (perm) 2 ahead, coordinates / D^-1/2 / v 1 ahead.
// Per sub-chunk each lane evaluates one point's d(2m+1) windows (v s folded
// into axis 0) into smem staging; then the lanes, which own disjoint blocks
// of the (2m+1)^d stencil, accumulate the sub-chunk's points in registers and
// flush into the warp's smem brick tile when the cell changes.  PERSIST
// (d <= 2: one brick = the whole sub-box) keeps the tile across segments and
// the CTA sums its warp tiles into one partial grid; otherwise every segment
// writes its own partial tile.  No atomics -> bitwise reproducible.
struct SubPos {
    int sub;   // global sub-chunk index, -1 = no more work
    int seg;   // its segment
    int end;   // one past the segment's last sub-chunk
};

__device__ __forceinline__ SubPos sub_first(const FsArgs& a, int seg, int seg_end) {
    SubPos p;
    if (seg >= seg_end) {
        p.sub = -1;
        p.seg = seg;
        p.end = 0;
        return p;
    }
    p.sub = __ldg(a.seg_sub + seg);
    p.end = __ldg(a.seg_sub + seg + 1);
    p.seg = seg;
    return p;
}

__device__ __forceinline__ SubPos sub_next(const FsArgs& a, SubPos p, int nwarps, int seg_end) {
    if (p.sub < 0) return p;
    if (p.sub + 1 < p.end) {
        p.sub += 1;
        return p;
    }
    return sub_first(a, p.seg + nwarps, seg_end);
}

// body of spread_kernel; `bid` / `nblk` stand for blockIdx.x / gridDim.x (the
// multi-layer launch gives every layer its own block count along x)
template <int D, int M, bool PERSIST, bool GROUPED>
__device__ __forceinline__ void spread_body(const FsArgs& a, const WinCoef& wc, const double* __restrict__ v,
                                            unsigned flags, int bid, int nblk) {
    using C = SpreadCfg<D, M>;
    constexpr int S = C::S;
    constexpr int SPAD = StageCfg<D, M>::pad;
    extern __shared__ double smem[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TL = a.g.TL;
    const int tile = a.tile_cells;
    double* my_tile = smem + (size_t)warp * tile;
    // (d = 2: + 8 doubles so the grouped reads of the last row's unused
    // offsets stay inside the warp's staging)
    constexpr int STAGE = 32 * D * SPAD + (D == 2 ? 8 : 0);
    double* my_stage = smem + (size_t)nw * tile + (size_t)warp * STAGE;
    for (int i = lane; i < STAGE; i += 32) my_stage[i] = 0.0;
    for (int i = lane; i < tile; i += 32) my_tile[i] = 0.0;
    pdl_wait();  // v (and the partial grids' previous readers) are stream predecessors

    const int l0 = lane / (C::P1 * C::P2), l1 = (lane / C::P2) % C::P1, l2 = lane % C::P2;
    const bool active = lane < C::P0 * C::P1 * C::P2;
    const int TL2 = (D == 3) ? TL * TL : 1;
    const int TL1 = (D >= 2) ? TL : 1;
    // segment walk: banded CTAs own a contiguous range, else global round-robin
    const bool banded = a.cta_seg != nullptr;
    const int gwarp = banded ? __ldg(a.cta_seg + bid) + warp : bid * nw + warp;
    const int nwarps = banded ? nw : nblk * nw;
    const int seg_end = banded ? __ldg(a.cta_seg + bid + 1) : a.nseg;
    const bool sorted = (flags & MLB_SORTED) != 0;
    const bool use_isd = (flags & MLB_USE_ISD) != 0;

    // d = 2: 8 groups of 4 lanes; group g accumulates points g, g + 8, ... of
    // a sub-chunk, lane (a, b) of a group owns the interleaved stencil block
    // rows a + 2i x cols b + 2k (GB x GB entries, GB = ceil(S / 2)): per
    // point 2 GB loads feed GB^2 FMAs, and all 32 lanes are busy.  The groups'
    // blocks meet by a fixed xor-shuffle tree at every flush.
    constexpr int GB = (S + 1) / 2;
    const int g2 = lane >> 2, a2 = (lane >> 1) & 1, b2 = lane & 1;
    constexpr bool G2 = (D == 2) && GROUPED;
    double acc2[G2 ? GB : 1][G2 ? GB : 1];
    if constexpr (G2) {
#pragma unroll
        for (int i = 0; i < GB; ++i)
#pragma unroll
            for (int k = 0; k < GB; ++k) acc2[i][k] = 0.0;
    }
    (void)g2;
    (void)a2;
    (void)b2;
    // d = 1: every lane owns its point (sub-chunks never straddle a cell) and
    // accumulates its S windows in registers; the warp's S sums meet by a
    // fixed xor-shuffle tree only when the cell changes (dense cells: a few
    // times per segment).  No staging, no shared-memory traffic per point.
    constexpr bool R1 = (D == 1);
    double acc1[R1 ? S : 1];
#pragma unroll
    for (int o = 0; o < (R1 ? S : 1); ++o) acc1[o] = 0.0;

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
            if constexpr (R1) {
                if (cell < 0) return;
#pragma unroll
                for (int o = 0; o < S; ++o) {
                    double t = acc1[o];
#pragma unroll
                    for (int sh = 16; sh > 0; sh >>= 1) t += __shfl_xor_sync(0xffffffffu, t, sh);
                    if (lane == 0 && !(flags & (1u << 18))) my_tile[cell + o] += t;
                    acc1[o] = 0.0;
                }
                return;
            }
            if constexpr (G2) {
                if (cell < 0) return;
                if (flags & (1u << 18)) return;  // ablation (profiling only)
#pragma unroll
                for (int i = 0; i < GB; ++i)
#pragma unroll
                    for (int k = 0; k < GB; ++k) {
                        double v = acc2[i][k];
                        v += __shfl_xor_sync(0xffffffffu, v, 4);
                        v += __shfl_xor_sync(0xffffffffu, v, 8);
                        v += __shfl_xor_sync(0xffffffffu, v, 16);
                        const int o0 = a2 + 2 * i, o1 = b2 + 2 * k;
                        if (g2 == 0 && o0 < S && o1 < S) my_tile[cell + o0 * TL1 + o1] += v;
                        acc2[i][k] = 0.0;
                    }
                return;
            }
            if (!active || cell < 0) return;
            if (flags & (1u << 18)) return;  // ablation (profiling only)
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

        // pipeline: p0 (compute), p1 (data in flight), p2 (perm in flight), p3 (descriptor in flight)
        SubPos p0 = sub_first(a, gwarp, seg_end);
        SubPos p1 = sub_next(a, p0, nwarps, seg_end);
        SubPos p2 = sub_next(a, p1, nwarps, seg_end);
        SubPos p3 = sub_next(a, p2, nwarps, seg_end);
        int2 d0 = (p0.sub >= 0) ? __ldg(a.sub_desc + p0.sub) : make_int2(0, 0);
        int2 d1 = (p1.sub >= 0) ? __ldg(a.sub_desc + p1.sub) : make_int2(0, 0);
        int2 d2 = (p2.sub >= 0) ? __ldg(a.sub_desc + p2.sub) : make_int2(0, 0);
        int2 d3 = (p3.sub >= 0) ? __ldg(a.sub_desc + p3.sub) : make_int2(0, 0);
        auto np_of = [](int2 d) { return d.y >> 24; };
        // branch-free loads: lanes past the sub-chunk's count re-read its last
        // point (always a valid index) and are masked with v = 0 when consumed
        auto pidx = [&](int2 d) { return d.x + min(lane, max(np_of(d) - 1, 0)); };
        auto node_of = [&](int2 d) -> int {
            const int p = pidx(d);
            return sorted ? p : __ldg(a.perm + p);
        };
        auto load_data = [&](int2 d, int node, double* f, double& s, double& vv) {
            const int p = pidx(d);
#pragma unroll
            for (int ax = 0; ax < D; ++ax) f[ax] = __ldg(a.frac + (int64_t)ax * a.n + p);
            s = use_isd ? __ldg(a.isd + p) : 1.0;
            vv = __ldg(v + node);
        };
        int n1 = node_of(d1);
        int n2 = node_of(d2);
        double f0[D], s0, v0;
        load_data(d0, node_of(d0), f0, s0, v0);
        double f1[D], s1, v1;
        load_data(d1, n1, f1, s1, v1);
        int seg_cur = p0.seg;

        while (p0.sub >= 0) {
            const int np = np_of(d0);
            const int cell = d0.y & 0xffffff;
            if (!PERSIST && p0.seg != seg_cur) {
                // segment boundary: finish the previous segment's partial tile
                flush(cur);
                cur = -1;
                __syncwarp();
                if (!(flags & (1u << 19))) {
                    double* out = a.partial + (size_t)seg_cur * tile;
                    for (int i = lane; i < tile; i += 32) {
                        out[i] = (pass ? out[i] : 0.0) + my_tile[i];  // same warp owns the segment in every pass
                        my_tile[i] = 0.0;
                    }
                }
                __syncwarp();
                seg_cur = p0.seg;
            }
            if (cell != cur) {
                flush(cur);
                cur = cell;
            }
            __syncwarp();
            if (R1 && !(flags & (1u << 17))) {
                const double sv0 = (lane < np && p0.sub >= 0) ? s0 * v0 : 0.0;
                double w[S];
                kb_windows<M>(f0[0], wc, w);
#pragma unroll
                for (int o = 0; o < S; ++o) acc1[o] = fma(w[o], sv0, acc1[o]);
            } else if (!(flags & (1u << 17))) {  // bit 17: ablation (profiling only)
                const double sv0 = (lane < np && p0.sub >= 0) ? s0 * v0 : 0.0;
                if constexpr (G2) {
                    double w[D][S];
                    kb_windows_k<M, D>(f0, wc, w);   // both axes at once (one coefficient read each)
#pragma unroll
                    for (int ax = 0; ax < D; ++ax) {
                        double* dst = my_stage + (lane * D + ax) * SPAD;
#pragma unroll
                        for (int o = 0; o < S; ++o) dst[o] = (ax == 0) ? w[ax][o] * sv0 : w[ax][o];
                    }
                } else {   // (plain lanes: the joint form costs the 2-CTA residency on config 2)
                    double w[S];
#pragma unroll
                    for (int ax = 0; ax < D; ++ax) {
                        kb_windows<M>(f0[ax], wc, w);
                        double* dst = my_stage + (lane * D + ax) * SPAD;
#pragma unroll
                        for (int o = 0; o < S; ++o) dst[o] = (ax == 0) ? w[o] * sv0 : w[o];
                    }
                }
            }
            // advance the pipeline (loads of later sub-chunks overlap the accumulation)
            SubPos p4 = sub_next(a, p3, nwarps, seg_end);
            const int2 d4 = (p4.sub >= 0) ? __ldg(a.sub_desc + p4.sub) : make_int2(0, 0);
            const int n3 = node_of(d3);
            double f2[D], s2, v2;
            load_data(d2, n2, f2, s2, v2);
            __syncwarp();
            if (R1) {
                // (accumulated above, in registers)
            } else if (G2 && !(flags & (1u << 16))) {
                // grouped lanes: 8 points per step (rows past np carry v = 0)
                for (int j0 = 0; j0 < np; j0 += 8) {
                    const double* ws = my_stage + (j0 + g2) * D * SPAD;
                    double w0[GB], w1[GB];
#pragma unroll
                    for (int i = 0; i < GB; ++i) w0[i] = ws[a2 + 2 * i];
#pragma unroll
                    for (int k = 0; k < GB; ++k) w1[k] = ws[SPAD + b2 + 2 * k];
#pragma unroll
                    for (int i = 0; i < GB; ++i)
#pragma unroll
                        for (int k = 0; k < GB; ++k) acc2[i][k] = fma(w0[i], w1[k], acc2[i][k]);
                }
            } else if (active && !(flags & (1u << 16))) {  // bit 16: ablation (profiling only)
                // rows past np carry v = 0, so the loop may run to an even count;
                // the next point's windows are loaded while this one accumulates
                auto ldw = [&](int j, double* w0, double* w1, double* w2) {
                    const double* ws = my_stage + j * D * SPAD;
#pragma unroll
                    for (int i = 0; i < C::B0; ++i) w0[i] = ws[l0 * C::B0 + i];
#pragma unroll
                    for (int jj = 0; jj < C::B1; ++jj) w1[jj] = (D >= 2) ? ws[SPAD + l1 * C::B1 + jj] : 1.0;
                    if constexpr (StageCfg<D, M>::vec2) {
                        const double* w2p = ws + 2 * SPAD + off2;  // 16-byte aligned (P2 = 1)
#pragma unroll
                        for (int k = 0; k + 1 < C::B2; k += 2) {
                            const double2 t = *reinterpret_cast<const double2*>(w2p + k);
                            w2[k] = t.x;
                            w2[k + 1] = t.y;
                        }
                        if (C::B2 & 1) w2[C::B2 - 1] = w2p[C::B2 - 1];
                    } else {
#pragma unroll
                        for (int k = 0; k < C::B2; ++k) w2[k] = (D == 3) ? ws[2 * SPAD + off2 + l2 * C::B2 + k] : 1.0;
                    }
                };
                auto acc_pt = [&](const double* w0, const double* w1, const double* w2) {
                    if constexpr (D == 2) {  // one FMA per stencil entry: acc += (s v w0) w1
#pragma unroll
                        for (int i = 0; i < C::B0; ++i)
#pragma unroll
                            for (int jj = 0; jj < C::B1; ++jj) acc[i][jj][0] = fma(w0[i], w1[jj], acc[i][jj][0]);
                        return;
                    }
#pragma unroll
                    for (int i = 0; i < C::B0; ++i)
#pragma unroll
                        for (int jj = 0; jj < C::B1; ++jj) {
                            const double w01 = w0[i] * w1[jj];
#pragma unroll
                            for (int k = 0; k < C::B2; ++k) acc[i][jj][k] = fma(w01, w2[k], acc[i][jj][k]);
                        }
                };
                double a0[C::B0], a1[C::B1], a2[C::B2], b0[C::B0], b1[C::B1], b2[C::B2];
                ldw(0, a0, a1, a2);
                for (int j = 0; j < np; j += 2) {
                    ldw(j + 1, b0, b1, b2);
                    acc_pt(a0, a1, a2);
                    ldw(min(j + 2, 31), a0, a1, a2);
                    acc_pt(b0, b1, b2);
                }
            }
            // rotate
            p0 = p1;
            p1 = p2;
            p2 = p3;
            p3 = p4;
            d0 = d1;
            d1 = d2;
            d2 = d3;
            d3 = d4;
            n2 = n3;
#pragma unroll
            for (int ax = 0; ax < D; ++ax) {
                f0[ax] = f1[ax];
                f1[ax] = f2[ax];
            }
            s0 = s1;
            s1 = s2;
            v0 = v1;
            v1 = v2;
        }
        flush(cur);
        __syncwarp();
        if (!PERSIST && seg_cur < seg_end && !(flags & (1u << 19))) {
            double* out = a.partial + (size_t)seg_cur * tile;
            for (int i = lane; i < tile; i += 32) {
                out[i] = (pass ? out[i] : 0.0) + my_tile[i];
                my_tile[i] = 0.0;
            }
            __syncwarp();
        }
    }
    pdl_launch();
    if (PERSIST) {
        __syncthreads();
        double* out = a.partial + (size_t)bid * tile;
        for (int i = threadIdx.x; i < tile; i += blockDim.x) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += smem[(size_t)w * tile + i];
            out[i] = t;
        }
    }
}

template <int D, int M, bool PERSIST, bool GROUPED = false>
__global__ void __launch_bounds__(PERSIST ? (GROUPED ? 32 * kBandWarps : 256) : 64, GROUPED ? kBandCtasPerSm : 1)
spread_kernel(FsArgs a, WinCoef wc, const double* __restrict__ v, unsigned flags, int* __restrict__ work) {
    (void)work;
    spread_body<D, M, PERSIST, GROUPED>(a, wc, v, flags, blockIdx.x, gridDim.x);
}

// ------------------------------------------------- d = 1: streaming kernels --
// d = 1 layers put 10^3..10^5 points in a cell, so per-32-point descriptors
// are pure overhead and the window polynomials are the work.  Each warp
// streams a contiguous range of the sorted points, K1 points per lane per
// step (lane l takes base + l + 32u): coalesced loads one step ahead (point
// indices two ahead), the lane's K1 windows formed together (one
// coefficient read feeds K1 FMAs) and consumed as they are formed.  A
// point's cell comes from the per-cell start table (cells are sorted).
constexpr int K1 = 4;
constexpr int K1STEP = 32 * K1;

__device__ __forceinline__ void warp_range(int64_t n, int64_t& lo, int64_t& hi) {
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const int64_t W = (int64_t)gridDim.x * nw, gw = (int64_t)blockIdx.x * nw + warp;
    const int64_t per = ((n + W - 1) / W + K1STEP - 1) / K1STEP * K1STEP;
    lo = gw * per;
    hi = lo + per < n ? lo + per : n;
}

// last key whose start is <= p
__device__ __forceinline__ int key_of(const FsArgs& a, int64_t p) {
    int kl = 0, kh = a.nkeys;
    while (kh - kl > 1) {
        const int mid = (kl + kh) >> 1;
        if (__ldg(a.key_start + mid) <= p) kl = mid;
        else kh = mid;
    }
    return kl;
}

// Spread: the lane's K1 points accumulate into registers for the warp's
// current cell; a step whose 32 K1 points all lie in it (almost every step)
// takes the fast path, otherwise the step is replayed slot by slot with a
// flush (fixed xor-shuffle tree, lane 0 adds to the warp's tile) at every
// cell boundary.  The CTA sums its warp tiles (grid_sum_kernel then sums the
// CTAs): deterministic.
template <int M>
__global__ void __launch_bounds__(256, 2) spread1_kernel(FsArgs a, WinCoef wc, const double* __restrict__ v,
                                                         unsigned flags) {
    constexpr int S = 2 * M + 1;
    extern __shared__ double smem[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = a.tile_cells;
    double* my_tile = smem + (size_t)warp * tile;
    for (int i = lane; i < tile; i += 32) my_tile[i] = 0.0;
    const bool sorted = (flags & MLB_SORTED) != 0, use_isd = (flags & MLB_USE_ISD) != 0;
    int64_t lo, hi;
    warp_range(a.n, lo, hi);
    pdl_wait();  // v (and D^-1/2) may come from the stream predecessor
    if (lo < hi) {
        int cur = key_of(a, lo);
        int64_t cstart = __ldg(a.key_start + cur), nxt = __ldg(a.key_start + cur + 1);
        // the current cell's even / odd pair sums and the o = -m sum (kb_accumulate_k)
        double ae[M], ao[M], a0 = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) ae[q] = ao[q] = 0.0;
        auto flush = [&]() {
            double acc[S];
            acc[0] = a0;
#pragma unroll
            for (int q = 1; q <= M; ++q) {
                acc[q + M] = ae[q - 1] + ao[q - 1];
                acc[1 - q + M] = ae[q - 1] - ao[q - 1];
            }
#pragma unroll
            for (int o = 0; o < S; ++o) {
                double t = acc[o];
#pragma unroll
                for (int sh = 16; sh > 0; sh >>= 1) t += __shfl_xor_sync(0xffffffffu, t, sh);
                if (lane == 0) my_tile[cur + o] += t;
            }
#pragma unroll
            for (int q = 0; q < M; ++q) ae[q] = ao[q] = 0.0;
            a0 = 0.0;
        };
        auto ld_node = [&](int64_t base, int (&nd)[K1]) {
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                const int64_t p = base + 32 * u + lane;
                nd[u] = (p < hi) ? (sorted ? (int)p : __ldg(a.perm + p)) : 0;
            }
        };
        // raw loads only: the product s v is formed when the step consumes them,
        // so the loads stay in flight across the previous step's arithmetic
        auto ld_data = [&](int64_t base, const int (&nd)[K1], double (&f)[K1], double (&sc)[K1], double (&vv)[K1]) {
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                const int64_t p = base + 32 * u + lane;
                const bool ok = p < hi;
                f[u] = ok ? __ldg(a.frac + p) : 0.5;
                sc[u] = (ok && use_isd) ? __ldg(a.isd + p) : 1.0;
                vv[u] = ok ? __ldg(v + nd[u]) : 0.0;
            }
        };
        int nd[K1];
        double f[K1], sc[K1], vv[K1];
        ld_node(lo, nd);
        ld_data(lo, nd, f, sc, vv);
        ld_node(lo + K1STEP, nd);
        for (int64_t base = lo; base < hi; base += K1STEP) {
            double fc[K1], svc[K1];
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                fc[u] = f[u];
                svc[u] = sc[u] * vv[u];
            }
            if (base + K1STEP < hi) ld_data(base + K1STEP, nd, f, sc, vv);   // next step's data
            if (base + 2 * K1STEP < hi) ld_node(base + 2 * K1STEP, nd);   // and the indices after it
            const int64_t last = (base + K1STEP < hi ? base + K1STEP : hi) - 1;
            if (last < nxt) {
                kb_accumulate_k<M, K1>(fc, svc, wc, ae, ao, a0);
                continue;
            }
#pragma unroll 1
            for (int u = 0; u < K1; ++u) {   // a cell boundary inside this step
                const int64_t g0 = base + 32 * u;
                if (g0 >= hi) break;
                const int64_t g1 = (g0 + 32 < hi ? g0 + 32 : hi) - 1;
                const int64_t p = g0 + lane;
                double fsel = fc[0], ssel = svc[0];   // slot u's values (constant indices: no stack)
#pragma unroll
                for (int k = 1; k < K1; ++k)
                    if (u == k) {
                        fsel = fc[k];
                        ssel = svc[k];
                    }
                const double fu[1] = {fsel};
                while (true) {
                    const double su[1] = {(p <= g1 && p >= cstart && p < nxt) ? ssel : 0.0};
                    kb_accumulate_k<M, 1>(fu, su, wc, ae, ao, a0);
                    if (g1 < nxt) break;
                    flush();
                    cstart = nxt;   // the next non-empty cell starts here
                    do {
                        ++cur;
                        nxt = __ldg(a.key_start + cur + 1);
                    } while (nxt <= cstart);
                }
            }
        }
        flush();
    }
    pdl_launch();
    __syncthreads();
    double* out = a.partial + (size_t)blockIdx.x * tile;
    for (int i = threadIdx.x; i < tile; i += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += smem[(size_t)w * tile + i];
        out[i] = t;
    }
}

// Gather: the whole (tiny) d = 1 grid sits in shared memory; every lane
// tracks its own points' cells (its points only move forward); epilogue
// y = alpha v + s (beta acc + gamma s v).
template <int M>
__global__ void __launch_bounds__(256, 2) gather1_kernel(FsArgs a, WinCoef wc, const double* __restrict__ grid,
                                                         const double* __restrict__ v, double* __restrict__ y,
                                                         double alpha, double beta, double gamma, unsigned flags) {
    constexpr int TS = 2 * M + 1;
    extern __shared__ double gs[];   // the grid (L), then per cell c: g[c], (GS, GD) per q (kb_dot_k)
    double* tab = gs + a.g.L;
    const int lane = threadIdx.x & 31;
    const bool sorted = (flags & MLB_SORTED) != 0, use_isd = (flags & MLB_USE_ISD) != 0;
    pdl_wait();  // the grid (convolution) and v come from stream predecessors
    for (int i = threadIdx.x; i < a.g.L; i += blockDim.x) gs[i] = __ldcg(grid + i);
    __syncthreads();
    for (int c = threadIdx.x; c < a.nkeys; c += blockDim.x) {
        tab[c * TS] = gs[c];
#pragma unroll
        for (int q = 1; q <= M; ++q) {
            const double hi_ = gs[c + q + M], lo_ = gs[c + 1 - q + M];
            tab[c * TS + 2 * q - 1] = hi_ + lo_;
            tab[c * TS + 2 * q] = hi_ - lo_;
        }
    }
    __syncthreads();
    int64_t lo, hi;
    warp_range(a.n, lo, hi);
    if (lo < hi) {
        int lc = key_of(a, lo + lane < hi ? lo + lane : hi - 1);
        int64_t lnxt = __ldg(a.key_start + lc + 1);
        auto ld_node = [&](int64_t base, int (&nd)[K1]) {
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                const int64_t p = base + 32 * u + lane;
                nd[u] = (p < hi) ? (sorted ? (int)p : __ldg(a.perm + p)) : 0;
            }
        };
        auto ld_data = [&](int64_t base, const int (&nd)[K1], double (&f)[K1], double (&sc)[K1], double (&vv)[K1]) {
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                const int64_t p = base + 32 * u + lane;
                const bool ok = p < hi;
                f[u] = ok ? __ldg(a.frac + p) : 0.5;
                sc[u] = (ok && use_isd) ? __ldg(a.isd + p) : 1.0;
                vv[u] = (ok && v) ? __ldg(v + nd[u]) : 0.0;
            }
        };
        int nd[K1], ndn[K1];
        double f[K1], sc[K1], vv[K1];
        ld_node(lo, nd);
        ld_data(lo, nd, f, sc, vv);
        ld_node(lo + K1STEP, ndn);
        for (int64_t base = lo; base < hi; base += K1STEP) {
            double fc[K1], scc[K1], vc[K1];
            int ndc[K1], cell[K1];
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                fc[u] = f[u];
                scc[u] = sc[u];
                vc[u] = vv[u];
                ndc[u] = nd[u];
                nd[u] = ndn[u];
                const int64_t p = base + 32 * u + lane;
                while (p < hi && p >= lnxt) {   // this lane's cell (points only move forward)
                    ++lc;
                    lnxt = __ldg(a.key_start + lc + 1);
                }
                cell[u] = lc;
            }
            if (base + K1STEP < hi) ld_data(base + K1STEP, nd, f, sc, vv);
            if (base + 2 * K1STEP < hi) ld_node(base + 2 * K1STEP, ndn);
            double acc[K1];
#pragma unroll
            for (int u = 0; u < K1; ++u) acc[u] = 0.0;
            kb_dot_k<M, K1>(fc, wc, tab, cell, acc);
#pragma unroll
            for (int u = 0; u < K1; ++u) {
                const int64_t p = base + 32 * u + lane;
                if (p >= hi) continue;
                const int node = ndc[u];
                double res = alpha * vc[u] + scc[u] * (beta * acc[u] + gamma * scc[u] * vc[u]);
                if (flags & MLB_ACCUMULATE) res += y[node];
                y[node] = res;
            }
        }
    }
    pdl_launch();
}

// ------------------------------------------------------ spread d=3: cells --
// The d = 3 spread works per CELL: all points of a cell (or of a part of at
// most cell_cap points of a heavy cell) share one (2m+1)^3 stencil position,
// so their contributions sum in registers into one block -- no per-warp
// brick tile in shared memory (which capped residency at ~10 warps/SM), no
// flushes.  A CTA of 8 warps walks a static list of items (bind time: blocks
// packed onto warps, largest first); within an item every warp walks its own
// precomputed stream of 32-point sub-chunks (one cell each): it evaluates
// the 32 points' windows (v s folded into axis 0) into its staging rows,
// then accumulates them with the SpreadCfg lane blocks (lane (i, j-block)
// owns one axis-0 offset, B1 axis-1 offsets and an axis-2 row).  At the end
// of an item the warps' sums meet in shared memory and each block is the
// fixed-order sum over its warps -> bitwise reproducible.  Global loads run
// two sub-chunks ahead (stream entries, point indices) and one ahead
// (coordinates, D^-1/2, v) across item boundaries.
template <int M>
__global__ void __launch_bounds__(256, (M >= 5) ? 1 : 2) spread_cells_kernel(FsArgs a, WinCoef wc, const double* __restrict__ v,
                                                              unsigned flags) {
    using C = SpreadCfg<3, M>;
    constexpr int S = C::S;
    constexpr int SPAD = StageCfg<3, M>::pad;
    constexpr int NRED = S * S * C::SP;       // one pass slice of a block
    // staging doubles per warp: >= one block slice, even (16-byte aligned rows)
    constexpr int STG = (((32 * 3 * SPAD > NRED) ? 32 * 3 * SPAD : NRED) + 1) & ~1;
    extern __shared__ __align__(16) double smem[];
    double* red = smem + kCellWarps * STG;     // kCellWarps x NRED
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* stage = smem + warp * STG;
    const int l0 = lane / C::P1, l1 = lane % C::P1;
    // m = 5: lanes own PPL consecutive (o0, o1) pairs (one pass, 31 of 32
    // lanes busy) instead of the (o0, o1-block) split (22 lanes)
    constexpr bool PAIRS = (M == 5);
    constexpr int PPL = (S * S + 31) / 32;
    const bool active = PAIRS ? (lane * PPL < S * S) : (lane < C::P0 * C::P1);
    const bool sorted = (flags & MLB_SORTED) != 0;
    const bool use_isd = (flags & MLB_USE_ISD) != 0;
    for (int i = lane; i < STG; i += 32) stage[i] = 0.0;
    const int e0 = __ldg(a.wstream_off + blockIdx.x * kCellWarps + warp);
    const int e1 = __ldg(a.wstream_off + blockIdx.x * kCellWarps + warp + 1);
    const int it0 = __ldg(a.citem_off + blockIdx.x);

    for (int pass = 0; pass < C::NPASS; ++pass) {
        const int off2 = pass * C::SP;
        double acc[C::B1][C::SP];
#pragma unroll
        for (int j = 0; j < C::B1; ++j)
#pragma unroll
            for (int k = 0; k < C::SP; ++k) acc[j][k] = 0.0;
        // pipeline: q0 compute, q1 data in flight, q2 point index in flight
        auto ent = [&](int e) { return (e < e1) ? __ldg(a.wstream + e) : make_int2(0, 0); };
        auto cnt_of = [](int2 q) { return (q.y >> 24) & 63; };
        auto pidx = [&](int2 q) { return q.x + min(lane, max(cnt_of(q) - 1, 0)); };
        auto node_of = [&](int2 q) -> int {
            const int p = pidx(q);
            return (sorted || cnt_of(q) == 0) ? p : __ldg(a.perm + p);
        };
        int e = e0;
        int2 q0 = ent(e), q1 = ent(e + 1), q2 = ent(e + 2);
        double f0[3], f1[3], s0 = 1.0, s1 = 1.0, v0 = 0.0, v1 = 0.0;
        auto load_data = [&](int2 q, int node, double* f, double& sv, double& vv) {
            const int p = pidx(q);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) f[ax] = __ldg(a.frac + (int64_t)ax * a.n + p);
            sv = use_isd ? __ldg(a.isd + p) : 1.0;
            vv = __ldg(v + node);
        };
        pdl_wait();  // v (and D^-1/2) may come from the stream predecessor
        load_data(q0, node_of(q0), f0, s0, v0);
        load_data(q1, node_of(q1), f1, s1, v1);
        int n2 = node_of(q2);
        int item = it0;
        for (; e < e1; ++e) {
            const int np = cnt_of(q0);
            if (np > 0 && !(flags & (1u << 17))) {  // bit 17: ablation (profiling only)
                const double sv = (lane < np) ? s0 * v0 : 0.0;
                double w[S];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {   // (the joint 3-axis form spills at m = 4, gains nothing at m = 5)
                    kb_windows<M>(f0[ax], wc, w);
                    double* dst = stage + (lane * 3 + ax) * SPAD;
#pragma unroll
                    for (int o = 0; o < S; ++o) dst[o] = (ax == 0) ? w[o] * sv : w[o];
                }
            }
            // advance the loads (they overlap the accumulation below)
            const int2 q3 = ent(e + 3);
            const int n3 = node_of(q3);
            double f2[3], s2, v2;
            load_data(q2, n2, f2, s2, v2);
            __syncwarp();
            if (np > 0 && active && !(flags & (1u << 16))) {  // bit 16: ablation (profiling only)
                auto ldw = [&](int j, double& w0, double* w1, double* w2) {
                    const double* ws = stage + j * 3 * SPAD;
                    w0 = ws[l0];
#pragma unroll
                    for (int jj = 0; jj < C::B1; ++jj) w1[jj] = ws[SPAD + l1 * C::B1 + jj];
                    if constexpr (StageCfg<3, M>::vec2) {
                        const double* w2p = ws + 2 * SPAD + off2;
#pragma unroll
                        for (int k = 0; k + 1 < C::SP; k += 2) {
                            const double2 t = *reinterpret_cast<const double2*>(w2p + k);
                            w2[k] = t.x;
                            w2[k + 1] = t.y;
                        }
                        if (C::SP & 1) w2[C::SP - 1] = w2p[C::SP - 1];
                    } else {
#pragma unroll
                        for (int k = 0; k < C::SP; ++k) w2[k] = ws[2 * SPAD + off2 + k];
                    }
                };
                auto acc_pt = [&](double w0, const double* w1, const double* w2) {
#pragma unroll
                    for (int jj = 0; jj < C::B1; ++jj) {
                        const double w01 = w0 * w1[jj];
#pragma unroll
                        for (int k = 0; k < C::SP; ++k) acc[jj][k] = fma(w01, w2[k], acc[jj][k]);
                    }
                };
                if constexpr (PAIRS) {
                    static_assert(C::NPASS == 1 && C::B1 >= PPL, "pair path: one pass, acc rows >= pairs");
                    for (int j = 0; j < np; ++j) {  // rows past np carry v = 0
                        const double* ws = stage + j * 3 * SPAD;
                        double w2[S];
#pragma unroll
                        for (int k = 0; k + 1 < S; k += 2) {
                            const double2 t = *reinterpret_cast<const double2*>(ws + 2 * SPAD + k);
                            w2[k] = t.x;
                            w2[k + 1] = t.y;
                        }
                        w2[S - 1] = ws[2 * SPAD + S - 1];
#pragma unroll
                        for (int i = 0; i < PPL; ++i) {
                            const int q = min(lane * PPL + i, S * S - 1);
                            const double w01 = ws[q / S] * ws[SPAD + q % S];
#pragma unroll
                            for (int k = 0; k < S; ++k) acc[i][k] = fma(w01, w2[k], acc[i][k]);
                        }
                    }
                } else {
                    double a0, a1[C::B1], a2[C::SP], b0, b1[C::B1], b2[C::SP];
                    ldw(0, a0, a1, a2);
                    for (int j = 0; j < np; j += 2) {  // rows past np carry v = 0
                        ldw(j + 1, b0, b1, b2);
                        acc_pt(a0, a1, a2);
                        ldw(min(j + 2, 31), a0, a1, a2);
                        acc_pt(b0, b1, b2);
                    }
                }
            }
            __syncwarp();
            if (q0.y & 1) {  // end of item: every warp of the CTA is here
                // the item row (L1-cached, read by every warp): this warp's block
                const int* ir = a.citem + (size_t)item * kItemInts;
                const int nb = __ldg(ir);
                int blk = -1, nwb = 0;
                bool multi = false;
                for (int eb = 0; eb < nb; ++eb) {
                    const int wlo = __ldg(ir + 2 + 3 * eb), nw = __ldg(ir + 3 + 3 * eb);
                    multi |= nw > 1;
                    if (warp >= wlo && warp < wlo + nw) {
                        blk = __ldg(ir + 1 + 3 * eb);
                        nwb = nw;
                    }
                }
                if (blk >= 0 && nwb == 1) {  // a one-warp block: transposed through the warp's staging, coalesced out
                    static_assert(NRED <= STG, "block slice must fit the warp's staging");
                    __syncwarp();
                    if (active) {
                        if constexpr (PAIRS) {
#pragma unroll
                            for (int i = 0; i < PPL; ++i)
                                if (lane * PPL + i < S * S)
#pragma unroll
                                    for (int k = 0; k < S; ++k) stage[(lane * PPL + i) * S + k] = acc[i][k];
                        } else {
                            double* r = stage + l0 * S * C::SP;
#pragma unroll
                            for (int jj = 0; jj < C::B1; ++jj)
#pragma unroll
                                for (int k = 0; k < C::SP; ++k)
                                    if (l1 * C::B1 + jj < S) r[(l1 * C::B1 + jj) * C::SP + k] = acc[jj][k];
                        }
                    }
                    __syncwarp();
                    double* out = a.blocks + (size_t)blk * (S * S * S);
                    for (int t = lane; t < NRED; t += 32) {
                        const int o01 = t / C::SP, k = t % C::SP;
                        if (off2 + k < S) {
                            if (a.agrid) atomicAdd(a.agrid + block_grid_index(a, blk, o01, off2 + k), stage[t]);
                            else out[o01 * S + off2 + k] = stage[t];
                        }
                    }
                    __syncwarp();
                }
                if (multi) {  // uniform over the CTA: multi-warp blocks meet in shared memory
                    __syncthreads();  // previous item's reduction reads of `red` are done
                    if (active && nwb > 1) {
                        if constexpr (PAIRS) {
#pragma unroll
                            for (int i = 0; i < PPL; ++i)
                                if (lane * PPL + i < S * S)
#pragma unroll
                                    for (int k = 0; k < S; ++k) red[warp * NRED + (lane * PPL + i) * S + k] = acc[i][k];
                        } else {
                            double* r = red + warp * NRED + l0 * S * C::SP;
#pragma unroll
                            for (int jj = 0; jj < C::B1; ++jj)
#pragma unroll
                                for (int k = 0; k < C::SP; ++k)
                                    if (l1 * C::B1 + jj < S) r[(l1 * C::B1 + jj) * C::SP + k] = acc[jj][k];
                        }
                    }
                    __syncthreads();
                    for (int eb = 0; eb < nb; ++eb) {
                        const int bk = __ldg(ir + 1 + 3 * eb), wlo = __ldg(ir + 2 + 3 * eb), nw = __ldg(ir + 3 + 3 * eb);
                        if (nw == 1) continue;
                        double* out = a.blocks + (size_t)bk * (S * S * S);
                        for (int t = threadIdx.x; t < NRED; t += blockDim.x) {
                            double sum = 0.0;
                            for (int r = 0; r < nw; ++r) sum += red[(wlo + r) * NRED + t];
                            const int o01 = t / C::SP, k = t % C::SP;
                            if (off2 + k < S) {
                                if (a.agrid) atomicAdd(a.agrid + block_grid_index(a, bk, o01, off2 + k), sum);
                                else out[o01 * S + off2 + k] = sum;
                            }
                        }
                    }
                }
#pragma unroll
                for (int jj = 0; jj < C::B1; ++jj)
#pragma unroll
                    for (int k = 0; k < C::SP; ++k) acc[jj][k] = 0.0;
                ++item;
            }
            q0 = q1;
            q1 = q2;
            q2 = q3;
            n2 = n3;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                f0[ax] = f1[ax];
                f1[ax] = f2[ax];
            }
            s0 = s1;
            s1 = s2;
            v0 = v1;
            v1 = v2;
        }
        __syncthreads();  // `red` reads of the last item done before the next pass
    }
    pdl_launch();
}

// d = 3 stage R1: brick tile = fixed-order sum of the brick's cell blocks,
// each placed at its cell.  CTA = (tile slab s0 along axis 0, active brick).
template <int M>
struct MergeCfg {
    static constexpr int TL = 4 + 2 * M;  // largest tile: d = 3 bricks are <= 4^3 cells
    static constexpr int MT = (TL * TL + 31) / 32 * 32;
};

template <int M>
__global__ void __launch_bounds__(MergeCfg<M>::MT, 2048 / MergeCfg<M>::MT) brick_merge_kernel(FsArgs a) {
    constexpr int S = 2 * M + 1;
    constexpr int SS = S * S;
    const int TL = a.g.TL;
    const int s0 = blockIdx.x, slot = blockIdx.y;
    const int q0 = __ldg(a.merge_off + slot * TL + s0), q1 = __ldg(a.merge_off + slot * TL + s0 + 1);
    double* out = a.partial + (size_t)slot * a.tile_cells + (size_t)s0 * TL * TL;
    // The block rows landing in this slab were listed at bind time (block
    // order) and are staged in shared memory with one cooperative load; the
    // thread of slab position t then sums them in list order, 8 independent
    // (branch-free) loads in flight.  One small CTA per (brick, slab): the
    // whole grid is resident at once, so the latency chain is paid once.
    __shared__ int2 pr[256];
    const int t = threadIdx.x;
    const bool live = t < TL * TL;
    const int i1 = live ? t / TL : 0, i2 = live ? t % TL : 0;
    double sum = 0.0;
    for (int base = q0; base < q1; base += 256) {
        const int nq = min(256, q1 - base);
        __syncthreads();
        for (int i = t; i < nq; i += blockDim.x) pr[i] = __ldg(reinterpret_cast<const int2*>(a.merge_pairs) + base + i);
        __syncthreads();
        pdl_wait();  // the cell blocks come from the spread
        for (int q = 0; q < nq; q += 8) {
            double vals[8];
            bool ok[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int2 p = pr[min(q + u, nq - 1)];
                const int o1 = i1 - (p.y >> 8), o2 = i2 - (p.y & 255);
                ok[u] = (q + u < nq) && (unsigned)o1 < (unsigned)S && (unsigned)o2 < (unsigned)S;
                vals[u] = __ldcg(a.blocks + (size_t)p.x * SS + (ok[u] ? o1 * S + o2 : 0));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += ok[u] ? vals[u] : 0.0;
        }
    }
    pdl_wait();  // (a slab without rows still orders its write after the predecessor)
    pdl_launch();
    if (live) out[t] = sum;
}

// ------------------------------------------------------------------ reduce --
// d <= 2: grid[u] = sum over the spread CTAs' partial grids.  Block = 8
// cells x 32 slices; slice k sums partials k, k+32, ...; the 32 slice sums
// combine through a fixed shuffle tree -> deterministic.
__device__ __forceinline__ void grid_sum_body(const double* __restrict__ partial, int nparts, int cells,
                                              const PeerOut& grid, int bid) {
    const int slice = threadIdx.x & 31;
    const int cell = bid * 8 + (threadIdx.x >> 5);
    double s = 0.0;
    pdl_wait();  // the partial grids come from the spread
    if (cell < cells) {
        int j = slice;
        for (; j + 96 < nparts; j += 128) {
            const double a0 = __ldcg(partial + (size_t)j * cells + cell);
            const double a1 = __ldcg(partial + (size_t)(j + 32) * cells + cell);
            const double a2 = __ldcg(partial + (size_t)(j + 64) * cells + cell);
            const double a3 = __ldcg(partial + (size_t)(j + 96) * cells + cell);
            s += a0;
            s += a1;
            s += a2;
            s += a3;
        }
        for (; j < nparts; j += 32) s += __ldcg(partial + (size_t)j * cells + cell);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    pdl_launch();
    if (slice == 0 && cell < cells) po_store(grid, cell, s);
    if (grid.n > 1) __threadfence_system();  // peer stores ordered before the exchange barrier
}

__global__ void grid_sum_kernel(const double* __restrict__ partial, int nparts, int cells, PeerOut grid) {
    grid_sum_body(partial, nparts, cells, grid, blockIdx.x);
}

// d = 2 banded spread: grid[u0, u1] = sum over the CTAs whose band covers
// row u0 (a contiguous CTA range, row_cta) of their band tiles.  Same
// 8 cells x 32 slices layout and fixed shuffle tree as grid_sum_kernel.
__global__ void band_sum_kernel(const double* __restrict__ partial, int band_tile, int TL,
                                const int32_t* __restrict__ cta_row0, const int2* __restrict__ row_cta, int cells,
                                PeerOut grid) {
    const int slice = threadIdx.x & 31;
    const int cell = blockIdx.x * 8 + (threadIdx.x >> 5);
    double s = 0.0;
    pdl_wait();  // the band tiles come from the spread
    if (cell < cells) {
        const int u0 = cell / TL, u1 = cell - u0 * TL;
        const int2 rc = __ldg(row_cta + u0);
        for (int c = rc.x + slice; c <= rc.y; c += 32)
            s += __ldcg(partial + (size_t)c * band_tile + (size_t)(u0 - __ldg(cta_row0 + c)) * TL + u1);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    pdl_launch();
    if (slice == 0 && cell < cells) po_store(grid, cell, s);
    if (grid.n > 1) __threadfence_system();  // peer stores ordered before the exchange barrier
}

// Stage R2: grid[u] = sum over the (<= 3^d) bricks whose tile covers u of
// that brick's (first-segment) tile value.  One thread per active cell.
template <int D, int TBC>
__global__ void reduce_kernel(FsArgs a, PeerOut grid) {
    const Geom g = a.g;
    const int L = g.L, nbr = g.nbr;
    const int Tb = TBC ? TBC : g.Tb;
    const int TL = TBC ? TBC + 2 * g.m : g.TL;
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
#pragma unroll
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
                    const int s0 = __ldg(a.brick_first + brick);
                    if (s0 >= 0) s += a.partial[(size_t)s0 * a.tile_cells + t];
                }
        po_store(grid, cidx, s);
    }
    if (grid.n > 1) __threadfence_system();
}

// Stage R2 for d = 3, block-centric: a CTA covers GB grid blocks of Tb^3
// cells; the <= R^3 source brick tiles of each grid block are resolved once
// into smem base pointers, then every cell issues its independent loads.
template <int TB, int M>
__global__ void __launch_bounds__(256) reduce3_kernel(FsArgs a, PeerOut grid) {
    constexpr int CPB = TB * TB * TB;  // cells per grid block
    constexpr int GB = 256 / CPB;      // grid blocks per CTA
    constexpr int TL = TB + 2 * M;
    constexpr int R = (TL + TB - 1) / TB;  // source bricks per axis
    constexpr int RRR = R * R * R;
    const Geom g = a.g;
    const int L = g.L, nbr = g.nbr;
    const int ngb = (L + TB - 1) / TB;  // grid blocks per axis
    __shared__ const double* base[GB][64];
    const int lb = threadIdx.x / CPB, c = threadIdx.x % CPB;
    const int gbid = blockIdx.x * GB + lb;
    const int gb0 = gbid / (ngb * ngb), gb1 = (gbid / ngb) % ngb, gb2 = gbid % ngb;
    const bool live = gbid < ngb * ngb * ngb;
    for (int q = c; q < RRR; q += CPB) {
        const int s0 = q / (R * R), s1 = (q / R) % R, s2 = q % R;
        const int b0 = gb0 - s0, b1 = gb1 - s1, b2 = gb2 - s2;
        const double* p = nullptr;
        if (live && b0 >= 0 && b1 >= 0 && b2 >= 0 && b0 < nbr && b1 < nbr && b2 < nbr) {
            const int f = __ldg(a.brick_first + (b0 * nbr + b1) * nbr + b2);
            if (f >= 0) p = a.partial + (size_t)f * a.tile_cells + ((s0 * TB) * TL + s1 * TB) * TL + s2 * TB;
        }
        base[lb][q] = p;
    }
    __syncthreads();
    pdl_wait();  // the brick tiles come from the merge
    if (!live) return;
    const int c0 = c / (TB * TB), c1 = (c / TB) % TB, c2 = c % TB;
    const int u0 = gb0 * TB + c0, u1 = gb1 * TB + c1, u2 = gb2 * TB + c2;
    if (u0 >= L || u1 >= L || u2 >= L) return;
    const int local = (c0 * TL + c1) * TL + c2;
    constexpr bool exact = (R * TB == TL);
    double sum = 0.0;
#pragma unroll
    for (int q = 0; q < RRR; ++q) {
        const double* p = base[lb][q];
        bool ok = p != nullptr;
        if (!exact) {
            const int s0 = q / (R * R), s1 = (q / R) % R, s2 = q % R;
            ok = ok && (s0 * TB + c0 < TL) && (s1 * TB + c1 < TL) && (s2 * TB + c2 < TL);
        }
        sum += ok ? __ldcg(p + local) : 0.0;
    }
    pdl_launch();
    po_store(grid, ((int64_t)u0 * L + u1) * L + u2, sum);
    if (grid.n > 1) __threadfence_system();
}

// ------------------------------------------------------------------ gather --
// Every warp owns a contiguous range of chunks; it stages the (2m+1)^d grid
// neighbourhood of the current chunk's cell in shared memory (reloaded only
// when the cell changes -- consecutive chunks usually share it) and each
// lane owns TWO points of the chunk (p0+lane, p0+32+lane), so every staged
// value read (a broadcast LDS: the whole chunk shares one cell) feeds two
// FMAs.  Epilogue: y = alpha v + s (beta acc + gamma s v).
template <int D, int M, bool PK>
struct GatherCfg {
    static constexpr int S = 2 * M + 1;
    // d = 3 packed (PK) stages a pencil: the neighbourhoods of <= Tb
    // consecutive axis-2 cells (Tb = 4, or 2 for m >= 6) share one
    // (2m+1)^2 x (2m+Tb) block
    static constexpr int SR = (D == 3 && PK) ? S + (M >= 6 ? 1 : 3) : S;
    static constexpr int NB = (D == 1) ? S : (D == 2 ? S * S : S * S * SR);
};

// body of gather_kernel; `bid` / `nblk` stand for blockIdx.x / gridDim.x
template <int D, int M, bool PK>
__device__ __forceinline__ void gather_body(const FsArgs& a, const WinCoef& wc, const double* __restrict__ grid,
                                            const double* __restrict__ v, double* __restrict__ y, double alpha,
                                            double beta, double gamma, unsigned flags, int bid, int nblk) {
    constexpr int S = 2 * M + 1;
    constexpr int SR = GatherCfg<D, M, PK>::SR;  // staged row length (d = 3 packed: a pencil of <= Tb cells)
    constexpr int NB = GatherCfg<D, M, PK>::NB;
    constexpr int W0S = 2 * S + 1;  // per-lane axis-0 window row (odd stride)
    extern __shared__ double nbs[];
    const int L = a.g.L;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    double* nb = nbs + wl * NB;
    double* w0s = nbs + 8 * NB + (wl * 32 + lane) * W0S;  // [0,S): point A, [S,2S): point B
    const int gw = (bid * (int)blockDim.x + (int)threadIdx.x) >> 5;
    const int nwt = (nblk * (int)blockDim.x) >> 5;
    const int nunits = (D == 3 && PK) ? a.ngrp : a.nchunks;  // pencil groups, or one-cell chunks
    const int c_lo = (int)(((long long)nunits * gw) / nwt);
    const int c_hi = (int)(((long long)nunits * (gw + 1)) / nwt);
    const int64_t rs = (D == 3) ? (int64_t)L * L : (int64_t)L;  // stride of axis 0
    long long cur = -1;
    // m >= 5 d = 3 chunks (one CTA per SM, registers to spare): the epilogue's
    // gathers are issued at the chunk's start (EPF) and the NEXT chunk's
    // offsets are loaded while this chunk contracts (PF)
    // (d = 2: the axis-0 windows go to shared memory like d = 3's, which
    // leaves the registers for both prefetches at 128 registers per thread)
    constexpr bool EPF = (D == 3 && M >= 5) || D <= 2;
    constexpr bool PF = ((D == 3 && M >= 5) || D <= 2) && !PK;
    double nf[6] = {0.5, 0.5, 0.5, 0.5, 0.5, 0.5};
    auto load_frac = [&](int c) {
        const int q0 = a.chunk_start[c];
        const int qn = a.chunk_start[c + 1] - q0;
        const bool oA = lane < qn, oB = lane + 32 < qn;
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
            nf[2 * ax] = oA ? __ldg(a.frac + ax * a.n + q0 + lane) : 0.5;
            nf[2 * ax + 1] = oB ? __ldg(a.frac + ax * a.n + q0 + 32 + lane) : 0.5;
        }
    };
    pdl_wait();  // the grid (convolution) and v come from stream predecessors
    if (PF && c_lo < c_hi) load_frac(c_lo);
    for (int ch = c_lo; ch < c_hi; ++ch) {
        int gbase, wst = S, dcA = 0, pA, pB;
        bool okA, okB, two;
        if (D == 3 && PK) {
            const int2 gg = __ldg(a.ggrp + ch);
            const int sA = __ldg(a.gslot + (int64_t)ch * 64 + lane);
            const int sB = __ldg(a.gslot + (int64_t)ch * 64 + 32 + lane);
            gbase = gg.x;
            wst = S - 1 + (gg.y & 255);  // staged cells along axis 2
            two = (gg.y >> 8) != 0;      // warp-uniform: one-point groups skip the second point
            okA = sA >= 0;
            okB = sB >= 0;
            pA = okA ? (sA & 0x1fffffff) : 0;
            pB = okB ? (sB & 0x1fffffff) : 0;
            dcA = okA ? (sA >> 29) : 0;  // a lane's two points share one cell
        } else {
            const int p0 = a.chunk_start[ch];
            const int np = a.chunk_start[ch + 1] - p0;
            gbase = a.chunk_gcell[ch];
            okA = lane < np;
            okB = lane + 32 < np;
            two = np > 32;  // warp-uniform: chunks of <= 32 points skip the second point
            pA = p0 + lane;
            pB = p0 + 32 + lane;
        }
        const long long key = (long long)gbase * 16 + wst;
        // d = 3: the epilogue's gathers (node index, D^-1/2, then v[node]) are
        // issued now and consumed after the contraction -- a random v[perm[p]]
        // read costs a full DRAM round trip that 2 warps per SMSP cannot hide
        int nodeA = 0, nodeB = 0;
        double sA = 1.0, sB = 1.0;
        if (EPF) {
            nodeA = (flags & MLB_SORTED) ? pA : (okA ? __ldg(a.perm + pA) : 0);
            nodeB = (flags & MLB_SORTED) ? pB : (okB ? __ldg(a.perm + pB) : 0);
            if (flags & MLB_USE_ISD) {
                sA = okA ? __ldg(a.isd + pA) : 1.0;
                sB = okB ? __ldg(a.isd + pB) : 1.0;
            }
        }
        // issue the point loads before (possibly) restaging the neighbourhood
        double fA0, fB0, fA1, fB1, fA2, fB2;
        if (PF) {
            fA0 = nf[0]; fB0 = nf[1]; fA1 = nf[2]; fB1 = nf[3]; fA2 = nf[4]; fB2 = nf[5];
        } else {
            fA0 = okA ? __ldg(a.frac + pA) : 0.5;
            fB0 = okB ? __ldg(a.frac + pB) : 0.5;
            fA1 = (D >= 2 && okA) ? __ldg(a.frac + a.n + pA) : 0.5;
            fB1 = (D >= 2 && okB) ? __ldg(a.frac + a.n + pB) : 0.5;
            fA2 = (D == 3 && okA) ? __ldg(a.frac + 2 * a.n + pA) : 0.5;
            fB2 = (D == 3 && okB) ? __ldg(a.frac + 2 * a.n + pB) : 0.5;
        }
        if (key != cur && !(flags & (1u << 18))) {  // bit 18: ablation (profiling only): no restaging
            __syncwarp();
            if (D == 3 && PK) {
                // rows (i, j) of the pencil block; columns past the group's width are not read
                for (int e = lane; e < S * S * SR; e += 32) {
                    const int row = e / SR, col = e % SR;
                    if (col < wst) cp_async8(nb + e, grid + gbase + (row / S) * rs + (row % S) * (int64_t)L + col);
                }
            } else {
                constexpr int NSRC = (D == 1) ? S : (D == 2 ? S * S : S * S * S);
                for (int e = lane; e < NSRC; e += 32) {
                    int64_t off;
                    if (D == 1) off = e;
                    else if (D == 2) off = (e / S) * rs + e % S;
                    else off = (e / (S * S)) * rs + ((e / S) % S) * (int64_t)L + e % S;
                    cp_async8(nb + e, grid + gbase + off);
                }
            }
            cp_async_wait_all();
            __syncwarp();
            cur = key;
        }
        // windows of both points and all axes: [A0 A1 A2 | B0 B1 B2] (first D of each)
        double wAB[2 * D][S];
        double (&wA0)[S] = wAB[0];
        double (&wA1)[S] = wAB[D >= 2 ? 1 : 0];
        double (&wA2)[S] = wAB[D == 3 ? 2 : 0];
        double (&wB0)[S] = wAB[D];
        double (&wB1)[S] = wAB[D >= 2 ? D + 1 : D];
        double (&wB2)[S] = wAB[D == 3 ? D + 2 : D];
        if (flags & (1u << 17)) {  // ablation (profiling only): constant windows
#pragma unroll
            for (int k = 0; k < 2 * D; ++k)
#pragma unroll
                for (int q = 0; q < S; ++q) wAB[k][q] = fA0 + fB1 + fA2;
        } else if (two) {   // one coefficient read feeds 2D FMAs
            double fk[2 * D];
            const double fa[3] = {fA0, fA1, fA2}, fb[3] = {fB0, fB1, fB2};
#pragma unroll
            for (int k = 0; k < D; ++k) {
                fk[k] = fa[k];
                fk[D + k] = fb[k];
            }
            kb_windows_k<M, 2 * D>(fk, wc, wAB);
        } else {
            double fk[D];
            const double fa[3] = {fA0, fA1, fA2};
#pragma unroll
            for (int k = 0; k < D; ++k) fk[k] = fa[k];
            double wa[D][S];
            kb_windows_k<M, D>(fk, wc, wa);
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
                for (int q = 0; q < S; ++q) {
                    wAB[k][q] = wa[k][q];
                    wAB[D + k][q] = 0.0;
                }
        }
        double vA = 0.0, vB = 0.0;
        if (D >= 2) {
#pragma unroll
            for (int q = 0; q < S; ++q) {
                w0s[q] = wA0[q];
                w0s[S + q] = wB0[q];
            }
        }
        if (EPF && v) {  // (the node indices have arrived during the window evaluation)
            vA = okA ? __ldg(v + nodeA) : 0.0;
            vB = okB ? __ldg(v + nodeB) : 0.0;
        }
        if (PF && ch + 1 < c_hi) load_frac(ch + 1);
        double accA = 0.0, accB = 0.0;
        if (flags & (1u << 16)) {  // ablation (profiling only): skip the contraction
            accA = wA0[0] + wA1[S - 1] + wA2[1];
            accB = wB0[0] + wB1[S - 1] + wB2[1] + nb[lane];
        } else if (D == 1) {
#pragma unroll
            for (int i = 0; i < S; ++i) {
                const double gv = nb[i];
                accA = fma(wA0[i], gv, accA);
                accB = fma(wB0[i], gv, accB);
            }
        } else if (D == 2) {
#pragma unroll
            for (int i = 0; i < S; ++i) {
                double rA = 0.0, rB = 0.0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const double gv = nb[i * S + j];
                    rA = fma(wA1[j], gv, rA);
                    rB = fma(wB1[j], gv, rB);
                }
                accA = fma(w0s[i], rA, accA);
                accB = fma(w0s[S + i], rB, accB);
            }
        } else if (!two) {
#pragma unroll 1
            for (int i = 0; i < S; ++i) {
                const double* gi = nb + dcA + i * S * SR;
                double rA = 0.0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    double qA = 0.0, qA2 = 0.0;  // two chains
#pragma unroll
                    for (int k = 0; k < S; ++k) {
                        if (k & 1) qA2 = fma(wA2[k], gi[j * SR + k], qA2);
                        else qA = fma(wA2[k], gi[j * SR + k], qA);
                    }
                    rA = fma(wA1[j], qA + qA2, rA);
                }
                accA = fma(w0s[i], rA, accA);
            }
        } else {
#pragma unroll 1
            for (int i = 0; i < S; ++i) {
                const double* gi = nb + dcA + i * S * SR;
                double rA = 0.0, rB = 0.0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    double qA = 0.0, qB = 0.0;
#pragma unroll
                    for (int k = 0; k < S; ++k) {
                        const double gv = gi[j * SR + k];
                        qA = fma(wA2[k], gv, qA);
                        qB = fma(wB2[k], gv, qB);
                    }
                    rA = fma(wA1[j], qA, rA);
                    rB = fma(wB1[j], qB, rB);
                }
                accA = fma(w0s[i], rA, accA);
                accB = fma(w0s[S + i], rB, accB);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool ok = h ? okB : okA;
            if (!ok) continue;
            const int p = h ? pB : pA;
            const double acc = h ? accB : accA;
            int node;
            double vv, s;
            if (EPF) {
                node = h ? nodeB : nodeA;
                vv = h ? vB : vA;
                s = h ? sB : sA;
            } else {
                node = (flags & MLB_SORTED) ? p : __ldg(a.perm + p);
                vv = v ? __ldg(v + node) : 0.0;
                s = (flags & MLB_USE_ISD) ? __ldg(a.isd + p) : 1.0;
            }
            double res = alpha * vv + s * (beta * acc + gamma * s * vv);
            if (flags & MLB_ACCUMULATE) res += y[node];
            y[node] = res;
        }
    }
    pdl_launch();
}

template <int D, int M, bool PK>
__global__ void __launch_bounds__(256, (D == 3 && M >= 5) ? 1 : 2) gather_kernel(FsArgs a, WinCoef wc,
                                                                                 const double* __restrict__ grid,
                                                                                 const double* __restrict__ v,
                                                                                 double* __restrict__ y, double alpha,
                                                                                 double beta, double gamma,
                                                                                 unsigned flags) {
    gather_body<D, M, PK>(a, wc, grid, v, y, alpha, beta, gamma, flags, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------ many small layers --
// mlb_apply_multi: T layers' fused Laplacians in one launch per stage,
// blockIdx.y = layer, each layer with its own block count along x (the CTAs
// past it exit at once).  For many small layers of one (d, m) -- config 3's
// 52 of 40,000 points -- whose per-layer launches are latency-bound.
struct MultiLayer {
    FsArgs a;
    double* grid;        // the layer's spread sum
    double* grid2;       // the convolved grid
    int spread_blocks;
    int gather_blocks;
    int cells;
};

// (the grouped d = 2 lanes: a small layer's few CTAs each walk thousands of points)
template <int D, int M>
__global__ void __launch_bounds__(32 * kBandWarps, kBandCtasPerSm) spread_multi_kernel(
    const MultiLayer* __restrict__ ml, WinCoef wc, const double* const* __restrict__ v, unsigned flags) {
    const MultiLayer& L = ml[blockIdx.y];
    if ((int)blockIdx.x >= L.spread_blocks) return;
    spread_body<D, M, true, true>(L.a, wc, v[blockIdx.y], flags, blockIdx.x, L.spread_blocks);
}

__global__ void grid_sum_multi_kernel(const MultiLayer* __restrict__ ml) {
    const MultiLayer& L = ml[blockIdx.y];
    if ((int)blockIdx.x * 8 >= L.cells) return;
    PeerOut out{};
    out.p[0] = L.grid;
    out.n = 1;
    grid_sum_body(L.a.partial, L.spread_blocks, L.cells, out, blockIdx.x);
}

template <int D, int M>
__global__ void __launch_bounds__(256, 2) gather_multi_kernel(const MultiLayer* __restrict__ ml, WinCoef wc,
                                                              const double* const* __restrict__ v,
                                                              double* const* __restrict__ y,
                                                              const double* __restrict__ abg, int T, unsigned flags) {
    const MultiLayer& L = ml[blockIdx.y];
    if ((int)blockIdx.x >= L.gather_blocks) return;
    const int t = blockIdx.y;
    gather_body<D, M, false>(L.a, wc, L.grid2, v[t], y[t], abg[t], abg[T + t], abg[2 * T + t], flags, blockIdx.x,
                             L.gather_blocks);
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
    a.chunk_gcell = b->chunk_gcell;
    a.sub_desc = reinterpret_cast<const int2*>(b->sub_desc);
    a.cblk = reinterpret_cast<const int4*>(b->cblk);
    a.wstream = reinterpret_cast<const int2*>(b->wstream);
    a.wstream_off = b->wstream_off;
    a.citem = b->citem;
    a.citem_off = b->citem_off;
    a.brick_blk = b->brick_blk;
    a.active_brick = b->active_brick;
    a.merge_off = b->merge_off;
    a.merge_pairs = b->merge_pairs;
    a.blocks = b->blocks;
    a.agrid = nullptr;
    a.cta_seg = nullptr;
    a.key_start = b->key_start;
    a.nkeys = b->nkeys;
    a.ggrp = reinterpret_cast<const int2*>(b->ggrp);
    a.gslot = b->gslot;
    a.ngrp = b->ngrp;
    a.seg_sub = b->seg_sub;
    a.seg_chunk = b->seg_chunk;
    a.seg_brick = b->seg_brick;
    a.brick_seg = b->brick_seg;
    a.brick_first = b->brick_first;
    a.isd = b->isd;
    a.partial = b->partial;
    a.tile_cells = b->tile_cells;
    a.nchunks = b->nchunks;
    a.nseg = b->nseg;
    return a;
}

template <int D, int M>
static size_t spread_smem(int nw, int tile_cells) {
    return (size_t)nw * tile_cells * 8 + (size_t)nw * (32 * D * StageCfg<D, M>::pad + (D == 2 ? 8 : 0)) * 8;
}

template <int D, int M>
static int spread_dm(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st) {
    FsArgs a = make_args(b);
    const int nsm = device_sms();
    (void)nsm;
    if constexpr (D == 1) {
        const size_t smem = (size_t)8 * b->tile_cells * sizeof(double);
        if (b->key_start && b->n >= kStream1MinN && smem <= 200 * 1024) {   // streaming d = 1 spread (fits: N <~ 3000)
            if (int rc = ensure_max_smem((const void*)spread1_kernel<M>, smem)) return rc;
            const int blocks = std::max(1, std::min(2 * nsm, (int)((b->n + 8 * K1STEP - 1) / (8 * K1STEP))));
            b->spread_parts = blocks;
            MLB_CUDA_TRY(launch_k(spread1_kernel<M>, dim3(blocks), dim3(256), smem, st, a, b->plan->wc, v, flags));
            note_launches(1);
            MLB_CUDA_TRY(cudaGetLastError());
            return MLB_OK;
        }
    }
    if constexpr (D <= 2) {
        // persistent CTAs of 8 warps, one partial grid per CTA; banded d = 2:
        // kBandWarps-warp CTAs over their own segment ranges, one band tile each
        const bool banded = D == 2 && b->ncta_band > 0;
        if (banded) {
            a.cta_seg = b->cta_seg;
            a.tile_cells = b->band_tile;
        }
        bool grouped = D == 2 && b->n >= (1 << 20);
        if (const char* env = std::getenv("MLB_D2_GROUPED")) grouped = D == 2 && env[0] == '1';  // tests / tuning
        int nw = (banded || grouped) ? kBandWarps : 8;   // (the grouped kernel's launch bounds: kBandWarps warps)
        while (!banded && nw > 1 && spread_smem<D, M>(nw, b->tile_cells) > 110 * 1024) --nw;
        const size_t smem = spread_smem<D, M>(nw, a.tile_cells);
        if (smem > 220 * 1024) return fail(MLB_ERR_CONFIG, "spread tile too large for shared memory");
        // grouped d = 2 lanes pay off on large layers (config 4: 622 -> 498
        // us); at config-2 size the plain lane blocks leave more room for
        // the concurrently running d = 3 layer (step 3.96 vs 3.86e9)
        auto kern = grouped ? spread_kernel<D, M, true, true> : spread_kernel<D, M, true, false>;
        MLB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int blocks = banded ? b->ncta_band : std::min(b->spread_parts_max, (b->nseg + nw - 1) / nw);
        if (blocks < 1) blocks = 1;
        b->spread_parts = blocks;
        MLB_CUDA_TRY(launch_k(kern, dim3(blocks), dim3(nw * 32), smem, st, a, b->plan->wc, v, flags, b->work));
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    } else {
        using C3 = SpreadCfg<3, M>;
        const size_t nred = (size_t)C3::S * C3::S * C3::SP;
        const size_t stg = (std::max<size_t>(32 * 3 * StageCfg<3, M>::pad, nred) + 1) & ~(size_t)1;
        const size_t smem = (size_t)kCellWarps * (stg + nred) * sizeof(double);
        if (smem > 220 * 1024) return fail(MLB_ERR_CONFIG, "spread staging too large for shared memory");
        auto kern3 = spread_cells_kernel<M>;
        if (int rc = ensure_max_smem((const void*)kern3, smem)) return rc;  // per (kernel, device)
        if (b->ncta_cells == 0) return MLB_OK;
        if (b->spread_atomic && b->atomic_target) {   // A/B mode: zero the target grid, blocks added atomically
            MLB_CUDA_TRY(cudaMemsetAsync(b->atomic_target, 0, b->grid_cells * sizeof(double), st));
            a.agrid = b->atomic_target;
        }
        MLB_CUDA_TRY(launch_k(kern3, dim3(b->ncta_cells), dim3(kCellWarps * 32), smem, st, a, b->plan->wc, v, flags));
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
}

template <int D, int M, bool PK>
static int gather_dmp(mlb_binding* b, const double* grid, const double* v, double* y, double alpha,
                      double beta, double gamma, unsigned flags, cudaStream_t st) {
    constexpr int S = 2 * M + 1;
    constexpr int NB = GatherCfg<D, M, PK>::NB;
    FsArgs a = make_args(b);
    const size_t smem = ((size_t)8 * NB + (size_t)256 * (2 * S + 1)) * sizeof(double);
    auto kern = gather_kernel<D, M, PK>;
    if (int rc = ensure_max_smem((const void*)kern, smem)) return rc;  // per (kernel, device)
    const int per_sm = occupancy_per_sm((const void*)kern, 256, smem);
    const int nsm = device_sms();
    int blocks = nsm * per_sm;
    const int need = ((D == 3 && PK ? b->ngrp : b->nchunks) + 7) / 8;  // at least one unit per warp
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    MLB_CUDA_TRY(launch_k(kern, dim3(blocks), dim3(256), smem, st, a, b->plan->wc, grid, v, y, alpha, beta, gamma, flags));
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

template <int D, int M>
static int gather_dm(mlb_binding* b, const double* grid, const double* v, double* y, double alpha,
                     double beta, double gamma, unsigned flags, cudaStream_t st) {
    if constexpr (D == 1) {
        const size_t smem = ((size_t)b->plan->g.L + (size_t)b->nkeys * (2 * M + 1)) * sizeof(double);
        if (b->key_start && b->n >= kStream1MinN && smem <= 200 * 1024) {   // streaming d = 1 gather
            FsArgs a = make_args(b);
            if (int rc = ensure_max_smem((const void*)gather1_kernel<M>, smem)) return rc;
            const int nsm = device_sms();
            const int blocks = std::max(1, std::min(2 * nsm, (int)((b->n + 8 * K1STEP - 1) / (8 * K1STEP))));
            MLB_CUDA_TRY(launch_k(gather1_kernel<M>, dim3(blocks), dim3(256), smem, st, a, b->plan->wc, grid, v, y,
                                  alpha, beta, gamma, flags));
            note_launches(1);
            MLB_CUDA_TRY(cudaGetLastError());
            return MLB_OK;
        }
    }
    if (D == 3 && b->gather_packed) return gather_dmp<D, M, true>(b, grid, v, y, alpha, beta, gamma, flags, st);
    return gather_dmp<D, M, false>(b, grid, v, y, alpha, beta, gamma, flags, st);
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
    if (b->lat_nitems > 0) return launch_lat_spread(b, v, flags, st);
    const Geom& g = b->plan->g;
    MLB_DISPATCH_DM(spread_dm, g.d, g.m, b, v, flags, st);
}

int launch_reduce(mlb_binding* b, double* grid_local, cudaStream_t st, const PeerOut* peers) {
    FsArgs a = make_args(b);
    PeerOut grid{};
    if (peers) {
        grid = *peers;
    } else {
        grid.p[0] = grid_local;
        grid.n = 1;
    }
    const Geom& G = b->plan->g;
    if (b->lat_nitems > 0) return launch_lat_reduce(b, grid, st);
    if (G.d == 2 && b->ncta_band > 0) {
        // the banded spread left one band tile per CTA
        const int cells = (int)b->grid_cells;
        MLB_CUDA_TRY(launch_k(band_sum_kernel, dim3((cells + 7) / 8), dim3(256), 0, st, (const double*)b->partial,
                              b->band_tile, G.TL, (const int32_t*)b->cta_row0,
                              reinterpret_cast<const int2*>(b->row_cta), cells, grid));
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    if (G.d <= 2) {
        // the spread left one partial grid per CTA
        const int cells = (int)b->grid_cells;
        MLB_CUDA_TRY(launch_k(grid_sum_kernel, dim3((cells + 7) / 8), dim3(256), 0, st, (const double*)b->partial,
                              b->spread_parts, cells, grid));
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    const int Tb = G.Tb;
    const int ngb = (G.L + Tb - 1) / Tb;
    const int64_t nblk = (int64_t)ngb * ngb * ngb;
    const int R = (G.TL + Tb - 1) / Tb;  // source bricks per axis
    if (b->nactive > 0) {
        const dim3 mg(G.TL, b->nactive);
        switch (G.m) {
            case 1: MLB_CUDA_TRY(launch_k(brick_merge_kernel<1>, mg, dim3(MergeCfg<1>::MT), 0, st, a)); break;
            case 2: MLB_CUDA_TRY(launch_k(brick_merge_kernel<2>, mg, dim3(MergeCfg<2>::MT), 0, st, a)); break;
            case 3: MLB_CUDA_TRY(launch_k(brick_merge_kernel<3>, mg, dim3(MergeCfg<3>::MT), 0, st, a)); break;
            case 4: MLB_CUDA_TRY(launch_k(brick_merge_kernel<4>, mg, dim3(MergeCfg<4>::MT), 0, st, a)); break;
            case 5: MLB_CUDA_TRY(launch_k(brick_merge_kernel<5>, mg, dim3(MergeCfg<5>::MT), 0, st, a)); break;
            default: MLB_CUDA_TRY(launch_k(brick_merge_kernel<6>, mg, dim3(MergeCfg<6>::MT), 0, st, a)); break;
        }
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
    }
    if (Tb == 4 && R * R * R <= 64) {
        const unsigned nb = (unsigned)((nblk + 3) / 4);
        switch (G.m) {
            case 2: MLB_CUDA_TRY(launch_k(reduce3_kernel<4, 2>, dim3(nb), dim3(256), 0, st, a, grid)); break;
            case 3: MLB_CUDA_TRY(launch_k(reduce3_kernel<4, 3>, dim3(nb), dim3(256), 0, st, a, grid)); break;
            case 4: MLB_CUDA_TRY(launch_k(reduce3_kernel<4, 4>, dim3(nb), dim3(256), 0, st, a, grid)); break;
            default: MLB_CUDA_TRY(launch_k(reduce3_kernel<4, 5>, dim3(nb), dim3(256), 0, st, a, grid)); break;
        }
        note_launches(1);
        MLB_CUDA_TRY(cudaGetLastError());
        return MLB_OK;
    }
    const int64_t total = b->grid_cells;
    int64_t blocks = (total + 255) / 256;
    if (blocks > device_sms() * 8) blocks = device_sms() * 8;
    if (Tb == 2) reduce_kernel<3, 2><<<(int)blocks, 256, 0, st>>>(a, grid);
    else reduce_kernel<3, 0><<<(int)blocks, 256, 0, st>>>(a, grid);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

// grid[i] = sum over ranks r (in rank order) of recv[r * cells + i]
__global__ void slot_sum_kernel(const double* __restrict__ recv, int world, int64_t cells, double* __restrict__ grid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < world; ++r) s += __ldcg(recv + (int64_t)r * cells + i);
        grid[i] = s;
    }
}

int launch_slot_sum(const double* recv, int world, int64_t cells, double* grid, cudaStream_t st) {
    if (cells <= 0) return MLB_OK;
    const int blocks = (int)std::min<int64_t>((cells + 255) / 256, (int64_t)device_sms() * 8);
    slot_sum_kernel<<<blocks, 256, 0, st>>>(recv, world, cells, grid);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_gather(mlb_binding* b, const double* grid, const double* v, double* y, double alpha, double beta,
                  double gamma, unsigned flags, cudaStream_t st) {
    if (b->nchunks == 0) return MLB_OK;
    if (b->lat_nitems > 0) return launch_lat_gather(b, grid, v, y, alpha, beta, gamma, flags, st);
    const Geom& g = b->plan->g;
    MLB_DISPATCH_DM(gather_dm, g.d, g.m, b, grid, v, y, alpha, beta, gamma, flags, st);
}

// ---------------------------------------------------------- many layers --
namespace {
struct MultiTab {
    MultiLayer* ml = nullptr;   // device, T entries
    ConvJob* jobs = nullptr;    // device, T entries
    int nw = 0, maxs = 0, maxg = 0, maxcells = 0;
};
std::mutex g_multi_mu;
std::map<std::vector<uint64_t>, MultiTab> g_multi;   // per binding set (binding uids)
}  // namespace

template <int M>
static int apply_multi_m(mlb_binding* const* b, int T, const double* const* v, double* const* y, const double* abg,
                         unsigned flags, cudaStream_t st) {
    constexpr int D = 2;
    constexpr int S = 2 * M + 1;
    constexpr int NB = GatherCfg<D, M, false>::NB;
    const int nsm = device_sms();
    const int tile = b[0]->tile_cells;
    int nw = kBandWarps;   // (spread_multi_kernel's launch bounds)
    while (nw > 1 && spread_smem<D, M>(nw, tile) > 72 * 1024) --nw;
    const size_t smem_s = spread_smem<D, M>(nw, tile);
    const size_t smem_g = ((size_t)8 * NB + (size_t)256 * (2 * S + 1)) * sizeof(double);
    auto ks = spread_multi_kernel<D, M>;
    auto kg = gather_multi_kernel<D, M>;
    if (int rc = ensure_max_smem((const void*)ks, smem_s)) return rc;
    if (int rc = ensure_max_smem((const void*)kg, smem_g)) return rc;
    std::vector<uint64_t> key(T);
    for (int t = 0; t < T; ++t) key[t] = b[t]->uid;
    MultiTab tab;
    {
        std::lock_guard<std::mutex> lk(g_multi_mu);
        auto it = g_multi.find(key);
        if (it != g_multi.end()) tab = it->second;
    }
    if (!tab.ml) {
        const int per_sm = occupancy_per_sm((const void*)kg, 256, smem_g);
        std::vector<MultiLayer> hml(T);
        std::vector<ConvJob> hjobs(T);
        for (int t = 0; t < T; ++t) {
            MultiLayer& L = hml[t];
            L.a = make_args(b[t]);
            L.grid = b[t]->grid;
            L.grid2 = b[t]->grid2;
            // the layers share the GPU: about two resident waves of CTAs in
            // total, so small layers get few CTAs (each spread CTA zeroes and
            // writes a whole sub-box tile: one CTA per segment would make the
            // tiles, not the points, the work)
            const int sshare = std::max(1, (2 * nsm + T - 1) / T);
            const int gshare = std::max(1, (2 * nsm * per_sm + T - 1) / T);
            L.spread_blocks = std::max(1, std::min(sshare, (b[t]->nseg + nw - 1) / nw));
            L.gather_blocks = std::max(1, std::min(gshare, (b[t]->nchunks + 7) / 8));
            L.cells = (int)b[t]->grid_cells;
            b[t]->spread_parts = L.spread_blocks;
            hjobs[t] = ConvJob{b[t]->grid, b[t]->grid2, b[t]->plan->sep};
            tab.maxs = std::max(tab.maxs, L.spread_blocks);
            tab.maxg = std::max(tab.maxg, L.gather_blocks);
            tab.maxcells = std::max(tab.maxcells, L.cells);
        }
        tab.nw = nw;
        MLB_CUDA_TRY(cudaMalloc(&tab.ml, sizeof(MultiLayer) * T));
        MLB_CUDA_TRY(cudaMalloc(&tab.jobs, sizeof(ConvJob) * T));
        MLB_CUDA_TRY(cudaMemcpy(tab.ml, hml.data(), sizeof(MultiLayer) * T, cudaMemcpyHostToDevice));
        MLB_CUDA_TRY(cudaMemcpy(tab.jobs, hjobs.data(), sizeof(ConvJob) * T, cudaMemcpyHostToDevice));
        std::lock_guard<std::mutex> lk(g_multi_mu);
        g_multi[key] = tab;
    }
    const Geom& g = b[0]->plan->g;
    MLB_CUDA_TRY(launch_k(ks, dim3(tab.maxs, T), dim3(32 * tab.nw), smem_s, st, (const MultiLayer*)tab.ml,
                          b[0]->plan->wc, v, flags));
    MLB_CUDA_TRY(launch_k(grid_sum_multi_kernel, dim3((tab.maxcells + 7) / 8, T), dim3(256), 0, st,
                          (const MultiLayer*)tab.ml));
    if (int rc = launch_sep_small_multi(tab.jobs, T, g.L, D, st)) return rc;
    MLB_CUDA_TRY(launch_k(kg, dim3(tab.maxg, T), dim3(256), smem_g, st, (const MultiLayer*)tab.ml, b[0]->plan->wc,
                          v, y, abg, T, flags));
    note_launches(3);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int launch_apply_multi(mlb_binding* const* b, int T, const double* const* v, double* const* y, const double* abg,
                       unsigned flags, cudaStream_t st) {
    // eligibility: one device, d = 2, one m, full-tile spreads (n < 2^20),
    // the separable one-CTA convolution, identical windows and tile sizes
    const mlb_plan* p0 = b[0]->plan;
    const int d = p0->g.d, m = p0->g.m, L = p0->g.L;
    const int64_t cells = b[0]->grid_cells;
    if (d != 2 || m < 2 || m > 5) return fail(MLB_ERR_CONFIG, "multi-layer apply covers d = 2, m <= 5");
    if ((2 * cells + 2 * L + 8) * 8 > 96 * 1024) return fail(MLB_ERR_CONFIG, "multi-layer apply: grid too large");
    for (int t = 0; t < T; ++t) {
        const mlb_binding* bt = b[t];
        const mlb_plan* p = bt->plan;
        if (p->device != p0->device || p->g.d != d || p->g.m != m || p->g.L != L || !p->sep ||
            bt->tile_cells != b[0]->tile_cells || bt->grid_cells != cells || bt->n < 1 || bt->n >= (1 << 20) ||
            bt->ncta_band > 0 || bt->lat_nitems > 0 || bt->spread_atomic || std::memcmp(&p->wc, &p0->wc, sizeof(WinCoef)) != 0)
            return fail(MLB_ERR_CONFIG, "multi-layer apply: layers differ in (d, m, grid, windows) or are large");
    }
    switch (m) {
        case 2: return apply_multi_m<2>(b, T, v, y, abg, flags, st);
        case 3: return apply_multi_m<3>(b, T, v, y, abg, flags, st);
        case 4: return apply_multi_m<4>(b, T, v, y, abg, flags, st);
        default: return apply_multi_m<5>(b, T, v, y, abg, flags, st);
    }
}

}  // namespace mlb
