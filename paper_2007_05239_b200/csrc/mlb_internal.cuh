// Internal declarations of libmlb.so (B200 / sm_100a NFFT Laplacian path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/multilap_b200.h"

namespace mlb {

void set_error(const std::string& msg);
void note_launches(int k);  // libmlb kernel-launch counter (bench evidence)
int fail(int code, const std::string& msg);

// Programmatic dependent launch: a kernel launched with launch_k may start
// (prologue: static tables, shared memory) while its stream predecessor is
// finishing; it must call pdl_wait() before touching anything a predecessor
// writes or reads, and calls pdl_launch() once its own main work is done.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // MLB_NO_PDL=1 disables (A/B)

// Outputs of the final grid reduction (R2): the local grid, or -- node-range
// sharding over NVLink -- this rank's slot in every peer's receive buffer
// (P2P stores from the reduction kernel itself: the spread's grid exchange
// is fused into the kernel that produces the grid).
constexpr int kMaxPeers = 8;
struct PeerOut {
    double* p[kMaxPeers];
    int n;
};
__device__ __forceinline__ void po_store(const PeerOut& o, int64_t i, double v) {
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
        if (q < o.n) o.p[q][i] = v;
}
int device_sms(int device = -1);  // SM count of `device` (-1: current), cached
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the CURRENT device,
// remembered per (kernel, device) so a second GPU in the process gets its own
// call (thread-safe); returns MLB_OK or MLB_ERR_CUDA
int ensure_max_smem(const void* kern, size_t smem);
// resident blocks per SM of `kern` at (threads, smem) on the current device, cached per (kernel, device)
int occupancy_per_sm(const void* kern, int threads, size_t smem);

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

#define MLB_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return ::mlb::fail(MLB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

constexpr int kMaxM = 6;          // window cutoffs supported by the kernels
constexpr int kChunk = 64;        // points per chunk (<= 2 per warp lane)
constexpr int kItemInts = 32;   // d = 3 spread item row: nb + 3 x (<= 8) entries, padded
constexpr int kCellWarps = 8;   // warps per d = 3 spread CTA
constexpr int kBandWarps = 4;    // warps per banded d = 2 spread CTA
#ifndef MLB_BAND_CTAS
#define MLB_BAND_CTAS 3
#endif
constexpr int kBandCtasPerSm = MLB_BAND_CTAS;   // resident banded spread CTAs per SM (launch bounds, grid; 4 = 128 registers: spills, d=2 spread 0.35 -> 0.56 ms)
constexpr int64_t kStream1MinN = 1 << 16;  // d = 1: streaming kernels from this many points
constexpr int kSegPoints = 256;   // points per spread work unit (one warp)
constexpr int kMaxWinCoef = 17;   // monomial degree <= 16

// Window polynomial coefficients, passed by value as a kernel parameter
// (lives in constant bank 0 so the DFMAs read coefficients as c[] operands).
// Even/odd split of the pairs P_q / P_{1-q}, q = 1..m, plus P_{-m}.
struct WinCoef {
    double e[kMaxM][9];   // even part of P_q in s^2 (up to 9 terms)
    double o[kMaxM][8];   // odd part of P_q: P_q = E(s^2) + s*O(s^2)
    double mm[kMaxWinCoef];  // P_{-m}, monomial in s
    int deg;
};

// one layer's convolution in the multi-layer launch (mlb_apply_multi)
struct ConvJob {
    const double* gin;
    double* gout;
    const double* c;   // the plan's separable kernel (2L - 1 taps)
};
int launch_sep_small_multi(const ConvJob* jobs_dev, int T, int L, int d, cudaStream_t st);

// Geometry shared by all kernels of one plan.
struct Geom {
    int d, N, m, ng;
    int S;        // 2m+1 stencil width
    int nb;       // bins per axis
    int L;        // active cells per axis = nb + 2m
    int ulo;      // first active cell (signed torus index) = bin_lo - m
    int K, Kh;    // N+1, N/2+1
    int Tb, TL;   // brick bins per axis, brick tile cells per axis (Tb + 2m)
    int nbr;      // bricks per axis
    double K0;
};

}  // namespace mlb

struct mlb_plan {
    int device;
    int nsm;                     // SM count of the device (grid sizing at bind time)
    mlb::Geom g;
    mlb::WinCoef wc;
    double* fused = nullptr;     // band weights (K^(d-1) x Kh)
    double2* twid = nullptr;     // L x K
    double* conv = nullptr;      // d <= 2: (2L-1)^d spatial kernel (nullptr: use the DFT stages)
    double* sep = nullptr;       // separable 1-D kernel (2L-1), nullptr if F is not rank-1
    std::vector<double> win_coef_host;
};

struct mlb_binding {
    const mlb_plan* plan;
    int device = 0;                  // plan->device, kept for destroy
    uint64_t uid = 0;                // unique per binding (multi-layer table cache key)
    int64_t n;
    int nchunks, nseg, nbricks;
    // device tables
    int32_t* perm = nullptr;         // sorted -> node
    double* frac = nullptr;          // d x n (SoA) fractional cell offsets f in [0,1)
    int32_t* chunk_start = nullptr;  // nchunks+1
    int32_t* chunk_cell = nullptr;   // nchunks: flat tile index of the chunk's bin base cell
    int32_t* chunk_gcell = nullptr;  // nchunks: flat sub-box (L^d) index of the bin base cell
    // d = 3 gather groups (bind: pencil packing)
    int32_t* ggrp = nullptr;         // ngrp x {grid index of the first staged cell, width | two << 8}
    int32_t* gslot = nullptr;        // ngrp x 64: sorted point | axis-2 offset << 29, -1 = empty
    int ngrp = 0;
    int gather_packed = 0;           // d = 3: gather on pencil groups (light cells) instead of one-cell chunks
    int32_t* seg_chunk = nullptr;    // nseg+1
    int32_t* sub_desc = nullptr;     // 2 x nsub: {first point, (count << 24) | tile cell}, segment order
    int32_t* seg_sub = nullptr;      // nseg+1: CSR of sub-chunks per segment
    int32_t* seg_brick = nullptr;    // nseg
    int32_t* brick_seg = nullptr;    // nbricks+1 (CSR, bricks lexicographic)
    int32_t* brick_first = nullptr;  // nbricks: first segment of the brick (d = 3: brick tile slot), -1 if empty
    // d = 3 cell blocks: every cell's points (split into parts of <= cell_cap)
    // spread into one (2m+1)^3 block; CTAs of 8 warps own static item lists
    int32_t* cblk = nullptr;         // nblk x {first point, count, tile cell, brick}
    int nblk = 0;
    int32_t* wstream = nullptr;      // per-warp sub-chunk streams: {first point, (count << 24) | end-of-item}
    int32_t* wstream_off = nullptr;  // ncta*8 + 1
    int32_t* citem = nullptr;        // items in CTA order, kItemInts ints each: nb, (block, warp lo, warps) x nb
    int32_t* citem_off = nullptr;    // ncta + 1
    int ncta_cells = 0;              // spread CTAs the streams were built for
    int32_t* brick_blk = nullptr;    // nbricks + 1: CSR of blocks per brick (merge)
    int32_t* active_brick = nullptr; // nactive: bricks with points, slot order
    int32_t* merge_off = nullptr;    // nactive*TL + 1: CSR of block rows per (brick slot, tile slab)
    int32_t* merge_pairs = nullptr;  // {block * S + row o0, (c1 << 8) | c2}
    int nactive = 0;
    double* blocks = nullptr;        // nblk x (2m+1)^3
    int* work = nullptr;             // spread work counter (reset before every launch)
    int spread_parts = 0;            // d <= 2: partial grids written by the last spread (one per CTA)
    int spread_parts_max = 0;        // capacity of `partial` in whole grids (d <= 2)
    double* isd = nullptr;           // sorted order
    // scratch
    double* partial = nullptr;       // nseg x TL^d
    double* grid = nullptr;          // L^d (spread result)
    double* grid2 = nullptr;         // L^d (convolved)
    double* stage_a = nullptr;       // complex DFT intermediates
    double* stage_b = nullptr;
    int64_t stage_elems = 0;         // doubles per stage buffer
    int tile_cells = 0;              // TL^d
    int64_t grid_cells = 0;          // L^d
    int max_seg_chunks = 0;
    // d = 3 A/B mode (env MLB_SPREAD_ATOMIC=1 at bind time): the spread adds
    // cell blocks into atomic_target with red.global.add (no merge / R2)
    int spread_atomic = 0;
    double* atomic_target = nullptr;
    // d = 2 banded spread (large layers): CTA c owns segments
    // [cta_seg[c], cta_seg[c+1]) and a tile of the sub-box rows
    // [cta_row0[c], cta_row0[c] + band_tile / TL); sub_desc cells are
    // band-relative; row_cta[u0] = {first, last} CTA whose band covers row u0
    int ncta_band = 0;               // 0: not banded
    int band_tile = 0;               // cells per band tile (rows x TL)
    int32_t* cta_seg = nullptr;      // ncta_band + 1
    int32_t* cta_row0 = nullptr;     // ncta_band
    int32_t* row_cta = nullptr;      // 2 x L
    // d = 1 streaming spread / gather: first sorted point of every cell
    int32_t* key_start = nullptr;    // nkeys + 1 (nullptr: sub-chunk kernels)
    int nkeys = 0;
    // d = 2 lattice items (mlb_lattice.cu; 0 items: the kernels above)
    int lat_nitems = 0;
    int64_t lat_points = 0;          // points in lattice cells of >= 2 x 2
    int lat_nf_max = 0;              // widest fast-axis window table of an item
    int lat_r_max = 0;               // most rows of an item
    int lat_sv_max = 0;              // largest staged s v block (rows at an odd stride)
    int32_t* lat_items = nullptr;    // nitems x {first point, rows, C | fast << 16 | diag << 17, sub-box cell}
    int32_t* lat_bin_off = nullptr;  // nb^2 + 1: CSR of items per bin (items stored in bin order)
    double* lat_blocks = nullptr;    // nitems x (2m+1)^2
};

namespace mlb {
// device half of the binding (mlb_bind.cu)
struct BindPointsIn {
    const double* points;     // n rows of `ld` doubles; columns cols[0..d) (or 0..d) are the coordinates
    int points_on_device;
    int64_t n;
    int ld;
    const int* cols;          // nullable (host)
    double scale;             // torus scale
    const double* box_mid;    // nullable (host, d): affine box map of raw features
    double box_half, box_s;
    double box_hw;            // > 0: validate_box on the box coordinates
    const int32_t* node_ids;  // nullable (host)
    void* stream;
};
struct BindPointsOut {
    int nkeys = 0;
    std::vector<int64_t> cnt;  // nkeys + 1: first sorted position of every key
    int32_t* perm = nullptr;   // device, sorted -> node (owned by the caller afterwards)
    double* frac = nullptr;    // device, d x n SoA
    double worst = 0.0;        // max |box coordinate|
};
int bind_points_device(const BindPointsIn& in, const Geom& g, BindPointsOut* out);

// kernels launchers (mlb_fastsum.cu)
int launch_spread(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st);
int launch_reduce(mlb_binding* b, double* grid, cudaStream_t st, const PeerOut* peers = nullptr);
int launch_slot_sum(const double* recv, int world, int64_t cells, double* grid, cudaStream_t st);
int launch_convolve(mlb_binding* b, const double* gin, double* gout, cudaStream_t st);
int launch_gather(mlb_binding* b, const double* grid, const double* v, double* y, double alpha,
                  double beta, double gamma, unsigned flags, cudaStream_t st);
// d = 2 lattice (separable-per-cell) kernels (mlb_lattice.cu)
#ifndef MLB_LAT_THREADS
#define MLB_LAT_THREADS 256
#endif
constexpr int kLatRowsMax = MLB_LAT_THREADS;   // rows per lattice item (<= one per thread)
constexpr int kLatThreads = MLB_LAT_THREADS;   // threads per lattice CTA
constexpr int kLatCols = kLatThreads;          // widest lattice run C (a gather thread owns a column)
constexpr int kLatPts = 8 * kLatThreads;       // points per lattice item (8 per spread thread)
constexpr int kLatGatherSlots = 8;             // points per gather thread and item
constexpr int64_t kLatMinN = 1 << 16;     // auto mode: layers from this many points
int build_lattice(mlb_binding* b, const std::vector<int64_t>& cnt, const std::vector<int32_t>& key_gcell, int mode,
                  cudaStream_t st);
int launch_lat_spread(mlb_binding* b, const double* v, unsigned flags, cudaStream_t st);
int launch_lat_reduce(mlb_binding* b, const PeerOut& grid, cudaStream_t st);
int launch_lat_gather(mlb_binding* b, const double* grid, const double* v, double* y, double alpha, double beta,
                      double gamma, unsigned flags, cudaStream_t st);
int launch_apply_multi(mlb_binding* const* b, int T, const double* const* v, double* const* y, const double* abg,
                       unsigned flags, cudaStream_t st);
}  // namespace mlb
