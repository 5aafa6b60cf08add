// Device binding: the per-point half of bind_points / _make_binding
// (fastsum.py:333-386) on the GPU.
//
// The reference builds, per point, the (2m+1)^d tensor product of flat grid
// indices and window weights and stable-argsorts it by grid index (16 C
// bytes per point: 213 GB at config 4).  The B200 binding is geometry only:
// per point the cell u = floor(ng * x * scale) and the fractional offset
// f = ng * x * scale - u per axis, the points stably sorted by
// (brick, cell-in-brick) key, and the per-key point counts from which the
// host builds the (cell-level) work tables.  Everything per point runs here:
//
//   1. bind_points_kernel   optional box map of raw feature columns
//                           x -> clip((x - mid) / half, -1, 1) * s
//                           (datapipe.py:100-123, bitwise as numpy), the box
//                           check |x| <= 1/4 - eps_b/2 (+1e-12, fastsum.py:66-80),
//                           cell / key / fractional offsets (fastsum.py:343-353)
//   2. cub radix sort       (key, point) pairs, LSD radix = stable: the same
//                           permutation as the reference's stable argsort by
//                           cell order within the brick layout
//   3. key_bounds_kernel    first / one-past-last sorted position of every key
//   4. sorted_soa_kernel    fractional offsets in sorted order (SoA) and the
//                           sorted -> node permutation (node ids of a
//                           component block, graphs.py:99-129)
//
// The host then receives 2 x nkeys int32 (nkeys = bricks x cells per brick,
// ~10^4-10^5) instead of walking n points.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <cstring>
#include <string>
#include <vector>

#include "mlb_internal.cuh"

namespace mlb {

struct BindGeomDev {
    int d, ng, bin_lo, nb, Tb, nbr, nloc;
    double scale;
    int ld;
    int cols[3];
    int affine;
    double mid[3];
    double half, s;
};

__device__ __forceinline__ void atomic_max_pos(unsigned long long* a, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(a, (unsigned long long)__double_as_longlong(v));
}

template <int D>
__global__ void bind_points_kernel(BindGeomDev G, const double* __restrict__ pts, int64_t n,
                                   int32_t* __restrict__ key, int32_t* __restrict__ idx, double* __restrict__ f,
                                   unsigned long long* __restrict__ worst, int* __restrict__ nonfinite,
                                   unsigned long long* __restrict__ first_bad) {
    double wmax = 0.0;
    int nf = 0;
    unsigned long long bad = (unsigned long long)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int brick = 0, local = 0;
        bool ok = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double x = pts[i * G.ld + G.cols[a]];
            if (G.affine) {
                // numpy: np.clip((X - mid) / half, -1, 1) * s, elementwise, IEEE round-to-nearest
                x = __ddiv_rn(__dsub_rn(x, G.mid[a]), G.half);
                x = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
                x = __dmul_rn(x, G.s);
            }
            if (!isfinite(x)) {
                nf = 1;
                ok = false;
                continue;
            }
            wmax = fmax(wmax, fabs(x));
            // tx = ng * (x * scale); u = floor(tx)  (fastsum.py:343-353, :386)
            const double tx = __dmul_rn((double)G.ng, __dmul_rn(x, G.scale));
            const double fl = floor(tx);
            const int bin = (int)fl - G.bin_lo;
            if (!(bin >= 0 && bin < G.nb)) {
                ok = false;
                continue;
            }
            f[i * D + a] = __dsub_rn(tx, fl);
            brick = brick * G.nbr + bin / G.Tb;
            local = local * G.Tb + bin % G.Tb;
        }
        if (!ok && (unsigned long long)i < bad) bad = (unsigned long long)i;
        key[i] = ok ? brick * G.nloc + local : 0;
        idx[i] = (int32_t)i;
    }
    // one atomic per warp for each reduction
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        wmax = fmax(wmax, __shfl_down_sync(0xffffffffu, wmax, off));
        nf |= __shfl_down_sync(0xffffffffu, nf, off);
        const unsigned long long ob = __shfl_down_sync(0xffffffffu, bad, off);
        bad = ob < bad ? ob : bad;
    }
    if ((threadIdx.x & 31) == 0) {
        if (wmax > 0.0) atomic_max_pos(worst, wmax);
        if (nf) atomicOr(nonfinite, 1);
        if (bad < (unsigned long long)n) atomicMin(first_bad, bad);
    }
}

__global__ void key_bounds_kernel(const int32_t* __restrict__ ks, int64_t n, int32_t* __restrict__ start,
                                  int32_t* __restrict__ end) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = ks[j];
        if (j == 0 || ks[j - 1] != k) start[k] = (int32_t)j;
        if (j == n - 1 || ks[j + 1] != k) end[k] = (int32_t)(j + 1);
    }
}

template <int D>
__global__ void sorted_soa_kernel(const int32_t* __restrict__ perm, const double* __restrict__ f, int64_t n,
                                  const int32_t* __restrict__ node_ids, double* __restrict__ fs,
                                  int32_t* __restrict__ perm_node) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = perm[j];
#pragma unroll
        for (int a = 0; a < D; ++a) fs[(int64_t)a * n + j] = f[(int64_t)p * D + a];
        perm_node[j] = node_ids ? node_ids[p] : p;
    }
}

static int grid1d(int64_t n, int per_block = 256) {
    int64_t b = (n + per_block - 1) / per_block;
    const int64_t cap = (int64_t)device_sms() * 16;
    if (b > cap) b = cap;
    return (int)(b < 1 ? 1 : b);
}

// RAII for the bind's temporary device buffers
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() {
        return static_cast<T*>(p);
    }
};

int bind_points_device(const BindPointsIn& in, const Geom& g, BindPointsOut* out) {
    const int64_t n = in.n;
    const int d = g.d;
    cudaStream_t st = (cudaStream_t)in.stream;
    BindGeomDev G{};
    G.d = d;
    G.ng = g.ng;
    G.bin_lo = g.ulo + g.m;
    G.nb = g.nb;
    G.Tb = g.Tb;
    G.nbr = g.nbr;
    G.nloc = 1;
    for (int a = 0; a < d; ++a) G.nloc *= g.Tb;
    G.scale = in.scale;
    G.ld = in.ld;
    for (int a = 0; a < d; ++a) G.cols[a] = in.cols ? in.cols[a] : a;
    G.affine = in.box_mid != nullptr;
    if (G.affine) {
        for (int a = 0; a < d; ++a) G.mid[a] = in.box_mid[a];
        G.half = in.box_half;
        G.s = in.box_s;
    }
    int nkeys = G.nloc;
    for (int a = 0; a < d; ++a) nkeys *= g.nbr;
    out->nkeys = nkeys;
    out->cnt.assign((size_t)nkeys + 1, 0);
    out->perm = nullptr;
    out->frac = nullptr;
    if (n == 0) return MLB_OK;
    int key_bits = 1;
    while (key_bits < 31 && ((int64_t)1 << key_bits) < nkeys) ++key_bits;

    DevBuf pts_buf, keys, keys_s, idx, idx_s, f, red, bounds, tmp, fs, perm_node, ids;
    const double* pts = in.points;
    if (!in.points_on_device) {
        const int lcols = in.ld;
        MLB_CUDA_TRY(cudaMalloc(&pts_buf.p, (size_t)n * lcols * sizeof(double)));
        MLB_CUDA_TRY(cudaMemcpyAsync(pts_buf.p, in.points, (size_t)n * lcols * sizeof(double),
                                     cudaMemcpyHostToDevice, st));
        pts = pts_buf.as<double>();
    }
    MLB_CUDA_TRY(cudaMalloc(&keys.p, (size_t)n * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMalloc(&keys_s.p, (size_t)n * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMalloc(&idx.p, (size_t)n * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMalloc(&idx_s.p, (size_t)n * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMalloc(&f.p, (size_t)n * d * sizeof(double)));
    MLB_CUDA_TRY(cudaMalloc(&red.p, 4 * sizeof(unsigned long long)));
    unsigned long long init[4] = {0ull, 0ull, (unsigned long long)n, 0ull};  // worst, nonfinite, first bad
    MLB_CUDA_TRY(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    unsigned long long* R = red.as<unsigned long long>();
    const int gb = grid1d(n);
    if (d == 1)
        bind_points_kernel<1><<<gb, 256, 0, st>>>(G, pts, n, keys.as<int32_t>(), idx.as<int32_t>(), f.as<double>(), R,
                                                 reinterpret_cast<int*>(R + 1), R + 2);
    else if (d == 2)
        bind_points_kernel<2><<<gb, 256, 0, st>>>(G, pts, n, keys.as<int32_t>(), idx.as<int32_t>(), f.as<double>(), R,
                                                 reinterpret_cast<int*>(R + 1), R + 2);
    else
        bind_points_kernel<3><<<gb, 256, 0, st>>>(G, pts, n, keys.as<int32_t>(), idx.as<int32_t>(), f.as<double>(), R,
                                                 reinterpret_cast<int*>(R + 1), R + 2);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    unsigned long long res[4];
    MLB_CUDA_TRY(cudaMemcpyAsync(res, red.p, sizeof(res), cudaMemcpyDeviceToHost, st));
    MLB_CUDA_TRY(cudaStreamSynchronize(st));
    double worst;
    std::memcpy(&worst, &res[0], sizeof(double));
    out->worst = worst;
    if ((int)res[1]) return fail(MLB_ERR_CONFIG, "points contain non-finite values");
    if (in.box_hw > 0.0 && worst > in.box_hw + 1e-12) {
        char msg[160];
        snprintf(msg, sizeof msg, "points exceed the admissible box: max |coord| = %.6g > 1/4 - eps_b/2 = %.6g", worst,
                 in.box_hw);
        return fail(MLB_ERR_CONFIG, msg);
    }
    if (res[2] < (unsigned long long)n)
        return fail(MLB_ERR_CONFIG, "point " + std::to_string(res[2]) + " lies outside the plan's admissible box");

    // 2. stable LSD radix sort of (key, point)
    size_t tmp_bytes = 0;
    MLB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.as<int32_t>(), keys_s.as<int32_t>(),
                                                 idx.as<int32_t>(), idx_s.as<int32_t>(), (int)n, 0, key_bits, st));
    MLB_CUDA_TRY(cudaMalloc(&tmp.p, tmp_bytes > 0 ? tmp_bytes : 16));
    MLB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.as<int32_t>(), keys_s.as<int32_t>(),
                                                 idx.as<int32_t>(), idx_s.as<int32_t>(), (int)n, 0, key_bits, st));
    note_launches(1);
    // 3. per-key bounds
    MLB_CUDA_TRY(cudaMalloc(&bounds.p, (size_t)2 * nkeys * sizeof(int32_t)));
    MLB_CUDA_TRY(cudaMemsetAsync(bounds.p, 0, (size_t)2 * nkeys * sizeof(int32_t), st));
    int32_t* start = bounds.as<int32_t>();
    int32_t* end = start + nkeys;
    key_bounds_kernel<<<grid1d(n), 256, 0, st>>>(keys_s.as<int32_t>(), n, start, end);
    note_launches(1);
    // 4. sorted SoA offsets and the sorted -> node permutation
    MLB_CUDA_TRY(cudaMalloc(&fs.p, (size_t)n * d * sizeof(double)));
    MLB_CUDA_TRY(cudaMalloc(&perm_node.p, (size_t)n * sizeof(int32_t)));
    if (in.node_ids) {
        MLB_CUDA_TRY(cudaMalloc(&ids.p, (size_t)n * sizeof(int32_t)));
        MLB_CUDA_TRY(cudaMemcpyAsync(ids.p, in.node_ids, (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    }
    if (d == 1)
        sorted_soa_kernel<1><<<grid1d(n), 256, 0, st>>>(idx_s.as<int32_t>(), f.as<double>(), n, ids.as<int32_t>(),
                                                        fs.as<double>(), perm_node.as<int32_t>());
    else if (d == 2)
        sorted_soa_kernel<2><<<grid1d(n), 256, 0, st>>>(idx_s.as<int32_t>(), f.as<double>(), n, ids.as<int32_t>(),
                                                        fs.as<double>(), perm_node.as<int32_t>());
    else
        sorted_soa_kernel<3><<<grid1d(n), 256, 0, st>>>(idx_s.as<int32_t>(), f.as<double>(), n, ids.as<int32_t>(),
                                                        fs.as<double>(), perm_node.as<int32_t>());
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    std::vector<int32_t> hb((size_t)2 * nkeys);
    MLB_CUDA_TRY(cudaMemcpyAsync(hb.data(), bounds.p, hb.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    MLB_CUDA_TRY(cudaStreamSynchronize(st));
    // cnt[k] = first sorted position of key k (empty keys: the next key's start)
    int64_t pos = 0;
    for (int k = 0; k < nkeys; ++k) {
        out->cnt[k] = pos;
        const int32_t e = hb[(size_t)nkeys + k];
        if (e > 0) {  // a non-empty key (sorted keys: its run starts where the previous one ended)
            if (hb[k] != pos || e <= pos) return fail(MLB_ERR_CUDA, "device binding: inconsistent key runs");
            pos = e;
        }
    }
    out->cnt[nkeys] = pos;
    if (pos != n) return fail(MLB_ERR_CUDA, "device binding: per-key bounds do not cover the points");
    out->frac = fs.as<double>();
    out->perm = perm_node.as<int32_t>();
    fs.p = nullptr;         // ownership moves to the binding
    perm_node.p = nullptr;
    return MLB_OK;
}

}  // namespace mlb
