// libmlb.so C ABI: errors, plans, bindings (host counting sort), apply.
//
// bind_points / _make_binding (fastsum.py:333-386) on the reference build the
// full (2m+1)^d tensor product of flat indices and weights per point (16 C
// bytes per point) and stable-argsort it.  Here the binding is geometry only:
// per point the fractional offsets f = ng*x - floor(ng*x) (8d bytes), the
// permutation to cell order, and chunk/segment tables; window weights are
// recomputed by the kernels on every apply.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <queue>
#include <cstdio>
#include <vector>

#include "mlb_internal.cuh"

namespace mlb {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MLB_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

void set_error(const std::string& msg) { g_err = msg; }

int device_sms(int device) {
    static int cache[64] = {0};
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) return 148;
    if (device >= 64) device = 63;
    if (cache[device] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
        cache[device] = n;
    }
    return cache[device];
}

int ensure_max_smem(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    MLB_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[{kern, dev}];
    if (smem <= cur) return MLB_OK;
    MLB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
    return MLB_OK;
}

int occupancy_per_sm(const void* kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, size_t>, int> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(kern, dev, threads, smem);
    auto it = done.find(key);
    if (it != done.end()) return it->second;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    done[key] = per_sm;
    return per_sm;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// Restores the caller's current device (torch keeps its own notion of it).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        // a failed switch must not leave cudaErrorInvalidDevice as the
        // runtime's last error: libcudart is shared with torch, whose next
        // launch check would report it
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) (void)cudaGetLastError();
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
static int dev_upload(T** dst, const T* src, size_t count) {
    if (count == 0) count = 1;
    MLB_CUDA_TRY(cudaMalloc((void**)dst, count * sizeof(T)));
    if (src) MLB_CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return MLB_OK;
}

template <typename T>
static void dev_free(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

static int ipow_h(int b, int e) {
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

}  // namespace mlb

using namespace mlb;

extern "C" {

int mlb_abi_version(void) { return MLB_ABI_VERSION; }

const char* mlb_last_error(void) { return g_err.c_str(); }

int64_t mlb_launch_count(void) { return g_launches.load(); }
void mlb_note_launches(int64_t k) {
    if (k > 0) g_launches += k;
}

int mlb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int mlb_plan_create(const mlb_plan_desc* desc, int device, mlb_plan** out) {
    if (!desc || !out) return fail(MLB_ERR_ARG, "null argument");
    const int d = desc->d, N = desc->N, m = desc->m, ng = desc->ng;
    if (d < 1 || d > 3) return fail(MLB_ERR_CONFIG, "fastsum supports d in {1, 2, 3}");
    if (N < 4 || N % 2) return fail(MLB_ERR_CONFIG, "N must be even and >= 4");
    if (m < 2 || m > kMaxM)
        return fail(MLB_ERR_CONFIG, "m_nfft must lie in [2, " + std::to_string(kMaxM) + "] on the GPU path");
    if (ng < N + 2 || ng % 2) return fail(MLB_ERR_CONFIG, "invalid oversampled grid size");
    if (desc->bin_hi < desc->bin_lo) return fail(MLB_ERR_CONFIG, "empty bin range");
    const int want_deg = (m <= 3) ? 15 : 13;   // mlb_window.cuh WinDeg
    if (desc->win_deg != want_deg)
        return fail(MLB_ERR_CONFIG, "window polynomial degree must be " + std::to_string(want_deg));
    DeviceGuard guard(device);
    mlb_plan* p = new mlb_plan();
    p->device = device;
    p->nsm = device_sms(device);
    Geom& g = p->g;
    g.d = d;
    g.N = N;
    g.m = m;
    g.ng = ng;
    g.S = 2 * m + 1;
    g.nb = desc->bin_hi - desc->bin_lo + 1;
    g.L = g.nb + 2 * m;
    g.ulo = desc->bin_lo - m;
    g.K = N + 1;
    g.Kh = N / 2 + 1;
    g.K0 = desc->K0;
    if (d <= 2) {
        g.Tb = g.nb;  // the whole sub-box is one brick
    } else {
        g.Tb = (m >= 6) ? 2 : 4;
        if (g.Tb > g.nb) g.Tb = g.nb;
    }
    g.TL = g.Tb + 2 * m;
    g.nbr = (g.nb + g.Tb - 1) / g.Tb;
    // window coefficients: split P_q (q=1..m) into even/odd parts in s
    const int nc = desc->win_deg + 1;
    p->win_coef_host.assign(desc->win_coef, desc->win_coef + (size_t)(2 * m + 1) * nc);
    std::memset(&p->wc, 0, sizeof(WinCoef));
    p->wc.deg = desc->win_deg;
    for (int q = 1; q <= m; ++q) {
        const double* c = desc->win_coef + (size_t)(q + m) * nc;  // o = q
        for (int j = 0; j < nc; ++j) {
            if (j % 2 == 0) p->wc.e[q - 1][j / 2] = c[j];
            else p->wc.o[q - 1][j / 2] = c[j];
        }
    }
    for (int j = 0; j < nc; ++j) p->wc.mm[j] = desc->win_coef[j];  // o = -m
    // device tables
    size_t nf = (size_t)g.Kh;
    for (int i = 1; i < d; ++i) nf *= g.K;
    int rc = dev_upload(&p->fused, desc->fused_band, nf);
    if (rc == MLB_OK) {
        std::vector<double2> tw((size_t)g.L * g.K);
        for (size_t i = 0; i < tw.size(); ++i) tw[i] = make_double2(desc->twiddle[2 * i], desc->twiddle[2 * i + 1]);
        rc = dev_upload(&p->twid, tw.data(), tw.size());
    }
    if (rc == MLB_OK && desc->sep_kernel) rc = dev_upload(&p->sep, desc->sep_kernel, (size_t)(2 * g.L - 1));
    if (rc == MLB_OK && d <= 2 && desc->conv_kernel) {
        const size_t nk = (d == 1) ? (size_t)(2 * g.L - 1) : (size_t)(2 * g.L - 1) * (2 * g.L - 1);
        // +2 doubles: TMA bulk copies round sizes up to 16 bytes
        std::vector<double> kc(nk + 2, 0.0);
        std::memcpy(kc.data(), desc->conv_kernel, nk * sizeof(double));
        rc = dev_upload(&p->conv, kc.data(), kc.size());
    }
    if (rc != MLB_OK) {
        dev_free(p->fused);
        dev_free(p->twid);
        dev_free(p->conv);
        dev_free(p->sep);
        delete p;
        return rc;
    }
    *out = p;
    return MLB_OK;
}

int mlb_plan_destroy(mlb_plan* p) {
    if (!p) return MLB_OK;
    DeviceGuard guard(p->device);
    dev_free(p->fused);
    dev_free(p->twid);
    dev_free(p->conv);
    dev_free(p->sep);
    delete p;
    return MLB_OK;
}

int mlb_binding_destroy(mlb_binding* b) {
    if (!b) return MLB_OK;
    // the binding's own copy of the device: a plan may be destroyed first
    // (finalizer order inside a collected reference cycle is arbitrary)
    DeviceGuard guard(b->device);
    dev_free(b->perm);
    dev_free(b->frac);
    dev_free(b->chunk_start);
    dev_free(b->chunk_cell);
    dev_free(b->chunk_gcell);
    dev_free(b->ggrp);
    dev_free(b->gslot);
    dev_free(b->seg_chunk);
    dev_free(b->sub_desc);
    dev_free(b->cblk);
    dev_free(b->wstream);
    dev_free(b->wstream_off);
    dev_free(b->citem);
    dev_free(b->citem_off);
    dev_free(b->brick_blk);
    dev_free(b->active_brick);
    dev_free(b->merge_off);
    dev_free(b->merge_pairs);
    dev_free(b->blocks);
    dev_free(b->seg_sub);
    dev_free(b->cta_seg);
    dev_free(b->key_start);
    dev_free(b->cta_row0);
    dev_free(b->row_cta);
    dev_free(b->seg_brick);
    dev_free(b->brick_seg);
    dev_free(b->brick_first);
    dev_free(b->work);
    dev_free(b->isd);
    dev_free(b->partial);
    dev_free(b->grid);
    dev_free(b->grid2);
    dev_free(b->stage_a);
    dev_free(b->stage_b);
    dev_free(b->lat_items);
    dev_free(b->lat_bin_off);
    dev_free(b->lat_blocks);
    delete b;
    return MLB_OK;
}

static int bind_impl(const mlb_plan* plan, const BindPointsIn& in, mlb_binding** out);

static int bind_guarded(const mlb_plan* plan, const BindPointsIn& in, mlb_binding** out) {
    // host-side allocation failures must not escape the C ABI
    try {
        return bind_impl(plan, in, out);
    } catch (const std::bad_alloc&) {
        return fail(MLB_ERR_CUDA, "mlb_bind: host allocation failed");
    } catch (const std::exception& e) {
        return fail(MLB_ERR_CUDA, std::string("mlb_bind: ") + e.what());
    } catch (...) {
        return fail(MLB_ERR_CUDA, "mlb_bind: unknown host exception");
    }
}

int mlb_bind(const mlb_plan* plan, const double* pts, int64_t n, double scale, const int32_t* node_ids,
             mlb_binding** out) {
    if (!plan) return fail(MLB_ERR_ARG, "null argument");
    BindPointsIn in{};
    in.points = pts;
    in.points_on_device = 0;
    in.n = n;
    in.ld = plan->g.d;
    in.scale = scale;
    in.node_ids = node_ids;
    return bind_guarded(plan, in, out);
}

int mlb_bind_ex(const mlb_plan* plan, const mlb_bind_desc* desc, mlb_binding** out) {
    if (!plan || !desc) return fail(MLB_ERR_ARG, "null argument");
    const int d = plan->g.d;
    if (desc->ld < d && !desc->cols) return fail(MLB_ERR_ARG, "row stride smaller than the dimension");
    if (desc->cols)
        for (int a = 0; a < d; ++a)
            if (desc->cols[a] < 0 || desc->cols[a] >= desc->ld) return fail(MLB_ERR_ARG, "column outside the row");
    if (desc->box_mid && !(desc->box_half > 0.0)) return fail(MLB_ERR_ARG, "box map needs half > 0");
    BindPointsIn in{};
    in.points = desc->points;
    in.points_on_device = desc->points_on_device;
    in.n = desc->n;
    in.ld = desc->ld;
    in.cols = desc->cols;
    in.scale = desc->scale;
    in.box_mid = desc->box_mid;
    in.box_half = desc->box_half;
    in.box_s = desc->box_s;
    in.box_hw = desc->box_hw;
    in.node_ids = desc->node_ids;
    in.stream = desc->stream;
    return bind_guarded(plan, in, out);
}

static int bind_impl(const mlb_plan* plan, const BindPointsIn& in, mlb_binding** out) {
    if (!plan || !out || (in.n > 0 && !in.points)) return fail(MLB_ERR_ARG, "null argument");
    const int64_t n = in.n;
    if (n < 0 || n >= (int64_t)1 << 31) return fail(MLB_ERR_ARG, "n out of range");
    const Geom& g = plan->g;
    const int d = g.d, Tb = g.Tb, nbr = g.nbr, TL = g.TL;
    const int nsm = plan->nsm;
    const int nloc = ipow_h(Tb, d);
    const int nbricks = ipow_h(nbr, d);
    DeviceGuard guard(plan->device);
    // 1-2. per point on the device (mlb_bind.cu): box map / box check, cell
    //      and fractional offsets exactly as _make_binding computes them
    //      (fastsum.py:343-353, :386), stable radix sort by (brick, cell)
    //      key, sorted SoA offsets; the host gets the per-key point counts
    BindPointsOut dev;
    struct Owned {  // device arrays not yet handed to the binding
        BindPointsOut* o;
        ~Owned() {
            if (o->perm) cudaFree(o->perm);
            if (o->frac) cudaFree(o->frac);
        }
    } owned{&dev};
    if (int rc = bind_points_device(in, g, &dev)) return rc;
    const int64_t nkeys = dev.nkeys;
    const std::vector<int64_t>& cnt = dev.cnt;
    // cell of a key: tile-local (TL^d) and sub-box (L^d) flat indices, the
    // digits of key = brick * nloc + local (axis 0 most significant)
    auto key_cells = [&](int64_t k, int32_t* tcell, int32_t* gcell) {
        int64_t brick = k / nloc, local = k % nloc;
        int bins[3], locs[3];
        for (int a = d - 1; a >= 0; --a) {
            locs[a] = (int)(local % Tb);
            bins[a] = (int)(brick % nbr) * Tb + locs[a];
            local /= Tb;
            brick /= nbr;
        }
        int32_t t = 0, gc = 0;
        for (int a = 0; a < d; ++a) {
            t = t * TL + locs[a];
            gc = gc * g.L + bins[a];
        }
        if (tcell) *tcell = t;
        if (gcell) *gcell = gc;
    };
    auto tcell_of = [&](int64_t k) { int32_t t; key_cells(k, &t, nullptr); return t; };
    auto gcell_of = [&](int64_t k) { int32_t gc; key_cells(k, nullptr, &gc); return gc; };
    // 3. chunks (<= kChunk points of one cell) and segments (<= maxseg chunks of one brick)
    std::vector<int32_t> chunk_start, chunk_cell, chunk_gcell, chunk_brick;
    for (int64_t k = 0; k < nkeys; ++k) {
        const int64_t lo = cnt[k], hi = cnt[k + 1];
        for (int64_t s = lo; s < hi; s += kChunk) {
            chunk_start.push_back((int32_t)s);
            chunk_cell.push_back(tcell_of(k));
            chunk_gcell.push_back(gcell_of(k));
            chunk_brick.push_back((int32_t)(k / nloc));
        }
    }
    const int nch = (int)chunk_cell.size();
    chunk_start.push_back((int32_t)n);
    // d = 3 gather groups: the points of one brick "pencil" (same brick and
    // axis-0/1 cell, <= Tb consecutive axis-2 cells) packed into 32 lanes.
    // Two-point groups pair points of the SAME cell in a lane (one staged
    // value read feeds both); a pencil's last group holding <= 32 points is a
    // one-point group.  Slot = sorted point | (axis-2 offset from the group's
    // first staged cell) << 29, -1 = empty.  Packing across the pencil's cells
    // fills the lanes that one-cell chunks leave idle on light cells.
    std::vector<int32_t> ggrp, gslot;
    // pack only where one-cell chunks leave lanes idle: lane fill of the
    // chunk path (64-point chunks; a tail of <= 32 points takes 32 lanes)
    bool packed = false;
    if (d == 3 && n > 0) {
        int64_t slots = 0;
        for (int64_t k = 0; k < nkeys; ++k) {
            const int64_t c = cnt[k + 1] - cnt[k], r = c % 64;
            slots += 64 * (c / 64) + (r == 0 ? 0 : (r <= 32 ? 32 : 64));
        }
        packed = (double)n / (double)slots < 0.9;
        if (const char* env = std::getenv("MLB_GATHER_PACKED")) packed = env[0] == '1';  // tuning
    }
    if (packed) {
        if (n >= ((int64_t)1 << 29)) return fail(MLB_ERR_CONFIG, "d = 3 bindings hold fewer than 2^29 points");
        struct Lane { int32_t a, b; int dc; int64_t k; };
        std::vector<Lane> lanes;
        int lo = 0, hi = 0;  // the pencil's occupied axis-2 range: one staging serves all its groups
        auto emit = [&](const std::vector<Lane>& ls, bool two) {
            // grid index of the first staged cell: any member's cell minus its offset
            const int32_t gb = gcell_of(ls[0].k) - (ls[0].dc - lo);
            ggrp.push_back(gb);
            ggrp.push_back((hi - lo + 1) | (two ? 256 : 0));
            const size_t base = gslot.size();
            gslot.resize(base + 64, -1);
            for (size_t i = 0; i < ls.size(); ++i) {
                gslot[base + i] = ls[i].a | ((ls[i].dc - lo) << 29);
                if (ls[i].b >= 0) gslot[base + 32 + i] = ls[i].b | ((ls[i].dc - lo) << 29);
            }
        };
        int64_t k = 0;
        while (k < nkeys) {
            const int64_t pen = k / Tb, kend = std::min<int64_t>(nkeys, (pen + 1) * Tb);
            lanes.clear();
            lo = 1 << 30;
            hi = -1;
            for (int64_t kk = k; kk < kend; ++kk) {
                const int dc = (int)(kk % Tb);
                if (cnt[kk + 1] > cnt[kk]) {
                    lo = std::min(lo, dc);
                    hi = std::max(hi, dc);
                }
                for (int64_t s = cnt[kk]; s < cnt[kk + 1]; s += 2)
                    lanes.push_back({(int32_t)s, s + 1 < cnt[kk + 1] ? (int32_t)(s + 1) : -1, dc, kk});
            }
            for (size_t g0 = 0; g0 < lanes.size(); g0 += 32) {
                const size_t g1 = std::min(lanes.size(), g0 + 32);
                std::vector<Lane> ls(lanes.begin() + g0, lanes.begin() + g1);
                int pts = 0;
                for (const Lane& l : ls) pts += 1 + (l.b >= 0);
                if (g1 == lanes.size() && pts <= 32) {  // tail: one point per lane
                    std::vector<Lane> one;
                    for (const Lane& l : ls) {
                        one.push_back({l.a, -1, l.dc, l.k});
                        if (l.b >= 0) one.push_back({l.b, -1, l.dc, l.k});
                    }
                    emit(one, false);
                } else {
                    emit(ls, true);
                }
            }
            k = kend;
        }
    }
    const int ngrp = (int)(ggrp.size() / 2);
    // segments (one warp's work unit): <= kSegPoints points of one brick,
    // never splitting a chunk; a bit smaller when n is small so every SM
    // gets work
    // (large n: grow segments so the partial tiles stay ~ nsm x 16 of them)
    // ~4 segments per spread warp (static round-robin): with about one per
    // warp, the few warps that get two set the kernel time (measured at
    // n = 1e7: d=1 spread 316 -> 212 us, config-4 d=2 spread 498 -> 461 us)
    int seg_points = (int)std::max<int64_t>(kSegPoints, n / (nsm * 64));
    while (seg_points > 64 && (n / seg_points) < nsm * 8) seg_points /= 2;
    if (const char* env = std::getenv("MLB_SEG_POINTS")) seg_points = std::max(32, std::atoi(env));  // tuning
    std::vector<int32_t> seg_chunk, seg_brick, brick_seg(nbricks + 1, 0);
    for (int c = 0; c < nch;) {
        const int br = chunk_brick[c];
        int e = c + 1;
        while (e < nch && chunk_brick[e] == br && chunk_start[e + 1] - chunk_start[c] <= seg_points) ++e;
        seg_chunk.push_back(c);
        seg_brick.push_back(br);
        brick_seg[br + 1]++;
        c = e;
    }
    const int nseg = (int)seg_brick.size();
    seg_chunk.push_back(nch);
    // sub-chunk descriptors (<= 32 points of one cell), in segment order
    std::vector<int32_t> sub_desc, seg_sub(nseg + 1, 0);
    for (int sg = 0; sg < nseg; ++sg) {
        seg_sub[sg] = (int)(sub_desc.size() / 2);
        for (int c = seg_chunk[sg]; c < seg_chunk[sg + 1]; ++c)
            for (int32_t p = chunk_start[c]; p < chunk_start[c + 1]; p += 32) {
                const int cnt = std::min<int32_t>(32, chunk_start[c + 1] - p);
                sub_desc.push_back(p);
                sub_desc.push_back((cnt << 24) | chunk_cell[c]);
            }
    }
    seg_sub[nseg] = (int)(sub_desc.size() / 2);
    for (int br = 0; br < nbricks; ++br) brick_seg[br + 1] += brick_seg[br];
    // d = 2 banded spread (large layers): CTA c takes the contiguous segment
    // range [cta_seg[c], cta_seg[c+1]); cells are sorted row-major, so its
    // points' stencils reach only the sub-box rows [row0, rmax + S) and its
    // warps' shared-memory tiles hold just that band (config 4: ~12 of 55
    // rows), which lets 12 instead of 6 warps run per SM.  The band sums
    // meet in launch_reduce (band_sum_kernel), in CTA order.
    std::vector<int32_t> cta_seg, cta_row0, row_cta;
    int ncta_band = 0, band_tile = 0;
    {
        bool banded = d == 2 && n >= (1 << 20);
        if (const char* env = std::getenv("MLB_D2_BANDED")) banded = d == 2 && env[0] == '1';  // tests / A/B
        if (banded && nseg > 0) {
            const int S = 2 * g.m + 1;
            const int nc = std::min(nsm * kBandCtasPerSm, std::max(1, nseg / kBandWarps));
            std::vector<int32_t> cs(nc + 1), r0(nc), r1(nc);
            int rows = 0;
            for (int c = 0; c <= nc; ++c) cs[c] = (int32_t)((int64_t)nseg * c / nc);
            for (int c = 0; c < nc; ++c) {
                int lo = 1 << 30, hi = -1;
                for (int ch = seg_chunk[cs[c]]; ch < seg_chunk[cs[c + 1]]; ++ch) {
                    lo = std::min(lo, chunk_cell[ch] / TL);
                    hi = std::max(hi, chunk_cell[ch] / TL);
                }
                r0[c] = lo;
                r1[c] = hi + S;   // one past the band's last row
                rows = std::max(rows, hi - lo + S);
            }
            if ((int64_t)rows * 2 <= TL) {   // only where the bands are much smaller than the sub-box
                ncta_band = nc;
                band_tile = rows * TL;
                cta_seg = cs;
                cta_row0 = r0;
                for (int c = 0; c < nc; ++c)
                    for (int j = seg_sub[cs[c]]; j < seg_sub[cs[c + 1]]; ++j) sub_desc[2 * j + 1] -= r0[c] * TL;
                // rows covered by CTA c: [r0[c], r1[c]); both bounds are non-decreasing in c
                row_cta.assign(2 * (size_t)g.L, 0);
                int first = 0, last = -1;
                for (int u = 0; u < g.L; ++u) {
                    while (first < nc && r1[first] <= u) ++first;
                    while (last + 1 < nc && r0[last + 1] <= u) ++last;
                    row_cta[2 * u] = first;
                    row_cta[2 * u + 1] = last;   // empty when last < first
                }
            }
            if (std::getenv("MLB_DEBUG"))
                fprintf(stderr, "[mlb] d2 bands: %d CTAs, band rows %d of %d (%s)\n", nc, rows, TL,
                        ncta_band ? "banded" : "full tiles");
        }
    }
    // d = 3: brick tile slot per brick (set with the cell blocks below), -1 if empty
    std::vector<int32_t> brick_first(nbricks, -1);
    // d = 3: cell blocks, CTA items and per-warp sub-chunk streams
    std::vector<int32_t> cblk, wstream, wstream_off, citem, citem_off, brick_blk, active_brick, merge_off, merge_pairs;
    int ncta_cells = 0;
    if (d == 3 && n > 0) {
        // points per block: >= 1024, and at large n about one CTA's share, so
        // a heavy cell splits into few parts (every part is a merge row set)
        int cap = (int)std::max<int64_t>(1024, ((n / (nsm * 2)) + 31) / 32 * 32);
        if (const char* env = std::getenv("MLB_CELL_CAP")) cap = std::max(32, std::atoi(env) / 32 * 32);  // tuning
        brick_blk.assign(nbricks + 1, 0);
        for (int64_t k = 0; k < nkeys; ++k) {
            const int64_t lo = cnt[k], hi = cnt[k + 1];
            if (hi == lo) continue;
            const int64_t np = hi - lo;
            const int64_t parts = (np + cap - 1) / cap;
            const int64_t per = ((np + parts - 1) / parts + 31) / 32 * 32;
            for (int64_t s0 = lo; s0 < hi; s0 += per) {
                cblk.push_back((int32_t)s0);
                cblk.push_back((int32_t)std::min<int64_t>(per, hi - s0));
                cblk.push_back(tcell_of(k));
                cblk.push_back((int32_t)(k / nloc));
                brick_blk[k / nloc + 1]++;
            }
        }
        for (int br = 0; br < nbricks; ++br) brick_blk[br + 1] += brick_blk[br];
        const int nb = (int)(cblk.size() / 4);
        // items: best-fit decreasing packing of blocks (w_b = min(8, sub-chunks) warps) into 8-warp CTAs
        std::vector<int> ord(nb), wb(nb), nsub(nb);
        int spw = 3;  // sub-chunks per warp before a block gets another warp (tuned on config 2)
        if (const char* env = std::getenv("MLB_WARP_SUBS")) spw = std::max(1, std::atoi(env));  // tuning
        for (int i = 0; i < nb; ++i) {
            ord[i] = i;
            nsub[i] = (cblk[4 * i + 1] + 31) / 32;
            wb[i] = std::min(kCellWarps, (nsub[i] + spw - 1) / spw);
        }
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return cblk[4 * x + 1] > cblk[4 * y + 1]; });
        struct Item { int used = 0, cost = 0; std::vector<int> blk; };
        std::vector<Item> items;
        std::vector<std::vector<int>> open(kCellWarps);  // open[r]: items with r free warps
        for (int i : ord) {
            const int w = wb[i];
            int it = -1;
            for (int r = w; r < kCellWarps && it < 0; ++r)
                while (!open[r].empty() && it < 0) {
                    const int c = open[r].back();
                    open[r].pop_back();
                    if (kCellWarps - items[c].used == r) it = c;  // stale entries are skipped
                }
            if (it < 0) {
                it = (int)items.size();
                items.emplace_back();
            }
            Item& I = items[it];
            I.blk.push_back(i);
            I.used += w;
            I.cost = std::max(I.cost, (nsub[i] + w - 1) / w);
            if (I.used < kCellWarps) open[kCellWarps - I.used].push_back(it);
        }
        std::vector<int> iord(items.size());
        for (size_t i = 0; i < items.size(); ++i) iord[i] = (int)i;
        std::stable_sort(iord.begin(), iord.end(), [&](int x, int y) { return items[x].cost > items[y].cost; });
        // item lists for as many CTAs as can be resident (m >= 5: one 8-warp
        // CTA per SM; m <= 4: two): one wave, so the LPT balance holds (two
        // waves of 148 at m = 5 cost config-4 rank shards at N = 8 +7 %)
        int cpsm = (g.m >= 5) ? 1 : 2;
        if (const char* env = std::getenv("MLB_CELL_CTAS")) cpsm = std::max(1, std::atoi(env));  // tuning
        ncta_cells = std::min<int>((int)items.size(), nsm * cpsm);
        // longest-processing-time-first: each item goes to the least loaded CTA
        std::vector<std::vector<int>> cta_items(ncta_cells);
        {
            using LC = std::pair<int64_t, int>;
            std::priority_queue<LC, std::vector<LC>, std::greater<LC>> pq;
            for (int c = 0; c < ncta_cells; ++c) pq.push({0, c});
            for (int k : iord) {
                LC t = pq.top();
                pq.pop();
                cta_items[t.second].push_back(k);
                pq.push({t.first + items[k].cost + 1, t.second});
            }
        }
        wstream_off.assign((size_t)ncta_cells * kCellWarps + 1, 0);
        citem_off.assign(ncta_cells + 1, 0);
        std::vector<std::vector<int32_t>> ws((size_t)ncta_cells * kCellWarps);
        for (int c = 0; c < ncta_cells; ++c) {
            citem_off[c] = (int)(citem.size() / kItemInts);
            for (int k : cta_items[c]) {
                const Item& I = items[k];
                std::vector<int32_t> row(kItemInts, 0);
                row[0] = (int)I.blk.size();
                int wlo = 0;
                for (size_t e = 0; e < I.blk.size(); ++e) {
                    const int bi = I.blk[e], w = wb[bi];
                    row[1 + 3 * e] = bi;
                    row[2 + 3 * e] = wlo;
                    row[3 + 3 * e] = w;
                    for (int r = 0; r < w; ++r) {
                        auto& st = ws[(size_t)c * kCellWarps + wlo + r];
                        for (int sc = r; sc < nsub[bi]; sc += w) {
                            const int32_t p0 = cblk[4 * bi] + 32 * sc;
                            const int32_t cntp = std::min(32, cblk[4 * bi + 1] - 32 * sc);
                            st.push_back(p0);
                            st.push_back(cntp << 24);
                        }
                    }
                    wlo += w;
                }
                for (int w = 0; w < kCellWarps; ++w) {  // end-of-item marker (an empty entry for idle warps)
                    auto& st = ws[(size_t)c * kCellWarps + w];
                    if (w >= wlo || st.empty() || (st.back() & 1)) {
                        st.push_back(0);
                        st.push_back(1);
                    } else {
                        st.back() |= 1;
                    }
                }
                citem.insert(citem.end(), row.begin(), row.end());
            }
        }
        citem_off[ncta_cells] = (int)(citem.size() / kItemInts);
        for (size_t i = 0; i < ws.size(); ++i) {
            wstream_off[i] = (int)(wstream.size() / 2);
            wstream.insert(wstream.end(), ws[i].begin(), ws[i].end());
        }
        wstream_off[ws.size()] = (int)(wstream.size() / 2);
        for (int br = 0; br < nbricks; ++br)
            if (brick_blk[br + 1] > brick_blk[br]) {
                brick_first[br] = (int)active_brick.size();
                active_brick.push_back(br);
            } else {
                brick_first[br] = -1;
            }
        // merge lists: for every (active brick, tile slab s0) the block rows
        // o0 = s0 - c0 that land in the slab, in block order
        const int S = 2 * g.m + 1;
        merge_off.assign(active_brick.size() * TL + 1, 0);
        for (size_t sl = 0; sl < active_brick.size(); ++sl) {
            const int br = active_brick[sl];
            for (int s0 = 0; s0 < TL; ++s0) {
                merge_off[sl * TL + s0] = (int)(merge_pairs.size() / 2);
                for (int bb = brick_blk[br]; bb < brick_blk[br + 1]; ++bb) {
                    const int tc = cblk[4 * bb + 2];
                    const int c2 = tc % TL, c1 = (tc / TL) % TL, c0 = tc / (TL * TL);
                    const int o0 = s0 - c0;
                    if (o0 < 0 || o0 >= S) continue;
                    merge_pairs.push_back(bb * S + o0);  // block row index: element offset (bb*S + o0) * S^2
                    merge_pairs.push_back((c1 << 8) | c2);
                }
            }
        }
        merge_off[active_brick.size() * TL] = (int)(merge_pairs.size() / 2);
        if (std::getenv("MLB_DEBUG")) {
            int mx = 0;
            for (size_t i = 0; i + 1 < merge_off.size(); ++i) mx = std::max(mx, merge_off[i + 1] - merge_off[i]);
            fprintf(stderr, "[mlb] d3 blocks %d items %zu ctas %d active bricks %zu merge rows %zu max/slab %d\n",
                    (int)(cblk.size() / 4), items.size(), ncta_cells, active_brick.size(), merge_pairs.size() / 2, mx);
        }
    }
    mlb_binding* b = new mlb_binding();
    b->plan = plan;
    b->device = plan->device;
    static std::atomic<uint64_t> next_uid{1};
    b->uid = next_uid++;
    b->n = n;
    b->nchunks = nch;
    b->ngrp = ngrp;
    b->gather_packed = packed ? 1 : 0;
    b->nseg = nseg;
    b->nbricks = nbricks;
    b->max_seg_chunks = seg_points;
    b->tile_cells = ipow_h(TL, d);
    b->nblk = (int)(cblk.size() / 4);
    b->ncta_cells = ncta_cells;
    b->nactive = (int)active_brick.size();
    if (const char* env = std::getenv("MLB_SPREAD_ATOMIC")) b->spread_atomic = (d == 3 && env[0] == '1');
    b->grid_cells = 1;
    for (int a = 0; a < d; ++a) b->grid_cells *= g.L;
    int64_t st = (int64_t)g.Kh;
    if (d == 2) st = std::max((int64_t)g.L * g.Kh, (int64_t)g.K * g.Kh);
    if (d == 3) {
        st = std::max((int64_t)g.L * g.L * g.Kh, (int64_t)g.L * g.K * g.Kh);
        st = std::max(st, (int64_t)g.K * g.K * g.Kh);
    }
    b->stage_elems = std::max<int64_t>(2 * st, b->grid_cells);  // >= one real grid (separable passes)
    int rc = MLB_OK;
    b->perm = dev.perm;  // the device binding's arrays move into the binding
    b->frac = dev.frac;
    dev.perm = nullptr;
    dev.frac = nullptr;
    if (rc == MLB_OK) rc = dev_upload(&b->chunk_start, chunk_start.data(), chunk_start.size());
    if (rc == MLB_OK) rc = dev_upload(&b->chunk_cell, chunk_cell.data(), chunk_cell.size());
    if (rc == MLB_OK) rc = dev_upload(&b->chunk_gcell, chunk_gcell.data(), chunk_gcell.size());
    if (rc == MLB_OK) rc = dev_upload(&b->seg_chunk, seg_chunk.data(), seg_chunk.size());
    if (rc == MLB_OK) rc = dev_upload(&b->sub_desc, sub_desc.data(), sub_desc.size());
    if (rc == MLB_OK) rc = dev_upload(&b->seg_sub, seg_sub.data(), seg_sub.size());
    if (rc == MLB_OK) rc = dev_upload(&b->seg_brick, seg_brick.data(), seg_brick.size());
    if (rc == MLB_OK) rc = dev_upload(&b->brick_seg, brick_seg.data(), brick_seg.size());
    if (rc == MLB_OK) rc = dev_upload(&b->brick_first, brick_first.data(), brick_first.size());
    if (d == 3 && n > 0) {
        if (rc == MLB_OK) rc = dev_upload(&b->cblk, cblk.data(), cblk.size());
        if (rc == MLB_OK) rc = dev_upload(&b->wstream, wstream.data(), wstream.size());
        if (rc == MLB_OK) rc = dev_upload(&b->wstream_off, wstream_off.data(), wstream_off.size());
        if (rc == MLB_OK) rc = dev_upload(&b->citem, citem.data(), citem.size());
        if (rc == MLB_OK) rc = dev_upload(&b->citem_off, citem_off.data(), citem_off.size());
        if (rc == MLB_OK) rc = dev_upload(&b->brick_blk, brick_blk.data(), brick_blk.size());
        if (rc == MLB_OK) rc = dev_upload(&b->active_brick, active_brick.data(), active_brick.size());
        if (rc == MLB_OK) rc = dev_upload(&b->merge_off, merge_off.data(), merge_off.size());
        if (rc == MLB_OK) rc = dev_upload(&b->merge_pairs, merge_pairs.data(), std::max<size_t>(2, merge_pairs.size()));
        if (packed && rc == MLB_OK) rc = dev_upload(&b->ggrp, ggrp.data(), ggrp.size());
        if (packed && rc == MLB_OK) rc = dev_upload(&b->gslot, gslot.data(), gslot.size());
        const int S = 2 * g.m + 1;
        if (rc == MLB_OK) rc = dev_upload<double>(&b->blocks, nullptr, (size_t)b->nblk * S * S * S);
    }
    const char* s1 = std::getenv("MLB_D1_STREAM");   // A/B: 0 = the sub-chunk kernels
    if (d == 1 && n > 0 && !(s1 && s1[0] == '0')) {   // per-cell starts for the streaming d = 1 kernels
        std::vector<int32_t> ks(cnt.begin(), cnt.end());
        b->nkeys = (int)nkeys;
        if (rc == MLB_OK) rc = dev_upload(&b->key_start, ks.data(), ks.size());
    }
    if (ncta_band > 0) {
        b->ncta_band = ncta_band;
        b->band_tile = band_tile;
        if (rc == MLB_OK) rc = dev_upload(&b->cta_seg, cta_seg.data(), cta_seg.size());
        if (rc == MLB_OK) rc = dev_upload(&b->cta_row0, cta_row0.data(), cta_row0.size());
        if (rc == MLB_OK) rc = dev_upload(&b->row_cta, row_cta.data(), row_cta.size());
    }
    if (rc == MLB_OK) rc = dev_upload<int>(&b->work, nullptr, 1);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->isd, nullptr, (size_t)n);
    // d <= 2: one partial grid per spread CTA (<= 2 per SM); d = 3: one per segment
    b->spread_parts_max = nsm * 2;
    const size_t nparts = (d <= 2) ? (size_t)std::max(nseg, b->spread_parts_max) : (size_t)std::max(1, b->nactive);  // d = 3: brick tiles
    const size_t partial_elems = std::max(nparts * (size_t)b->tile_cells, (size_t)ncta_band * band_tile);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->partial, nullptr, partial_elems);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->grid, nullptr, (size_t)b->grid_cells + 2);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->grid2, nullptr, (size_t)b->grid_cells + 2);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->stage_a, nullptr, (size_t)b->stage_elems);
    if (rc == MLB_OK) rc = dev_upload<double>(&b->stage_b, nullptr, (size_t)b->stage_elems);
    if (rc == MLB_OK && d == 2 && n > 0) {   // lattice items (image layers): MLB_LATTICE=0 off, 1 forced
        int mode = -1;
        if (const char* env = std::getenv("MLB_LATTICE")) mode = env[0] == '1' ? 1 : (env[0] == '0' ? 0 : -1);
        std::vector<int32_t> key_gcell((size_t)nkeys);
        for (int64_t k = 0; k < nkeys; ++k) key_gcell[k] = gcell_of(k);
        rc = build_lattice(b, cnt, key_gcell, mode, (cudaStream_t)in.stream);
    }
    if (rc != MLB_OK) {
        std::string msg = g_err;
        mlb_binding_destroy(b);
        return fail(rc, msg);
    }
    *out = b;
    return MLB_OK;
}

int64_t mlb_binding_n(const mlb_binding* b) { return b ? b->n : -1; }

int mlb_binding_perm(const mlb_binding* b, int32_t* perm_host) {
    if (!b || !perm_host) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(b->plan->device);
    if (b->n) MLB_CUDA_TRY(cudaMemcpy(perm_host, b->perm, b->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    return MLB_OK;
}

int mlb_binding_stats(const mlb_binding* b, int64_t* o) {
    if (!b || !o) return fail(MLB_ERR_ARG, "null argument");
    o[0] = b->n;
    o[1] = b->nchunks;
    o[2] = b->nseg;
    o[3] = b->nbricks;
    o[4] = b->tile_cells;
    o[5] = b->grid_cells;
    o[6] = b->ncta_band;
    o[7] = b->band_tile;
    return MLB_OK;
}

int mlb_binding_lattice(const mlb_binding* b, int64_t* out2) {
    if (!b || !out2) return fail(MLB_ERR_ARG, "null argument");
    out2[0] = b->lat_nitems;
    out2[1] = b->lat_points;
    return MLB_OK;
}

int mlb_grid_cells(const mlb_binding* b, int64_t* cells, int* L, int* ulo) {
    if (!b) return fail(MLB_ERR_ARG, "null argument");
    if (cells) *cells = b->grid_cells;
    if (L) *L = b->plan->g.L;
    if (ulo) *ulo = b->plan->g.ulo;
    return MLB_OK;
}

}  // extern "C"

// ------------------------------------------------------------ permutations --
namespace mlb {
__global__ void gather_perm_kernel(const int32_t* __restrict__ perm, const double* __restrict__ src,
                                   double* __restrict__ dst, int64_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        dst[j] = src[perm[j]];
}
__global__ void scatter_perm_kernel(const int32_t* __restrict__ perm, const double* __restrict__ src,
                                    double* __restrict__ dst, int64_t n, int acc) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = perm[j];
        dst[i] = acc ? dst[i] + src[j] : src[j];
    }
}
static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > device_sms() * 16) b = device_sms() * 16;
    return (int)(b < 1 ? 1 : b);
}
}  // namespace mlb

extern "C" {

int mlb_binding_set_isd(mlb_binding* b, const double* isd_dev, void* stream) {
    if (!b || (!isd_dev && b->n)) return fail(MLB_ERR_ARG, "null argument");
    if (!b->n) return MLB_OK;
    DeviceGuard guard(b->plan->device);
    gather_perm_kernel<<<grid_for(b->n), 256, 0, (cudaStream_t)stream>>>(b->perm, isd_dev, b->isd, b->n);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_to_sorted(const mlb_binding* b, const double* v, double* vs, void* stream) {
    if (!b) return fail(MLB_ERR_ARG, "null argument");
    if (!b->n) return MLB_OK;
    DeviceGuard guard(b->plan->device);
    gather_perm_kernel<<<grid_for(b->n), 256, 0, (cudaStream_t)stream>>>(b->perm, v, vs, b->n);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_to_node(const mlb_binding* b, const double* vs, double* v, int accumulate, void* stream) {
    if (!b) return fail(MLB_ERR_ARG, "null argument");
    if (!b->n) return MLB_OK;
    DeviceGuard guard(b->plan->device);
    scatter_perm_kernel<<<grid_for(b->n), 256, 0, (cudaStream_t)stream>>>(b->perm, vs, v, b->n, accumulate);
    note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

int mlb_spread(mlb_binding* b, const double* v, double* grid, unsigned flags, void* stream) {
    if (!b || !grid) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(b->plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    b->atomic_target = grid;
    int rc = launch_spread(b, v, flags & ~MLB_SPREAD_ONLY, st);
    if (rc != MLB_OK) return rc;
    if (flags & MLB_SPREAD_ONLY || b->spread_atomic) return MLB_OK;
    if (b->nseg == 0) {
        MLB_CUDA_TRY(cudaMemsetAsync(grid, 0, b->grid_cells * sizeof(double), st));
        return MLB_OK;
    }
    return launch_reduce(b, grid, st);
}

int mlb_spread_peers(mlb_binding* b, const double* v, double* const* peer_slots, int world, unsigned flags,
                     void* stream) {
    if (!b || !peer_slots) return fail(MLB_ERR_ARG, "null argument");
    if (world < 1 || world > kMaxPeers) return fail(MLB_ERR_ARG, "world size outside [1, 8]");
    DeviceGuard guard(b->plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    PeerOut po{};
    po.n = world;
    for (int q = 0; q < world; ++q) {
        if (!peer_slots[q]) return fail(MLB_ERR_ARG, "null peer slot");
        po.p[q] = peer_slots[q];
    }
    if (b->nseg == 0) {
        for (int q = 0; q < world; ++q)
            MLB_CUDA_TRY(cudaMemsetAsync(po.p[q], 0, b->grid_cells * sizeof(double), st));
        return MLB_OK;
    }
    b->atomic_target = nullptr;   // (the peer exchange always takes the deterministic blocks)
    int rc = launch_spread(b, v, flags & ~MLB_SPREAD_ONLY, st);
    if (rc != MLB_OK) return rc;
    return launch_reduce(b, nullptr, st, &po);
}

int mlb_grid_sum_slots(const double* recv, int world, int64_t cells, double* grid, void* stream) {
    if (!recv || !grid) return fail(MLB_ERR_ARG, "null argument");
    if (world < 1) return fail(MLB_ERR_ARG, "world size must be >= 1");
    return launch_slot_sum(recv, world, cells, grid, (cudaStream_t)stream);
}

int mlb_ipc_handle(const void* dev_ptr, unsigned char* handle64) {
    if (!dev_ptr || !handle64) return fail(MLB_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    MLB_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, 64);
    return MLB_OK;
}

int mlb_ipc_open(const unsigned char* handle64, int device, void** dev_ptr) {
    if (!handle64 || !dev_ptr) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    MLB_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MLB_OK;
}

int mlb_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return MLB_OK;
    MLB_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return MLB_OK;
}

int mlb_reduce(mlb_binding* b, double* grid, void* stream) {
    if (!b || !grid) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(b->plan->device);
    if (b->spread_atomic) return MLB_OK;   // the atomic spread wrote the grid itself
    if (b->nseg == 0) {
        MLB_CUDA_TRY(cudaMemsetAsync(grid, 0, b->grid_cells * sizeof(double), (cudaStream_t)stream));
        return MLB_OK;
    }
    return launch_reduce(b, grid, (cudaStream_t)stream);
}

int mlb_convolve(mlb_binding* b, const double* gin, double* gout, void* stream) {
    if (!b || !gin || !gout) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(b->plan->device);
    return launch_convolve(b, gin, gout, (cudaStream_t)stream);
}

int mlb_gather(mlb_binding* b, const double* grid, double* y, unsigned flags, void* stream) {
    if (!b || !grid || !y) return fail(MLB_ERR_ARG, "null argument");
    DeviceGuard guard(b->plan->device);
    return launch_gather(b, grid, nullptr, y, 0.0, 1.0, 0.0, flags & (MLB_SORTED | MLB_ACCUMULATE | 0x70000u),
                         (cudaStream_t)stream);
}

int mlb_gather_apply(mlb_binding* b, const double* grid, const double* v, double* y, double alpha, double beta,
                     double gamma, unsigned flags, void* stream) {
    if (!b || (b->n && (!grid || !v || !y))) return fail(MLB_ERR_ARG, "null argument");
    if (!b->n) return MLB_OK;
    DeviceGuard guard(b->plan->device);
    flags &= (MLB_USE_ISD | MLB_ACCUMULATE | MLB_SORTED);
    return launch_gather(b, grid, v, y, alpha, beta, gamma, flags, (cudaStream_t)stream);
}

int mlb_apply(mlb_binding* b, const double* v, double* y, double alpha, double beta, double gamma, unsigned flags,
              void* stream) {
    if (!b || (b->n && (!v || !y))) return fail(MLB_ERR_ARG, "null argument");
    if (!b->n) return MLB_OK;
    DeviceGuard guard(b->plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    flags &= (MLB_USE_ISD | MLB_ACCUMULATE | MLB_SORTED);  // the public bits only
    b->atomic_target = b->grid;
    int rc = launch_spread(b, v, flags, st);
    if (rc == MLB_OK && !b->spread_atomic) rc = launch_reduce(b, b->grid, st);
    if (rc == MLB_OK) rc = launch_convolve(b, b->grid, b->grid2, st);
    if (rc == MLB_OK) rc = launch_gather(b, b->grid2, v, y, alpha, beta, gamma, flags, st);
    return rc;
}

int mlb_apply_multi(mlb_binding* const* b, int T, const double* const* v_dev, double* const* y_dev,
                    const double* abg_dev, unsigned flags, void* stream) {
    if (T < 1 || !b || !v_dev || !y_dev || !abg_dev) return fail(MLB_ERR_ARG, "null argument");
    for (int t = 0; t < T; ++t)
        if (!b[t]) return fail(MLB_ERR_ARG, "null binding");
    DeviceGuard guard(b[0]->plan->device);
    flags &= (MLB_USE_ISD | MLB_ACCUMULATE | MLB_SORTED);
    return launch_apply_multi(b, T, v_dev, y_dev, abg_dev, flags, (cudaStream_t)stream);
}

int mlb_apply_batched(mlb_binding* const* b, int T, const double* v, double* const* y, const double* alpha,
                      const double* beta, const double* gamma, unsigned flags, void* stream) {
    if (T < 0 || (T > 0 && (!b || !y || !alpha || !beta || !gamma))) return fail(MLB_ERR_ARG, "null argument");
    if (T == 0) return MLB_OK;
    if (T == 1) return mlb_apply(b[0], v, y[0], alpha[0], beta[0], gamma[0], flags, stream);
    for (int t = 0; t < T; ++t)
        if (!b[t] || b[t]->plan->device != b[0]->plan->device)
            return fail(MLB_ERR_ARG, "batched layers must be bound on one device");
    DeviceGuard guard(b[0]->plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    // the layers are independent: each runs on its own stream (forked from
    // and joined back into the caller's stream), so the cheap layers fill
    // the SMs the costly one leaves idle in its low-occupancy phases
    // streams and events belong to a device: one pool per (thread, device)
    struct Pool {
        std::vector<cudaStream_t> streams;
        std::vector<cudaEvent_t> evs;
    };
    static thread_local std::map<int, Pool> pools;
    Pool& P = pools[b[0]->plan->device];
    while ((int)P.streams.size() < T) {
        cudaStream_t s;
        MLB_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        P.streams.push_back(s);
    }
    while ((int)P.evs.size() < T + 1) {
        cudaEvent_t e;
        MLB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P.evs.push_back(e);
    }
    MLB_CUDA_TRY(cudaEventRecord(P.evs[T], st));
    int rc = MLB_OK;
    int forked = 0;  // streams that waited on the fork event: each must be joined back
    for (int t = 0; t < T && rc == MLB_OK; ++t) {
        cudaError_t e = cudaStreamWaitEvent(P.streams[t], P.evs[T], 0);
        if (e != cudaSuccess) {
            rc = fail(MLB_ERR_CUDA, std::string("cudaStreamWaitEvent: ") + cudaGetErrorString(e));
            break;
        }
        ++forked;
        rc = mlb_apply(b[t], v, y[t], alpha[t], beta[t], gamma[t], flags, P.streams[t]);
    }
    // always join every forked stream into the caller's stream (also on the
    // error path: an unjoined fork would break a surrounding graph capture)
    for (int t = 0; t < forked; ++t) {
        cudaError_t e = cudaEventRecord(P.evs[t], P.streams[t]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, P.evs[t], 0);
        if (e != cudaSuccess && rc == MLB_OK)
            rc = fail(MLB_ERR_CUDA, std::string("stream join: ") + cudaGetErrorString(e));
    }
    return rc;
}

}  // extern "C"

// ------------------------------------------------------------ FP64 probe --
namespace mlb {
__global__ void dfma_probe_kernel(int64_t iters, double* out) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double b = 0.999999999, c = 1e-12;
    for (int64_t i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void dmma_probe_kernel(int64_t iters, double* out) {
    // 4 independent m8n8k4 fp64 MMA chains per warp
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
    for (int64_t i = 0; i < iters; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
    }
    const double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
    if (s == 12345.678) out[0] = s;
}
}  // namespace mlb

extern "C" int mlb_probe_dmma(int64_t iters, int blocks, double* out_dev, void* stream) {
    mlb::dmma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, out_dev);
    mlb::note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}

extern "C" int mlb_probe_fp64(int64_t iters, int blocks, double* out_dev, void* stream) {
    mlb::dfma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, out_dev);
    mlb::note_launches(1);
    MLB_CUDA_TRY(cudaGetLastError());
    return MLB_OK;
}
