/*
 * multilap_b200.h -- C ABI of libmlb.so, the B200 (sm_100a) NFFT
 * normalized-Laplacian matvec path of arXiv 2007.05239 ("multilap").
 *
 * The reference (/root/reference/pkg/src/multilap, pure Python) has no FFI;
 * its seam is Python duck typing.  Every entry point
 * below replaces one reference function, cited as file:line; the Python
 * package paper_2007_05239_b200 binds them with ctypes (INTEGRATION.md shows
 * the binding a maintainer of the reference would add).
 *
 * Conventions
 *   - Return 0 (MLB_OK) on success, otherwise an MLB_ERR_* code; the message
 *     is in mlb_last_error() (thread-local).  MLB_ERR_CONFIG maps to the
 *     reference's ConfigError, MLB_ERR_NUMERICAL to NumericalError.
 *   - All vectors are fp64.  "dev" pointers are CUDA device pointers, "host"
 *     pointers are CPU memory.  Inputs are never written.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Handles own their device buffers until *_destroy.  A binding may be
 *     used from one stream at a time; plans are read-only and shareable.
 *   - No torch types: plain pointers, sizes and C structs only.
 */
#ifndef MULTILAP_B200_H
#define MULTILAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLB_ABI_VERSION 1

#define MLB_OK 0
#define MLB_ERR_CONFIG 1      /* reference ConfigError    (errors.py:11-12) */
#define MLB_ERR_NUMERICAL 2   /* reference NumericalError (errors.py:19-21) */
#define MLB_ERR_CUDA 3        /* CUDA runtime failure */
#define MLB_ERR_ARG 4         /* NULL handle / bad size */

/* flags for mlb_apply */
#define MLB_USE_ISD 1u        /* s = D^-1/2 (set by mlb_binding_set_isd), else s = 1 */
#define MLB_ACCUMULATE 2u     /* y += result instead of y = result */
#define MLB_SORTED 4u         /* v and y are in the binding's sorted (cell) order */
#define MLB_SPREAD_ONLY 8u    /* mlb_spread: run the spread kernel only (partials, no reduction) */
/* bits 16-19 of the mlb_spread / mlb_gather stage hooks switch parts of those
   kernels off for profiling ablations (tools/ablate_spread.py); mlb_apply
   ignores every bit but MLB_USE_ISD | MLB_ACCUMULATE | MLB_SORTED */

typedef struct mlb_plan mlb_plan;
typedef struct mlb_binding mlb_binding;

/* Plan description: the host computes the plan math (fastsum.py:256-313)
 * and passes the device-facing tables.  Layouts:
 *   fused_band : (K,)*(d-1) x Kh real, K = N+1 (k = -N/2..N/2), Kh = N/2+1
 *                (k = 0..N/2 on the last axis); the reference's
 *                fused_weights / ng^d restricted to the band |k| <= N/2.
 *   twiddle    : L x K complex (re,im interleaved): exp(-2 pi i k u / ng)
 *                for the active cells u = u_lo..u_lo+L-1, k = -N/2..N/2.
 *   win_coef   : (2m+1) x (win_deg+1): monomial coefficients in s = 2f-1 of
 *                phi(f - o), o = -m..m, f in [0,1) (the Kaiser-Bessel window
 *                of fastsum.py:158-167 as an exact-to-1e-14 polynomial).
 *   conv_kernel: d <= 2 only (NULL for d = 3): (2L-1)^d real spatial kernel
 *                Kc[D] = sum_{|k|<=N/2} F(k) cos(2 pi k.D / ng), D = -(L-1)..L-1,
 *                so the convolution stage is a direct sub-box convolution.
 *   sep_kernel : nullable, 2L-1 reals: when the band weights are a rank-1
 *                tensor F(k) = prod_a f(k_a) (checked on the host to 1e-13),
 *                c[D] = sum_k f(k) cos(2 pi k D / ng) and the convolution runs
 *                as d one-dimensional passes. */
typedef struct mlb_plan_desc {
    int d, N, m, ng;
    int bin_lo, bin_hi;       /* admissible floor(ng*x) range per axis */
    int win_deg;
    double K0;                /* kernel value at 0 (kernels.py:38-39) */
    const double* fused_band; /* host */
    const double* twiddle;    /* host */
    const double* win_coef;   /* host */
    const double* conv_kernel;/* host, d <= 2 (nullable for d = 3) */
    const double* sep_kernel; /* host, nullable: separable 1-D kernel */
} mlb_plan_desc;

int mlb_abi_version(void);
const char* mlb_last_error(void);
int mlb_device_count(void);
/* number of kernels libmlb has launched in this process (bench evidence) */
int64_t mlb_launch_count(void);
/* add k launches to that count: kernels replayed from a captured CUDA graph
   (the graph's launches were counted once, at capture) */
void mlb_note_launches(int64_t k);
/* FP64 FMA throughput probe: `blocks` x 256 threads x iters x 8 DFMA (roofline
 * denominator; MEASURED_PEAKS.json carries no FP64 figure) */
int mlb_probe_fp64(int64_t iters, int blocks, double* out_dev, void* stream);
/* FP64 tensor-core probe: blocks x 8 warps x iters x 4 DMMA.8x8x4 (m8n8k4 f64) */
int mlb_probe_dmma(int64_t iters, int blocks, double* out_dev, void* stream);

/* build_plan (fastsum.py:256-313): upload plan tables to `device`. */
int mlb_plan_create(const mlb_plan_desc* desc, int device, mlb_plan** out);
int mlb_plan_destroy(mlb_plan* plan);

/* bind_points / _make_binding (fastsum.py:333-386): bin the n points
 * (row-major n x d box coordinates, host memory) by cell floor(ng*x*scale)
 * with `scale` = 1/sqrt(d) (1 for the bare torus transforms), counting-sort
 * them by (brick, cell), build the chunk/segment tables and upload.  The box
 * check is the caller's (validate_box, fastsum.py:66-80).  `node_ids_host`
 * (nullable) maps point i to its node index in the vectors passed to
 * mlb_apply -- one binding per component block (graphs.py:99-129). */
int mlb_bind(const mlb_plan* plan, const double* points_host, int64_t n, double scale,
             const int32_t* node_ids_host, mlb_binding** out);
/* The same binding from a row-major point / feature matrix on the host OR the
 * device, with the box map of feature_group folded in (datapipe.py:100-123:
 * x_box = clip((x - mid) / half, -1, 1) * box_s per column, then the torus
 * scale) and validate_box (fastsum.py:66-80) done on the device.  Every
 * per-point step (map, check, cells, stable sort, sorted offsets) runs on
 * the GPU; the host builds the cell-level work tables from per-cell counts. */
typedef struct mlb_bind_desc {
    const double* points;     /* n rows of ld doubles */
    int points_on_device;     /* 1: device pointer, 0: host pointer */
    int64_t n;
    int ld;                   /* row stride in doubles */
    const int* cols;          /* nullable, host: the d columns of a row (default 0..d-1) */
    double scale;             /* 1/sqrt(d) for the fastsum box, 1 for the bare torus transforms */
    const double* box_mid;    /* nullable, host, d values: raw features -> box (mode "fastsum-box") */
    double box_half, box_s;   /* half-range and box half-width of that map */
    double box_hw;            /* > 0: reject |x_box|_inf > box_hw + 1e-12 (ConfigError, validate_box) */
    const int32_t* node_ids;  /* nullable, host: point -> node index (component blocks) */
    void* stream;             /* the bind's stream (it synchronises it) */
} mlb_bind_desc;
int mlb_bind_ex(const mlb_plan* plan, const mlb_bind_desc* desc, mlb_binding** out);
int mlb_binding_destroy(mlb_binding* b);
int64_t mlb_binding_n(const mlb_binding* b);
/* sorted position -> original node index (int32, host out, n entries) */
int mlb_binding_perm(const mlb_binding* b, int32_t* perm_host);
/* binding statistics: [n, nchunks, nsegments, nbricks, tile_cells, grid_cells,
   band_ctas (d = 2 banded spread CTAs, 0 = full tiles), band_tile_cells] */
int mlb_binding_stats(const mlb_binding* b, int64_t* out8);
/* d = 2 lattice items (image layers: the points of a cell form an R x C
   product set; spread / gather as two small contractions per cell, see
   DESIGN.md 3.3b): [items (0 = the general kernels), points in lattice cells].
   Bind-time env MLB_LATTICE=0 / 1 turns the mode off / on regardless of size. */
int mlb_binding_lattice(const mlb_binding* b, int64_t* out2);

/* Store D^-1/2 (graphs.py:159-165) for the fused Laplacian; node order, device. */
int mlb_binding_set_isd(mlb_binding* b, const double* isd_dev, void* stream);

/* The hot path.  With s = isd (MLB_USE_ISD) or 1 and acc = W~(s.v) -- the
 * spread / rFFT * fused / irFFT / gather chain of fastsum_apply
 * (fastsum.py:475-497) without the diagonal removal:
 *     y (=|+=) alpha*v + s.(beta*acc + gamma*s.v)
 *   W v              (fastsum_apply, fastsum.py:475-497):   1, 0, alpha=-K0, beta=1, gamma=0
 *   L_sym+delta v    (apply_sym_laplacian, graphs.py:197-201): USE_ISD, 1+delta, -1, K0
 *   D^-1/2 W D^-1/2 v (apply_one_minus_L1 term, powermean.py:75-76): USE_ISD, 0, 1, -K0
 * v, y: device, node order (or sorted order with MLB_SORTED). */
int mlb_apply(mlb_binding* b, const double* v_dev, double* y_dev, double alpha, double beta,
              double gamma, unsigned flags, void* stream);

/* T independent layers applied to one vector (SURVEY 8(b)'s proposed
 * mlb_apply_lsym_batched; apply_sym_laplacians for C hosts): y[t] = layer
 * t's mlb_apply of v with coefficients alpha[t], beta[t], gamma[t] (host
 * arrays).  The layers run concurrently on library-owned streams forked
 * from and joined back into `stream`; all bindings on one device. */
/* The fused Laplacian of T layers with one launch per stage (blockIdx.y =
 * layer) -- for many small layers of one (d, m), e.g. config 3's 52, whose
 * per-layer launches are latency-bound (graphs.py:197-201 per layer).
 * b: HOST array of T bindings (d = 2, same m <= 5, same grid and windows,
 * < 2^20 points each, separable convolution); v_dev / y_dev: DEVICE arrays
 * of T device pointers; abg_dev: DEVICE array alpha[T] | beta[T] | gamma[T].
 * y_t (=|+=) alpha_t v_t + s_t (beta_t W~ (s_t v_t) + gamma_t s_t v_t) as
 * mlb_apply.  MLB_ERR_CONFIG when the layers are not eligible (the caller
 * falls back to mlb_apply per layer). */
int mlb_apply_multi(mlb_binding* const* b, int T, const double* const* v_dev, double* const* y_dev,
                    const double* abg_dev, unsigned flags, void* stream);
int mlb_apply_batched(mlb_binding* const* b, int T, const double* v_dev, double* const* y_dev, const double* alpha,
                      const double* beta, const double* gamma, unsigned flags, void* stream);

/* Test hooks on the three stages (sub-box grid of L^d cells, row-major):
 * spread (fastsum.py:389-391), convolution rfftn*fused*irfftn
 * (fastsum.py:492-495), gather (fastsum.py:400-406). */
int mlb_grid_cells(const mlb_binding* b, int64_t* cells, int* L, int* u_lo);
int mlb_spread(mlb_binding* b, const double* v_dev, double* grid_dev, unsigned flags, void* stream);
/* the deterministic partial-tile reduction of the last spread into grid_dev */
int mlb_reduce(mlb_binding* b, double* grid_dev, void* stream);

/* Node-range sharding (the per-matvec sum of the ranks'
 * sub-box grids; replaces the all-reduce of dist.py's NCCL path): spread
 * this rank's points and let the final reduction kernel store the grid
 * straight into every rank's receive buffer -- peer_slots[q] = this rank's
 * slot (rank * cells) in rank q's buffer, device pointers (own buffer or
 * CUDA-IPC-mapped peer memory over NVLink), world <= 8.  After a barrier
 * every rank sums its buffer's slots in rank order (mlb_grid_sum_slots):
 * bitwise the same grid on all ranks. */
int mlb_spread_peers(mlb_binding* b, const double* v_dev, double* const* peer_slots, int world, unsigned flags,
                     void* stream);
int mlb_grid_sum_slots(const double* recv_dev, int world, int64_t cells, double* grid_dev, void* stream);
/* CUDA IPC of device buffers (64-byte handles) for the peer slots above */
int mlb_ipc_handle(const void* dev_ptr, unsigned char* handle64);
int mlb_ipc_open(const unsigned char* handle64, int device, void** dev_ptr);
int mlb_ipc_close(void* dev_ptr);
int mlb_convolve(mlb_binding* b, const double* grid_in_dev, double* grid_out_dev, void* stream);
int mlb_gather(mlb_binding* b, const double* grid_dev, double* y_dev, unsigned flags, void* stream);

/* Node-range sharding, NCCL path: the gather of mlb_gather with
 * mlb_apply's fused epilogue, from a grid the caller summed over the ranks
 * (mlb_spread -> all-reduce of the sub-box grid -> mlb_convolve -> this):
 *     y (=|+=) alpha*v + s.(beta*gather(grid) + gamma*s.v)
 * v, y: this binding's points (node order, or sorted with MLB_SORTED). */
int mlb_gather_apply(mlb_binding* b, const double* grid_dev, const double* v_dev, double* y_dev, double alpha,
                     double beta, double gamma, unsigned flags, void* stream);

/* Complex band DFT between the active sub-box (L^d complex cells) and the full
 * band (K^d complex, k = -N/2..N/2 per axis): forward sum_u in[u] e^{-2 pi i k.u/ng},
 * inverse sum_k in[k] e^{+2 pi i k.u/ng} (unnormalised).  Building block of the
 * bare transforms nfft_adjoint / nfft_forward (fastsum.py:418-468). */
int mlb_band_dft(mlb_binding* b, const double* in_dev, double* out_dev, int inverse, void* stream);

/* Permutations between node order and the binding's sorted order. */
int mlb_to_sorted(const mlb_binding* b, const double* v_node_dev, double* v_sorted_dev, void* stream);
int mlb_to_node(const mlb_binding* b, const double* v_sorted_dev, double* v_node_dev, int accumulate,
                void* stream);

/* ---- Krylov kernels (krylov.py:65-71, :172-216) -------------------------
 * V is column-major n x ldcols (column j at V + j*ld).  Deterministic
 * fixed-order reductions; `work` is device scratch of mlb_krylov_work_size. */
int64_t mlb_krylov_work_size(int64_t n, int maxcols);
/* h[0..cols) = V[:, :cols]^T w (device out) */
int mlb_gemv_t(const double* V, int64_t ld, int64_t n, int cols, const double* w, double* h,
               double* work, void* stream);
/* two-pass classical Gram-Schmidt of w against V[:, :cols] (krylov.py:65-71):
 * h_out = h1+h2 (device, cols), h1_out = first-pass projections (device,
 * cols, nullable; h1[cols-1] is the Lanczos alpha of krylov.py:198),
 * nrm2_out = ||w||^2 after (device, 1, nullable) */
int mlb_cgs2(const double* V, int64_t ld, int64_t n, int cols, double* w, double* h_out,
             double* h1_out, double* nrm2_out, double* work, void* stream);
/* CGS2 of T Lanczos chains in one launch per phase (the lockstep PKSM of many
 * layers): chain t has basis V[t] (same ld, n, cols for all), w[t] is
 * orthogonalised in place; h_out[t] = h1 + h2, h1_out[t] = first-pass
 * projections, nrm2_out[t][0] = ||w||^2 after; with vnext (nullable) also
 * V[t] column `cols` = w / sqrt(||w||^2).  Pointer arrays are DEVICE arrays of
 * T device pointers; cols <= 64.  Per chain bitwise the same as mlb_cgs2 +
 * mlb_scale_by.  work: mlb_cgs2_batched_work_size(T) doubles. */
int64_t mlb_cgs2_batched_work_size(int T);
int mlb_cgs2_batched(int T, const double* const* V, int64_t ld, int64_t n, int cols, double* const* w,
                     double* const* h_out, double* const* h1_out, double* const* nrm2_out, double* const* vnext,
                     double* work, void* stream);
/* Lockstep PKSM coefficients of step j for T chains (krylov.py:196-216),
 * one warp per chain, no host eigh: AB row t (device, ld >= 2 dim + 5
 * doubles) = [h1 (alpha_j at j) | ||w_j||^2 at dim + j | <v,v> at 2 dim |
 * stats out: min eigenvalue, ||c||^2, ||c - [c_prev; 0]||^2, status];
 * hist (device, T x 2 dim) receives alpha_j / beta_j; C (device, T x dim x
 * dim) receives c_j = ||v|| Q f(Lambda) Q[0,:]^T of T_{j+1} with f = max(.,0)^p,
 * eigenpairs by implicit QL.  status 1 = QL did not converge (recompute). */
int mlb_tridiag_fn_batched(int T, double* AB, int64_t ld, int dim, int j, double p, double* hist, double* C,
                           void* stream);
/* y = V[:, :cols] c  (c device) ; out may alias nothing */
int mlb_gemv_n(const double* V, int64_t ld, int64_t n, int cols, const double* c, double* y,
               double scale, int accumulate, void* stream);
/* Out[:, :k] = V[:, :s] S[:s, :k]  (S column-major s x k, device); Out must not alias V */
int mlb_gemm_vs(const double* V, int64_t ld, int64_t n, int s, const double* S, int k, double* Out,
                int64_t ldo, void* stream);
/* dot products / norms (device scalar out) */
int mlb_dot(const double* x, const double* y, int64_t n, double* out, double* work, void* stream);
/* y = a*x + b*y */
int mlb_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream);
/* y = x * scale_dev[0]^pow  (pow = -0.5 -> normalise by sqrt of a norm^2) */
int mlb_scale_by(const double* x, double* y, int64_t n, const double* s_dev, double pw, void* stream);

/* z = x .* y */
int mlb_hadamard(const double* x, const double* y, double* z, int64_t n, void* stream);

/* Exact dense kernel sums (direct_apply, fastsum.py:500-553) with the same
 * epilogue as mlb_apply: y (=|+=) alpha v + s.(beta sum_j K(x_i-x_j) s_j v_j
 * + gamma s.v), the sum INCLUDING j = i.  X: n x d row-major (device);
 * family 0 = gaussian, 1 = laplacian; s nullable (= 1). */
int mlb_direct(const double* X, int64_t n, int d, int family, double sigma, const double* v, const double* s,
               double* y, double alpha, double beta, double gamma, int accumulate, void* stream);

/* Exact sums at nt targets Xt (nt x d, device): yt[t] = sum_j K(|Xt_t - X_j|) v_j
 * over ALL n sources (a target that is also a source includes its K(0) v
 * term); the accuracy check of run_fastsum_bench (runner.py:496-512).  work:
 * mlb_direct_targets_work_size(nt) doubles. */
int64_t mlb_direct_targets_work_size(int64_t nt);
int mlb_direct_targets(const double* X, int64_t n, int d, int family, double sigma, const double* v, const double* Xt,
                       int64_t nt, double* yt, double* work, void* stream);

/* ---- Allen-Cahn (allencahn.py:172-223) ----------------------------------
 * Phi: n x k row-major, U/F: n x m row-major, fid: n.  One iteration:
 *   R = (1+c dt) U - dt/(2 eps) T(U) - dt fid (U-F);  Vc = Phi^T R / denom;
 *   U_next = proj_simplex(Phi Vc);  stats = [max_i |dU_i|^2, max_i |U_next_i|^2]. */
int64_t mlb_ac_work_size(int64_t n, int k, int m);
int mlb_ac_step(const double* Phi, int64_t n, int k, int m, const double* U, const double* F,
                const double* fid, const double* denom, double c_dt, double dt_2eps, double dt,
                double* U_next, double* stats, double* work, void* stream);
/* the same step with one pass over Phi (m <= 8): the update of iteration t and
   the right-hand side of iteration t+1 share the staged Phi tile; first = 1 on
   the first call of a solve (it also forms R(U_0)); the right-hand side stays
   in `work` between calls (m > 8: the two-pass mlb_ac_step) */
int mlb_ac_step2(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                 const double* denom, double c_dt, double dt_2eps, double dt, int first, double* U_next,
                 double* stats, double* work, void* stream);
/* the multiclass step split for node-range sharding: this
   rank's rows only.  rhs_partial: PtR (k x m, device) = Phi^T R(U) over the n
   local rows (fixed-order block sums); the caller all-reduces PtR over the
   ranks; update_from: Vc = PtR / denom, U_next = proj_simplex(Phi Vc), stats =
   the local [max |dU_i|^2, max |U_next_i|^2] (the caller max-reduces them).
   work: mlb_ac_work_size doubles. */
int mlb_ac_rhs_partial(const double* Phi, int64_t n, int k, int m, const double* U, const double* F, const double* fid,
                       double c_dt, double dt_2eps, double dt, double* PtR, double* work, void* stream);
int mlb_ac_update_from(const double* Phi, int64_t n, int k, int m, const double* PtR, const double* denom,
                       const double* U, double* U_next, double* stats, double* work, void* stream);
/* one binary Allen-Cahn step (allencahn.py:261-309): v_next = (lead v - dt/eps Phi^T u^3
   - dt Phi^T (fid (u - f))) / denom, u_next = Phi v_next; stats = (max (u_next-u)^2, max u_next^2);
   work: mlb_ac_work_size(n, k, 1) doubles */
int mlb_bac_step(const double* Phi, int64_t n, int k, const double* u, const double* f, const double* fid,
                 const double* v, const double* denom, double lead, double dt_eps, double dt, double* v_next,
                 double* u_next, double* stats, double* work, void* stream);
/* Ginzburg-Landau energy terms (allencahn.py:232-252): per block (fixed partition)
   [Phi^T U (k x m, only if Phi) | sum_i prod_q A_iq^2/4 | sum_i fid_i |F_i - U_i|^2];
   the caller sums the *nblocks rows in order.  partial: mlb_gl_energy_work_size doubles */
int64_t mlb_gl_energy_work_size(int k, int m);
int mlb_gl_energy_partials(const double* Phi, int64_t n, int k, int m, const double* U, const double* F,
                           const double* fid, double* partial, int* nblocks, void* stream);
/* argmax per row, ties to the lowest class (allencahn.py:226-229) */
int mlb_argmax_rows(const double* U, int64_t n, int m, int32_t* labels, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MULTILAP_B200_H */
