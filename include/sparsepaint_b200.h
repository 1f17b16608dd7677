/*
 * sparsepaint_b200.h -- C-ABI of libsparsepaint_b200.so, the sm_100a
 * implementation of the data-optimization hot path of arXiv 2401.06747
 * (reference package `sparsepaint` 0.1.0 under /root/reference/pkg).
 *
 * Conventions
 *   - every entry returns 0 on success, < 0 on failure; the message is
 *     available from sp_last_error() (thread-local).  Nothing throws.
 *   - pointers named x/u/out/... are DEVICE pointers unless suffixed _h.
 *   - images are planar (C, H, W), contiguous, dtype code 0 = float32,
 *     1 = float64 (MultigridConfig.dtype, solver.py:49-82); masks are
 *     (H, W) uint8 (0/1), labels int32, seeds int64 (m, 2) rows (y, x).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work
 *     is stream-ordered; calls return before the GPU finishes unless stated.
 *   - buffers are caller-owned; temporaries come from the stream-ordered
 *     allocator; handles (sp_hier_*) own their device pyramids.
 *
 * Boundary B1 below replaces, entry by entry, the 16-name kernel table the
 * reference selects at import time (kernels/__init__.py:12-29, 43-66); the
 * Python binding paper_2401_06747_b200/kernels/cuda_impl.py exposes them
 * with the reference's numpy signatures so that
 * `monkeypatch.setattr(sparsepaint.kernels, name, cuda_impl.<name>)`
 * (test_backends.py:132-152) drives the reference orchestration on the GPU.
 * Boundary B2 is the device-resident path behind the public entry points
 * inpaint / delaunay_densify / voronoi_richardson_init / ras_tonal /
 * cgnr_tonal (sparsepaint/__init__.py:9-56).
 */
#ifndef SPARSEPAINT_B200_H
#define SPARSEPAINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 1
#define SP_DTYPE_F32 0
#define SP_DTYPE_F64 1

const char* sp_last_error(void);
int sp_abi_version(void);

/* ======================= B1: kernel table ================================ */

/* numba_impl.py:13-36  negated_laplacian(x, inv_h2) */
int sp_negated_laplacian(int dtype, const void* x, void* out, int C, int H, int W,
                         double inv_h2, void* stream);
/* numba_impl.py:39-65  inpaint_matvec(x, mask, inv_h2) */
int sp_inpaint_matvec(int dtype, const void* x, const uint8_t* mask, void* out, int C,
                      int H, int W, double inv_h2, void* stream);
/* numba_impl.py:68-98  sym_matvec(x, mask, inv_h2) */
int sp_sym_matvec(int dtype, const void* x, const uint8_t* mask, void* out, int C, int H,
                  int W, double inv_h2, void* stream);
/* numba_impl.py:101-121  sym_rhs(b, mask, inv_h2) */
int sp_sym_rhs(int dtype, const void* b, const uint8_t* mask, void* out, int C, int H,
               int W, double inv_h2, void* stream);
/* numba_impl.py:124-144  ct_apply(w, mask, inv_h2) */
int sp_ct_apply(int dtype, const void* w, const uint8_t* mask, void* out, int C, int H,
                int W, double inv_h2, void* stream);
/* numba_impl.py:147-158  sym_residual(u, bsym, mask, inv_h2) -> (r, norms);
 * norms is a device double[C] */
int sp_sym_residual(int dtype, const void* u, const void* bsym, const uint8_t* mask,
                    void* r, double* norms, int C, int H, int W, double inv_h2,
                    void* stream);
/* numba_impl.py:161-263  oras_apply(u, r, mask, xs, ys, bh, bw, gamma, taus, cap,
 * weights, inv_h2) -- mutates u.  xs_h/ys_h/taus_h are HOST arrays, weights a
 * device (nby*nbx, bh, bw) array of dtype.  Synchronizes the stream. */
int sp_oras_apply(int dtype, void* u, const void* r, const uint8_t* mask,
                  const int64_t* xs_h, int nbx, const int64_t* ys_h, int nby, int bh,
                  int bw, double gamma, const double* taus_h, long cap,
                  const void* weights, double inv_h2, int C, int H, int W, void* stream);
/* numba_impl.py:266-284  restrict_values(fine) -> (C, ceil(H/2), ceil(W/2)) */
int sp_restrict_values(int dtype, const void* fine, void* out, int C, int H, int W,
                       void* stream);
/* numba_impl.py:287-313  restrict_mask(mask, values) -> (cmask, cvals) */
int sp_restrict_mask(int dtype, const uint8_t* mask, const void* values, uint8_t* cmask,
                     void* cvals, int C, int H, int W, void* stream);
/* numba_impl.py:316-348  prolongate(coarse, h, w) */
int sp_prolongate(int dtype, const void* coarse, void* out, int C, int ch, int cw, int H,
                  int W, void* stream);
/* numba_impl.py:351-396  jfa_run(labels, seeds, steps); steps_h is HOST int64 */
int sp_jfa_run(const int32_t* labels, int32_t* out, const int64_t* seeds, long m,
               const int64_t* steps_h, int nsteps, int H, int W, void* stream);
/* numba_impl.py:399-409  jfa_dist2(labels, seeds) -> int64 (H, W); out may be
 * NULL; dmax (device uint64, may be NULL) receives max d^2 (geometry.py:108-110) */
int sp_jfa_dist2(const int32_t* labels, const int64_t* seeds, long m, int64_t* out, int H,
                 int W, uint64_t* dmax, void* stream);
/* numba_impl.py:412-439  fs_dither(dens) -> uint8 (serial, bit-exact) */
int sp_fs_dither(const double* dens, uint8_t* out, int H, int W, void* stream);
/* numba_impl.py:442-466  assign_triangles(tris, vy, vx, h, w) -> int32 */
int sp_assign_triangles(const int64_t* tris, long ntris, const int64_t* vy,
                        const int64_t* vx, int H, int W, int32_t* out, void* stream);
/* numba_impl.py:469-481  fallback_assign(assign, labels, seed_min_tri) */
int sp_fallback_assign(const int32_t* assign, const int32_t* labels,
                       const int32_t* seed_min_tri, int32_t* out, int H, int W,
                       void* stream);
/* numba_impl.py:484-498  reduce_cells(assign, err, ntris) -> (sums, amax, amax_val) */
int sp_reduce_cells(const int32_t* assign, const double* err, long ntris, double* sums,
                    int64_t* amax_idx, double* amax_val, int H, int W, void* stream);

/* helpers used by the device-resident path */
int sp_masked_sym_rhs(int dtype, const void* x, const uint8_t* mask, void* out, int C,
                      int H, int W, void* stream); /* sym_rhs(where(mask, x, 0)) */
int sp_enforce(int dtype, void* u, const void* src, const uint8_t* mask, int C, int H,
               int W, int zero_off, void* stream); /* u[mask] = src[mask] */

/* deterministic per-channel reductions over C planes of n elements; out is a
 * device double[C].  mode 0: sum x^2, 1: sum x*y, 2: sum (x - z)^2 with z a
 * double array, 3: sum (x - y)^2 with y of x's dtype (tonal.py:86-97
 * _mse/_chan_dot, grid.py:188-193 quality) */
int sp_chan_reduce(int dtype, int mode, const void* x, const void* y, const double* z, long n,
                   int C, double* out, void* stream);
/* e = sum_c (u_c - f_c)^2 in double, f double (spatial.py:184-186 _error_map) */
int sp_error_map(int dtype, const void* u, const double* f, double* e, int C, long n,
                 void* stream);
/* sp_error_map plus *total = sum of e (device double; the MSE numerator of
 * grid.py:188-193, summed in a fixed order) in the same pass */
int sp_error_map_sum(int dtype, const void* u, const double* f, double* e, int C, long n,
                     double* total, void* stream);

/* ======================= B2: device-resident solver ====================== */

/* GridHierarchy (solver.py:205-372).  One handle per (dtype, C, H, W, cfg);
 * sp_hier_set_mask rebuilds the mask/value pyramid in place, so a handle is
 * reused across the masks of a densification run. */
typedef struct sp_solve_report {
  int iterations; /* V-cycles run (SolverReport.iterations) */
  int converged;
  int nres;       /* entries used in residuals[] */
  int pad;
  double residuals[256]; /* relative residual before each V-cycle */
} sp_solve_report;

/* ntile independent problems of the same (C, H, W) share one handle; their
 * masks/vectors are stacked [tile][...] and each tile stops on its own
 * tolerance test (the RAS block-local systems, tonal.py:343-354) */
int sp_hier_create(void** out, int dtype, int C, int H, int W, int block, int overlap,
                   int levels, int pre, int post, double alpha, double rho,
                   int with_values, int ntile);
int sp_hier_destroy(void* hier);
int sp_hier_levels(void* hier, int* nlevels, int* dims, int cap);
int sp_hier_use_graphs(void* hier, int on);
int sp_hier_set_mask(void* hier, const uint8_t* mask, const void* values, void* stream);
int sp_hier_level_mask(void* hier, int level, uint8_t* out, void* stream);
/* solve_sym (solver.py:328-372): init_mode 0 = zeros, 1 = u holds the warm
 * start, 2 = FMG cascade (needs values); tol < 0 = run exactly `cycles`
 * V-cycles.  Synchronizes the stream once per V-cycle in tolerance mode. */
int sp_hier_solve(void* hier, const void* bsym, void* u, int init_mode, double tol,
                  int cycles, int max_cycles, sp_solve_report* rep, void* stream);
/* sp_hier_solve with separate start and result buffers (no copy of the
 * caller's warm start) and, for src_mode 1, the right-hand side formed from
 * stored values: src = x, b~ = sym_rhs(where(mask, x, 0)) (solver.py:501-502,
 * tonal.py:136-137) written straight into the hierarchy.  src_mode 0: src is
 * b~.  u_in is read for init_mode 1 only (NULL = u_out holds the start). */
int sp_hier_solve_ex(void* hier, const void* src, int src_mode, const void* u_in, void* u_out,
                     int init_mode, double tol, int cycles, int max_cycles,
                     sp_solve_report* rep, void* stream);
int sp_hier_vcycle(void* hier, const void* bsym, void* u, void* stream);
/* batched solve_sym: active_h (HOST int[ntile], NULL = all) selects the tiles
 * to solve; iters_h / conv_h (HOST int[ntile], may be NULL) receive the
 * per-tile V-cycle counts and converged flags */
int sp_hier_solve_tiles(void* hier, const void* bsym, void* u, int init_mode, double tol,
                        int cycles, int max_cycles, const int* active_h, int* iters_h,
                        int* conv_h, void* stream);

/* ============ B2: row-strip partitioned solve ============== */
/* The north_star's multi-GPU layout for large images: the finest `La`
 * levels of the inpainting hierarchy are cut into P row strips (owned rows
 * o0/o1, int[La][P], multiples of 16 except the image end), each computed
 * on its owned rows widened by `halo` (>= 33, multiple of 16) rows; the
 * coarser levels are replicated.  Per smoothing sweep: halo exchange, ORAS
 * on the view, and the residual norms combined across strips as
 * partition-independent row-band partials, so the solve is bit-identical for
 * every P.  This process holds strips [first, first + nloc); strips on other
 * ranks are reached through the NCCL communicator `comm` (one strip per
 * rank, rank = strip index), strips in this process through device copies.
 * Same semantics as sp_hier_solve (solver.py:328-372) on a float32 image;
 * bsym / u are full-size, u returns the gathered solution on every rank.
 * No reference counterpart: the reference is single-process CPU code. */
int sp_nccl_unique_id(uint8_t* out128);
int sp_nccl_comm_create(void** comm, const uint8_t* id128, int nranks, int rank);
int sp_nccl_comm_destroy(void* comm);
int sp_strip_create(void** out, int C, int H, int W, int block, int overlap, int levels,
                    int pre, int post, double alpha, double rho, int P, int nloc, int first,
                    int La, int halo, const int* o0_h, const int* o1_h, void* comm);
int sp_strip_destroy(void* group);
int sp_strip_set_mask(void* group, const uint8_t* mask, const void* values, void* stream);
int sp_strip_solve(void* group, const void* bsym, void* u, int init_mode, double tol,
                   int cycles, int max_cycles, sp_solve_report* rep, void* stream);
int sp_strip_levels(void* group, int* nlev, int* dims, int cap);
/* Host-staged transport for a strip group whose strips live on other ranks
 * (instead of the NCCL communicator of sp_strip_create): halo rows, the
 * band-sum all-reduce and the agglomeration broadcasts go through these
 * callbacks on pinned host buffers, stream-synchronously, and the V-cycle is
 * not graph-captured.  It runs the multi-rank protocol where NCCL cannot
 * (several ranks sharing one GPU: the CI harness; a gloo world).
 *   int sendrecv(void* user, int peer, const void* send, size_t send_bytes,
 *                void* recv, size_t recv_bytes);
 *   int allreduce_f64(void* user, double* buf, size_t n);      (sum)
 *   int bcast(void* user, void* buf, size_t bytes, int root);
 * Each returns 0 on success.  Replaces the NCCL path of csrc/strips.cu;
 * reference counterpart: none (the reference is single-process). */
int sp_strip_set_host_transport(void* group, void* sendrecv, void* allreduce_f64, void* bcast,
                                void* user);

/* ================ B2: densification geometry workspace ================== */
/* One workspace per (H, W).  Replaces, per densification iteration,
 * jump_flood_voronoi (geometry.py:92-110), delaunay_from_voronoi (:113-185),
 * accumulate_errors / voronoi_cell_errors (:197-244) and the pick loop of
 * delaunay_densify (spatial.py:245-259). */
int sp_geo_create(void** out, int H, int W);
int sp_geo_destroy(void* geo);
/* seeds = row-major nonzero of mask; start_hint < 1 means None; returns m,
 * max_radius = sqrt(max d^2) and the number of JFA passes.  Syncs. */
int sp_geo_voronoi(void* geo, const uint8_t* mask, double start_hint, long* m,
                   double* max_radius, int* nsteps, void* stream);
int sp_geo_delaunay(void* geo, long* ntris, void* stream); /* syncs */
/* Seed count from which sp_geo_delaunay sorts wide triangle keys (a, b << 32
 * | c) by two stable radix passes instead of packed 3 x 21-bit keys
 * (default and maximum 2^21, i.e. any mask the reference accepts works;
 * v <= 0 queries).  Lowered only by tests of the wide path. */
long sp_geo_wide_threshold(long v);
/* err: device double (H, W); voronoi != 0 buckets by cell instead of triangle */
int sp_geo_accumulate(void* geo, const double* err, int voronoi, void* stream);
/* implementation of sp_geo_accumulate (partition "delaunay"): 1 = tile-binned
 * rasteriser with shared-memory minima + per-triangle bounding-box walk
 * (default), 0 = global atomicMin rasteriser + pixel radix sort; both are
 * bit-identical to numba_impl.py:442-498.  v < 0 only reads the setting. */
int sp_geo_accumulate_mode(int v);
/* Programmatic dependent launch for the V-cycle kernels of the multigrid
 * levels >= v (the small levels; measured neutral, so off by default: -1); -1 turns it
 * off, v < -1 only reads the setting.  Results are identical either way. */
int sp_pdl_from_level(int v);
/* marks the argmax pixels of the `want` best eligible buckets in mask */
int sp_geo_select(void* geo, uint8_t* mask, long nbuckets, long want, long* picked,
                  void* stream);
/* spatial.py:189-197 */
int sp_geo_fill_highest_error(void* geo, const double* err, uint8_t* mask, long want,
                              void* stream);
/* Row-strip partition of the Delaunay step and the accumulate (SURVEY.md
 * section 8e; every rank holds the full labels -- jump flooding stays
 * replicated).  Replaces, across P ranks, sp_geo_delaunay + sp_geo_accumulate
 * (geometry.py:113-223) with bit-identical triangles and buckets:
 *   corner keys of rows [r0, r1) -> all-gather -> sp_geo_delaunay_from_keys;
 *   sp_geo_raster_rows(own rows) -> all-gather the assignment rows
 *   (sp_geo_assign_rows) -> sp_geo_reduce_range(own triangle range) ->
 *   all-gather the bucket ranges (sp_geo_set_buckets).
 * A triangle's sequential f64 sum is never split across ranks. */
int sp_geo_corner_keys(void* geo, int r0, int r1, long* nkeys, void* stream);
int sp_geo_keys_copy(void* geo, uint64_t* dst, long n, void* stream);
int sp_geo_delaunay_from_keys(void* geo, const uint64_t* keys, long n, long* ntris,
                              void* stream);
int sp_geo_raster_rows(void* geo, int r0, int r1, void* stream);
/* dir 0: rows [r0, r1) of the assignment to buf; dir 1: from buf */
int sp_geo_assign_rows(void* geo, int32_t* buf, int r0, int r1, int dir, void* stream);
int sp_geo_reduce_range(void* geo, const double* err, long t0, long t1, void* stream);
int sp_geo_set_buckets(void* geo, const double* sums, const int64_t* amax,
                       const double* amax_val, long t0, long t1, void* stream);
/* load caller labels (H,W) i32 + seed rows sy/sx (m) i32 into the workspace */
int sp_geo_load(void* geo, const int32_t* labels, const int32_t* sy, const int32_t* sx,
                long m, void* stream);
int sp_geo_export(void* geo, int32_t* labels, int32_t* sy, int32_t* sx, int32_t* tris,
                  double* sums, int64_t* amax, double* amax_val, long nbuckets,
                  void* stream);

/* ================ B2: dithered initial mask (spatial.py:107-148) ========== */
/* dens (H,W) double = clip(sum_c |L(gauss_sigma f_c)| * density*n/total, 0, 1);
 * gauss_h: 2r+1 HOST weights exactly as scipy's _gaussian_kernel1d; total_h
 * (HOST) receives the numpy pairwise total (0 = constant image).  Syncs. */
int sp_density_map(const double* f, int C, int H, int W, double density,
                   const double* gauss_h, int radius, double* dens, double* total_h,
                   void* stream);
/* analytic_mask(dither="random") + _exact_count; pcg_h = HOST {state_lo,
 * state_hi, inc_lo, inc_hi} of numpy default_rng(seed)'s PCG64.  Sets
 * *degenerate_h = 1 (mask untouched) when the Laplacian vanishes. */
int sp_init_mask_random(const double* f, int C, int H, int W, long target, double density,
                        const double* gauss_h, int radius, const uint64_t* pcg_h,
                        uint8_t* mask, int* degenerate_h, void* stream);
/* doubles start..start+count-1 of numpy Generator(PCG64).random (tests) */
int sp_pcg64_doubles(const uint64_t* pcg_h, long long start, long long count, double* out,
                     void* stream);
/* numpy pairwise sum of a device double array (result on the HOST) */
int sp_pairwise_sum(const double* a, long long n, double* out_h, void* stream);

/* ======================= B2: tonal optimizers (tonal.py) ================== */
/* pixels stably sorted by label: perm (H*W), per-cell [start, end) */
int sp_cell_index(const int32_t* labels, int H, int W, long m, int32_t* perm, int32_t* start,
                  int32_t* end, void* stream);
/* voronoi_weights (geometry.py:247-264): scheme 0 constant, 1 inverse-log */
int sp_vi_weights(const int32_t* labels, const int32_t* sy, const int32_t* sx,
                  const int32_t* perm, const int32_t* start, const int32_t* end, int H, int W,
                  long m, int scheme, double* w, void* stream);
/* per-cell sequential sums in pixel order (np.bincount) */
int sp_cell_sum(const int32_t* perm, const int32_t* start, const int32_t* end, const double* v,
                long m, double* out, void* stream);
/* g[seed_t] += T(tau * sum_cell w (f - u)) per channel (tonal.py:459-464) */
int sp_vi_step(int dtype, const int32_t* perm, const int32_t* start, const int32_t* end,
               const double* w, const void* f, const void* u, const int32_t* sy,
               const int32_t* sx, long m, int C, int H, int W, double tau, void* g,
               void* stream);
/* out[plane] = sum x*y (y NULL: x*x), planes of len elements, double */
int sp_plane_dot(int dtype, const void* x, const void* y, long len, long nplanes, int C,
                 const int32_t* active, double* out, void* stream);
/* yout = x + sign * T(coef[plane]) * z, per plane (CG vector updates) */
int sp_plane_axpy(int dtype, void* yout, const void* x, const void* z, const double* coef,
                  double sign, long len, long nplanes, int C, const int32_t* active,
                  void* stream);
int sp_gather_tiles(int dtype, const void* img, const int32_t* oy, const int32_t* ox, int ntile,
                    int C, int H, int W, int bh, int bw, void* out, void* stream);
int sp_gather_mask_tiles(const uint8_t* mask, const int32_t* oy, const int32_t* ox, int ntile,
                         int H, int W, int bh, int bw, uint8_t* out, void* stream);
/* g += sum over covering RAS blocks of T(1/cover) * v_b (tonal.py:375-380) */
int sp_ras_scatter(int dtype, void* g, const void* v, const int32_t* tile_of,
                   const int32_t* ys, const int32_t* xs, const int32_t* row_k0,
                   const int32_t* row_n, const int32_t* col_k0, const int32_t* col_n, int nbx,
                   int bh, int bw, int C, int H, int W, void* stream);
int sp_where_mask(int dtype, const void* x, const uint8_t* mask, void* out, int C, int H, int W,
                  void* stream);
/* neighbor_balance_init (tonal.py:389-414, scipy.ndimage.correlate with a
 * 3x3 ones kernel, mode="constant"): g = T(u + box(f - u) / box(1)) on the
 * mask, 0 elsewhere.  f is the f64 image [C,H,W]; u, g are [C,H,W] of dtype. */
int sp_neighbor_balance(int dtype, const double* f, const void* u, const uint8_t* mask, void* g,
                        int C, int H, int W, void* stream);
int sp_masked_sym_rhs_tiles(int dtype, const void* x, const uint8_t* mask, void* out, int C,
                            int H, int W, int ntile, const int32_t* active, void* stream);
int sp_ct_apply_tiles(int dtype, const void* w, const uint8_t* mask, void* out, int C, int H,
                      int W, int ntile, const int32_t* active, void* stream);

/* ======================= tracing / measurement =========================== */
/* ORAS local-CG statistics {jobs, iterations, converged-on-entry, max it};
 * enable 1 = reset+start, 0 = reset+stop, -1 = read only */
int sp_stats(int enable, uint64_t* out_h);
/* float ORAS kernel for blocks <= 32x32: 4 = one warp per job, registers
 * only (default), 0 = register-resident 4-warp job kernel, one job per CTA
 * (bit-identical to 4), 1 = 256-thread CTA kernel, 3 = the 4-warp kernel
 * persistent with cp.async prefetch; v < 0 query */
int sp_oras_variant(int v);
/* Batched cold tile solves (sp_hier_solve_tiles, the RAS block-local
 * products tonal.py:120-131) on the fused on-chip kernel (tilesolve.cu: one
 * cluster of C CTAs per block, whole solve in shared memory) when the
 * hierarchy qualifies (float, two levels, <= 64x64): 1 = on (default),
 * 0 = the batched V-cycle path; v < 0 queries.  A/B aid. */
int sp_tile_fused(int v);
/* V-cycle graphs of multi-channel hierarchies captured afterwards run the C
 * channels as parallel graph branches (solver.cu run_vcycle): 1 = on,
 * 0 = one sequential chain (default, measured faster); v < 0 queries.
 * Results are identical either way.  A/B aid. */
int sp_channel_parallel(int v);
/* Tolerance-mode solves of one image as ONE graph launch: a WHILE
 * conditional node around {stop test kernel; IF{V-cycle; residual}}, the
 * stop test (solver.py:358-368) on the device, no host round trip per
 * V-cycle: 1 = on, 0 = host-driven loop (default: equal speed, and the
 * host-driven form keeps every kernel visible to CUPTI profilers); v < 0
 * queries.  Results, iteration counts and residual histories are identical. */
int sp_graph_loop(int v);
/* Default sweep kernels of hierarchies created afterwards (all bit-identical
 * per element): 2 = TMA-staged residual sweeps on wide float levels
 * (mgtma.cu, default), 1 = row-marching register kernels (mgfast.cu), 0 =
 * the per-pixel kernels everywhere; v < 0 queries.  A/B measurement aid, no
 * reference counterpart. */
int sp_march_variant(int v);
/* Within sweep variant 2: 1 = warp-streamed TMA kernels (each warp marches
 * its own range of 8-row chunks through a private TMA ring, default), 0 =
 * the CTA-tile TMA kernels.  Residuals, restrictions and prolongations are
 * bit-identical; the residual norms group their float partials differently.
 * Applies to launches made afterwards; v < 0 queries.  A/B aid, no
 * reference counterpart. */
int sp_ws_variant(int v);
/* Chunks each warp of the warp-streamed sweeps keeps prefetched into L2
 * ahead of its shared-memory ring (cp.async.bulk.prefetch.tensor; default 0,
 * measured slower); v < 0 queries.  Timing only, results unchanged. */
int sp_ws_prefetch(int v);
/* Shared-memory stages per warp of the warp-streamed sweeps: 1 or 2 for
 * every sweep, 0 = the measured per-sweep defaults (residual 2, restriction
 * and prolongation 1); v < 0 queries.  Timing only, results unchanged. */
int sp_ws_stages(int v);
/* ORAS local-CG jobs read per-job row-mask words precomputed with the mask
 * pyramid (1, default) or load and test their mask bytes (0); bit-identical.
 * v < 0 queries.  A/B aid, no reference counterpart. */
int sp_oras_offbits(int v);
/* Fused RAS block solves of a partly active batch launch their grids over
 * the list of active blocks (1, default) or over every block with early
 * exits (0); identical results.  v < 0 queries. */
int sp_tile_list(int v);
/* One-image tolerance solves form ||b~||^2 (the tolerance scale,
 * solver.py:351-352) in the masked_sym_rhs pass (1, default) or by a
 * separate reduction (0); the sums group differently (rounding only).
 * v < 0 queries. */
int sp_fused_bnorm(int v);
/* Multigrid levels with fewer than v pixels per plane run the per-pixel
 * sweep kernels instead of the TMA / warp-streamed ones (identical
 * results); v < 0 queries. */
long sp_tma_min_pixels(long v);
/* Jump-flooding passes of step 1 and 2 on pixel quads with aligned 16-byte
 * candidate loads (1, default) or per pixel (0); bit-identical labels.
 * v < 0 queries. */
int sp_jfa_short4(int v);
/* C = 3 float blend: 2 = packed cover words on column pairs (two pixels per
 * 8-byte access where W and every block start are even, else 1; default),
 * 3 = the same with two rows per thread, 1 = packed per-row / per-column
 * cover words (one table load each), 0 = the cover-table chains; all
 * bit-identical.  v < 0 queries.  A/B aid, no reference counterpart. */
int sp_blend_packed(int v);
/* residual r = b~ - A~ u and per-plane sum r^2 of level lv's current iterate
 * (after a solve), computed by the hierarchy's sweep kernel, into device
 * buffers r_out [ntile][C][h][w], norms_out [ntile][C] (kernel-variant
 * checks; the residual of solver.py:256-258) */
int sp_hier_residual(void* hier, int lv, void* r_out, double* norms_out, void* stream);
/* kernels launched by the library since the last reset */
long long sp_launch_count(int reset);
/* finest-level pixel x V-cycle work of the solves since the last reset
 * (Mpixel-iterations of the metric): kind 0 = image-level solves, kind 1 =
 * batched block-local (RAS) solves */
long long sp_work_count(int kind, int reset);
/* CUDA-event timing of a finest-level kernel (0 residual, 1 ORAS local CG,
 * 2 blend, 3 residual+restrict, 4 prolongation+add+enforce): mean ms and algorithmic bytes per launch */
int sp_hier_bench(void* hier, int which, int reps, double* ms_h, double* bytes_h,
                  void* stream);

/* ---- PNM wire formats, encoded on the device (pnm.py:40-127) ------------ */
/* P4 body of write_mask (pnm.py:78-84): np.packbits(mask != 0, axis=1), i.e.
 * H rows of ceil(W/8) bytes, MSB first; out holds H * ceil(W/8) bytes */
int sp_pack_mask_bits(const uint8_t* mask, int H, int W, uint8_t* out, void* stream);
/* inverse of the above (read_mask, pnm.py:87-95): mask u8 0/1 [H,W] */
int sp_unpack_mask_bits(const uint8_t* bits, int H, int W, uint8_t* mask, void* stream);
/* PGM/PPM body of values [C,H,W] (dtype code) as interleaved [H,W,C]:
 * wide = 0: clip(rint(v), 0, 255) u8 (write_image / 8-bit write_tonal,
 * grid.py:216-218); wide = 1: big-endian u16 clip(rint((v+256)*64), 0,
 * 65535) (pnm.py:106-117).  mask != NULL applies where(mask, v, 0) first
 * (write_tonal).  out holds H*W*C*(1 + wide) bytes. */
int sp_encode_pnm(int dtype, const void* values, const uint8_t* mask, int C, int H, int W,
                  int wide, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEPAINT_B200_H */
