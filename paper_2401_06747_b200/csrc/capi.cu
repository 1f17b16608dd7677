// capi.cu -- the C-ABI boundary (declared in include/sparsepaint_b200.h).
//
// Plain pointers and sizes only; every entry returns 0 on success and a
// negative code on failure with the message in sp_last_error().  Nothing
// throws across the boundary.  Device buffers are caller-owned (PyTorch on
// the Python side); temporaries come from the stream-ordered allocator.
#include <stdarg.h>

#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "solver.cuh"
#include "geometry.cuh"
#include "../../include/sparsepaint_b200.h"

namespace sp {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

void retain_pool_memory() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

static thread_local bool g_pdl_now = false;
bool pdl_now() { return g_pdl_now; }
void pdl_set(bool on) { g_pdl_now = on; }

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

void cover_tables(const std::vector<int>& starts, int size, int dim, std::vector<int>& k0,
                  std::vector<int>& n);

}  // namespace sp

using namespace sp;

#define STREAM(s) ((cudaStream_t)(s))
#define DISPATCH(dtype, CALL_F32, CALL_F64)                                   \
  do {                                                                        \
    if ((dtype) == SP_F32) return CALL_F32;                                   \
    if ((dtype) == SP_F64) return CALL_F64;                                   \
    set_error("unsupported dtype code %d", (int)(dtype));                     \
    return -2;                                                                \
  } while (0)

extern "C" {

const char* sp_last_error(void) { return last_error(); }

int sp_abi_version(void) { return SP_ABI_VERSION; }

// ---- B1: kernel table (kernels/__init__.py:12-29) ---------------------------

int sp_negated_laplacian(int dtype, const void* x, void* out, int C, int H, int W,
                         double inv_h2, void* s) {
  DISPATCH(dtype, neglap<float>((const float*)x, (float*)out, C, H, W, inv_h2, STREAM(s)),
           neglap<double>((const double*)x, (double*)out, C, H, W, inv_h2, STREAM(s)));
}

int sp_inpaint_matvec(int dtype, const void* x, const uint8_t* m, void* out, int C, int H,
                      int W, double inv_h2, void* s) {
  DISPATCH(dtype,
           inpaint_matvec<float>((const float*)x, m, (float*)out, C, H, W, inv_h2, STREAM(s)),
           inpaint_matvec<double>((const double*)x, m, (double*)out, C, H, W, inv_h2, STREAM(s)));
}

int sp_sym_matvec(int dtype, const void* x, const uint8_t* m, void* out, int C, int H, int W,
                  double inv_h2, void* s) {
  DISPATCH(dtype,
           sym_matvec<float>((const float*)x, m, (float*)out, C, H, W, inv_h2, STREAM(s)),
           sym_matvec<double>((const double*)x, m, (double*)out, C, H, W, inv_h2, STREAM(s)));
}

int sp_sym_rhs(int dtype, const void* b, const uint8_t* m, void* out, int C, int H, int W,
               double inv_h2, void* s) {
  DISPATCH(dtype,
           sym_rhs<float>((const float*)b, m, (float*)out, nullptr, C, H, W, inv_h2, STREAM(s)),
           sym_rhs<double>((const double*)b, m, (double*)out, nullptr, C, H, W, inv_h2,
                           STREAM(s)));
}

int sp_ct_apply(int dtype, const void* w, const uint8_t* m, void* out, int C, int H, int W,
                double inv_h2, void* s) {
  DISPATCH(dtype,
           ct_apply<float>((const float*)w, m, (float*)out, C, H, W, inv_h2, STREAM(s)),
           ct_apply<double>((const double*)w, m, (double*)out, C, H, W, inv_h2, STREAM(s)));
}

int sp_masked_sym_rhs(int dtype, const void* x, const uint8_t* m, void* out, int C, int H,
                      int W, void* s) {
  DISPATCH(dtype, masked_sym_rhs<float>((const float*)x, m, (float*)out, C, H, W, STREAM(s)),
           masked_sym_rhs<double>((const double*)x, m, (double*)out, C, H, W, STREAM(s)));
}

int sp_sym_residual(int dtype, const void* u, const void* bsym, const uint8_t* m, void* r,
                    double* norms, int C, int H, int W, double inv_h2, void* s) {
  cudaStream_t st = STREAM(s);
  size_t np = residual_partials(H, W);
  Scratch scr(st);
  SP_TRY(scr.alloc(sizeof(double) * C * np + sizeof(unsigned) * C + 256));
  unsigned* counter = (unsigned*)((char*)scr.p + sizeof(double) * C * np);
  SP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned) * C, st));
  double* part = (double*)scr.p;
  DISPATCH(dtype,
           residual<float>((const float*)u, (const float*)bsym, m, (float*)r, part, counter,
                           norms, C, H, W, inv_h2, st),
           residual<double>((const double*)u, (const double*)bsym, m, (double*)r, part,
                            counter, norms, C, H, W, inv_h2, st));
}

int sp_oras_apply(int dtype, void* u, const void* r, const uint8_t* m, const int64_t* xs_h,
                  int nbx, const int64_t* ys_h, int nby, int bh, int bw, double gamma,
                  const double* taus_h, long cap, const void* weights, double inv_h2, int C,
                  int H, int W, void* s) {
  cudaStream_t st = STREAM(s);
  if (bh > H || bw > W || bh < 1 || bw < 1) {
    set_error("block (%d, %d) does not fit the grid (%d, %d)", bh, bw, H, W);
    return -2;
  }
  std::vector<int> ys(nby), xs(nbx), rk0, rn, ck0, cn;
  for (int i = 0; i < nby; ++i) ys[i] = (int)ys_h[i];
  for (int i = 0; i < nbx; ++i) xs[i] = (int)xs_h[i];
  for (int i = 1; i < nby; ++i)
    if (ys[i] < ys[i - 1]) { set_error("block starts must be sorted"); return -2; }
  for (int i = 1; i < nbx; ++i)
    if (xs[i] < xs[i - 1]) { set_error("block starts must be sorted"); return -2; }
  cover_tables(ys, bh, H, rk0, rn);
  cover_tables(xs, bw, W, ck0, cn);
  for (int y = 0; y < H; ++y)
    if (rn[y] > 3) { set_error("more than 3 blocks cover row %d", y); return -2; }
  for (int x = 0; x < W; ++x)
    if (cn[x] > 3) { set_error("more than 3 blocks cover column %d", x); return -2; }
  size_t es = dtype == SP_F64 ? 8 : 4;
  size_t ncorr = (size_t)C * nby * nbx * bh * bw;
  size_t ints = (size_t)nby + nbx + 2 * (size_t)H + 2 * (size_t)W;
  Scratch scr(st);
  SP_TRY(scr.alloc(es * ncorr + sizeof(double) * C + sizeof(int) * ints + 64));
  char* base = (char*)scr.p;
  void* corr = base;
  double* taus = (double*)(base + es * ncorr);
  int* ip = (int*)(taus + C);
  int *dys = ip, *dxs = dys + nby, *drk0 = dxs + nbx, *drn = drk0 + H, *dck0 = drn + H,
      *dcn = dck0 + W;
  std::vector<int> packed;
  packed.reserve(ints);
  packed.insert(packed.end(), ys.begin(), ys.end());
  packed.insert(packed.end(), xs.begin(), xs.end());
  packed.insert(packed.end(), rk0.begin(), rk0.end());
  packed.insert(packed.end(), rn.begin(), rn.end());
  packed.insert(packed.end(), ck0.begin(), ck0.end());
  packed.insert(packed.end(), cn.begin(), cn.end());
  SP_CUDA(cudaMemcpyAsync(taus, taus_h, sizeof(double) * C, cudaMemcpyHostToDevice, st));
  SP_CUDA(cudaMemcpyAsync(ip, packed.data(), sizeof(int) * ints, cudaMemcpyHostToDevice, st));
  if (dtype == SP_F32) {
    SP_TRY(oras_local_launch<float>((const float*)r, m, taus, 1.0, dys, dxs, nby, nbx, bh, bw,
                                    H, W, C, gamma, cap, inv_h2, (const float*)weights,
                                    (float*)corr, st));
    SP_TRY(oras_blend_launch<float>((float*)u, (const float*)corr, dys, dxs, drk0, drn, dck0,
                                    dcn, nby, nbx, bh, bw, H, W, C, st));
  } else if (dtype == SP_F64) {
    SP_TRY(oras_local_launch<double>((const double*)r, m, taus, 1.0, dys, dxs, nby, nbx, bh,
                                     bw, H, W, C, gamma, cap, inv_h2, (const double*)weights,
                                     (double*)corr, st));
    SP_TRY(oras_blend_launch<double>((double*)u, (const double*)corr, dys, dxs, drk0, drn,
                                     dck0, dcn, nby, nbx, bh, bw, H, W, C, st));
  } else {
    set_error("unsupported dtype code %d", dtype);
    return -2;
  }
  // keep the host staging vectors alive until the copies are consumed
  SP_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sp_restrict_values(int dtype, const void* f, void* out, int C, int H, int W, void* s) {
  DISPATCH(dtype, restrict_values<float>((const float*)f, (float*)out, C, H, W, STREAM(s)),
           restrict_values<double>((const double*)f, (double*)out, C, H, W, STREAM(s)));
}

int sp_restrict_mask(int dtype, const uint8_t* m, const void* v, uint8_t* cm, void* cv, int C,
                     int H, int W, void* s) {
  DISPATCH(dtype,
           restrict_mask<float>(m, (const float*)v, cm, (float*)cv, C, H, W, STREAM(s)),
           restrict_mask<double>(m, (const double*)v, cm, (double*)cv, C, H, W, STREAM(s)));
}

int sp_prolongate(int dtype, const void* co, void* out, int C, int ch, int cw, int H, int W,
                  void* s) {
  DISPATCH(dtype,
           prolongate<float>((const float*)co, (float*)out, C, ch, cw, H, W, STREAM(s)),
           prolongate<double>((const double*)co, (double*)out, C, ch, cw, H, W, STREAM(s)));
}

int sp_enforce(int dtype, void* u, const void* src, const uint8_t* m, int C, int H, int W,
               int zero_off, void* s) {
  DISPATCH(dtype, enforce<float>((float*)u, (const float*)src, m, C, H, W, zero_off, STREAM(s)),
           enforce<double>((double*)u, (const double*)src, m, C, H, W, zero_off, STREAM(s)));
}

// ---- vector reductions (deterministic; tonal.py:86-97, grid.py:188-193) ------
// mode 0: out[c] = sum x_c^2; 1: sum x_c*y_c; 2: sum (x_c - z_c)^2 (z double);
// 3: sum (x_c - y_c)^2 (y of x's dtype)
int sp_chan_reduce(int dtype, int mode, const void* x, const void* y, const double* z, long n,
                   int C, double* out, void* s) {
  cudaStream_t st = STREAM(s);
  Scratch scr(st);
  SP_TRY(scr.alloc(sizeof(double) * 1024 * (size_t)C + 64));
  unsigned* counter = (unsigned*)((double*)scr.p + 1024 * (size_t)C);
  SP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), st));
  DISPATCH(dtype,
           chan_reduce<float>(mode, (const float*)x, (const float*)y, z, (size_t)n, C,
                              (double*)scr.p, counter, out, st),
           chan_reduce<double>(mode, (const double*)x, (const double*)y, z, (size_t)n, C,
                               (double*)scr.p, counter, out, st));
}

int sp_error_map(int dtype, const void* u, const double* f, double* e, int C, long n, void* s) {
  DISPATCH(dtype, error_map<float>((const float*)u, f, e, C, (size_t)n, STREAM(s)),
           error_map<double>((const double*)u, f, e, C, (size_t)n, STREAM(s)));
}

// the error map and its total (the MSE numerator) in one pass
int sp_error_map_sum(int dtype, const void* u, const double* f, double* e, int C, long n,
                     double* total, void* s) {
  DISPATCH(dtype, error_map<float>((const float*)u, f, e, C, (size_t)n, STREAM(s), total),
           error_map<double>((const double*)u, f, e, C, (size_t)n, STREAM(s), total));
}

// ---- B2: device-resident hierarchy (solver.py:205-372) ----------------------

int sp_hier_create(void** out, int dtype, int C, int H, int W, int block, int overlap,
                   int levels, int pre, int post, double alpha, double rho, int with_values,
                   int ntile) {
  if (dtype != SP_F32 && dtype != SP_F64) {
    set_error("unsupported dtype code %d", dtype);
    return -2;
  }
  HierCfg cfg;
  cfg.block = block;
  cfg.overlap = overlap;
  cfg.levels = levels;
  cfg.pre = pre;
  cfg.post = post;
  cfg.alpha = alpha;
  cfg.rho = rho;
  Hier* h = nullptr;
  SP_TRY(hier_create(&h, dtype, C, H, W, cfg, with_values, ntile));
  *out = h;
  return 0;
}

int sp_hier_destroy(void* h) {
  delete (Hier*)h;
  return 0;
}

int sp_hier_levels(void* hp, int* nlevels, int* dims, int cap) {
  Hier* h = (Hier*)hp;
  *nlevels = (int)h->lv.size();
  for (int i = 0; i < (int)h->lv.size() && 2 * i + 1 < cap; ++i) {
    dims[2 * i] = h->lv[i].H;
    dims[2 * i + 1] = h->lv[i].W;
  }
  return 0;
}

int sp_hier_use_graphs(void* hp, int on) {
  Hier* h = (Hier*)hp;
  h->use_graphs = on != 0;
  if (!h->use_graphs && h->graph_exec) {
    cudaGraphExecDestroy(h->graph_exec);
    h->graph_exec = nullptr;
  }
  return 0;
}

int sp_hier_set_mask(void* h, const uint8_t* mask, const void* values, void* s) {
  return hier_set_mask((Hier*)h, mask, values, STREAM(s));
}

// level mask / values read-back (tests: restrict_mask chain parity)
int sp_hier_level_mask(void* hp, int lv, uint8_t* out, void* s) {
  Hier* h = (Hier*)hp;
  if (lv < 0 || lv >= (int)h->lv.size()) { set_error("bad level %d", lv); return -2; }
  Level& L = h->lv[lv];
  SP_CUDA(cudaMemcpyAsync(out, L.mask, (size_t)L.H * L.W, cudaMemcpyDeviceToDevice, STREAM(s)));
  return 0;
}

int sp_hier_solve(void* h, const void* bsym, void* u, int init_mode, double tol, int cycles,
                  int max_cycles, sp_solve_report* rep, void* s) {
  static_assert(sizeof(sp_solve_report) == sizeof(SolveReport), "report layout");
  return hier_solve((Hier*)h, bsym, u, init_mode, tol, cycles, max_cycles, STREAM(s),
                    nullptr, nullptr, nullptr, (SolveReport*)rep);
}

int sp_hier_solve_ex(void* h, const void* src, int src_mode, const void* u_in, void* u_out,
                     int init_mode, double tol, int cycles, int max_cycles, sp_solve_report* rep,
                     void* s) {
  if (src_mode != 0 && src_mode != 1) { sp::set_error("bad src_mode %d", src_mode); return -3; }
  return hier_solve((Hier*)h, src, u_out, init_mode, tol, cycles, max_cycles, STREAM(s),
                    nullptr, nullptr, nullptr, (SolveReport*)rep, u_in, src_mode);
}

int sp_hier_solve_tiles(void* h, const void* bsym, void* u, int init_mode, double tol,
                        int cycles, int max_cycles, const int* active_h, int* iters_h,
                        int* conv_h, void* s) {
  return hier_solve((Hier*)h, bsym, u, init_mode, tol, cycles, max_cycles, STREAM(s),
                    active_h, iters_h, conv_h, nullptr);
}

int sp_hier_vcycle(void* h, const void* bsym, void* u, void* s) {
  return hier_vcycle((Hier*)h, bsym, u, STREAM(s));
}


// ---- B1: geometry kernels ----------------------------------------------------

int sp_jfa_run(const int32_t* labels, int32_t* out, const int64_t* seeds, long m,
               const int64_t* steps_h, int nsteps, int H, int W, void* s) {
  cudaStream_t st = STREAM(s);
  size_t n = (size_t)H * W;
  Scratch scr(st);
  SP_TRY(scr.alloc(sizeof(int) * (2 * n + 2 * (size_t)(m > 0 ? m : 1))));
  int* a = (int*)scr.p;
  int* b = a + n;
  int* sy = b + n;
  int* sx = sy + (m > 0 ? m : 1);
  SP_TRY(seeds_to_soa((const long long*)seeds, m, sy, sx, st));
  SP_CUDA(cudaMemcpyAsync(a, labels, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  int* res = nullptr;
  SP_TRY(jfa_passes(a, b, sy, sx, (const long long*)steps_h, nsteps, H, W, &res, st));
  SP_CUDA(cudaMemcpyAsync(out, res, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  return 0;
}

int sp_jfa_dist2(const int32_t* labels, const int64_t* seeds, long m, int64_t* out, int H,
                   int W, uint64_t* dmax, void* s) {
  cudaStream_t st = STREAM(s);
  Scratch scr(st);
  SP_TRY(scr.alloc(sizeof(int) * 2 * (size_t)(m > 0 ? m : 1)));
  int* sy = (int*)scr.p;
  int* sx = sy + (m > 0 ? m : 1);
  SP_TRY(seeds_to_soa((const long long*)seeds, m, sy, sx, st));
  return dist2(labels, sy, sx, (long long*)out, (unsigned long long*)dmax, H, W, (int)m, st);
}

int sp_fs_dither(const double* dens, uint8_t* out, int H, int W, void* s) {
  return fs_dither(dens, out, H, W, STREAM(s));
}

int sp_assign_triangles(const int64_t* tris, long ntris, const int64_t* vy, const int64_t* vx,
                        int H, int W, int32_t* out, void* s) {
  return assign_tris<long long>((const long long*)tris, ntris, (const long long*)vy,
                                (const long long*)vx, H, W, out, true, STREAM(s));
}

int sp_fallback_assign(const int32_t* assign, const int32_t* labels, const int32_t* smt,
                       int32_t* out, int H, int W, void* s) {
  return fallback(assign, labels, smt, out, (size_t)H * W, STREAM(s));
}

int sp_reduce_cells(const int32_t* assign, const double* err, long ntris, double* sums,
                    int64_t* amax_idx, double* amax_val, int H, int W, void* s) {
  return reduce_cells(assign, err, ntris, sums, (long long*)amax_idx, amax_val, H, W,
                      STREAM(s));
}

// ---- B2: densification geometry workspace -------------------------------------

int sp_geo_create(void** out, int H, int W) {
  Geo* g = nullptr;
  SP_TRY(geo_create(&g, H, W));
  *out = g;
  return 0;
}

int sp_geo_destroy(void* g) {
  delete (Geo*)g;
  return 0;
}

int sp_geo_voronoi(void* g, const uint8_t* mask, double start_hint, long* m, double* max_radius,
                   int* nsteps, void* s) {
  return geo_voronoi((Geo*)g, mask, start_hint, m, max_radius, nsteps, STREAM(s));
}

int sp_geo_delaunay(void* g, long* ntris, void* s) {
  return geo_delaunay((Geo*)g, ntris, STREAM(s));
}

// seed count from which sp_geo_delaunay sorts wide (2 x 32-bit) triangle
// keys instead of packed 3 x 21-bit ones (default and maximum 2^21; v <= 0
// queries) -- lowered only to test the wide path on small images
long sp_geo_wide_threshold(long v) { return geo_wide_threshold(v); }

// programmatic dependent launch of the V-cycle kernels on levels >= v
// (v = -1: off; v < -1: read only); returns the setting
int sp_pdl_from_level(int v) { return sp::pdl_from_level(v); }

// accumulate implementation (A/B and tests): 1 = tile-binned rasteriser +
// bbox-order reduction (default), 0 = global atomics + pixel sort; v < 0 reads
int sp_geo_accumulate_mode(int v) { return sp::geo_accumulate_mode(v); }

int sp_geo_accumulate(void* g, const double* err, int voronoi, void* s) {
  return geo_accumulate((Geo*)g, err, voronoi, STREAM(s));
}

int sp_geo_select(void* g, uint8_t* mask, long nbuckets, long want, long* picked, void* s) {
  return geo_select((Geo*)g, mask, nbuckets, want, picked, STREAM(s));
}

int sp_geo_fill_highest_error(void* g, const double* err, uint8_t* mask, long want, void* s) {
  return fill_highest_error((Geo*)g, err, mask, want, STREAM(s));
}

// load caller-provided labels (H,W) i32 and seed rows sy/sx (m) i32 into the
// workspace (delaunay_from_voronoi / accumulate on user VoronoiLabels)
int sp_geo_load(void* gp, const int32_t* labels, const int32_t* sy, const int32_t* sx, long m,
                void* s) {
  Geo* g = (Geo*)gp;
  cudaStream_t st = STREAM(s);
  size_t n = (size_t)g->H * g->W;
  if (m < 0 || (size_t)m > n) { set_error("bad seed count %ld", m); return -2; }
  SP_CUDA(cudaMemcpyAsync(g->lab_a, labels, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  if (m) {
    SP_CUDA(cudaMemcpyAsync(g->sy, sy, sizeof(int) * m, cudaMemcpyDeviceToDevice, st));
    SP_CUDA(cudaMemcpyAsync(g->sx, sx, sizeof(int) * m, cudaMemcpyDeviceToDevice, st));
  }
  g->m = m;
  g->T = 0;
  return 0;
}

// ---- row-strip partition of the Delaunay step and the accumulate ------------
// (geometry.cu geo_corner_keys ...).  Row ranges are
// image rows [r0, r1); triangle ranges [t0, t1).

// sorted unique triangle keys of the corners in rows [r0, r1) (left in the
// workspace; sp_geo_keys_copy reads them out)
int sp_geo_corner_keys(void* g, int r0, int r1, long* nkeys, void* s) {
  return geo_corner_keys((Geo*)g, r0, r1, nkeys, STREAM(s));
}

int sp_geo_keys_copy(void* gp, uint64_t* dst, long n, void* s) {
  Geo* g = (Geo*)gp;
  if (n < 0 || (size_t)n > g->key_cap) { set_error("bad key count %ld", n); return -2; }
  if (n) SP_CUDA(cudaMemcpyAsync(dst, g->keys, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice,
                                 STREAM(s)));
  return 0;
}

// the triangles of the merged (concatenated) key lists of all strips
int sp_geo_delaunay_from_keys(void* g, const uint64_t* keys, long n, long* ntris, void* s) {
  return geo_delaunay_from_keys((Geo*)g, (const unsigned long long*)keys, n, ntris, STREAM(s));
}

// pixel -> triangle assignment of rows [r0, r1) only
int sp_geo_raster_rows(void* g, int r0, int r1, void* s) {
  return geo_raster_rows((Geo*)g, r0, r1, STREAM(s));
}

// assignment rows [r0, r1) to (dir 0) or from (dir 1) buf, int32 [r1-r0][W]
int sp_geo_assign_rows(void* gp, int32_t* buf, int r0, int r1, int dir, void* s) {
  Geo* g = (Geo*)gp;
  if (r0 < 0 || r1 > g->H || r1 < r0) { set_error("bad row range [%d, %d)", r0, r1); return -2; }
  const size_t off = (size_t)r0 * g->W, n = (size_t)(r1 - r0) * g->W;
  if (!n) return 0;
  if (dir == 0)
    SP_CUDA(cudaMemcpyAsync(buf, g->assign + off, sizeof(int) * n, cudaMemcpyDeviceToDevice,
                            STREAM(s)));
  else
    SP_CUDA(cudaMemcpyAsync(g->assign + off, buf, sizeof(int) * n, cudaMemcpyDeviceToDevice,
                            STREAM(s)));
  return 0;
}

// per-triangle sums / argmax of triangles [t0, t1) over the full assignment
int sp_geo_reduce_range(void* g, const double* err, long t0, long t1, void* s) {
  return geo_reduce_range((Geo*)g, err, t0, t1, STREAM(s));
}

// install bucket results [t0, t1) (the all-gathered ranges) for sp_geo_select
int sp_geo_set_buckets(void* gp, const double* sums, const int64_t* amax,
                       const double* amax_val, long t0, long t1, void* s) {
  Geo* g = (Geo*)gp;
  if (t0 < 0 || t1 < t0 || (size_t)t1 > g->tri_cap) { set_error("bad bucket range"); return -2; }
  const size_t n = (size_t)(t1 - t0);
  if (!n) return 0;
  cudaStream_t st = STREAM(s);
  SP_CUDA(cudaMemcpyAsync(g->sums + t0, sums, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaMemcpyAsync(g->amax + t0, amax, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaMemcpyAsync(g->amax_val + t0, amax_val, sizeof(double) * n,
                          cudaMemcpyDeviceToDevice, st));
  return 0;
}

// copies of the workspace state for the public API objects (any pointer may
// be NULL): labels (H,W) i32, seed rows sy/sx (m) i32, triangles (T,3) i32,
// bucket sums / argmax / argmax value (T, or m for the Voronoi partition)
int sp_geo_export(void* gp, int32_t* labels, int32_t* sy, int32_t* sx, int32_t* tris,
                  double* sums, int64_t* amax, double* amax_val, long nbuckets, void* s) {
  Geo* g = (Geo*)gp;
  cudaStream_t st = STREAM(s);
  size_t n = (size_t)g->H * g->W;
  if (labels) SP_CUDA(cudaMemcpyAsync(labels, g->lab_a, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  if (sy) SP_CUDA(cudaMemcpyAsync(sy, g->sy, sizeof(int) * g->m, cudaMemcpyDeviceToDevice, st));
  if (sx) SP_CUDA(cudaMemcpyAsync(sx, g->sx, sizeof(int) * g->m, cudaMemcpyDeviceToDevice, st));
  if (tris && g->T) SP_CUDA(cudaMemcpyAsync(tris, g->tris, sizeof(int) * 3 * g->T, cudaMemcpyDeviceToDevice, st));
  if (nbuckets > 0) {
    if (sums) SP_CUDA(cudaMemcpyAsync(sums, g->sums, sizeof(double) * nbuckets, cudaMemcpyDeviceToDevice, st));
    if (amax) SP_CUDA(cudaMemcpyAsync(amax, g->amax, sizeof(int64_t) * nbuckets, cudaMemcpyDeviceToDevice, st));
    if (amax_val) SP_CUDA(cudaMemcpyAsync(amax_val, g->amax_val, sizeof(double) * nbuckets, cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

}  // extern "C"

// ---- tracing: ORAS local-solve statistics -----------------------------------
namespace sp {
int oras_stats(int enable, unsigned long long* out);
}
extern "C" int sp_stats(int enable, uint64_t* out) {
  // enable: 1 = reset + start, 0 = reset + stop, -1 = read only.  out (HOST,
  // may be NULL) receives {ORAS jobs, local CG iterations, jobs converged on
  // entry, 0} accumulated since the last reset
  return sp::oras_stats(enable, (unsigned long long*)out);
}

namespace sp {
int oras_variant(int v);
}
// select the float ORAS kernel for blocks <= 32x32: 1 = warp per job
// (default), 0 = CTA per job; v < 0 only queries.  Returns the current value.
extern "C" int sp_oras_variant(int v) { return sp::oras_variant(v); }

namespace sp {
int march_default(int v);
}
extern "C" int sp_march_variant(int v) { return sp::march_default(v); }
extern "C" int sp_ws_variant(int v) { return sp::ws_variant(v); }
extern "C" int sp_ws_prefetch(int v) { return sp::ws_prefetch(v); }
extern "C" int sp_ws_stages(int v) { return sp::ws_stages(v); }
extern "C" int sp_oras_offbits(int v) { return sp::oras_offbits(v); }
namespace sp { int tile_list(int v); }
extern "C" int sp_tile_list(int v) { return sp::tile_list(v); }
namespace sp { int jfa_short4(int v); }
extern "C" int sp_jfa_short4(int v) { return sp::jfa_short4(v); }
namespace sp { long tma_min_pixels(long v); }
extern "C" long sp_tma_min_pixels(long v) { return sp::tma_min_pixels(v); }
namespace sp { int fused_bnorm(int v); }
extern "C" int sp_fused_bnorm(int v) { return sp::fused_bnorm(v); }
extern "C" int sp_blend_packed(int v) { return sp::blend_packed(v); }
namespace sp { int tile_fused(int v); int channel_parallel(int v); int graph_loop(int v); }
extern "C" int sp_tile_fused(int v) { return sp::tile_fused(v); }
extern "C" int sp_channel_parallel(int v) { return sp::channel_parallel(v); }
extern "C" int sp_graph_loop(int v) { return sp::graph_loop(v); }

// ---- dithered initial mask (spatial.py:107-148) -------------------------------
namespace sp {
int density_map(const double* f, int C, int H, int W, double density, const double* gauss_h,
                int radius, double* dens, double* total_out, cudaStream_t s);
int init_mask_random(const double* f, int C, int H, int W, long target, double density,
                     const double* gauss_h, int radius, const uint64_t* pcg_h, uint8_t* mask,
                     int* degenerate, cudaStream_t s);
int pcg_doubles(const uint64_t* pcg_h, long long start, long long count, double* out,
                cudaStream_t s);
int pairwise_sum(const double* a, long long n, double* out, cudaStream_t s);

}

extern "C" {
int sp_density_map(const double* f, int C, int H, int W, double density, const double* gauss_h,
                   int radius, double* dens, double* total_h, void* s) {
  return sp::density_map(f, C, H, W, density, gauss_h, radius, dens, total_h, STREAM(s));
}

int sp_init_mask_random(const double* f, int C, int H, int W, long target, double density,
                        const double* gauss_h, int radius, const uint64_t* pcg_h, uint8_t* mask,
                        int* degenerate_h, void* s) {
  return sp::init_mask_random(f, C, H, W, target, density, gauss_h, radius, pcg_h, mask,
                              degenerate_h, STREAM(s));
}

int sp_pcg64_doubles(const uint64_t* pcg_h, long long start, long long count, double* out,
                     void* s) {
  return sp::pcg_doubles(pcg_h, start, count, out, STREAM(s));
}

int sp_pairwise_sum(const double* a, long long n, double* out_h, void* s) {
  return sp::pairwise_sum(a, n, out_h, STREAM(s));
}
}  // extern "C"

// ---- B2: row-strip partitioned solve (strips.cu) -----------------
namespace sp {
struct StripGroup;
int strip_create(StripGroup** out, int C, int H, int W, const HierCfg& cfg, int P, int nloc,
                 int first, int La, int halo, const int* o0, const int* o1, void* comm);
void strip_destroy(StripGroup* g);
int strip_set_mask(StripGroup* g, const uint8_t* mask, const float* values, cudaStream_t s);
int strip_solve(StripGroup* g, const float* bsym, float* u_io, int init_mode, double tol,
                int cycles, int max_cycles, cudaStream_t s, SolveReport* rep);
int strip_levels(StripGroup* g, int* nlev, int* dims, int cap);
int strip_set_host_transport(StripGroup* g, const HostTransport& t);
int nccl_unique_id(uint8_t* out);
int nccl_comm_create(void** comm, const uint8_t* id_bytes, int nranks, int rank);
int nccl_comm_destroy(void* comm);
}  // namespace sp

extern "C" {
int sp_nccl_unique_id(uint8_t* out128) { return sp::nccl_unique_id(out128); }
int sp_nccl_comm_create(void** comm, const uint8_t* id128, int nranks, int rank) {
  return sp::nccl_comm_create(comm, id128, nranks, rank);
}
int sp_nccl_comm_destroy(void* comm) { return sp::nccl_comm_destroy(comm); }

int sp_strip_create(void** out, int C, int H, int W, int block, int overlap, int levels,
                    int pre, int post, double alpha, double rho, int P, int nloc, int first,
                    int La, int halo, const int* o0_h, const int* o1_h, void* comm) {
  HierCfg cfg;
  cfg.block = block;
  cfg.overlap = overlap;
  cfg.levels = levels;
  cfg.pre = pre;
  cfg.post = post;
  cfg.alpha = alpha;
  cfg.rho = rho;
  return sp::strip_create((sp::StripGroup**)out, C, H, W, cfg, P, nloc, first, La, halo, o0_h,
                          o1_h, comm);
}
int sp_strip_destroy(void* g) {
  sp::strip_destroy((sp::StripGroup*)g);
  return 0;
}
int sp_strip_set_mask(void* g, const uint8_t* mask, const void* values, void* s) {
  return sp::strip_set_mask((sp::StripGroup*)g, mask, (const float*)values, STREAM(s));
}
int sp_strip_solve(void* g, const void* bsym, void* u, int init_mode, double tol, int cycles,
                   int max_cycles, sp_solve_report* rep, void* s) {
  return sp::strip_solve((sp::StripGroup*)g, (const float*)bsym, (float*)u, init_mode, tol,
                         cycles, max_cycles, STREAM(s), (sp::SolveReport*)rep);
}
int sp_strip_levels(void* g, int* nlev, int* dims, int cap) {
  return sp::strip_levels((sp::StripGroup*)g, nlev, dims, cap);
}
int sp_strip_set_host_transport(void* g, void* sendrecv, void* allreduce_f64, void* bcast,
                                void* user) {
  sp::HostTransport t;
  t.sendrecv = (decltype(t.sendrecv))sendrecv;
  t.allreduce_f64 = (decltype(t.allreduce_f64))allreduce_f64;
  t.bcast = (decltype(t.bcast))bcast;
  t.user = user;
  return sp::strip_set_host_transport((sp::StripGroup*)g, t);
}
}  // extern "C"

// ---- measurement hooks (bench.py) ---------------------------------------------
#include <atomic>
namespace sp {
static std::atomic<long long> g_launches{0};
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// finest-level pixel x V-cycle work of every solve (Mpixel-iterations)
static std::atomic<long long> g_work[2]{{0}, {0}};
void count_work(int kind, long long px_cycles) {
  g_work[kind & 1].fetch_add(px_cycles, std::memory_order_relaxed);
}
int hier_bench(Hier* h, int which, int reps, cudaStream_t s, double* ms, double* bytes);
int hier_residual_out(Hier* h, int lv, void* r_out, double* norms_out, cudaStream_t s);
}  // namespace sp

extern "C" {
// kernels launched by the library since the last reset (reset != 0 zeroes it)
long long sp_launch_count(int reset) {
  long long v = sp::g_launches.load();
  if (reset) sp::g_launches.store(0);
  return v;
}

// finest-level pixel-V-cycles of the solves since the last reset: kind 0 =
// image-level solves (one hierarchy per image / strip group), kind 1 =
// batched block-local solves (RAS 64x64 products)
long long sp_work_count(int kind, int reset) {
  long long v = sp::g_work[kind & 1].load();
  if (reset) sp::g_work[kind & 1].store(0);
  return v;
}

// mean time (ms, CUDA events on `stream`) of `reps` launches of a finest-level
// kernel of the hierarchy (0 residual, 1 ORAS local CG, 2 ORAS blend, 3
// residual+restriction) and its algorithmic bytes per launch
int sp_hier_bench(void* h, int which, int reps, double* ms_h, double* bytes_h, void* s) {
  return sp::hier_bench((sp::Hier*)h, which, reps, (cudaStream_t)s, ms_h, bytes_h);
}

// residual (r, per-plane sum r^2) of level lv's current iterate with the
// hierarchy's sweep kernel, into device buffers
int sp_hier_residual(void* h, int lv, void* r_out, double* norms_out, void* s) {
  return sp::hier_residual_out((sp::Hier*)h, lv, r_out, norms_out, (cudaStream_t)s);
}
}  // extern "C"
