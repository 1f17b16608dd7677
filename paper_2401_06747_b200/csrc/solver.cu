// solver.cu -- device-resident multigrid-ORAS hierarchy (native runtime).
//
// Reference: solver.py:205-372 (GridHierarchy build / _smooth / _vcycle /
// _cascade / solve_sym).  The whole level pyramid (masks, iterates,
// right-hand sides, residuals, ORAS corrections) lives in HBM and is reused
// across mask changes of the same geometry.  A V-cycle is recorded once into
// a CUDA graph and replayed; the only host synchronisation in a solve is the
// read-back of the per-channel residual norms for the tolerance test
// (solver.py:358-368), one small copy per V-cycle.
//
// A hierarchy holds `ntile` independent problems of the same shape (each
// with its own mask): ntile = 1 is the global image; the RAS tonal
// optimizer solves all of its 64x64 block-local systems as one batch
// (tonal.py:343-354, 120-131).  Each tile keeps its own stopping decision:
// tiles that have converged are switched off through a device flag array
// that every kernel of the (graph-captured) V-cycle reads.
#include <cmath>
#include <cstring>
#include <vector>

#include "kernels.cuh"
#include "solver.cuh"

namespace sp {

// one-image tolerance solves take ||b~||^2 from the masked_sym_rhs pass (1)
// or from a separate reduction of b~ (0): sp_fused_bnorm
static int fused_bnorm_on = 1;
int fused_bnorm(int v) {
  if (v >= 0) fused_bnorm_on = v;
  return fused_bnorm_on;
}

// sweep kernels of new hierarchies (sp_march_variant): 2 = TMA-staged
// residual sweeps (default), 1 = row-marching register kernels, 0 = the
// per-pixel kernels everywhere.  The row-strip solver always uses the
// row-marching kernels (their band-norm mode).
int march_default(int v) {
  static int on = 2;
  if (v >= 0) on = v;
  return on;
}

// covering tables for sorted block starts (host)
void cover_tables(const std::vector<int>& starts, int size, int dim, std::vector<int>& k0,
                  std::vector<int>& n) {
  k0.assign(dim, 0);
  n.assign(dim, 0);
  for (int y = 0; y < dim; ++y) {
    int first = -1, cnt = 0;
    for (size_t k = 0; k < starts.size(); ++k) {
      if (starts[k] <= y && y < starts[k] + size) {
        if (first < 0) first = (int)k;
        ++cnt;
      }
    }
    k0[y] = first < 0 ? 0 : first;
    n[y] = cnt;
  }
}

static int dalloc(void** p, size_t bytes) {
  *p = nullptr;
  if (!bytes) return 0;
  SP_CUDA(cudaMalloc(p, bytes));
  return 0;
}

Hier::~Hier() {
  if (!owner) return;  // a channel view: the buffers belong to its parent
  for (Hier* v : chv) delete v;
  for (cudaStream_t st : ch_streams) cudaStreamDestroy(st);
  for (cudaEvent_t ev : ch_events) cudaEventDestroy(ev);
  if (up_ev) cudaEventDestroy(up_ev);
  if (loop_exec) cudaGraphExecDestroy(loop_exec);
  if (loop_ctl) cudaFree(loop_ctl);
  if (h_loop) cudaFreeHost(h_loop);
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  if (cap_stream) cudaStreamDestroy(cap_stream);
  for (auto& L : lv) {
    for (void* p : {(void*)L.mask, L.values, L.u, L.b, L.r, L.corr, L.weights, (void*)L.partial,
                    (void*)L.counter, (void*)L.norms, (void*)L.ys, (void*)L.xs,
                    (void*)L.row_k0, (void*)L.row_n, (void*)L.col_k0, (void*)L.col_n,
                    (void*)L.wdelta, (void*)L.offbits, (void*)L.rowinfo, (void*)L.colinfo})
      if (p) cudaFree(p);
  }
  if (d_active) cudaFree(d_active);
  if (d_scratch) cudaFree(d_scratch);
  if (d_list) cudaFree(d_list);
  if (h_list) cudaFreeHost(h_list);
  if (list_ev) cudaEventDestroy(list_ev);
  if (h_norms) cudaFreeHost(h_norms);
  if (h_active) cudaFreeHost(h_active);
}

int hier_create(Hier** out, int dtype, int C, int H, int W, const HierCfg& cfg,
                int with_values, int ntile) {
  *out = nullptr;
  if (H < 1 || W < 1 || C < 1 || ntile < 1) {
    set_error("bad hierarchy shape (%d tiles, %d, %d, %d)", ntile, C, H, W);
    return -2;
  }
  if ((long)ntile * C > 65535) {
    set_error("at most 65535 tile-channels per hierarchy (got %d x %d)", ntile, C);
    return -2;
  }
  if (cfg.block < cfg.overlap + 2 || cfg.overlap < 1) {
    set_error("block size must be at least overlap + 2");
    return -2;
  }
  if (tma_ok(64, 128, 1) && tma_prepare()) return -1;
  Hier* h = new Hier();
  h->sweep = march_default(-1);
  h->dtype = dtype;
  h->C = C;
  h->ntile = ntile;
  h->cfg = cfg;
  h->gamma = (1.0 - cfg.alpha) / (1.0 + cfg.alpha);
  const size_t es = dtype == SP_F64 ? 8 : 4;
  const size_t ntc = (size_t)ntile * C;
  int hh = H, ww = W, level = 0;
  while (true) {
    Level L{};
    L.H = hh;
    L.W = ww;
    L.bh = std::min(cfg.block, hh);
    L.bw = std::min(cfg.block, ww);
    int stride = cfg.block - cfg.overlap;
    L.nby = num_starts(hh, L.bh, stride);
    L.nbx = num_starts(ww, L.bw, stride);
    std::vector<int> ys(L.nby), xs(L.nbx);
    for (int k = 0; k < L.nby; ++k) ys[k] = block_start(k, stride, hh, L.bh);
    for (int k = 0; k < L.nbx; ++k) xs[k] = block_start(k, stride, ww, L.bw);
    std::vector<int> rk0, rn, ck0, cn;
    cover_tables(ys, L.bh, hh, rk0, rn);
    cover_tables(xs, L.bw, ww, ck0, cn);
    // solver.py:262-264: tau_c = rho * (bh*bw / N) * ||r_c||^2, cap = bh*bw
    L.tau_scale = cfg.rho * ((double)(L.bh * L.bw) / (double)((long)hh * ww));
    size_t plane = (size_t)hh * ww, nb = (size_t)L.nby * L.nbx;
    size_t vec = es * ntc * plane;
    int rc = 0;
    rc |= dalloc((void**)&L.mask, plane * ntile);
    rc |= dalloc(&L.u, vec);
    rc |= dalloc(&L.b, vec);
    rc |= dalloc(&L.r, vec);
    rc |= dalloc(&L.corr, es * ntc * nb * L.bh * L.bw);
    rc |= dalloc(&L.weights, es * nb * L.bh * L.bw);
    if (with_values) rc |= dalloc(&L.values, vec);
    L.npart = residual_partials(hh, ww);
    rc |= dalloc((void**)&L.partial, sizeof(double) * ntc * L.npart);
    rc |= dalloc((void**)&L.counter, sizeof(unsigned) * ntc);
    rc |= dalloc((void**)&L.norms, sizeof(double) * ntc);
    rc |= dalloc((void**)&L.ys, sizeof(int) * L.nby);
    rc |= dalloc((void**)&L.xs, sizeof(int) * L.nbx);
    rc |= dalloc((void**)&L.row_k0, sizeof(int) * hh);
    rc |= dalloc((void**)&L.row_n, sizeof(int) * hh);
    rc |= dalloc((void**)&L.col_k0, sizeof(int) * ww);
    rc |= dalloc((void**)&L.col_n, sizeof(int) * ww);
    L.wdelta = nullptr;
    if (dtype != SP_F64) rc |= dalloc((void**)&L.wdelta, sizeof(int) * nb);
    L.offbits = nullptr;
    if (dtype != SP_F64 && L.bh <= 32 && L.bw <= 32)
      rc |= dalloc((void**)&L.offbits, sizeof(uint32_t) * 32 * nb * ntile);
    std::vector<int> rinfo, cinfo;
    L.rowinfo = L.colinfo = nullptr;
    L.pair_cols = ww % 2 == 0;
    for (int x0 : xs) L.pair_cols = L.pair_cols && x0 % 2 == 0;
    if (dtype != SP_F64 && L.bh == 32 && L.bw == 32 && blend_pack(ys, 32, hh, rinfo) &&
        blend_pack(xs, 32, ww, cinfo)) {
      rc |= dalloc((void**)&L.rowinfo, sizeof(int) * hh);
      rc |= dalloc((void**)&L.colinfo, sizeof(int) * ww);
    }
    h->lv.push_back(L);
    if (rc) { delete h; return -1; }
    Level& B = h->lv.back();
    if (cudaMemset(B.counter, 0, sizeof(unsigned) * ntc) != cudaSuccess ||
        cudaMemcpy(B.ys, ys.data(), sizeof(int) * B.nby, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(B.xs, xs.data(), sizeof(int) * B.nbx, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(B.row_k0, rk0.data(), sizeof(int) * hh, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(B.row_n, rn.data(), sizeof(int) * hh, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(B.col_k0, ck0.data(), sizeof(int) * ww, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(B.col_n, cn.data(), sizeof(int) * ww, cudaMemcpyHostToDevice) != cudaSuccess ||
        (B.rowinfo && cudaMemcpy(B.rowinfo, rinfo.data(), sizeof(int) * hh,
                                 cudaMemcpyHostToDevice) != cudaSuccess) ||
        (B.colinfo && cudaMemcpy(B.colinfo, cinfo.data(), sizeof(int) * ww,
                                 cudaMemcpyHostToDevice) != cudaSuccess)) {
      set_error("hierarchy upload failed");
      delete h;
      return -1;
    }
    int wrc = dtype == SP_F64
                  ? block_weights_launch<double>((double*)B.weights, B.ys, B.xs, B.row_k0,
                                                 B.row_n, B.col_k0, B.col_n, B.nby, B.nbx,
                                                 B.bh, B.bw, hh, ww, cfg.overlap, 0)
                  : block_weights_launch<float>((float*)B.weights, B.ys, B.xs, B.row_k0,
                                                B.row_n, B.col_k0, B.col_n, B.nby, B.nbx,
                                                B.bh, B.bw, hh, ww, cfg.overlap, 0);
    if (!wrc && B.wdelta)
      wrc = weight_aliases((const float*)B.weights, B.nby, B.nbx, B.bh, B.bw, B.wdelta, 0);
    if (wrc || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("partition-of-unity weights failed");
      delete h;
      return -1;
    }
    ++level;
    // solver.py:238-243: auto levels coarsen until max(h, w) <= block
    if (cfg.levels > 0) {
      if (level >= cfg.levels || std::max(hh, ww) <= 2) break;
    } else if (std::max(hh, ww) <= cfg.block) {
      break;
    }
    hh = (hh + 1) / 2;
    ww = (ww + 1) / 2;
  }
  // reduction partials: 1024 per tile (4096 for one image: the fused
  // ||b~||^2 of masked_sym_rhs), the norms and a counter behind them
  const size_t nslot = ntile == 1 ? 4096 : 1024;
  size_t scratch = sizeof(double) * (nslot + 8) * (size_t)ntile + 256;
  if (cudaMallocHost((void**)&h->h_norms, sizeof(double) * ntc) != cudaSuccess ||
      cudaMallocHost((void**)&h->h_active, sizeof(int) * ntile) != cudaSuccess ||
      cudaMallocHost(&h->h_loop, 4096) != cudaSuccess ||
      cudaMalloc((void**)&h->d_active, sizeof(int) * ntile) != cudaSuccess ||
      cudaMalloc(&h->d_scratch, scratch) != cudaSuccess) {
    set_error("hierarchy bookkeeping alloc failed");
    delete h;
    return -1;
  }
  *out = h;
  return 0;
}

// ---------------------------------------------------------------------------

template <typename T>
static int set_mask_t(Hier* h, const uint8_t* mask, const T* values, cudaStream_t s) {
  Level& L0 = h->lv[0];
  size_t plane = (size_t)L0.H * L0.W * h->ntile;
  SP_CUDA(cudaMemcpyAsync(L0.mask, mask, plane, cudaMemcpyDeviceToDevice, s));
  bool vals = values != nullptr && L0.values != nullptr;
  if (vals)
    SP_CUDA(cudaMemcpyAsync(L0.values, values, sizeof(T) * h->C * plane,
                            cudaMemcpyDeviceToDevice, s));
  for (size_t i = 1; i < h->lv.size(); ++i) {
    Level& F = h->lv[i - 1];
    Level& G = h->lv[i];
    SP_TRY(restrict_mask<T>(F.mask, vals ? (const T*)F.values : nullptr, G.mask,
                            vals ? (T*)G.values : nullptr, h->C, F.H, F.W, s, h->ntile));
  }
  for (Level& L : h->lv)
    if (L.offbits)
      SP_TRY(oras_offbits_launch(L.mask, L.ys, L.xs, L.nby, L.nbx, L.bh, L.bw, L.H, L.W,
                                 h->ntile, L.offbits, s));
  h->has_values = vals;
  return 0;
}

int hier_set_mask(Hier* h, const uint8_t* mask, const void* values, cudaStream_t s) {
  if (h->dtype == SP_F64) return set_mask_t<double>(h, mask, (const double*)values, s);
  return set_mask_t<float>(h, mask, (const float*)values, s);
}

// ---- V-cycle ----------------------------------------------------------------

// the level sweeps on wide float levels: TMA-staged kernels (mgtma.cu,
// sweep variant 2, default), row-marching register kernels (mgfast.cu, 1),
// or the per-pixel reference-exact kernels (mg.cu, 0 -- also every narrow or
// double level).  All three are bit-identical per element.
template <typename T>
static bool aligned_level(const Level& L) {
  return (((uintptr_t)L.u | (uintptr_t)L.b | (uintptr_t)L.r | (uintptr_t)L.mask) & 15u) == 0;
}
// levels below this many pixels per plane take the per-pixel sweep kernels
// instead of the TMA ones (whose fixed start-up -- descriptor prefetch,
// barrier init, the one-wave grid's partial sums -- dominates a small
// plane): sp_tma_min_pixels.  300,000: at 4K the levels from 270 x 480 down
// (ws residual 6.9-9.5 us vs 4.3 us per-pixel); warm V-cycle 0.971 ->
// 0.951 ms, pipeline -2 ms (probe_perf.py / probe_switch.py)
static long tma_min_px = 300000;
long tma_min_pixels(long v) {
  if (v >= 0) tma_min_px = v;
  return tma_min_px;
}

template <typename T>
static bool use_tma(const Hier* h, const Level& L) {
  return sizeof(T) == 4 && h->sweep == 2 && (long)L.H * L.W >= tma_min_px &&
         tma_ok(L.H, L.W, L.npart) && aligned_level<T>(L);
}
template <typename T>
static bool use_march(const Hier* h, const Level& L) {
  return sizeof(T) == 4 && h->sweep == 1 && march_ok(L.H, L.W, L.npart) && aligned_level<T>(L);
}

template <typename T>
static int residual_lv(Hier* h, int lv, bool with_norms, cudaStream_t s) {
  Level& L = h->lv[lv];
  if (use_tma<T>(h, L))
    return resid_tma((const float*)L.u, (const float*)L.b, L.mask, (float*)L.r, L.partial,
                     L.counter, with_norms ? L.norms : nullptr, h->C, L.H, L.W, s, h->ntile,
                     h->d_active, nullptr, 0, 0, 0, L.npart);
  if (use_march<T>(h, L))
    return resid_march((const float*)L.u, (const float*)L.b, L.mask, (float*)L.r, L.partial,
                       L.counter, with_norms ? L.norms : nullptr, h->C, L.H, L.W, s, h->ntile,
                       h->d_active);
  return residual<T>((const T*)L.u, (const T*)L.b, L.mask, (T*)L.r, L.partial, L.counter,
                     with_norms ? L.norms : nullptr, h->C, L.H, L.W, 1.0, s, h->ntile,
                     h->d_active);
}

template <typename T>
static int residual_restrict_lv(Hier* h, int lv, cudaStream_t s) {
  Level& F = h->lv[lv];
  Level& G = h->lv[lv + 1];
  if (use_tma<T>(h, F))
    return resid_restrict_tma((const float*)F.u, (const float*)F.b, F.mask, (float*)G.r, h->C,
                              F.H, F.W, s, h->ntile, h->d_active);
  if (use_march<T>(h, F))
    return resid_restrict_march((const float*)F.u, (const float*)F.b, F.mask, (float*)G.r,
                                h->C, F.H, F.W, s, h->ntile, h->d_active);
  return residual_restrict<T>((const T*)F.u, (const T*)F.b, F.mask, (T*)G.r, h->C, F.H, F.W,
                              1.0, s, h->ntile, h->d_active);
}

template <typename T>
int prolong_lv(Hier* h, int lv, int add, cudaStream_t s) {
  Level& F = h->lv[lv];
  Level& G = h->lv[lv + 1];
  if (sizeof(T) == 4 && h->sweep == 2 && (long)F.H * F.W >= tma_min_px &&
      tma_prolong_ok(F.H, F.W) && aligned_level<T>(F))
    return prolong_tma((const float*)G.u, (float*)F.u, (const float*)F.b, F.mask, h->C, G.H,
                       G.W, F.H, F.W, add, s, h->ntile, h->d_active);
  if (use_march<T>(h, F))
    return prolong_march((const float*)G.u, (float*)F.u, (const float*)F.b, F.mask, h->C, G.H,
                         G.W, F.H, F.W, add, s, h->ntile, h->d_active);
  return prolong_enforce<T>((const T*)G.u, (T*)F.u, (const T*)F.b, F.mask, h->C, G.H, G.W, F.H,
                            F.W, add, s, h->ntile, h->d_active);
}

template <typename T>
static int oras_lv(Hier* h, Level& L, cudaStream_t s) {
  return oras_local_launch<T>((const T*)L.r, L.mask, L.norms, L.tau_scale, L.ys, L.xs, L.nby,
                              L.nbx, L.bh, L.bw, L.H, L.W, h->C, h->gamma, (long)L.bh * L.bw,
                              1.0, (const T*)L.weights, (T*)L.corr, s, h->ntile, h->d_active,
                              h->cfg.block - h->cfg.overlap, 0, 0, L.wdelta, L.offbits);
}

// u += the level's weighted block corrections (block order)
template <typename T>
static int blend_lv(Hier* h, Level& L, T* u, cudaStream_t s) {
  return oras_blend_launch<T>(u, (const T*)L.corr, L.ys, L.xs, L.row_k0, L.row_n, L.col_k0,
                              L.col_n, L.nby, L.nbx, L.bh, L.bw, L.H, L.W, h->C, s, h->ntile,
                              h->d_active, 0, 0, L.rowinfo, L.colinfo, L.pair_cols);
}

template <typename T>
int smooth_lv(Hier* h, int lv, int sweeps, bool first_done, cudaStream_t s) {
  Level& L = h->lv[lv];
  for (int sw = 0; sw < sweeps; ++sw) {
    if (!(sw == 0 && first_done)) SP_TRY(residual_lv<T>(h, lv, true, s));
    SP_TRY(oras_lv<T>(h, L, s));
    SP_TRY(blend_lv<T>(h, L, (T*)L.u, s));
  }
  return 0;
}

// programmatic dependent launch for the V-cycle kernels of the levels
// >= pdl_from (the launch-latency-bound small levels); < 0: off
static int pdl_from = -1;  // measured neutral on the 4K pipeline (probe_pdl.py): off
int pdl_from_level(int v) {
  if (v >= -1) pdl_from = v;
  return pdl_from;
}

// solver.py:283-300; `first_done`: level lv's residual r/norms for the
// current u are already in place (computed by the caller's tolerance check)
template <typename T>
int vcycle_lv(Hier* h, int lv, bool first_done, cudaStream_t s) {
  const HierCfg& cfg = h->cfg;
  int last = (int)h->lv.size() - 1;
  const bool pdl = pdl_from >= 0 && lv >= pdl_from;
  struct Restore {
    ~Restore() { pdl_set(false); }
  } restore;
  pdl_set(pdl);
  if (lv == last) return smooth_lv<T>(h, lv, cfg.pre + cfg.post, first_done, s);
  SP_TRY(smooth_lv<T>(h, lv, cfg.pre, first_done, s));
  Level& F = h->lv[lv];
  Level& G = h->lv[lv + 1];
  SP_TRY(residual_restrict_lv<T>(h, lv, s));
  SP_TRY(sym_rhs<T>((const T*)G.r, G.mask, (T*)G.b, (T*)G.u, h->C, G.H, G.W, 1.0, s,
                    h->ntile, h->d_active));
  SP_TRY(vcycle_lv<T>(h, lv + 1, false, s));
  pdl_set(pdl);
  SP_TRY(prolong_lv<T>(h, lv, 1, s));
  SP_TRY(smooth_lv<T>(h, lv, cfg.post, false, s));
  return 0;
}

// Channel-parallel V-cycles.  The C channels of an image are C independent
// systems through a whole V-cycle (shared mask, per-channel norms and ORAS
// thresholds; only the solve's tolerance test sums them), so the captured
// graph runs them as C parallel branches: the compute-bound ORAS local CG of
// one channel overlaps the HBM-bound sweeps of another, and the
// launch-latency-bound coarse levels of the channels run side by side.
// Every kernel is launched on a one-channel view that aliases the parent's
// buffers at the channel's offset (results are identical: the kernels are
// per plane and the per-plane reduction partials keep their slots).
// Measured slower on the 4K RGB pipeline (335 vs 305 ms): the one-channel
// launches lose the channel-fused kernels' amortised index work (the blend
// gathers each pixel's covering blocks once for all C channels) and the
// branches' ORAS launches mostly collide rather than interleave.  Off by
// default (sp_channel_parallel), kept as a measured A/B option.
static int channel_parallel_on = 0;
int channel_parallel(int v) {
  if (v >= 0) channel_parallel_on = v;
  return channel_parallel_on;
}

static int make_channel_views(Hier* h) {
  const size_t es = h->dtype == SP_F64 ? 8 : 4;
  for (int c = 0; c < h->C; ++c) {
    Hier* v = new Hier();
    v->owner = false;
    v->dtype = h->dtype;
    v->C = 1;
    v->ntile = 1;
    v->cfg = h->cfg;
    v->gamma = h->gamma;
    v->has_values = h->has_values;
    v->use_graphs = false;
    v->sweep = h->sweep;
    v->h_norms = h->h_norms;
    v->h_active = h->h_active;
    v->d_active = h->d_active;
    v->d_scratch = h->d_scratch;
    for (const Level& P : h->lv) {
      Level L = P;
      const size_t plane = (size_t)P.H * P.W, nbp = (size_t)P.nby * P.nbx * P.bh * P.bw;
      auto off = [&](void* p, size_t n) { return p ? (void*)((char*)p + c * n * es) : p; };
      L.u = off(P.u, plane);
      L.b = off(P.b, plane);
      L.r = off(P.r, plane);
      L.values = off(P.values, plane);
      L.corr = off(P.corr, nbp);
      L.partial = P.partial + (size_t)c * P.npart;
      L.counter = P.counter + c;
      L.norms = P.norms + c;
      v->lv.push_back(L);
    }
    h->chv.push_back(v);
    cudaStream_t st;
    cudaEvent_t ev;
    SP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    SP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    h->ch_streams.push_back(st);
    h->ch_events.push_back(ev);
  }
  cudaEvent_t fork;
  SP_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  h->ch_events.push_back(fork);  // the last event forks the branches
  return 0;
}

template <typename T>
static int vcycle_channels(Hier* h, cudaStream_t cap) {
  if (h->chv.empty()) SP_TRY(make_channel_views(h));
  cudaEvent_t fork = h->ch_events.back();
  SP_CUDA(cudaEventRecord(fork, cap));
  for (int c = 0; c < h->C; ++c) {
    SP_CUDA(cudaStreamWaitEvent(h->ch_streams[c], fork, 0));
    SP_TRY(vcycle_lv<T>(h->chv[c], 0, true, h->ch_streams[c]));
    SP_CUDA(cudaEventRecord(h->ch_events[c], h->ch_streams[c]));
    SP_CUDA(cudaStreamWaitEvent(cap, h->ch_events[c], 0));
  }
  return 0;
}

template <typename T>
static int run_vcycle(Hier* h, cudaStream_t s) {
  // precondition: level-0 r/norms are current (residual_lv(0) ran)
  if (!h->use_graphs) return vcycle_lv<T>(h, 0, true, s);
  if (!h->graph_exec) {
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on `s`
    if (!h->cap_stream) SP_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g;
    SP_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    const bool par = channel_parallel_on && h->C > 1 && h->ntile == 1 && h->C <= 8;
    int rc = par ? vcycle_channels<T>(h, h->cap_stream) : vcycle_lv<T>(h, 0, true, h->cap_stream);
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc) { if (e == cudaSuccess) cudaGraphDestroy(g); return rc; }
    SP_CUDA(e);
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    h->graph_nodes = (long long)nn;
    cudaError_t ie = cudaGraphInstantiate(&h->graph_exec, g, 0);
    cudaGraphDestroy(g);
    SP_CUDA(ie);
  }
  SP_CUDA(cudaGraphLaunch(h->graph_exec, s));
  count_launches(h->graph_nodes);
  return 0;
}

template <typename T>
static int cascade_t(Hier* h, cudaStream_t s) {
  int last = (int)h->lv.size() - 1;
  const int nt = h->ntile;
  Level& Lc = h->lv[last];
  // solver.py:302-317: coarsest: u = 0, b = level rhs, enforce, smooth 1
  SP_TRY(masked_sym_rhs<T>((const T*)Lc.values, Lc.mask, (T*)Lc.b, h->C, Lc.H, Lc.W, s, nt,
                           h->d_active));
  SP_TRY(enforce<T>((T*)Lc.u, (const T*)Lc.b, Lc.mask, h->C, Lc.H, Lc.W, 1, s, nt,
                    h->d_active));
  SP_TRY(smooth_lv<T>(h, last, 1, false, s));
  for (int lv = last - 1; lv >= 0; --lv) {
    Level& F = h->lv[lv];
    Level& G = h->lv[lv + 1];
    SP_TRY(masked_sym_rhs<T>((const T*)F.values, F.mask, (T*)F.b, h->C, F.H, F.W, s, nt,
                             h->d_active));
    SP_TRY(prolong_lv<T>(h, lv, 0, s));
    SP_TRY(smooth_lv<T>(h, lv, 1, false, s));
  }
  return 0;
}

int upload_active(Hier* h, cudaStream_t s) {
  if (!h->up_ev) SP_CUDA(cudaEventCreateWithFlags(&h->up_ev, cudaEventDisableTiming));
  SP_CUDA(cudaMemcpyAsync(h->d_active, h->h_active, sizeof(int) * h->ntile,
                          cudaMemcpyHostToDevice, s));
  SP_CUDA(cudaEventRecord(h->up_ev, s));
  return 0;
}

// waits for the last upload from h_active only, not for all queued work
int active_host_ready(Hier* h) {
  if (h->up_ev) SP_CUDA(cudaEventSynchronize(h->up_ev));
  return 0;
}

// ---- device-driven tolerance loop --------------------------------------------
// solver.py:351-369 without a host round trip per V-cycle: the stop test
// (relative residual over the channels, tolerance, cycle cap) runs in a
// one-thread kernel that sets the conditions of a WHILE node (continue the
// loop) and of an IF node (run the V-cycle + residual of this iteration).
// The whole solve is one graph launch; the host reads the iteration record
// (count, converged flag, relative residual history) once at the end.
// Measured equal to the host-driven loop on the 4K pipeline (300.7 vs
// 300.5 ms: the host turnaround it removes is offset by the conditional
// nodes' own scheduling), and CUPTI-based profilers do not list the
// kernels of conditional bodies, so it is off by default (sp_graph_loop).
static int graph_loop_on = 0;
int graph_loop(int v) {
  if (v >= 0) graph_loop_on = v;
  return graph_loop_on;
}

struct LoopCtl {  // <= 4096 bytes (h_loop)
  double tol;
  double scale;
  int max_cycles;
  int done;
  int conv;
  int nres;
  double res[SP_MAX_RES];
};

__global__ void k_loop_init(LoopCtl* c, double tol, int max_cycles, const double* bn) {
  const double b = sqrt(bn[0]);
  c->tol = tol;
  c->scale = b > 0 ? b : 1.0;
  c->max_cycles = max_cycles;
  c->done = 0;
  c->conv = 0;
  c->nres = 0;
}

__global__ void k_loop_check(LoopCtl* c, const double* norms, int C,
                             cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  double tot = 0.0;
  for (int ch = 0; ch < C; ++ch) tot += norms[ch];
  const double rel = sqrt(tot) / c->scale;
  if (c->nres < SP_MAX_RES) c->res[c->nres++] = rel;
  unsigned go = 0;
  if (rel <= c->tol) c->conv = 1;
  else if (c->done < c->max_cycles) { go = 1; c->done += 1; }
  cudaGraphSetConditional(hw, go);
  cudaGraphSetConditional(hi, go);
}

template <typename T>
static int build_loop_graph(Hier* h) {
  Level& L0 = h->lv[0];
  if (!h->cap_stream) SP_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  if (!h->loop_ctl) SP_CUDA(cudaMalloc(&h->loop_ctl, sizeof(LoopCtl)));
  cudaGraph_t g;
  SP_CUDA(cudaGraphCreate(&g, 0));
  int rc = 0;
  cudaGraphConditionalHandle hw, hi;
  cudaGraphNode_t wnode, cnode, inode;
  cudaGraphNodeParams wp = {};
  cudaGraphNodeParams ip = {};
  cudaGraph_t body, ifbody;
  size_t nn = 0;
  cudaError_t e = cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    e = cudaGraphAddNode(&wnode, g, nullptr, 0, &wp);
  }
  if (e == cudaSuccess) {
    body = wp.conditional.phGraph_out[0];
    e = cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault);
  }
  if (e == cudaSuccess) {
    // the stop test (captured: a kernel node of the WHILE body)
    e = cudaStreamBeginCaptureToGraph(h->cap_stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      k_loop_check<<<1, 1, 0, h->cap_stream>>>((LoopCtl*)h->loop_ctl, L0.norms, h->C, hw, hi);
      cudaError_t le = cudaGetLastError();
      e = cudaStreamEndCapture(h->cap_stream, &body);
      if (e == cudaSuccess) e = le;
    }
  }
  if (e == cudaSuccess) {
    size_t nb = 1;
    e = cudaGraphGetNodes(body, &cnode, &nb);
  }
  if (e == cudaSuccess) {
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    e = cudaGraphAddNode(&inode, body, &cnode, 1, &ip);
  }
  if (e == cudaSuccess) {
    ifbody = ip.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(h->cap_stream, ifbody, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      // precondition of vcycle_lv: level-0 r/norms current (the previous
      // iteration's residual, or the one launched before the graph)
      rc = vcycle_lv<T>(h, 0, true, h->cap_stream);
      if (!rc) rc = residual_lv<T>(h, 0, true, h->cap_stream);
      e = cudaStreamEndCapture(h->cap_stream, &ifbody);
    }
  }
  if (e == cudaSuccess && !rc) {
    cudaGraphGetNodes(ifbody, nullptr, &nn);
    h->loop_nodes = (long long)nn;
    e = cudaGraphInstantiate(&h->loop_exec, g, 0);
  }
  cudaGraphDestroy(g);
  if (rc) return rc;
  SP_CUDA(e);
  return 0;
}

// tolerance mode of solve_t for one image: L0.u / L0.b set and enforced;
// bn = ||b~||^2 on the device.  Fills done[0] / cv[0] and the report.
template <typename T>
static int solve_loop_t(Hier* h, double tol, int max_cycles, const double* bn, cudaStream_t s,
                        int* done, int* cv, SolveReport* rep) {
  if (!h->loop_exec) SP_TRY(build_loop_graph<T>(h));
  LoopCtl* c = (LoopCtl*)h->loop_ctl;
  k_loop_init<<<1, 1, 0, s>>>(c, tol, max_cycles, bn);
  SP_CHECK_LAUNCH();
  SP_TRY(residual_lv<T>(h, 0, true, s));
  SP_CUDA(cudaGraphLaunch(h->loop_exec, s));
  LoopCtl* hc = (LoopCtl*)h->h_loop;
  SP_CUDA(cudaMemcpyAsync(hc, c, sizeof(LoopCtl), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  count_launches(2 + (long long)hc->done * h->loop_nodes);
  done[0] = hc->done;
  cv[0] = hc->conv;
  if (rep) {
    rep->nres = 0;
    for (int i = 0; i < hc->nres && i < SP_MAX_RES; ++i) rep->residuals[rep->nres++] = hc->res[i];
  }
  return 0;
}

template <typename T>
static int solve_t(Hier* h, const T* bsym, T* u_io, int init_mode, double tol, int cycles,
                   int max_cycles, cudaStream_t s, const int* active_in, int* iters,
                   int* conv, SolveReport* rep, const T* u_in = nullptr, int src_mode = 0) {
  // batched cold tile solves to a tolerance (RAS block-local products): the
  // fused on-chip kernel when the hierarchy qualifies (tilesolve.cu)
  if (sizeof(T) == 4 && active_in && !rep && init_mode == 0 && tol >= 0 && src_mode == 0 &&
      tile_fused_ok(h))
    return tile_solve_fused(h, (const float*)bsym, (float*)u_io, tol, max_cycles, s, active_in,
                            iters, conv);
  Level& L0 = h->lv[0];
  const int C = h->C, nt = h->ntile;
  size_t per = (size_t)C * L0.H * L0.W, n = per * nt;
  if (rep) { rep->iterations = 0; rep->nres = 0; rep->converged = 0; }
  // the pinned flag buffer may still feed an earlier async upload
  SP_TRY(active_host_ready(h));
  for (int t = 0; t < nt; ++t) h->h_active[t] = active_in ? (active_in[t] != 0) : 1;
  SP_TRY(upload_active(h, s));
  if (init_mode == 1) {
    SP_CUDA(cudaMemcpyAsync(L0.u, u_in ? u_in : u_io, sizeof(T) * n, cudaMemcpyDeviceToDevice,
                            s));
  } else if (init_mode == 2 && h->lv.size() > 1) {
    if (!h->has_values) {
      set_error("hierarchy was built without stored values");
      return -2;
    }
    SP_TRY(cascade_t<T>(h, s));
  } else {
    SP_CUDA(cudaMemsetAsync(L0.u, 0, sizeof(T) * n, s));
  }
  // scratch layout: partials [nslot * nt], then ||b~||^2 [nt], then a counter
  const size_t nslot = nt == 1 ? 4096 : 1024;
  double* part = (double*)h->d_scratch;
  double* bn = part + nslot * (size_t)nt;
  unsigned* counter = (unsigned*)(bn + nt);
  bool bn_done = false;
  if (src_mode == 1) {
    // b~ = sym_rhs(where(mask, x, 0)) straight into level 0, u = b~ on the
    // mask in the same pass -- and, for a tolerance solve of one image,
    // ||b~||^2 of the tolerance scale (solver.py:351-352) too
    const bool fuse = tol >= 0 && nt == 1 && sizeof(T) == 4 && fused_bnorm_on &&
                      L0.W % 4 == 0 &&
                      (((uintptr_t)bsym | (uintptr_t)L0.b | (uintptr_t)L0.mask) & 15u) == 0;
    if (fuse) SP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
    SP_TRY(masked_sym_rhs<T>(bsym, L0.mask, (T*)L0.b, C, L0.H, L0.W, s, nt, h->d_active,
                             (T*)L0.u, fuse ? bn : nullptr, fuse ? part : nullptr,
                             fuse ? counter : nullptr));
    bn_done = fuse;
  } else {
    SP_CUDA(cudaMemcpyAsync(L0.b, bsym, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
    SP_TRY(enforce<T>((T*)L0.u, (const T*)L0.b, L0.mask, C, L0.H, L0.W, 0, s, nt, h->d_active));
  }
  std::vector<int> done(nt, 0), cv(nt, 0);
  if (tol < 0) {
    // solver.py:345-350: exactly `cycles` V-cycles, converged = True
    for (int c = 0; c < cycles; ++c) {
      SP_TRY(residual_lv<T>(h, 0, true, s));
      SP_TRY(run_vcycle<T>(h, s));
    }
    for (int t = 0; t < nt; ++t) {
      done[t] = h->h_active[t] ? cycles : 0;
      cv[t] = 1;
    }
    if (rep) { rep->iterations = cycles; rep->converged = 1; }
  } else {
    // solver.py:351-369, per tile: ||b~|| over all channels of the tile
    if (!bn_done) {
      SP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
      SP_TRY(chan_reduce<T>(0, (const T*)L0.b, nullptr, nullptr, per, nt, part, counter, bn, s));
    }
    if (nt == 1 && h->use_graphs && graph_loop_on && h->h_loop) {
      SP_TRY(solve_loop_t<T>(h, tol, max_cycles, bn, s, done.data(), cv.data(), rep));
      count_work(0, (long long)done[0] * L0.H * L0.W);
      if (rep) { rep->iterations = done[0]; rep->converged = cv[0]; }
      if (iters) iters[0] = done[0];
      if (conv) conv[0] = cv[0];
      SP_CUDA(cudaMemcpyAsync(u_io, L0.u, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
      return 0;
    }
    std::vector<double> scale(nt);
    SP_CUDA(cudaMemcpyAsync(h->h_norms, bn, sizeof(double) * nt, cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    for (int t = 0; t < nt; ++t) {
      double bnorm = std::sqrt(h->h_norms[t]);
      scale[t] = bnorm > 0 ? bnorm : 1.0;
    }
    while (true) {
      SP_TRY(residual_lv<T>(h, 0, true, s));
      SP_CUDA(cudaMemcpyAsync(h->h_norms, L0.norms, sizeof(double) * C * nt,
                              cudaMemcpyDeviceToHost, s));
      SP_CUDA(cudaStreamSynchronize(s));
      int live = 0;
      bool changed = false;
      for (int t = 0; t < nt; ++t) {
        if (!h->h_active[t]) continue;
        double tot = 0.0;
        for (int c = 0; c < C; ++c) tot += h->h_norms[(size_t)t * C + c];
        double rel = std::sqrt(tot) / scale[t];
        if (t == 0 && rep && rep->nres < SP_MAX_RES) rep->residuals[rep->nres++] = rel;
        if (rel <= tol) { cv[t] = 1; h->h_active[t] = 0; changed = true; continue; }
        if (done[t] >= max_cycles) { h->h_active[t] = 0; changed = true; continue; }
        ++live;
      }
      if (!live) break;
      // the device flags already match unless a tile stopped (one image:
      // never), so the common V-cycle goes straight to the graph launch
      if (changed) SP_TRY(upload_active(h, s));
      SP_TRY(run_vcycle<T>(h, s));
      for (int t = 0; t < nt; ++t) done[t] += h->h_active[t];
    }
    if (rep) { rep->iterations = done[0]; rep->converged = cv[0]; }
  }
  if (iters) for (int t = 0; t < nt; ++t) iters[t] = done[t];
  if (conv) for (int t = 0; t < nt; ++t) conv[t] = cv[t];
  {
    long long cyc = 0;
    for (int t = 0; t < nt; ++t) cyc += done[t];
    count_work(nt > 1 ? 1 : 0, cyc * (long long)L0.H * L0.W);
  }
  SP_CUDA(cudaMemcpyAsync(u_io, L0.u, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int hier_solve(Hier* h, const void* bsym, void* u_io, int init_mode, double tol,
               int cycles, int max_cycles, cudaStream_t s, const int* active_in, int* iters,
               int* conv, SolveReport* rep, const void* u_in, int src_mode) {
  if (h->dtype == SP_F64)
    return solve_t<double>(h, (const double*)bsym, (double*)u_io, init_mode, tol, cycles,
                           max_cycles, s, active_in, iters, conv, rep, (const double*)u_in,
                           src_mode);
  return solve_t<float>(h, (const float*)bsym, (float*)u_io, init_mode, tol, cycles,
                        max_cycles, s, active_in, iters, conv, rep, (const float*)u_in,
                        src_mode);
}

template <typename T>
static int vcycle_once_t(Hier* h, const T* bsym, T* u_io, cudaStream_t s) {
  Level& L0 = h->lv[0];
  size_t n = (size_t)h->C * L0.H * L0.W * h->ntile;
  SP_TRY(active_host_ready(h));
  for (int t = 0; t < h->ntile; ++t) h->h_active[t] = 1;
  SP_TRY(upload_active(h, s));
  SP_CUDA(cudaMemcpyAsync(L0.u, u_io, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  SP_CUDA(cudaMemcpyAsync(L0.b, bsym, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  SP_TRY(residual_lv<T>(h, 0, true, s));
  SP_TRY(run_vcycle<T>(h, s));
  SP_CUDA(cudaMemcpyAsync(u_io, L0.u, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int hier_vcycle(Hier* h, const void* bsym, void* u_io, cudaStream_t s) {
  if (h->dtype == SP_F64) return vcycle_once_t<double>(h, (const double*)bsym, (double*)u_io, s);
  return vcycle_once_t<float>(h, (const float*)bsym, (float*)u_io, s);
}

}  // namespace sp

namespace sp {

// ---- per-kernel timing on the finest level (bench.py roofline) ---------------
// which: 0 = residual + norms sweep, 1 = ORAS local CG, 2 = ORAS blend,
// 3 = fused residual + restriction, 4 = prolongation + add + enforce.  Runs
// `reps` launches on the current level-0 state (after a solve) between CUDA events on `s`; returns the mean
// milliseconds per launch and the algorithmic bytes per launch.
template <typename T>
static int bench_t(Hier* h, int which, int reps, cudaStream_t s, double* ms, double* bytes) {
  Level& L = h->lv[0];
  const size_t es = sizeof(T), C = h->C, plane = (size_t)L.H * L.W, nt = h->ntile;
  const size_t vec = C * plane * nt;
  const size_t nb = (size_t)L.nby * L.nbx, npx = (size_t)L.bh * L.bw;
  // algorithmic bytes (SURVEY.md section 8d conventions, mask shared by channels)
  switch (which) {
    case 0: *bytes = (double)(3 * es * vec + plane * nt); break;          // u, b, r + mask
    case 1: {
      // r + corr per job, mask once per block, weights: the blocks whose
      // weights are not aliased to the shared interior pattern, plus it once
      size_t own = nb;
      if (L.wdelta) {
        std::vector<int> wd(nb);
        SP_CUDA(cudaMemcpy(wd.data(), L.wdelta, sizeof(int) * nb, cudaMemcpyDeviceToHost));
        own = 1;
        for (int d : wd) own += d == 0;
      }
      // the job's row masks: one 32-bit word per column with offbits, else
      // the mask bytes
      const size_t mb = L.offbits && oras_offbits(-1) ? nb * 32 * 4 * nt : nb * npx * nt;
      *bytes = (double)(es * C * nb * npx * nt * 2 + mb + es * own * npx);
      break;
    }
    case 2: *bytes = (double)(es * C * nb * npx * nt + 2 * es * vec); break;       // corr + u rw
    case 3: *bytes = (double)(2 * es * vec + plane * nt + es * vec / 4); break;    // u, b, mask, rc
    case 4: *bytes = (double)(2 * es * vec + plane * nt + es * vec / 4); break;    // u rw, mask, e
    default: set_error("unknown kernel id %d", which); return -2;
  }
  SP_TRY(active_host_ready(h));
  for (int t = 0; t < nt; ++t) h->h_active[t] = 1;
  SP_TRY(upload_active(h, s));
  Level* G = h->lv.size() > 1 ? &h->lv[1] : nullptr;
  auto launch = [&]() -> int {
    switch (which) {
      case 0:
        return residual_lv<T>(h, 0, true, s);
      case 1:
        return oras_lv<T>(h, L, s);
      case 2:
        // blend into a scratch copy so the solver state is not disturbed
        return blend_lv<T>(h, L, (T*)L.r, s);
      case 3:
        if (!G) { set_error("single-level hierarchy"); return -2; }
        return residual_restrict_lv<T>(h, 0, s);
      default: {
        // u += P e, u = b~ on the mask, into the r buffer (scratch) so the
        // solver state is not disturbed
        if (!G) { set_error("single-level hierarchy"); return -2; }
        if (sizeof(T) == 4 && h->sweep == 2 && tma_prolong_ok(L.H, L.W) && aligned_level<T>(L))
          return prolong_tma((const float*)G->u, (float*)L.r, (const float*)L.b, L.mask, h->C,
                             G->H, G->W, L.H, L.W, 1, s, h->ntile, h->d_active);
        return prolong_enforce<T>((const T*)G->u, (T*)L.r, (const T*)L.b, L.mask, h->C, G->H,
                                  G->W, L.H, L.W, 1, s, h->ntile, h->d_active);
      }
    }
  };
  // the ORAS local kernel needs current r/norms
  SP_TRY(residual_lv<T>(h, 0, true, s));
  SP_TRY(launch());  // warm-up
  cudaEvent_t e0, e1;
  SP_CUDA(cudaEventCreate(&e0));
  SP_CUDA(cudaEventCreate(&e1));
  SP_CUDA(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) SP_TRY(launch());
  SP_CUDA(cudaEventRecord(e1, s));
  SP_CUDA(cudaEventSynchronize(e1));
  float t = 0.f;
  SP_CUDA(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = (double)t / reps;
  // leave r / norms consistent with u for the next solve
  SP_TRY(residual_lv<T>(h, 0, true, s));
  return 0;
}

// residual of level lv's current state (u, b) into r_out / norms_out, with
// the sweep kernel the hierarchy uses (kernel-variant tests)
template <typename T>
static int residual_out_t(Hier* h, int lv, void* r_out, double* norms_out, cudaStream_t s) {
  if (lv < 0 || lv >= (int)h->lv.size()) { set_error("no level %d", lv); return -2; }
  Level& L = h->lv[lv];
  SP_TRY(active_host_ready(h));
  for (int t = 0; t < h->ntile; ++t) h->h_active[t] = 1;
  SP_TRY(upload_active(h, s));
  SP_TRY(residual_lv<T>(h, lv, true, s));
  const size_t n = (size_t)h->C * L.H * L.W * h->ntile;
  SP_CUDA(cudaMemcpyAsync(r_out, L.r, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  SP_CUDA(cudaMemcpyAsync(norms_out, L.norms, sizeof(double) * h->C * h->ntile,
                          cudaMemcpyDeviceToDevice, s));
  return 0;
}

int hier_residual_out(Hier* h, int lv, void* r_out, double* norms_out, cudaStream_t s) {
  if (h->dtype == SP_F64) return residual_out_t<double>(h, lv, r_out, norms_out, s);
  return residual_out_t<float>(h, lv, r_out, norms_out, s);
}

int hier_bench(Hier* h, int which, int reps, cudaStream_t s, double* ms, double* bytes) {
  if (h->dtype == SP_F64) return bench_t<double>(h, which, reps, s, ms, bytes);
  return bench_t<float>(h, which, reps, s, ms, bytes);
}

// level operations shared with the row-strip solver (strips.cu)
template int prolong_lv<float>(Hier*, int, int, cudaStream_t);
template int smooth_lv<float>(Hier*, int, int, bool, cudaStream_t);
template int vcycle_lv<float>(Hier*, int, bool, cudaStream_t);

}  // namespace sp
