// kernels.cuh -- launcher declarations shared by the .cu translation units.
#pragma once
#include <vector>
#include "common.cuh"

namespace sp {

// ---- stencil.cu (ntile/active: batched independent problems, see stencil.cu)
template <typename T> int neglap(const T* x, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int inpaint_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int sym_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int sym_rhs(const T* b, const uint8_t* m, T* out, T* e, int C, int H, int W, double inv_h2, cudaStream_t s, int ntile = 1, const int* active = nullptr);
// b~ = sym_rhs(where(m, x, 0)); enforce_u (optional): u = b~ on the stored
// pixels in the same pass (sparse stores)
// nrm (one image): also *nrm = sum of out^2 over all planes in the same pass
// (partial: >= 4096 doubles, counter: zeroed)
template <typename T> int masked_sym_rhs(const T* x, const uint8_t* m, T* out, int C, int H, int W, cudaStream_t s, int ntile = 1, const int* active = nullptr, T* enforce_u = nullptr, double* nrm = nullptr, double* partial = nullptr, unsigned* counter = nullptr);
template <typename T> int ct_apply(const T* w, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s, int ntile = 1, const int* active = nullptr);
size_t residual_partials(int H, int W);
template <typename T> int residual(const T* u, const T* b, const uint8_t* m, T* r, double* partial, unsigned* counter, double* norms, int C, int H, int W, double inv_h2, cudaStream_t s, int ntile = 1, const int* active = nullptr);
template <typename T> int residual_restrict(const T* u, const T* b, const uint8_t* m, T* rc, int C, int H, int W, double inv_h2, cudaStream_t s, int ntile = 1, const int* active = nullptr);
template <typename T> int restrict_values(const T* f, T* out, int C, int H, int W, cudaStream_t s);
template <typename T> int restrict_mask(const uint8_t* m, const T* v, uint8_t* cm, T* cv, int C, int H, int W, cudaStream_t s, int ntile = 1);
template <typename T> int prolongate(const T* co, T* out, int C, int chh, int cww, int H, int W, cudaStream_t s);
template <typename T> int prolong_enforce(const T* e, T* u, const T* b, const uint8_t* m, int C, int chh, int cww, int H, int W, int add, cudaStream_t s, int ntile = 1, const int* active = nullptr);
template <typename T> int enforce(T* u, const T* src, const uint8_t* m, int C, int H, int W, int zero_off, cudaStream_t s, int ntile = 1, const int* active = nullptr);

// ---- oras.cu ---------------------------------------------------------------
// local CG per (block, channel, tile) -> corr = T(w_b) * v_b
template <typename T>
int oras_local_launch(const T* r, const uint8_t* m, const double* tau_src, double tau_scale,
                      const int* ys, const int* xs, int nby, int nbx, int bh, int bw, int H,
                      int W, int C, double gamma, long cap, double inv_h2, const T* weights,
                      T* corr, cudaStream_t s, int ntile = 1, const int* active = nullptr,
                      int stride = 0, int corr_nb = 0, size_t ps = 0,
                      const int* wdelta = nullptr, const uint32_t* offbits = nullptr,
                      const int* tile_list = nullptr, int nlist = 0);
int oras_offbits(int v);  // sp_oras_offbits
int oras_variant(int v);  // the ORAS local-CG kernel (sp_oras_variant)
// per-job row-mask words of the ORAS blocks ([ntile][nb][32], see Level)
int oras_offbits_launch(const uint8_t* m, const int* ys, const int* xs, int nby, int nbx, int bh,
                        int bw, int H, int W, int ntile, uint32_t* offbits, cudaStream_t s);
// wdelta[b] = c - b where block c holds weights identical to block b's
// (interior blocks share one 32x32 pattern): the ORAS epilogue reads the
// shared pattern (cache-resident) instead of every block's own weights
int weight_aliases(const float* weights, int nby, int nbx, int bh, int bw, int* wdelta,
                   cudaStream_t s);
// u += weighted corrections of the covering blocks, in block order
template <typename T>
int oras_blend_launch(T* u, const T* corr, const int* ys, const int* xs, const int* row_k0,
                      const int* row_n, const int* col_k0, const int* col_n, int nby, int nbx,
                      int bh, int bw, int H, int W, int C, cudaStream_t s, int ntile = 1,
                      const int* active = nullptr, int corr_nb = 0, size_t ps = 0,
                      const int* rowinfo = nullptr, const int* colinfo = nullptr,
                      bool pair_cols = false);
// packed per-row / per-column cover words for the C = 3 float blend
// (k_oras_blend3p); sp_blend_packed
bool blend_pack(const std::vector<int>& starts, int size, int dim, std::vector<int>& info);
int blend_packed(int v);
// partition-of-unity weights [nb][bh][bw] (solver.py:142-197)
template <typename T>
int block_weights_launch(T* weights, const int* ys, const int* xs, const int* row_k0,
                         const int* row_n, const int* col_k0, const int* col_n, int nby,
                         int nbx, int bh, int bw, int H, int W, int overlap, cudaStream_t s);

// ---- mgfast.cu: row-marching float sweeps (W % 4 == 0, W >= 128, inv_h2 = 1) --
bool march_ok(int H, int W, size_t npart);
int resid_march(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
                unsigned* counter, double* norms, int C, int H, int W, cudaStream_t s,
                int ntile, const int* active, double* bandcol = nullptr, int band0 = 0,
                int nbt = 0);
int march_band_rows();  // rows per norm band (bandcol mode)
int resid_restrict_march(const float* u, const float* b, const uint8_t* m, float* rc, int C,
                         int H, int W, cudaStream_t s, int ntile, const int* active);
int prolong_march(const float* e, float* u, const float* b, const uint8_t* m, int C, int chh,
                  int cww, int H, int W, int add, cudaStream_t s, int ntile,
                  const int* active);

// ---- mgtma.cu: TMA-staged float sweeps (W % 16 == 0, W >= 128, inv_h2 = 1) -----
bool tma_ok(int H, int W, size_t npart);
int resid_tma(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
              unsigned* counter, double* norms, int C, int H, int W, cudaStream_t s, int ntile,
              const int* active, double* bandcol = nullptr, int band0 = 0, int nbt = 0,
              size_t ps = 0, size_t npart = 0);
// warp-streamed sweeps (default 1) vs the CTA-tile kernels (0): sp_ws_variant
int ws_variant(int v);
int ws_prefetch(int v);  // chunks per warp prefetched into L2 (sp_ws_prefetch, default 0)
int ws_stages(int v);    // shared-memory stages per warp, 1 or 2 (sp_ws_stages)
bool tma_view_ok(int W);
int tma_prepare();  // one-time kernel attributes (outside graph capture)
// ps / cps: fine / coarse plane strides in elements (0 = H*W / its coarse
// level's); a row-strip view passes its full level's strides
int resid_restrict_tma(const float* u, const float* b, const uint8_t* m, float* rc, int C,
                       int H, int W, cudaStream_t s, int ntile, const int* active,
                       size_t ps = 0, size_t cps = 0);
bool tma_prolong_ok(int H, int W);
int prolong_tma(const float* e, float* u, const float* b, const uint8_t* m, int C, int chh,
                int cww, int H, int W, int add, cudaStream_t s, int ntile, const int* active,
                size_t ps = 0, size_t cps = 0);

// ---- vec.cu ------------------------------------------------------------------
template <typename T>
int chan_reduce(int mode, const T* x, const T* y, const double* z, size_t n, int C,
                double* partial, unsigned* counter, double* out, cudaStream_t s);
template <typename T>
int error_map(const T* u, const double* f, double* e, int C, size_t n, cudaStream_t s,
              double* total = nullptr);  // total: sum of e (deterministic), optional

}  // namespace sp
