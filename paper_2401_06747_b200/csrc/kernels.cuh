// kernels.cuh -- launcher declarations shared by the .cu translation units.
#pragma once
#include "common.cuh"

namespace sp {

// ---- stencil.cu ------------------------------------------------------------
template <typename T> int neglap(const T* x, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int inpaint_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int sym_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int sym_rhs(const T* b, const uint8_t* m, T* out, T* e, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int masked_sym_rhs(const T* x, const uint8_t* m, T* out, int C, int H, int W, cudaStream_t s);
template <typename T> int ct_apply(const T* w, const uint8_t* m, T* out, int C, int H, int W, double inv_h2, cudaStream_t s);
size_t residual_partials(int H, int W);
template <typename T> int residual(const T* u, const T* b, const uint8_t* m, T* r, double* partial, unsigned* counter, double* norms, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int residual_restrict(const T* u, const T* b, const uint8_t* m, T* rc, int C, int H, int W, double inv_h2, cudaStream_t s);
template <typename T> int restrict_values(const T* f, T* out, int C, int H, int W, cudaStream_t s);
template <typename T> int restrict_mask(const uint8_t* m, const T* v, uint8_t* cm, T* cv, int C, int H, int W, cudaStream_t s);
template <typename T> int prolongate(const T* co, T* out, int C, int chh, int cww, int H, int W, cudaStream_t s);
template <typename T> int prolong_add_enforce(const T* e, T* u, const T* b, const uint8_t* m, int C, int chh, int cww, int H, int W, cudaStream_t s);
template <typename T> int prolong_enforce(const T* uc, T* u, const T* b, const uint8_t* m, int C, int chh, int cww, int H, int W, cudaStream_t s);
template <typename T> int enforce(T* u, const T* src, const uint8_t* m, int C, int H, int W, int zero_off, cudaStream_t s);

// ---- oras.cu ---------------------------------------------------------------
// One ORAS sweep given the residual r and per-channel norms (device):
// local CG per (block, channel) -> corr, then the ordered blend into u.
struct OrasGeom {
  int H, W, C;
  int bh, bw, nby, nbx, stride_y, stride_x, overlap;
  double gamma, rho, inv_h2;
  long cap;
};
template <typename T> int oras_local(const T* r, const uint8_t* m, const double* norms, const double* taus_host, T* corr, const OrasGeom& g, cudaStream_t s);
template <typename T> int oras_blend(T* u, const T* corr, const T* weights, const OrasGeom& g, cudaStream_t s);

// ---- vec.cu ------------------------------------------------------------------
int mse_partial_count(size_t n);

}  // namespace sp
