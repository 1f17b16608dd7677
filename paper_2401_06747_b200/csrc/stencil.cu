// stencil.cu -- the 5-point stencil family and grid transfers (sm_100a).
//
// Reference semantics: numba_impl.py:13-158 (stencils, residual),
// :266-348 (restrict_values / restrict_mask / prolongate).  Every stencil
// accumulates in double in the reference order (up, down, left, right) and
// rounds once to T, so outputs are bit-identical to the CPU oracle.
// One thread owns one pixel and loops over the C channels (planar layout,
// mask shared by channels); warps run along x so every load is coalesced.
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int BX = 32, BY = 8, NT = BX * BY;

__device__ __forceinline__ bool in_img(int y, int x, int H, int W) {
  return y >= 0 && y < H && x >= 0 && x < W;
}

// negated Laplacian (numba_impl.py:13-36)
template <typename T>
__global__ void k_neglap(const T* __restrict__ x, T* __restrict__ out, int C,
                         int H, int W, double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  for (int c = 0; c < C; ++c) {
    const T* xc = x + c * plane;
    double d = 0.0, a = 0.0;
    if (y > 0) { d += 1.0; a += (double)xc[k - W]; }
    if (y < H - 1) { d += 1.0; a += (double)xc[k + W]; }
    if (xx > 0) { d += 1.0; a += (double)xc[k - 1]; }
    if (xx < W - 1) { d += 1.0; a += (double)xc[k + 1]; }
    out[c * plane + k] = (T)((d * (double)xc[k] - a) * inv_h2);
  }
}

// A x = C x + (I-C) L x (numba_impl.py:39-65)
template <typename T>
__global__ void k_inpaint_matvec(const T* __restrict__ x, const uint8_t* __restrict__ m,
                                 T* __restrict__ out, int C, int H, int W,
                                 double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  for (int c = 0; c < C; ++c) {
    const T* xc = x + c * plane;
    if (mk) { out[c * plane + k] = xc[k]; continue; }
    double d = 0.0, a = 0.0;
    if (y > 0) { d += 1.0; a += (double)xc[k - W]; }
    if (y < H - 1) { d += 1.0; a += (double)xc[k + W]; }
    if (xx > 0) { d += 1.0; a += (double)xc[k - 1]; }
    if (xx < W - 1) { d += 1.0; a += (double)xc[k + 1]; }
    out[c * plane + k] = (T)((d * (double)xc[k] - a) * inv_h2);
  }
}

// neighbour code: bit0 up, bit1 down, bit2 left, bit3 right are inside the
// image; bits 4..7 the same neighbours are unmasked.
__device__ __forceinline__ unsigned nbr_code(const uint8_t* __restrict__ m, size_t k,
                                             int y, int xx, int H, int W) {
  unsigned code = 0;
  if (y > 0) { code |= 1u; if (!m[k - W]) code |= 16u; }
  if (y < H - 1) { code |= 2u; if (!m[k + W]) code |= 32u; }
  if (xx > 0) { code |= 4u; if (!m[k - 1]) code |= 64u; }
  if (xx < W - 1) { code |= 8u; if (!m[k + 1]) code |= 128u; }
  return code;
}

// symmetrized matvec at an unmasked pixel (numba_impl.py:78-97)
template <typename T>
__device__ __forceinline__ T sym_row(const T* __restrict__ xc, size_t k, int W,
                                     unsigned code, double inv_h2) {
  double d = 0.0, a = 0.0;
  if (code & 1u) { d += 1.0; if (code & 16u) a += (double)xc[k - W]; }
  if (code & 2u) { d += 1.0; if (code & 32u) a += (double)xc[k + W]; }
  if (code & 4u) { d += 1.0; if (code & 64u) a += (double)xc[k - 1]; }
  if (code & 8u) { d += 1.0; if (code & 128u) a += (double)xc[k + 1]; }
  return (T)((d * (double)xc[k] - a) * inv_h2);
}

template <typename T>
__global__ void k_sym_matvec(const T* __restrict__ x, const uint8_t* __restrict__ m,
                             T* __restrict__ out, int C, int H, int W, double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  unsigned code = mk ? 0u : nbr_code(m, k, y, xx, H, W);
  for (int c = 0; c < C; ++c) {
    const T* xc = x + c * plane;
    out[c * plane + k] = mk ? xc[k] : sym_row(xc, k, W, code, inv_h2);
  }
}

// C~ b (numba_impl.py:101-121); optionally also writes e = mask ? out : 0
// (the coarse-grid "e = 0; _enforce(e, bsym_c)" of solver.py:289-292)
template <typename T>
__global__ void k_sym_rhs(const T* __restrict__ b, const uint8_t* __restrict__ m,
                          T* __restrict__ out, T* __restrict__ e, int C, int H, int W,
                          double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  bool up = y > 0 && m[k - W], dn = y < H - 1 && m[k + W];
  bool lf = xx > 0 && m[k - 1], rt = xx < W - 1 && m[k + 1];
  for (int c = 0; c < C; ++c) {
    const T* bc = b + c * plane;
    T o;
    if (mk) {
      o = bc[k];
    } else {
      double a = 0.0;
      if (up) a += (double)bc[k - W];
      if (dn) a += (double)bc[k + W];
      if (lf) a += (double)bc[k - 1];
      if (rt) a += (double)bc[k + 1];
      o = (T)((double)bc[k] + a * inv_h2);
    }
    out[c * plane + k] = o;
    if (e) e[c * plane + k] = mk ? o : (T)0;
  }
}

// where(mask, x, 0) followed by sym_rhs, fused (tonal.py:136-137, solver.py:501-502)
template <typename T>
__global__ void k_masked_sym_rhs(const T* __restrict__ x, const uint8_t* __restrict__ m,
                                 T* __restrict__ out, int C, int H, int W) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  bool up = y > 0 && m[k - W], dn = y < H - 1 && m[k + W];
  bool lf = xx > 0 && m[k - 1], rt = xx < W - 1 && m[k + 1];
  for (int c = 0; c < C; ++c) {
    const T* xc = x + c * plane;
    T o;
    if (mk) {
      o = xc[k];
    } else {
      // b(k) = 0 off-mask; numba adds 0.0 + acc (exact)
      double a = 0.0;
      if (up) a += (double)xc[k - W];
      if (dn) a += (double)xc[k + W];
      if (lf) a += (double)xc[k - 1];
      if (rt) a += (double)xc[k + 1];
      o = (T)(0.0 + a);
    }
    out[c * plane + k] = o;
  }
}

// (C - C L (I-C)) w, zero off-mask (numba_impl.py:124-144)
template <typename T>
__global__ void k_ct_apply(const T* __restrict__ w, const uint8_t* __restrict__ m,
                           T* __restrict__ out, int C, int H, int W, double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  bool up = y > 0 && !m[k - W], dn = y < H - 1 && !m[k + W];
  bool lf = xx > 0 && !m[k - 1], rt = xx < W - 1 && !m[k + 1];
  for (int c = 0; c < C; ++c) {
    const T* wc = w + c * plane;
    if (!mk) { out[c * plane + k] = (T)0; continue; }
    double a = 0.0;
    if (up) a += (double)wc[k - W];
    if (dn) a += (double)wc[k + W];
    if (lf) a += (double)wc[k - 1];
    if (rt) a += (double)wc[k + 1];
    out[c * plane + k] = (T)((double)wc[k] + a * inv_h2);
  }
}

// r = b~ - A~ u (T arithmetic) and per-channel sum of r^2 in double
// (numba_impl.py:147-158).  The squares are reduced deterministically: CTA
// tree, then the last CTA to finish adds the per-CTA partials in fixed order.
template <typename T>
__global__ void __launch_bounds__(NT) k_residual(
    const T* __restrict__ u, const T* __restrict__ b, const uint8_t* __restrict__ m,
    T* __restrict__ r, double* __restrict__ partial, unsigned* __restrict__ counter,
    double* __restrict__ norms, int C, int H, int W, double inv_h2) {
  __shared__ double s0[NT / 32], s1[NT / 32];
  __shared__ bool am_last;
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  int tid = threadIdx.y * BX + threadIdx.x;
  unsigned nblk = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  bool live = xx < W && y < H;
  size_t plane = (size_t)H * W, k = live ? (size_t)y * W + xx : 0;
  bool mk = live ? m[k] : true;
  unsigned code = (live && !mk) ? nbr_code(m, k, y, xx, H, W) : 0u;
  for (int c = 0; c < C; ++c) {
    double sq = 0.0;
    if (live) {
      const T* uc = u + c * plane;
      T ax = mk ? uc[k] : sym_row(uc, k, W, code, inv_h2);
      T rv = (T)(b[c * plane + k] - ax);
      if (r) r[c * plane + k] = rv;
      sq = (double)rv * (double)rv;
    }
    double s = cta_sum<NT>(sq, (c & 1) ? s1 : s0);
    if (tid == 0) partial[(size_t)bid * C + c] = s;
  }
  if (!norms) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(counter, 1u) == nblk - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (unsigned i = tid; i < nblk; i += NT)
      s += ((volatile double*)partial)[(size_t)i * C + c];
    s = cta_sum<NT>(s, (c & 1) ? s1 : s0);
    if (tid == 0) norms[c] = s;
  }
  if (tid == 0) *counter = 0u;
}

// fused residual + 2x2 restriction (solver.py:289-290: restrict_values(r)).
// One thread per coarse pixel recomputes its (up to four) fine residuals in
// T and averages them in double in row-major order (numba_impl.py:266-284).
template <typename T>
__global__ void k_residual_restrict(const T* __restrict__ u, const T* __restrict__ b,
                                    const uint8_t* __restrict__ m, T* __restrict__ rc,
                                    int C, int H, int W, double inv_h2) {
  int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
  if (j >= cw || i >= ch_) return;
  size_t plane = (size_t)H * W, cplane = (size_t)ch_ * cw;
  int y1 = min(2 * i + 2, H), x1 = min(2 * j + 2, W);
  unsigned codes[4];
  bool mks[4];
  int n = 0;
  for (int y = 2 * i; y < y1; ++y)
    for (int x = 2 * j; x < x1; ++x) {
      size_t k = (size_t)y * W + x;
      mks[n] = m[k];
      codes[n] = mks[n] ? 0u : nbr_code(m, k, y, x, H, W);
      ++n;
    }
  for (int c = 0; c < C; ++c) {
    const T* uc = u + c * plane;
    const T* bc = b + c * plane;
    double acc = 0.0;
    int q = 0;
    for (int y = 2 * i; y < y1; ++y)
      for (int x = 2 * j; x < x1; ++x, ++q) {
        size_t k = (size_t)y * W + x;
        T ax = mks[q] ? uc[k] : sym_row(uc, k, W, codes[q], inv_h2);
        acc += (double)(T)(bc[k] - ax);
      }
    rc[c * cplane + (size_t)i * cw + j] = (T)(acc / (double)n);
  }
}

// 2x2 box average (numba_impl.py:266-284)
template <typename T>
__global__ void k_restrict_values(const T* __restrict__ f, T* __restrict__ out, int C,
                                  int H, int W) {
  int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
  if (j >= cw || i >= ch_) return;
  size_t plane = (size_t)H * W, cplane = (size_t)ch_ * cw;
  int y1 = min(2 * i + 2, H), x1 = min(2 * j + 2, W);
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
    int n = 0;
    for (int y = 2 * i; y < y1; ++y)
      for (int x = 2 * j; x < x1; ++x) { acc += (double)f[c * plane + (size_t)y * W + x]; ++n; }
    out[c * cplane + (size_t)i * cw + j] = (T)(acc / (double)n);
  }
}

// OR mask + mean of covered stored values (numba_impl.py:287-313)
template <typename T>
__global__ void k_restrict_mask(const uint8_t* __restrict__ m, const T* __restrict__ v,
                                uint8_t* __restrict__ cm, T* __restrict__ cv, int C,
                                int H, int W) {
  int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
  if (j >= cw || i >= ch_) return;
  size_t plane = (size_t)H * W, cplane = (size_t)ch_ * cw, ck = (size_t)i * cw + j;
  int y1 = min(2 * i + 2, H), x1 = min(2 * j + 2, W);
  int cnt = 0;
  for (int y = 2 * i; y < y1; ++y)
    for (int x = 2 * j; x < x1; ++x) cnt += m[(size_t)y * W + x] ? 1 : 0;
  cm[ck] = cnt > 0;
  if (!cv) return;
  for (int c = 0; c < C; ++c) {
    T o = (T)0;
    if (cnt) {
      double acc = 0.0;
      for (int y = 2 * i; y < y1; ++y)
        for (int x = 2 * j; x < x1; ++x)
          if (m[(size_t)y * W + x]) acc += (double)v[c * plane + (size_t)y * W + x];
      o = (T)(acc / (double)cnt);
    }
    cv[c * cplane + ck] = o;
  }
}

// cell-centred bilinear weights, clamped (numba_impl.py:321-341)
__device__ __forceinline__ void prolong_axis(int y, int n, int& y0, int& y1, double& wy) {
  double fy = ((double)y + 0.5) / 2.0 - 0.5;
  y0 = (int)floor(fy);
  wy = fy - (double)y0;
  if (y0 < 0) { y0 = 0; wy = 0.0; }
  if (y0 > n - 1) { y0 = n - 1; wy = 0.0; }
  y1 = min(y0 + 1, n - 1);
}

template <typename T>
__device__ __forceinline__ T prolong_at(const T* __restrict__ cc, int cww, int y0, int y1,
                                        double wy, int x0, int x1, double wx) {
  double v = (1.0 - wy) * ((1.0 - wx) * (double)cc[(size_t)y0 * cww + x0] +
                           wx * (double)cc[(size_t)y0 * cww + x1]) +
             wy * ((1.0 - wx) * (double)cc[(size_t)y1 * cww + x0] +
                   wx * (double)cc[(size_t)y1 * cww + x1]);
  return (T)v;
}

template <typename T>
__global__ void k_prolongate(const T* __restrict__ co, T* __restrict__ out, int C,
                             int chh, int cww, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  int y0, y1, x0, x1;
  double wy, wx;
  prolong_axis(y, chh, y0, y1, wy);
  prolong_axis(x, cww, x0, x1, wx);
  size_t plane = (size_t)H * W, cplane = (size_t)chh * cww;
  for (int c = 0; c < C; ++c)
    out[c * plane + (size_t)y * W + x] =
        prolong_at(co + c * cplane, cww, y0, y1, wy, x0, x1, wx);
}

// u += prolongate(e); u[mask] = b~[mask]  (solver.py:294-296)
template <typename T>
__global__ void k_prolong_add_enforce(const T* __restrict__ e, T* __restrict__ u,
                                      const T* __restrict__ b,
                                      const uint8_t* __restrict__ m, int C, int chh,
                                      int cww, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  size_t plane = (size_t)H * W, cplane = (size_t)chh * cww, k = (size_t)y * W + x;
  if (m[k]) {
    for (int c = 0; c < C; ++c) u[c * plane + k] = b[c * plane + k];
    return;
  }
  int y0, y1, x0, x1;
  double wy, wx;
  prolong_axis(y, chh, y0, y1, wy);
  prolong_axis(x, cww, x0, x1, wx);
  for (int c = 0; c < C; ++c) {
    T p = prolong_at(e + c * cplane, cww, y0, y1, wy, x0, x1, wx);
    u[c * plane + k] = (T)(u[c * plane + k] + p);
  }
}

// u = prolongate(uc) then u[mask] = b[mask]  (FMG cascade, solver.py:309-312)
template <typename T>
__global__ void k_prolong_enforce(const T* __restrict__ uc, T* __restrict__ u,
                                  const T* __restrict__ b, const uint8_t* __restrict__ m,
                                  int C, int chh, int cww, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  size_t plane = (size_t)H * W, cplane = (size_t)chh * cww, k = (size_t)y * W + x;
  if (m[k]) {
    for (int c = 0; c < C; ++c) u[c * plane + k] = b[c * plane + k];
    return;
  }
  int y0, y1, x0, x1;
  double wy, wx;
  prolong_axis(y, chh, y0, y1, wy);
  prolong_axis(x, cww, x0, x1, wx);
  for (int c = 0; c < C; ++c)
    u[c * plane + k] = prolong_at(uc + c * cplane, cww, y0, y1, wy, x0, x1, wx);
}

// u[mask] = src[mask] (solver.py:275-281, 508-510); optional zero elsewhere
template <typename T>
__global__ void k_enforce(T* __restrict__ u, const T* __restrict__ src,
                          const uint8_t* __restrict__ m, int C, size_t plane,
                          int zero_off) {
  size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= plane) return;
  bool mk = m[k];
  for (int c = 0; c < C; ++c) {
    if (mk) u[c * plane + k] = src[c * plane + k];
    else if (zero_off) u[c * plane + k] = (T)0;
  }
}

inline dim3 grid2(int W, int H) { return dim3(cdiv(W, BX), cdiv(H, BY)); }
const dim3 kBlock(BX, BY);

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <typename T>
int neglap(const T* x, T* out, int C, int H, int W, double inv_h2, cudaStream_t s) {
  k_neglap<T><<<grid2(W, H), kBlock, 0, s>>>(x, out, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int inpaint_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W,
                   double inv_h2, cudaStream_t s) {
  k_inpaint_matvec<T><<<grid2(W, H), kBlock, 0, s>>>(x, m, out, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int sym_matvec(const T* x, const uint8_t* m, T* out, int C, int H, int W,
               double inv_h2, cudaStream_t s) {
  k_sym_matvec<T><<<grid2(W, H), kBlock, 0, s>>>(x, m, out, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int sym_rhs(const T* b, const uint8_t* m, T* out, T* e, int C, int H, int W,
            double inv_h2, cudaStream_t s) {
  k_sym_rhs<T><<<grid2(W, H), kBlock, 0, s>>>(b, m, out, e, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int masked_sym_rhs(const T* x, const uint8_t* m, T* out, int C, int H, int W,
                   cudaStream_t s) {
  k_masked_sym_rhs<T><<<grid2(W, H), kBlock, 0, s>>>(x, m, out, C, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int ct_apply(const T* w, const uint8_t* m, T* out, int C, int H, int W, double inv_h2,
             cudaStream_t s) {
  k_ct_apply<T><<<grid2(W, H), kBlock, 0, s>>>(w, m, out, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

size_t residual_partials(int H, int W) { return (size_t)cdiv(W, BX) * cdiv(H, BY); }

template <typename T>
int residual(const T* u, const T* b, const uint8_t* m, T* r, double* partial,
             unsigned* counter, double* norms, int C, int H, int W, double inv_h2,
             cudaStream_t s) {
  k_residual<T><<<grid2(W, H), kBlock, 0, s>>>(u, b, m, r, partial, counter, norms, C,
                                               H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int residual_restrict(const T* u, const T* b, const uint8_t* m, T* rc, int C, int H,
                      int W, double inv_h2, cudaStream_t s) {
  k_residual_restrict<T><<<grid2((W + 1) / 2, (H + 1) / 2), kBlock, 0, s>>>(
      u, b, m, rc, C, H, W, inv_h2);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int restrict_values(const T* f, T* out, int C, int H, int W, cudaStream_t s) {
  k_restrict_values<T><<<grid2((W + 1) / 2, (H + 1) / 2), kBlock, 0, s>>>(f, out, C, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int restrict_mask(const uint8_t* m, const T* v, uint8_t* cm, T* cv, int C, int H, int W,
                  cudaStream_t s) {
  k_restrict_mask<T><<<grid2((W + 1) / 2, (H + 1) / 2), kBlock, 0, s>>>(m, v, cm, cv, C,
                                                                       H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int prolongate(const T* co, T* out, int C, int chh, int cww, int H, int W,
               cudaStream_t s) {
  k_prolongate<T><<<grid2(W, H), kBlock, 0, s>>>(co, out, C, chh, cww, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int prolong_add_enforce(const T* e, T* u, const T* b, const uint8_t* m, int C, int chh,
                        int cww, int H, int W, cudaStream_t s) {
  k_prolong_add_enforce<T><<<grid2(W, H), kBlock, 0, s>>>(e, u, b, m, C, chh, cww, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int prolong_enforce(const T* uc, T* u, const T* b, const uint8_t* m, int C, int chh,
                    int cww, int H, int W, cudaStream_t s) {
  k_prolong_enforce<T><<<grid2(W, H), kBlock, 0, s>>>(uc, u, b, m, C, chh, cww, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int enforce(T* u, const T* src, const uint8_t* m, int C, int H, int W, int zero_off,
            cudaStream_t s) {
  size_t plane = (size_t)H * W;
  k_enforce<T><<<cdiv(plane, 256), 256, 0, s>>>(u, src, m, C, plane, zero_off);
  SP_CHECK_LAUNCH();
  return 0;
}

#define INST(T)                                                                       \
  template int neglap<T>(const T*, T*, int, int, int, double, cudaStream_t);            \
  template int inpaint_matvec<T>(const T*, const uint8_t*, T*, int, int, int, double,   \
                                 cudaStream_t);                                         \
  template int sym_matvec<T>(const T*, const uint8_t*, T*, int, int, int, double,       \
                             cudaStream_t);                                             \
  template int sym_rhs<T>(const T*, const uint8_t*, T*, T*, int, int, int, double,      \
                          cudaStream_t);                                                \
  template int masked_sym_rhs<T>(const T*, const uint8_t*, T*, int, int, int,           \
                                 cudaStream_t);                                         \
  template int ct_apply<T>(const T*, const uint8_t*, T*, int, int, int, double,         \
                           cudaStream_t);                                               \
  template int residual<T>(const T*, const T*, const uint8_t*, T*, double*, unsigned*,  \
                           double*, int, int, int, double, cudaStream_t);               \
  template int residual_restrict<T>(const T*, const T*, const uint8_t*, T*, int, int,   \
                                    int, double, cudaStream_t);                         \
  template int restrict_values<T>(const T*, T*, int, int, int, cudaStream_t);           \
  template int restrict_mask<T>(const uint8_t*, const T*, uint8_t*, T*, int, int, int,  \
                                cudaStream_t);                                          \
  template int prolongate<T>(const T*, T*, int, int, int, int, int, cudaStream_t);      \
  template int prolong_add_enforce<T>(const T*, T*, const T*, const uint8_t*, int, int, \
                                      int, int, int, cudaStream_t);                     \
  template int prolong_enforce<T>(const T*, T*, const T*, const uint8_t*, int, int,     \
                                  int, int, int, cudaStream_t);                         \
  template int enforce<T>(T*, const T*, const uint8_t*, int, int, int, int, cudaStream_t);

INST(float)
INST(double)

}  // namespace sp
