// stencil.cu -- stencil / transfer kernels used only through the kernel
// table (boundary B1): negated_laplacian, inpaint_matvec, sym_matvec,
// restrict_values, prolongate.  The multigrid path uses the persistent
// kernels of mg.cu.
//
// Reference semantics: numba_impl.py:13-98, 266-284, 316-348.  Every stencil
// accumulates in double in the reference order (up, down, left, right) and
// rounds once to T, so outputs are bit-identical to the CPU oracle.
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int BX = 32, BY = 8;

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

// A~ x = C x + (I-C) L (I-C) x (numba_impl.py:68-98)
template <typename T>
__global__ void k_sym_matvec(const T* __restrict__ x, const uint8_t* __restrict__ m,
                             T* __restrict__ out, int C, int H, int W, double inv_h2) {
  int xx = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (xx >= W || y >= H) return;
  size_t plane = (size_t)H * W, k = (size_t)y * W + xx;
  bool mk = m[k];
  for (int c = 0; c < C; ++c) {
    const T* xc = x + c * plane;
    if (mk) { out[c * plane + k] = xc[k]; continue; }
    double d = 0.0, a = 0.0;
    if (y > 0) { d += 1.0; if (!m[k - W]) a += (double)xc[k - W]; }
    if (y < H - 1) { d += 1.0; if (!m[k + W]) a += (double)xc[k + W]; }
    if (xx > 0) { d += 1.0; if (!m[k - 1]) a += (double)xc[k - 1]; }
    if (xx < W - 1) { d += 1.0; if (!m[k + 1]) a += (double)xc[k + 1]; }
    out[c * plane + k] = (T)((d * (double)xc[k] - a) * inv_h2);
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

// cell-centred bilinear interpolation, clamped (numba_impl.py:316-348)
__device__ __forceinline__ void axis_w(int y, int n, int& y0, int& y1, double& wy) {
  double fy = ((double)y + 0.5) / 2.0 - 0.5;
  y0 = (int)floor(fy);
  wy = fy - (double)y0;
  if (y0 < 0) { y0 = 0; wy = 0.0; }
  if (y0 > n - 1) { y0 = n - 1; wy = 0.0; }
  y1 = min(y0 + 1, n - 1);
}

template <typename T>
__global__ void k_prolongate(const T* __restrict__ co, T* __restrict__ out, int C,
                             int chh, int cww, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  int y0, y1, x0, x1;
  double wy, wx;
  axis_w(y, chh, y0, y1, wy);
  axis_w(x, cww, x0, x1, wx);
  size_t plane = (size_t)H * W, cplane = (size_t)chh * cww;
  for (int c = 0; c < C; ++c) {
    const T* cc = co + c * cplane;
    double v = (1.0 - wy) * ((1.0 - wx) * (double)cc[(size_t)y0 * cww + x0] +
                             wx * (double)cc[(size_t)y0 * cww + x1]) +
               wy * ((1.0 - wx) * (double)cc[(size_t)y1 * cww + x0] +
                     wx * (double)cc[(size_t)y1 * cww + x1]);
    out[c * plane + (size_t)y * W + x] = (T)v;
  }
}

inline dim3 grid2(int W, int H) { return dim3(cdiv(W, BX), cdiv(H, BY)); }
const dim3 kBlock(BX, BY);

}  // namespace

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
int restrict_values(const T* f, T* out, int C, int H, int W, cudaStream_t s) {
  k_restrict_values<T><<<grid2((W + 1) / 2, (H + 1) / 2), kBlock, 0, s>>>(f, out, C, H, W);
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

#define INST(T)                                                                     \
  template int neglap<T>(const T*, T*, int, int, int, double, cudaStream_t);          \
  template int inpaint_matvec<T>(const T*, const uint8_t*, T*, int, int, int, double, \
                                 cudaStream_t);                                       \
  template int sym_matvec<T>(const T*, const uint8_t*, T*, int, int, int, double,     \
                             cudaStream_t);                                           \
  template int restrict_values<T>(const T*, T*, int, int, int, cudaStream_t);         \
  template int prolongate<T>(const T*, T*, int, int, int, int, int, cudaStream_t);

INST(float)
INST(double)

}  // namespace sp
