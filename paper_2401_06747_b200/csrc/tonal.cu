// tonal.cu -- kernels of the tonal optimizers (tonal.py) on the device.
//
//   cell index        pixels stably sorted by Voronoi label: per-cell sums
//                     then add in row-major order, exactly like np.bincount
//                     (geometry.py:259-272)
//   vi weights        w = (1/ln(2 + sqrt(d2))) / cell_total (geometry.py:247-264)
//   vi step           g[seed_t] += T(tau * sum_cell w (f - u))  (tonal.py:459-464)
//   plane dot         per-(tile, channel) double dots (tonal.py:91-97), one CTA
//                     per plane, deterministic tree
//   plane axpy        y = x + T(coef[plane]) * z for the CG/CGNR vector
//                     updates (tonal.py:246-262, 283-292)
//   tile gather       the 64x64 RAS block copies of the normal-equation rhs
//                     and of the mask (tonal.py:343-354, 376-378)
//   RAS scatter       g += sum over covering blocks (block order) of
//                     T(1/cover) * v_b (tonal.py:297-306, 379-380)
#include <cub/cub.cuh>

#include "geometry.cuh"

namespace sp {

namespace {

constexpr int NT = 256;

__global__ void k_iota32(int* __restrict__ p, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int)i;
}

__global__ void k_bounds(const int* __restrict__ keys, size_t n, int* __restrict__ start,
                         int* __restrict__ end) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = keys[i];
  if (i == 0 || keys[i - 1] != k) start[k] = (int)i;
  if (i == n - 1 || keys[i + 1] != k) end[k] = (int)i + 1;
}

// raw weights 1/ln(2 + sqrt(d2)) ("inverse-log") or 1 ("constant")
__global__ void k_raw_weights(const int* __restrict__ lab, const int* __restrict__ sy,
                              const int* __restrict__ sx, int H, int W, int scheme,
                              double* __restrict__ raw) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)H * W) return;
  if (scheme == 0) {
    raw[i] = 1.0;
    return;
  }
  int y = (int)(i / W), x = (int)(i - (size_t)y * W);
  int s = lab[i];
  long long dy = (long long)y - sy[s], dx = (long long)x - sx[s];
  double d2 = (double)(dy * dy + dx * dx);
  raw[i] = 1.0 / log(2.0 + sqrt(d2));
}

// sequential per-cell sums in pixel order (np.bincount semantics)
__global__ void k_cell_sum(const int* __restrict__ perm, const int* __restrict__ start,
                           const int* __restrict__ end, const double* __restrict__ v, int m,
                           double* __restrict__ out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  double s = 0.0;
  for (int i = start[t]; i < end[t]; ++i) s += v[perm[i]];
  out[t] = s;
}

__global__ void k_normalize(const int* __restrict__ lab, const double* __restrict__ tot,
                            double* __restrict__ w, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = w[i] / tot[lab[i]];
}

// VI update: one thread per (cell, channel)
template <typename T>
__global__ void k_vi_step(const int* __restrict__ perm, const int* __restrict__ start,
                          const int* __restrict__ end, const double* __restrict__ w,
                          const T* __restrict__ f, const T* __restrict__ u,
                          const int* __restrict__ sy, const int* __restrict__ sx, int m, int C,
                          int W, size_t n, double tau, T* __restrict__ g) {
  int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= m * C) return;
  int t = id % m, c = id / m;
  const T* fc = f + (size_t)c * n;
  const T* uc = u + (size_t)c * n;
  double s = 0.0;
  for (int i = start[t]; i < end[t]; ++i) {
    int p = perm[i];
    s += w[p] * ((double)fc[p] - (double)uc[p]);
  }
  size_t k = (size_t)c * n + (size_t)sy[t] * W + sx[t];
  g[k] = g[k] + (T)(tau * s);
}

// out[plane] = sum x*y (mode 1) / x*x (mode 0) over `len` elements
template <typename T>
__global__ void __launch_bounds__(NT) k_plane_dot(const T* __restrict__ x,
                                                  const T* __restrict__ y, size_t len,
                                                  int mode, const int* __restrict__ active,
                                                  int C, double* __restrict__ out) {
  __shared__ double sc[NT / 32];
  const size_t pl = blockIdx.x;
  if (active && !active[pl / C]) return;
  const T* xp = x + pl * len;
  const T* yp = (mode == 1 ? y : x) + pl * len;
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < len; i += NT) acc += (double)xp[i] * (double)yp[i];
  acc = cta_sum<NT>(acc, sc);
  if (threadIdx.x == 0) out[pl] = acc;
}

// y = x + T(coef[plane]) * z (elementwise in T), planes of `len` elements
template <typename T>
__global__ void k_plane_axpy(T* yout, const T* x, const T* z, const double* __restrict__ coef,
                             double sign, size_t len, long nplanes, int C,
                             const int* __restrict__ active) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len * nplanes) return;
  size_t pl = i / len;
  if (active && !active[pl / C]) return;
  const T a = (T)coef[pl];
  const T prod = a * z[i];
  yout[i] = sign > 0 ? (T)(x[i] + prod) : (T)(x[i] - prod);
}

// float planes of a multiple of 4 elements (16-byte aligned): one CTA per
// plane, the plane's active flag and coefficient read once, float4 traffic
// (the per-element kernel above pays a 64-bit division per element)
__global__ void __launch_bounds__(256) k_plane_axpy4(float* yout, const float* x, const float* z,
                                                     const double* __restrict__ coef,
                                                     double sign, int len4, int C,
                                                     const int* __restrict__ active) {
  const long pl = blockIdx.x;
  if (active && !active[pl / C]) return;
  const float a = (float)coef[pl];
  const float4* x4 = reinterpret_cast<const float4*>(x) + pl * len4;
  const float4* z4 = reinterpret_cast<const float4*>(z) + pl * len4;
  float4* y4 = reinterpret_cast<float4*>(yout) + pl * len4;
  for (int i = threadIdx.x; i < len4; i += blockDim.x) {
    const float4 xv = x4[i], zv = z4[i];
    float4 o;
    if (sign > 0) {
      o.x = xv.x + a * zv.x; o.y = xv.y + a * zv.y; o.z = xv.z + a * zv.z; o.w = xv.w + a * zv.w;
    } else {
      o.x = xv.x - a * zv.x; o.y = xv.y - a * zv.y; o.z = xv.z - a * zv.z; o.w = xv.w - a * zv.w;
    }
    y4[i] = o;
  }
}

// rhs tiles [tile][C][bh][bw] from the image (C, H, W) at block origins
template <typename T>
__global__ void k_gather_tiles(const T* __restrict__ img, const int* __restrict__ oy,
                               const int* __restrict__ ox, int ntile, int C, int H, int W,
                               int bh, int bw, T* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t per = (size_t)bh * bw;
  if (i >= per * C * ntile) return;
  size_t pl = i / per, k = i - pl * per;
  int t = (int)(pl / C), c = (int)(pl % C);
  int yy = oy[t] + (int)(k / bw), xx = ox[t] + (int)(k % bw);
  out[i] = img[((size_t)c * H + yy) * W + xx];
}

__global__ void k_gather_mask_tiles(const uint8_t* __restrict__ m, const int* __restrict__ oy,
                                    const int* __restrict__ ox, int ntile, int H, int W, int bh,
                                    int bw, uint8_t* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t per = (size_t)bh * bw;
  if (i >= per * ntile) return;
  int t = (int)(i / per);
  size_t k = i - (size_t)t * per;
  int yy = oy[t] + (int)(k / bw), xx = ox[t] + (int)(k % bw);
  out[i] = m[(size_t)yy * W + xx];
}

// g += upd with upd = sum over covering blocks (ascending block index, only
// blocks that own a tile) of T(1/cover) * v_b, cover = number of covering
// blocks of the full decomposition (tonal.py:297-306, 375-380)
template <typename T>
__global__ void k_ras_scatter(T* __restrict__ g, const T* __restrict__ v,
                              const int* __restrict__ tile_of, const int* __restrict__ ys,
                              const int* __restrict__ xs, const int* __restrict__ row_k0,
                              const int* __restrict__ row_n, const int* __restrict__ col_k0,
                              const int* __restrict__ col_n, int nbx, int bh, int bw, int C,
                              int H, int W) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n = (size_t)H * W;
  if (idx >= n * C) return;
  const int c = (int)(idx / n);
  const size_t k = idx - (size_t)c * n;
  const int y = (int)(k / W), x = (int)(k - (size_t)y * W);
  const int ky0 = row_k0[y], nky = row_n[y], kx0 = col_k0[x], nkx = col_n[x];
  const T w = (T)(1.0 / (double)(nky * nkx));
  T upd = (T)0;
  for (int a = 0; a < nky; ++a)
    for (int b = 0; b < nkx; ++b) {
      const int ky = ky0 + a, kx = kx0 + b;
      const int t = tile_of[ky * nbx + kx];
      if (t < 0) continue;
      const int i = y - ys[ky], j = x - xs[kx];
      upd = upd + w * v[(((size_t)t * C + c) * bh + i) * bw + j];
    }
  g[idx] = g[idx] + upd;
}

// g = where(mask, x, 0)
template <typename T>
__global__ void k_where_mask(const T* __restrict__ x, const uint8_t* __restrict__ m,
                             T* __restrict__ out, int C, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * C) return;
  out[i] = m[i % n] ? x[i] : (T)0;
}

// neighbor_balance_init (tonal.py:389-414): g = T(u + s / cnt) on the mask,
// 0 elsewhere, with s = correlate(f - u, ones(3, 3), mode="constant") and
// cnt = correlate(ones, ones(3, 3)) summed in scipy's footprint order
// (row-major offsets (-1,-1) .. (1,1)); an out-of-image offset adds
// cval * weight = +0.0, which leaves every sum unchanged.  f is the f64 image.
template <typename T>
__global__ void k_neighbor_balance(const double* __restrict__ f, const T* __restrict__ u,
                                   const uint8_t* __restrict__ m, T* __restrict__ g, int C,
                                   int H, int W) {
  const size_t n = (size_t)H * W;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * C) return;
  const size_t p = i % n;
  if (!m[p]) {
    g[i] = (T)0;
    return;
  }
  const int y = (int)(p / W), x = (int)(p - (size_t)y * W);
  const double* fc = f + (i - p);
  const T* uc = u + (i - p);
  double s = 0.0, cnt = 0.0;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int yy = y + dy, xx = x + dx;
      if (yy < 0 || yy >= H || xx < 0 || xx >= W) {
        s = __dadd_rn(s, 0.0);
        cnt = __dadd_rn(cnt, 0.0);
        continue;
      }
      const size_t q = (size_t)yy * W + xx;
      s = __dadd_rn(s, __dsub_rn(fc[q], (double)uc[q]));
      cnt = __dadd_rn(cnt, 1.0);
    }
  g[i] = (T)__dadd_rn((double)u[i], __ddiv_rn(s, cnt));
}

}  // namespace

template <typename T>
int neighbor_balance(const double* f, const T* u, const uint8_t* m, T* g, int C, int H, int W,
                     cudaStream_t s) {
  const size_t n = (size_t)H * W * C;
  if (!n) return 0;
  k_neighbor_balance<T><<<cdiv(n, 256), 256, 0, s>>>(f, u, m, g, C, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

// ---- cell index ----------------------------------------------------------------
int cell_index(const int* lab, int H, int W, long m, int* perm, int* start, int* end,
               cudaStream_t s) {
  size_t n = (size_t)H * W;
  int nbits = 1;
  while ((1L << nbits) < m + 1 && nbits < 31) ++nbits;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const int*)nullptr, (int*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)n, 0, nbits, s);
  Scratch scr(s);
  SP_TRY(scr.alloc(tmp_bytes + sizeof(int) * 2 * n + 64));
  int* keys_out = (int*)scr.p;
  int* iota = keys_out + n;
  void* tmp = (void*)(iota + n + 8);
  k_iota32<<<cdiv(n, 256), 256, 0, s>>>(iota, n);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, lab, keys_out, iota, perm, (int)n, 0,
                                          nbits, s));
  SP_CUDA(cudaMemsetAsync(start, 0, sizeof(int) * m, s));
  SP_CUDA(cudaMemsetAsync(end, 0, sizeof(int) * m, s));
  k_bounds<<<cdiv(n, 256), 256, 0, s>>>(keys_out, n, start, end);
  SP_CHECK_LAUNCH();
  return 0;
}

int vi_weights(const int* lab, const int* sy, const int* sx, const int* perm, const int* start,
               const int* end, int H, int W, long m, int scheme, double* w, cudaStream_t s) {
  size_t n = (size_t)H * W;
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(double) * (size_t)m + 64));
  double* tot = (double*)scr.p;
  k_raw_weights<<<cdiv(n, 256), 256, 0, s>>>(lab, sy, sx, H, W, scheme, w);
  SP_CHECK_LAUNCH();
  k_cell_sum<<<cdiv(m, 128), 128, 0, s>>>(perm, start, end, w, (int)m, tot);
  SP_CHECK_LAUNCH();
  k_normalize<<<cdiv(n, 256), 256, 0, s>>>(lab, tot, w, n);
  SP_CHECK_LAUNCH();
  return 0;
}

int cell_sum(const int* perm, const int* start, const int* end, const double* v, long m,
             double* out, cudaStream_t s) {
  k_cell_sum<<<cdiv(m, 128), 128, 0, s>>>(perm, start, end, v, (int)m, out);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int vi_step(const int* perm, const int* start, const int* end, const double* w, const T* f,
            const T* u, const int* sy, const int* sx, long m, int C, int H, int W, double tau,
            T* g, cudaStream_t s) {
  k_vi_step<T><<<cdiv(m * C, 128), 128, 0, s>>>(perm, start, end, w, f, u, sy, sx, (int)m, C, W,
                                                 (size_t)H * W, tau, g);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int plane_dot(const T* x, const T* y, size_t len, long nplanes, int C, const int* active,
              double* out, cudaStream_t s) {
  if (nplanes <= 0) return 0;
  k_plane_dot<T><<<(unsigned)nplanes, NT, 0, s>>>(x, y, len, y ? 1 : 0, active, C, out);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int plane_axpy(T* yout, const T* x, const T* z, const double* coef, double sign, size_t len,
               long nplanes, int C, const int* active, cudaStream_t s) {
  size_t n = len * nplanes;
  if (!n) return 0;
  if (sizeof(T) == 4 && len % 4 == 0 && len / 4 < (1u << 30) &&
      ((((uintptr_t)yout) | ((uintptr_t)x) | ((uintptr_t)z)) & 15) == 0) {
    // same operations per element: a = T(coef), x +- a * z (no contraction)
    k_plane_axpy4<<<(unsigned)nplanes, 256, 0, s>>>((float*)yout, (const float*)x,
                                                    (const float*)z, coef, sign, (int)(len / 4),
                                                    C, active);
    SP_CHECK_LAUNCH();
    return 0;
  }
  k_plane_axpy<T><<<cdiv(n, 256), 256, 0, s>>>(yout, x, z, coef, sign, len, nplanes, C, active);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int gather_tiles(const T* img, const int* oy, const int* ox, int ntile, int C, int H, int W,
                 int bh, int bw, T* out, cudaStream_t s) {
  size_t n = (size_t)bh * bw * C * ntile;
  if (!n) return 0;
  k_gather_tiles<T><<<cdiv(n, 256), 256, 0, s>>>(img, oy, ox, ntile, C, H, W, bh, bw, out);
  SP_CHECK_LAUNCH();
  return 0;
}

int gather_mask_tiles(const uint8_t* m, const int* oy, const int* ox, int ntile, int H, int W,
                      int bh, int bw, uint8_t* out, cudaStream_t s) {
  size_t n = (size_t)bh * bw * ntile;
  if (!n) return 0;
  k_gather_mask_tiles<<<cdiv(n, 256), 256, 0, s>>>(m, oy, ox, ntile, H, W, bh, bw, out);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int ras_scatter(T* g, const T* v, const int* tile_of, const int* ys, const int* xs,
                const int* row_k0, const int* row_n, const int* col_k0, const int* col_n,
                int nbx, int bh, int bw, int C, int H, int W, cudaStream_t s) {
  size_t n = (size_t)H * W * C;
  k_ras_scatter<T><<<cdiv(n, 256), 256, 0, s>>>(g, v, tile_of, ys, xs, row_k0, row_n, col_k0,
                                                col_n, nbx, bh, bw, C, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int where_mask(const T* x, const uint8_t* m, T* out, int C, int H, int W, cudaStream_t s) {
  size_t n = (size_t)H * W;
  k_where_mask<T><<<cdiv(n * C, 256), 256, 0, s>>>(x, m, out, C, n);
  SP_CHECK_LAUNCH();
  return 0;
}

#define INST(T)                                                                              \
  template int vi_step<T>(const int*, const int*, const int*, const double*, const T*,        \
                          const T*, const int*, const int*, long, int, int, int, double, T*,  \
                          cudaStream_t);                                                      \
  template int plane_dot<T>(const T*, const T*, size_t, long, int, const int*, double*,       \
                            cudaStream_t);                                                    \
  template int plane_axpy<T>(T*, const T*, const T*, const double*, double, size_t, long, int, \
                             const int*, cudaStream_t);                                       \
  template int gather_tiles<T>(const T*, const int*, const int*, int, int, int, int, int, int, \
                               T*, cudaStream_t);                                             \
  template int ras_scatter<T>(T*, const T*, const int*, const int*, const int*, const int*,   \
                              const int*, const int*, const int*, int, int, int, int, int,    \
                              int, cudaStream_t);                                             \
  template int where_mask<T>(const T*, const uint8_t*, T*, int, int, int, cudaStream_t);     \
  template int neighbor_balance<T>(const double*, const T*, const uint8_t*, T*, int, int, int, \
                                   cudaStream_t);
INST(float)
INST(double)

}  // namespace sp
