// mg.cu -- multigrid level kernels (sm_100a), persistent grid-stride form.
//
// Reference semantics (bit-identical per element; double accumulation in
// the reference order, one rounding to T):
//   sym_rhs        numba_impl.py:101-121      ct_apply   :124-144
//   sym_residual   numba_impl.py:147-158      restrict_values/_mask :266-313
//   prolongate     numba_impl.py:316-348      _enforce   solver.py:275-281
//
// Layout: a launch covers `nz = ntile * C` planes ([tile][C][H][W] vectors,
// [tile][H][W] masks).  The grid is (nbx, nz): CTA (bx, z) walks the
// plane's 32x8 pixel tiles with stride nbx.  nbx is chosen so that the
// whole launch is about two waves of resident CTAs (148 SMs x 8): each
// thread handles many pixels, so CTA launch / wave-transition overhead
// (~2.4k cycles per wave) no longer dominates these HBM-bound sweeps.
// `active` (nullable, [ntile]) switches whole tiles off (per-tile stopping
// of the batched RAS block solves).
#include <initializer_list>

#include "kernels.cuh"

namespace sp {

namespace {

constexpr int BX = 32, BY = 8, NT = BX * BY;
constexpr long kTargetCtas = 2 * 148 * 8;
constexpr size_t kNrmSlots = 4096;  // partial slots of the fused ||b~||^2 (>= the grid)

struct PlaneTiles {
  int ntx, nty;
  int per_plane;
};

__host__ __device__ inline PlaneTiles plane_tiles(int H, int W) {
  PlaneTiles p;
  p.ntx = (W + BX - 1) / BX;
  p.nty = (H + BY - 1) / BY;
  p.per_plane = p.ntx * p.nty;
  return p;
}

inline dim3 mg_grid(int H, int W, long nz) {
  PlaneTiles p = plane_tiles(H, W);
  long nbx = (kTargetCtas + nz - 1) / nz;
  if (nbx < 1) nbx = 1;
  if (nbx > p.per_plane) nbx = p.per_plane;
  return dim3((unsigned)nbx, (unsigned)nz, 1);
}

// iterate over this CTA's tiles of plane z: x, y are the thread's pixel
#define FOR_PIXELS(H, W)                                                      \
  const PlaneTiles _pt = plane_tiles(H, W);                                   \
  for (int _t = blockIdx.x; _t < _pt.per_plane; _t += gridDim.x)              \
    for (int _once = 1, y = (_t / _pt.ntx) * BY + threadIdx.y,                \
                        x = (_t % _pt.ntx) * BX + threadIdx.x;                \
         _once; _once = 0)

#define PLANE_SETUP(C)                                                       \
  const int z = blockIdx.y, tile = z / (C), c = z - tile * (C);              \
  (void)c;                                                                   \
  if (active && !active[tile]) return;

// unmasked-pixel row of A~ x (numba_impl.py:78-97)
template <typename T>
__device__ __forceinline__ T sym_row_at(const T* __restrict__ xc,
                                        const uint8_t* __restrict__ m, size_t k, int y,
                                        int x, int H, int W, double inv_h2) {
  double d = 0.0, a = 0.0;
  if (y > 0) { d += 1.0; if (!m[k - W]) a += (double)xc[k - W]; }
  if (y < H - 1) { d += 1.0; if (!m[k + W]) a += (double)xc[k + W]; }
  if (x > 0) { d += 1.0; if (!m[k - 1]) a += (double)xc[k - 1]; }
  if (x < W - 1) { d += 1.0; if (!m[k + 1]) a += (double)xc[k + 1]; }
  return (T)((d * (double)xc[k] - a) * inv_h2);
}

// C~ b; optionally e = mask ? out : 0 (solver.py:289-292)
template <typename T>
__global__ void __launch_bounds__(NT) k_sym_rhs(const T* __restrict__ b,
                                                const uint8_t* __restrict__ m,
                                                T* __restrict__ out, T* __restrict__ e,
                                                int C, int H, int W, double inv_h2,
                                                const int* __restrict__ active) {
  pdl_enter();
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* bc = b + vo;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    bool mk = m[k];
    T o;
    if (mk) {
      o = bc[k];
    } else {
      double a = 0.0;
      if (y > 0 && m[k - W]) a += (double)bc[k - W];
      if (y < H - 1 && m[k + W]) a += (double)bc[k + W];
      if (x > 0 && m[k - 1]) a += (double)bc[k - 1];
      if (x < W - 1 && m[k + 1]) a += (double)bc[k + 1];
      o = (T)((double)bc[k] + a * inv_h2);
    }
    out[vo + k] = o;
    if (e) e[vo + k] = mk ? o : (T)0;
  }
}

// sym_rhs(where(mask, x, 0)) fused (tonal.py:136-137, solver.py:501-502)
template <typename T>
__global__ void __launch_bounds__(NT) k_masked_sym_rhs(const T* __restrict__ xs,
                                                       const uint8_t* __restrict__ m,
                                                       T* __restrict__ out, int C, int H,
                                                       int W, const int* __restrict__ active) {
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* xc = xs + vo;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    T o;
    if (m[k]) {
      o = xc[k];
    } else {
      // b(k) = 0 off-mask; the reference adds 0.0 + acc (exact)
      double a = 0.0;
      if (y > 0 && m[k - W]) a += (double)xc[k - W];
      if (y < H - 1 && m[k + W]) a += (double)xc[k + W];
      if (x > 0 && m[k - 1]) a += (double)xc[k - 1];
      if (x < W - 1 && m[k + 1]) a += (double)xc[k + 1];
      o = (T)(0.0 + a);
    }
    out[vo + k] = o;
  }
}

// (C - C L (I-C)) w, zero off-mask
template <typename T>
__global__ void __launch_bounds__(NT) k_ct_apply(const T* __restrict__ w,
                                                 const uint8_t* __restrict__ m,
                                                 T* __restrict__ out, int C, int H, int W,
                                                 double inv_h2,
                                                 const int* __restrict__ active) {
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* wc = w + vo;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    if (!m[k]) { out[vo + k] = (T)0; continue; }
    double a = 0.0;
    if (y > 0 && !m[k - W]) a += (double)wc[k - W];
    if (y < H - 1 && !m[k + W]) a += (double)wc[k + W];
    if (x > 0 && !m[k - 1]) a += (double)wc[k - 1];
    if (x < W - 1 && !m[k + 1]) a += (double)wc[k + 1];
    out[vo + k] = (T)((double)wc[k] + a * inv_h2);
  }
}

// r = b~ - A~ u in T; sum r^2 per plane in double, deterministically: each
// thread sums its pixels in a fixed order, CTA tree, then the last CTA of the
// plane adds the per-CTA partials in index order.
template <typename T>
__global__ void __launch_bounds__(NT) k_residual(
    const T* __restrict__ u, const T* __restrict__ b, const uint8_t* __restrict__ m,
    T* __restrict__ r, double* __restrict__ partial, unsigned* __restrict__ counter,
    double* __restrict__ norms, int C, int H, int W, double inv_h2,
    const int* __restrict__ active) {
  pdl_enter();
  __shared__ double s0[NT / 32];
  __shared__ bool am_last;
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* uc = u + vo;
  const T* bc = b + vo;
  double sq = 0.0;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    T ax = m[k] ? uc[k] : sym_row_at(uc, m, k, y, x, H, W, inv_h2);
    T rv = (T)(bc[k] - ax);
    if (r) r[vo + k] = rv;
    sq += (double)rv * (double)rv;
  }
  if (!norms) return;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const unsigned nblk = gridDim.x;
  double s = cta_sum<NT>(sq, s0);
  if (nblk == 1) {
    if (tid == 0) norms[z] = s;
    return;
  }
  if (tid == 0) {
    partial[(size_t)z * nblk + blockIdx.x] = s;
    __threadfence();
    am_last = atomicAdd(counter + z, 1u) == nblk - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned i = tid; i < nblk; i += NT) t += ((volatile double*)partial)[(size_t)z * nblk + i];
  t = cta_sum<NT>(t, s0);
  if (tid == 0) {
    norms[z] = t;
    counter[z] = 0u;
  }
}

// fused residual + 2x2 restriction (solver.py:289-290).  Each thread
// computes one fine residual (T); the 2x2 groups are combined through shared
// memory in the reference's row-major order ((a + b) + c) + d in double.
template <typename T>
__global__ void __launch_bounds__(NT) k_residual_restrict(
    const T* __restrict__ u, const T* __restrict__ b, const uint8_t* __restrict__ m,
    T* __restrict__ rc, int C, int H, int W, double inv_h2, const int* __restrict__ active) {
  pdl_enter();
  __shared__ T rs[BY][BX + 1];
  PLANE_SETUP(C);
  const int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* uc = u + vo;
  const T* bc = b + vo;
  T* out = rc + (size_t)z * ch_ * cw;
  FOR_PIXELS(H, W) {
    if (x < W && y < H) {
      size_t k = (size_t)y * W + x;
      T ax = m[k] ? uc[k] : sym_row_at(uc, m, k, y, x, H, W, inv_h2);
      rs[threadIdx.y][threadIdx.x] = (T)(bc[k] - ax);
    }
    __syncthreads();
    if (!(threadIdx.x & 1) && !(threadIdx.y & 1) && x < W && y < H) {
      const int ty = threadIdx.y, tx = threadIdx.x;
      bool xr = x + 1 < W, yd = y + 1 < H;
      double acc = (double)rs[ty][tx];
      int n = 1;
      if (xr) { acc += (double)rs[ty][tx + 1]; ++n; }
      if (yd) { acc += (double)rs[ty + 1][tx]; ++n; }
      if (xr && yd) { acc += (double)rs[ty + 1][tx + 1]; ++n; }
      out[(size_t)(y >> 1) * cw + (x >> 1)] = (T)(acc / (double)n);
    }
    __syncthreads();
  }
}

// OR mask + mean of covered stored values (numba_impl.py:287-313); one
// thread per coarse pixel, all channels
template <typename T>
__global__ void __launch_bounds__(NT) k_restrict_mask(const uint8_t* __restrict__ m,
                                                      const T* __restrict__ v,
                                                      uint8_t* __restrict__ cm,
                                                      T* __restrict__ cv, int C, int H, int W) {
  const int tile = blockIdx.y;
  const int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  const size_t plane = (size_t)H * W, cplane = (size_t)ch_ * cw;
  m += (size_t)tile * plane;
  cm += (size_t)tile * cplane;
  if (v) v += (size_t)tile * C * plane;
  if (cv) cv += (size_t)tile * C * cplane;
  FOR_PIXELS(ch_, cw) {
    const int i = y, j = x;
    if (j >= cw || i >= ch_) continue;
    size_t ck = (size_t)i * cw + j;
    int y1 = min(2 * i + 2, H), x1 = min(2 * j + 2, W);
    int cnt = 0;
    for (int yy = 2 * i; yy < y1; ++yy)
      for (int xx = 2 * j; xx < x1; ++xx) cnt += m[(size_t)yy * W + xx] ? 1 : 0;
    cm[ck] = cnt > 0;
    if (!cv) continue;
    for (int cc = 0; cc < C; ++cc) {
      T o = (T)0;
      if (cnt) {
        double acc = 0.0;
        for (int yy = 2 * i; yy < y1; ++yy)
          for (int xx = 2 * j; xx < x1; ++xx)
            if (m[(size_t)yy * W + xx]) acc += (double)v[cc * plane + (size_t)yy * W + xx];
        o = (T)(acc / (double)cnt);
      }
      cv[cc * cplane + ck] = o;
    }
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

// u += prolongate(e); u[mask] = b~[mask] (solver.py:294-296); with
// add == 0 the FMG step u = prolongate(uc); enforce (solver.py:309-312)
template <typename T>
__global__ void __launch_bounds__(NT) k_prolong_enforce(
    const T* __restrict__ e, T* __restrict__ u, const T* __restrict__ b,
    const uint8_t* __restrict__ m, int C, int chh, int cww, int H, int W, int add,
    const int* __restrict__ active) {
  pdl_enter();
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* ec = e + (size_t)z * chh * cww;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    if (m[k]) {
      u[vo + k] = b[vo + k];
      continue;
    }
    int y0, y1, x0, x1;
    double wy, wx;
    prolong_axis(y, chh, y0, y1, wy);
    prolong_axis(x, cww, x0, x1, wx);
    double v = (1.0 - wy) * ((1.0 - wx) * (double)ec[(size_t)y0 * cww + x0] +
                             wx * (double)ec[(size_t)y0 * cww + x1]) +
               wy * ((1.0 - wx) * (double)ec[(size_t)y1 * cww + x0] +
                     wx * (double)ec[(size_t)y1 * cww + x1]);
    T p = (T)v;
    u[vo + k] = add ? (T)(u[vo + k] + p) : p;
  }
}

// u[mask] = src[mask]; optional zero elsewhere
template <typename T>
__global__ void __launch_bounds__(NT) k_enforce(T* __restrict__ u, const T* __restrict__ src,
                                                const uint8_t* __restrict__ m, int C, int H,
                                                int W, int zero_off,
                                                const int* __restrict__ active) {
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  FOR_PIXELS(H, W) {
    if (x >= W || y >= H) continue;
    size_t k = (size_t)y * W + x;
    if (m[k]) u[vo + k] = src[vo + k];
    else if (zero_off) u[vo + k] = (T)0;
  }
}

// ===========================================================================
// Vectorized forms (W % 4 == 0, 16-byte aligned planes): every thread owns a
// quad of 4 consecutive pixels of a row, the CTA a 128 x 8 pixel tile.  Row
// neighbours come from one wide load each, the left/right halo from two
// scalar loads; the tile index math is paid once per 1024 pixels.  Element
// arithmetic is unchanged (same double accumulation order), so the results
// are bit-identical to the scalar kernels.
// ===========================================================================

template <typename T>
struct V4 {
  T a[4];
};

__device__ __forceinline__ V4<float> ld4(const float* p) {
  float4 v = *reinterpret_cast<const float4*>(p);
  return {{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
  double2 v0 = reinterpret_cast<const double2*>(p)[0];
  double2 v1 = reinterpret_cast<const double2*>(p)[1];
  return {{v0.x, v0.y, v1.x, v1.y}};
}
__device__ __forceinline__ void st4(float* p, const V4<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.a[0], v.a[1], v.a[2], v.a[3]);
}
__device__ __forceinline__ void st4(double* p, const V4<double>& v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v.a[0], v.a[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.a[2], v.a[3]);
}
template <typename T>
__device__ __forceinline__ V4<T> zero4() {
  return {{(T)0, (T)0, (T)0, (T)0}};
}
__device__ __forceinline__ uint32_t ldm4(const uint8_t* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ bool mbit(uint32_t w, int i) { return (w >> (8 * i)) & 0xFFu; }

// iterate over this CTA's 128x8 tiles of the plane; x0 is the quad start
#define FOR_QUADS(H, W)                                                       \
  const int _ntx = ((W) / 4 + BX - 1) / BX;                                   \
  const int _per = _ntx * (((H) + BY - 1) / BY);                              \
  for (int _t = blockIdx.x; _t < _per; _t += gridDim.x)                       \
    for (int _once = 1, y = (_t / _ntx) * BY + threadIdx.y,                   \
                        x0 = ((_t % _ntx) * BX + threadIdx.x) * 4;            \
         _once; _once = 0)

inline dim3 mg_grid4(int H, int W, long nz) {
  long per = (long)((W / 4 + BX - 1) / BX) * ((H + BY - 1) / BY);
  long nbx = (kTargetCtas + nz - 1) / nz;
  if (nbx < 1) nbx = 1;
  if (nbx > per) nbx = per;
  return dim3((unsigned)nbx, (unsigned)nz, 1);
}

// the four neighbour rows/columns of a quad (masks as packed bytes)
template <typename T>
struct Quad {
  uint32_t mc, mu, md;
  bool hu, hd, hl, hr;
  uint8_t ml, mr;
  V4<T> c, up, dn;
  T l, r;
};

template <typename T>
__device__ __forceinline__ void load_quad(Quad<T>& q, const T* __restrict__ xc,
                                          const uint8_t* __restrict__ m, size_t k, int x0,
                                          int y, int H, int W, bool need_vals) {
  q.hu = y > 0;
  q.hd = y < H - 1;
  q.hl = x0 > 0;
  q.hr = x0 + 4 < W;
  q.mc = ldm4(m + k);
  q.mu = q.hu ? ldm4(m + k - W) : 0u;
  q.md = q.hd ? ldm4(m + k + W) : 0u;
  q.ml = q.hl ? m[k - 1] : (uint8_t)0;
  q.mr = q.hr ? m[k + 4] : (uint8_t)0;
  if (need_vals) {
    q.c = ld4(xc + k);
    q.up = q.hu ? ld4(xc + k - W) : zero4<T>();
    q.dn = q.hd ? ld4(xc + k + W) : zero4<T>();
    q.l = q.hl ? xc[k - 1] : (T)0;
    q.r = q.hr ? xc[k + 4] : (T)0;
  }
}

// neighbour i of the quad: exists / masked / value, in the order up, down,
// left, right of numba_impl.py:78-97
template <typename T>
__device__ __forceinline__ T sym_quad(const Quad<T>& q, int i, double inv_h2) {
  double d = 0.0, a = 0.0;
  if (q.hu) { d += 1.0; if (!mbit(q.mu, i)) a += (double)q.up.a[i]; }
  if (q.hd) { d += 1.0; if (!mbit(q.md, i)) a += (double)q.dn.a[i]; }
  if (i > 0 || q.hl) {
    d += 1.0;
    bool lm = i > 0 ? mbit(q.mc, i - 1) : (bool)q.ml;
    if (!lm) a += (double)(i > 0 ? q.c.a[i - 1] : q.l);
  }
  if (i < 3 || q.hr) {
    d += 1.0;
    bool rm = i < 3 ? mbit(q.mc, i + 1) : (bool)q.mr;
    if (!rm) a += (double)(i < 3 ? q.c.a[i + 1] : q.r);
  }
  return (T)((d * (double)q.c.a[i] - a) * inv_h2);
}

// sum of the MASKED (want_masked) or UNMASKED neighbours (sym_rhs / ct_apply)
template <typename T>
__device__ __forceinline__ double nbr_sum_quad(const Quad<T>& q, int i, bool want_masked) {
  double a = 0.0;
  if (q.hu && mbit(q.mu, i) == want_masked) a += (double)q.up.a[i];
  if (q.hd && mbit(q.md, i) == want_masked) a += (double)q.dn.a[i];
  if (i > 0 || q.hl) {
    bool lm = i > 0 ? mbit(q.mc, i - 1) : (bool)q.ml;
    if (lm == want_masked) a += (double)(i > 0 ? q.c.a[i - 1] : q.l);
  }
  if (i < 3 || q.hr) {
    bool rm = i < 3 ? mbit(q.mc, i + 1) : (bool)q.mr;
    if (rm == want_masked) a += (double)(i < 3 ? q.c.a[i + 1] : q.r);
  }
  return a;
}

template <typename T>
__global__ void __launch_bounds__(NT) k4_residual(
    const T* __restrict__ u, const T* __restrict__ b, const uint8_t* __restrict__ m,
    T* __restrict__ r, double* __restrict__ partial, unsigned* __restrict__ counter,
    double* __restrict__ norms, int C, int H, int W, double inv_h2,
    const int* __restrict__ active) {
  pdl_enter();
  __shared__ double s0[NT / 32];
  __shared__ bool am_last;
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* uc = u + vo;
  const T* bc = b + vo;
  double sq = 0.0;
  FOR_QUADS(H, W) {
    if (x0 >= W || y >= H) continue;
    size_t k = (size_t)y * W + x0;
    Quad<T> q;
    load_quad(q, uc, m, k, x0, y, H, W, true);
    V4<T> bb = ld4(bc + k), rr;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      T ax = mbit(q.mc, i) ? q.c.a[i] : sym_quad(q, i, inv_h2);
      rr.a[i] = (T)(bb.a[i] - ax);
      sq += (double)rr.a[i] * (double)rr.a[i];
    }
    if (r) st4(r + vo + k, rr);
  }
  if (!norms) return;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const unsigned nblk = gridDim.x;
  double s = cta_sum<NT>(sq, s0);
  if (nblk == 1) {
    if (tid == 0) norms[z] = s;
    return;
  }
  if (tid == 0) {
    partial[(size_t)z * nblk + blockIdx.x] = s;
    __threadfence();
    am_last = atomicAdd(counter + z, 1u) == nblk - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned i = tid; i < nblk; i += NT) t += ((volatile double*)partial)[(size_t)z * nblk + i];
  t = cta_sum<NT>(t, s0);
  if (tid == 0) {
    norms[z] = t;
    counter[z] = 0u;
  }
}

// mode 0: sym_rhs (+ optional e); 1: masked_sym_rhs; 2: ct_apply
// NRM (one image, MODE 1): also the sum of out^2 over all planes -- the
// ||b~||^2 of the solve's tolerance scale (solver.py:351-352) -- in the same
// pass: per-thread double sums, CTA partials in grid order, the last CTA of
// the grid adds them in index order (deterministic)
template <typename T, int MODE, bool NRM = false>
__global__ void __launch_bounds__(NT) k4_rhs(const T* __restrict__ xin,
                                             const uint8_t* __restrict__ m,
                                             T* __restrict__ out, T* __restrict__ e, int C,
                                             int H, int W, double inv_h2,
                                             const int* __restrict__ active,
                                             double* __restrict__ partial,
                                             unsigned* __restrict__ counter,
                                             double* __restrict__ nrm) {
  pdl_enter();
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* xc = xin + vo;
  double nacc = 0.0;
  FOR_QUADS(H, W) {
    if (x0 >= W || y >= H) continue;
    size_t k = (size_t)y * W + x0;
    Quad<T> q;
    load_quad(q, xc, m, k, x0, y, H, W, true);
    V4<T> o, ee;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      bool mk = mbit(q.mc, i);
      if (MODE == 0) {
        o.a[i] = mk ? q.c.a[i] : (T)((double)q.c.a[i] + nbr_sum_quad(q, i, true) * inv_h2);
        ee.a[i] = mk ? o.a[i] : (T)0;
      } else if (MODE == 1) {
        o.a[i] = mk ? q.c.a[i] : (T)(0.0 + nbr_sum_quad(q, i, true));
        // fused enforce (solver.py:275-281): u = b~ on the stored pixels
        if (e && mk) e[vo + k + i] = o.a[i];
      } else {
        o.a[i] = mk ? (T)((double)q.c.a[i] + nbr_sum_quad(q, i, false) * inv_h2) : (T)0;
      }
    }
    st4(out + vo + k, o);
    if (MODE == 0 && e) st4(e + vo + k, ee);
    if (NRM) {
#pragma unroll
      for (int i = 0; i < 4; ++i) nacc += (double)o.a[i] * (double)o.a[i];
    }
  }
  if (!NRM) return;
  // one partial per CTA (grid order); k_sum_parts adds them in index order --
  // no atomics: with the grid-stride loop every CTA ends at the same time
  __shared__ double s0[NT / 32];
  const double sb = cta_sum<NT>(nacc, s0);
  if (threadIdx.y * BX + threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = sb;
}

__global__ void __launch_bounds__(1024) k_sum_parts(const double* __restrict__ partial, int n,
                                                    double* __restrict__ total) {
  __shared__ double s0[1024 / 32];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) t += partial[i];
  t = cta_sum<1024>(t, s0);
  if (threadIdx.x == 0) *total = t;
}

template <typename T>
__global__ void __launch_bounds__(NT) k4_enforce(T* __restrict__ u, const T* __restrict__ src,
                                                 const uint8_t* __restrict__ m, int C, int H,
                                                 int W, int zero_off,
                                                 const int* __restrict__ active) {
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  FOR_QUADS(H, W) {
    if (x0 >= W || y >= H) continue;
    size_t k = (size_t)y * W + x0;
    uint32_t mc = ldm4(m + k);
    if (!mc && !zero_off) continue;
    V4<T> s4 = mc ? ld4(src + vo + k) : zero4<T>();
    V4<T> u4 = (mc == 0x01010101u || zero_off) ? zero4<T>() : ld4(u + vo + k);
#pragma unroll
    for (int i = 0; i < 4; ++i) u4.a[i] = mbit(mc, i) ? s4.a[i] : (zero_off ? (T)0 : u4.a[i]);
    st4(u + vo + k, u4);
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) k4_prolong_enforce(
    const T* __restrict__ e, T* __restrict__ u, const T* __restrict__ b,
    const uint8_t* __restrict__ m, int C, int chh, int cww, int H, int W, int add,
    const int* __restrict__ active) {
  pdl_enter();
  PLANE_SETUP(C);
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* ec = e + (size_t)z * chh * cww;
  FOR_QUADS(H, W) {
    if (x0 >= W || y >= H) continue;
    size_t k = (size_t)y * W + x0;
    uint32_t mc = ldm4(m + k);
    V4<T> bb = mc ? ld4(b + vo + k) : zero4<T>();
    V4<T> uu = add ? ld4(u + vo + k) : zero4<T>();
    int y0, y1;
    double wy;
    prolong_axis(y, chh, y0, y1, wy);
    const T* r0 = ec + (size_t)y0 * cww;
    const T* r1 = ec + (size_t)y1 * cww;
    V4<T> o;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (mbit(mc, i)) {
        o.a[i] = bb.a[i];
        continue;
      }
      int xa, xb;
      double wx;
      prolong_axis(x0 + i, cww, xa, xb, wx);
      double v = (1.0 - wy) * ((1.0 - wx) * (double)r0[xa] + wx * (double)r0[xb]) +
                 wy * ((1.0 - wx) * (double)r1[xa] + wx * (double)r1[xb]);
      T p = (T)v;
      o.a[i] = add ? (T)(uu.a[i] + p) : p;
    }
    st4(u + vo + k, o);
  }
}

// residual + 2x2 restriction: the CTA's 128x8 fine tile maps to 64x4 coarse
// pixels, one per thread, combined from shared memory in row-major order
template <typename T>
__global__ void __launch_bounds__(NT) k4_residual_restrict(
    const T* __restrict__ u, const T* __restrict__ b, const uint8_t* __restrict__ m,
    T* __restrict__ rc, int C, int H, int W, double inv_h2, const int* __restrict__ active) {
  pdl_enter();
  __shared__ T rs[BY][4 * BX + 1];
  PLANE_SETUP(C);
  const int ch_ = (H + 1) / 2, cw = (W + 1) / 2;
  const size_t plane = (size_t)H * W, vo = (size_t)z * plane;
  m += (size_t)tile * plane;
  const T* uc = u + vo;
  const T* bc = b + vo;
  T* out = rc + (size_t)z * ch_ * cw;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const int ci = tid / 64, cj = tid % 64;  // coarse pixel of this thread in the tile
  FOR_QUADS(H, W) {
    if (x0 < W && y < H) {
      size_t k = (size_t)y * W + x0;
      Quad<T> q;
      load_quad(q, uc, m, k, x0, y, H, W, true);
      V4<T> bb = ld4(bc + k);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        T ax = mbit(q.mc, i) ? q.c.a[i] : sym_quad(q, i, inv_h2);
        rs[threadIdx.y][threadIdx.x * 4 + i] = (T)(bb.a[i] - ax);
      }
    }
    __syncthreads();
    {
      const int ty0 = (_t / _ntx) * BY, tx0 = (_t % _ntx) * BX * 4;
      const int fy = ty0 + 2 * ci, fx = tx0 + 2 * cj;
      if (fy < H && fx < W) {
        const bool xr = fx + 1 < W, yd = fy + 1 < H;
        double acc = (double)rs[2 * ci][2 * cj];
        int n = 1;
        if (xr) { acc += (double)rs[2 * ci][2 * cj + 1]; ++n; }
        if (yd) { acc += (double)rs[2 * ci + 1][2 * cj]; ++n; }
        if (xr && yd) { acc += (double)rs[2 * ci + 1][2 * cj + 1]; ++n; }
        out[(size_t)(fy >> 1) * cw + (fx >> 1)] = (T)(acc / (double)n);
      }
    }
    __syncthreads();
  }
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

const dim3 kBlock(BX, BY);

}  // namespace

size_t residual_partials(int H, int W) {
  // per-plane partial slots; mg_grid never exceeds this many CTAs per plane
  PlaneTiles p = plane_tiles(H, W);
  long cap = kTargetCtas;
  return (size_t)(p.per_plane < cap ? p.per_plane : cap);
}

#define VEC_OK(...) (W % 4 == 0 && all_aligned({__VA_ARGS__}))
static bool all_aligned(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (p && !aligned16(p)) return false;
  return true;
}

template <typename T>
int sym_rhs(const T* b, const uint8_t* m, T* out, T* e, int C, int H, int W, double inv_h2,
            cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(b, m, out, e))
    SP_CUDA(launch_k(k4_rhs<T, 0>, mg_grid4(H, W, nz), kBlock, 0, s, b, m, out, e, C, H, W, inv_h2, active,
                     (double*)nullptr, (unsigned*)nullptr, (double*)nullptr));
  else
    SP_CUDA(launch_k(k_sym_rhs<T>, mg_grid(H, W, nz), kBlock, 0, s, b, m, out, e, C, H, W, inv_h2, active));
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int masked_sym_rhs(const T* x, const uint8_t* m, T* out, int C, int H, int W, cudaStream_t s,
                   int ntile, const int* active, T* enforce_u, double* nrm, double* partial,
                   unsigned* counter) {
  long nz = (long)ntile * C;
  if (nrm && !(ntile == 1 && VEC_OK(x, m, out) && partial && counter)) {
    set_error("fused ||b~||^2: one image, aligned quads");
    return -2;
  }
  if (VEC_OK(x, m, out)) {
    const dim3 g = mg_grid4(H, W, nz);
    if (nrm) {
      if ((size_t)g.x * g.y > kNrmSlots) {
        set_error("fused ||b~||^2: %u CTAs exceed the partial slots", g.x * g.y);
        return -2;
      }
      SP_CUDA(launch_k(k4_rhs<T, 1, true>, g, kBlock, 0, s, x, m, out, enforce_u, C, H, W, 1.0,
                       active, partial, counter, nrm));
      SP_CHECK_LAUNCH();
      k_sum_parts<<<1, 1024, 0, s>>>(partial, (int)(g.x * g.y), nrm);
    } else {
      SP_CUDA(launch_k(k4_rhs<T, 1>, g, kBlock, 0, s, x, m, out, enforce_u, C, H, W, 1.0, active,
                       (double*)nullptr, (unsigned*)nullptr, (double*)nullptr));
    }
  } else {
    k_masked_sym_rhs<T><<<mg_grid(H, W, nz), kBlock, 0, s>>>(x, m, out, C, H, W, active);
    if (enforce_u) {
      SP_CHECK_LAUNCH();
      return enforce<T>(enforce_u, out, m, C, H, W, 0, s, ntile, active);
    }
  }
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int ct_apply(const T* w, const uint8_t* m, T* out, int C, int H, int W, double inv_h2,
             cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(w, m, out))
    SP_CUDA(launch_k(k4_rhs<T, 2>, mg_grid4(H, W, nz), kBlock, 0, s, w, m, out, nullptr, C, H, W, inv_h2,
                     active, (double*)nullptr, (unsigned*)nullptr, (double*)nullptr));
  else
    k_ct_apply<T><<<mg_grid(H, W, nz), kBlock, 0, s>>>(w, m, out, C, H, W, inv_h2, active);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int residual(const T* u, const T* b, const uint8_t* m, T* r, double* partial,
             unsigned* counter, double* norms, int C, int H, int W, double inv_h2,
             cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(u, b, m, r))
    SP_CUDA(launch_k(k4_residual<T>, mg_grid4(H, W, nz), kBlock, 0, s, u, b, m, r, partial, counter, norms,
                                                         C, H, W, inv_h2, active));
  else
    SP_CUDA(launch_k(k_residual<T>, mg_grid(H, W, nz), kBlock, 0, s, u, b, m, r, partial, counter, norms, C,
                                                       H, W, inv_h2, active));
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int residual_restrict(const T* u, const T* b, const uint8_t* m, T* rc, int C, int H, int W,
                      double inv_h2, cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(u, b, m))
    SP_CUDA(launch_k(k4_residual_restrict<T>, mg_grid4(H, W, nz), kBlock, 0, s, u, b, m, rc, C, H, W,
                                                                  inv_h2, active));
  else
    SP_CUDA(launch_k(k_residual_restrict<T>, mg_grid(H, W, nz), kBlock, 0, s, u, b, m, rc, C, H, W, inv_h2,
                                                                active));
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int restrict_mask(const uint8_t* m, const T* v, uint8_t* cm, T* cv, int C, int H, int W,
                  cudaStream_t s, int ntile) {
  k_restrict_mask<T><<<mg_grid((H + 1) / 2, (W + 1) / 2, ntile), kBlock, 0, s>>>(m, v, cm,
                                                                                  cv, C, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int prolong_enforce(const T* e, T* u, const T* b, const uint8_t* m, int C, int chh, int cww,
                    int H, int W, int add, cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(u, b, m))
    SP_CUDA(launch_k(k4_prolong_enforce<T>, mg_grid4(H, W, nz), kBlock, 0, s, e, u, b, m, C, chh, cww, H, W,
                                                                add, active));
  else
    SP_CUDA(launch_k(k_prolong_enforce<T>, mg_grid(H, W, nz), kBlock, 0, s, e, u, b, m, C, chh, cww, H, W,
                                                              add, active));
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int enforce(T* u, const T* src, const uint8_t* m, int C, int H, int W, int zero_off,
            cudaStream_t s, int ntile, const int* active) {
  long nz = (long)ntile * C;
  if (VEC_OK(u, src, m))
    k4_enforce<T><<<mg_grid4(H, W, nz), kBlock, 0, s>>>(u, src, m, C, H, W, zero_off, active);
  else
    k_enforce<T><<<mg_grid(H, W, nz), kBlock, 0, s>>>(u, src, m, C, H, W, zero_off, active);
  SP_CHECK_LAUNCH();
  return 0;
}

#define INST(T)                                                                          \
  template int sym_rhs<T>(const T*, const uint8_t*, T*, T*, int, int, int, double,         \
                          cudaStream_t, int, const int*);                                  \
  template int masked_sym_rhs<T>(const T*, const uint8_t*, T*, int, int, int,              \
                                 cudaStream_t, int, const int*, T*, double*, double*,      \
                                 unsigned*);                                               \
  template int ct_apply<T>(const T*, const uint8_t*, T*, int, int, int, double,            \
                           cudaStream_t, int, const int*);                                 \
  template int residual<T>(const T*, const T*, const uint8_t*, T*, double*, unsigned*,     \
                           double*, int, int, int, double, cudaStream_t, int, const int*); \
  template int residual_restrict<T>(const T*, const T*, const uint8_t*, T*, int, int, int, \
                                    double, cudaStream_t, int, const int*);                \
  template int restrict_mask<T>(const uint8_t*, const T*, uint8_t*, T*, int, int, int,     \
                                cudaStream_t, int);                                        \
  template int prolong_enforce<T>(const T*, T*, const T*, const uint8_t*, int, int, int,   \
                                  int, int, int, cudaStream_t, int, const int*);           \
  template int enforce<T>(T*, const T*, const uint8_t*, int, int, int, int, cudaStream_t,  \
                          int, const int*);

INST(float)
INST(double)

}  // namespace sp
