// oras.cu -- optimized restricted additive Schwarz sweep (sm_100a).
//
// Reference: numba_impl.py:161-263 (oras_apply) driven by solver.py:259-273.
// Kernel 1 (k_oras_local): one CTA per (block, channel).  The block's
// residual is staged into registers (each thread owns PPT pixels, strided by
// the CTA size so warps read whole rows), the search direction p lives in
// shared memory for the 5-point stencil, and the local CG runs entirely
// on-chip: dots are double, reduced by warp shuffles plus a fixed-order
// cross-warp sum (deterministic); alpha/beta are rounded to T and the vector
// updates use T arithmetic exactly like the reference.  The correction v is
// written to `corr` ([C][nb][bh][bw]).
// Kernel 2 (k_oras_blend): the reference blends u += w_b * v_b sequentially
// in block order.  Here every pixel gathers its (at most 3x3) covering
// blocks in ascending block index, which is the same summation order, so the
// blend is race-free and bit-identical.  The partition-of-unity weights are
// either read (kernel-table path) or recomputed on the fly in double with
// the exact operation order of build_decomposition (solver.py:142-197),
// which saves streaming a weight array of the size of the image.
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int NT = 256;

template <typename T, int PPT>
__global__ void __launch_bounds__(NT) k_oras_local(
    const T* __restrict__ r, const uint8_t* __restrict__ m,
    const double* __restrict__ tau_src, double tau_scale,
    const int* __restrict__ ys, const int* __restrict__ xs, int nbx, int bh, int bw,
    int H, int W, double gamma, long cap, double inv_h2, T* __restrict__ corr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ps = reinterpret_cast<T*>(smem_raw);
  __shared__ double red0[NT / 32], red1[NT / 32], red2[NT / 32];
  const int bi = blockIdx.x, ch = blockIdx.y, C = gridDim.y, nb = gridDim.x;
  const int y0 = ys[bi / nbx], x0 = xs[bi % nbx];
  const int npx = bh * bw;
  const size_t plane = (size_t)H * W;
  const T* rc = r + (size_t)ch * plane;

  T res[PPT], v[PPT], p[PPT], ap[PPT];
  double diag[PPT];
  unsigned flags[PPT];  // bit0 valid, bit1 masked, bits4..7 in-block unmasked nbr
  int kk[PPT];
  double rs_part = 0.0;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    int k = threadIdx.x + s * NT;
    kk[s] = k;
    flags[s] = 0;
    res[s] = v[s] = p[s] = ap[s] = (T)0;
    diag[s] = 0.0;
    if (k < npx) {
      int i = k / bw, j = k - (k / bw) * bw;
      int gy = y0 + i, gx = x0 + j;
      size_t g = (size_t)gy * W + gx;
      unsigned f = 1u;
      if (m[g]) f |= 2u;
      double d = 0.0;
      if (gy > 0) {
        if (i > 0) { d += 1.0; if (!m[g - W]) f |= 16u; } else d += 1.0 - gamma;
      }
      if (gy < H - 1) {
        if (i < bh - 1) { d += 1.0; if (!m[g + W]) f |= 32u; } else d += 1.0 - gamma;
      }
      if (gx > 0) {
        if (j > 0) { d += 1.0; if (!m[g - 1]) f |= 64u; } else d += 1.0 - gamma;
      }
      if (gx < W - 1) {
        if (j < bw - 1) { d += 1.0; if (!m[g + 1]) f |= 128u; } else d += 1.0 - gamma;
      }
      flags[s] = f;
      diag[s] = d;
      res[s] = rc[g];
      p[s] = res[s];
      rs_part += (double)res[s] * (double)res[s];
    }
  }
  double rs = cta_sum<NT>(rs_part, red0);
  const double tau = tau_scale * tau_src[ch];
  long it = 0;
  int phase = 0;
  while (rs > tau && it < cap) {
    // stage p for the stencil
#pragma unroll
    for (int s = 0; s < PPT; ++s)
      if (flags[s] & 1u) ps[kk[s]] = p[s];
    __syncthreads();
    double pap_part = 0.0;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      unsigned f = flags[s];
      if (!(f & 1u)) continue;
      T a;
      if (f & 2u) {
        a = p[s];
      } else {
        int k = kk[s];
        double acc = 0.0;
        if (f & 16u) acc += (double)ps[k - bw];
        if (f & 32u) acc += (double)ps[k + bw];
        if (f & 64u) acc += (double)ps[k - 1];
        if (f & 128u) acc += (double)ps[k + 1];
        a = (T)((diag[s] * (double)p[s] - acc) * inv_h2);
      }
      ap[s] = a;
      pap_part += (double)p[s] * (double)a;
    }
    double pap = cta_sum<NT>(pap_part, phase ? red2 : red1);
    if (pap <= 0.0) break;
    T alpha = (T)(rs / pap);
    double rsn_part = 0.0;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      if (!(flags[s] & 1u)) continue;
      v[s] = v[s] + alpha * p[s];
      res[s] = res[s] - alpha * ap[s];
      rsn_part += (double)res[s] * (double)res[s];
    }
    double rsn = cta_sum<NT>(rsn_part, phase ? red1 : red2);
    T beta = (T)(rsn / rs);
    rs = rsn;
#pragma unroll
    for (int s = 0; s < PPT; ++s)
      if (flags[s] & 1u) p[s] = res[s] + beta * p[s];
    ++it;
    phase ^= 1;
  }
  T* out = corr + ((size_t)ch * nb + bi) * (size_t)npx;
#pragma unroll
  for (int s = 0; s < PPT; ++s)
    if (flags[s] & 1u) out[kk[s]] = v[s];
}

// covering-block tables: for row y, blocks ky in [row_k0[y], row_k0[y]+row_n[y])
template <typename T>
__global__ void k_oras_blend(T* __restrict__ u, const T* __restrict__ corr,
                             const T* __restrict__ weights,
                             const int* __restrict__ ys, const int* __restrict__ xs,
                             const int* __restrict__ row_k0, const int* __restrict__ row_n,
                             const int* __restrict__ col_k0, const int* __restrict__ col_n,
                             int nby, int nbx, int bh, int bw, int H, int W, int C,
                             int overlap) {
  int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
  if (x >= W || y >= H) return;
  const int nb = nby * nbx;
  const size_t plane = (size_t)H * W, k = (size_t)y * W + x, npx = (size_t)bh * bw;
  const int ky0 = row_k0[y], nky = row_n[y], kx0 = col_k0[x], nkx = col_n[x];
  // weights of the covering blocks in block order (<= 3x3)
  double wv[9];
  int cnt = 0;
  if (weights) {
    for (int a = 0; a < nky; ++a)
      for (int b = 0; b < nkx; ++b) {
        int ky = ky0 + a, kx = kx0 + b, bi = ky * nbx + kx;
        int i = y - ys[ky], j = x - xs[kx];
        wv[cnt++] = (double)weights[(size_t)bi * npx + (size_t)i * bw + j];
      }
  } else {
    // solver.py:160-197: raw = min(dist_to_inner_edge + 1, overlap),
    // normalized by the pointwise total; the last covering block takes the
    // exact complement 1 - (sum of the earlier normalized weights).
    const double big = (double)(H > W ? H : W);
    double raw[9], total = 0.0;
    for (int a = 0; a < nky; ++a)
      for (int b = 0; b < nkx; ++b) {
        int yb = ys[ky0 + a], xb = xs[kx0 + b];
        double ii = (double)(y - yb), jj = (double)(x - xb);
        double di = big;
        if (yb > 0) di = fmin(di, ii);
        if (yb + bh < H) di = fmin(di, (double)(bh - 1) - ii);
        if (xb > 0) di = fmin(di, jj);
        if (xb + bw < W) di = fmin(di, (double)(bw - 1) - jj);
        double rw = fmin(di + 1.0, (double)overlap);
        raw[cnt++] = rw;
      }
    // total accumulates over all blocks in block order (same adds)
    for (int q = 0; q < cnt; ++q) total += raw[q];
    double acc = 0.0;
    for (int q = 0; q < cnt; ++q) {
      double wn = (q == cnt - 1) ? 1.0 - acc : raw[q] / total;
      acc += wn;
      wv[q] = wn;
    }
  }
  for (int c = 0; c < C; ++c) {
    T uv = u[c * plane + k];
    int q = 0;
    for (int a = 0; a < nky; ++a)
      for (int b = 0; b < nkx; ++b, ++q) {
        int ky = ky0 + a, kx = kx0 + b, bi = ky * nbx + kx;
        int i = y - ys[ky], j = x - xs[kx];
        T cv = corr[((size_t)c * nb + bi) * npx + (size_t)i * bw + j];
        uv = uv + (T)wv[q] * cv;
      }
    u[c * plane + k] = uv;
  }
}

}  // namespace

template <typename T>
int oras_local_launch(const T* r, const uint8_t* m, const double* tau_src,
                      double tau_scale, const int* ys, const int* xs, int nby, int nbx,
                      int bh, int bw, int H, int W, int C, double gamma, long cap,
                      double inv_h2, T* corr, cudaStream_t s) {
  int npx = bh * bw;
  dim3 grid(nby * nbx, C);
  size_t sm = (size_t)npx * sizeof(T);
  if (npx <= NT * 4) {
    k_oras_local<T, 4><<<grid, NT, sm, s>>>(r, m, tau_src, tau_scale, ys, xs, nbx, bh,
                                            bw, H, W, gamma, cap, inv_h2, corr);
  } else if (npx <= NT * 16) {
    auto kern = k_oras_local<T, 16>;
    if (sm > 48 * 1024) SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, NT, sm, s>>>(r, m, tau_src, tau_scale, ys, xs, nbx, bh, bw, H, W, gamma,
                              cap, inv_h2, corr);
  } else {
    set_error("oras block of %d pixels exceeds the 4096-pixel kernel limit", npx);
    return -2;
  }
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int oras_blend_launch(T* u, const T* corr, const T* weights, const int* ys, const int* xs,
                      const int* row_k0, const int* row_n, const int* col_k0,
                      const int* col_n, int nby, int nbx, int bh, int bw, int H, int W,
                      int C, int overlap, cudaStream_t s) {
  dim3 grid(cdiv(W, 32), cdiv(H, 8));
  k_oras_blend<T><<<grid, dim3(32, 8), 0, s>>>(u, corr, weights, ys, xs, row_k0, row_n,
                                               col_k0, col_n, nby, nbx, bh, bw, H, W, C,
                                               overlap);
  SP_CHECK_LAUNCH();
  return 0;
}

#define INST(T)                                                                        \
  template int oras_local_launch<T>(const T*, const uint8_t*, const double*, double,    \
                                    const int*, const int*, int, int, int, int, int,    \
                                    int, int, double, long, double, T*, cudaStream_t);  \
  template int oras_blend_launch<T>(T*, const T*, const T*, const int*, const int*,     \
                                    const int*, const int*, const int*, const int*,     \
                                    int, int, int, int, int, int, int, int, cudaStream_t);
INST(float)
INST(double)

}  // namespace sp
