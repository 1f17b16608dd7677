// mgfast.cu -- row-marching float stencil sweeps for the multigrid hierarchy.
//
// The V-cycle's HBM-bound sweeps on the wide levels (W >= 128, W % 4 == 0):
//   residual          r = b~ - A~ u, per-plane sum r^2     (numba_impl.py:147-158)
//   residual+restrict r_H = restrict(b~ - A~ u)          (solver.py:289-291)
//   prolong+enforce   u += P e, u[mask] = b~[mask]         (solver.py:294-296)
//
// Thread layout: a warp owns 32 float4 column quads (128 columns) and marches
// down a band of rows, holding the rows above / at / below the current one
// in registers, so every u element comes from DRAM once; the two horizontal
// neighbours of a quad come from the adjacent lanes by shuffle (lanes 0 and
// 31 fetch one extra scalar).  Masks are read as 4-byte words.  Loads run two
// rows ahead of the arithmetic.
//
// Arithmetic is the reference's, bit for bit (the same as mg.cu's per-pixel
// kernels): neighbour sums in double in the order up, down, left, right,
// one rounding to float, residual r = b - A u in float; the restriction
// averages in double, the prolongation interpolates in double.  Norm
// reductions are deterministic: per-thread double sums, warp / CTA trees in
// fixed order, the last CTA of a plane adds the CTA partials in index order.
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int MRB = 16;            // rows per warp band
constexpr int MWARPS = 4;          // warps per CTA (stacked bands)
constexpr int MNT = MWARPS * 32;
constexpr int MROWS = MRB * MWARPS;  // rows per CTA

__device__ __forceinline__ float4 ldq(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// one quad row: u, its neighbour-sum values q (u where unmasked, 0 where
// masked or outside the image) and the mask word
struct Row {
  float4 u, q;
  uint32_t m;
};

__device__ __forceinline__ bool mk(uint32_t mw, int i) { return (mw >> (8 * i)) & 0xFFu; }
__device__ __forceinline__ float f4(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ Row load_row(const float* __restrict__ uc,
                                        const uint8_t* __restrict__ mt, int y, int H, int W,
                                        int x0) {
  Row r;
  if (y >= 0 && y < H && x0 < W) {
    const size_t k = (size_t)y * W + x0;
    r.u = ldq(uc + k);
    r.m = *reinterpret_cast<const uint32_t*>(mt + k);
  } else {
    r.u = make_float4(0.f, 0.f, 0.f, 0.f);
    r.m = 0u;
  }
  r.q = make_float4(mk(r.m, 0) ? 0.f : r.u.x, mk(r.m, 1) ? 0.f : r.u.y,
                    mk(r.m, 2) ? 0.f : r.u.z, mk(r.m, 3) ? 0.f : r.u.w);
  return r;
}

// r = b - A~ u for one quad row (numba_impl.py:78-97, 147-158), bit-exact:
// the neighbour sum in double in the order up, down, left, right (absent or
// masked neighbours add an exact +0), (d u - sum) rounded once to float.
// ql / qr: the quad's outer horizontal neighbour values (0 outside).
__device__ __forceinline__ float4 resid_quad(const Row& up, const Row& c, const Row& dn,
                                             float ql, float qr, float4 bb, int y, int H,
                                             int x0, int W) {
  const double dv = 2.0 + (y > 0 ? 1.0 : 0.0) + (y < H - 1 ? 1.0 : 0.0);
  const double d0 = dv - (x0 > 0 ? 0.0 : 1.0);
  const double d3 = dv - (x0 + 4 < W ? 0.0 : 1.0);
  const float qs[6] = {ql, c.q.x, c.q.y, c.q.z, c.q.w, qr};
  float out[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double a = (((double)f4(up.q, i) + (double)f4(dn.q, i)) + (double)qs[i]) +
                     (double)qs[i + 2];
    const float uv = f4(c.u, i);
    const double d = i == 0 ? d0 : (i == 3 ? d3 : dv);
    const float ax = mk(c.m, i) ? uv : (float)(d * (double)uv - a);
    out[i] = f4(bb, i) - ax;
  }
  return make_float4(out[0], out[1], out[2], out[3]);
}

// the quad's outer horizontal neighbour values for row y (adjacent lanes by
// shuffle; lanes 0 / 31 read one scalar + mask byte)
__device__ __forceinline__ void side(const Row& c, int lane, const float* __restrict__ uc,
                                     const uint8_t* __restrict__ mt, int y, int H, int W,
                                     int x0, float& ql, float& qr) {
  ql = __shfl_up_sync(0xFFFFFFFFu, c.q.w, 1);
  qr = __shfl_down_sync(0xFFFFFFFFu, c.q.x, 1);
  if (lane == 0) {
    ql = 0.0f;
    if (x0 > 0 && x0 < W && y < H) {
      const size_t k = (size_t)y * W + x0 - 1;
      ql = mt[k] ? 0.0f : uc[k];
    }
  }
  if (lane == 31) {
    qr = 0.0f;
    if (x0 + 4 < W && y < H) {
      const size_t k = (size_t)y * W + x0 + 4;
      qr = mt[k] ? 0.0f : uc[k];
    }
  }
}

template <bool NORMS>
__global__ void __launch_bounds__(MNT) k_resid_march(
    const float* __restrict__ u, const float* __restrict__ b, const uint8_t* __restrict__ m,
    float* __restrict__ r, double* __restrict__ partial, unsigned* __restrict__ counter,
    double* __restrict__ norms, int C, int H, int W, const int* __restrict__ active,
    double* __restrict__ bandcol, int band0, int nbt) {
  __shared__ double wsum[MWARPS];
  __shared__ bool am_last;
  const int z = blockIdx.z, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * 32 + lane) * 4;
  const int ys = blockIdx.y * MROWS + w * MRB, ye = min(ys + MRB, H);
  const size_t plane = (size_t)H * W;
  const float* uc = u + (size_t)z * plane;
  const float* bc = b + (size_t)z * plane;
  float* rc = r + (size_t)z * plane;
  const uint8_t* mt = m + (size_t)tile * plane;
  float sq = 0.0f;
  if (ys < H) {
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    Row ru = load_row(uc, mt, ys - 1, H, W, x0);
    Row rc0 = load_row(uc, mt, ys, H, W, x0);
    Row rd = load_row(uc, mt, ys + 1, H, W, x0);
    Row rd2 = load_row(uc, mt, ys + 2 <= ye ? ys + 2 : H, H, W, x0);
    float4 bb = x0 < W ? ldq(bc + (size_t)ys * W + x0) : z4;
    float4 bn = (ys + 1 < ye && x0 < W) ? ldq(bc + (size_t)(ys + 1) * W + x0) : z4;
#pragma unroll 1
    for (int t = 0; t < MRB; ++t) {
      const int y = ys + t;
      if (y < ye) {
        // loads run two rows ahead of the arithmetic
        Row rn = load_row(uc, mt, y + 3 <= ye ? y + 3 : H, H, W, x0);
        float4 bn2 = (y + 2 < ye && x0 < W) ? ldq(bc + (size_t)(y + 2) * W + x0) : z4;
        float ql, qr;
        side(rc0, lane, uc, mt, y, H, W, x0, ql, qr);
        if (x0 < W) {
          const float4 rr = resid_quad(ru, rc0, rd, ql, qr, bb, y, H, x0, W);
          *reinterpret_cast<float4*>(rc + (size_t)y * W + x0) = rr;
          if (NORMS) {
            sq = __fmaf_rn(rr.x, rr.x, sq);
            sq = __fmaf_rn(rr.y, rr.y, sq);
            sq = __fmaf_rn(rr.z, rr.z, sq);
            sq = __fmaf_rn(rr.w, rr.w, sq);
          }
        }
        ru = rc0; rc0 = rd; rd = rd2; rd2 = rn;
        bb = bn; bn = bn2;
      }
    }
  }
  if (!NORMS) return;
  // deterministic plane reduction: warp butterfly -> CTA (warp order)
  // -> last CTA of the plane sums the CTA partials in index order
  double sqd = (double)sq;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sqd += __shfl_xor_sync(0xFFFFFFFFu, sqd, o);
  if (bandcol) {
    // row-band partials for the strip-partitioned solve (strips.cu): one
    // double per (plane, 16-row band of the level, 128-column group); the
    // view starts on a band boundary, so band indices are global
    if (lane == 0 && ys < H)
      bandcol[((size_t)z * nbt + band0 + (ys / MRB)) * gridDim.x + blockIdx.x] = sqd;
    return;
  }
  if (lane == 0) wsum[w] = sqd;
  __syncthreads();
  const unsigned ncta = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < MWARPS; ++q) s += wsum[q];
    if (ncta == 1) {
      norms[z] = s;
      am_last = false;
    } else {
      partial[(size_t)z * ncta + cta] = s;
      __threadfence();
      am_last = atomicAdd(counter + z, 1u) == ncta - 1;
    }
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned i = threadIdx.x; i < ncta; i += MNT)
    t += ((volatile double*)partial)[(size_t)z * ncta + i];
  t = cta_sum<MNT>(t, wsum);
  if (threadIdx.x == 0) {
    norms[z] = t;
    counter[z] = 0u;
  }
}

// residual fused with the 2x2 box restriction (restrict_values,
// numba_impl.py:266-284): a warp marches down its band two fine rows per
// step and emits one coarse row of 64 pixels (two per lane).  Bands have an
// even number of rows, so every 2x2 cell lies inside one band.
__global__ void __launch_bounds__(MNT) k_resid_restrict_march(
    const float* __restrict__ u, const float* __restrict__ b, const uint8_t* __restrict__ m,
    float* __restrict__ rcoarse, int C, int H, int W, const int* __restrict__ active) {
  const int z = blockIdx.z, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * 32 + lane) * 4;
  const int ys = blockIdx.y * MROWS + w * MRB, ye = min(ys + MRB, H);
  if (ys >= H) return;
  const int cw = (W + 1) / 2;
  const size_t plane = (size_t)H * W;
  const float* uc = u + (size_t)z * plane;
  const float* bc = b + (size_t)z * plane;
  const uint8_t* mt = m + (size_t)tile * plane;
  float* out = rcoarse + (size_t)z * ((size_t)((H + 1) / 2) * cw);
  Row ru = load_row(uc, mt, ys - 1, H, W, x0);
  Row r0 = load_row(uc, mt, ys, H, W, x0);
  Row r1 = load_row(uc, mt, ys + 1, H, W, x0);
  Row r2 = load_row(uc, mt, ys + 2 <= ye ? ys + 2 : H, H, W, x0);
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int t = 0; t < MRB; t += 2) {
    const int y = ys + t;
    if (y < ye) {
      const bool two = y + 1 < H;
      // next step's rows (needed up to row ye: the band's lower neighbour)
      Row n1 = load_row(uc, mt, y + 3 <= ye ? y + 3 : H, H, W, x0);
      Row n2 = load_row(uc, mt, y + 4 <= ye ? y + 4 : H, H, W, x0);
      float4 b0 = x0 < W ? ldq(bc + (size_t)y * W + x0) : z4;
      float4 b1 = (two && x0 < W) ? ldq(bc + (size_t)(y + 1) * W + x0) : z4;
      float ql0, qr0, ql1, qr1;
      side(r0, lane, uc, mt, y, H, W, x0, ql0, qr0);
      side(r1, lane, uc, mt, two ? y + 1 : H, H, W, x0, ql1, qr1);
      if (x0 < W) {
        const float4 e0 = resid_quad(ru, r0, r1, ql0, qr0, b0, y, H, x0, W);
        float2 o;
        // restrict_values (numba_impl.py:266-284): ((a + b) + c) + d in double
        if (two) {
          const float4 e1 = resid_quad(r0, r1, r2, ql1, qr1, b1, y + 1, H, x0, W);
          o.x = (float)(((((double)e0.x + (double)e0.y) + (double)e1.x) + (double)e1.y) / 4.0);
          o.y = (float)(((((double)e0.z + (double)e0.w) + (double)e1.z) + (double)e1.w) / 4.0);
        } else {
          o.x = (float)(((double)e0.x + (double)e0.y) / 2.0);
          o.y = (float)(((double)e0.z + (double)e0.w) / 2.0);
        }
        *reinterpret_cast<float2*>(out + (size_t)(y >> 1) * cw + (x0 >> 1)) = o;
      }
      ru = r1; r0 = r2; r1 = n1; r2 = n2;
    }
  }
}

// cell-centred bilinear prolongation (numba_impl.py:316-348), clamped,
// fused with u += P e and u[mask] = b~[mask]; add == 0: u = P e (FMG step)
__device__ __forceinline__ void paxis(int y, int n, int& y0, int& y1, double& wy) {
  double fy = ((double)y + 0.5) / 2.0 - 0.5;
  y0 = (int)floor(fy);
  wy = fy - (double)y0;
  if (y0 < 0) { y0 = 0; wy = 0.0; }
  if (y0 > n - 1) { y0 = n - 1; wy = 0.0; }
  y1 = min(y0 + 1, n - 1);
}

__global__ void __launch_bounds__(MNT) k_prolong_march(
    const float* __restrict__ e, float* __restrict__ u, const float* __restrict__ b,
    const uint8_t* __restrict__ m, int C, int chh, int cww, int H, int W, int add,
    const int* __restrict__ active) {
  const int z = blockIdx.z, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * 32 + lane) * 4;
  const int ys = blockIdx.y * MROWS + w * MRB, ye = min(ys + MRB, H);
  if (ys >= H || x0 >= W) return;
  const size_t plane = (size_t)H * W;
  float* uc = u + (size_t)z * plane;
  const float* bc = b + (size_t)z * plane;
  const uint8_t* mt = m + (size_t)tile * plane;
  const float* ec = e + (size_t)z * chh * cww;
  int xa[4], xb[4];
  double wx[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) paxis(x0 + i, cww, xa[i], xb[i], wx[i]);
  for (int y = ys; y < ye; ++y) {
    const size_t k = (size_t)y * W + x0;
    const uint32_t mw = *reinterpret_cast<const uint32_t*>(mt + k);
    const float4 bb = mw ? ldq(bc + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 uu = add ? ldq(uc + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    int y0, y1;
    double wy;
    paxis(y, chh, y0, y1, wy);
    const float* e0 = ec + (size_t)y0 * cww;
    const float* e1 = ec + (size_t)y1 * cww;
    float o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (mk(mw, i)) {
        o[i] = f4(bb, i);
        continue;
      }
      // numba_impl.py:316-348: the bilinear value in double, one rounding
      const double v = (1.0 - wy) * ((1.0 - wx[i]) * (double)e0[xa[i]] + wx[i] * (double)e0[xb[i]]) +
                       wy * ((1.0 - wx[i]) * (double)e1[xa[i]] + wx[i] * (double)e1[xb[i]]);
      const float p = (float)v;
      o[i] = add ? f4(uu, i) + p : p;
    }
    *reinterpret_cast<float4*>(uc + k) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace

int march_band_rows() { return MRB; }

bool march_ok(int H, int W, size_t npart) {
  if (W % 4 != 0 || W < 128) return false;
  const size_t ncta = (size_t)cdiv(W, 128) * cdiv(H, MROWS);
  return ncta <= npart;
}

int resid_march(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
                unsigned* counter, double* norms, int C, int H, int W, cudaStream_t s,
                int ntile, const int* active, double* bandcol, int band0, int nbt) {
  dim3 grid(cdiv(W, 128), cdiv(H, MROWS), (unsigned)((long)ntile * C));
  if (norms || bandcol)
    k_resid_march<true><<<grid, MNT, 0, s>>>(u, b, m, r, partial, counter, norms, C, H, W,
                                             active, bandcol, band0, nbt);
  else
    k_resid_march<false><<<grid, MNT, 0, s>>>(u, b, m, r, partial, counter, norms, C, H, W,
                                              active, nullptr, 0, 0);
  SP_CHECK_LAUNCH();
  return 0;
}

int resid_restrict_march(const float* u, const float* b, const uint8_t* m, float* rc, int C,
                         int H, int W, cudaStream_t s, int ntile, const int* active) {
  dim3 grid(cdiv(W, 128), cdiv(H, MROWS), (unsigned)((long)ntile * C));
  k_resid_restrict_march<<<grid, MNT, 0, s>>>(u, b, m, rc, C, H, W, active);
  SP_CHECK_LAUNCH();
  return 0;
}

int prolong_march(const float* e, float* u, const float* b, const uint8_t* m, int C, int chh,
                  int cww, int H, int W, int add, cudaStream_t s, int ntile,
                  const int* active) {
  dim3 grid(cdiv(W, 128), cdiv(H, MROWS), (unsigned)((long)ntile * C));
  k_prolong_march<<<grid, MNT, 0, s>>>(e, u, b, m, C, chh, cww, H, W, add, active);
  SP_CHECK_LAUNCH();
  return 0;
}

}  // namespace sp
