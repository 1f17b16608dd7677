// geometry.cu -- jump flooding, Delaunay-from-Voronoi, triangle buckets and
// pixel selection (sm_100a).  Everything here is integer or order-exact and
// therefore bit-identical to the reference:
//   jfa pass            numba_impl.py:351-396   (one thread per pixel)
//   jfa_dist2 / max     numba_impl.py:399-409, geometry.py:108-110
//   corner scan         geometry.py:140-181     (packed 63-bit keys, radix
//                                                sort + unique == np.unique)
//   assign_triangles    numba_impl.py:442-466   (lowest index wins ==
//                                                atomicMin, order-independent)
//   seed_min_triangle   geometry.py:188-194     (atomicMin)
//   fallback_assign     numba_impl.py:469-481
//   reduce_cells        numba_impl.py:484-498   (stable sort of pixels by
//                                                triangle, then a sequential
//                                                row-major double sum per
//                                                triangle: same adds, same
//                                                order; first strict max)
//   selection           spatial.py:245-259      (stable sort on ~bits(sum))
//   fill_highest_error  spatial.py:189-197
//   fs_dither           numba_impl.py:412-439   (serial; `aa` baseline only)
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <vector>

#include "geometry.cuh"

namespace sp {

namespace {

constexpr int BX = 32, BY = 8;

template <typename D>
__global__ void k_jfa_pass(const int* __restrict__ cur, int* __restrict__ nxt,
                           const int* __restrict__ sy, const int* __restrict__ sx,
                           int step, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  int best = cur[(size_t)y * W + x];
  D bd;
  if (best >= 0) {
    D dy = (D)y - (D)sy[best], dx = (D)x - (D)sx[best];
    bd = dy * dy + dx * dx;
  } else {
    bd = (D)4 * ((D)H * (D)H + (D)W * (D)W);
  }
#pragma unroll
  for (int oy = -1; oy <= 1; ++oy) {
    int ny = y + oy * step;
    if (ny < 0 || ny >= H) continue;
#pragma unroll
    for (int ox = -1; ox <= 1; ++ox) {
      if (oy == 0 && ox == 0) continue;
      int nx = x + ox * step;
      if (nx < 0 || nx >= W) continue;
      int cand = cur[(size_t)ny * W + nx];
      if (cand < 0) continue;
      D dy = (D)y - (D)sy[cand], dx = (D)x - (D)sx[cand];
      D cd = dy * dy + dx * dx;
      if (cd < bd || (cd == bd && best >= 0 && cand < best)) {
        bd = cd;
        best = cand;
      }
    }
  }
  nxt[(size_t)y * W + x] = best;
}

__global__ void k_dist2(const int* __restrict__ lab, const int* __restrict__ sy,
                        const int* __restrict__ sx, long long* __restrict__ out,
                        unsigned long long* __restrict__ dmax, int H, int W, int m) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  long long d = 0;
  bool live = x < W && y < H;
  if (live) {
    int s = lab[(size_t)y * W + x];
    if (s < 0) s += m;  // unlabelled pixel: numba's wraparound seeds[-1]
    long long dy = (long long)y - sy[s], dx = (long long)x - sx[s];
    d = dy * dy + dx * dx;
    if (out) out[(size_t)y * W + x] = d;
  }
  if (dmax) {
    unsigned long long v = (unsigned long long)d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
      v = w > v ? w : v;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(dmax, v);
  }
}

__global__ void k_seeds_i64_to_soa(const long long* __restrict__ seeds, long m,
                                   int* __restrict__ sy, int* __restrict__ sx) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  sy[i] = (int)seeds[2 * i];
  sx[i] = (int)seeds[2 * i + 1];
}

// seeds are the row-major np.nonzero order (geometry.py:99-105)
__global__ void k_seed_init(const int* __restrict__ idx, long m, int W, int* __restrict__ sy,
                            int* __restrict__ sx, int* __restrict__ lab) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int p = idx[i];
  sy[i] = p / W;
  sx[i] = p - (p / W) * W;
  lab[p] = (int)i;
}


// ---- jump flooding on packed seed coordinates ---------------------------------
// The pipeline's seeds are the stored pixels in row-major order
// (np.nonzero, geometry.py:92-110), so seed index order IS the row-major
// order of the seed coordinates: a label can carry the seed's coordinates
// key = (sy << 16) | sx instead of its index, and "lower index wins a tie"
// becomes "lower key wins".  A pass then needs no seed-table gathers (the
// index form reads sy/sx of all nine candidates, 18 scattered L2 reads per
// pixel); the keys are mapped back to indices once at the end.
//
// "No seed yet" is the key of a phantom seed at (32767, 32767): for images
// of at most kKeyMax rows and columns its squared distance (>= 2 * 16767^2)
// exceeds every real one (<= 2 * 16000^2) and its key every real key, so
// the pass rule "nearer wins, lower key wins a tie, unlabelled candidates
// are skipped, an unlabelled pixel takes any labelled candidate" is exactly
// the minimum of the 64-bit word (d2 << 32 | key) -- no special cases.
constexpr unsigned KNONE = 0x7FFF7FFFu;
constexpr int kKeyMax = 16000;

__global__ void k_jfa_key_init(const uint8_t* __restrict__ m, unsigned* __restrict__ lab, int H,
                               int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  size_t k = (size_t)y * W + x;
  lab[k] = m[k] ? (((unsigned)y << 16) | (unsigned)x) : KNONE;
}

// (squared distance of the key's seed to (y, x)) << 32 | key
__device__ __forceinline__ unsigned long long key_dk(unsigned key, int y, int x) {
  const int dy = y - (int)(key >> 16), dx = x - (int)(key & 0xFFFFu);
  const unsigned d = (unsigned)(dy * dy) + (unsigned)(dx * dx);
  return ((unsigned long long)d << 32) | key;
}

__global__ void k_jfa_pass_key(const unsigned* __restrict__ cur, unsigned* __restrict__ nxt,
                               int step, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x >= W || y >= H) return;
  unsigned long long best = key_dk(cur[(size_t)y * W + x], y, x);
#pragma unroll
  for (int oy = -1; oy <= 1; ++oy) {
    int ny = y + oy * step;
    if (ny < 0 || ny >= H) continue;
#pragma unroll
    for (int ox = -1; ox <= 1; ++ox) {
      if (oy == 0 && ox == 0) continue;
      int nx = x + ox * step;
      if (nx < 0 || nx >= W) continue;
      const unsigned long long c = key_dk(cur[(size_t)ny * W + nx], y, x);
      best = c < best ? c : best;
    }
  }
  nxt[(size_t)y * W + x] = (unsigned)best;
}

// four pixels per thread for steps that are multiples of 4 (W % 4 == 0): the
// quad x0..x0+3 and each of its 3x3 candidate quads start on a multiple of
// 4, so every candidate row is one 16-byte load and the four pixels share
// the bounds tests; per pixel the candidates are visited in the same order
// with the same rule, so the labels are those of k_jfa_pass_key
__global__ void k_jfa_pass_key4(const unsigned* __restrict__ cur, unsigned* __restrict__ nxt,
                                int step, int H, int W) {
  const int x0 = (blockIdx.x * BX + threadIdx.x) * 4, y = blockIdx.y * BY + threadIdx.y;
  if (x0 >= W || y >= H) return;
  const uint4 self = *reinterpret_cast<const uint4*>(cur + (size_t)y * W + x0);
  unsigned long long best[4] = {key_dk(self.x, y, x0), key_dk(self.y, y, x0 + 1),
                                key_dk(self.z, y, x0 + 2), key_dk(self.w, y, x0 + 3)};
#pragma unroll
  for (int oy = -1; oy <= 1; ++oy) {
    const int ny = y + oy * step;
    if (ny < 0 || ny >= H) continue;
#pragma unroll
    for (int ox = -1; ox <= 1; ++ox) {
      if (oy == 0 && ox == 0) continue;
      const int nx = x0 + ox * step;
      if (nx < 0 || nx >= W) continue;
      const uint4 q = *reinterpret_cast<const uint4*>(cur + (size_t)ny * W + nx);
      const unsigned cand[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned long long c = key_dk(cand[i], y, x0 + i);
        best[i] = c < best[i] ? c : best[i];
      }
    }
  }
  *reinterpret_cast<uint4*>(nxt + (size_t)y * W + x0) =
      make_uint4((unsigned)best[0], (unsigned)best[1], (unsigned)best[2], (unsigned)best[3]);
}

// four pixels per thread for the short steps (1, 2; W % 4 == 0): the
// candidate columns x0 - step .. x0 + 3 + step of a row lie in the three
// aligned quads at x0 - 4, x0, x0 + 4, so each candidate row is three
// 16-byte loads instead of twelve scalar ones; out-of-image candidates are
// the phantom "no seed" key, which never wins.  Same minimum as
// k_jfa_pass_key (the rule is a total order): bit-identical labels.
__global__ void k_jfa_pass_key4s(const unsigned* __restrict__ cur, unsigned* __restrict__ nxt,
                                 int step, int H, int W) {
  const int x0 = (blockIdx.x * BX + threadIdx.x) * 4, y = blockIdx.y * BY + threadIdx.y;
  if (x0 >= W || y >= H) return;
  const uint4 none = make_uint4(KNONE, KNONE, KNONE, KNONE);
  unsigned long long best[4];
#pragma unroll
  for (int oy = -1; oy <= 1; ++oy) {
    const int ny = y + oy * step;
    const bool rok = ny >= 0 && ny < H;
    const unsigned* row = cur + (size_t)(rok ? ny : y) * W;
    const uint4 l = rok && x0 > 0 ? *reinterpret_cast<const uint4*>(row + x0 - 4) : none;
    const uint4 c = rok ? *reinterpret_cast<const uint4*>(row + x0) : none;
    const uint4 r = rok && x0 + 4 < W ? *reinterpret_cast<const uint4*>(row + x0 + 4) : none;
    const unsigned w[12] = {l.x, l.y, l.z, l.w, c.x, c.y, c.z, c.w, r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (oy == -1) best[i] = ~0ull;
      // step is 1 or 2: the window index of x0 + i + ox * step
      const unsigned long long a = key_dk(step == 1 ? w[3 + i] : w[2 + i], y, x0 + i);
      const unsigned long long m = key_dk(w[4 + i], y, x0 + i);
      const unsigned long long b = key_dk(step == 1 ? w[5 + i] : w[6 + i], y, x0 + i);
      unsigned long long t = a < m ? a : m;
      t = b < t ? b : t;
      best[i] = t < best[i] ? t : best[i];
    }
  }
  *reinterpret_cast<uint4*>(nxt + (size_t)y * W + x0) =
      make_uint4((unsigned)best[0], (unsigned)best[1], (unsigned)best[2], (unsigned)best[3]);
}

// keys -> seed indices (rank of the seed pixel), in place; fused with the
// max squared distance of jfa_dist2 (unlabelled pixels: numba's seeds[-1])
__global__ void k_jfa_key_finish(unsigned* __restrict__ lab, const int* __restrict__ rank,
                                 const int* __restrict__ sy, const int* __restrict__ sx, long m,
                                 unsigned long long* __restrict__ dmax, int H, int W) {
  int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  long long d = 0;
  if (x < W && y < H) {
    size_t k = (size_t)y * W + x;
    unsigned key = lab[k];
    long long dy, dx;
    int s;
    if (key == KNONE) {
      s = -1;
      dy = (long long)y - sy[m - 1];
      dx = (long long)x - sx[m - 1];
    } else {
      const int ky = (int)(key >> 16), kx = (int)(key & 0xFFFFu);
      s = rank[(size_t)ky * W + kx];
      dy = (long long)y - ky;
      dx = (long long)x - kx;
    }
    d = dy * dy + dx * dx;
    lab[k] = (unsigned)s;
  }
  // CTA max, one atomic per CTA (same-address atomics serialise in L2)
  __shared__ unsigned long long wmax[BX * BY / 32];
  unsigned long long v = (unsigned long long)d;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  const int tid = threadIdx.y * BX + threadIdx.x;
  if ((tid & 31) == 0) wmax[tid >> 5] = v;
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < BX * BY / 32; ++i) v = wmax[i] > v ? wmax[i] : v;
    atomicMax(dmax, v);
  }
}

__global__ void k_fill_i32(int* __restrict__ p, size_t n, int v) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_mask_flags(const uint8_t* __restrict__ m, uint8_t* __restrict__ flags,
                             size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = m[i] != 0;
}

// ---- corner scan (geometry.py:140-181) ----------------------------------------
__device__ __forceinline__ unsigned long long tri_key(unsigned a, unsigned b, unsigned c) {
  // a < b < c after sorting; 21 bits each
  return ((unsigned long long)a << 42) | ((unsigned long long)b << 21) | (unsigned long long)c;
}

__device__ __forceinline__ void sort3(unsigned& a, unsigned& b, unsigned& c) {
  unsigned t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > c) { t = b; b = c; c = t; }
  if (a > b) { t = a; a = b; b = t; }
}

// corner rows [y0c, y1c) (a corner row y reads label rows y and y + 1; the
// whole image is y0c = 0, y1c = H - 1)
// WIDE (>= 2^21 seeds): the triple as keys2 = a (the high word) and keys =
// b << 32 | c, sorted lexicographically by two stable passes (wide_sort)
template <bool WIDE>
__global__ void k_corner_scan(const int* __restrict__ lab, int H, int W,
                              unsigned long long* __restrict__ keys,
                              unsigned long long* __restrict__ nkeys, int y0c, int y1c,
                              unsigned* __restrict__ keys2) {
  int x = blockIdx.x * BX + threadIdx.x, y = y0c + blockIdx.y * BY + threadIdx.y;
  unsigned long long k0 = 0, k1 = 0;
  unsigned h0 = 0, h1 = 0;
  auto key = [&](unsigned a, unsigned b, unsigned c, unsigned& hi) {
    hi = a;
    return WIDE ? (((unsigned long long)b << 32) | c) : tri_key(a, b, c);
  };
  int nk = 0;
  if (x < W - 1 && y < y1c) {
    size_t p = (size_t)y * W + x;
    int tl = lab[p], tr = lab[p + 1], bl = lab[p + W], br = lab[p + W + 1];
    int s0 = tl, s1 = tr, s2 = bl, s3 = br, t;
    // sort 4
    if (s0 > s1) { t = s0; s0 = s1; s1 = t; }
    if (s2 > s3) { t = s2; s2 = s3; s3 = t; }
    if (s0 > s2) { t = s0; s0 = s2; s2 = t; }
    if (s1 > s3) { t = s1; s1 = s3; s3 = t; }
    if (s1 > s2) { t = s1; s1 = s2; s2 = t; }
    bool d0 = s1 == s0, d1 = s2 == s1, d2 = s3 == s2;
    int nd = 4 - (int)d0 - (int)d1 - (int)d2;
    if (nd == 3) {
      unsigned a = s0, b = d0 ? s2 : s1, c = d2 ? s2 : s3;
      k0 = key(a, b, c, h0);
      nk = 1;
    } else if (nd == 4) {
      int a = tl, b = tr, c = bl, d = br;
      int d1lo = min(a, d), d1hi = max(a, d), d2lo = min(b, c), d2hi = max(b, c);
      bool use1 = (d1lo < d2lo) || (d1lo == d2lo && d1hi <= d2hi);
      unsigned p0, p1, p2, q0, q1, q2;
      if (use1) { p0 = a; p1 = b; p2 = d; q0 = a; q1 = c; q2 = d; }
      else { p0 = a; p1 = b; p2 = c; q0 = b; q1 = c; q2 = d; }
      sort3(p0, p1, p2);
      sort3(q0, q1, q2);
      k0 = key(p0, p1, p2, h0);
      k1 = key(q0, q1, q2, h1);
      nk = 2;
    }
  }
  // warp-aggregated append
  unsigned lane = threadIdx.x & 31;
  unsigned cnt = (unsigned)nk;
  unsigned incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += v;
  }
  // CTA-aggregated: one atomic per CTA (same-address atomics serialise in L2)
  __shared__ unsigned wtot[BY];
  __shared__ unsigned long long cbase;
  if (lane == 31) wtot[threadIdx.y] = incl;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned acc = 0;
    for (int i = 0; i < BY; ++i) {
      const unsigned t = wtot[i];
      wtot[i] = acc;
      acc += t;
    }
    cbase = acc ? atomicAdd(nkeys, (unsigned long long)acc) : 0ull;
  }
  __syncthreads();
  unsigned long long pos = cbase + wtot[threadIdx.y] + incl - cnt;
  if (nk >= 1) keys[pos] = k0;
  if (nk == 2) keys[pos + 1] = k1;
  if (WIDE) {
    if (nk >= 1) keys2[pos] = h0;
    if (nk == 2) keys2[pos + 1] = h1;
  }
}

__global__ void k_decode_tris(const unsigned long long* __restrict__ keys, long T,
                              int* __restrict__ tris) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  unsigned long long k = keys[i];
  tris[3 * i] = (int)(k >> 42);
  tris[3 * i + 1] = (int)((k >> 21) & 0x1FFFFFull);
  tris[3 * i + 2] = (int)(k & 0x1FFFFFull);
}

__global__ void k_decode_tris_wide(const unsigned long long* __restrict__ lo,
                                   const unsigned* __restrict__ hi, long T,
                                   int* __restrict__ tris) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  tris[3 * i] = (int)hi[i];
  tris[3 * i + 1] = (int)(lo[i] >> 32);
  tris[3 * i + 2] = (int)(lo[i] & 0xFFFFFFFFull);
}

// wide keys: flags of the first of every run of equal (hi, lo) pairs
__global__ void k_wide_uniq_flags(const unsigned long long* __restrict__ lo,
                                  const unsigned* __restrict__ hi, long n,
                                  uint8_t* __restrict__ flag) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = i == 0 || lo[i] != lo[i - 1] || hi[i] != hi[i - 1];
}

__global__ void k_gather_u64_u32(const int* __restrict__ idx, long n,
                                 const unsigned long long* __restrict__ lo_in,
                                 const unsigned* __restrict__ hi_in,
                                 unsigned long long* __restrict__ lo_out,
                                 unsigned* __restrict__ hi_out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = idx[i];
  if (lo_out) lo_out[i] = lo_in[j];
  if (hi_out) hi_out[i] = hi_in[j];
}

// ---- rasterization (numba_impl.py:442-466) --------------------------------
template <typename V>
__global__ void k_assign_tris(const V* __restrict__ tris, long T, const V* __restrict__ vy,
                              const V* __restrict__ vx, int H, int W, int* __restrict__ assign) {
  // one 4-lane group per triangle (Delaunay triangles cover ~20-40 box
  // pixels): eight triangles in flight per warp, so the per-triangle vertex
  // gathers overlap instead of serialising a warp's whole triangle list
  constexpr int G = 4;
  long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  int lane = threadIdx.x & (G - 1);
  long nwarps = ((long)gridDim.x * blockDim.x) / G;
  for (long t = warp; t < T; t += nwarps) {
    long long ay = vy[tris[3 * t]], ax = vx[tris[3 * t]];
    long long by = vy[tris[3 * t + 1]], bx = vx[tris[3 * t + 1]];
    long long cy = vy[tris[3 * t + 2]], cx = vx[tris[3 * t + 2]];
    long long ylo = max(0LL, min(ay, min(by, cy))), yhi = min((long long)H - 1, max(ay, max(by, cy)));
    long long xlo = max(0LL, min(ax, min(bx, cx))), xhi = min((long long)W - 1, max(ax, max(bx, cx)));
    if (ylo > yhi || xlo > xhi) continue;
    // the clamped box lies inside the image: 32-bit pixel coordinates and
    // box index (no 64-bit division), 64-bit edge-function products
    const int bw = (int)(xhi - xlo + 1), y0 = (int)ylo, x0 = (int)xlo;
    const long long area = (yhi - ylo + 1) * (long long)bw;
    const long long lim = 1LL << 30;
    const bool in32 = ay > -lim && ay < lim && ax > -lim && ax < lim && by > -lim && by < lim &&
                      bx > -lim && bx < lim && cy > -lim && cy < lim && cx > -lim && cx < lim;
    if (area >= (1LL << 31) || !in32) {
      for (long long q = lane; q < area; q += G) {
        long long y = ylo + q / bw, x = xlo + q % bw;
        long long e0 = (bx - ax) * (y - ay) - (by - ay) * (x - ax);
        long long e1 = (cx - bx) * (y - by) - (cy - by) * (x - bx);
        long long e2 = (ax - cx) * (y - cy) - (ay - cy) * (x - cx);
        if ((e0 >= 0 && e1 >= 0 && e2 >= 0) || (e0 <= 0 && e1 <= 0 && e2 <= 0))
          atomicMin(&assign[y * W + x], (int)t);
      }
      continue;
    }
    const int iay = (int)ay, iax = (int)ax, iby = (int)by, ibx = (int)bx, icy = (int)cy,
              icx = (int)cx;
    for (int q = lane; q < (int)area; q += G) {
      const int r = q / bw, y = y0 + r, x = x0 + (q - r * bw);
      long long e0 = (long long)(ibx - iax) * (y - iay) - (long long)(iby - iay) * (x - iax);
      long long e1 = (long long)(icx - ibx) * (y - iby) - (long long)(icy - iby) * (x - ibx);
      long long e2 = (long long)(iax - icx) * (y - icy) - (long long)(iay - icy) * (x - icx);
      if ((e0 >= 0 && e1 >= 0 && e2 >= 0) || (e0 <= 0 && e1 <= 0 && e2 <= 0))
        atomicMin(&assign[(size_t)y * W + x], (int)t);
    }
  }
}

__global__ void k_unset_to_neg(int* __restrict__ a, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && a[i] == INT_MAX) a[i] = -1;
}

template <typename V>
__global__ void k_seed_min_tri(const V* __restrict__ tris, long T, int* __restrict__ smt) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * T) return;
  atomicMin(&smt[tris[i]], (int)(i / 3));
}

__global__ void k_fallback(const int* __restrict__ assign, const int* __restrict__ lab,
                           const int* __restrict__ smt, int* __restrict__ out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int t = assign[i];
  if (t < 0 || t == INT_MAX) {
    t = smt[lab[i]];
    if (t < 0 || t == INT_MAX) t = 0;
  }
  out[i] = t;
}

__global__ void k_iota(int* __restrict__ p, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int)i;
}

__global__ void k_segment_bounds(const int* __restrict__ keys, size_t n, int* __restrict__ start,
                                 int* __restrict__ end) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = keys[i];
  if (i == 0 || keys[i - 1] != k) start[k] = (int)i;
  if (i == n - 1 || keys[i + 1] != k) end[k] = (int)i + 1;
}

// sequential row-major double sum + first strict max per segment
__global__ void k_reduce_segments(const int* __restrict__ start, const int* __restrict__ end,
                                  const int* __restrict__ pix, const double* __restrict__ err,
                                  long ntris, double* __restrict__ sums,
                                  long long* __restrict__ amax_idx,
                                  double* __restrict__ amax_val) {
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  int b = start[t], e = end[t];
  double s = 0.0, best = -1.0;
  long long bi = -1;
  for (int i = b; i < e; ++i) {
    int p = pix[i];
    double v = err[p];
    s += v;
    if (v > best) { best = v; bi = p; }
  }
  sums[t] = s;
  if (amax_idx) amax_idx[t] = bi;
  if (amax_val) amax_val[t] = best;
}


// ---- tile-binned rasterisation + bbox-order reduction (B2 path) ----------
// The same three results as assign_triangles -> fallback_assign ->
// reduce_cells (numba_impl.py:442-498), without a global atomic per covered
// pixel and without sorting the 8.3 M pixels by triangle:
//  1. bin: every triangle is listed in the 64 x 32 screen tiles its clamped
//     bounding box overlaps (count, scan, scatter; order inside a tile's
//     list is irrelevant because the winner is the minimum index);
//  2. raster: one CTA per tile takes the minimum containing triangle per
//     pixel in shared memory (inclusive edge test, exact 32-bit integer
//     edge functions: |coordinates| < 2^15), then the fallback for
//     uncovered pixels (seed's lowest incident triangle, else 0).  Fallback
//     pixels are stored with the sign bit set and listed as (t, pixel) keys;
//  3. reduce: one thread per triangle walks its bounding box in row-major
//     order and takes the pixels rasterised to it, merged in pixel order
//     with its (sorted) fallback pixels -- exactly the row-major sequence
//     reduce_cells visits, so the double sums and the first strict maxima
//     are bit-identical.
constexpr int RTW = 64, RTH = 32, RTN = RTW * RTH;

__device__ __forceinline__ bool tri_box(const int* __restrict__ tris, long t,
                                        const int* __restrict__ vy, const int* __restrict__ vx,
                                        int H, int W, int4& v, int2& c, int4& box) {
  const int a = tris[3 * t], b = tris[3 * t + 1], cc = tris[3 * t + 2];
  v = make_int4(vy[a], vx[a], vy[b], vx[b]);
  c = make_int2(vy[cc], vx[cc]);
  box.x = max(0, min(v.x, min(v.z, c.x)));          // ylo
  box.z = min(H - 1, max(v.x, max(v.z, c.x)));      // yhi
  box.y = max(0, min(v.y, min(v.w, c.y)));          // xlo
  box.w = min(W - 1, max(v.y, max(v.w, c.y)));      // xhi
  return box.x <= box.z && box.y <= box.w;
}

__global__ void k_bin_count(const int* __restrict__ tris, long T, const int* __restrict__ vy,
                            const int* __restrict__ vx, int H, int W, int ntx,
                            int4* __restrict__ tv, int2* __restrict__ tc,
                            int4* __restrict__ tbox, unsigned* __restrict__ cnt) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int4 v, box;
  int2 c;
  const bool ok = tri_box(tris, t, vy, vx, H, W, v, c, box);
  tv[t] = v;
  tc[t] = c;
  if (!ok) box = make_int4(1, 1, 0, 0);
  tbox[t] = box;
  if (!ok) return;
  for (int ty = box.x / RTH; ty <= box.z / RTH; ++ty)
    for (int tx = box.y / RTW; tx <= box.w / RTW; ++tx) atomicAdd(&cnt[ty * ntx + tx], 1u);
}

__global__ void k_bin_scatter(const int4* __restrict__ tbox, long T, int ntx,
                              const unsigned* __restrict__ off, unsigned* __restrict__ fill,
                              int* __restrict__ list) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int4 box = tbox[t];
  if (box.x > box.z) return;
  for (int ty = box.x / RTH; ty <= box.z / RTH; ++ty)
    for (int tx = box.y / RTW; tx <= box.w / RTW; ++tx) {
      const int tile = ty * ntx + tx;
      list[off[tile] + atomicAdd(&fill[tile], 1u)] = (int)t;
    }
}

// The pixels of row y inside triangle (v, c) under the reference's
// inclusive test (numba_impl.py:456-462) form one run [x0, x1] (empty when
// x0 > x1): each edge function is affine in x, e_i = K_i - B_i x, and with
// D = e0 + e1 + e2 (twice the signed area, constant) the test is "all
// e_i >= 0" for D >= 0 (for D == 0 that is "all e_i == 0", the same set as
// "all <= 0") and "all e_i <= 0" for D < 0.  Each half-line bound is an
// exact integer floor / ceil, so the run equals the per-pixel test.
__device__ __forceinline__ int fdiv_floor(int a, int b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}
// |K_i| <= 2 (H - 1)(W - 1) < 2^31 for H, W < 32768 (the caller's bound)
__device__ __forceinline__ void tri_span(int y, const int4& v, const int2& c, int lo, int hi,
                                         int& x0, int& x1) {
  const int ay = v.x, ax = v.y, by = v.z, bx = v.w, cy = c.x, cx = c.y;
  int B[3] = {by - ay, cy - by, ay - cy};
  int K[3] = {(bx - ax) * (y - ay) + (by - ay) * ax, (cx - bx) * (y - by) + (cy - by) * bx,
              (ax - cx) * (y - cy) + (ay - cy) * cx};
  // D = e0 + e1 + e2 = K0 + K1 + K2 (the B_i sum to 0): twice the signed area
  const long long D = (long long)K[0] + K[1] + K[2];
  int l = lo, h = hi;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int k = K[i], b = B[i];
    if (D < 0) { k = -k; b = -b; }
    // k - b x >= 0
    if (b == 0) {
      if (k < 0) { l = 1; h = 0; }
    } else if (b > 0) {
      h = min(h, fdiv_floor(k, b));
    } else {
      l = max(l, -fdiv_floor(k, -b));  // ceil(k / b) for b < 0
    }
  }
  x0 = max(l, lo);
  x1 = min(h, hi);
}

// tiles tile0 + blockIdx.x; only image rows [r0, r1) are rasterised and
// written (a row strip; the whole image is 0, H); fb == NULL: no fallback
// list (the strip path collects it from the gathered assignment)
__global__ void __launch_bounds__(256) k_raster_tiles(
    const unsigned* __restrict__ off, const unsigned* __restrict__ cnt,
    const int* __restrict__ list, const int4* __restrict__ tv, const int2* __restrict__ tc,
    const int4* __restrict__ tbox, const int* __restrict__ lab, const int* __restrict__ smt,
    int H, int W, int ntx, int* __restrict__ assign, unsigned long long* __restrict__ fb,
    unsigned long long* __restrict__ nfb, int tile0, int r0, int r1) {
  __shared__ int best[RTN];
  __shared__ unsigned wcount[8];
  __shared__ unsigned long long cbase;
  const int tile = tile0 + blockIdx.x, ty0 = (tile / ntx) * RTH, tx0 = (tile % ntx) * RTW;
  for (int i = threadIdx.x; i < RTN; i += 256) best[i] = INT_MAX;
  __syncthreads();
  // 4 lanes per triangle, 8 triangles per warp in flight.  Rows of the
  // clipped box: wide rows take the exact run (tri_span, three integer
  // divisions per row), narrow rows test their few pixels directly (the
  // reference's inclusive edge functions, exact in 32 bits)
  const int grp = threadIdx.x >> 2, sub = threadIdx.x & 3;
  const unsigned n = cnt[tile], o = off[tile];
  // few (large) triangles: (triangle, row) items so all 64 groups work
  const bool by_row = n < 64;
  const unsigned nitems = by_row ? n * RTH : n;
  for (unsigned item = grp; item < nitems; item += 64) {
    const unsigned i = by_row ? item / RTH : item;
    const int t = list[o + i];
    const int4 v = tv[t];
    const int2 c = tc[t];
    const int4 box = tbox[t];
    int ylo = max(max(box.x, ty0), r0), yhi = min(min(box.z, ty0 + RTH - 1), r1 - 1);
    if (by_row) {
      const int yr = ty0 + (int)(item % RTH);
      if (yr < ylo || yr > yhi) continue;
      ylo = yhi = yr;
    }
    const int xlo = max(box.y, tx0), xhi = min(box.w, tx0 + RTW - 1);
    const int ay = v.x, ax = v.y, by = v.z, bx = v.w, cy = c.x, cx = c.y;
    const bool wide = xhi - xlo >= 24;
    for (int y = ylo; y <= yhi; ++y) {
      int* row = best + (y - ty0) * RTW - tx0;
      if (wide) {
        int x0, x1;
        tri_span(y, v, c, xlo, xhi, x0, x1);
        for (int x = x0 + sub; x <= x1; x += 4) atomicMin(&row[x], t);
      } else {
        const int f0 = (bx - ax) * (y - ay), f1 = (cx - bx) * (y - by), f2 = (ax - cx) * (y - cy);
        for (int x = xlo + sub; x <= xhi; x += 4) {
          const int e0 = f0 - (by - ay) * (x - ax);
          const int e1 = f1 - (cy - by) * (x - bx);
          const int e2 = f2 - (ay - cy) * (x - cx);
          if ((e0 >= 0 && e1 >= 0 && e2 >= 0) || (e0 <= 0 && e1 <= 0 && e2 <= 0))
            atomicMin(&row[x], t);
        }
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i0 = 0; i0 < RTN; i0 += 256) {
    const int i = i0 + threadIdx.x;
    const int y = ty0 + i / RTW, x = tx0 + (i % RTW);
    bool isfb = false;
    int t = 0;
    size_t p = 0;
    if (y < H && x < W && y >= r0 && y < r1) {
      p = (size_t)y * W + x;
      t = best[i];
      if (t == INT_MAX) {
        t = smt[lab[p]];
        if (t < 0 || t == INT_MAX) t = 0;
        isfb = true;
        assign[p] = (int)((unsigned)t | 0x80000000u);
      } else {
        assign[p] = t;
      }
    }
    if (!fb) continue;  // uniform: no fallback list
    // CTA-aggregated append of the fallback pixels
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, isfb);
    if (lane == 0) wcount[w] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned acc = 0;
      for (int k = 0; k < 8; ++k) {
        const unsigned c2 = wcount[k];
        wcount[k] = acc;
        acc += c2;
      }
      cbase = acc ? atomicAdd(nfb, (unsigned long long)acc) : 0ull;
    }
    __syncthreads();
    if (isfb)
      fb[cbase + wcount[w] + __popc(bal & ((1u << lane) - 1u))] =
          ((unsigned long long)(unsigned)t << 32) | (unsigned long long)p;
    __syncthreads();
  }
}

__global__ void k_fb_bounds(const unsigned long long* __restrict__ keys, long n,
                            int* __restrict__ start, int* __restrict__ end) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned t = (unsigned)(keys[i] >> 32);
  if (i == 0 || (unsigned)(keys[i - 1] >> 32) != t) start[t] = (int)i;
  if (i == n - 1 || (unsigned)(keys[i + 1] >> 32) != t) end[t] = (int)i + 1;
}

// one thread per triangle (dense triangulations: boxes of a few dozen
// pixels): the box in row-major order, eight pixels per step with their
// assign / err loads issued together, the triangle's fallback pixels merged
// in pixel order
__global__ void __launch_bounds__(128) k_reduce_tris_small(
    const int4* __restrict__ tbox, long T, const int* __restrict__ assign,
    const double* __restrict__ err, int W, const unsigned long long* __restrict__ fb,
    const int* __restrict__ fs, const int* __restrict__ fe, double* __restrict__ sums,
    long long* __restrict__ amax_idx, double* __restrict__ amax_val, long t0) {
  // triangles [t0, T)
  const long t = t0 + (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int4 box = tbox[t];
  int fi = fs[t];
  const int fend = fe[t];
  long long nfp = fi < fend ? (long long)(fb[fi] & 0xFFFFFFFFull) : LLONG_MAX;
  double s = 0.0, best = -1.0;
  long long bi = -1;
  for (int y = box.x; y <= box.z; ++y) {
    const long long row = (long long)y * W;
    for (int x0 = box.y; x0 <= box.w; x0 += 8) {
      int a[8];
      double e[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = x0 + k <= box.w ? assign[row + x0 + k] : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = a[k] == (int)t ? err[row + x0 + k] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long p = row + x0 + k;
        while (nfp < p) {
          const double v = err[nfp];
          s += v;
          if (v > best) { best = v; bi = nfp; }
          ++fi;
          nfp = fi < fend ? (long long)(fb[fi] & 0xFFFFFFFFull) : LLONG_MAX;
        }
        if (a[k] == (int)t) {
          s += e[k];
          if (e[k] > best) { best = e[k]; bi = p; }
        }
      }
    }
  }
  while (nfp != LLONG_MAX) {
    const double v = err[nfp];
    s += v;
    if (v > best) { best = v; bi = nfp; }
    ++fi;
    nfp = fi < fend ? (long long)(fb[fi] & 0xFFFFFFFFull) : LLONG_MAX;
  }
  sums[t] = s;
  amax_idx[t] = bi;
  amax_val[t] = best;
}

// one warp per triangle: the run of each row of the triangle (tri_span) in
// 32-pixel chunks -- lanes load assign / err coalesced, then lane 0 adds
// the chunk's pixels of this triangle in pixel order from shared memory.
// The triangle's fallback pixels (outside every triangle, hence never inside
// one of its runs) are merged in pixel order between runs.
__global__ void __launch_bounds__(256) k_reduce_tris(
    const int4* __restrict__ tv, const int2* __restrict__ tc, const int4* __restrict__ tbox,
    long T, const int* __restrict__ assign, const double* __restrict__ err, int W,
    const unsigned long long* __restrict__ fb, const int* __restrict__ fs,
    const int* __restrict__ fe, double* __restrict__ sums, long long* __restrict__ amax_idx,
    double* __restrict__ amax_val, unsigned* __restrict__ next, long t0) {
  // triangles [t0, T)
  constexpr int RB = 4;  // rows per batch
  __shared__ double vals[8][RB * 32];
  __shared__ double fv[8][32];
  __shared__ long long qv[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // persistent warps take triangles from a work counter: a few large
  // triangles must not hold a whole wave of CTAs
  while (true) {
    unsigned tt = 0;
    if (lane == 0) tt = atomicAdd(next, 1u);
    const long t = t0 + (long)__shfl_sync(0xFFFFFFFFu, tt, 0);
    if (t >= T) break;
    const int4 box = tbox[t];
    const int4 v = tv[t];
    const int2 c = tc[t];
    int fi = fs[t];  // warp-uniform
    const int fend = fe[t];
    double s = 0.0, best = -1.0;  // meaningful in lane 0
    long long bi = -1;
    // all lanes: consume the fallback pixels below `lim`, 32 per step (the
    // list is sorted, so the taken ones are a prefix), added by lane 0
    auto drain = [&](long long lim) {
      while (fi < fend) {
        const int j = fi + lane;
        const long long q = j < fend ? (long long)(fb[j] & 0xFFFFFFFFull) : LLONG_MAX;
        const bool take = q < lim;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, take);
        if (!bal) break;
        fv[w][lane] = take ? err[q] : 0.0;
        qv[w][lane] = q;
        __syncwarp();
        if (lane == 0) {
          for (unsigned b = bal; b; b &= b - 1) {
            const int k = __ffs(b) - 1;
            const double ev = fv[w][k];
            s += ev;
            if (ev > best) { best = ev; bi = qv[w][k]; }
          }
        }
        __syncwarp();
        const int nt = __popc(bal);
        fi += nt;
        if (nt < 32) break;
      }
    };
    // add the chunk of `row` starting at column xc (hits in `bal`, values
    // staged in vals[w][slot]) in pixel order, after the earlier fallbacks
    auto take = [&](long long row, int xc, unsigned bal, int slot) {
      drain(row + xc);
      if (lane == 0) {
        for (unsigned b = bal; b; b &= b - 1) {
          const int k = __ffs(b) - 1;
          const double ev = vals[w][slot * 32 + k];
          s += ev;
          if (ev > best) { best = ev; bi = row + xc + k; }
        }
      }
      __syncwarp();
    };
    for (int yb = box.x; yb <= box.z; yb += RB) {
      int x0[RB], x1[RB];
      bool narrow = true;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        x0[r] = 1;
        x1[r] = 0;
        if (yb + r <= box.z) tri_span(yb + r, v, c, box.y, box.w, x0[r], x1[r]);
        narrow = narrow && x1[r] - x0[r] < 32;
      }
      if (narrow) {
        // RB rows of at most one chunk each: all loads in flight together
        bool hit[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int x = x0[r] + lane;
          hit[r] = x <= x1[r] && assign[(long long)(yb + r) * W + x] == (int)t;
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
          vals[w][r * 32 + lane] = hit[r] ? err[(long long)(yb + r) * W + x0[r] + lane] : 0.0;
        unsigned bal[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) bal[r] = __ballot_sync(0xFFFFFFFFu, hit[r]);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (bal[r]) take((long long)(yb + r) * W, x0[r], bal[r], r);
        continue;
      }
      for (int r = 0; r < RB && yb + r <= box.z; ++r) {
        const long long row = (long long)(yb + r) * W;
        for (int xc = x0[r]; xc <= x1[r]; xc += 32) {
          const int x = xc + lane;
          const bool h = x <= x1[r] && assign[row + x] == (int)t;
          vals[w][lane] = h ? err[row + x] : 0.0;
          const unsigned b = __ballot_sync(0xFFFFFFFFu, h);
          __syncwarp();
          if (b) take(row, xc, b, 0);
        }
      }
    }
    drain(LLONG_MAX);
    if (lane == 0) {
      sums[t] = s;
      amax_idx[t] = bi;
      amax_val[t] = best;
    }
  }
}

__global__ void k_fs_dither(const double* __restrict__ dens, double* __restrict__ buf,
                            uint8_t* __restrict__ out, int H, int W) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (size_t i = 0; i < (size_t)H * W; ++i) buf[i] = dens[i];
  for (int y = 0; y < H; ++y) {
    int x0 = (y % 2 == 0) ? 0 : W - 1, x1 = (y % 2 == 0) ? W : -1, sgn = (y % 2 == 0) ? 1 : -1;
    for (int x = x0; x != x1; x += sgn) {
      size_t k = (size_t)y * W + x;
      double val = buf[k];
      int bit = val >= 0.5 ? 1 : 0;
      out[k] = (uint8_t)bit;
      double e = val - (double)bit;
      int xn = x + sgn;
      if (xn >= 0 && xn < W) buf[k + sgn] += e * (7.0 / 16.0);
      if (y + 1 < H) {
        int xb = x - sgn;
        if (xb >= 0 && xb < W) buf[k + W - sgn] += e * (3.0 / 16.0);
        buf[k + W] += e * (5.0 / 16.0);
        if (xn >= 0 && xn < W) buf[k + W + sgn] += e * (1.0 / 16.0);
      }
    }
  }
}

// ---- selection (spatial.py:245-259) -----------------------------------------
__global__ void k_valid_flags(const long long* __restrict__ amax,
                              const uint8_t* __restrict__ mask, long T,
                              uint8_t* __restrict__ flags) {
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  long long px = amax[t];
  flags[t] = px >= 0 && !mask[px];
}

__global__ void k_not_mask(const uint8_t* __restrict__ mask, size_t n,
                           uint8_t* __restrict__ flags) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = !mask[i];
}

// sort keys of non-negative doubles: the IEEE bit pattern orders them
// ascending, its complement descending
__global__ void k_desc_keys(const int* __restrict__ idx, long n, const double* __restrict__ v,
                            unsigned long long* __restrict__ keys, int descending) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long b = (unsigned long long)__double_as_longlong(v[idx[i]]);
  keys[i] = descending ? ~b : b;
}

__global__ void k_set_mask_val(const int* __restrict__ idx, long n, uint8_t* __restrict__ mask,
                               uint8_t val) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) mask[idx[i]] = val;
}

__global__ void k_apply_picks(const int* __restrict__ order, long npick,
                              const long long* __restrict__ amax, uint8_t* __restrict__ mask) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npick) mask[amax[order[i]]] = 1;
}

__global__ void k_set_mask(const int* __restrict__ idx, long n, uint8_t* __restrict__ mask) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) mask[idx[i]] = 1;
}

inline dim3 grid2(int W, int H) { return dim3(cdiv(W, BX), cdiv(H, BY)); }

int bits_for(long n) {
  int b = 1;
  while ((1L << b) < n + 1 && b < 31) ++b;
  return b;
}

}  // namespace

// ---------------------------------------------------------------------------
// helpers shared with the B1 wrappers and the B2 workspace
// ---------------------------------------------------------------------------

int jfa_passes(int* a, int* b, const int* sy, const int* sx, const long long* steps,
               int nsteps, int H, int W, int** result, cudaStream_t s) {
  bool small = 4.0 * ((double)H * H + (double)W * W) < 2.0e9;
  int* cur = a;
  int* nxt = b;
  for (int i = 0; i < nsteps; ++i) {
    if (small)
      k_jfa_pass<int><<<grid2(W, H), dim3(BX, BY), 0, s>>>(cur, nxt, sy, sx, (int)steps[i], H, W);
    else
      k_jfa_pass<long long><<<grid2(W, H), dim3(BX, BY), 0, s>>>(cur, nxt, sy, sx,
                                                                  (int)steps[i], H, W);
    SP_CHECK_LAUNCH();
    int* t = cur;
    cur = nxt;
    nxt = t;
  }
  *result = cur;
  return 0;
}

int dist2(const int* lab, const int* sy, const int* sx, long long* out,
          unsigned long long* dmax, int H, int W, int m, cudaStream_t s) {
  if (dmax) SP_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s));
  k_dist2<<<grid2(W, H), dim3(BX, BY), 0, s>>>(lab, sy, sx, out, dmax, H, W, m);
  SP_CHECK_LAUNCH();
  return 0;
}

int seeds_to_soa(const long long* seeds, long m, int* sy, int* sx, cudaStream_t s) {
  if (m <= 0) return 0;
  k_seeds_i64_to_soa<<<cdiv(m, 256), 256, 0, s>>>(seeds, m, sy, sx);
  SP_CHECK_LAUNCH();
  return 0;
}

int fs_dither(const double* dens, uint8_t* out, int H, int W, cudaStream_t s) {
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(double) * (size_t)H * W));
  k_fs_dither<<<1, 1, 0, s>>>(dens, (double*)scr.p, out, H, W);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename V>
int assign_tris(const V* tris, long T, const V* vy, const V* vx, int H, int W, int* assign,
                bool neg_unset, cudaStream_t s) {
  size_t n = (size_t)H * W;
  k_fill_i32<<<cdiv(n, 256), 256, 0, s>>>(assign, n, INT_MAX);
  SP_CHECK_LAUNCH();
  if (T > 0) {
    long warps = std::min<long>(T, (long)num_sms() * 64);
    k_assign_tris<V><<<cdiv(warps * 32, 256), 256, 0, s>>>(tris, T, vy, vx, H, W, assign);
    SP_CHECK_LAUNCH();
  }
  if (neg_unset) {
    k_unset_to_neg<<<cdiv(n, 256), 256, 0, s>>>(assign, n);
    SP_CHECK_LAUNCH();
  }
  return 0;
}
template int assign_tris<long long>(const long long*, long, const long long*, const long long*,
                                    int, int, int*, bool, cudaStream_t);
template int assign_tris<int>(const int*, long, const int*, const int*, int, int, int*, bool,
                              cudaStream_t);

int fallback(const int* assign, const int* lab, const int* smt, int* out, size_t n,
             cudaStream_t s) {
  k_fallback<<<cdiv(n, 256), 256, 0, s>>>(assign, lab, smt, out, n);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename V>
int seed_min_tri(const V* tris, long T, int* smt, long m, cudaStream_t s) {
  k_fill_i32<<<cdiv(m, 256), 256, 0, s>>>(smt, (size_t)m, INT_MAX);
  SP_CHECK_LAUNCH();
  if (T > 0) {
    k_seed_min_tri<V><<<cdiv(3 * T, 256), 256, 0, s>>>(tris, T, smt);
    SP_CHECK_LAUNCH();
  }
  return 0;
}
template int seed_min_tri<int>(const int*, long, int*, long, cudaStream_t);

// per-segment sequential reduction; `assign` values must lie in [0, nseg)
int reduce_cells(const int* assign, const double* err, long nseg, double* sums,
                 long long* amax_idx, double* amax_val, int H, int W, cudaStream_t s) {
  size_t n = (size_t)H * W;
  int nbits = bits_for(nseg);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const int*)nullptr, (int*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)n, 0, nbits, s);
  Scratch scr(s);
  size_t ints = 3 * n + 2 * (size_t)nseg + 64;
  SP_TRY(scr.alloc(tmp_bytes + sizeof(int) * ints));
  int* keys_out = (int*)scr.p;
  int* vals_in = keys_out + n;
  int* vals_out = vals_in + n;
  int* start = vals_out + n;
  int* end = start + nseg;
  void* tmp = (void*)(end + nseg + 32);
  k_iota<<<cdiv(n, 256), 256, 0, s>>>(vals_in, n);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, assign, keys_out, vals_in, vals_out,
                                          (int)n, 0, nbits, s));
  SP_CUDA(cudaMemsetAsync(start, 0, sizeof(int) * 2 * nseg, s));
  k_segment_bounds<<<cdiv(n, 256), 256, 0, s>>>(keys_out, n, start, end);
  SP_CHECK_LAUNCH();
  if (nseg > 0) {
    k_reduce_segments<<<cdiv(nseg, 128), 128, 0, s>>>(start, end, vals_out, err, nseg, sums,
                                                      amax_idx, amax_val);
    SP_CHECK_LAUNCH();
  }
  return 0;
}

// ---------------------------------------------------------------------------
// B2 workspace
// ---------------------------------------------------------------------------

Geo::~Geo() {
  for (void* p : {(void*)lab_a, (void*)lab_b, (void*)rank, (void*)sy, (void*)sx, (void*)keys,
                  (void*)keys2,
                  (void*)nkeys, (void*)tris, (void*)assign, (void*)smt, (void*)sums,
                  (void*)amax, (void*)amax_val, (void*)dmax, (void*)flags, (void*)idx,
                  (void*)nsel, (void*)h_small})
    if (p) {
      if (p == (void*)h_small) cudaFreeHost(p);
      else cudaFree(p);
    }
}

int geo_create(Geo** out, int H, int W) {
  *out = nullptr;
  Geo* g = new Geo();
  g->H = H;
  g->W = W;
  size_t n = (size_t)H * W;
  size_t ncorner = (size_t)(H > 1 ? H - 1 : 0) * (W > 1 ? W - 1 : 0);
  g->key_cap = 2 * ncorner + 2;
  g->tri_cap = g->key_cap;
  bool ok = cudaMalloc(&g->lab_a, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->lab_b, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->rank, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->sy, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->sx, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->idx, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->flags, n) == cudaSuccess &&
            cudaMalloc(&g->keys, sizeof(unsigned long long) * g->key_cap) == cudaSuccess &&
            cudaMalloc(&g->nkeys, sizeof(unsigned long long) * 4) == cudaSuccess &&
            cudaMalloc(&g->tris, sizeof(int) * 3 * g->tri_cap) == cudaSuccess &&
            cudaMalloc(&g->assign, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->smt, sizeof(int) * n) == cudaSuccess &&
            cudaMalloc(&g->sums, sizeof(double) * g->tri_cap) == cudaSuccess &&
            cudaMalloc(&g->amax, sizeof(long long) * g->tri_cap) == cudaSuccess &&
            cudaMalloc(&g->amax_val, sizeof(double) * g->tri_cap) == cudaSuccess &&
            cudaMalloc(&g->dmax, sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&g->nsel, sizeof(int) * 4) == cudaSuccess &&
            cudaMallocHost(&g->h_small, 64) == cudaSuccess;
  if (!ok) {
    set_error("geometry workspace allocation failed (%d x %d)", H, W);
    delete g;
    return -1;
  }
  *out = g;
  return 0;
}

// geometry.py:76-89
// short JFA steps on pixel quads (k_jfa_pass_key4s, 1) or per pixel (0)
static int jfa_short4_on = 1;
int jfa_short4(int v) {
  if (v >= 0) jfa_short4_on = v;
  return jfa_short4_on;
}

static std::vector<long long> steps_for(int max_dim, double hint) {
  long long start;
  if (hint >= 1.0) {
    double lg = std::ceil(std::log2(std::max(1.0, hint)));
    start = 1LL << std::max(0, (int)lg);
    start = std::min(start, (long long)std::max(1, max_dim / 2));
  } else if (max_dim >= 2) {
    start = 1LL << ((int)std::ceil(std::log2((double)max_dim)) - 1);
  } else {
    start = 1;
  }
  std::vector<long long> out{1};
  for (long long v = start; v >= 1; v /= 2) out.push_back(v);
  return out;
}

int geo_voronoi(Geo* g, const uint8_t* mask, double hint, long* m_out, double* radius,
                int* nsteps_out, cudaStream_t s) {
  const int H = g->H, W = g->W;
  size_t n = (size_t)H * W;
  // seeds: row-major nonzero (cub select on a counting iterator)
  k_mask_flags<<<cdiv(n, 256), 256, 0, s>>>(mask, g->flags, n);
  SP_CHECK_LAUNCH();
  cub::CountingInputIterator<int> it(0);
  size_t tmp_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, g->flags, g->idx, g->nsel, (int)n, s);
  {
    Scratch scr(s);
    SP_TRY(scr.alloc(tmp_bytes));
    SP_CUDA(cub::DeviceSelect::Flagged(scr.p, tmp_bytes, it, g->flags, g->idx, g->nsel, (int)n, s));
  }
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  long m = ((int*)g->h_small)[0];
  if (m == 0) {
    set_error("mask has no stored pixels to seed from");
    return -3;
  }
  g->m = m;
  std::vector<long long> steps = steps_for(std::max(H, W), hint);
  const bool keyed = H <= kKeyMax && W <= kKeyMax;
  if (keyed) {
    // packed-coordinate labels (k_jfa_pass_key); rank[] maps keys back
    k_seed_init<<<cdiv(m, 256), 256, 0, s>>>(g->idx, m, W, g->sy, g->sx, g->rank);
    SP_CHECK_LAUNCH();
    unsigned* cur = (unsigned*)g->lab_a;
    unsigned* nxt = (unsigned*)g->lab_b;
    k_jfa_key_init<<<grid2(W, H), dim3(BX, BY), 0, s>>>(mask, cur, H, W);
    SP_CHECK_LAUNCH();
    for (size_t i = 0; i < steps.size(); ++i) {
      if (steps[i] % 4 == 0 && W % 4 == 0)
        k_jfa_pass_key4<<<grid2(W / 4, H), dim3(BX, BY), 0, s>>>(cur, nxt, (int)steps[i], H, W);
      else if (steps[i] <= 2 && W % 4 == 0 && jfa_short4_on)
        k_jfa_pass_key4s<<<grid2(W / 4, H), dim3(BX, BY), 0, s>>>(cur, nxt, (int)steps[i], H, W);
      else
        k_jfa_pass_key<<<grid2(W, H), dim3(BX, BY), 0, s>>>(cur, nxt, (int)steps[i], H, W);
      SP_CHECK_LAUNCH();
      std::swap(cur, nxt);
    }
    if ((int*)cur != g->lab_a) std::swap(g->lab_a, g->lab_b);  // labels live in lab_a
    SP_CUDA(cudaMemsetAsync(g->dmax, 0, sizeof(unsigned long long), s));
    k_jfa_key_finish<<<grid2(W, H), dim3(BX, BY), 0, s>>>((unsigned*)g->lab_a, g->rank, g->sy,
                                                          g->sx, m, g->dmax, H, W);
    SP_CHECK_LAUNCH();
  } else {
    k_fill_i32<<<cdiv(n, 256), 256, 0, s>>>(g->lab_a, n, -1);
    SP_CHECK_LAUNCH();
    k_seed_init<<<cdiv(m, 256), 256, 0, s>>>(g->idx, m, W, g->sy, g->sx, g->lab_a);
    SP_CHECK_LAUNCH();
    int* res = nullptr;
    SP_TRY(jfa_passes(g->lab_a, g->lab_b, g->sy, g->sx, steps.data(), (int)steps.size(), H, W,
                      &res, s));
    if (res != g->lab_a) std::swap(g->lab_a, g->lab_b);  // labels live in lab_a
    SP_TRY(dist2(g->lab_a, g->sy, g->sx, nullptr, g->dmax, H, W, (int)g->m, s));
  }
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->dmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  unsigned long long d2 = ((unsigned long long*)g->h_small)[0];
  *m_out = m;
  *radius = std::sqrt((double)d2);
  if (nsteps_out) *nsteps_out = (int)steps.size();
  g->T = 0;
  return 0;
}

static int sort_unique_keys(Geo* g, long nk, long* n_out, bool decode, cudaStream_t s);

// >= 2^21 seeds: the packed 3 x 21-bit keys would overflow.  The corner
// triples are kept as (a, b << 32 | c) pairs and sorted lexicographically by
// two stable radix passes (low word, then high word, the payload an index),
// then deduplicated -- the same sorted unique triangle list.
static int delaunay_wide(Geo* g, long* T_out, cudaStream_t s) {
  const int H = g->H, W = g->W;
  if (!g->keys2) SP_CUDA(cudaMalloc(&g->keys2, sizeof(unsigned) * g->key_cap));
  SP_CUDA(cudaMemsetAsync(g->nkeys, 0, sizeof(unsigned long long) * 2, s));
  k_corner_scan<true><<<grid2(W, H), dim3(BX, BY), 0, s>>>(g->lab_a, H, W, g->keys, g->nkeys,
                                                           0, H - 1, g->keys2);
  SP_CHECK_LAUNCH();
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nkeys, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long nk = (long)((unsigned long long*)g->h_small)[0];
  if (nk == 0) return 0;
  const int nb = bits_for(g->m - 1);
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, (int)nk, 0, 32 + nb, s);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const unsigned*)nullptr, (unsigned*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)nk, 0, nb, s);
  cub::CountingInputIterator<int> it(0);
  cub::DeviceSelect::Flagged(nullptr, b3, it, (const uint8_t*)nullptr, (int*)nullptr,
                             (int*)nullptr, (int)nk, s);
  const size_t nn = (size_t)nk;
  Scratch scr(s);
  SP_TRY(scr.alloc(nn * (8 + 8 + 4 + 4 + 4 + 4 + 4 + 1) + std::max(b1, std::max(b2, b3)) + 1024));
  unsigned long long* lo_s = (unsigned long long*)scr.p;
  unsigned long long* lo_f = lo_s + nn;
  unsigned* hi_g = (unsigned*)(lo_f + nn);
  unsigned* hi_s = hi_g + nn;
  int* idx0 = (int*)(hi_s + nn);
  int* idx1 = idx0 + nn;
  int* idx2 = idx1 + nn;
  uint8_t* flag = (uint8_t*)(idx2 + nn);
  void* tmp = (void*)(((uintptr_t)(flag + nn) + 255) & ~(uintptr_t)255);
  k_iota<<<cdiv(nn, 256), 256, 0, s>>>(idx0, nn);
  SP_CHECK_LAUNCH();
  // pass 1: by the low word (b, c); pass 2 (stable): by the high word a
  SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b1, g->keys, lo_s, idx0, idx1, (int)nk, 0,
                                          32 + nb, s));
  k_gather_u64_u32<<<cdiv(nn, 256), 256, 0, s>>>(idx1, nk, g->keys, g->keys2, nullptr, hi_g);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b2, hi_g, hi_s, idx1, idx2, (int)nk, 0, nb, s));
  k_gather_u64_u32<<<cdiv(nn, 256), 256, 0, s>>>(idx2, nk, g->keys, g->keys2, lo_f, nullptr);
  SP_CHECK_LAUNCH();
  k_wide_uniq_flags<<<cdiv(nn, 256), 256, 0, s>>>(lo_f, hi_s, nk, flag);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceSelect::Flagged(tmp, b3, it, flag, idx0, g->nsel, (int)nk, s));
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long T = ((int*)g->h_small)[0];
  // unique pairs into keys / keys2, then the triangles
  k_gather_u64_u32<<<cdiv(T, 256), 256, 0, s>>>(idx0, T, lo_f, hi_s, g->keys, g->keys2);
  SP_CHECK_LAUNCH();
  k_decode_tris_wide<<<cdiv(T, 256), 256, 0, s>>>(g->keys, g->keys2, T, g->tris);
  SP_CHECK_LAUNCH();
  g->T = T;
  *T_out = T;
  return 0;
}

// seed count from which the wide keys are used (2^21; lower only for tests)
static long wide_from = 1L << 21;
long geo_wide_threshold(long v) {
  if (v > 0 && v <= (1L << 21)) wide_from = v;
  return wide_from;
}

int geo_delaunay(Geo* g, long* T_out, cudaStream_t s) {
  const int H = g->H, W = g->W;
  g->T = 0;
  *T_out = 0;
  if (H < 2 || W < 2 || g->m < 3) return 0;
  SP_CUDA(cudaMemsetAsync(g->nkeys, 0, sizeof(unsigned long long) * 2, s));
  if (g->m >= wide_from) return delaunay_wide(g, T_out, s);
  k_corner_scan<false><<<grid2(W, H), dim3(BX, BY), 0, s>>>(g->lab_a, H, W, g->keys, g->nkeys,
                                                            0, H - 1, nullptr);
  SP_CHECK_LAUNCH();
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nkeys, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  long nk = (long)((unsigned long long*)g->h_small)[0];
  if (nk == 0) return 0;
  long T = 0;
  SP_TRY(sort_unique_keys(g, nk, &T, true, s));
  g->T = T;
  *T_out = T;
  return 0;
}

// sort + unique of g->keys[0, nk) in place (np.unique(axis=0) on sorted
// triples == sorted packed keys); decode: the triangles of the unique keys
static int sort_unique_keys(Geo* g, long nk, long* n_out, bool decode, cudaStream_t s) {
  *n_out = 0;
  if (nk == 0) return 0;
  int nbits = bits_for(g->m - 1);
  int endbit = 42 + nbits;
  size_t sort_bytes = 0, uniq_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int)nk, 0, endbit, s);
  cub::DeviceSelect::Unique(nullptr, uniq_bytes, (const unsigned long long*)nullptr,
                            (unsigned long long*)nullptr, (int*)nullptr, (int)nk, s);
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(unsigned long long) * nk + std::max(sort_bytes, uniq_bytes) + 256));
  unsigned long long* sorted = (unsigned long long*)scr.p;
  void* tmp = (void*)(sorted + nk + 16);
  SP_CUDA(cub::DeviceRadixSort::SortKeys(tmp, sort_bytes, g->keys, sorted, (int)nk, 0, endbit, s));
  SP_CUDA(cub::DeviceSelect::Unique(tmp, uniq_bytes, sorted, g->keys, g->nsel, (int)nk, s));
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  long T = ((int*)g->h_small)[0];
  if (decode) {
    k_decode_tris<<<cdiv(T, 256), 256, 0, s>>>(g->keys, T, g->tris);
    SP_CHECK_LAUNCH();
  }
  *n_out = T;
  return 0;
}

// B2 accumulate (geometry.py:197-223) through the tile-binned rasteriser and
// the bbox-order reduction (see k_raster_tiles): bit-identical to the
// assign_tris / fallback / reduce_cells sequence, which stays the kernel-table
// (B1) path and the fallback for images of 2^15 pixels or more per side or
// pixel counts that do not fit the 32-bit fallback keys.
static int accumulate_tiled(Geo* g, const double* err, cudaStream_t s) {
  const int H = g->H, W = g->W;
  const long T = g->T;
  const size_t n = (size_t)H * W;
  const int ntx = cdiv(W, RTW), nty = cdiv(H, RTH), ntile = ntx * nty;
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const unsigned*)nullptr,
                                (unsigned*)nullptr, ntile, s);
  Scratch scr(s);
  const size_t tb = sizeof(int4) * 2 * (size_t)T + sizeof(int2) * (size_t)T;
  const size_t ub = sizeof(unsigned) * 3 * (size_t)ntile + 64;
  SP_TRY(scr.alloc(tb + ub + scan_bytes + 256));
  int4* tv = (int4*)scr.p;
  int4* tbox = tv + T;
  int2* tc = (int2*)(tbox + T);
  unsigned* cnt = (unsigned*)(tc + T);
  unsigned* off = cnt + ntile;
  unsigned* fill = off + ntile;
  void* scan_tmp = (void*)(((uintptr_t)(fill + ntile) + 255) & ~(uintptr_t)255);
  SP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * ntile, s));
  SP_CUDA(cudaMemsetAsync(fill, 0, sizeof(unsigned) * ntile, s));
  k_bin_count<<<cdiv(T, 256), 256, 0, s>>>(g->tris, T, g->sy, g->sx, H, W, ntx, tv, tc, tbox,
                                           cnt);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, off, ntile, s));
  unsigned* hs = (unsigned*)g->h_small;
  SP_CUDA(cudaMemcpyAsync(hs, off + ntile - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaMemcpyAsync(hs + 1, cnt + ntile - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const size_t nlist = (size_t)hs[0] + hs[1];
  Scratch lst(s);
  SP_TRY(lst.alloc(sizeof(int) * (nlist + 1)));
  k_bin_scatter<<<cdiv(T, 256), 256, 0, s>>>(tbox, T, ntx, off, fill, (int*)lst.p);
  SP_CHECK_LAUNCH();
  SP_TRY(seed_min_tri<int>(g->tris, T, g->smt, g->m, s));
  unsigned long long* fbk = (unsigned long long*)g->keys;  // n <= key_cap scratch keys
  SP_CUDA(cudaMemsetAsync(g->nkeys + 2, 0, sizeof(unsigned long long), s));
  k_raster_tiles<<<ntile, 256, 0, s>>>(off, cnt, (const int*)lst.p, tv, tc, tbox, g->lab_a,
                                       g->smt, H, W, ntx, g->assign, fbk, g->nkeys + 2, 0, 0,
                                       H);
  SP_CHECK_LAUNCH();
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nkeys + 2, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long nfb = (long)((unsigned long long*)g->h_small)[0];
  // fallback pixels sorted by (triangle, pixel); per-triangle ranges
  Scratch fbs(s);
  size_t sort_bytes = 0;
  if (nfb > 0)
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int)nfb, 0,
                                   32 + bits_for(T), s);
  SP_TRY(fbs.alloc(sizeof(unsigned long long) * (nfb + 1) + sizeof(int) * 2 * (size_t)T +
                   sort_bytes + 512));
  unsigned long long* fsorted = (unsigned long long*)fbs.p;
  int* fs = (int*)(fsorted + nfb + 1);
  int* fe = fs + T;
  void* sort_tmp = (void*)(((uintptr_t)(fe + T) + 255) & ~(uintptr_t)255);
  SP_CUDA(cudaMemsetAsync(fs, 0, sizeof(int) * 2 * (size_t)T, s));
  if (nfb > 0) {
    SP_CUDA(cub::DeviceRadixSort::SortKeys(sort_tmp, sort_bytes, fbk, fsorted, (int)nfb, 0,
                                           32 + bits_for(T), s));
    k_fb_bounds<<<cdiv(nfb, 256), 256, 0, s>>>(fsorted, nfb, fs, fe);
    SP_CHECK_LAUNCH();
  }
  if ((double)T * 128.0 >= (double)n) {
    // dense: boxes of a few dozen pixels, one thread per triangle
    k_reduce_tris_small<<<cdiv(T, 128), 128, 0, s>>>(tbox, T, g->assign, err, W, fsorted, fs,
                                                     fe, g->sums, g->amax, g->amax_val, 0);
  } else {
    const long rblocks = std::min<long>(cdiv(T, 8), (long)num_sms() * 4);
    SP_CUDA(cudaMemsetAsync(g->nkeys + 3, 0, sizeof(unsigned long long), s));
    k_reduce_tris<<<rblocks, 256, 0, s>>>(tv, tc, tbox, T, g->assign, err, W, fsorted, fs, fe,
                                          g->sums, g->amax, g->amax_val,
                                          (unsigned*)(g->nkeys + 3), 0);
  }
  SP_CHECK_LAUNCH();
  return 0;
}

// ---- row-strip partition of the Delaunay step and the accumulate (SURVEY.md
// section 8e): every rank holds the full labels (jump flooding stays
// replicated: each pass reads the whole previous field) and
//   1. scans the corners of its own rows, sort + unique locally
//      (geo_corner_keys); the ranks' key lists are all-gathered and merged
//      by one more sort + unique (geo_delaunay_from_keys) -- the union of
//      the corner triples in sorted order, the same triangle list and
//      indices as the unpartitioned scan;
//   2. rasterises its own rows (geo_raster_rows); the assignment rows are
//      all-gathered, so every rank holds the full pixel -> triangle map;
//   3. reduces a contiguous range of triangles over the FULL map, each in
//      the reference's sequential row-major order (geo_reduce_range); the
//      (sum, argmax) ranges are all-gathered.  A triangle's sum is never
//      split across ranks, so the f64 rounding is the unpartitioned one.

int geo_corner_keys(Geo* g, int r0, int r1, long* n_out, cudaStream_t s) {
  const int H = g->H, W = g->W;
  *n_out = 0;
  g->T = 0;
  if (H < 2 || W < 2 || g->m < 3) return 0;
  if (g->m >= (1L << 21)) {
    set_error("the strip-partitioned Delaunay step packs keys for < 2^21 stored pixels");
    return -2;
  }
  const int y0c = std::max(0, r0), y1c = std::min(r1, H - 1);
  SP_CUDA(cudaMemsetAsync(g->nkeys, 0, sizeof(unsigned long long) * 2, s));
  if (y1c > y0c) {
    k_corner_scan<false><<<dim3(cdiv(W, BX), cdiv(y1c - y0c, BY)), dim3(BX, BY), 0, s>>>(
        g->lab_a, H, W, g->keys, g->nkeys, y0c, y1c, nullptr);
    SP_CHECK_LAUNCH();
  }
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nkeys, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long nk = (long)((unsigned long long*)g->h_small)[0];
  return sort_unique_keys(g, nk, n_out, false, s);
}

int geo_delaunay_from_keys(Geo* g, const unsigned long long* keys, long n, long* T_out,
                           cudaStream_t s) {
  *T_out = 0;
  g->T = 0;
  if ((size_t)n > g->key_cap) {
    set_error("%ld keys exceed the workspace's %zu", n, g->key_cap);
    return -2;
  }
  if (n == 0) return 0;
  if (keys != g->keys)
    SP_CUDA(cudaMemcpyAsync(g->keys, keys, sizeof(unsigned long long) * n,
                            cudaMemcpyDeviceToDevice, s));
  long T = 0;
  SP_TRY(sort_unique_keys(g, n, &T, true, s));
  g->T = T;
  *T_out = T;
  return 0;
}

// the triangles' vertices / boxes (k_bin_count) and their per-tile lists
struct TriBins {
  int4* tv;
  int4* tbox;
  int2* tc;
  unsigned *cnt, *off, *fill;
  int* list;
  int ntx, ntile;
};

static int bin_triangles(Geo* g, Scratch& scr, Scratch& lst, TriBins& b, cudaStream_t s) {
  const int H = g->H, W = g->W;
  const long T = g->T;
  b.ntx = cdiv(W, RTW);
  b.ntile = b.ntx * cdiv(H, RTH);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const unsigned*)nullptr,
                                (unsigned*)nullptr, b.ntile, s);
  const size_t tb = sizeof(int4) * 2 * (size_t)T + sizeof(int2) * (size_t)T;
  const size_t ub = sizeof(unsigned) * 3 * (size_t)b.ntile + 64;
  SP_TRY(scr.alloc(tb + ub + scan_bytes + 256));
  b.tv = (int4*)scr.p;
  b.tbox = b.tv + T;
  b.tc = (int2*)(b.tbox + T);
  b.cnt = (unsigned*)(b.tc + T);
  b.off = b.cnt + b.ntile;
  b.fill = b.off + b.ntile;
  void* scan_tmp = (void*)(((uintptr_t)(b.fill + b.ntile) + 255) & ~(uintptr_t)255);
  SP_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(unsigned) * b.ntile, s));
  SP_CUDA(cudaMemsetAsync(b.fill, 0, sizeof(unsigned) * b.ntile, s));
  k_bin_count<<<cdiv(T, 256), 256, 0, s>>>(g->tris, T, g->sy, g->sx, H, W, b.ntx, b.tv, b.tc,
                                           b.tbox, b.cnt);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, b.cnt, b.off, b.ntile, s));
  unsigned* hs = (unsigned*)g->h_small;
  SP_CUDA(cudaMemcpyAsync(hs, b.off + b.ntile - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaMemcpyAsync(hs + 1, b.cnt + b.ntile - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const size_t nlist = (size_t)hs[0] + hs[1];
  SP_TRY(lst.alloc(sizeof(int) * (nlist + 1)));
  b.list = (int*)lst.p;
  k_bin_scatter<<<cdiv(T, 256), 256, 0, s>>>(b.tbox, T, b.ntx, b.off, b.fill, b.list);
  SP_CHECK_LAUNCH();
  return 0;
}

static bool strip_geometry_ok(const Geo* g) {
  const size_t n = (size_t)g->H * g->W;
  return g->H < 32768 && g->W < 32768 && n < (1ull << 32) && n <= g->key_cap;
}

int geo_raster_rows(Geo* g, int r0, int r1, cudaStream_t s) {
  const int H = g->H, W = g->W;
  if (!strip_geometry_ok(g)) {
    set_error("strip geometry needs < 2^15 pixels per side");
    return -2;
  }
  r0 = std::max(0, r0);
  r1 = std::min(H, r1);
  if (g->T == 0 || r1 <= r0) return 0;
  Scratch scr(s), lst(s);
  TriBins b;
  SP_TRY(bin_triangles(g, scr, lst, b, s));
  SP_TRY(seed_min_tri<int>(g->tris, g->T, g->smt, g->m, s));
  const int ty0 = r0 / RTH, ty1 = (r1 - 1) / RTH;
  k_raster_tiles<<<(ty1 - ty0 + 1) * b.ntx, 256, 0, s>>>(
      b.off, b.cnt, b.list, b.tv, b.tc, b.tbox, g->lab_a, g->smt, H, W, b.ntx, g->assign,
      nullptr, nullptr, ty0 * b.ntx, r0, r1);
  SP_CHECK_LAUNCH();
  return 0;
}

// fallback pixels (assignment high bit) of the full map, (triangle, pixel) keys
__global__ void k_fb_collect(const int* __restrict__ assign, size_t n,
                             unsigned long long* __restrict__ fb,
                             unsigned long long* __restrict__ nfb) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int a = p < n ? assign[p] : 0;
  const bool isfb = p < n && (a & 0x80000000);
  const unsigned bal = __ballot_sync(0xFFFFFFFFu, isfb);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(nfb, (unsigned long long)__popc(bal));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (isfb)
    fb[base + __popc(bal & ((1u << lane) - 1u))] =
        ((unsigned long long)((unsigned)a & 0x7FFFFFFFu) << 32) | (unsigned long long)p;
}

int geo_reduce_range(Geo* g, const double* err, long t0, long t1, cudaStream_t s) {
  const int H = g->H, W = g->W;
  const long T = g->T;
  const size_t n = (size_t)H * W;
  if (!strip_geometry_ok(g)) {
    set_error("strip geometry needs < 2^15 pixels per side");
    return -2;
  }
  t0 = std::max(0L, t0);
  t1 = std::min(T, t1);
  if (T == 0 || t1 <= t0) return 0;
  Scratch scr(s), lst(s);
  TriBins b;
  SP_TRY(bin_triangles(g, scr, lst, b, s));
  unsigned long long* fbk = (unsigned long long*)g->keys;  // n <= key_cap scratch keys
  SP_CUDA(cudaMemsetAsync(g->nkeys + 2, 0, sizeof(unsigned long long), s));
  k_fb_collect<<<cdiv(n, 256), 256, 0, s>>>(g->assign, n, fbk, g->nkeys + 2);
  SP_CHECK_LAUNCH();
  SP_CUDA(cudaMemcpyAsync(g->h_small, g->nkeys + 2, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long nfb = (long)((unsigned long long*)g->h_small)[0];
  Scratch fbs(s);
  size_t sort_bytes = 0;
  if (nfb > 0)
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int)nfb, 0,
                                   32 + bits_for(T), s);
  SP_TRY(fbs.alloc(sizeof(unsigned long long) * (nfb + 1) + sizeof(int) * 2 * (size_t)T +
                   sort_bytes + 512));
  unsigned long long* fsorted = (unsigned long long*)fbs.p;
  int* fs = (int*)(fsorted + nfb + 1);
  int* fe = fs + T;
  void* sort_tmp = (void*)(((uintptr_t)(fe + T) + 255) & ~(uintptr_t)255);
  SP_CUDA(cudaMemsetAsync(fs, 0, sizeof(int) * 2 * (size_t)T, s));
  if (nfb > 0) {
    SP_CUDA(cub::DeviceRadixSort::SortKeys(sort_tmp, sort_bytes, fbk, fsorted, (int)nfb, 0,
                                           32 + bits_for(T), s));
    k_fb_bounds<<<cdiv(nfb, 256), 256, 0, s>>>(fsorted, nfb, fs, fe);
    SP_CHECK_LAUNCH();
  }
  const long nt = t1 - t0;
  if ((double)T * 128.0 >= (double)n) {
    k_reduce_tris_small<<<cdiv(nt, 128), 128, 0, s>>>(b.tbox, t1, g->assign, err, W, fsorted,
                                                      fs, fe, g->sums, g->amax, g->amax_val,
                                                      t0);
  } else {
    const long rblocks = std::min<long>(cdiv(nt, 8), (long)num_sms() * 4);
    SP_CUDA(cudaMemsetAsync(g->nkeys + 3, 0, sizeof(unsigned long long), s));
    k_reduce_tris<<<rblocks, 256, 0, s>>>(b.tv, b.tc, b.tbox, t1, g->assign, err, W, fsorted,
                                          fs, fe, g->sums, g->amax, g->amax_val,
                                          (unsigned*)(g->nkeys + 3), t0);
  }
  SP_CHECK_LAUNCH();
  return 0;
}

static int accumulate_mode = 1;  // 1: tiled (default), 0: global atomics + pixel sort
int geo_accumulate_mode(int v) {
  if (v >= 0) accumulate_mode = v;
  return accumulate_mode;
}

// geometry.py:197-223 (partition="delaunay") or :226-244 ("voronoi")
int geo_accumulate(Geo* g, const double* err, int voronoi, cudaStream_t s) {
  const int H = g->H, W = g->W;
  size_t n = (size_t)H * W;
  if (voronoi) {
    return reduce_cells(g->lab_a, err, g->m, g->sums, g->amax, g->amax_val, H, W, s);
  }
  if (g->T == 0) return 0;
  if (accumulate_mode == 1 && H < 32768 && W < 32768 && n < (1ull << 32) &&
      n <= g->key_cap)
    return accumulate_tiled(g, err, s);
  SP_TRY(assign_tris<int>(g->tris, g->T, g->sy, g->sx, H, W, g->assign, false, s));
  SP_TRY(seed_min_tri<int>(g->tris, g->T, g->smt, g->m, s));
  SP_TRY(fallback(g->assign, g->lab_a, g->smt, g->assign, n, s));
  return reduce_cells(g->assign, err, g->T, g->sums, g->amax, g->amax_val, H, W, s);
}

// Ordered selection of the `want` first entries of sort((-value, index))
// among flagged indices; `apply(order, k)` consumes the sorted index list.
// Order-preserving compaction (cub select) + one stable radix sort on the
// complemented key == np.lexsort((index, -value)).
template <typename Apply>
static int top_by_desc(const uint8_t* flags, const double* vals, long n, long want,
                       int* nsel, long* taken, cudaStream_t s, Apply apply,
                       bool descending = true) {
  *taken = 0;
  if (want <= 0 || n <= 0) return 0;
  cub::CountingInputIterator<int> it(0);
  size_t sel_bytes = 0, sort_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, sel_bytes, it, flags, (int*)nullptr, nsel, (int)n, s);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, (int)n, 0, 64, s);
  size_t nn = (size_t)n;
  Scratch scr(s);
  SP_TRY(scr.alloc(2 * sizeof(unsigned long long) * nn + 2 * sizeof(int) * nn +
                   std::max(sel_bytes, sort_bytes) + 512));
  unsigned long long* k_in = (unsigned long long*)scr.p;
  unsigned long long* k_out = k_in + nn;
  int* v_in = (int*)(k_out + nn);
  int* v_out = v_in + nn;
  void* tmp = (void*)(v_out + nn + 16);
  SP_CUDA(cub::DeviceSelect::Flagged(tmp, sel_bytes, it, flags, v_in, nsel, (int)n, s));
  int nv_h = 0;
  SP_CUDA(cudaMemcpyAsync(&nv_h, nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  long nv = nv_h;
  if (nv == 0) return 0;
  k_desc_keys<<<cdiv(nv, 256), 256, 0, s>>>(v_in, nv, vals, k_in, descending ? 1 : 0);
  SP_CHECK_LAUNCH();
  SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, k_in, k_out, v_in, v_out, (int)nv,
                                          0, 64, s));
  long k = std::min(nv, want);
  SP_TRY(apply(v_out, k));
  *taken = k;
  return 0;
}

// spatial.py:245-259: picks the argmax pixel of the `want` highest-error
// buckets whose argmax is not stored yet; updates mask in place.
int geo_select(Geo* g, uint8_t* mask, long nbuckets, long want, long* picked,
               cudaStream_t s) {
  *picked = 0;
  if (want <= 0 || nbuckets <= 0) return 0;
  k_valid_flags<<<cdiv(nbuckets, 256), 256, 0, s>>>(g->amax, mask, nbuckets, g->flags);
  SP_CHECK_LAUNCH();
  return top_by_desc(g->flags, g->sums, nbuckets, want, g->nsel, picked, s,
                     [&](const int* order, long k) {
                       k_apply_picks<<<cdiv(k, 256), 256, 0, s>>>(order, k, g->amax, mask);
                       SP_CHECK_LAUNCH();
                       return 0;
                     });
}

// spatial.py:189-197: store the `want` highest-error free pixels
int fill_highest_error(Geo* g, const double* err, uint8_t* mask, long want, cudaStream_t s) {
  size_t n = (size_t)g->H * g->W;
  k_not_mask<<<cdiv(n, 256), 256, 0, s>>>(mask, n, g->flags);
  SP_CHECK_LAUNCH();
  long taken = 0;
  return top_by_desc(g->flags, err, (long)n, want, g->nsel, &taken, s,
                     [&](const int* order, long k) {
                       k_set_mask<<<cdiv(k, 256), 256, 0, s>>>(order, k, mask);
                       SP_CHECK_LAUNCH();
                       return 0;
                     });
}

// spatial.py:90-104 (_exact_count): among the flagged pixels (flags == NULL:
// the pixels with mask_set == 0) take the `want` first of the order
// (value descending or ascending, index ascending) and set them to
// `set_value` in mask_set
int top_select(const uint8_t* flags, const double* vals, long n, long want, bool descending,
               int* nsel, cudaStream_t s, uint8_t* mask_set, uint8_t set_value) {
  Scratch fl(s);
  if (!flags) {
    SP_TRY(fl.alloc((size_t)n));
    k_not_mask<<<cdiv(n, 256), 256, 0, s>>>(mask_set, (size_t)n, (uint8_t*)fl.p);
    SP_CHECK_LAUNCH();
    flags = (const uint8_t*)fl.p;
  }
  long taken = 0;
  return top_by_desc(flags, vals, n, want, nsel, &taken, s,
                     [&](const int* order, long k) {
                       k_set_mask_val<<<cdiv(k, 256), 256, 0, s>>>(order, k, mask_set,
                                                                   set_value);
                       SP_CHECK_LAUNCH();
                       return 0;
                     },
                     descending);
}

}  // namespace sp
