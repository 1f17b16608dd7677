// dither.cu -- the dithered initial mask of delaunay_densify on the device
// (spatial.py:107-148 analytic_mask(dither="random") + _exact_count :90-104),
// bit-exact against the reference:
//   1. scipy.ndimage.gaussian_filter(sigma, mode="reflect") per channel:
//      separable correlate1d along axis 0 then axis 1, symmetric branch
//      out = x0*w0; for jj = -r..-1: out += (x[jj] + x[-jj]) * w[jj]
//      (scipy ni_filters.c), reflect = "dcba|abcd|dcba"; weights come from
//      the host exactly as scipy's _gaussian_kernel1d computes them;
//   2. negated Laplacian in double (numba_impl.py:13-36);
//   3. mag = |L0| + |L1| + ... in channel order (numpy sum over axis 0);
//   4. total = numpy pairwise sum of mag (blocks of <= 128 with 8
//      accumulators, split at n/2 rounded down to a multiple of 8): the
//      leaves are summed on the device, the (tiny) tree is combined on the
//      host in the same recursion order;
//   5. dens = clip(mag * scale, 0, 1) with scale = (density * n) / total;
//   6. bits = u_i < dens_i, u_i the i-th numpy PCG64 double: PCG64 XSL-RR
//      128-bit LCG (numpy pcg64.h), (next64 >> 11) * 2^-53, each thread
//      jumping ahead to its chunk with the O(log n) LCG advance;
//   7. exact count: drop the lowest-(dens, index) set pixels or add the
//      highest-dens / lowest-index unset pixels (stable radix sort).
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "geometry.cuh"

namespace sp {

namespace {

struct u128 {
  unsigned long long lo, hi;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  unsigned __int128 x = ((unsigned __int128)a.hi << 64) | a.lo;
  unsigned __int128 y = ((unsigned __int128)b.hi << 64) | b.lo;
  unsigned __int128 z = x * y;
  r.lo = (unsigned long long)z;
  r.hi = (unsigned long long)(z >> 64);
#endif
  return r;
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

// PCG_DEFAULT_MULTIPLIER_128 (numpy/random/src/pcg64/pcg64.h)
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return {0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__host__ __device__ inline u128 pcg_advance(u128 state, unsigned long long delta, u128 inc) {
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  u128 acc_mult = {1ull, 0ull}, acc_plus = {0ull, 0ull};
  while (delta > 0) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, {1ull, 0ull}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}

// XSL-RR output of the (already advanced) state
__host__ __device__ __forceinline__ unsigned long long pcg_output(u128 s) {
  unsigned rot = (unsigned)(s.hi >> 58);
  unsigned long long x = s.hi ^ s.lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int CHUNK = 64;

// bits[i] = (pcg double i) < dens[i]; each thread owns CHUNK consecutive i
__global__ void k_coin(const double* __restrict__ dens, uint8_t* __restrict__ bits, size_t n,
                       unsigned long long s_lo, unsigned long long s_hi,
                       unsigned long long inc_lo, unsigned long long inc_hi,
                       unsigned long long* __restrict__ count) {
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t i0 = t * CHUNK;
  unsigned c = 0;
  if (i0 < n) {
    u128 inc = {inc_lo, inc_hi};
    u128 s = pcg_advance({s_lo, s_hi}, (unsigned long long)i0, inc);
    const u128 mult = pcg_mult();
    size_t i1 = i0 + CHUNK < n ? i0 + CHUNK : n;
    for (size_t i = i0; i < i1; ++i) {
      s = add128(mul128(s, mult), inc);  // step, then output (numpy next64)
      double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
      uint8_t b = u < dens[i];
      bits[i] = b;
      c += b;
    }
  }
  // warp-aggregated count
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// separable symmetric correlation with reflect boundary along rows (axis 1)
// or columns (axis 0); one thread per output pixel
__device__ __forceinline__ int reflect_idx(int i, int n) {
  // scipy "reflect": d c b a | a b c d | d c b a
  if (n == 1) return 0;
  const int period = 2 * n;
  i %= period;
  if (i < 0) i += period;
  return i < n ? i : period - 1 - i;
}

__global__ void k_gauss_axis(const double* __restrict__ in, double* __restrict__ out, int C,
                             int H, int W, int axis, const double* __restrict__ wts, int radius) {
  const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
  const int c = blockIdx.z;
  if (x >= W || y >= H) return;
  const double* src = in + (size_t)c * H * W;
  const double* fw = wts + radius;  // centre
  double acc;
  if (axis == 0) {
    acc = src[(size_t)y * W + x] * fw[0];
    for (int jj = -radius; jj < 0; ++jj)
      acc += (src[(size_t)reflect_idx(y + jj, H) * W + x] +
              src[(size_t)reflect_idx(y - jj, H) * W + x]) * fw[jj];
  } else {
    const double* row = src + (size_t)y * W;
    acc = row[x] * fw[0];
    for (int jj = -radius; jj < 0; ++jj)
      acc += (row[reflect_idx(x + jj, W)] + row[reflect_idx(x - jj, W)]) * fw[jj];
  }
  out[(size_t)c * H * W + (size_t)y * W + x] = acc;
}

// mag = sum_c |L_c| (channel order, numpy sum over axis 0)
__global__ void k_abs_chan_sum(const double* __restrict__ lap, double* __restrict__ mag, int C,
                               size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = fabs(lap[i]);
  for (int c = 1; c < C; ++c) s = s + fabs(lap[(size_t)c * n + i]);
  mag[i] = s;
}

// numpy pairwise leaf (n <= 128): 8 accumulators, then the remainder
__global__ void k_pairwise_leaves(const double* __restrict__ a, const long long* __restrict__ off,
                                  const int* __restrict__ len, int nleaves,
                                  double* __restrict__ out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const double* p = a + off[t];
  const int n = len[t];
  double res;
  if (n < 8) {
    res = 0.0;
    for (int i = 0; i < n; ++i) res += p[i];
  } else {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = p[k];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += p[i + k];
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += p[i];
  }
  out[t] = res;
}

__global__ void k_clip_scale(double* __restrict__ mag, size_t n, double scale) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = mag[i] * scale;
  mag[i] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

// host recursion of numpy's pairwise_sum: leaves in order
void pairwise_plan(long long lo, long long n, std::vector<long long>& off,
                   std::vector<int>& len) {
  if (n <= 128) {
    off.push_back(lo);
    len.push_back((int)n);
    return;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  pairwise_plan(lo, n2, off, len);
  pairwise_plan(lo + n2, n - n2, off, len);
}

double pairwise_combine(long long n, const double* leaves, size_t& k) {
  if (n <= 128) return leaves[k++];
  long long n2 = n / 2;
  n2 -= n2 % 8;
  double a = pairwise_combine(n2, leaves, k);
  double b = pairwise_combine(n - n2, leaves, k);
  return a + b;
}

}  // namespace

int top_select(const uint8_t* flags, const double* vals, long n, long want, bool descending,
               int* nsel, cudaStream_t s, uint8_t* mask_set, uint8_t set_value);

// numpy pairwise sum of a device array (double)
int pairwise_sum(const double* a, long long n, double* out, cudaStream_t s) {
  std::vector<long long> off;
  std::vector<int> len;
  pairwise_plan(0, n, off, len);
  int nl = (int)off.size();
  Scratch scr(s);
  SP_TRY(scr.alloc((sizeof(long long) + sizeof(int) + sizeof(double)) * (size_t)nl + 64));
  long long* d_off = (long long*)scr.p;
  double* d_out = (double*)(d_off + nl);
  int* d_len = (int*)(d_out + nl);
  SP_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, s));
  SP_CUDA(cudaMemcpyAsync(d_len, len.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, s));
  k_pairwise_leaves<<<cdiv(nl, 256), 256, 0, s>>>(a, d_off, d_len, nl, d_out);
  SP_CHECK_LAUNCH();
  std::vector<double> leaves(nl);
  SP_CUDA(cudaMemcpyAsync(leaves.data(), d_out, sizeof(double) * nl, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  size_t k = 0;
  *out = pairwise_combine(n, leaves.data(), k);
  return 0;
}

// spatial.py:107-120 laplacian_density_map: dens (device, H*W) and the
// pairwise total; *total_out == 0 means the Laplacian vanishes (constant
// image) and dens is left unscaled
int density_map(const double* f, int C, int H, int W, double density, const double* gauss_h,
                int radius, double* dens, double* total_out, cudaStream_t s) {
  const size_t n = (size_t)H * W, cn = (size_t)C * n;
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(double) * (2 * cn + 2 * (size_t)radius + 8)));
  double* a = (double*)scr.p;
  double* b = a + cn;
  double* wts = b + cn;
  const double* src = f;
  dim3 g(cdiv(W, 32), cdiv(H, 8), C);
  if (radius > 0) {
    SP_CUDA(cudaMemcpyAsync(wts, gauss_h, sizeof(double) * (2 * radius + 1),
                            cudaMemcpyHostToDevice, s));
    k_gauss_axis<<<g, dim3(32, 8), 0, s>>>(f, a, C, H, W, 0, wts, radius);
    SP_CHECK_LAUNCH();
    k_gauss_axis<<<g, dim3(32, 8), 0, s>>>(a, b, C, H, W, 1, wts, radius);
    SP_CHECK_LAUNCH();
    src = b;
  }
  SP_TRY(neglap<double>(src, a, C, H, W, 1.0, s));
  k_abs_chan_sum<<<cdiv(n, 256), 256, 0, s>>>(a, dens, C, n);
  SP_CHECK_LAUNCH();
  double total = 0.0;
  SP_TRY(pairwise_sum(dens, (long long)n, &total, s));
  *total_out = total;
  if (total == 0.0) return 0;
  // spatial.py:120: mag * (density * n / total), clipped to [0, 1]
  const double scale = density * (double)n / total;
  k_clip_scale<<<cdiv(n, 256), 256, 0, s>>>(dens, n, scale);
  SP_CHECK_LAUNCH();
  return 0;
}

// spatial.py:123-148 with dither="random"; `density` is target / n.
// *degenerate = 1 when the Laplacian vanishes (the caller falls back to the
// uniform random mask, spatial.py:136-140), else `mask` is written.
int init_mask_random(const double* f, int C, int H, int W, long target, double density,
                     const double* gauss_h, int radius, const uint64_t* pcg_h, uint8_t* mask,
                     int* degenerate, cudaStream_t s) {
  const size_t n = (size_t)H * W;
  *degenerate = 0;
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(double) * n + 64));
  double* dens = (double*)scr.p;
  unsigned long long* dcount = (unsigned long long*)(dens + n);
  int* nsel = (int*)(dcount + 1);
  double total = 0.0;
  SP_TRY(density_map(f, C, H, W, density, gauss_h, radius, dens, &total, s));
  if (total == 0.0) {
    *degenerate = 1;
    return 0;
  }
  SP_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), s));
  size_t nthreads = (n + CHUNK - 1) / CHUNK;
  k_coin<<<cdiv(nthreads, 256), 256, 0, s>>>(dens, mask, n, pcg_h[0], pcg_h[1], pcg_h[2],
                                             pcg_h[3], dcount);
  SP_CHECK_LAUNCH();
  unsigned long long cnt_h = 0;
  SP_CUDA(cudaMemcpyAsync(&cnt_h, dcount, sizeof(cnt_h), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const long cnt = (long)cnt_h;
  // spatial.py:90-104 _exact_count
  if (cnt > target)  // drop the (cnt - target) set pixels of lowest (dens, index)
    SP_TRY(top_select(mask, dens, (long)n, cnt - target, false, nsel, s, mask, 0));
  else if (cnt < target)  // add the unset pixels of highest dens, lowest index
    SP_TRY(top_select(nullptr, dens, (long)n, target - cnt, true, nsel, s, mask, 1));
  return 0;
}

namespace {
__global__ void k_pcg_doubles(unsigned long long s_lo, unsigned long long s_hi,
                              unsigned long long inc_lo, unsigned long long inc_hi,
                              long long start, long long count, double* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  u128 inc = {inc_lo, inc_hi};
  u128 st = pcg_advance({s_lo, s_hi}, (unsigned long long)(start + i + 1), inc);
  out[i] = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
}
}  // namespace

// doubles start .. start+count-1 of numpy's PCG64 Generator.random stream
int pcg_doubles(const uint64_t* pcg_h, long long start, long long count, double* out,
                cudaStream_t s) {
  if (count <= 0) return 0;
  k_pcg_doubles<<<cdiv(count, 256), 256, 0, s>>>(pcg_h[0], pcg_h[1], pcg_h[2], pcg_h[3], start,
                                                 count, out);
  SP_CHECK_LAUNCH();
  return 0;
}

}  // namespace sp
