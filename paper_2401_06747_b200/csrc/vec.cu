// vec.cu -- deterministic vector reductions and elementwise helpers.
//
// Reductions never use floating atomics: a fixed number of CTAs (a function
// of the length only) each reduce a fixed strided subset, then the last CTA
// to finish sums the partials in index order.  Results are therefore
// bit-identical run to run.  Used for the ||b~|| scale of solve_sym
// (solver.py:355-358), the per-channel dots of the tonal CG loops
// (tonal.py:91-97) and the MSE (tonal.py:86-88, grid.py:188-193).
#include "solver.cuh"

namespace sp {

namespace {
constexpr int NT = 256;
constexpr int MAXB = 1024;

inline int nblocks_for(size_t n) {
  size_t b = (n + NT * 8 - 1) / (NT * 8);
  if (b < 1) b = 1;
  if (b > MAXB) b = MAXB;
  return (int)b;
}

// mode 0: sum x^2; mode 1: sum x*y; mode 2: sum (x - z)^2 with z double;
// mode 3: sum (x - y)^2 with y of x's type (both widened exactly to double)
template <typename T, int MODE>
__global__ void __launch_bounds__(NT) k_reduce(const T* __restrict__ x,
                                               const T* __restrict__ y,
                                               const double* __restrict__ z, size_t n,
                                               int C, double* __restrict__ partial,
                                               unsigned* __restrict__ counter,
                                               double* __restrict__ out) {
  __shared__ double s0[NT / 32], s1[NT / 32];
  __shared__ bool am_last;
  const size_t stride = (size_t)gridDim.x * NT;
  for (int c = 0; c < C; ++c) {
    const size_t off = (size_t)c * n;
    double acc = 0.0;
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < n; i += stride) {
      double a = (double)x[off + i];
      if (MODE == 0) acc += a * a;
      else if (MODE == 1) acc += a * (double)y[off + i];
      else if (MODE == 3) { double d = a - (double)y[off + i]; acc += d * d; }
      else { double d = a - z[off + i]; acc += d * d; }
    }
    double s = cta_sum<NT>(acc, (c & 1) ? s1 : s0);
    if (threadIdx.x == 0) partial[(size_t)blockIdx.x * C + c] = s;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += NT)
      s += ((volatile double*)partial)[(size_t)i * C + c];
    s = cta_sum<NT>(s, (c & 1) ? s1 : s0);
    if (threadIdx.x == 0) out[c] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}
// many short segments (the batched RAS tiles: thousands of (tile) planes of
// a few thousand elements): one CTA per segment, fixed per-thread strides and
// a fixed-order CTA sum, so results are still run-to-run bit-identical
template <typename T, int MODE>
__global__ void __launch_bounds__(NT) k_reduce_seg(const T* __restrict__ x,
                                                   const T* __restrict__ y,
                                                   const double* __restrict__ z, size_t n,
                                                   double* __restrict__ out) {
  __shared__ double s0[NT / 32];
  const size_t off = (size_t)blockIdx.x * n;
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < n; i += NT) {
    double a = (double)x[off + i];
    if (MODE == 0) acc += a * a;
    else if (MODE == 1) acc += a * (double)y[off + i];
    else if (MODE == 3) { double d = a - (double)y[off + i]; acc += d * d; }
    else { double d = a - z[off + i]; acc += d * d; }
  }
  double s = cta_sum<NT>(acc, s0);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}
}  // namespace

size_t red_partials() { return MAXB; }

template <typename T>
int dot_self(const T* x, size_t n, double* partial, unsigned* counter, double* out,
             cudaStream_t s) {
  k_reduce<T, 0><<<nblocks_for(n), NT, 0, s>>>(x, nullptr, nullptr, n, 1, partial, counter,
                                               out);
  SP_CHECK_LAUNCH();
  return 0;
}

// per-channel sums over C planes of n elements each
template <typename T>
int chan_reduce(int mode, const T* x, const T* y, const double* z, size_t n, int C,
                double* partial, unsigned* counter, double* out, cudaStream_t s) {
  int nb = nblocks_for(n);
  if (C >= 2 * num_sms() && n <= (size_t)NT * 64) {
    if (mode == 0) k_reduce_seg<T, 0><<<C, NT, 0, s>>>(x, y, z, n, out);
    else if (mode == 1) k_reduce_seg<T, 1><<<C, NT, 0, s>>>(x, y, z, n, out);
    else if (mode == 3) k_reduce_seg<T, 3><<<C, NT, 0, s>>>(x, y, z, n, out);
    else k_reduce_seg<T, 2><<<C, NT, 0, s>>>(x, y, z, n, out);
    SP_CHECK_LAUNCH();
    return 0;
  }
  if (mode == 0) k_reduce<T, 0><<<nb, NT, 0, s>>>(x, y, z, n, C, partial, counter, out);
  else if (mode == 1) k_reduce<T, 1><<<nb, NT, 0, s>>>(x, y, z, n, C, partial, counter, out);
  else if (mode == 3) k_reduce<T, 3><<<nb, NT, 0, s>>>(x, y, z, n, C, partial, counter, out);
  else k_reduce<T, 2><<<nb, NT, 0, s>>>(x, y, z, n, C, partial, counter, out);
  SP_CHECK_LAUNCH();
  return 0;
}

// e = sum_c (u_c - f_c)^2 in double, channel order (spatial.py:184-186)
template <typename T>
__global__ void k_error_map(const T* __restrict__ u, const double* __restrict__ f,
                            double* __restrict__ e, int C, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int c = 0; c < C; ++c) {
    double d = (double)u[(size_t)c * n + i] - f[(size_t)c * n + i];
    double sq = d * d;
    acc = c == 0 ? sq : acc + sq;
  }
  e[i] = acc;
}

// the same error map plus one partial sum per CTA (the MSE numerator,
// grid.py:188-193): one pixel per thread like k_error_map, a fixed-order
// CTA sum; k_sum_partials adds the CTA partials in index order (no atomics:
// a last-CTA reduction serialised ~1,000 same-address atomics at the end of
// a grid whose CTAs all finish together)
template <typename T>
__global__ void __launch_bounds__(256) k_error_map_part(const T* __restrict__ u,
                                                       const double* __restrict__ f,
                                                       double* __restrict__ e, int C, size_t n,
                                                       double* __restrict__ partial) {
  __shared__ double s0[256 / 32];
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (i < n) {
    for (int c = 0; c < C; ++c) {
      double d = (double)u[(size_t)c * n + i] - f[(size_t)c * n + i];
      double sq = d * d;
      acc = c == 0 ? sq : acc + sq;
    }
    e[i] = acc;
  }
  const double sb = cta_sum<256>(acc, s0);
  if (threadIdx.x == 0) partial[blockIdx.x] = sb;
}

__global__ void __launch_bounds__(1024) k_sum_partials(const double* __restrict__ partial,
                                                       int n, double* __restrict__ total) {
  __shared__ double s0[1024 / 32];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) t += partial[i];
  t = cta_sum<1024>(t, s0);
  if (threadIdx.x == 0) *total = t;
}

template <typename T>
int error_map(const T* u, const double* f, double* e, int C, size_t n, cudaStream_t s,
              double* total) {
  if (!total) {
    k_error_map<T><<<cdiv(n, 256), 256, 0, s>>>(u, f, e, C, n);
    SP_CHECK_LAUNCH();
    return 0;
  }
  const unsigned nb = cdiv(n, 256);
  Scratch scr(s);
  SP_TRY(scr.alloc(sizeof(double) * nb + 64));
  k_error_map_part<T><<<nb, 256, 0, s>>>(u, f, e, C, n, (double*)scr.p);
  SP_CHECK_LAUNCH();
  k_sum_partials<<<1, 1024, 0, s>>>((const double*)scr.p, (int)nb, total);
  SP_CHECK_LAUNCH();
  return 0;
}
template int error_map<float>(const float*, const double*, double*, int, size_t, cudaStream_t,
                              double*);
template int error_map<double>(const double*, const double*, double*, int, size_t, cudaStream_t,
                               double*);

template int dot_self<float>(const float*, size_t, double*, unsigned*, double*, cudaStream_t);
template int dot_self<double>(const double*, size_t, double*, unsigned*, double*, cudaStream_t);
template int chan_reduce<float>(int, const float*, const float*, const double*, size_t, int,
                                double*, unsigned*, double*, cudaStream_t);
template int chan_reduce<double>(int, const double*, const double*, const double*, size_t,
                                 int, double*, unsigned*, double*, cudaStream_t);

}  // namespace sp
