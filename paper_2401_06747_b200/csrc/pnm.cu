// pnm.cu -- the on-disk formats of masks and stored values, encoded where
// the data lives (reference pnm.py:40-127).
//
//   P4 mask body      np.packbits(indicator, axis=1): per row ceil(W/8)
//                     bytes, most significant bit first, tail bits zero
//                     (pnm.py:78-84).  One thread per output byte; the eight
//                     mask bytes it needs are one 8-byte load when aligned.
//   P4 unpack         the inverse (pnm.py:87-95), so a mask file is uploaded
//                     as its packed body (8x fewer bytes than u8)
//   8-bit body        clamp_to_bytes: clip(rint(v), 0, 255) -> u8, planar
//                     [C,H,W] -> interleaved [H,W,C] (grid.py:216-218,
//                     pnm.py:42-55); optionally where(mask, v, 0) first
//                     (write_tonal, pnm.py:98-105)
//   16-bit sidecar    clip(rint((v + 256) * 64), 0, 65535) as big-endian u16,
//                     interleaved (pnm.py:106-117).  The arithmetic runs in
//                     the value dtype, as numpy does for a float32 array and
//                     Python float scalars (weak scalars, NEP 50); no FMA.
#include "common.cuh"

namespace sp {

namespace {

__global__ void k_pack_bits(const uint8_t* __restrict__ m, int H, int W, uint8_t* __restrict__ out) {
  const int rb = (W + 7) >> 3;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)H * rb) return;
  const int y = (int)(i / rb), bx = (int)(i - (size_t)y * rb);
  const uint8_t* row = m + (size_t)y * W;
  const int x0 = bx * 8;
  unsigned v = 0;
  if (x0 + 8 <= W && ((((uintptr_t)(row + x0)) & 7) == 0)) {
    const unsigned long long q = *(const unsigned long long*)(row + x0);
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((q >> (8 * k)) & 0xFFull) != 0 ? 1u : 0u) << (7 - k);
  } else {
    for (int k = 0; k < 8 && x0 + k < W; ++k) v |= (row[x0 + k] != 0 ? 1u : 0u) << (7 - k);
  }
  out[i] = (uint8_t)v;
}

__global__ void k_unpack_bits(const uint8_t* __restrict__ bits, int H, int W, uint8_t* __restrict__ m) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)H * W) return;
  const int rb = (W + 7) >> 3;
  const int y = (int)(i / W), x = (int)(i - (size_t)y * W);
  m[i] = (bits[(size_t)y * rb + (x >> 3)] >> (7 - (x & 7))) & 1u;
}

template <typename T>
__device__ __forceinline__ T vclip(T v, T lo, T hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// one thread per pixel, all C channels -> C contiguous output bytes
template <typename T>
__global__ void k_bytes_hwc(const T* __restrict__ v, const uint8_t* __restrict__ m, int C,
                            size_t n, uint8_t* __restrict__ out) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const bool on = m == nullptr || m[p] != 0;
  for (int c = 0; c < C; ++c) {
    const T x = on ? v[(size_t)c * n + p] : (T)0;
    // NaN never reaches here (images are validated finite, grid.py:57-60)
    out[p * C + c] = (uint8_t)vclip<T>(rint(x), (T)0, (T)255);
  }
}

template <typename T>
__global__ void k_tonal16_hwc(const T* __restrict__ v, const uint8_t* __restrict__ m, int C,
                              size_t n, uint8_t* __restrict__ out) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const bool on = m == nullptr || m[p] != 0;
  for (int c = 0; c < C; ++c) {
    const T x = on ? v[(size_t)c * n + p] : (T)0;
    T e = (x + (T)256) * (T)64;
    e = vclip<T>(rint(e), (T)0, (T)65535);
    const unsigned u = (unsigned)e;
    out[2 * (p * C + c)] = (uint8_t)(u >> 8);
    out[2 * (p * C + c) + 1] = (uint8_t)(u & 0xFFu);
  }
}

}  // namespace

int pack_bits(const uint8_t* m, int H, int W, uint8_t* out, cudaStream_t s) {
  const size_t n = (size_t)H * ((W + 7) >> 3);
  if (!n) return 0;
  k_pack_bits<<<cdiv(n, 256), 256, 0, s>>>(m, H, W, out);
  SP_CHECK_LAUNCH();
  return 0;
}

int unpack_bits(const uint8_t* bits, int H, int W, uint8_t* m, cudaStream_t s) {
  const size_t n = (size_t)H * W;
  if (!n) return 0;
  k_unpack_bits<<<cdiv(n, 256), 256, 0, s>>>(bits, H, W, m);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int encode_pnm(const T* v, const uint8_t* m, int C, int H, int W, int wide, uint8_t* out,
               cudaStream_t s) {
  const size_t n = (size_t)H * W;
  if (!n) return 0;
  if (wide) k_tonal16_hwc<T><<<cdiv(n, 256), 256, 0, s>>>(v, m, C, n, out);
  else k_bytes_hwc<T><<<cdiv(n, 256), 256, 0, s>>>(v, m, C, n, out);
  SP_CHECK_LAUNCH();
  return 0;
}

template int encode_pnm<float>(const float*, const uint8_t*, int, int, int, int, uint8_t*,
                               cudaStream_t);
template int encode_pnm<double>(const double*, const uint8_t*, int, int, int, int, uint8_t*,
                                cudaStream_t);

}  // namespace sp

extern "C" {

int sp_pack_mask_bits(const uint8_t* mask, int H, int W, uint8_t* out, void* s) {
  return sp::pack_bits(mask, H, W, out, (cudaStream_t)s);
}

int sp_unpack_mask_bits(const uint8_t* bits, int H, int W, uint8_t* mask, void* s) {
  return sp::unpack_bits(bits, H, W, mask, (cudaStream_t)s);
}

int sp_encode_pnm(int dtype, const void* values, const uint8_t* mask, int C, int H, int W,
                  int wide, uint8_t* out, void* s) {
  if (dtype == sp::SP_F32)
    return sp::encode_pnm<float>((const float*)values, mask, C, H, W, wide, out,
                                 (cudaStream_t)s);
  if (dtype == sp::SP_F64)
    return sp::encode_pnm<double>((const double*)values, mask, C, H, W, wide, out,
                                  (cudaStream_t)s);
  sp::set_error("unsupported dtype code %d", dtype);
  return -2;
}

}  // extern "C"
