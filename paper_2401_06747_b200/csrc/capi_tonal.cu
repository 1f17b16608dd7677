// capi_tonal.cu -- C-ABI of the tonal-optimizer kernels (csrc/tonal.cu).
// Declared in include/sparsepaint_b200.h; same conventions as capi.cu.
#include "geometry.cuh"
#include "../../include/sparsepaint_b200.h"

namespace sp {
int cell_index(const int* lab, int H, int W, long m, int* perm, int* start, int* end,
               cudaStream_t s);
int vi_weights(const int* lab, const int* sy, const int* sx, const int* perm, const int* start,
               const int* end, int H, int W, long m, int scheme, double* w, cudaStream_t s);
int cell_sum(const int* perm, const int* start, const int* end, const double* v, long m,
             double* out, cudaStream_t s);
template <typename T>
int vi_step(const int* perm, const int* start, const int* end, const double* w, const T* f,
            const T* u, const int* sy, const int* sx, long m, int C, int H, int W, double tau,
            T* g, cudaStream_t s);
template <typename T>
int plane_dot(const T* x, const T* y, size_t len, long nplanes, int C, const int* active,
              double* out, cudaStream_t s);
template <typename T>
int plane_axpy(T* yout, const T* x, const T* z, const double* coef, double sign, size_t len,
               long nplanes, int C, const int* active, cudaStream_t s);
template <typename T>
int gather_tiles(const T* img, const int* oy, const int* ox, int ntile, int C, int H, int W,
                 int bh, int bw, T* out, cudaStream_t s);
int gather_mask_tiles(const uint8_t* m, const int* oy, const int* ox, int ntile, int H, int W,
                      int bh, int bw, uint8_t* out, cudaStream_t s);
template <typename T>
int ras_scatter(T* g, const T* v, const int* tile_of, const int* ys, const int* xs,
                const int* row_k0, const int* row_n, const int* col_k0, const int* col_n,
                int nbx, int bh, int bw, int C, int H, int W, cudaStream_t s);
template <typename T>
int where_mask(const T* x, const uint8_t* m, T* out, int C, int H, int W, cudaStream_t s);
template <typename T>
int neighbor_balance(const double* f, const T* u, const uint8_t* m, T* g, int C, int H, int W,
                     cudaStream_t s);
}  // namespace sp

using namespace sp;
#define STREAM(s) ((cudaStream_t)(s))
#define DISPATCH(dtype, CALL_F32, CALL_F64)                                   \
  do {                                                                        \
    if ((dtype) == SP_F32) return CALL_F32;                                   \
    if ((dtype) == SP_F64) return CALL_F64;                                   \
    set_error("unsupported dtype code %d", (int)(dtype));                     \
    return -2;                                                                \
  } while (0)

extern "C" {

int sp_cell_index(const int32_t* labels, int H, int W, long m, int32_t* perm, int32_t* start,
                  int32_t* end, void* s) {
  return cell_index(labels, H, W, m, perm, start, end, STREAM(s));
}

int sp_vi_weights(const int32_t* labels, const int32_t* sy, const int32_t* sx,
                  const int32_t* perm, const int32_t* start, const int32_t* end, int H, int W,
                  long m, int scheme, double* w, void* s) {
  return vi_weights(labels, sy, sx, perm, start, end, H, W, m, scheme, w, STREAM(s));
}

int sp_cell_sum(const int32_t* perm, const int32_t* start, const int32_t* end, const double* v,
                long m, double* out, void* s) {
  return cell_sum(perm, start, end, v, m, out, STREAM(s));
}

int sp_vi_step(int dtype, const int32_t* perm, const int32_t* start, const int32_t* end,
               const double* w, const void* f, const void* u, const int32_t* sy,
               const int32_t* sx, long m, int C, int H, int W, double tau, void* g, void* s) {
  DISPATCH(dtype,
           vi_step<float>(perm, start, end, w, (const float*)f, (const float*)u, sy, sx, m, C, H,
                          W, tau, (float*)g, STREAM(s)),
           vi_step<double>(perm, start, end, w, (const double*)f, (const double*)u, sy, sx, m, C,
                           H, W, tau, (double*)g, STREAM(s)));
}

int sp_plane_dot(int dtype, const void* x, const void* y, long len, long nplanes, int C,
                 const int32_t* active, double* out, void* s) {
  DISPATCH(dtype,
           plane_dot<float>((const float*)x, (const float*)y, (size_t)len, nplanes, C, active,
                            out, STREAM(s)),
           plane_dot<double>((const double*)x, (const double*)y, (size_t)len, nplanes, C,
                             active, out, STREAM(s)));
}

int sp_plane_axpy(int dtype, void* yout, const void* x, const void* z, const double* coef,
                  double sign, long len, long nplanes, int C, const int32_t* active, void* s) {
  DISPATCH(dtype,
           plane_axpy<float>((float*)yout, (const float*)x, (const float*)z, coef, sign,
                             (size_t)len, nplanes, C, active, STREAM(s)),
           plane_axpy<double>((double*)yout, (const double*)x, (const double*)z, coef, sign,
                              (size_t)len, nplanes, C, active, STREAM(s)));
}

int sp_gather_tiles(int dtype, const void* img, const int32_t* oy, const int32_t* ox, int ntile,
                    int C, int H, int W, int bh, int bw, void* out, void* s) {
  DISPATCH(dtype,
           gather_tiles<float>((const float*)img, oy, ox, ntile, C, H, W, bh, bw, (float*)out,
                               STREAM(s)),
           gather_tiles<double>((const double*)img, oy, ox, ntile, C, H, W, bh, bw,
                                (double*)out, STREAM(s)));
}

int sp_gather_mask_tiles(const uint8_t* m, const int32_t* oy, const int32_t* ox, int ntile,
                         int H, int W, int bh, int bw, uint8_t* out, void* s) {
  return gather_mask_tiles(m, oy, ox, ntile, H, W, bh, bw, out, STREAM(s));
}

int sp_ras_scatter(int dtype, void* g, const void* v, const int32_t* tile_of,
                   const int32_t* ys, const int32_t* xs, const int32_t* row_k0,
                   const int32_t* row_n, const int32_t* col_k0, const int32_t* col_n, int nbx,
                   int bh, int bw, int C, int H, int W, void* s) {
  DISPATCH(dtype,
           ras_scatter<float>((float*)g, (const float*)v, tile_of, ys, xs, row_k0, row_n,
                              col_k0, col_n, nbx, bh, bw, C, H, W, STREAM(s)),
           ras_scatter<double>((double*)g, (const double*)v, tile_of, ys, xs, row_k0, row_n,
                               col_k0, col_n, nbx, bh, bw, C, H, W, STREAM(s)));
}

int sp_where_mask(int dtype, const void* x, const uint8_t* m, void* out, int C, int H, int W,
                  void* s) {
  DISPATCH(dtype, where_mask<float>((const float*)x, m, (float*)out, C, H, W, STREAM(s)),
           where_mask<double>((const double*)x, m, (double*)out, C, H, W, STREAM(s)));
}

int sp_neighbor_balance(int dtype, const double* f, const void* u, const uint8_t* m, void* g,
                        int C, int H, int W, void* s) {
  DISPATCH(dtype,
           neighbor_balance<float>(f, (const float*)u, m, (float*)g, C, H, W, STREAM(s)),
           neighbor_balance<double>(f, (const double*)u, m, (double*)g, C, H, W, STREAM(s)));
}

int sp_masked_sym_rhs_tiles(int dtype, const void* x, const uint8_t* m, void* out, int C, int H,
                            int W, int ntile, const int32_t* active, void* s) {
  DISPATCH(dtype,
           masked_sym_rhs<float>((const float*)x, m, (float*)out, C, H, W, STREAM(s), ntile,
                                 active),
           masked_sym_rhs<double>((const double*)x, m, (double*)out, C, H, W, STREAM(s), ntile,
                                  active));
}

int sp_ct_apply_tiles(int dtype, const void* w, const uint8_t* m, void* out, int C, int H, int W,
                      int ntile, const int32_t* active, void* s) {
  DISPATCH(dtype,
           ct_apply<float>((const float*)w, m, (float*)out, C, H, W, 1.0, STREAM(s), ntile,
                           active),
           ct_apply<double>((const double*)w, m, (double*)out, C, H, W, 1.0, STREAM(s), ntile,
                            active));
}

}  // extern "C"
