// geometry.cuh -- jump flooding / Delaunay / bucket workspace (geometry.cu).
#pragma once
#include "kernels.cuh"

namespace sp {

// Reusable per-(H, W) workspace of the densification geometry.
struct Geo {
  int H = 0, W = 0;
  long m = 0, T = 0;
  size_t key_cap = 0, tri_cap = 0;
  int *lab_a = nullptr, *lab_b = nullptr;  // labels live in lab_a after geo_voronoi
  int *sy = nullptr, *sx = nullptr;        // seed coordinates (row-major order)
  int* idx = nullptr;
  int* rank = nullptr;                     // seed index at each seed pixel
  uint8_t* flags = nullptr;
  unsigned long long* keys = nullptr;
  unsigned* keys2 = nullptr;               // high words of wide keys (>= 2^21 seeds)
  unsigned long long* nkeys = nullptr;
  int* tris = nullptr;                     // (T, 3) ascending triples, sorted
  int* assign = nullptr;
  int* smt = nullptr;
  double* sums = nullptr;
  long long* amax = nullptr;
  double* amax_val = nullptr;
  unsigned long long* dmax = nullptr;
  int* nsel = nullptr;
  void* h_small = nullptr;
  ~Geo();
};

int geo_create(Geo** out, int H, int W);
int geo_voronoi(Geo* g, const uint8_t* mask, double hint, long* m_out, double* radius,
                int* nsteps_out, cudaStream_t s);
int geo_delaunay(Geo* g, long* T_out, cudaStream_t s);
long geo_wide_threshold(long v);  // seeds from which the wide (2 x 32-bit) keys apply
int geo_accumulate(Geo* g, const double* err, int voronoi, cudaStream_t s);
int geo_accumulate_mode(int v);
int geo_select(Geo* g, uint8_t* mask, long nbuckets, long want, long* picked, cudaStream_t s);
int fill_highest_error(Geo* g, const double* err, uint8_t* mask, long want, cudaStream_t s);
// row-strip partition of the Delaunay step and the accumulate (geometry.cu)
int geo_corner_keys(Geo* g, int r0, int r1, long* n_out, cudaStream_t s);
int geo_delaunay_from_keys(Geo* g, const unsigned long long* keys, long n, long* T_out,
                           cudaStream_t s);
int geo_raster_rows(Geo* g, int r0, int r1, cudaStream_t s);
int geo_reduce_range(Geo* g, const double* err, long t0, long t1, cudaStream_t s);

// B1 building blocks
int jfa_passes(int* a, int* b, const int* sy, const int* sx, const long long* steps,
               int nsteps, int H, int W, int** result, cudaStream_t s);
int dist2(const int* lab, const int* sy, const int* sx, long long* out,
          unsigned long long* dmax, int H, int W, int m, cudaStream_t s);
int seeds_to_soa(const long long* seeds, long m, int* sy, int* sx, cudaStream_t s);
int fs_dither(const double* dens, uint8_t* out, int H, int W, cudaStream_t s);
template <typename V>
int assign_tris(const V* tris, long T, const V* vy, const V* vx, int H, int W, int* assign,
                bool neg_unset, cudaStream_t s);
int fallback(const int* assign, const int* lab, const int* smt, int* out, size_t n,
             cudaStream_t s);
int reduce_cells(const int* assign, const double* err, long nseg, double* sums,
                 long long* amax_idx, double* amax_val, int H, int W, cudaStream_t s);

}  // namespace sp
