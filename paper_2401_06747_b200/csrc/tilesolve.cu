// tilesolve.cu -- batched cold solves of the RAS block-local systems with
// the level sweeps fused per block (sm_100a).
//
// Reference: tonal.py:120-131 / 343-354 (the block-local products B_b and
// B_b^T are cold inpainting solves on each 64x64 RAS block to
// local_product_tol) running solver.py:328-372 (solve_sym: tolerance loop;
// V-cycle solver.py:283-300; ORAS smoother numba_impl.py:161-263).
//
// The generic batched hierarchy (solver.cu, ntile > 1) runs a two-level
// V-cycle over all 2,546 blocks of a 4K image as ~15 full sweeps (residual,
// blend, restriction, rhs, prolongation, enforcement), each streaming the
// whole block set through HBM (≈ 125 MB per level-0 vector at 4K RGB, well
// over the L2), plus a host round trip per V-cycle for the stopping test.
//
// A 64x64 block plane is 16 KB, so everything between two ORAS local-CG
// launches can run on ONE CTA per block out of shared memory:
//
//   P0  u = enforce(0, b~); r = b~ - A~ u; ||r_c||^2; ||b~||; stop test
//   [ORAS level 0: one warp per (32x32 job, channel, block) -- k_oras_warp]
//   P1  u0 += corr (blend) ; r1 = restrict(b~ - A~ u0) ; b1 = C~ r1 ;
//       u1 = mask ? b1 : 0 ; r1 = b1 - A~ u1 ; ||r1_c||^2
//   [ORAS level 1]  P2  u1 += corr1 ; r1 ; ||r1_c||^2   [ORAS level 1]
//   P3  u1 += corr1 ; u0 += P u1, u0[mask] = b~ ; r0 ; ||r0_c||^2
//   [ORAS level 0]  P4  u0 += corr ; r0 ; ||r0_c||^2 ; stop test, count
//
// so a V-cycle is 8 launches and moves each block's u/r/corr a couple of
// times instead of ~15 times, while the ORAS jobs keep the full-device
// occupancy of the one-warp kernel.  The stopping test (per block, over all
// its channels, solver.py:358-368) runs on the device: P0/P4 clear the
// block's `active` flag and count the live blocks; the host reads one
// integer per V-cycle.
//
// Arithmetic contract: every element operation is the one of mg.cu / oras.cu
// (same double accumulation orders and roundings); the residual norms (and
// so the ORAS thresholds tau_c and the stopping test) are summed per block
// in a different order than the generic sweeps, so iterates agree with the
// generic batched path to rounding (tests/test_tonal_gpu.py), not bitwise.
#include <cmath>

#include "kernels.cuh"
#include "solver.cuh"

namespace sp {

static int tile_fused_on = 1;
int tile_fused(int v) {
  if (v >= 0) tile_fused_on = v;
  return tile_fused_on;
}

namespace {

constexpr int PT = 512;       // threads per block-CTA
constexpr int TMAX = 64;      // level-0 side limit
constexpr int CMAX = 1024;    // level-1 pixels limit (32 x 32)

struct TV {
  float *u0, *b0, *r0, *corr0, *u1, *b1, *r1, *corr1;
  const uint8_t *m0, *m1;
  double *n0, *n1;       // [tile][C] sum r^2 of the level
  double* scale;         // [tile] ||b~|| (or 1)
  int* active;           // [tile]
  int *done, *conv;      // [tile]
  int* live;             // live-block counter of the last stop test
  const int* list;       // the grid covers these tiles (compacted active set) or null
  int C, H0, W0, H1, W1, bh0, bw0, nby0, nbx0, stride;
  double tol;
  int max_cycles;
};

template <int NT>
__device__ __forceinline__ double cta_sum_d(double v, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += buf[w];
  __syncthreads();
  return s;
}

// A~ x at pixel k (mg.cu sym_row_at with inv_h2 = 1; masked rows: x)
__device__ __forceinline__ float sym_ax(const float* X, const uint8_t* M, int k, int y, int x,
                                        int H, int W) {
  if (M[k]) return X[k];
  double d = 0.0, a = 0.0;
  if (y > 0) { d += 1.0; if (!M[k - W]) a += (double)X[k - W]; }
  if (y < H - 1) { d += 1.0; if (!M[k + W]) a += (double)X[k + W]; }
  if (x > 0) { d += 1.0; if (!M[k - 1]) a += (double)X[k - 1]; }
  if (x < W - 1) { d += 1.0; if (!M[k + 1]) a += (double)X[k + 1]; }
  return (float)((d * (double)X[k] - a) * 1.0);
}

// r = b~ - A~ u of a plane held in shared memory (U, M); b~ and r in global
// memory; returns sum r^2 (CTA-uniform)
__device__ __forceinline__ double plane_residual(const float* U, const uint8_t* M,
                                                 const float* __restrict__ B,
                                                 float* __restrict__ R, int H, int W,
                                                 double* buf) {
  double sq = 0.0;
#pragma unroll 4
  for (int k = threadIdx.x; k < H * W; k += PT) {
    const int y = k / W, x = k - y * W;
    const float r = (float)(B[k] - sym_ax(U, M, k, y, x, H, W));
    R[k] = r;
    sq += (double)r * (double)r;
  }
  return cta_sum_d<PT>(sq, buf);
}

// u += the weighted corrections of the covering level-0 blocks, in block
// index order (oras.cu k_oras_blend): one barrier-separated phase per block,
// so every pixel receives its corrections in ascending block order while
// each phase reads one block's corrections contiguously
template <int TH0, int TW0>
__device__ __forceinline__ void blend0(const TV& a, float* U, const float* __restrict__ u,
                                       const float* __restrict__ corr) {
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int bh = TH0 ? 32 : a.bh0, bw = TW0 ? 32 : a.bw0;
  const int nby = TH0 ? 3 : a.nby0, nbx = TW0 ? 3 : a.nbx0, stride = TH0 ? 26 : a.stride;
  const int npx = bh * bw;
  if (TH0 == 64 && TW0 == 64) {
    // every global load first (u, then the thread's pixels of all nine
    // blocks), so their latencies overlap; the phases then run on-chip
    constexpr int NU = 64 * 64 / PT, NC = 32 * 32 / PT;
    float uv[NU], cv[9][NC];
#pragma unroll
    for (int q = 0; q < NU; ++q) uv[q] = u[threadIdx.x + q * PT];
#pragma unroll
    for (int kb = 0; kb < 9; ++kb)
#pragma unroll
      for (int q = 0; q < NC; ++q) cv[kb][q] = corr[kb * 1024 + threadIdx.x + q * PT];
#pragma unroll
    for (int q = 0; q < NU; ++q) U[threadIdx.x + q * PT] = uv[q];
#pragma unroll
    for (int kb = 0; kb < 9; ++kb) {
      const int ys = block_start(kb / 3, 26, 64, 32), xs = block_start(kb % 3, 26, 64, 32);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const int k = threadIdx.x + q * PT, i = k >> 5, j = k & 31;
        const int g = (ys + i) * 64 + xs + j;
        U[g] = U[g] + cv[kb][q];
      }
    }
    return;
  }
  for (int k = threadIdx.x; k < H0 * W0; k += PT) U[k] = u[k];
  for (int kb = 0; kb < nby * nbx; ++kb) {
    const int ky = kb / nbx, kx = kb - ky * nbx;
    const int ys = block_start(ky, stride, H0, bh), xs = block_start(kx, stride, W0, bw);
    const float* cb = corr + (size_t)kb * npx;
    __syncthreads();
    for (int k = threadIdx.x; k < npx; k += PT) {
      const int i = k / bw, j = k - i * bw;
      const int g = (ys + i) * W0 + xs + j;
      U[g] = U[g] + cb[k];
    }
  }
}

__device__ __forceinline__ void load_mask(uint8_t* M, const uint8_t* __restrict__ m, int n) {
  for (int k = threadIdx.x; k < n; k += PT) M[k] = m[k];
}

// the stop test of solver.py:358-368 for one block (thread 0)
__device__ __forceinline__ void stop_test(const TV& a, int tile, const double* nrm) {
  double tot = 0.0;
  for (int c = 0; c < a.C; ++c) tot += nrm[c];
  const double rel = sqrt(tot) / a.scale[tile];
  if (rel <= a.tol) {
    a.conv[tile] = 1;
    a.active[tile] = 0;
  } else if (a.done[tile] >= a.max_cycles) {
    a.active[tile] = 0;
  } else {
    atomicAdd(a.live, 1);
  }
}

// P0: cold start u = mask ? b~ : 0 (solver.cu solve_t), residual, ||b~||
template <int TH0, int TW0, int TH1, int TW1>
__global__ void __launch_bounds__(PT) k_tv_init(TV a) {
  __shared__ float U[TMAX * TMAX];
  __shared__ uint8_t M[TMAX * TMAX];
  __shared__ double buf[PT / 32];
  __shared__ double nrm[8];
  const int tile = a.list ? a.list[blockIdx.x] : blockIdx.x;
  if (!a.active[tile]) return;
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int H1 = TH1 ? TH1 : a.H1, W1 = TW1 ? TW1 : a.W1;
  (void)H1; (void)W1; (void)H0; (void)W0;
  const int n0 = H0 * W0;
  load_mask(M, a.m0 + (size_t)tile * n0, n0);
  double bb = 0.0;
  for (int c = 0; c < a.C; ++c) {
    const size_t o = ((size_t)tile * a.C + c) * n0;
    __syncthreads();
    for (int k = threadIdx.x; k < n0; k += PT) {
      const float b = a.b0[o + k];
      const float u = M[k] ? b : 0.0f;
      U[k] = u;
      a.u0[o + k] = u;
      bb += (double)b * (double)b;
    }
    __syncthreads();
    const double s = plane_residual(U, M, a.b0 + o, a.r0 + o, H0, W0, buf);
    if (threadIdx.x == 0) {
      nrm[c] = s;
      a.n0[(size_t)tile * a.C + c] = s;
    }
  }
  bb = cta_sum_d<PT>(bb, buf);
  if (threadIdx.x == 0) {
    const double bn = sqrt(bb);
    a.scale[tile] = bn > 0 ? bn : 1.0;
    a.done[tile] = 0;
    a.conv[tile] = 0;
    stop_test(a, tile, nrm);
  }
}

// P1: blend level 0, restrict the residual, coarse rhs / start, coarse residual
template <int TH0, int TW0, int TH1, int TW1>
__global__ void __launch_bounds__(PT) k_tv_down(TV a) {
  __shared__ float U[TMAX * TMAX];
  __shared__ uint8_t M[TMAX * TMAX];
  __shared__ float R1[CMAX], B1[CMAX], U1[CMAX];
  __shared__ uint8_t M1[CMAX];
  __shared__ double buf[PT / 32];
  const int tile = a.list ? a.list[blockIdx.x] : blockIdx.x;
  if (!a.active[tile]) return;
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int H1 = TH1 ? TH1 : a.H1, W1 = TW1 ? TW1 : a.W1;
  (void)H1; (void)W1; (void)H0; (void)W0;
  const int n0 = H0 * W0, n1 = H1 * W1, npx = a.bh0 * a.bw0;
  load_mask(M, a.m0 + (size_t)tile * n0, n0);
  load_mask(M1, a.m1 + (size_t)tile * n1, n1);
  for (int c = 0; c < a.C; ++c) {
    const size_t o = ((size_t)tile * a.C + c) * n0, o1 = ((size_t)tile * a.C + c) * n1;
    const float* B0 = a.b0 + o;
    __syncthreads();
    blend0<TH0, TW0>(a, U, a.u0 + o, a.corr0 + ((size_t)tile * a.C + c) * a.nby0 * a.nbx0 * npx);
    __syncthreads();
    for (int k = threadIdx.x; k < n0; k += PT) a.u0[o + k] = U[k];
    // fused residual + 2x2 restriction (mg.cu k_residual_restrict)
    for (int k = threadIdx.x; k < n1; k += PT) {
      const int i = k / W1, j = k - i * W1;
      const int y = 2 * i, x = 2 * j, f = y * W0 + x;
      const bool xr = x + 1 < W0, yd = y + 1 < H0;
      double acc = (double)(float)(B0[f] - sym_ax(U, M, f, y, x, H0, W0));
      int n = 1;
      if (xr) { acc += (double)(float)(B0[f + 1] - sym_ax(U, M, f + 1, y, x + 1, H0, W0)); ++n; }
      if (yd) {
        acc += (double)(float)(B0[f + W0] - sym_ax(U, M, f + W0, y + 1, x, H0, W0));
        ++n;
      }
      if (xr && yd) {
        acc += (double)(float)(B0[f + W0 + 1] -
                               sym_ax(U, M, f + W0 + 1, y + 1, x + 1, H0, W0));
        ++n;
      }
      R1[k] = (float)(acc / (double)n);
    }
    __syncthreads();
    // coarse rhs C~ r and start e = mask ? rhs : 0 (mg.cu k_sym_rhs)
    for (int k = threadIdx.x; k < n1; k += PT) {
      const int y = k / W1, x = k - y * W1;
      float ov;
      if (M1[k]) {
        ov = R1[k];
      } else {
        double s = 0.0;
        if (y > 0 && M1[k - W1]) s += (double)R1[k - W1];
        if (y < H1 - 1 && M1[k + W1]) s += (double)R1[k + W1];
        if (x > 0 && M1[k - 1]) s += (double)R1[k - 1];
        if (x < W1 - 1 && M1[k + 1]) s += (double)R1[k + 1];
        ov = (float)((double)R1[k] + s * 1.0);
      }
      B1[k] = ov;
      const float e = M1[k] ? ov : 0.0f;
      U1[k] = e;
      a.b1[o1 + k] = ov;
      a.u1[o1 + k] = e;
    }
    __syncthreads();
    // coarsest level, first sweep: fresh residual (solver.cu smooth_lv)
    const double s = plane_residual(U1, M1, B1, a.r1 + o1, H1, W1, buf);
    if (threadIdx.x == 0) a.n1[(size_t)tile * a.C + c] = s;
  }
}

// P2: coarse blend + residual (between the two coarsest sweeps)
template <int TH0, int TW0, int TH1, int TW1>
__global__ void __launch_bounds__(PT) k_tv_coarse(TV a) {
  __shared__ float U1[CMAX];
  __shared__ uint8_t M1[CMAX];
  __shared__ double buf[PT / 32];
  const int tile = a.list ? a.list[blockIdx.x] : blockIdx.x;
  if (!a.active[tile]) return;
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int H1 = TH1 ? TH1 : a.H1, W1 = TW1 ? TW1 : a.W1;
  (void)H1; (void)W1; (void)H0; (void)W0;
  const int n1 = H1 * W1;
  load_mask(M1, a.m1 + (size_t)tile * n1, n1);
  for (int c = 0; c < a.C; ++c) {
    const size_t o1 = ((size_t)tile * a.C + c) * n1;
    __syncthreads();
    for (int k = threadIdx.x; k < n1; k += PT) {
      const float v = a.u1[o1 + k] + a.corr1[o1 + k];
      U1[k] = v;
      a.u1[o1 + k] = v;
    }
    __syncthreads();
    const double s = plane_residual(U1, M1, a.b1 + o1, a.r1 + o1, H1, W1, buf);
    if (threadIdx.x == 0) a.n1[(size_t)tile * a.C + c] = s;
  }
}

// cell-centred bilinear axis weights, clamped (mg.cu prolong_axis)
__device__ __forceinline__ void paxis(int y, int n, int& y0, int& y1, double& wy) {
  double fy = ((double)y + 0.5) / 2.0 - 0.5;
  y0 = (int)floor(fy);
  wy = fy - (double)y0;
  if (y0 < 0) { y0 = 0; wy = 0.0; }
  if (y0 > n - 1) { y0 = n - 1; wy = 0.0; }
  y1 = min(y0 + 1, n - 1);
}

// P3: coarse blend, prolongation + enforcement into level 0, residual
template <int TH0, int TW0, int TH1, int TW1>
__global__ void __launch_bounds__(PT, 4) k_tv_up(TV a) {
  __shared__ float U[TMAX * TMAX];
  __shared__ uint8_t M[TMAX * TMAX];
  __shared__ float U1[CMAX];
  __shared__ double buf[PT / 32];
  const int tile = a.list ? a.list[blockIdx.x] : blockIdx.x;
  if (!a.active[tile]) return;
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int H1 = TH1 ? TH1 : a.H1, W1 = TW1 ? TW1 : a.W1;
  (void)H1; (void)W1; (void)H0; (void)W0;
  const int n0 = H0 * W0, n1 = H1 * W1;
  // the bilinear axis weights of every fine row / column, once per CTA
  __shared__ int ay0[TMAX], ay1[TMAX], ax0[TMAX], ax1[TMAX];
  __shared__ double awy[TMAX], awx[TMAX];
  if (threadIdx.x < H0) paxis(threadIdx.x, H1, ay0[threadIdx.x], ay1[threadIdx.x], awy[threadIdx.x]);
  if (threadIdx.x >= 64 && threadIdx.x - 64 < W0) {
    const int x = threadIdx.x - 64;
    paxis(x, W1, ax0[x], ax1[x], awx[x]);
  }
  load_mask(M, a.m0 + (size_t)tile * n0, n0);
  for (int c = 0; c < a.C; ++c) {
    const size_t o = ((size_t)tile * a.C + c) * n0, o1 = ((size_t)tile * a.C + c) * n1;
    __syncthreads();
    for (int k = threadIdx.x; k < n1; k += PT) U1[k] = a.u1[o1 + k] + a.corr1[o1 + k];
    __syncthreads();
    // u += prolongate(e); u[mask] = b~[mask] (mg.cu k_prolong_enforce, add)
    for (int k = threadIdx.x; k < n0; k += PT) {
      float v;
      if (M[k]) {
        v = a.b0[o + k];
      } else {
        const int y = k / W0, x = k - y * W0;
        const int y0 = ay0[y], y1 = ay1[y], x0 = ax0[x], x1 = ax1[x];
        const double wy = awy[y], wx = awx[x];
        const double e = (1.0 - wy) * ((1.0 - wx) * (double)U1[y0 * W1 + x0] +
                                       wx * (double)U1[y0 * W1 + x1]) +
                         wy * ((1.0 - wx) * (double)U1[y1 * W1 + x0] +
                               wx * (double)U1[y1 * W1 + x1]);
        v = a.u0[o + k] + (float)e;
      }
      U[k] = v;
      a.u0[o + k] = v;
    }
    __syncthreads();
    const double s = plane_residual(U, M, a.b0 + o, a.r0 + o, H0, W0, buf);
    if (threadIdx.x == 0) a.n0[(size_t)tile * a.C + c] = s;
  }
}

// P4: blend level 0 (post-smoothing), residual, stop test
template <int TH0, int TW0, int TH1, int TW1>
__global__ void __launch_bounds__(PT) k_tv_close(TV a) {
  __shared__ float U[TMAX * TMAX];
  __shared__ uint8_t M[TMAX * TMAX];
  __shared__ double buf[PT / 32];
  __shared__ double nrm[8];
  const int tile = a.list ? a.list[blockIdx.x] : blockIdx.x;
  if (!a.active[tile]) return;
  const int H0 = TH0 ? TH0 : a.H0, W0 = TW0 ? TW0 : a.W0;
  const int H1 = TH1 ? TH1 : a.H1, W1 = TW1 ? TW1 : a.W1;
  (void)H1; (void)W1; (void)H0; (void)W0;
  const int n0 = H0 * W0, npx = a.bh0 * a.bw0;
  load_mask(M, a.m0 + (size_t)tile * n0, n0);
  for (int c = 0; c < a.C; ++c) {
    const size_t o = ((size_t)tile * a.C + c) * n0;
    __syncthreads();
    blend0<TH0, TW0>(a, U, a.u0 + o,
                     a.corr0 + ((size_t)tile * a.C + c) * a.nby0 * a.nbx0 * npx);
    __syncthreads();
    for (int k = threadIdx.x; k < n0; k += PT) a.u0[o + k] = U[k];
    const double s = plane_residual(U, M, a.b0 + o, a.r0 + o, H0, W0, buf);
    if (threadIdx.x == 0) {
      nrm[c] = s;
      a.n0[(size_t)tile * a.C + c] = s;
    }
  }
  if (threadIdx.x == 0) {
    a.done[tile] += 1;
    stop_test(a, tile, nrm);
  }
}

}  // namespace

// partly active batches launch over the list of active tiles (1) or over
// every tile with early exits (0): sp_tile_list
static int tile_list_on = 1;
int tile_list(int v) {
  if (v >= 0) tile_list_on = v;
  return tile_list_on;
}

bool tile_fused_ok(const Hier* h) {
  if (!tile_fused_on || h->dtype != SP_F32 || h->lv.size() != 2) return false;
  if (h->C < 1 || h->C > 8 || h->cfg.pre != 1 || h->cfg.post != 1) return false;
  const Level& L0 = h->lv[0];
  const Level& L1 = h->lv[1];
  if (L0.H > TMAX || L0.W > TMAX || L0.bh > 32 || L0.bw > 32) return false;
  return L1.nby * L1.nbx == 1 && L1.H * L1.W <= CMAX;
}

// solver.cu solve_t for a batch of tiles: cold start (init_mode 0),
// tolerance mode; per-block stopping on the device
int tile_solve_fused(Hier* h, const float* bsym, float* u_out, double tol, int max_cycles,
                     cudaStream_t s, const int* active_in, int* iters, int* conv) {
  const int nt = h->ntile, C = h->C;
  Level& L0 = h->lv[0];
  Level& L1 = h->lv[1];
  const size_t n = (size_t)nt * C * L0.H * L0.W;
  // the pinned flags may still feed an earlier upload (waits for that copy
  // only, not for the caller's queued work)
  SP_TRY(active_host_ready(h));
  int nact = 0;
  for (int t = 0; t < nt; ++t) {
    h->h_active[t] = active_in ? (active_in[t] != 0) : 1;
    nact += h->h_active[t];
  }
  SP_TRY(upload_active(h, s));
  // the block kernels read b~ straight from the caller's batch ([nt][C][h][w],
  // the level-0 layout): no staging copy
  // a partly active batch (the tail of the RAS local CG: a few blocks still
  // iterating) launches its grids over the list of active tiles only -- the
  // full-size grids of early-exiting CTAs cost ~1 ms per solve at 4K
  const int* list = nullptr;
  int ngrid = nt;
  if (nact < nt && tile_list_on && oras_variant(-1) >= 6) {  // one-warp ORAS jobs
    if (!h->d_list) SP_CUDA(cudaMalloc(&h->d_list, sizeof(int) * nt));
    if (!h->h_list) SP_CUDA(cudaMallocHost(&h->h_list, sizeof(int) * nt));
    // the pinned list may still feed the previous solve's upload
    if (h->list_ev) SP_CUDA(cudaEventSynchronize(h->list_ev));
    else SP_CUDA(cudaEventCreateWithFlags(&h->list_ev, cudaEventDisableTiming));
    int k = 0;
    for (int t = 0; t < nt; ++t)
      if (h->h_active[t]) h->h_list[k++] = t;
    SP_CUDA(cudaMemcpyAsync(h->d_list, h->h_list, sizeof(int) * nact, cudaMemcpyHostToDevice, s));
    SP_CUDA(cudaEventRecord(h->list_ev, s));
    list = h->d_list;
    ngrid = nact;
  }
  double* scale = (double*)h->d_scratch;
  int* done = (int*)(scale + nt);
  int* cvd = done + nt;
  int* live = cvd + nt;
  TV a;
  // with every block active the block kernels iterate in the caller's output
  // directly (each block's u is written by k_tv_init before any read); a
  // partly active batch keeps the hierarchy's buffer and copies it out whole
  // (the inactive blocks' stale values, as the unfused path returns them)
  const bool direct = nact == nt && (u_out + n <= bsym || bsym + n <= u_out);
  a.u0 = direct ? u_out : (float*)L0.u;
  a.b0 = const_cast<float*>(bsym);
  a.r0 = (float*)L0.r;
  a.corr0 = (float*)L0.corr;
  a.u1 = (float*)L1.u; a.b1 = (float*)L1.b; a.r1 = (float*)L1.r; a.corr1 = (float*)L1.corr;
  a.m0 = L0.mask; a.m1 = L1.mask;
  a.n0 = L0.norms; a.n1 = L1.norms;
  a.scale = scale; a.active = h->d_active; a.done = done; a.conv = cvd; a.live = live;
  a.list = list;
  a.C = C; a.H0 = L0.H; a.W0 = L0.W; a.H1 = L1.H; a.W1 = L1.W;
  a.bh0 = L0.bh; a.bw0 = L0.bw; a.nby0 = L0.nby; a.nbx0 = L0.nbx;
  a.stride = h->cfg.block - h->cfg.overlap;
  a.tol = tol; a.max_cycles = max_cycles;
  const int stride = a.stride;
  // never-active blocks keep done = conv = 0
  SP_CUDA(cudaMemsetAsync(done, 0, sizeof(int) * (2 * (size_t)nt + 1), s));
  const bool sp64 = L0.H == 64 && L0.W == 64 && L0.bh == 32 && L0.bw == 32 && stride == 26 &&
                    L1.H == 32 && L1.W == 32;
  auto k_init = sp64 ? k_tv_init<64, 64, 32, 32> : k_tv_init<0, 0, 0, 0>;
  auto k_down = sp64 ? k_tv_down<64, 64, 32, 32> : k_tv_down<0, 0, 0, 0>;
  auto k_coarse = sp64 ? k_tv_coarse<64, 64, 32, 32> : k_tv_coarse<0, 0, 0, 0>;
  auto k_up = sp64 ? k_tv_up<64, 64, 32, 32> : k_tv_up<0, 0, 0, 0>;
  auto k_close = sp64 ? k_tv_close<64, 64, 32, 32> : k_tv_close<0, 0, 0, 0>;
  if (ngrid == 0) {
    SP_CUDA(cudaMemcpyAsync(u_out, L0.u, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    for (int t = 0; t < nt; ++t) {
      if (iters) iters[t] = 0;
      if (conv) conv[t] = 0;
    }
    return 0;
  }
  k_init<<<ngrid, PT, 0, s>>>(a);
  SP_CHECK_LAUNCH();
  int* hl = (int*)h->h_norms;  // pinned staging (>= ntile * C doubles)
  auto oras = [&](Level& L) {
    return oras_local_launch<float>((const float*)L.r, L.mask, L.norms, L.tau_scale, L.ys, L.xs,
                                    L.nby, L.nbx, L.bh, L.bw, L.H, L.W, C, h->gamma,
                                    (long)L.bh * L.bw, 1.0, (const float*)L.weights,
                                    (float*)L.corr, s, nt, h->d_active, stride, 0, 0,
                                    L.wdelta, L.offbits, list, ngrid);
  };
  // V-cycles run in batches between reads of the live-block count: a block
  // that stops inside a batch is skipped by every later launch (each kernel
  // tests `active`), so batching changes no result, only the number of host
  // round trips.  The local products converge in 3 V-cycles (4K RAS), so the
  // first batch is 3, then one V-cycle per read.
  int batch = 3;
  while (true) {
    for (int b = 0; b < batch; ++b) {
      SP_CUDA(cudaMemsetAsync(live, 0, sizeof(int), s));
      SP_TRY(oras(L0));                     // pre-smoothing, level 0
      k_down<<<ngrid, PT, 0, s>>>(a);
      SP_CHECK_LAUNCH();
      SP_TRY(oras(L1));                     // coarsest, sweep 1
      k_coarse<<<ngrid, PT, 0, s>>>(a);
      SP_CHECK_LAUNCH();
      SP_TRY(oras(L1));                     // coarsest, sweep 2
      k_up<<<ngrid, PT, 0, s>>>(a);
      SP_CHECK_LAUNCH();
      SP_TRY(oras(L0));                     // post-smoothing, level 0
      k_close<<<ngrid, PT, 0, s>>>(a);
      SP_CHECK_LAUNCH();
    }
    SP_CUDA(cudaMemcpyAsync(hl, live, sizeof(int), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    if (hl[0] == 0) break;
    batch = 1;
  }
  if (!direct)
    SP_CUDA(cudaMemcpyAsync(u_out, L0.u, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
  SP_CUDA(cudaMemcpyAsync(hl, done, sizeof(int) * 2 * nt, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  long long cyc = 0;
  for (int t = 0; t < nt; ++t) {
    if (iters) iters[t] = hl[t];
    if (conv) conv[t] = hl[nt + t];
    cyc += hl[t];
  }
  count_work(1, cyc * (long long)L0.H * L0.W);
  return 0;
}

}  // namespace sp
