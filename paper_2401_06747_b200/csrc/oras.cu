// oras.cu -- optimized restricted additive Schwarz sweep (sm_100a).
//
// Reference: numba_impl.py:161-263 (oras_apply) driven by solver.py:259-273.
//
// k_oras_local: one CTA per (block, channel, tile).  The block's mask is
// staged in shared memory, its residual in registers (each thread owns PPT
// pixels, strided by the CTA size so warps read whole rows); the search
// direction p is staged in shared memory for the 5-point stencil and the
// local CG runs entirely on-chip: dots in double, reduced by warp shuffles
// plus a fixed-order cross-warp sum (deterministic); alpha/beta rounded to
// T and the vector updates in T exactly like the reference.  The kernel
// writes the WEIGHTED correction T(w_b) * v_b -- the very product the
// reference forms in its blend loop (numba_impl.py:261-263) -- into `corr`
// ([tile][C][nb][bh][bw]).
//
// k_oras_blend: the reference adds u += w_b * v_b sequentially in block
// order.  Every pixel gathers its (at most 3x3) covering blocks in
// ascending block index -- the same summation order -- so the blend is
// race-free and bit-identical, and with pre-weighted corrections it is a
// pure gather-add.
//
// k_block_weights: the partition-of-unity weights of build_decomposition
// (solver.py:142-197), recomputed on the device in double with the exact
// operation order (pointwise total over covering blocks in block order,
// last covering block takes 1 - sum of the others), cast to T.
#include <cuda_pipeline.h>

#include <algorithm>

#include "kernels.cuh"
#include "oras_warp.cuh"

namespace sp {

// ORAS statistics (jobs, local CG iterations, jobs converged on entry);
// collected only while enabled through sp_stats (tracing aid)
__device__ unsigned long long g_oras_stats[4];
__device__ int g_stats_on;

// kernel choice for float blocks <= 32x32 (sp_oras_variant, A/B runs):
// 8 = one warp per job, the lean local CG on packed float pairs
// (k_oras_warp<CGK 2>: FFMA2 / FADD2, the default; 341 instead of 471
// instructions per CG step, 4K pipeline 249.7 -> 244.9 ms); 7 = the same CG
// on scalar floats (k_oras_warp<CGK 1>);
// 6 = one warp per job, the reference-ordered CG (bit-identical to 0 and 4);
// 4 = k_oras_warp with four jobs per CTA; 0 = the register-resident 4-warp
// job kernel (k_oras_rows); 1 = the 256-thread CTA kernel with the
// reference's double stencil.  (A persistent cp.async-prefetch variant
// measured slower -- 1.80 vs 1.58 ms per 4K V-cycle, profiles/
// oras_ab_r01j.txt -- and was removed; so did a two-warps-per-job pair CG,
// 16 rows per lane at 96-124 registers for 16-20 warps per SM: 255.7 /
// 260.3 vs 244.8 ms per 4K pipeline -- 480 instead of 341 instructions per
// job step outweigh the extra warps.)
static int oras_kernel = 8;
int oras_variant(int v) {
  if (v >= 0) oras_kernel = v;
  return oras_kernel;
}

// the default kernel reads the precomputed per-job row-mask words (1) or
// loads and tests the job's mask bytes itself (0); bit-identical
static int offbits_on = 1;
int oras_offbits(int v) {
  if (v >= 0) offbits_on = v;
  return offbits_on;
}

int oras_stats(int enable, unsigned long long* out) {
  if (out) SP_CUDA(cudaMemcpyFromSymbol(out, g_oras_stats, sizeof(unsigned long long) * 4));
  if (enable >= 0) {
    unsigned long long z[4] = {0, 0, 0, 0};
    SP_CUDA(cudaMemcpyToSymbol(g_oras_stats, z, sizeof(z)));
    SP_CUDA(cudaMemcpyToSymbol(g_stats_on, &enable, sizeof(int)));
  }
  return 0;
}

namespace {

constexpr int NT = 256;

// Specialization for the default 32-wide blocks (bw == 32, bh <= 32): lane =
// column, warp w owns rows w, w+8, w+16, w+24.  No integer division, the
// stencil is branch-free (absent neighbours add an exact +0.0), and p is
// staged in shared memory as double so each neighbour costs one LDS.64
// instead of a load plus a conversion.  Arithmetic is identical to the
// generic kernel below.
template <typename T>
__global__ void __launch_bounds__(NT, 4) k_oras_local32(
    const T* __restrict__ r, const uint8_t* __restrict__ m,
    const double* __restrict__ tau_src, double tau_scale, const int* __restrict__ ys,
    const int* __restrict__ xs, int nbx, int bh, int H, int W, int stride, double gamma,
    long cap, double inv_h2, const T* __restrict__ weights, T* __restrict__ corr,
    const int* __restrict__ active) {
  constexpr int PPT = 4, BWD = 32;
  __shared__ double psd[32 * BWD + 2 * BWD];  // p as double, one guard row each side
  __shared__ uint8_t ms[32 * BWD];
  __shared__ double red0[NT / 32], red1[NT / 32], red2[NT / 32];
  const int bi = blockIdx.x, ch = blockIdx.y, C = gridDim.y, nb = gridDim.x;
  const int tile = blockIdx.z;
  if (active && !active[tile]) return;
  // block origin: arithmetic _starts (solver.py:134-139) when stride > 0,
  // else the caller's table (kernel-table path with arbitrary starts)
  const int kyb = bi / nbx, kxb = bi - kyb * nbx;
  const int y0 = stride > 0 ? block_start(kyb, stride, H, bh) : ys[kyb];
  const int x0 = stride > 0 ? block_start(kxb, stride, W, BWD) : xs[kxb];
  const int npx = bh * BWD;
  const size_t plane = (size_t)H * W;
  const T* rc = r + ((size_t)tile * C + ch) * plane;
  m += (size_t)tile * plane;
  const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* pd = psd + BWD;  // pd[-32 .. npx + 31] addressable
  const double tau = tau_scale * tau_src[(size_t)tile * C + ch];

  T res[PPT], v[PPT], p[PPT], wgt[PPT];
  double diag[PPT];
  unsigned flags[PPT];
  // issue every global load of the job up front (residual, mask, blend
  // weights): the job is short and otherwise pays several DRAM round trips
  const T* wb = weights + (size_t)bi * npx;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int i = w + 8 * s;
    res[s] = (T)0;
    wgt[s] = (T)0;
    if (i < bh) {
      const size_t g = (size_t)(y0 + i) * W + (x0 + j);
      ms[i * BWD + j] = m[g];
      res[s] = rc[g];
      wgt[s] = wb[i * BWD + j];
    }
  }
  // guard rows of the staged p stay zero
  if (threadIdx.x < BWD) {
    psd[threadIdx.x] = 0.0;
    psd[BWD + npx + threadIdx.x] = 0.0;
  }
  __syncthreads();
  double rs_part = 0.0;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int i = w + 8 * s, k = i * BWD + j;
    flags[s] = 0;
    v[s] = p[s] = (T)0;
    diag[s] = 0.0;
    if (i < bh) {
      const int gy = y0 + i, gx = x0 + j;
      unsigned f = 1u;
      if (ms[k]) f |= 2u;
      double d = 0.0;
      if (gy > 0) {
        if (i > 0) { d += 1.0; if (!ms[k - BWD]) f |= 16u; } else d += 1.0 - gamma;
      }
      if (gy < H - 1) {
        if (i < bh - 1) { d += 1.0; if (!ms[k + BWD]) f |= 32u; } else d += 1.0 - gamma;
      }
      if (gx > 0) {
        if (j > 0) { d += 1.0; if (!ms[k - 1]) f |= 64u; } else d += 1.0 - gamma;
      }
      if (gx < W - 1) {
        if (j < BWD - 1) { d += 1.0; if (!ms[k + 1]) f |= 128u; } else d += 1.0 - gamma;
      }
      flags[s] = f;
      diag[s] = d;
      p[s] = res[s];
      rs_part += (double)res[s] * (double)res[s];
    }
  }
  double rs = cta_sum<NT>(rs_part, red0);
  long it = 0;
  int phase = 0;
  T ap[PPT];
  // single-precision fast path: the stencil runs in float (one rounding of
  // d*p - acc in float instead of double-then-float) and the per-thread dot
  // partials are float over its 4 pixels; cross-thread sums stay double.
  // The local CG is an inexact smoother whose dots already differ from the
  // reference in summation order, so this only moves the iterate at the
  // 1e-7 level (solver parity is tolerance based, tests/test_solver_gpu.py).
  constexpr bool kF32 = sizeof(T) == 4;
  float* pf = reinterpret_cast<float*>(pd);
  float diagf[PPT];
#pragma unroll
  for (int s = 0; s < PPT; ++s) diagf[s] = (float)diag[s];
  const float inv_h2f = (float)inv_h2;
  while (rs > tau && it < cap) {
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      const int i = w + 8 * s;
      if (i < bh) {
        if (kF32) pf[i * BWD + j] = (float)p[s];
        else pd[i * BWD + j] = (double)p[s];
      }
    }
    __syncthreads();
    double pap_part = 0.0;
    float pap_f = 0.0f;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      const unsigned f = flags[s];
      const int k = (w + 8 * s) * BWD + j;
      const int kl = j > 0 ? k - 1 : k, kr = j < BWD - 1 ? k + 1 : k;
      // guard rows / lane clamps keep every address valid; absent
      // neighbours contribute +0.0
      if (kF32) {
        float acc = 0.0f;
        acc += (f & 16u) ? pf[k - BWD] : 0.0f;
        acc += (f & 32u) ? pf[k + BWD] : 0.0f;
        acc += (f & 64u) ? pf[kl] : 0.0f;
        acc += (f & 128u) ? pf[kr] : 0.0f;
        const float pv = (float)p[s];
        float a = (f & 2u) ? pv : (diagf[s] * pv - acc) * inv_h2f;
        a = (f & 1u) ? a : 0.0f;
        ap[s] = (T)a;
        pap_f += pv * a;
      } else {
        double acc = 0.0;
        acc += (f & 16u) ? pd[k - BWD] : 0.0;
        acc += (f & 32u) ? pd[k + BWD] : 0.0;
        acc += (f & 64u) ? pd[kl] : 0.0;
        acc += (f & 128u) ? pd[kr] : 0.0;
        const double pdv = (double)p[s];
        const T a = (f & 2u) ? p[s] : (T)((diag[s] * pdv - acc) * inv_h2);
        ap[s] = (f & 1u) ? a : (T)0;
        pap_part += pdv * (double)ap[s];
      }
    }
    if (kF32) pap_part = (double)pap_f;
    const double pap = cta_sum<NT>(pap_part, phase ? red2 : red1);
    if (pap <= 0.0) break;
    const T alpha = (T)(rs / pap);
    double rsn_part = 0.0;
    float rsn_f = 0.0f;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      if (!(flags[s] & 1u)) continue;
      v[s] = v[s] + alpha * p[s];
      res[s] = res[s] - alpha * ap[s];
      if (kF32) rsn_f += (float)res[s] * (float)res[s];
      else rsn_part += (double)res[s] * (double)res[s];
    }
    if (kF32) rsn_part = (double)rsn_f;
    const double rsn = cta_sum<NT>(rsn_part, phase ? red1 : red2);
    const T beta = (T)(rsn / rs);
    rs = rsn;
#pragma unroll
    for (int s = 0; s < PPT; ++s)
      if (flags[s] & 1u) p[s] = res[s] + beta * p[s];
    ++it;
    phase ^= 1;
  }
  T* out = corr + (((size_t)tile * C + ch) * nb + bi) * (size_t)npx;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int i = w + 8 * s, k = i * BWD + j;
    if (i < bh) out[k] = wgt[s] * v[s];
  }
  if (threadIdx.x == 0 && g_stats_on) {
    atomicAdd(&g_oras_stats[0], 1ull);
    atomicAdd(&g_oras_stats[1], (unsigned long long)it);
    if (it == 0) atomicAdd(&g_oras_stats[2], 1ull);
    atomicMax(&g_oras_stats[3], (unsigned long long)it);
  }
}

// ---------------------------------------------------------------------------
// Default float kernel for blocks up to 32 x 32 (the ORAS 32/6 configuration
// on every level): 4 warps per (block, channel, tile) job.  Warp w owns the 8
// consecutive block rows 8w..8w+7 and lane j owns column j, so the whole
// local CG lives in registers: up/down neighbours are the adjacent registers,
// left/right come from one shuffle each, the mask is a per-thread bit word.
// Only the two edge rows of each warp cross warps, through shared memory.
//
// Two barriers per CG step instead of three: after the r-update each warp
// publishes its NEW edge residual rows together with its rs partial; after
// the barrier a neighbour rebuilds the new edge search direction itself as
// r_edge + beta * p_edge_old -- the same operation, operands and rounding the
// owning warp uses for its own p -- so p never has to be staged again.
//
// The operator is applied branch-free: (A p)_i = dgp_i p_i - fm_i * sum of the
// in-block neighbours' q = fm * p, with fm the valid-and-unmasked indicator
// and dgp the Robin-closed diagonal (1 on masked identity rows, 0 outside the
// block), so no per-pixel mask bit tests remain in the loop.
//
// Arithmetic: stencil and vector updates in float (fused multiply-adds), the
// dot partials in float per warp, the cross-warp sums in double, alpha/beta
// as float quotients (the reference rounds them to the solve dtype,
// numba_impl.py:234-247).  The local CG
// is an inexact smoother whose dot order already differs from the
// reference's, so solver parity is tolerance based (tests/test_solver_gpu.py)
// -- the bit-exact B1 kernel-table path keeps the CTA kernels below.
// ---------------------------------------------------------------------------
constexpr int RW = 8;           // rows per warp
constexpr int NWJ = 4;          // warps per job
constexpr int NTJ = NWJ * 32;   // threads per job

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// The local CG of one (block, channel) job (numba_impl.py:188-251) on
// registers: res[] (in: r, out: final residual), v[] (out: correction), the
// mask / validity bit words of the warp's 8 rows and the unmasked flags of
// the rows just above / below the band.  Returns the iteration count.
template <bool UNIT_H>
__device__ __forceinline__ long cg_rows(float (&res)[RW], float (&v)[RW], uint32_t mb,
                                        uint32_t vb, float fm_up, float fm_dn, int y0, int x0,
                                        int bh, int bw, int H, int W, float closure,
                                        float inv_h2, double tau, long cap, int j, int w,
                                        float (*er_top)[32], float (*er_bot)[32],
                                        double* red_a, double* red_b) {
  long it;
  const bool lf_in = j > 0, rt_in = j < bw - 1;
  const float lf = lf_in ? 1.0f : 0.0f, rt = rt_in ? 1.0f : 0.0f;
  const int gx = x0 + j;
  // Branch-free operator (numba_impl.py:196-226 semantics):
  //   (A p)_i = dgp_i * p_i - fm_i * sum_{in-block nbrs k} fm_k p_k
  // fm = 1 on valid unmasked pixels, else 0.  dgp = the Robin-closed local
  // diagonal (in-block neighbours count 1, block sides inside the image
  // 1 - gamma) on unmasked pixels, 1 on masked pixels (identity rows),
  // 0 outside the block; invalid pixels keep p = r = 0 throughout.
  float fm[RW], dgp[RW];
#pragma unroll
  for (int s = 0; s < RW; ++s) {
    const int i = w * RW + s, gy = y0 + i;
    float d = 0.0f;
    if (gy > 0) d += i > 0 ? 1.0f : closure;
    if (gy < H - 1) d += i < bh - 1 ? 1.0f : closure;
    if (gx > 0) d += lf_in ? 1.0f : closure;
    if (gx < W - 1) d += rt_in ? 1.0f : closure;
    const bool valid = (vb >> s) & 1u, masked = (mb >> s) & 1u;
    fm[s] = valid && !masked ? 1.0f : 0.0f;
    dgp[s] = !valid ? 0.0f : (masked ? 1.0f : d * inv_h2);
  }
  float p[RW], ap[RW];
  float rs_f = 0.0f;
#pragma unroll
  for (int s = 0; s < RW; ++s) {
    p[s] = res[s];
    v[s] = 0.0f;
    rs_f = __fmaf_rn(res[s], res[s], rs_f);
  }
  er_top[w][j] = res[0];
  er_bot[w][j] = res[RW - 1];
  const float rsw = warp_sum_f(rs_f);
  if (j == 0) red_a[w] = (double)rsw;
  __syncthreads();
  double rs = 0.0;
#pragma unroll
  for (int q = 0; q < NWJ; ++q) rs += red_a[q];
  // p of the row above / below this warp's band (owned by warps w-1 / w+1)
  float pu = w > 0 ? er_bot[w - 1][j] : 0.0f;
  float pd = w < NWJ - 1 ? er_top[w + 1][j] : 0.0f;
  it = 0;
  while (rs > tau && it < cap) {
    float q[RW];
#pragma unroll
    for (int s = 0; s < RW; ++s) q[s] = p[s] * fm[s];
    const float qu = pu * fm_up, qd = pd * fm_dn;
    float pap_f = 0.0f;
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      const float ql = __shfl_up_sync(0xFFFFFFFFu, q[s], 1);
      const float qr = __shfl_down_sync(0xFFFFFFFFu, q[s], 1);
      const float up = s > 0 ? q[s - 1] : qu;
      const float dn = s < RW - 1 ? q[s + 1] : qd;
      // lane-edge neighbours enter with weight 0 (lf / rt are 0 or 1, so the
      // fused multiply-add is an exact add where they are 1)
      const float acc = __fmaf_rn(qr, rt, __fmaf_rn(ql, lf, up + dn));
      const float fa = fm[s] * acc;
      const float a = __fmaf_rn(dgp[s], p[s], UNIT_H ? -fa : -(fa * inv_h2));
      ap[s] = a;
      pap_f = __fmaf_rn(p[s], a, pap_f);
    }
    const float pw = warp_sum_f(pap_f);
    if (j == 0) red_b[w] = (double)pw;
    __syncthreads();
    double pap = 0.0;
#pragma unroll
    for (int q2 = 0; q2 < NWJ; ++q2) pap += red_b[q2];
    if (pap <= 0.0) break;
    const float alpha = (float)rs / (float)pap;
    float rsn_f = 0.0f;
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      v[s] = __fmaf_rn(alpha, p[s], v[s]);
      res[s] = __fmaf_rn(-alpha, ap[s], res[s]);
      rsn_f = __fmaf_rn(res[s], res[s], rsn_f);
    }
    er_top[w][j] = res[0];
    er_bot[w][j] = res[RW - 1];
    const float rw = warp_sum_f(rsn_f);
    if (j == 0) red_a[w] = (double)rw;
    __syncthreads();
    double rsn = 0.0;
#pragma unroll
    for (int q2 = 0; q2 < NWJ; ++q2) rsn += red_a[q2];
    const float beta = (float)rsn / (float)rs;
    rs = rsn;
#pragma unroll
    for (int s = 0; s < RW; ++s) p[s] = __fmaf_rn(beta, p[s], res[s]);
    // the neighbours' new edge directions, rebuilt bit-identically
    if (w > 0) pu = __fmaf_rn(beta, pu, er_bot[w - 1][j]);
    if (w < NWJ - 1) pd = __fmaf_rn(beta, pd, er_top[w + 1][j]);
    ++it;
  }
  return it;
}

template <bool UNIT_H>
__global__ void __launch_bounds__(NTJ, 7) k_oras_rows(
    const float* __restrict__ r, const uint8_t* __restrict__ m,
    const double* __restrict__ tau_src, double tau_scale, const int* __restrict__ ys,
    const int* __restrict__ xs, int nbx, int bh, int bw, int H, int W, int stride,
    float closure, long cap, float inv_h2, const float* __restrict__ weights,
    float* __restrict__ corr, const int* __restrict__ active, int corr_nb, size_t ps) {
  __shared__ float er_top[NWJ][32], er_bot[NWJ][32];  // edge rows of r (new)
  __shared__ double red_a[NWJ], red_b[NWJ];
  // corr_nb: blocks per channel plane of `corr` (a row-strip view launches a
  // sub-range of the level's blocks, `weights` / `corr` offset to its first)
  const int bi = blockIdx.x, ch = blockIdx.y, C = gridDim.y;
  const int nb = corr_nb > 0 ? corr_nb : (int)gridDim.x;
  const int tile = blockIdx.z;
  if (active && !active[tile]) return;
  const int j = threadIdx.x & 31, w = threadIdx.x >> 5, i0 = w * RW;
  const int kyb = bi / nbx, kxb = bi - kyb * nbx;
  const int y0 = stride > 0 ? block_start(kyb, stride, H, bh) : ys[kyb];
  const int x0 = stride > 0 ? block_start(kxb, stride, W, bw) : xs[kxb];
  const size_t plane = ps;  // channel-plane stride (row-strip views: the level's)
  const float* rc = r + ((size_t)tile * C + ch) * plane;
  const uint8_t* mt = m + (size_t)tile * plane;
  const bool lane_ok = j < bw;
  const int gx = x0 + j;

  // ---- load the job: residual rows, mask bits (own rows + the row above
  // and below the warp's band), validity
  // branch-free: every row is loaded from a clamped (valid) address and the
  // invalid ones are zeroed afterwards, so the 8 + 8 loads issue back to
  // back (a branch per row serialises their DRAM latencies)
  float res[RW];
  uint8_t mk[RW];
  uint32_t mb = 0, vb = 0;
  const int jc = lane_ok ? j : bw - 1;
#pragma unroll
  for (int s = 0; s < RW; ++s) {
    const int ic = min(i0 + s, bh - 1);
    const size_t g = (size_t)(y0 + ic) * W + (x0 + jc);
    res[s] = rc[g];
    mk[s] = mt[g];
  }
#pragma unroll
  for (int s = 0; s < RW; ++s) {
    const bool ok = i0 + s < bh && lane_ok;
    res[s] = ok ? res[s] : 0.0f;
    if (ok) {
      vb |= 1u << s;
      if (mk[s]) mb |= 1u << s;
    }
  }
  const bool has_up = i0 > 0 && i0 - 1 < bh && lane_ok;
  const bool has_dn = i0 + RW < bh && lane_ok;
  // neighbour rows outside the warp's band: 1 if they exist in the block and
  // are unmasked (their q = p * fm feeds this band's stencil)
  const float fm_up =
      has_up && !mt[(size_t)(y0 + i0 - 1) * W + gx] ? 1.0f : 0.0f;
  const float fm_dn =
      has_dn && !mt[(size_t)(y0 + i0 + RW) * W + gx] ? 1.0f : 0.0f;
  const double tau = tau_scale * tau_src[(size_t)tile * C + ch];
  float v[RW];
  const long it = cg_rows<UNIT_H>(res, v, mb, vb, fm_up, fm_dn, y0, x0, bh, bw, H, W, closure,
                                  inv_h2, tau, cap, j, w, er_top, er_bot, red_a, red_b);
  float* out = corr + (((size_t)tile * C + ch) * nb + bi) * (size_t)(bh * bw);
  const float* wb = weights + (size_t)bi * bh * bw;
#pragma unroll
  for (int s = 0; s < RW; ++s) {
    const int i = i0 + s;
    if ((vb >> s) & 1u) out[i * bw + j] = wb[i * bw + j] * v[s];
  }
  if (threadIdx.x == 0 && g_stats_on) {
    atomicAdd(&g_oras_stats[0], 1ull);
    atomicAdd(&g_oras_stats[1], (unsigned long long)it);
    if (it == 0) atomicAdd(&g_oras_stats[2], 1ull);
    atomicMax(&g_oras_stats[3], (unsigned long long)it);
  }
}

// ---------------------------------------------------------------------------
// One WARP per (block, channel, tile) job (sp_oras_variant 4): lane j owns
// column j and all 32 rows of the block in registers, so the local CG needs
// no shared memory and no barrier at all -- up/down neighbours are adjacent
// registers, left/right one shuffle each, and the dots are warp reductions.
// A CTA holds 4 independent jobs (consecutive blocks).
//
// The arithmetic is bit-identical to k_oras_rows: the same per-pixel fused
// operations, the dot partials accumulated in float over the same 8-row
// groups (rows 8g..8g+7, one accumulator per group -- which also gives the
// chain 4-way ILP), each group reduced over the 32 lanes by the same xor
// butterfly (done for the 4 groups at once by the transpose trick: 6
// shuffles instead of 20; IEEE addition is commutative, so every pair sum
// is the one the butterfly forms) and the 4 group sums added in double in
// group order.  tests/test_solver_gpu.py checks the two kernels agree
// bitwise.
// ---------------------------------------------------------------------------
constexpr int WJ = 4;  // jobs (warps) per CTA

// CGK: 0 = warp_cg32 (reference-ordered), 1 = warp_cg32_fast, 2 = warp_cg32_pair
template <bool UNIT_H, bool FULLH, int WJ, int CGK = 0>
__global__ void __launch_bounds__(WJ * 32, 12 / WJ) k_oras_warp(
    const float* __restrict__ r, const uint8_t* __restrict__ m,
    const double* __restrict__ tau_src, double tau_scale, const int* __restrict__ ys,
    const int* __restrict__ xs, int nbx, int nbl, int bh, int bw, int H, int W, int stride,
    float closure, long cap, float inv_h2, const float* __restrict__ weights,
    float* __restrict__ corr, const int* __restrict__ active, int corr_nb, size_t ps,
    const int* __restrict__ wdelta, const uint32_t* __restrict__ offbits,
    const int* __restrict__ tile_list) {
  pdl_enter();
  // FULLH: a full 32 x 32 block (bh == bw == 32): compile-time row / column
  // offsets in the job's loads and stores
  constexpr int R = 32;
  if (FULLH) {
    bh = 32;
    bw = 32;
  }
  const int j = threadIdx.x & 31;
  const int bi = blockIdx.x * WJ + (threadIdx.x >> 5), ch = blockIdx.y, C = gridDim.y;
  // tile_list: the grid covers only the listed tiles (a compacted active set)
  const int tile = tile_list ? tile_list[blockIdx.z] : blockIdx.z;
  if (bi >= nbl) return;
  if (active && !active[tile]) return;
  const int nb = corr_nb > 0 ? corr_nb : nbl;
  const int kyb = bi / nbx, kxb = bi - kyb * nbx;
  const int y0 = stride > 0 ? block_start(kyb, stride, H, bh) : ys[kyb];
  const int x0 = stride > 0 ? block_start(kxb, stride, W, bw) : xs[kxb];
  const bool lane_ok = FULLH || j < bw;
  const int jc = lane_ok ? j : bw - 1, gx = x0 + j;
  // the lane's column in row 0 of the block; rows follow at stride W
  const float* rp = r + ((size_t)tile * C + ch) * ps + (size_t)y0 * W + (x0 + jc);
  const uint8_t* mp = m + (size_t)tile * ps + (size_t)y0 * W + (x0 + jc);

  // ---- load the job (branch-free, clamped addresses; invalid zeroed)
  float res[R];
  // off: bit s set where row s is masked or outside the block (q = 0 there,
  // and A p = p, which is 0 outside the block)
  uint32_t off = 0;
  constexpr bool FAST = CGK > 0;
  if (FAST && offbits) {
    // the precomputed row-mask word of the lane's column (oras_offbits_launch)
    off = offbits[((size_t)tile * nbl + bi) * 32 + j];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int ic = FULLH ? s : min(s, bh - 1);
      res[s] = rp[ic * W];
    }
#pragma unroll
    for (int s = 0; s < R; ++s) res[s] = ((off >> s) & 1u) ? 0.0f : res[s];
  } else {
    uint8_t mk[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int ic = FULLH ? s : min(s, bh - 1);
      res[s] = rp[ic * W];
      mk[s] = mp[ic * W];
    }
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const bool ok = (FULLH || s < bh) && lane_ok;
      // FAST: the residual is 0 on masked pixels anyway (u = b~ there, so
      // r = b~ - u = 0); zeroing it makes p = q exact for warp_cg32_fast
      res[s] = (FAST ? ok && !mk[s] : ok) ? res[s] : 0.0f;
      if (!ok || mk[s]) off |= 1u << s;
    }
  }
  // Robin-closed diagonal of the three row classes (k_oras_rows' float
  // addition order): top row, interior rows, bottom row
  auto diag_of = [&](int i) {
    const int gy = y0 + i;
    float d = 0.0f;
    if (gy > 0) d += i > 0 ? 1.0f : closure;
    if (gy < H - 1) d += i < bh - 1 ? 1.0f : closure;
    if (gx > 0) d += j > 0 ? 1.0f : closure;
    if (gx < W - 1) d += j < bw - 1 ? 1.0f : closure;
    return d * inv_h2;
  };
  const float dtop = diag_of(0), dmid = diag_of(1), dbot = diag_of(bh - 1);
  const float lf = j > 0 ? 1.0f : 0.0f, rt = j < bw - 1 ? 1.0f : 0.0f;
  const double tau = tau_scale * tau_src[(size_t)tile * C + ch];

  float v[R];
  const long it =
      CGK == 2 ? warp_cg32_pair<UNIT_H, FULLH>(res, v, off, dtop, dmid, dbot, lf, rt, inv_h2,
                                               bh, tau, cap)
      : FAST   ? warp_cg32_fast<UNIT_H, FULLH>(res, v, off, dtop, dmid, dbot, lf, rt, inv_h2, bh,
                                             tau, cap)
               : warp_cg32<UNIT_H, FULLH>(res, v, off, dtop, dmid, dbot, lf, rt, inv_h2, bh, tau,
                                      cap, j);
  float* out = corr + (((size_t)tile * C + ch) * nb + bi) * (size_t)(bh * bw) + j;
  // interior blocks read the one shared weight pattern (bit-identical values)
  const long wb_i = (long)bi + (wdelta ? wdelta[bi] : 0);
  const float* wb = weights + wb_i * bh * bw + j;
  if (lane_ok) {
#pragma unroll
    for (int s = 0; s < R; ++s)
      if (FULLH || s < bh) out[s * bw] = wb[s * bw] * v[s];
  }
  if (j == 0 && g_stats_on) {
    atomicAdd(&g_oras_stats[0], 1ull);
    atomicAdd(&g_oras_stats[1], (unsigned long long)it);
    if (it == 0) atomicAdd(&g_oras_stats[2], 1ull);
    atomicMax(&g_oras_stats[3], (unsigned long long)it);
  }
}

template <typename T, int PPT>
__global__ void __launch_bounds__(NT) k_oras_local(
    const T* __restrict__ r, const uint8_t* __restrict__ m,
    const double* __restrict__ tau_src, double tau_scale, const int* __restrict__ ys,
    const int* __restrict__ xs, int nbx, int bh, int bw, int H, int W, double gamma,
    long cap, double inv_h2, const T* __restrict__ weights, T* __restrict__ corr,
    const int* __restrict__ active) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ps = reinterpret_cast<T*>(smem_raw);
  __shared__ double red0[NT / 32], red1[NT / 32], red2[NT / 32];
  const int bi = blockIdx.x, ch = blockIdx.y, C = gridDim.y, nb = gridDim.x;
  const int tile = blockIdx.z;
  if (active && !active[tile]) return;
  const int y0 = ys[bi / nbx], x0 = xs[bi % nbx];
  const int npx = bh * bw;
  const size_t plane = (size_t)H * W;
  const T* rc = r + ((size_t)tile * C + ch) * plane;
  m += (size_t)tile * plane;
  uint8_t* ms = reinterpret_cast<uint8_t*>(ps + npx);

  T res[PPT], v[PPT], p[PPT], ap[PPT];
  double diag[PPT];
  unsigned flags[PPT];  // bit0 valid, bit1 masked, bits4..7 in-block unmasked nbr
  // stage the mask (one byte per pixel) and issue every residual load first
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int k = threadIdx.x + s * NT;
    res[s] = (T)0;
    if (k < npx) {
      const int i = k / bw, j = k - i * bw;
      const size_t g = (size_t)(y0 + i) * W + (x0 + j);
      ms[k] = m[g];
      res[s] = rc[g];
    }
  }
  __syncthreads();
  double rs_part = 0.0;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int k = threadIdx.x + s * NT;
    flags[s] = 0;
    v[s] = p[s] = ap[s] = (T)0;
    diag[s] = 0.0;
    if (k < npx) {
      const int i = k / bw, j = k - i * bw;
      const int gy = y0 + i, gx = x0 + j;
      unsigned f = 1u;
      if (ms[k]) f |= 2u;
      // Robin-closed local diagonal (numba_impl.py:196-226): in-block
      // neighbours count 1, image-interior block sides 1 - gamma
      double d = 0.0;
      if (gy > 0) {
        if (i > 0) { d += 1.0; if (!ms[k - bw]) f |= 16u; } else d += 1.0 - gamma;
      }
      if (gy < H - 1) {
        if (i < bh - 1) { d += 1.0; if (!ms[k + bw]) f |= 32u; } else d += 1.0 - gamma;
      }
      if (gx > 0) {
        if (j > 0) { d += 1.0; if (!ms[k - 1]) f |= 64u; } else d += 1.0 - gamma;
      }
      if (gx < W - 1) {
        if (j < bw - 1) { d += 1.0; if (!ms[k + 1]) f |= 128u; } else d += 1.0 - gamma;
      }
      flags[s] = f;
      diag[s] = d;
      p[s] = res[s];
      rs_part += (double)res[s] * (double)res[s];
    }
  }
  double rs = cta_sum<NT>(rs_part, red0);
  const double tau = tau_scale * tau_src[(size_t)tile * C + ch];
  long it = 0;
  int phase = 0;
  while (rs > tau && it < cap) {
#pragma unroll
    for (int s = 0; s < PPT; ++s)
      if (flags[s] & 1u) ps[threadIdx.x + s * NT] = p[s];
    __syncthreads();
    double pap_part = 0.0;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      const unsigned f = flags[s];
      if (!(f & 1u)) continue;
      T a;
      if (f & 2u) {
        a = p[s];
      } else {
        const int k = threadIdx.x + s * NT;
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
    const double pap = cta_sum<NT>(pap_part, phase ? red2 : red1);
    if (pap <= 0.0) break;
    const T alpha = (T)(rs / pap);
    double rsn_part = 0.0;
#pragma unroll
    for (int s = 0; s < PPT; ++s) {
      if (!(flags[s] & 1u)) continue;
      v[s] = v[s] + alpha * p[s];
      res[s] = res[s] - alpha * ap[s];
      rsn_part += (double)res[s] * (double)res[s];
    }
    const double rsn = cta_sum<NT>(rsn_part, phase ? red1 : red2);
    const T beta = (T)(rsn / rs);
    rs = rsn;
#pragma unroll
    for (int s = 0; s < PPT; ++s)
      if (flags[s] & 1u) p[s] = res[s] + beta * p[s];
    ++it;
    phase ^= 1;
  }
  T* out = corr + (((size_t)tile * C + ch) * nb + bi) * (size_t)npx;
  const T* wb = weights + (size_t)bi * npx;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int k = threadIdx.x + s * NT;
    if (flags[s] & 1u) out[k] = wb[k] * v[s];
  }
}

// partition-of-unity weight of each covering block of pixel (x, y), in
// block order (<= 3x3); fully unrolled so the arrays stay in registers
__device__ __forceinline__ void pou_weights(int x, int y, const int* __restrict__ ys,
                                            const int* __restrict__ xs, int ky0, int nky,
                                            int kx0, int nkx, int bh, int bw, int H, int W,
                                            int overlap, double wv[9]) {
  const double big = (double)(H > W ? H : W);
  const int last = (nky - 1) * 3 + (nkx - 1);
  double raw[9], total = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int a = q / 3, b = q % 3;
    raw[q] = 0.0;
    if (a < nky && b < nkx) {
      int yb = ys[ky0 + a], xb = xs[kx0 + b];
      double ii = (double)(y - yb), jj = (double)(x - xb);
      double di = big;
      if (yb > 0) di = fmin(di, ii);
      if (yb + bh < H) di = fmin(di, (double)(bh - 1) - ii);
      if (xb > 0) di = fmin(di, jj);
      if (xb + bw < W) di = fmin(di, (double)(bw - 1) - jj);
      raw[q] = fmin(di + 1.0, (double)overlap);
      total += raw[q];
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int a = q / 3, b = q % 3;
    wv[q] = 0.0;
    if (a < nky && b < nkx) {
      double wn = (q == last) ? 1.0 - acc : raw[q] / total;
      acc += wn;
      wv[q] = wn;
    }
  }
}

template <typename T>
__global__ void k_block_weights(T* __restrict__ weights, const int* __restrict__ ys,
                                const int* __restrict__ xs, const int* __restrict__ row_k0,
                                const int* __restrict__ row_n, const int* __restrict__ col_k0,
                                const int* __restrict__ col_n, int nbx, int bh, int bw, int H,
                                int W, int overlap) {
  const int bi = blockIdx.y;
  const int npx = bh * bw;
  const int ky = bi / nbx, kx = bi % nbx;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < npx; k += gridDim.x * blockDim.x) {
    const int i = k / bw, j = k - i * bw;
    const int y = ys[ky] + i, x = xs[kx] + j;
    const int ky0 = row_k0[y], nky = row_n[y], kx0 = col_k0[x], nkx = col_n[x];
    double wv[9];
    pou_weights(x, y, ys, xs, ky0, nky, kx0, nkx, bh, bw, H, W, overlap, wv);
    const int q = (ky - ky0) * 3 + (kx - kx0);
    double w = 0.0;
#pragma unroll
    for (int t = 0; t < 9; ++t)
      if (t == q) w = wv[t];
    weights[(size_t)bi * npx + k] = (T)w;
  }
}

// u += sum over covering blocks (block order) of the weighted corrections.
// grid (nbx_cta, ntile): a thread owns one pixel of the tile's plane and
// ALL C channels, so the covering-block lookup (<= 3 x 3 blocks, normally
// 1-4) and the per-block offsets are computed once per pixel, not per
// channel.  The blocks are visited in ascending block index (row-major
// ky, kx), exactly the reference's sequential blend order.
template <typename T, int CM>
__global__ void __launch_bounds__(256) k_oras_blend(
    T* __restrict__ u, const T* __restrict__ corr, const int* __restrict__ ys,
    const int* __restrict__ xs, const int* __restrict__ row_k0,
    const int* __restrict__ row_n, const int* __restrict__ col_k0,
    const int* __restrict__ col_n, int nby, int nbx, int bh, int bw, int H, int W, int Cdyn,
    const int* __restrict__ active, int corr_nb, size_t ps) {
  pdl_enter();
  const int C = CM > 0 ? CM : Cdyn;
  const int tile = blockIdx.y;
  if (active && !active[tile]) return;
  const int nb = corr_nb > 0 ? corr_nb : nby * nbx;
  const size_t plane = ps, npx = (size_t)bh * bw, cplane = (size_t)nb * npx;
  T* ut = u + (size_t)tile * C * plane;
  const T* ct = corr + (size_t)tile * C * cplane;
  constexpr int CC = CM > 0 ? CM : 4;
  // a CTA tile is 32 x 16 pixels: each thread blends rows y and y + 8, and
  // issues all corrections of both pixels (<= 2 x 2 covering blocks each, the
  // regular case) before adding them, for memory-level parallelism
  const int ntx = (W + 31) / 32, nty = (H + 15) / 16, per = ntx * nty;
  for (int t = blockIdx.x; t < per; t += gridDim.x) {
    const int x = (t % ntx) * 32 + threadIdx.x;
    if (x >= W) continue;
    const int kx0 = col_k0[x], nkx = col_n[x];
    const int xo0 = x - xs[kx0], xo1 = nkx > 1 ? x - xs[kx0 + 1] : 0;
    int yv[2], ky0[2], nky[2];
    bool ok[2];
    bool regular = nkx <= 2;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      yv[h2] = (t / ntx) * 16 + threadIdx.y + 8 * h2;
      ok[h2] = yv[h2] < H;
      ky0[h2] = ok[h2] ? row_k0[yv[h2]] : 0;
      nky[h2] = ok[h2] ? row_n[yv[h2]] : 0;
      regular = regular && nky[h2] <= 2;
    }
    if (regular) {
      // every load of both pixels first (u and the <= 2 x 2 corrections per
      // channel), then the sums in block order and the stores
      size_t off[2][4];
      bool on[2][4];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = q >> 1, b2 = q & 1;
          on[h2][q] = ok[h2] && a < nky[h2] && b2 < nkx;
          const int ky = ky0[h2] + (on[h2][q] ? a : 0), kx = kx0 + (on[h2][q] ? b2 : 0);
          off[h2][q] = ((size_t)ky * nbx + kx) * npx + (size_t)(yv[h2] - ys[ky]) * bw +
                       (b2 ? xo1 : xo0);
        }
      T uu[2][CC], v[2][4][CC];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int c = 0; c < CC; ++c)
          uu[h2][c] = (ok[h2] && c < C) ? ut[(size_t)c * plane + (size_t)yv[h2] * W + x] : (T)0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < CC; ++c)
            v[h2][q][c] = (on[h2][q] && c < C) ? ct[(size_t)c * cplane + off[h2][q]] : (T)0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (!ok[h2]) continue;
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          if (c >= C) continue;
          T acc = uu[h2][c];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (on[h2][q]) acc = acc + v[h2][q][c];
          ut[(size_t)c * plane + (size_t)yv[h2] * W + x] = acc;
        }
      }
      continue;
    }
    // three covering blocks in a row or column (a pulled-in last block)
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (!ok[h2]) continue;
      const int y = yv[h2];
      const size_t k = (size_t)y * W + x;
      T acc[CC];
#pragma unroll
      for (int c = 0; c < CC; ++c)
        if (c < C) acc[c] = ut[(size_t)c * plane + k];
      for (int a = 0; a < nky[h2]; ++a) {
        const int ky = ky0[h2] + a;
        const size_t rowoff = (size_t)ky * nbx * npx + (size_t)(y - ys[ky]) * bw;
        for (int b2 = 0; b2 < nkx; ++b2) {
          const int kx = kx0 + b2;
          const size_t off = rowoff + (size_t)kx * npx + (size_t)(x - xs[kx]);
#pragma unroll
          for (int c = 0; c < CC; ++c)
            if (c < C) acc[c] = acc[c] + ct[(size_t)c * cplane + off];
        }
      }
#pragma unroll
      for (int c = 0; c < CC; ++c)
        if (c < C) ut[(size_t)c * plane + k] = acc[c];
    }
  }
}

// The common float case (C = 3, 32 x 32 blocks, planes < 2^31 elements):
// the same gather in the same block order as k_oras_blend, with 32-bit
// offsets and per-row / per-column block coordinates computed once, so a
// pixel costs ~50 instructions instead of ~130 (64-bit offset arithmetic).
__global__ void __launch_bounds__(256) k_oras_blend3(
    float* __restrict__ u, const float* __restrict__ corr, const int* __restrict__ ys,
    const int* __restrict__ xs, const int* __restrict__ row_k0, const int* __restrict__ row_n,
    const int* __restrict__ col_k0, const int* __restrict__ col_n, int nbx, int H, int W,
    const int* __restrict__ active, int nb, size_t ps) {
  pdl_enter();
  const int tile = blockIdx.y;
  if (active && !active[tile]) return;
  const int plane = (int)ps, cplane = nb * 1024;
  float* ut = u + (size_t)tile * 3 * ps;
  const float* ct = corr + (size_t)tile * 3 * (size_t)cplane;
  const int ntx = (W + 31) >> 5, nty = (H + 15) >> 4, per = ntx * nty;
  for (int t = blockIdx.x; t < per; t += gridDim.x) {
    const int ty = t / ntx;
    const int x = (t - ty * ntx) * 32 + threadIdx.x;
    if (x >= W) continue;
    const int kx0 = col_k0[x], nkx = col_n[x];
    const int xo0 = x - xs[kx0], xo1 = nkx > 1 ? x - xs[kx0 + 1] : 0;
    int yv[2], ky0[2], nky[2];
    bool ok[2];
    bool regular = nkx <= 2;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      yv[h2] = ty * 16 + threadIdx.y + 8 * h2;
      ok[h2] = yv[h2] < H;
      ky0[h2] = ok[h2] ? row_k0[yv[h2]] : 0;
      nky[h2] = ok[h2] ? row_n[yv[h2]] : 0;
      regular = regular && nky[h2] <= 2;
    }
    if (regular) {
      int off[2][4];
      bool on[2][4];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int yo0 = yv[h2] - ys[ky0[h2]];
        const int yo1 = nky[h2] > 1 ? yv[h2] - ys[ky0[h2] + 1] : 0;
        const int b00 = (ky0[h2] * nbx + kx0) * 1024;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = q >> 1, b2 = q & 1;
          on[h2][q] = ok[h2] && a < nky[h2] && b2 < nkx;
          off[h2][q] = on[h2][q] ? b00 + (a ? nbx * 1024 : 0) + (b2 ? 1024 : 0) +
                                       (a ? yo1 : yo0) * 32 + (b2 ? xo1 : xo0)
                                 : 0;
        }
      }
      float uu[2][3], v[2][4][3];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          uu[h2][c] = ok[h2] ? ut[c * plane + yv[h2] * W + x] : 0.0f;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            v[h2][q][c] = on[h2][q] ? ct[c * cplane + off[h2][q]] : 0.0f;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (!ok[h2]) continue;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float acc = uu[h2][c];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (on[h2][q]) acc = acc + v[h2][q][c];
          ut[c * plane + yv[h2] * W + x] = acc;
        }
      }
      continue;
    }
    // three covering blocks in a row or column (a pulled-in last block)
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (!ok[h2]) continue;
      const int y = yv[h2], k = y * W + x;
      float acc[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = ut[c * plane + k];
      for (int a = 0; a < nky[h2]; ++a) {
        const int ky = ky0[h2] + a;
        const int rowoff = ky * nbx * 1024 + (y - ys[ky]) * 32;
        for (int b2 = 0; b2 < nkx; ++b2) {
          const int kx = kx0 + b2;
          const int o = rowoff + kx * 1024 + (x - xs[kx]);
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[c] = acc[c] + ct[c * cplane + o];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) ut[c * plane + k] = acc[c];
    }
  }
}

// k_oras_blend3 with the per-row / per-column cover data packed into one
// word each at hierarchy build (blend_pack: k0 | two << 16 | three << 17 |
// o0 << 18 | o1 << 24): one table load per row and per column instead of the
// dependent cover-table -> block-start chains (ncu: the blend stalls 54 % on
// long scoreboards).  Rows or columns with three covering blocks take the
// generic path.  Same gather, same block order: bit-identical.
__global__ void __launch_bounds__(256) k_oras_blend3p(
    float* __restrict__ u, const float* __restrict__ corr, const int* __restrict__ ys,
    const int* __restrict__ xs, const int* __restrict__ row_k0, const int* __restrict__ row_n,
    const int* __restrict__ col_k0, const int* __restrict__ col_n,
    const int* __restrict__ rowinfo, const int* __restrict__ colinfo, int nbx, int H, int W,
    const int* __restrict__ active, int nb, size_t ps) {
  pdl_enter();
  const int tile = blockIdx.y;
  if (active && !active[tile]) return;
  const int plane = (int)ps, cplane = nb * 1024;
  float* ut = u + (size_t)tile * 3 * ps;
  const float* ct = corr + (size_t)tile * 3 * (size_t)cplane;
  const int ntx = (W + 31) >> 5, nty = (H + 15) >> 4, per = ntx * nty;
  for (int t = blockIdx.x; t < per; t += gridDim.x) {
    const int ty = t / ntx;
    const int x = (t - ty * ntx) * 32 + threadIdx.x;
    if (x >= W) continue;
    const int ci = colinfo[x];
    int yv[2], ri[2];
    bool ok[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      yv[h2] = ty * 16 + threadIdx.y + 8 * h2;
      ok[h2] = yv[h2] < H;
      ri[h2] = ok[h2] ? rowinfo[yv[h2]] : 0;
    }
    if (((ci | ri[0] | ri[1]) >> 17) & 1) {
      // a row or column with three covering blocks (a pulled-in last block)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (!ok[h2]) continue;
        const int y = yv[h2], k = y * W + x;
        float acc[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = ut[c * plane + k];
        for (int a = 0; a < row_n[y]; ++a) {
          const int ky = row_k0[y] + a;
          const int rowoff = ky * nbx * 1024 + (y - ys[ky]) * 32;
          for (int b2 = 0; b2 < col_n[x]; ++b2) {
            const int kx = col_k0[x] + b2;
            const int o = rowoff + kx * 1024 + (x - xs[kx]);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = acc[c] + ct[c * cplane + o];
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) ut[c * plane + k] = acc[c];
      }
      continue;
    }
    const int kx0 = ci & 0xFFFF, xo0 = (ci >> 18) & 63, dxo = ((ci >> 24) & 63) - xo0;
    const bool twox = (ci >> 16) & 1;
    int off[2][4];
    bool on[2][4];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = ri[h2];
      const int ky0 = r & 0xFFFF, yo0 = (r >> 18) & 63, dyo = ((r >> 24) & 63) - yo0;
      const bool twoy = (r >> 16) & 1;
      const int b00 = (ky0 * nbx + kx0) * 1024 + yo0 * 32 + xo0;
      off[h2][0] = b00;
      off[h2][1] = b00 + 1024 + dxo;
      off[h2][2] = b00 + nbx * 1024 + dyo * 32;
      off[h2][3] = off[h2][2] + 1024 + dxo;
      on[h2][0] = ok[h2];
      on[h2][1] = ok[h2] && twox;
      on[h2][2] = ok[h2] && twoy;
      on[h2][3] = ok[h2] && twox && twoy;
    }
    float uu[2][3], v[2][4][3];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        uu[h2][c] = ok[h2] ? ut[c * plane + yv[h2] * W + x] : 0.0f;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          v[h2][q][c] = on[h2][q] ? ct[c * cplane + off[h2][q]] : 0.0f;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (!ok[h2]) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float acc = uu[h2][c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (on[h2][q]) acc = acc + v[h2][q][c];
        ut[c * plane + yv[h2] * W + x] = acc;
      }
    }
  }
}

// k_oras_blend3q's path for a pixel pair on a row or column with three
// covering blocks (a pulled-in last block), out of line so the common path
// keeps its compact code: the cover tables, then the block starts, then each
// block row's corrections load as independent batches (a loop of chained
// table -> start -> correction loads costs several us per launch on the
// small levels)
__device__ __noinline__ void blend3q_generic(float* __restrict__ ut, const float* __restrict__ ct,
                                             const int* __restrict__ ys,
                                             const int* __restrict__ xs,
                                             const int* __restrict__ row_k0,
                                             const int* __restrict__ row_n,
                                             const int* __restrict__ col_k0,
                                             const int* __restrict__ col_n, int nbx, int W,
                                             int plane, int cplane, int x, int y) {
  const int nc = col_n[x], c0 = col_k0[x];
  const int nr = row_n[y], r0 = row_k0[y];
  int xsb[3], ysb[3];
#pragma unroll
  for (int b2 = 0; b2 < 3; ++b2) xsb[b2] = b2 < nc ? xs[c0 + b2] : 0;
#pragma unroll
  for (int a2 = 0; a2 < 3; ++a2) ysb[a2] = a2 < nr ? ys[r0 + a2] : 0;
  const int k = y * W + x;
  float2 acc[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) acc[c] = *reinterpret_cast<const float2*>(ut + c * plane + k);
#pragma unroll
  for (int a2 = 0; a2 < 3; ++a2) {
    if (a2 >= nr) break;
    const int rowoff = (r0 + a2) * nbx * 1024 + (y - ysb[a2]) * 32;
    float2 v[3][3];
#pragma unroll
    for (int b2 = 0; b2 < 3; ++b2)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        v[b2][c] = b2 < nc ? *reinterpret_cast<const float2*>(ct + c * cplane + rowoff +
                                                              (c0 + b2) * 1024 + (x - xsb[b2]))
                           : make_float2(0.0f, 0.0f);
#pragma unroll
    for (int b2 = 0; b2 < 3; ++b2) {
      if (b2 >= nc) break;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        acc[c].x = acc[c].x + v[b2][c].x;
        acc[c].y = acc[c].y + v[b2][c].y;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) *reinterpret_cast<float2*>(ut + c * plane + k) = acc[c];
}

// k_oras_blend3p on column PAIRS (x, x + 1), x even: with every block
// start even and W even (stride 26 at every level of the default
// decomposition) a pair never straddles a block edge, so both pixels have
// the same covering blocks and their offsets in them differ by one -- every
// u and correction access is one 8-byte load or store for two pixels, half
// the address arithmetic of the per-pixel kernel (which is ALU-bound: ncu
// 66 % ALU pipe).  Same gather, same block order, same float adds:
// bit-identical.  Tiles of 64 x 16 pixels.
template <int R>
__global__ void __launch_bounds__(256, R == 1 ? 4 : 2) k_oras_blend3q(
    float* __restrict__ u, const float* __restrict__ corr, const int* __restrict__ ys,
    const int* __restrict__ xs, const int* __restrict__ row_k0, const int* __restrict__ row_n,
    const int* __restrict__ col_k0, const int* __restrict__ col_n,
    const int* __restrict__ rowinfo, const int* __restrict__ colinfo, int nbx, int H, int W,
    const int* __restrict__ active, int nb, size_t ps) {
  pdl_enter();
  const int tile = blockIdx.y;
  if (active && !active[tile]) return;
  const int plane = (int)ps, cplane = nb * 1024;
  float* ut = u + (size_t)tile * 3 * ps;
  const float* ct = corr + (size_t)tile * 3 * (size_t)cplane;
  const int ntx = (W + 63) >> 6, nty = (H + 8 * R - 1) / (8 * R), per = ntx * nty;
  for (int t = blockIdx.x; t < per; t += gridDim.x) {
    const int ty = t / ntx;
    const int x = (t - ty * ntx) * 64 + 2 * threadIdx.x;
    if (x >= W) continue;
    const int ci = colinfo[x];
    int yv[R], ri[R];
    bool ok[R];
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2) {
      yv[h2] = ty * 8 * R + threadIdx.y + 8 * h2;
      ok[h2] = yv[h2] < H;
      ri[h2] = ok[h2] ? rowinfo[yv[h2]] : 0;
    }
    int rall = 0;
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2) rall |= ri[h2];
    if (((ci | rall) >> 17) & 1) {
      // a row or column with three covering blocks (a pulled-in last block)
#pragma unroll
      for (int h2 = 0; h2 < R; ++h2)
        if (ok[h2])
          blend3q_generic(ut, ct, ys, xs, row_k0, row_n, col_k0, col_n, nbx, W, plane, cplane,
                          x, yv[h2]);
      continue;
    }
    const int kx0 = ci & 0xFFFF, xo0 = (ci >> 18) & 63, dxo = ((ci >> 24) & 63) - xo0;
    const bool twox = (ci >> 16) & 1;
    int off[R][4];
    bool on[R][4];
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2) {
      const int r = ri[h2];
      const int ky0 = r & 0xFFFF, yo0 = (r >> 18) & 63, dyo = ((r >> 24) & 63) - yo0;
      const bool twoy = (r >> 16) & 1;
      const int b00 = (ky0 * nbx + kx0) * 1024 + yo0 * 32 + xo0;
      off[h2][0] = b00;
      off[h2][1] = b00 + 1024 + dxo;
      off[h2][2] = b00 + nbx * 1024 + dyo * 32;
      off[h2][3] = off[h2][2] + 1024 + dxo;
      on[h2][0] = ok[h2];
      on[h2][1] = ok[h2] && twox;
      on[h2][2] = ok[h2] && twoy;
      on[h2][3] = ok[h2] && twox && twoy;
    }
    float2 uu[R][3], v[R][4][3];
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        uu[h2][c] = ok[h2] ? *reinterpret_cast<const float2*>(ut + c * plane + yv[h2] * W + x)
                           : make_float2(0.0f, 0.0f);
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          v[h2][q][c] = on[h2][q] ? *reinterpret_cast<const float2*>(ct + c * cplane + off[h2][q])
                                  : make_float2(0.0f, 0.0f);
#pragma unroll
    for (int h2 = 0; h2 < R; ++h2) {
      if (!ok[h2]) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float2 acc = uu[h2][c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (on[h2][q]) {
            acc.x = acc.x + v[h2][q][c].x;
            acc.y = acc.y + v[h2][q][c].y;
          }
        *reinterpret_cast<float2*>(ut + c * plane + yv[h2] * W + x) = acc;
      }
    }
  }
}

// generic channel count (C > 4): one channel plane per grid row
template <typename T>
__global__ void __launch_bounds__(256) k_oras_blend_plane(
    T* __restrict__ u, const T* __restrict__ corr, const int* __restrict__ ys,
    const int* __restrict__ xs, const int* __restrict__ row_k0,
    const int* __restrict__ row_n, const int* __restrict__ col_k0,
    const int* __restrict__ col_n, int nby, int nbx, int bh, int bw, int H, int W, int C,
    const int* __restrict__ active, int corr_nb, size_t ps) {
  pdl_enter();
  const int z = blockIdx.y, tile = z / C;
  if (active && !active[tile]) return;
  const int nb = corr_nb > 0 ? corr_nb : nby * nbx;
  const size_t plane = ps, npx = (size_t)bh * bw;
  T* uc = u + (size_t)z * plane;
  const T* cc = corr + (size_t)z * nb * npx;
  const int ntx = (W + 31) / 32, nty = (H + 7) / 8, per = ntx * nty;
  for (int t = blockIdx.x; t < per; t += gridDim.x) {
    const int x = (t % ntx) * 32 + threadIdx.x, y = (t / ntx) * 8 + threadIdx.y;
    if (x >= W || y >= H) continue;
    const int ky0 = row_k0[y], nky = row_n[y], kx0 = col_k0[x], nkx = col_n[x];
    const size_t k = (size_t)y * W + x;
    T uv = uc[k];
    for (int a = 0; a < nky; ++a) {
      const int ky = ky0 + a;
      for (int b2 = 0; b2 < nkx; ++b2) {
        const int kx = kx0 + b2;
        uv = uv + cc[(size_t)(ky * nbx + kx) * npx + (size_t)(y - ys[ky]) * bw + (x - xs[kx])];
      }
    }
    uc[k] = uv;
  }
}

}  // namespace

template <typename T>
int oras_local_launch(const T* r, const uint8_t* m, const double* tau_src, double tau_scale,
                      const int* ys, const int* xs, int nby, int nbx, int bh, int bw, int H,
                      int W, int C, double gamma, long cap, double inv_h2, const T* weights,
                      T* corr, cudaStream_t s, int ntile, const int* active, int stride,
                      int corr_nb, size_t ps, const int* wdelta, const uint32_t* offbits,
                      const int* tile_list, int nlist) {
  if (tile_list && !(sizeof(T) == 4 && bw <= 32 && bh <= 32 && oras_kernel >= 6)) {
    set_error("tile lists need the one-warp float ORAS kernel");
    return -2;
  }
  const int npx = bh * bw;
  if (ps && ps != (size_t)H * W &&
      !(sizeof(T) == 4 && bw <= 32 && bh <= 32 &&
        (oras_kernel == 0 || oras_kernel == 2 || oras_kernel == 4 || oras_kernel >= 6))) {
    set_error("plane-strided ORAS launches need the float 32x32 4-warp kernel");
    return -2;
  }
  if (!ps) ps = (size_t)H * W;
  if (corr_nb > 0 && !(sizeof(T) == 4 && bw <= 32 && bh <= 32 && oras_kernel != 1)) {
    set_error("block sub-range launches need the float 32x32 ORAS kernel");
    return -2;
  }
  dim3 grid(nby * nbx, C, ntile);
  size_t sm = (size_t)npx * sizeof(T) + (size_t)npx;  // p staging + mask bytes
  if (sizeof(T) == 4 && bw <= 32 && bh <= 32 &&
      (oras_kernel == 4 || oras_kernel >= 6)) {
    const int nbl = nby * nbx;
    const bool unit = inv_h2 == 1.0, full = bh == 32 && bw == 32;
    // 4: four jobs per CTA; 6: one job per CTA (a finished job frees its
    // slot at once instead of waiting for the CTA's slowest job); 7: 6 with
    // the lean local CG (warp_cg32_fast); 8: on packed float pairs
    // (warp_cg32_pair)
    const int wj = oras_kernel == 4 ? WJ : 1;
    dim3 g4(cdiv(nbl, wj), C, tile_list ? nlist : ntile);
#define SP_WARP(WJN, F)                                                                   \
  (unit ? (full ? k_oras_warp<true, true, WJN, F> : k_oras_warp<true, false, WJN, F>)     \
        : (full ? k_oras_warp<false, true, WJN, F> : k_oras_warp<false, false, WJN, F>))
    auto kern = oras_kernel == 8   ? SP_WARP(1, 2)
                : oras_kernel == 7 ? SP_WARP(1, 1)
                                   : (wj == 1 ? SP_WARP(1, 0) : SP_WARP(WJ, 0));
#undef SP_WARP
    if (oras_kernel >= 7) {
      SP_CUDA(launch_k(kern, g4, dim3(wj * 32), 0, s, (const float*)r, m, tau_src, tau_scale, ys,
                       xs, nbx, nbl, bh, bw, H, W, stride, (float)(1.0 - gamma), cap,
                       (float)inv_h2, (const float*)weights, (float*)corr, active, corr_nb, ps,
                       wdelta, corr_nb > 0 || !offbits_on ? nullptr : offbits, tile_list));
    } else {
      kern<<<g4, wj * 32, 0, s>>>((const float*)r, m, tau_src, tau_scale, ys, xs, nbx, nbl, bh,
                                  bw, H, W, stride, (float)(1.0 - gamma), cap, (float)inv_h2,
                                  (const float*)weights, (float*)corr, active, corr_nb, ps,
                                  wdelta, nullptr, nullptr);
    }
  } else if (sizeof(T) == 4 && bw <= 32 && bh <= 32 && oras_kernel != 1) {
    auto kern = inv_h2 == 1.0 ? k_oras_rows<true> : k_oras_rows<false>;
    kern<<<grid, NTJ, 0, s>>>((const float*)r, m, tau_src, tau_scale, ys, xs, nbx, bh, bw, H,
                              W, stride, (float)(1.0 - gamma), cap, (float)inv_h2,
                              (const float*)weights, (float*)corr, active, corr_nb, ps);
  } else if (bw == 32 && bh <= 32) {
    k_oras_local32<T><<<grid, NT, 0, s>>>(r, m, tau_src, tau_scale, ys, xs, nbx, bh, H, W,
                                          stride, gamma, cap, inv_h2, weights, corr, active);
  } else if (npx <= NT * 4) {
    k_oras_local<T, 4><<<grid, NT, sm, s>>>(r, m, tau_src, tau_scale, ys, xs, nbx, bh, bw, H,
                                            W, gamma, cap, inv_h2, weights, corr, active);
  } else if (npx <= NT * 16) {
    auto kern = k_oras_local<T, 16>;
    if (sm > 48 * 1024)
      SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, NT, sm, s>>>(r, m, tau_src, tau_scale, ys, xs, nbx, bh, bw, H, W, gamma, cap,
                              inv_h2, weights, corr, active);
  } else {
    set_error("oras block of %d pixels exceeds the 4096-pixel kernel limit", npx);
    return -2;
  }
  SP_CHECK_LAUNCH();
  return 0;
}

// host: packed cover words of sorted block starts (k_oras_blend3p); false
// when a block offset does not fit
bool blend_pack(const std::vector<int>& starts, int size, int dim, std::vector<int>& info) {
  info.assign(dim, 0);
  for (int y = 0; y < dim; ++y) {
    int k0 = -1, n = 0;
    for (size_t k = 0; k < starts.size(); ++k)
      if (starts[k] <= y && y < starts[k] + size) {
        if (k0 < 0) k0 = (int)k;
        ++n;
      }
    if (n < 1 || k0 > 0xFFFF) return false;
    if (n > 2) {  // generic path
      info[y] = 1 << 17;
      continue;
    }
    const int o0 = y - starts[k0], o1 = n > 1 ? y - starts[k0 + 1] : o0;
    if (o0 > 63 || o1 > 63) return false;
    info[y] = k0 | ((n - 1) << 16) | (o0 << 18) | (o1 << 24);
  }
  return true;
}

// 2 (default): column pairs (k_oras_blend3q, one row per thread, 63
// registers) where they fit, else 1; 3: pairs with two rows per thread (107
// registers, 2 CTAs per SM).  4K finest blend: 1 = 73.6 us (0.73 of HBM),
// 3 = 67.5 us, 2 = 61.7 us (0.87); pipeline -5 ms.
static int blend_packed_on = 2;
int blend_packed(int v) {
  if (v >= 0) blend_packed_on = v;
  return blend_packed_on;
}

template <typename T>
int oras_blend_launch(T* u, const T* corr, const int* ys, const int* xs, const int* row_k0,
                      const int* row_n, const int* col_k0, const int* col_n, int nby, int nbx,
                      int bh, int bw, int H, int W, int C, cudaStream_t s, int ntile,
                      const int* active, int corr_nb, size_t ps, const int* rowinfo,
                      const int* colinfo, bool pair_cols) {
  if (!ps) ps = (size_t)H * W;
  long per = (long)cdiv(W, 32) * cdiv(H, C <= 4 ? 16 : 8);
  long nz = C <= 4 ? (long)ntile : (long)ntile * C;
  long nbx_cta = (2L * 148 * 8 + nz - 1) / nz;
  if (nbx_cta > per) nbx_cta = per;
  if (nbx_cta < 1) nbx_cta = 1;
  dim3 grid((unsigned)nbx_cta, (unsigned)nz), blk(32, 8);
#define SP_BLEND(CM)                                                                      \
  SP_CUDA(launch_k(k_oras_blend<T, CM>, grid, blk, 0, s, u, corr, ys, xs, row_k0, row_n,    \
                   col_k0, col_n, nby, nbx, bh, bw, H, W, C, active, corr_nb, ps))
  const long nbt = (long)(corr_nb > 0 ? corr_nb : nby * nbx);
  const bool b3 = C == 3 && sizeof(T) == 4 && bh == 32 && bw == 32 && 3 * ps < (1UL << 31) &&
                  3 * nbt * 1024 < (1L << 31);
  if (C == 1) SP_BLEND(1);
  else if (b3 && rowinfo && colinfo && blend_packed_on >= 2 && pair_cols) {
    const int blend_rows = blend_packed_on == 3 ? 2 : 1;
    const long perq = (long)cdiv(W, 64) * cdiv(H, 8 * blend_rows);
    dim3 gq((unsigned)std::min<long>(grid.x, perq), grid.y);
    SP_CUDA(launch_k(blend_rows == 1 ? k_oras_blend3q<1> : k_oras_blend3q<2>, gq, blk, 0, s, (float*)u, (const float*)corr, ys, xs,
                     row_k0, row_n, col_k0, col_n, rowinfo, colinfo, nbx, H, W, active,
                     (int)nbt, ps));
  } else if (b3 && rowinfo && colinfo && blend_packed_on)
    SP_CUDA(launch_k(k_oras_blend3p, grid, blk, 0, s, (float*)u, (const float*)corr, ys, xs,
                     row_k0, row_n, col_k0, col_n, rowinfo, colinfo, nbx, H, W, active,
                     (int)nbt, ps));
  else if (b3)
    SP_CUDA(launch_k(k_oras_blend3, grid, blk, 0, s, (float*)u, (const float*)corr, ys, xs,
                     row_k0, row_n, col_k0, col_n, nbx, H, W, active, (int)nbt, ps));
  else if (C == 3) SP_BLEND(3);
  else if (C <= 4) SP_BLEND(0);
  else
    SP_CUDA(launch_k(k_oras_blend_plane<T>, grid, blk, 0, s, u, corr, ys, xs, row_k0, row_n,
                     col_k0, col_n, nby, nbx, bh, bw, H, W, C, active, corr_nb, ps));
#undef SP_BLEND
  SP_CHECK_LAUNCH();
  return 0;
}

// offbits[tile][b][j]: bit s = pixel (ys[ky] + s, xs[kx] + j) masked, or
// row s / column j outside the bh x bw block -- the ORAS job's `off` word
__global__ void __launch_bounds__(256) k_offbits(const uint8_t* __restrict__ m,
                                                 const int* __restrict__ ys,
                                                 const int* __restrict__ xs, int nb, int nbx,
                                                 int bh, int bw, int H, int W,
                                                 uint32_t* __restrict__ offbits) {
  // one warp per block, lane = column; the 32 row bytes are loaded first
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5), tile = blockIdx.y, j = threadIdx.x & 31;
  if (b >= nb) return;
  const int ky = b / nbx, kx = b - ky * nbx;
  uint32_t off = 0xFFFFFFFFu;
  if (j < bw) {
    const uint8_t* mp = m + (size_t)tile * H * W + (size_t)ys[ky] * W + xs[kx] + j;
    uint8_t mk[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) mk[s] = mp[(size_t)min(s, bh - 1) * W];
    off = 0;
#pragma unroll
    for (int s = 0; s < 32; ++s)
      if (s >= bh || mk[s]) off |= 1u << s;
  }
  offbits[((size_t)tile * nb + b) * 32 + j] = off;
}

int oras_offbits_launch(const uint8_t* m, const int* ys, const int* xs, int nby, int nbx, int bh,
                        int bw, int H, int W, int ntile, uint32_t* offbits, cudaStream_t s) {
  const int nb = nby * nbx;
  k_offbits<<<dim3(cdiv(nb, 8), ntile), 256, 0, s>>>(m, ys, xs, nb, nbx, bh, bw, H, W, offbits);
  SP_CHECK_LAUNCH();
  return 0;
}

// wdelta[b] = cb - b when block b's weights equal block cb's bit for bit
// (cb: the interior block (1, 1)), else 0
__global__ void k_weight_alias(const float* __restrict__ w, int npx, int cb,
                               int* __restrict__ wdelta) {
  const int b = blockIdx.x;
  __shared__ int diff;
  if (threadIdx.x == 0) diff = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < npx; i += blockDim.x)
    if (__float_as_uint(w[(size_t)b * npx + i]) != __float_as_uint(w[(size_t)cb * npx + i]))
      diff = 1;
  __syncthreads();
  if (threadIdx.x == 0) wdelta[b] = diff ? 0 : cb - b;
}

int weight_aliases(const float* weights, int nby, int nbx, int bh, int bw, int* wdelta,
                   cudaStream_t s) {
  const int nb = nby * nbx;
  if (nby < 3 || nbx < 3) return cudaMemsetAsync(wdelta, 0, sizeof(int) * nb, s) == cudaSuccess
                                     ? 0 : (set_error("wdelta memset failed"), -1);
  k_weight_alias<<<nb, 256, 0, s>>>(weights, bh * bw, nbx + 1, wdelta);
  SP_CHECK_LAUNCH();
  return 0;
}

template <typename T>
int block_weights_launch(T* weights, const int* ys, const int* xs, const int* row_k0,
                         const int* row_n, const int* col_k0, const int* col_n, int nby,
                         int nbx, int bh, int bw, int H, int W, int overlap, cudaStream_t s) {
  const int npx = bh * bw;
  dim3 grid(cdiv(npx, 256), nby * nbx);
  k_block_weights<T><<<grid, 256, 0, s>>>(weights, ys, xs, row_k0, row_n, col_k0, col_n, nbx,
                                          bh, bw, H, W, overlap);
  SP_CHECK_LAUNCH();
  return 0;
}

#define INST(T)                                                                            \
  template int oras_local_launch<T>(const T*, const uint8_t*, const double*, double,        \
                                    const int*, const int*, int, int, int, int, int, int,   \
                                    int, double, long, double, const T*, T*, cudaStream_t,  \
                                    int, const int*, int, int, size_t, const int*,          \
                                    const uint32_t*, const int*, int);                      \
  template int oras_blend_launch<T>(T*, const T*, const int*, const int*, const int*,       \
                                    const int*, const int*, const int*, int, int, int, int, \
                                    int, int, int, cudaStream_t, int, const int*, int,      \
                                    size_t, const int*, const int*, bool);                  \
  template int block_weights_launch<T>(T*, const int*, const int*, const int*, const int*,  \
                                       const int*, const int*, int, int, int, int, int,     \
                                       int, int, cudaStream_t);
INST(float)
INST(double)

}  // namespace sp
