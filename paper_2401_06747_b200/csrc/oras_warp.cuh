// oras_warp.cuh -- the ORAS local CG of one 32x32 block job on ONE warp
// (numba_impl.py:188-251 semantics; see k_oras_warp in oras.cu for the
// design and the arithmetic contract).  Shared by the global ORAS sweep
// (oras.cu) and the fused on-chip tile solver (tilesolve.cu).
#pragma once
#include "common.cuh"

namespace sp {

// the xor-butterfly sums of x[0..3] over the warp, all four in every lane
__device__ __forceinline__ void warp_sum4(const float (&x)[4], float (&t)[4], int j) {
  const bool hi16 = j & 16, hi8 = j & 8;
  // o = 16: keep groups {0,1} (low half) or {2,3} (high half)
  const float s0 = hi16 ? x[0] : x[2], s1 = hi16 ? x[1] : x[3];
  const float k0 = hi16 ? x[2] : x[0], k1 = hi16 ? x[3] : x[1];
  const float y0 = k0 + __shfl_xor_sync(0xFFFFFFFFu, s0, 16);
  const float y1 = k1 + __shfl_xor_sync(0xFFFFFFFFu, s1, 16);
  // o = 8: keep the first or second of the pair
  const float sd = hi8 ? y0 : y1, kp = hi8 ? y1 : y0;
  float z = kp + __shfl_xor_sync(0xFFFFFFFFu, sd, 8);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) z += __shfl_xor_sync(0xFFFFFFFFu, z, o);
  // lanes 0 / 8 / 16 / 24 hold the totals of groups 0 / 1 / 2 / 3
#pragma unroll
  for (int g = 0; g < 4; ++g) t[g] = __shfl_sync(0xFFFFFFFFu, z, 8 * g);
}

__device__ __forceinline__ double sum4_double(const float (&t)[4]) {
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < 4; ++g) s += (double)t[g];
  return s;
}

// Local CG on the block held in registers: lane j = column j, res[s] = row s
// (in: the block residual, out: the final local residual), v (out: the
// local correction).  off bit s: row s masked or outside the block.  dtop /
// dmid / dbot: the Robin-closed diagonal (times inv_h2) of the top, interior
// and bottom rows; lf / rt: 1 where the lane has an in-block left / right
// neighbour.  Stops on rs <= tau or after cap steps or on pap <= 0.
// Returns the number of CG steps.
template <bool UNIT_H, bool FULLH>
__device__ __forceinline__ long warp_cg32(float (&res)[32], float (&v)[32], uint32_t off,
                                          float dtop, float dmid, float dbot, float lf,
                                          float rt, float inv_h2, int bh, double tau, long cap,
                                          int j) {
  constexpr int R = 32;
  float p[R], ap[R];
#pragma unroll
  for (int s = 0; s < R; ++s) v[s] = 0.0f;
  float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f}, t4[4];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    p[s] = res[s];
    acc4[s >> 3] = __fmaf_rn(res[s], res[s], acc4[s >> 3]);
  }
  warp_sum4(acc4, t4, j);
  double rs = sum4_double(t4);
  long it = 0;
  while (rs > tau && it < cap) {
    float q[R];
#pragma unroll
    for (int s = 0; s < R; ++s) q[s] = ((off >> s) & 1u) ? 0.0f : p[s];
#pragma unroll
    for (int g = 0; g < 4; ++g) acc4[g] = 0.0f;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const float ql = __shfl_up_sync(0xFFFFFFFFu, q[s], 1);
      const float qr = __shfl_down_sync(0xFFFFFFFFu, q[s], 1);
      const float up = s > 0 ? q[s - 1] : 0.0f;
      const float dn = s < R - 1 ? q[s + 1] : 0.0f;
      const float acc = __fmaf_rn(qr, rt, __fmaf_rn(ql, lf, up + dn));
      float dg;
      if (FULLH) dg = s == 0 ? dtop : (s == R - 1 ? dbot : dmid);
      else dg = s == 0 ? dtop : (s == bh - 1 ? dbot : dmid);
      const float a = __fmaf_rn(dg, p[s], UNIT_H ? -acc : -(acc * inv_h2));
      ap[s] = ((off >> s) & 1u) ? p[s] : a;
      acc4[s >> 3] = __fmaf_rn(p[s], ap[s], acc4[s >> 3]);
    }
    warp_sum4(acc4, t4, j);
    const double pap = sum4_double(t4);
    if (pap <= 0.0) break;
    const float alpha = (float)rs / (float)pap;
#pragma unroll
    for (int g = 0; g < 4; ++g) acc4[g] = 0.0f;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      v[s] = __fmaf_rn(alpha, p[s], v[s]);
      res[s] = __fmaf_rn(-alpha, ap[s], res[s]);
      acc4[s >> 3] = __fmaf_rn(res[s], res[s], acc4[s >> 3]);
    }
    warp_sum4(acc4, t4, j);
    const double rsn = sum4_double(t4);
    const float beta = (float)rsn / (float)rs;
    rs = rsn;
#pragma unroll
    for (int s = 0; s < R; ++s) p[s] = __fmaf_rn(beta, p[s], res[s]);
    ++it;
  }
  return it;
}

// sum of a0..a3 over the warp, in every lane: ((a0 + a1) + (a2 + a3)), then
// one xor butterfly in float.  The closing broadcast of lane 0 makes the
// result provably warp-uniform, so the CG loop's exit tests stay uniform
// branches (without it the compiler wraps every shuffle of the loop in
// WARPSYNC / collective fix-up code).
__device__ __forceinline__ float warp_sum_f(float a0, float a1, float a2, float a3) {
  float x = (a0 + a1) + (a2 + a3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  return __shfl_sync(0xFFFFFFFFu, x, 0);
}

// The same local CG with a leaner instruction stream (the default kernel,
// sp_oras_variant 7).  Differences from warp_cg32, all below the float
// rounding of the vectors themselves:
//   - q = p: the caller zeroes the residual on `off` rows (masked or outside
//     the block), so p, v and the residual stay exactly 0 there and only the
//     operator row needs the select (A p = p = 0 on those rows);
//   - dots: four interleaved float accumulators per lane (rows s mod 4),
//     combined pairwise, one float xor butterfly, compared in double;
//   - alpha = rs / pap and beta = rs' / rs by the fast float division (the
//     reference rounds both to the vector dtype, numba_impl.py:234-247).
// Stop rule, cap, breakdown test and the update order are warp_cg32's.
template <bool UNIT_H, bool FULLH>
__device__ __forceinline__ long warp_cg32_fast(float (&res)[32], float (&v)[32], uint32_t off,
                                               float dtop, float dmid, float dbot, float lf,
                                               float rt, float inv_h2, int bh, double tau,
                                               long cap) {
  constexpr int R = 32;
  float p[R], ap[R];
  float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
  for (int s = 0; s < R; s += 4) {
    v[s] = v[s + 1] = v[s + 2] = v[s + 3] = 0.0f;
    p[s] = res[s];
    p[s + 1] = res[s + 1];
    p[s + 2] = res[s + 2];
    p[s + 3] = res[s + 3];
    a0 = __fmaf_rn(res[s], res[s], a0);
    a1 = __fmaf_rn(res[s + 1], res[s + 1], a1);
    a2 = __fmaf_rn(res[s + 2], res[s + 2], a2);
    a3 = __fmaf_rn(res[s + 3], res[s + 3], a3);
  }
  float rs = warp_sum_f(a0, a1, a2, a3);
  long it = 0;
  while ((double)rs > tau && it < cap) {
    float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const float ql = __shfl_up_sync(0xFFFFFFFFu, p[s], 1);
      const float qr = __shfl_down_sync(0xFFFFFFFFu, p[s], 1);
      const float up = s > 0 ? p[s - 1] : 0.0f;
      const float dn = s < R - 1 ? p[s + 1] : 0.0f;
      const float acc = __fmaf_rn(qr, rt, __fmaf_rn(ql, lf, up + dn));
      float dg;
      if (FULLH) dg = s == 0 ? dtop : (s == R - 1 ? dbot : dmid);
      else dg = s == 0 ? dtop : (s == bh - 1 ? dbot : dmid);
      const float a = __fmaf_rn(dg, p[s], UNIT_H ? -acc : -(acc * inv_h2));
      ap[s] = ((off >> s) & 1u) ? 0.0f : a;
      acc4[s & 3] = __fmaf_rn(p[s], ap[s], acc4[s & 3]);
    }
    const float pap = warp_sum_f(acc4[0], acc4[1], acc4[2], acc4[3]);
    if (pap <= 0.0f) break;
    const float alpha = __fdividef(rs, pap);
#pragma unroll
    for (int g = 0; g < 4; ++g) acc4[g] = 0.0f;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      v[s] = __fmaf_rn(alpha, p[s], v[s]);
      res[s] = __fmaf_rn(-alpha, ap[s], res[s]);
      acc4[s & 3] = __fmaf_rn(res[s], res[s], acc4[s & 3]);
    }
    const float rsn = warp_sum_f(acc4[0], acc4[1], acc4[2], acc4[3]);
    const float beta = __fdividef(rsn, rs);
    rs = rsn;
#pragma unroll
    for (int s = 0; s < R; ++s) p[s] = __fmaf_rn(beta, p[s], res[s]);
    ++it;
  }
  return it;
}

// warp_sum_f over eight float chains held as four pairs: pairwise FADD2s,
// the two halves, one xor butterfly.  No closing broadcast: at every level
// lanes i and i ^ o add the same two operands (IEEE addition commutes), so
// all lanes hold the same bits; the CG's exit tests vote on them
// (__all_sync / __any_sync) to give the compiler its uniform branches, which
// takes a shuffle latency off each of the step's two reductions.
__device__ __forceinline__ float warp_sum_f2(const float2 (&d)[4]) {
  const float2 t = __fadd2_rn(__fadd2_rn(d[0], d[1]), __fadd2_rn(d[2], d[3]));
  float x = t.x + t.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  return x;
}

// The lean local CG on packed float pairs (sp_oras_variant 8): the lane's
// 32 rows live as 16 register pairs {row k, row k + 16}, so every vector
// update, the operator and the dots run as FFMA2 / FADD2 (two IEEE float
// operations per instruction, each rounded exactly like the scalar one) --
// the kernel is issue-bound and this halves its floating-point instruction
// count.  The {k, k + 16} pairing keeps the vertical neighbours aligned: the
// rows above / below pair k are pairs k - 1 / k + 1 (two seam pairs are
// assembled from halves).  Same arithmetic as warp_cg32_fast per pixel; the
// dots accumulate rows {k mod 4} x {low, high half} in eight float chains
// (4 rows each: FFMA2 chains stall on their latency), combined pairwise.
template <bool UNIT_H, bool FULLH>
__device__ __forceinline__ long warp_cg32_pair(float (&res)[32], float (&v)[32], uint32_t off,
                                               float dtop, float dmid, float dbot, float lf,
                                               float rt, float inv_h2, int bh, double tau,
                                               long cap) {
  constexpr int K = 16;
  float2 r2[K], p2[K], v2[K], ap2[K];
  float2 d4[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) d4[g] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    r2[k] = make_float2(res[k], res[k + K]);
    p2[k] = r2[k];
    v2[k] = make_float2(0.0f, 0.0f);
    d4[k & 3] = __ffma2_rn(r2[k], r2[k], d4[k & 3]);
  }
  float rs = warp_sum_f2(d4);
  const float2 lf2 = make_float2(lf, lf), rt2 = make_float2(rt, rt);
  const float2 ih2 = make_float2(inv_h2, inv_h2);
  long it = 0;
  while (__all_sync(0xFFFFFFFFu, (double)rs > tau) && it < cap) {
#pragma unroll
    for (int g = 0; g < 4; ++g) d4[g] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float2 ql = make_float2(__shfl_up_sync(0xFFFFFFFFu, p2[k].x, 1),
                                    __shfl_up_sync(0xFFFFFFFFu, p2[k].y, 1));
      const float2 qr = make_float2(__shfl_down_sync(0xFFFFFFFFu, p2[k].x, 1),
                                    __shfl_down_sync(0xFFFFFFFFu, p2[k].y, 1));
      const float2 up = k > 0 ? p2[k - 1] : make_float2(0.0f, p2[K - 1].x);
      const float2 dn = k < K - 1 ? p2[k + 1] : make_float2(p2[0].y, 0.0f);
      const float2 acc = __ffma2_rn(qr, rt2, __ffma2_rn(ql, lf2, __fadd2_rn(up, dn)));
      float2 dg;
      if (FULLH) {
        dg.x = k == 0 ? dtop : dmid;
        dg.y = k == K - 1 ? dbot : dmid;
      } else {
        dg.x = k == 0 ? dtop : (k == bh - 1 ? dbot : dmid);
        dg.y = k + K == bh - 1 ? dbot : dmid;
      }
      const float2 sc = UNIT_H ? acc : __fmul2_rn(acc, ih2);
      const float2 a = __ffma2_rn(dg, p2[k], make_float2(-sc.x, -sc.y));
      ap2[k].x = ((off >> k) & 1u) ? 0.0f : a.x;
      ap2[k].y = ((off >> (k + K)) & 1u) ? 0.0f : a.y;
      d4[k & 3] = __ffma2_rn(p2[k], ap2[k], d4[k & 3]);
    }
    const float pap = warp_sum_f2(d4);
    if (__any_sync(0xFFFFFFFFu, pap <= 0.0f)) break;
    const float alpha = __fdividef(rs, pap);
    const float2 al2 = make_float2(alpha, alpha), nal2 = make_float2(-alpha, -alpha);
#pragma unroll
    for (int g = 0; g < 4; ++g) d4[g] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v2[k] = __ffma2_rn(al2, p2[k], v2[k]);
      r2[k] = __ffma2_rn(nal2, ap2[k], r2[k]);
      d4[k & 3] = __ffma2_rn(r2[k], r2[k], d4[k & 3]);
    }
    const float rsn = warp_sum_f2(d4);
    const float beta = __fdividef(rsn, rs);
    rs = rsn;
    const float2 be2 = make_float2(beta, beta);
#pragma unroll
    for (int k = 0; k < K; ++k) p2[k] = __ffma2_rn(be2, p2[k], r2[k]);
    ++it;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    res[k] = r2[k].x;
    res[k + K] = r2[k].y;
    v[k] = v2[k].x;
    v[k + K] = v2[k].y;
  }
  return it;
}

}  // namespace sp
