/*
 * sp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's 16-entry kernel table
 * (/root/reference/pkg/src/sparsepaint/kernels/numba_impl.py, the default
 * "numba" backend selected by kernels/__init__.py:43-66).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_2401_06747_b200) never does.
 *
 * Arithmetic follows the numba semantics exactly so that the oracle is
 * bit-identical to the reference (pinned by tests/test_oracle_golden.py
 * against fixtures produced by the reference itself, tests/golden/):
 *   - stencil accumulators are double, the result is rounded once to the
 *     storage type T (numba_impl.py:21-35, 50-64, 79-97, 111-120, 132-141);
 *   - sym_residual subtracts in T and sums squares sequentially in double
 *     (numba_impl.py:147-158);
 *   - the ORAS local CG computes dots in double and rounds alpha/beta to T,
 *     vector updates in T (numba_impl.py:161-263);
 *   - compile with -ffp-contract=off: no FMA contraction anywhere.
 * Parallel loops (OpenMP) only write disjoint memory; every floating-point
 * reduction runs in the reference's sequential order.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX3(c, y, x) (((size_t)(c) * H + (size_t)(y)) * W + (size_t)(x))
#define IDX2(y, x) ((size_t)(y) * W + (size_t)(x))

/* ---- stencil family (numba_impl.py:13-144) ------------------------------ */

#define DEF_STENCILS(T, SUF)                                                        \
  void ora_negated_laplacian_##SUF(const T *x, T *out, int C, int H, int W,        \
                                   double inv_h2) {                                \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      for (int c = 0; c < C; ++c)                                                  \
        for (int xx = 0; xx < W; ++xx) {                                           \
          double d = 0.0, a = 0.0;                                                 \
          if (y > 0) { d += 1.0; a += (double)x[IDX3(c, y - 1, xx)]; }             \
          if (y < H - 1) { d += 1.0; a += (double)x[IDX3(c, y + 1, xx)]; }         \
          if (xx > 0) { d += 1.0; a += (double)x[IDX3(c, y, xx - 1)]; }            \
          if (xx < W - 1) { d += 1.0; a += (double)x[IDX3(c, y, xx + 1)]; }        \
          out[IDX3(c, y, xx)] = (T)((d * (double)x[IDX3(c, y, xx)] - a) * inv_h2); \
        }                                                                          \
    }                                                                              \
  }                                                                                \
  void ora_inpaint_matvec_##SUF(const T *x, const uint8_t *m, T *out, int C,       \
                                int H, int W, double inv_h2) {                     \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      for (int c = 0; c < C; ++c)                                                  \
        for (int xx = 0; xx < W; ++xx) {                                           \
          if (m[IDX2(y, xx)]) { out[IDX3(c, y, xx)] = x[IDX3(c, y, xx)]; continue; } \
          double d = 0.0, a = 0.0;                                                 \
          if (y > 0) { d += 1.0; a += (double)x[IDX3(c, y - 1, xx)]; }             \
          if (y < H - 1) { d += 1.0; a += (double)x[IDX3(c, y + 1, xx)]; }         \
          if (xx > 0) { d += 1.0; a += (double)x[IDX3(c, y, xx - 1)]; }            \
          if (xx < W - 1) { d += 1.0; a += (double)x[IDX3(c, y, xx + 1)]; }        \
          out[IDX3(c, y, xx)] = (T)((d * (double)x[IDX3(c, y, xx)] - a) * inv_h2); \
        }                                                                          \
    }                                                                              \
  }                                                                                \
  void ora_sym_matvec_##SUF(const T *x, const uint8_t *m, T *out, int C, int H,    \
                            int W, double inv_h2) {                                \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      for (int c = 0; c < C; ++c)                                                  \
        for (int xx = 0; xx < W; ++xx) {                                           \
          if (m[IDX2(y, xx)]) { out[IDX3(c, y, xx)] = x[IDX3(c, y, xx)]; continue; } \
          double d = 0.0, a = 0.0;                                                 \
          if (y > 0) { d += 1.0; if (!m[IDX2(y - 1, xx)]) a += (double)x[IDX3(c, y - 1, xx)]; } \
          if (y < H - 1) { d += 1.0; if (!m[IDX2(y + 1, xx)]) a += (double)x[IDX3(c, y + 1, xx)]; } \
          if (xx > 0) { d += 1.0; if (!m[IDX2(y, xx - 1)]) a += (double)x[IDX3(c, y, xx - 1)]; } \
          if (xx < W - 1) { d += 1.0; if (!m[IDX2(y, xx + 1)]) a += (double)x[IDX3(c, y, xx + 1)]; } \
          out[IDX3(c, y, xx)] = (T)((d * (double)x[IDX3(c, y, xx)] - a) * inv_h2); \
        }                                                                          \
    }                                                                              \
  }                                                                                \
  void ora_sym_rhs_##SUF(const T *b, const uint8_t *m, T *out, int C, int H,       \
                         int W, double inv_h2) {                                   \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      for (int c = 0; c < C; ++c)                                                  \
        for (int xx = 0; xx < W; ++xx) {                                           \
          if (m[IDX2(y, xx)]) { out[IDX3(c, y, xx)] = b[IDX3(c, y, xx)]; continue; } \
          double a = 0.0;                                                          \
          if (y > 0 && m[IDX2(y - 1, xx)]) a += (double)b[IDX3(c, y - 1, xx)];     \
          if (y < H - 1 && m[IDX2(y + 1, xx)]) a += (double)b[IDX3(c, y + 1, xx)]; \
          if (xx > 0 && m[IDX2(y, xx - 1)]) a += (double)b[IDX3(c, y, xx - 1)];    \
          if (xx < W - 1 && m[IDX2(y, xx + 1)]) a += (double)b[IDX3(c, y, xx + 1)]; \
          out[IDX3(c, y, xx)] = (T)((double)b[IDX3(c, y, xx)] + a * inv_h2);       \
        }                                                                          \
    }                                                                              \
  }                                                                                \
  void ora_ct_apply_##SUF(const T *wi, const uint8_t *m, T *out, int C, int H,     \
                          int W, double inv_h2) {                                  \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      for (int c = 0; c < C; ++c)                                                  \
        for (int xx = 0; xx < W; ++xx) {                                           \
          if (!m[IDX2(y, xx)]) { out[IDX3(c, y, xx)] = (T)0; continue; }           \
          double a = 0.0;                                                          \
          if (y > 0 && !m[IDX2(y - 1, xx)]) a += (double)wi[IDX3(c, y - 1, xx)];   \
          if (y < H - 1 && !m[IDX2(y + 1, xx)]) a += (double)wi[IDX3(c, y + 1, xx)]; \
          if (xx > 0 && !m[IDX2(y, xx - 1)]) a += (double)wi[IDX3(c, y, xx - 1)];  \
          if (xx < W - 1 && !m[IDX2(y, xx + 1)]) a += (double)wi[IDX3(c, y, xx + 1)]; \
          out[IDX3(c, y, xx)] = (T)((double)wi[IDX3(c, y, xx)] + a * inv_h2);      \
        }                                                                          \
    }                                                                              \
  }                                                                                \
  /* numba_impl.py:147-158: r in T, per-channel sequential double sum */          \
  void ora_sym_residual_##SUF(const T *u, const T *bs, const uint8_t *m, T *r,     \
                              double *norms, int C, int H, int W, double inv_h2) { \
    ora_sym_matvec_##SUF(u, m, r, C, H, W, inv_h2);                                \
    size_t n = (size_t)C * H * W;                                                  \
    _Pragma("omp parallel for schedule(static)") for (long i = 0; i < (long)n; ++i) \
      r[i] = (T)(bs[i] - r[i]);                                                    \
    size_t plane = (size_t)H * W;                                                  \
    for (int c = 0; c < C; ++c) {                                                  \
      double acc = 0.0;                                                            \
      const T *rc = r + (size_t)c * plane;                                         \
      for (size_t i = 0; i < plane; ++i) acc += (double)rc[i] * (double)rc[i];     \
      norms[c] = acc;                                                              \
    }                                                                              \
  }

DEF_STENCILS(float, f32)
DEF_STENCILS(double, f64)

/* ---- ORAS sweep (numba_impl.py:161-263) --------------------------------- */

#define DEF_ORAS(T, SUF)                                                            \
  void ora_oras_apply_##SUF(T *u, const T *r, const uint8_t *m, const int64_t *xs, \
                            int nbx, const int64_t *ys, int nby, int bh, int bw,   \
                            double gamma, const double *taus, long cap,            \
                            const T *weights, double inv_h2, int C, int H, int W) { \
    long nb = (long)nbx * nby;                                                     \
    size_t bsz = (size_t)bh * bw;                                                  \
    T *corr = (T *)calloc((size_t)nb * C * bsz, sizeof(T));                        \
    _Pragma("omp parallel") {                                                      \
      T *res = (T *)malloc(bsz * sizeof(T));                                       \
      T *v = (T *)malloc(bsz * sizeof(T));                                         \
      T *p = (T *)malloc(bsz * sizeof(T));                                         \
      T *ap = (T *)malloc(bsz * sizeof(T));                                        \
      _Pragma("omp for schedule(dynamic, 4)") for (long job = 0; job < nb * C; ++job) { \
        long bi = job / C;                                                         \
        int ch = (int)(job % C);                                                   \
        long y0 = ys[bi / nbx], x0 = xs[bi % nbx];                                 \
        for (int i = 0; i < bh; ++i)                                               \
          for (int j = 0; j < bw; ++j) {                                           \
            res[i * bw + j] = r[IDX3(ch, y0 + i, x0 + j)];                         \
            v[i * bw + j] = (T)0;                                                  \
            p[i * bw + j] = res[i * bw + j];                                       \
          }                                                                        \
        double rs = 0.0;                                                           \
        for (size_t k = 0; k < bsz; ++k) rs += (double)res[k] * (double)res[k];    \
        double tau = taus[ch];                                                     \
        long it = 0;                                                               \
        while (rs > tau && it < cap) {                                             \
          for (int i = 0; i < bh; ++i) {                                           \
            long gy = y0 + i;                                                      \
            for (int j = 0; j < bw; ++j) {                                         \
              long gx = x0 + j;                                                    \
              if (m[IDX2(gy, gx)]) { ap[i * bw + j] = p[i * bw + j]; continue; }   \
              double d = 0.0, a = 0.0;                                             \
              if (gy > 0) {                                                        \
                if (i > 0) { d += 1.0; if (!m[IDX2(gy - 1, gx)]) a += (double)p[(i - 1) * bw + j]; } \
                else d += 1.0 - gamma;                                             \
              }                                                                    \
              if (gy < H - 1) {                                                    \
                if (i < bh - 1) { d += 1.0; if (!m[IDX2(gy + 1, gx)]) a += (double)p[(i + 1) * bw + j]; } \
                else d += 1.0 - gamma;                                             \
              }                                                                    \
              if (gx > 0) {                                                        \
                if (j > 0) { d += 1.0; if (!m[IDX2(gy, gx - 1)]) a += (double)p[i * bw + j - 1]; } \
                else d += 1.0 - gamma;                                             \
              }                                                                    \
              if (gx < W - 1) {                                                    \
                if (j < bw - 1) { d += 1.0; if (!m[IDX2(gy, gx + 1)]) a += (double)p[i * bw + j + 1]; } \
                else d += 1.0 - gamma;                                             \
              }                                                                    \
              ap[i * bw + j] = (T)((d * (double)p[i * bw + j] - a) * inv_h2);      \
            }                                                                      \
          }                                                                        \
          double pap = 0.0;                                                        \
          for (size_t k = 0; k < bsz; ++k) pap += (double)p[k] * (double)ap[k];    \
          if (pap <= 0.0) break;                                                   \
          T alpha = (T)(rs / pap);                                                 \
          for (size_t k = 0; k < bsz; ++k) {                                       \
            v[k] = (T)(v[k] + (T)(alpha * p[k]));                                  \
            res[k] = (T)(res[k] - (T)(alpha * ap[k]));                             \
          }                                                                        \
          double rsn = 0.0;                                                        \
          for (size_t k = 0; k < bsz; ++k) rsn += (double)res[k] * (double)res[k]; \
          T beta = (T)(rsn / rs);                                                  \
          rs = rsn;                                                                \
          for (size_t k = 0; k < bsz; ++k) p[k] = (T)(res[k] + (T)(beta * p[k]));  \
          ++it;                                                                    \
        }                                                                          \
        memcpy(corr + ((size_t)bi * C + ch) * bsz, v, bsz * sizeof(T));            \
      }                                                                            \
      free(res); free(v); free(p); free(ap);                                       \
    }                                                                              \
    /* deterministic sequential blend in block order (numba_impl.py:255-263) */   \
    for (long bi = 0; bi < nb; ++bi) {                                             \
      long y0 = ys[bi / nbx], x0 = xs[bi % nbx];                                   \
      for (int ch = 0; ch < C; ++ch)                                               \
        for (int i = 0; i < bh; ++i)                                               \
          for (int j = 0; j < bw; ++j) {                                           \
            T w = weights[(size_t)bi * bsz + (size_t)i * bw + j];                  \
            T cv = corr[((size_t)bi * C + ch) * bsz + (size_t)i * bw + j];         \
            size_t k = IDX3(ch, y0 + i, x0 + j);                                   \
            u[k] = (T)(u[k] + (T)(w * cv));                                        \
          }                                                                        \
    }                                                                              \
    free(corr);                                                                    \
  }

DEF_ORAS(float, f32)
DEF_ORAS(double, f64)

/* ---- grid transfers (numba_impl.py:266-348) ----------------------------- */

#define DEF_TRANSFERS(T, SUF)                                                       \
  void ora_restrict_values_##SUF(const T *f, T *out, int C, int H, int W) {        \
    int ch = (H + 1) / 2, cw = (W + 1) / 2;                                        \
    for (int k = 0; k < C; ++k)                                                    \
      for (int i = 0; i < ch; ++i) {                                               \
        int y1 = 2 * i + 2 < H ? 2 * i + 2 : H;                                    \
        for (int j = 0; j < cw; ++j) {                                             \
          int x1 = 2 * j + 2 < W ? 2 * j + 2 : W;                                  \
          double acc = 0.0; int cnt = 0;                                           \
          for (int y = 2 * i; y < y1; ++y)                                         \
            for (int x = 2 * j; x < x1; ++x) { acc += (double)f[IDX3(k, y, x)]; ++cnt; } \
          out[((size_t)k * ch + i) * cw + j] = (T)(acc / (double)cnt);            \
        }                                                                          \
      }                                                                            \
  }                                                                                \
  void ora_restrict_mask_##SUF(const uint8_t *m, const T *vals, uint8_t *cm,       \
                               T *cv, int C, int H, int W) {                       \
    int ch = (H + 1) / 2, cw = (W + 1) / 2;                                        \
    memset(cm, 0, (size_t)ch * cw);                                                \
    memset(cv, 0, (size_t)C * ch * cw * sizeof(T));                                \
    for (int i = 0; i < ch; ++i) {                                                 \
      int y1 = 2 * i + 2 < H ? 2 * i + 2 : H;                                      \
      for (int j = 0; j < cw; ++j) {                                               \
        int x1 = 2 * j + 2 < W ? 2 * j + 2 : W;                                    \
        int cnt = 0;                                                               \
        for (int y = 2 * i; y < y1; ++y)                                           \
          for (int x = 2 * j; x < x1; ++x) cnt += m[IDX2(y, x)] ? 1 : 0;           \
        if (!cnt) continue;                                                        \
        cm[(size_t)i * cw + j] = 1;                                                \
        for (int k = 0; k < C; ++k) {                                              \
          double acc = 0.0;                                                        \
          for (int y = 2 * i; y < y1; ++y)                                         \
            for (int x = 2 * j; x < x1; ++x)                                       \
              if (m[IDX2(y, x)]) acc += (double)vals[IDX3(k, y, x)];               \
          cv[((size_t)k * ch + i) * cw + j] = (T)(acc / (double)cnt);             \
        }                                                                          \
      }                                                                            \
    }                                                                              \
  }                                                                                \
  void ora_prolongate_##SUF(const T *co, T *out, int C, int chh, int cww, int H,   \
                            int W) {                                               \
    _Pragma("omp parallel for schedule(static)") for (int y = 0; y < H; ++y) {     \
      double fy = ((double)y + 0.5) / 2.0 - 0.5;                                   \
      long y0 = (long)floor(fy);                                                   \
      double wy = fy - (double)y0;                                                 \
      if (y0 < 0) { y0 = 0; wy = 0.0; }                                            \
      if (y0 > chh - 1) { y0 = chh - 1; wy = 0.0; }                                \
      long y1 = y0 + 1 < chh - 1 ? y0 + 1 : chh - 1;                               \
      for (int x = 0; x < W; ++x) {                                                \
        double fx = ((double)x + 0.5) / 2.0 - 0.5;                                 \
        long x0 = (long)floor(fx);                                                 \
        double wx = fx - (double)x0;                                               \
        if (x0 < 0) { x0 = 0; wx = 0.0; }                                          \
        if (x0 > cww - 1) { x0 = cww - 1; wx = 0.0; }                              \
        long x1 = x0 + 1 < cww - 1 ? x0 + 1 : cww - 1;                             \
        for (int k = 0; k < C; ++k) {                                              \
          const T *c = co + (size_t)k * chh * cww;                                 \
          double v = (1.0 - wy) * ((1.0 - wx) * (double)c[y0 * cww + x0] +         \
                                   wx * (double)c[y0 * cww + x1]) +                \
                     wy * ((1.0 - wx) * (double)c[y1 * cww + x0] +                 \
                           wx * (double)c[y1 * cww + x1]);                         \
          out[IDX3(k, y, x)] = (T)v;                                               \
        }                                                                          \
      }                                                                            \
    }                                                                              \
  }

DEF_TRANSFERS(float, f32)
DEF_TRANSFERS(double, f64)

/* ---- jump flooding (numba_impl.py:351-409) ------------------------------ */

static void jfa_pass(const int32_t *cur, int32_t *nxt, const int64_t *sy,
                     const int64_t *sx, long step, int H, int W) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int32_t best = cur[IDX2(y, x)];
      int64_t bd;
      if (best >= 0) {
        int64_t dy = y - sy[best], dx = x - sx[best];
        bd = dy * dy + dx * dx;
      } else {
        bd = (int64_t)4 * ((int64_t)H * H + (int64_t)W * W);
      }
      for (int oy = -1; oy <= 1; ++oy) {
        long ny = y + oy * step;
        if (ny < 0 || ny >= H) continue;
        for (int ox = -1; ox <= 1; ++ox) {
          if (!oy && !ox) continue;
          long nx = x + ox * step;
          if (nx < 0 || nx >= W) continue;
          int32_t cand = cur[IDX2(ny, nx)];
          if (cand < 0) continue;
          int64_t dy = y - sy[cand], dx = x - sx[cand];
          int64_t cd = dy * dy + dx * dx;
          if (cd < bd || (cd == bd && best >= 0 && cand < best)) {
            bd = cd;
            best = cand;
          }
        }
      }
      nxt[IDX2(y, x)] = best;
    }
}

void ora_jfa_run(const int32_t *labels, int32_t *out, const int64_t *seeds, long m,
                 const int64_t *steps, int nsteps, int H, int W) {
  size_t n = (size_t)H * W;
  int64_t *sy = (int64_t *)malloc((m ? m : 1) * sizeof(int64_t));
  int64_t *sx = (int64_t *)malloc((m ? m : 1) * sizeof(int64_t));
  for (long i = 0; i < m; ++i) { sy[i] = seeds[2 * i]; sx[i] = seeds[2 * i + 1]; }
  int32_t *a = (int32_t *)malloc(n * sizeof(int32_t));
  int32_t *b = (int32_t *)malloc(n * sizeof(int32_t));
  memcpy(a, labels, n * sizeof(int32_t));
  for (int s = 0; s < nsteps; ++s) {
    jfa_pass(a, b, sy, sx, (long)steps[s], H, W);
    int32_t *t = a; a = b; b = t;
  }
  memcpy(out, a, n * sizeof(int32_t));
  free(a); free(b); free(sy); free(sx);
}

void ora_jfa_dist2(const int32_t *labels, const int64_t *seeds, long m, int64_t *out, int H,
                   int W) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int32_t s = labels[IDX2(y, x)];
      if (s < 0) s += (int32_t)m;  /* numba wraparound indexing (seeds[-1]) */
      int64_t dy = (int64_t)y - seeds[2 * (int64_t)s];
      int64_t dx = (int64_t)x - seeds[2 * (int64_t)s + 1];
      out[IDX2(y, x)] = dy * dy + dx * dx;
    }
}

/* ---- Floyd-Steinberg (numba_impl.py:412-439) ---------------------------- */

void ora_fs_dither(const double *dens, uint8_t *out, int H, int W) {
  size_t n = (size_t)H * W;
  double *buf = (double *)malloc(n * sizeof(double));
  memcpy(buf, dens, n * sizeof(double));
  memset(out, 0, n);
  for (int y = 0; y < H; ++y) {
    int x0 = (y % 2 == 0) ? 0 : W - 1, x1 = (y % 2 == 0) ? W : -1;
    int sgn = (y % 2 == 0) ? 1 : -1;
    for (int x = x0; x != x1; x += sgn) {
      double val = buf[IDX2(y, x)];
      int bit = val >= 0.5 ? 1 : 0;
      out[IDX2(y, x)] = (uint8_t)bit;
      double err = val - (double)bit;
      int xn = x + sgn;
      if (xn >= 0 && xn < W) buf[IDX2(y, xn)] += err * (7.0 / 16.0);
      if (y + 1 < H) {
        int xb = x - sgn;
        if (xb >= 0 && xb < W) buf[IDX2(y + 1, xb)] += err * (3.0 / 16.0);
        buf[IDX2(y + 1, x)] += err * (5.0 / 16.0);
        if (xn >= 0 && xn < W) buf[IDX2(y + 1, xn)] += err * (1.0 / 16.0);
      }
    }
  }
  free(buf);
}

/* ---- triangle buckets (numba_impl.py:442-498) --------------------------- */

void ora_assign_triangles(const int64_t *tris, long T, const int64_t *vy,
                          const int64_t *vx, int H, int W, int32_t *assign) {
  for (size_t i = 0; i < (size_t)H * W; ++i) assign[i] = -1;
  for (long t = 0; t < T; ++t) {
    int64_t ay = vy[tris[3 * t]], ax = vx[tris[3 * t]];
    int64_t by = vy[tris[3 * t + 1]], bx = vx[tris[3 * t + 1]];
    int64_t cy = vy[tris[3 * t + 2]], cx = vx[tris[3 * t + 2]];
    int64_t ylo = ay < by ? ay : by; ylo = ylo < cy ? ylo : cy; if (ylo < 0) ylo = 0;
    int64_t yhi = ay > by ? ay : by; yhi = yhi > cy ? yhi : cy; if (yhi > H - 1) yhi = H - 1;
    int64_t xlo = ax < bx ? ax : bx; xlo = xlo < cx ? xlo : cx; if (xlo < 0) xlo = 0;
    int64_t xhi = ax > bx ? ax : bx; xhi = xhi > cx ? xhi : cx; if (xhi > W - 1) xhi = W - 1;
    for (int64_t y = ylo; y <= yhi; ++y)
      for (int64_t x = xlo; x <= xhi; ++x) {
        if (assign[IDX2(y, x)] >= 0) continue;
        int64_t e0 = (bx - ax) * (y - ay) - (by - ay) * (x - ax);
        int64_t e1 = (cx - bx) * (y - by) - (cy - by) * (x - bx);
        int64_t e2 = (ax - cx) * (y - cy) - (ay - cy) * (x - cx);
        if ((e0 >= 0 && e1 >= 0 && e2 >= 0) || (e0 <= 0 && e1 <= 0 && e2 <= 0))
          assign[IDX2(y, x)] = (int32_t)t;
      }
  }
}

void ora_fallback_assign(const int32_t *assign, const int32_t *labels,
                         const int32_t *smt, int32_t *out, int H, int W) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int32_t t = assign[IDX2(y, x)];
      if (t < 0) {
        t = smt[labels[IDX2(y, x)]];
        if (t < 0) t = 0;
      }
      out[IDX2(y, x)] = t;
    }
}

void ora_reduce_cells(const int32_t *assign, const double *err, long ntris,
                      double *sums, int64_t *amax_idx, double *amax_val, int H,
                      int W) {
  for (long t = 0; t < ntris; ++t) { sums[t] = 0.0; amax_idx[t] = -1; amax_val[t] = -1.0; }
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int32_t t = assign[IDX2(y, x)];
      double e = err[IDX2(y, x)];
      sums[t] += e;
      if (e > amax_val[t]) { amax_val[t] = e; amax_idx[t] = (int64_t)y * W + x; }
    }
}

/* thread control for the CPU baseline timings (bench.py reference arm) */
void ora_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int ora_get_threads(void) { return omp_get_max_threads(); }
