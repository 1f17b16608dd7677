// mgtma.cu -- TMA-staged stencil sweeps of the multigrid hierarchy (sm_100a).
//
// The two HBM-bound sweeps of every V-cycle on the wide float levels:
//   residual           r = b~ - A~ u, per-plane sum r^2     (numba_impl.py:147-158)
//   residual+restrict  r_H = restrict(b~ - A~ u)          (solver.py:289-291)
//
// Data movement: a CTA owns a 128-column x 64-row tile of one plane and
// streams it in 8-row chunks through a 4-stage shared-memory ring filled by
// the Tensor Memory Accelerator (cp.async.bulk.tensor.3d, one elected
// thread, completion on an mbarrier with expect_tx).  Each chunk brings the
// u rows y-1 .. y+8 with a 4-column halo (136 x 10 floats), the mask rows
// with a 16-byte halo (160 x 10 bytes) and the b rows (128 x 8 floats); the
// tensor maps are 3-D ([plane][H][W]) so the image border is the TMA
// out-of-bounds zero fill -- no edge special cases in the load path.  While
// the 8 warps compute chunk k, chunks k+1..k+3 are in flight: the memory
// level parallelism comes from the TMA engine, not from registers.
//
// Arithmetic is the reference's bit for bit (the same as mg.cu's per-pixel
// kernels): the neighbour sum in double in the order up, down, left, right,
// (d u - sum) rounded once to float, r = b - A u in float; the restriction
// averages ((a + b) + c) + d in double.  Norms: per-thread float sums, then
// double warp / CTA trees in fixed order and the last CTA of a plane adds
// the CTA partials in index order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace sp {

namespace {

constexpr int TC = 128;              // tile columns
constexpr int TR = 64;               // tile rows
constexpr int CR = 8;                // rows per chunk (= warps)
constexpr int NCH = TR / CR;         // chunks per tile
constexpr int NS = 4;                // pipeline stages
constexpr int UW = TC + 8;           // u row: 4-column halo each side
constexpr int MW = TC + 32;          // mask row: 16-byte halo each side (TMA
                                     // x coordinates must be 16-byte aligned)
constexpr int U_BYTES = UW * (CR + 2) * 4;
constexpr int M_BYTES = MW * (CR + 2);
constexpr int B_BYTES = TC * CR * 4;
constexpr int U_OFF = 0;
constexpr int M_OFF = (U_BYTES + 127) / 128 * 128;
constexpr int B_OFF = M_OFF + (M_BYTES + 127) / 128 * 128;
constexpr int STAGE = B_OFF + (B_BYTES + 127) / 128 * 128;
constexpr int SMEM = NS * STAGE + 128;
constexpr int TX_BYTES = U_BYTES + M_BYTES + B_BYTES;
// (dynamic + static shared memory exceeds the 48 KB default for MODE 1: the
// opt-in attribute is set once by tma_prepare(), outside any graph capture)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of a tensor box (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   (uint64_t)map),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

struct Maps {
  CUtensorMap u, b, m;
};

// issue the three TMA loads of chunk `ck` of the tile into stage `st`
__device__ __forceinline__ void issue_chunk(const Maps& mp, unsigned char* sm, uint64_t* bars,
                                            int st, int x0, int ychunk, int z, int tile) {
  unsigned char* base = sm + st * STAGE;
  mbar_expect_tx(&bars[st], TX_BYTES);
  tma_load_3d(base + U_OFF, &mp.u, x0 - 4, ychunk - 1, z, &bars[st]);
  tma_load_3d(base + M_OFF, &mp.m, x0 - 16, ychunk - 1, tile, &bars[st]);
  tma_load_3d(base + B_OFF, &mp.b, x0, ychunk, z, &bars[st]);
}

__device__ __forceinline__ float f4g(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// r = b - A~ u for the lane's quad of chunk row `w` (stage buffers)
__device__ __forceinline__ float4 resid_smem(const float* us, const unsigned char* ms,
                                             const float* bs, int w, int lane, int y, int H,
                                             int xq, int W) {
  const float* uc = us + (w + 1) * UW + 4 + 4 * lane;
  const float4 c = *reinterpret_cast<const float4*>(uc);
  const float4 up = *reinterpret_cast<const float4*>(uc - UW);
  const float4 dn = *reinterpret_cast<const float4*>(uc + UW);
  const float ul = uc[-1], ur = uc[4];
  const unsigned char* mc = ms + (w + 1) * MW + 16 + 4 * lane;
  const uint32_t m = *reinterpret_cast<const uint32_t*>(mc);
  const uint32_t mu = *reinterpret_cast<const uint32_t*>(mc - MW);
  const uint32_t md = *reinterpret_cast<const uint32_t*>(mc + MW);
  const bool ml = mc[-1] != 0, mr = mc[4] != 0;
  const float4 bb = *reinterpret_cast<const float4*>(bs + w * TC + 4 * lane);
  const bool hu = y > 0, hd = y < H - 1, hl = xq > 0, hr = xq + 4 < W;
  // q: the value as it enters a neighbour's sum (0 where masked)
  auto q = [](float v, uint32_t mw, int i) { return ((mw >> (8 * i)) & 0xFFu) ? 0.0 : (double)v; };
  const double dv = (hu ? 1.0 : 0.0) + (hd ? 1.0 : 0.0);  // vertical neighbours
  float out[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float uv = f4g(c, i);
    float ax;
    if ((m >> (8 * i)) & 0xFFu) {
      ax = uv;
    } else {
      // absent neighbours (outside the image) are TMA zero fill: +0.0 exactly
      const double qu = q(f4g(up, i), mu, i), qd = q(f4g(dn, i), md, i);
      const double ql = i > 0 ? q(f4g(c, i - 1), m, i - 1) : (ml ? 0.0 : (double)ul);
      const double qr = i < 3 ? q(f4g(c, i + 1), m, i + 1) : (mr ? 0.0 : (double)ur);
      const double a = ((qu + qd) + ql) + qr;
      const double d = dv + (i > 0 || hl ? 1.0 : 0.0) + (i < 3 || hr ? 1.0 : 0.0);
      ax = (float)(d * (double)uv - a);
    }
    out[i] = f4g(bb, i) - ax;
  }
  return make_float4(out[0], out[1], out[2], out[3]);
}

// MODE 0: residual (+ norms); MODE 1: residual + 2x2 restriction
template <int MODE, bool NORMS>
__global__ void __launch_bounds__(CR * 32) k_resid_tma(
    const __grid_constant__ Maps mp, float* __restrict__ r, double* __restrict__ partial,
    unsigned* __restrict__ counter, double* __restrict__ norms, float* __restrict__ rcoarse,
    int C, int H, int W, const int* __restrict__ active, double* __restrict__ bandcol,
    int band0, int nbt, size_t ps, size_t cps) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 127) & ~(uintptr_t)127);
  __shared__ uint64_t bars[NS];
  __shared__ double wsum[CR];
  __shared__ bool am_last;
  __shared__ __align__(16) float rrow[MODE == 1 ? 2 : 1][MODE == 1 ? CR : 1][MODE == 1 ? TC + 4 : 1];
  const int z = blockIdx.z, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TC, y0 = blockIdx.y * TR;
  const int nck = min(NCH, (H - y0 + CR - 1) / CR);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NS && k < nck; ++k) issue_chunk(mp, sm, bars, k, x0, y0 + k * CR, z, tile);
  const int xq = x0 + 4 * lane;
  const size_t plane = ps;  // plane stride (a row-strip view: the full level's)
  float sq = 0.0f;
  for (int k = 0; k < nck; ++k) {
    const int st = k % NS;
    mbar_wait(&bars[st], (uint32_t)((k / NS) & 1));
    const unsigned char* base = sm + st * STAGE;
    const int y = y0 + k * CR + w;
    float4 rr = make_float4(0.f, 0.f, 0.f, 0.f);
    if (y < H && xq < W) {
      rr = resid_smem((const float*)(base + U_OFF), base + M_OFF, (const float*)(base + B_OFF),
                      w, lane, y, H, xq, W);
      if (MODE == 0) {
        *reinterpret_cast<float4*>(r + (size_t)z * plane + (size_t)y * W + xq) = rr;
        if (NORMS) {
          sq = __fmaf_rn(rr.x, rr.x, sq);
          sq = __fmaf_rn(rr.y, rr.y, sq);
          sq = __fmaf_rn(rr.z, rr.z, sq);
          sq = __fmaf_rn(rr.w, rr.w, sq);
        }
      }
    }
    if (MODE == 1) *reinterpret_cast<float4*>(&rrow[k & 1][w][4 * lane]) = rr;
    if (MODE == 0 && NORMS && bandcol && ((k & 1) || k == nck - 1)) {
      // row-band partials for the strip-partitioned solve (strips.cu): the
      // CTA's sum over each 16-row band (2 chunks), one double per (plane,
      // band, 128-column group); views start on a band boundary
      double d = (double)sq;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xFFFFFFFFu, d, o);
      if (lane == 0) wsum[w] = d;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < CR; ++q2) t += wsum[q2];
        bandcol[((size_t)z * nbt + band0 + (y0 + k * CR) / 16) * gridDim.x + blockIdx.x] = t;
      }
      sq = 0.0f;
    }
    __syncthreads();  // stage st fully consumed (and the chunk's r rows staged)
    if (threadIdx.x == 0 && k + NS < nck)
      issue_chunk(mp, sm, bars, st, x0, y0 + (k + NS) * CR, z, tile);
    if (MODE == 1) {
      // restrict_values (numba_impl.py:266-284): all 8 warps, one coarse
      // pixel per lane -- warp w takes coarse row w/2 of the chunk and the
      // 32-column half w&1, ((a + b) + c) + d in double.  rrow is double
      // buffered, so the next chunk's rows never overwrite rows still being
      // restricted (no second barrier per chunk).
      const int yf = y0 + k * CR + 2 * (w >> 1);
      const int xc = (x0 >> 1) + 32 * (w & 1) + lane;
      const int cw = W / 2;
      if (yf < H && xc < cw) {
        const float* ra = &rrow[k & 1][2 * (w >> 1)][2 * (32 * (w & 1) + lane)];
        const float2 a = *reinterpret_cast<const float2*>(ra);
        float o;
        if (yf + 1 < H) {
          const float2 b2 = *reinterpret_cast<const float2*>(ra + (TC + 4));
          o = (float)(((((double)a.x + (double)a.y) + (double)b2.x) + (double)b2.y) / 4.0);
        } else {
          o = (float)(((double)a.x + (double)a.y) / 2.0);
        }
        rcoarse[(size_t)z * cps + (size_t)(yf >> 1) * cw + xc] = o;
      }
    }
  }
  if (MODE != 0 || !NORMS || bandcol) return;
  double sqd = (double)sq;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sqd += __shfl_xor_sync(0xFFFFFFFFu, sqd, o);
  if (lane == 0) wsum[w] = sqd;
  __syncthreads();
  const unsigned ncta = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < CR; ++q) s += wsum[q];
    if (ncta == 1) {
      norms[z] = s;
      am_last = false;
    } else {
      partial[(size_t)z * ncta + cta] = s;
      __threadfence();
      am_last = atomicAdd(counter + z, 1u) == ncta - 1;
    }
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned i = threadIdx.x; i < ncta; i += CR * 32)
    t += ((volatile double*)partial)[(size_t)z * ncta + i];
  t = cta_sum<CR * 32>(t, wsum);
  if (threadIdx.x == 0) {
    norms[z] = t;
    counter[z] = 0u;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool make_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, size_t esize, int W,
              int H, int nz, int box_w, int box_h, size_t ps = 0) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)W * esize,
                           (cuuint64_t)(ps ? ps : (size_t)W * H) * esize};
  cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_maps(Maps& mp, const float* u, const float* b, const uint8_t* m, int C, int H, int W,
               int ntile, size_t ps) {
  const int nz = C * ntile;
  return make_map(&mp.u, u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, W, H, nz, UW, CR + 2, ps) &&
         make_map(&mp.b, b, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, W, H, nz, TC, CR, ps) &&
         make_map(&mp.m, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, H, ntile, MW, CR + 2);
}

template <int MODE, bool NORMS>
int launch(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
           unsigned* counter, double* norms, float* rc, int C, int H, int W, cudaStream_t s,
           int ntile, const int* active, double* bandcol = nullptr, int band0 = 0,
           int nbt = 0, size_t ps = 0, size_t cps = 0) {
  if (!ps) ps = (size_t)H * W;
  if (!cps) cps = (size_t)((H + 1) / 2) * (W / 2);
  Maps mp;
  if (!make_maps(mp, u, b, m, C, H, W, ntile, ps)) {
    set_error("cuTensorMapEncodeTiled failed (%d x %d x %d)", C * ntile, H, W);
    return -1;
  }
  dim3 grid(cdiv(W, TC), cdiv(H, TR), (unsigned)((long)C * ntile));
  SP_CUDA(launch_k(k_resid_tma<MODE, NORMS>, grid, dim3(CR * 32), SMEM, s, mp, r, partial,
                   counter, norms, rc, C, H, W, active, bandcol, band0, nbt, ps, cps));
  SP_CHECK_LAUNCH();
  return 0;
}

// ---- prolongation + enforce (solver.py:294-296, numba_impl.py:316-348) -------
// u = (add ? u : 0) + P e on unmasked pixels, u = b~ on masked pixels.  A
// chunk is 8 fine rows x 128 columns: TMA brings the u rows (add only), the
// mask rows and the 6 x 72 coarse rows / columns the bilinear stencil of
// the chunk touches; the overwrite form (FMG cascade) reads b~ directly for
// quads holding a stored pixel, the add form never reads it (see below).  The interpolation is the reference's double
// expression with its clamped, cell-centred indices, one rounding.
constexpr int EW = TC / 2 + 8;     // coarse columns per chunk (4-column halo)
constexpr int EH = CR / 2 + 2;     // coarse rows per chunk
constexpr int PU_BYTES = TC * CR * 4;
constexpr int PM_BYTES = TC * CR;
constexpr int PE_BYTES = EW * EH * 4;
constexpr int PU_OFF = 0;
constexpr int PM_OFF = PU_BYTES;
constexpr int PE_OFF = PM_OFF + (PM_BYTES + 127) / 128 * 128;
constexpr int PSTAGE = PE_OFF + (PE_BYTES + 127) / 128 * 128;
constexpr int PSMEM = NS * PSTAGE + 128;

struct PMaps {
  CUtensorMap u, m, e;
};

__device__ __forceinline__ void paxis_d(int y, int n, int& y0, int& y1, double& wy) {
  double fy = ((double)y + 0.5) / 2.0 - 0.5;
  y0 = (int)floor(fy);
  wy = fy - (double)y0;
  if (y0 < 0) { y0 = 0; wy = 0.0; }
  if (y0 > n - 1) { y0 = n - 1; wy = 0.0; }
  y1 = min(y0 + 1, n - 1);
}

template <bool ADD>
__global__ void __launch_bounds__(CR * 32) k_prolong_tma(
    const __grid_constant__ PMaps mp, float* __restrict__ u, const float* __restrict__ b,
    const uint8_t* __restrict__ m, int C, int chh, int cww, int H, int W,
    const int* __restrict__ active, size_t ps) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 127) & ~(uintptr_t)127);
  __shared__ uint64_t bars[NS];
  const int z = blockIdx.z, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TC, y0 = blockIdx.y * TR;
  const int nck = min(NCH, (H - y0 + CR - 1) / CR);
  const uint32_t tx = (ADD ? PU_BYTES : 0) + PM_BYTES + PE_BYTES;
  auto issue = [&](int st, int yc) {
    unsigned char* base = sm + st * PSTAGE;
    mbar_expect_tx(&bars[st], tx);
    if (ADD) tma_load_3d(base + PU_OFF, &mp.u, x0, yc, z, &bars[st]);
    tma_load_3d(base + PM_OFF, &mp.m, x0, yc, tile, &bars[st]);
    tma_load_3d(base + PE_OFF, &mp.e, x0 / 2 - 4, yc / 2 - 1, z, &bars[st]);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NS && k < nck; ++k) issue(k, y0 + k * CR);
  const int xq = x0 + 4 * lane;
  const size_t plane = ps;
  // x interpolation of the lane's 4 pixels (chunk-independent)
  int xa[4], xb[4];
  double wx[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    paxis_d(xq + i, cww, xa[i], xb[i], wx[i]);
    xa[i] -= x0 / 2 - 4;
    xb[i] -= x0 / 2 - 4;
  }
  for (int k = 0; k < nck; ++k) {
    const int st = k % NS;
    mbar_wait(&bars[st], (uint32_t)((k / NS) & 1));
    const unsigned char* base = sm + st * PSTAGE;
    const int yc = y0 + k * CR, y = yc + w;
    if (y < H && xq < W) {
      const uint32_t mw = *reinterpret_cast<const uint32_t*>(base + PM_OFF + w * TC + 4 * lane);
      const float4 uu = ADD ? *reinterpret_cast<const float4*>(base + PU_OFF + (w * TC + 4 * lane) * 4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      // masked pixels take b~.  With ADD the V-cycle invariant u == b~ on
      // the mask holds on entry (solver.py:293-296 enforces before every
      // smoothing sweep, and ORAS corrections vanish on masked pixels: the
      // local residual, and hence p and v, are exactly 0 there), so the
      // TMA-staged u already holds b~ and b~ is never read; the FMG
      // cascade's overwrite (ADD false) reads it.
      const float4 bb = ADD ? uu
                            : (mw ? *reinterpret_cast<const float4*>(b + (size_t)z * plane +
                                                                      (size_t)y * W + xq)
                                  : make_float4(0.f, 0.f, 0.f, 0.f));
      int ya, yb;
      double wy;
      paxis_d(y, chh, ya, yb, wy);
      const float* es = (const float*)(base + PE_OFF);
      const float* e0 = es + (ya - (yc / 2 - 1)) * EW;
      const float* e1 = es + (yb - (yc / 2 - 1)) * EW;
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if ((mw >> (8 * i)) & 0xFFu) {
          o[i] = f4g(bb, i);
          continue;
        }
        const double v = (1.0 - wy) * ((1.0 - wx[i]) * (double)e0[xa[i]] + wx[i] * (double)e0[xb[i]]) +
                         wy * ((1.0 - wx[i]) * (double)e1[xa[i]] + wx[i] * (double)e1[xb[i]]);
        const float p = (float)v;
        o[i] = ADD ? f4g(uu, i) + p : p;
      }
      *reinterpret_cast<float4*>(u + (size_t)z * plane + (size_t)y * W + xq) =
          make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + NS < nck) issue(st, y0 + (k + NS) * CR);
  }
}

// ---- warp-streamed sweeps (the default: sp_ws_variant) ----------------------
// The CTA-tile kernels above spend 60-70 issued instructions per
// pixel-channel (ncu: issue-bound at 69-75% with the DRAM at 4.4 TB/s): one
// row per warp, so every value is converted and mask-tested once for each
// of the up to five stencil rows that read it, and a CTA-wide barrier per
// chunk.  Here every WARP is an independent streaming unit:
//   - it owns a contiguous range of the plane's 8-row x 128-column chunks,
//     taken down one 128-column strip (consecutive chunks share their halo
//     rows, which then come from L2);
//   - a private ring of SPW shared-memory stages, filled by its own elected
//     lane through TMA (the same tensor maps and boxes as above, image
//     borders are the TMA zero fill), completion on per-stage mbarriers;
//   - the lane owns a 4-pixel column quad and MARCHES the chunk's 8 rows:
//     each value is converted to double and masked once and reused as the
//     down, centre and up neighbour, no barriers at all (__syncwarp only);
//   - the grid is sized to the resident warp slots (one wave), the chunk
//     ranges are balanced to one chunk, so there is no tail wave.
// Arithmetic is the kernels' above bit for bit (numba_impl.py:68-98 /
// 147-158 / 266-284 / 316-348): the residual, the restriction and the
// prolongation are identical per element; only the float partials of the
// residual norms group differently (per warp range instead of per tile), and
// they are still reduced in a fixed order (deterministic).
constexpr int WS_NW = 8;  // warps per CTA

// the value as it enters a neighbour's sum: 0 where masked (selected in
// float, then one conversion)
__device__ __forceinline__ double qmask(float v, uint32_t mw, int i) {
  return (double)(((mw >> (8 * i)) & 0xFFu) ? 0.0f : v);
}

__device__ __forceinline__ unsigned char* ws_smem(unsigned char* raw) {
  // 128-byte aligned base of the dynamic shared memory, as a shared-space
  // pointer (LDS, not generic loads)
  return raw + ((128u - (smem_u32(raw) & 127u)) & 127u);
}

// the warp's chunk range [q0, q1) of a plane of nq chunks split over gwp warps
__device__ __forceinline__ void ws_range(long nq, int gw, int gwp, long& q0, long& q1) {
  q0 = nq * gw / gwp;
  q1 = nq * (gw + 1) / gwp;
}

// MODE 0: residual (+ norms); MODE 1: residual + 2x2 restriction
template <int MODE, bool NORMS, int SPW>
__global__ void __launch_bounds__(WS_NW * 32) k_ws_resid(
    const __grid_constant__ Maps mp, float* __restrict__ r, double* __restrict__ partial,
    unsigned* __restrict__ counter, double* __restrict__ norms, float* __restrict__ rcoarse,
    int C, int H, int W, const int* __restrict__ active, size_t ps, size_t cps, int pf) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t bars[WS_NW][SPW];
  const int z = blockIdx.y, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* sm = ws_smem(smraw) + (size_t)w * SPW * STAGE;
  uint64_t* bar = bars[w];
  const int nrc = (H + CR - 1) / CR;
  const long nq = (long)((W + TC - 1) / TC) * nrc;
  const int gwp = gridDim.x * WS_NW, gw = blockIdx.x * WS_NW + w;
  long q0, q1;
  ws_range(nq, gw, gwp, q0, q1);
  const int n = (int)(q1 - q0);
  if (lane == 0) {
    for (int i = 0; i < SPW; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // chunks SPW.. SPW+pf-1 ahead of the ring are prefetched into L2 (more
  // bytes in flight than the shared-memory ring holds)
  auto prefetch = [&](int k) {
    if (k >= n) return;
    const long q = q0 + k;
    const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
    tma_prefetch_3d(&mp.u, tx * TC - 4, rc * CR - 1, z);
    tma_prefetch_3d(&mp.b, tx * TC, rc * CR, z);
  };
  if (lane == 0) {
    for (int k = 0; k < SPW && k < n; ++k) {
      const long q = q0 + k;
      const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
      issue_chunk(mp, sm, bar, k, tx * TC, rc * CR, z, tile);
    }
    for (int k = SPW; k < SPW + pf; ++k) prefetch(k);
  }
  const size_t plane = ps;
  const int cw = W / 2;
  float sq = 0.0f;
  for (int k = 0; k < n; ++k) {
    const int st = k % SPW;
    const long q = q0 + k;
    const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
    const int x0 = tx * TC, y0 = rc * CR, xq = x0 + 4 * lane;
    mbar_wait(&bar[st], (uint32_t)((k / SPW) & 1));
    const unsigned char* base = sm + st * STAGE;
    const float* us = (const float*)(base + U_OFF) + 4 + 4 * lane;
    const unsigned char* ms = base + M_OFF + 16 + 4 * lane;
    const float* bs = (const float*)(base + B_OFF) + 4 * lane;
    if (xq < W) {
      // diagonal (numba_impl.py:80-95 counts each existing neighbour once;
      // integer-valued, so order-free): interior rows, per lane pixel
      float* const rrow0 = MODE == 0 ? r + (size_t)z * plane + (size_t)y0 * W + xq : nullptr;
      double dmid[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dmid[i] = 2.0 + (xq + i > 0 ? 1.0 : 0.0) + (xq + i < W - 1 ? 1.0 : 0.0);
      // rolling rows: a = row above, b = centre row, n = row below
      double qa[4], qb[4];
      float4 ub;
      uint32_t mb;
      {
        const float4 u0 = *reinterpret_cast<const float4*>(us);
        const uint32_t m0 = *reinterpret_cast<const uint32_t*>(ms);
        ub = *reinterpret_cast<const float4*>(us + UW);
        mb = *reinterpret_cast<const uint32_t*>(ms + MW);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          qa[i] = qmask(f4g(u0, i), m0, i);
          qb[i] = qmask(f4g(ub, i), mb, i);
        }
      }
      float4 rprev = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int t = 0; t < CR; ++t) {
        const int y = y0 + t;
        const float4 un = *reinterpret_cast<const float4*>(us + (t + 2) * UW);
        const uint32_t mn = *reinterpret_cast<const uint32_t*>(ms + (t + 2) * MW);
        double qn[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qn[i] = qmask(f4g(un, i), mn, i);
        float4 rr = make_float4(0.f, 0.f, 0.f, 0.f);
        if (y < H) {
          const float* uc = us + (t + 1) * UW;
          const unsigned char* mc = ms + (t + 1) * MW;
          const double qL = (double)(mc[-1] ? 0.0f : uc[-1]);
          const double qR = (double)(mc[4] ? 0.0f : uc[4]);
          const float4 bb = *reinterpret_cast<const float4*>(bs + t * TC);
          double a[4];
          float o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double ql = i > 0 ? qb[i - 1] : qL;
            const double qr = i < 3 ? qb[i + 1] : qR;
            a[i] = ((qa[i] + qn[i]) + ql) + qr;
            // d * u is exact (d <= 4, u a float), so the fused form rounds
            // exactly like the reference's (d * u - acc); masked pixels are
            // identity rows (branch-free select)
            const float axu = (float)__fma_rn(dmid[i], qb[i], -a[i]);
            const float ax = ((mb >> (8 * i)) & 0xFFu) ? f4g(ub, i) : axu;
            o[i] = f4g(bb, i) - ax;
          }
          if (y == 0 || y == H - 1) {
            // the image's first / last row: one vertical neighbour less
            const double dtb = (y > 0 ? 0.0 : 1.0) + (y < H - 1 ? 0.0 : 1.0);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float axu = (float)__fma_rn(dmid[i] - dtb, qb[i], -a[i]);
              const float ax = ((mb >> (8 * i)) & 0xFFu) ? f4g(ub, i) : axu;
              o[i] = f4g(bb, i) - ax;
            }
          }
          rr = make_float4(o[0], o[1], o[2], o[3]);
          if (MODE == 0) {
            *reinterpret_cast<float4*>(rrow0 + (size_t)t * W) = rr;
            if (NORMS) {
              sq = __fmaf_rn(rr.x, rr.x, sq);
              sq = __fmaf_rn(rr.y, rr.y, sq);
              sq = __fmaf_rn(rr.z, rr.z, sq);
              sq = __fmaf_rn(rr.w, rr.w, sq);
            }
          }
        }
        if (MODE == 1 && (t & 1)) {
          // restrict_values (numba_impl.py:266-284): rows y-1, y -> coarse
          // row (y-1)/2, ((a + b) + c) + d in double, a 1-row tail halves
          const int ye = y - 1;
          if (ye < H) {
            float c0, c1;
            if (y < H) {
              c0 = (float)(((((double)rprev.x + (double)rprev.y) + (double)rr.x) + (double)rr.y) / 4.0);
              c1 = (float)(((((double)rprev.z + (double)rprev.w) + (double)rr.z) + (double)rr.w) / 4.0);
            } else {
              c0 = (float)(((double)rprev.x + (double)rprev.y) / 2.0);
              c1 = (float)(((double)rprev.z + (double)rprev.w) / 2.0);
            }
            *reinterpret_cast<float2*>(rcoarse + (size_t)z * cps + (size_t)(ye >> 1) * cw +
                                       (xq >> 1)) = make_float2(c0, c1);
          }
        }
        rprev = rr;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          qa[i] = qb[i];
          qb[i] = qn[i];
        }
        ub = un;
        mb = mn;
      }
    }
    __syncwarp();  // every lane is done with stage st
    if (lane == 0 && k + SPW < n) {
      const long q2 = q + SPW;
      const int tx2 = (int)(q2 / nrc), rc2 = (int)(q2 - (long)tx2 * nrc);
      issue_chunk(mp, sm, bar, st, tx2 * TC, rc2 * CR, z, tile);
      if (pf > 0) prefetch(k + SPW + pf);
    }
  }
  if (MODE != 0 || !NORMS) return;
  // deterministic norms: one double per warp (its fixed chunk range), the
  // plane's last warp adds them in warp order
  double d = (double)sq;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xFFFFFFFFu, d, o);
  unsigned last = 0;
  if (lane == 0) {
    partial[(size_t)z * gwp + gw] = d;
    __threadfence();
    last = atomicAdd(counter + z, 1u) == (unsigned)gwp - 1;
  }
  last = __shfl_sync(0xFFFFFFFFu, last, 0);
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = lane; i < gwp; i += 32) t += ((volatile double*)partial)[(size_t)z * gwp + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
  if (lane == 0) {
    norms[z] = t;
    counter[z] = 0u;
  }
}

// prolongation + enforce, warp-streamed (the same stage layout and
// arithmetic as k_prolong_tma): u = (ADD ? u : 0) + P e on unmasked pixels
template <bool ADD, int SPW>
__global__ void __launch_bounds__(WS_NW * 32) k_ws_prolong(
    const __grid_constant__ PMaps mp, float* __restrict__ u, const float* __restrict__ b,
    int C, int chh, int cww, int H, int W, const int* __restrict__ active, size_t ps, int pf) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t bars[WS_NW][SPW];
  const int z = blockIdx.y, tile = z / C;
  if (active && !active[tile]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* sm = ws_smem(smraw) + (size_t)w * SPW * PSTAGE;
  uint64_t* bar = bars[w];
  const int nrc = (H + CR - 1) / CR;
  const long nq = (long)((W + TC - 1) / TC) * nrc;
  const int gwp = gridDim.x * WS_NW, gw = blockIdx.x * WS_NW + w;
  long q0, q1;
  ws_range(nq, gw, gwp, q0, q1);
  const int n = (int)(q1 - q0);
  const uint32_t tx_bytes = (ADD ? PU_BYTES : 0) + PM_BYTES + PE_BYTES;
  auto issue = [&](int st, long q) {
    const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
    const int x0 = tx * TC, yc = rc * CR;
    unsigned char* base = sm + st * PSTAGE;
    mbar_expect_tx(&bar[st], tx_bytes);
    if (ADD) tma_load_3d(base + PU_OFF, &mp.u, x0, yc, z, &bar[st]);
    tma_load_3d(base + PM_OFF, &mp.m, x0, yc, tile, &bar[st]);
    tma_load_3d(base + PE_OFF, &mp.e, x0 / 2 - 4, yc / 2 - 1, z, &bar[st]);
  };
  if (lane == 0) {
    for (int i = 0; i < SPW; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto prefetch = [&](int k) {
    if (!ADD || k >= n) return;
    const long q = q0 + k;
    const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
    tma_prefetch_3d(&mp.u, tx * TC, rc * CR, z);
  };
  if (lane == 0) {
    for (int k = 0; k < SPW && k < n; ++k) issue(k, q0 + k);
    for (int k = SPW; k < SPW + pf; ++k) prefetch(k);
  }
  const size_t plane = ps;
  for (int k = 0; k < n; ++k) {
    const int st = k % SPW;
    const long q = q0 + k;
    const int tx = (int)(q / nrc), rc = (int)(q - (long)tx * nrc);
    const int x0 = tx * TC, yc = rc * CR, xq = x0 + 4 * lane;
    mbar_wait(&bar[st], (uint32_t)((k / SPW) & 1));
    const unsigned char* base = sm + st * PSTAGE;
    if (xq < W) {
      // x interpolation (numba_impl.py:333-344) of the lane's 4 pixels in
      // closed form: coarse columns c-1 .. c+2 (c = xq/2), weights 1/4, 3/4;
      // the left image edge clamps pixel 0 to (c, c+1) with weights (1, 0),
      // the right edge clamps column c+2 to cww-1.  E columns are relative
      // to the box origin x0/2 - 4.
      const int c = xq >> 1, cb = c - (x0 / 2 - 4);
      int ia[4], ib[4];
      double wa[4], wb[4];
      ia[0] = cb - 1; ib[0] = cb;     wa[0] = 0.25; wb[0] = 0.75;
      ia[1] = cb;     ib[1] = cb + 1; wa[1] = 0.75; wb[1] = 0.25;
      ia[2] = cb;     ib[2] = cb + 1; wa[2] = 0.25; wb[2] = 0.75;
      ia[3] = cb + 1; ib[3] = c + 2 <= cww - 1 ? cb + 2 : cb + 1;
      wa[3] = 0.75;   wb[3] = 0.25;
      if (xq == 0) {
        ia[0] = cb;
        ib[0] = cww > 1 ? cb + 1 : cb;
        wa[0] = 1.0;
        wb[0] = 0.0;
      }
      const float* es = (const float*)(base + PE_OFF);
      // one coarse row's x interpolations (exact products: the weights are
      // 0, 1/4, 3/4 or 1 and E is float, so the fused form equals the
      // reference's (1 - wx) * e0 + wx * e1)
      auto hrow = [&](int l, double (&h)[4]) {
        const float* e = es + l * EW;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          h[i] = __fma_rn(wb[i], (double)e[ib[i]], wa[i] * (double)e[ia[i]]);
      };
      const int yb0 = yc / 2 - 1;  // coarse row of local index 0
      double hlo[4], hhi[4];
      hrow(0, hlo);
      hrow(1, hhi);
      const uint32_t* mrow = (const uint32_t*)(base + PM_OFF) + lane;
      const float4* urow = (const float4*)(base + PU_OFF) + lane;
#pragma unroll
      for (int t = 0; t < CR; ++t) {
        if (t & 1) {
          // generic rows: t -> coarse local rows ((t+1)/2, (t+1)/2 + 1)
#pragma unroll
          for (int i = 0; i < 4; ++i) hlo[i] = hhi[i];
          hrow((t + 1) / 2 + 1, hhi);
        }
        const int y = yc + t;
        if (y >= H) break;
        int ya, yb;
        double wy;
        paxis_d(y, chh, ya, yb, wy);
        double ha[4], hb[4];
        if (ya - yb0 == (t + 1) / 2 && yb == ya + 1) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            ha[i] = hlo[i];
            hb[i] = hhi[i];
          }
        } else {  // clamped edge rows (y = 0, the last row)
          hrow(ya - yb0, ha);
          hrow(yb - yb0, hb);
        }
        const uint32_t mw = mrow[t * (TC / 4)];
        const float4 uu = ADD ? urow[t * (TC / 4)] : make_float4(0.f, 0.f, 0.f, 0.f);
        float* dst = u + (size_t)z * plane + (size_t)y * W + xq;
        // masked pixels: u == b~ there (V-cycle invariant, see k_prolong_tma)
        // with ADD; the overwrite form reads b~
        const float4 bb = ADD ? uu
                              : (mw ? *reinterpret_cast<const float4*>(b + (size_t)z * plane +
                                                                        (size_t)y * W + xq)
                                    : make_float4(0.f, 0.f, 0.f, 0.f));
        float o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if ((mw >> (8 * i)) & 0xFFu) {
            o[i] = f4g(bb, i);
          } else {
            const double v = (1.0 - wy) * ha[i] + wy * hb[i];
            o[i] = ADD ? f4g(uu, i) + (float)v : (float)v;
          }
        }
        *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncwarp();
    if (lane == 0 && k + SPW < n) {
      issue(st, q + SPW);
      if (pf > 0) prefetch(k + SPW + pf);
    }
  }
}

// shared-memory stages per warp: 2 (default) or 1 (half the shared memory,
// twice the resident warps), sp_ws_stages
constexpr int ws_smem(int spw) { return WS_NW * spw * STAGE + 128; }
constexpr int ws_psmem(int spw) { return WS_NW * spw * PSTAGE + 128; }

}  // namespace

// warp-streamed sweeps on/off (sp_ws_variant; A/B against the CTA-tile
// kernels, which stay as the bandcol / strip-norm path)
static int ws_on = 1;
int ws_variant(int v) {
  if (v >= 0) ws_on = v;
  return ws_on;
}

// chunks each warp keeps prefetched into L2 ahead of its shared-memory ring
// (sp_ws_prefetch)
static int ws_pf = 0;  // measured slower at 1, 2, 4, 8 (profiles/ws_ab_r02u.txt)
int ws_prefetch(int v) {
  if (v >= 0) ws_pf = v;
  return ws_pf;
}

// stages per warp (1 or 2) of launches made afterwards: the residual sweep
// runs best with 2 stages (8 warps per SM), the restriction and the
// prolongation with 1 (16 warps per SM): 57.5 / 51.4 / 47.4 us on the 4K RGB
// finest level vs 61.8 / 62.0 / 48.3 with the other choice
// (profiles/ws_ab_r02u.txt).  0 = these defaults.
static int ws_spw = 0;
int ws_stages(int v) {
  if (v >= 0 && v <= 2) ws_spw = v;
  return ws_spw;
}
static int spw_for(int kind) {  // 0 residual, 1 restriction, 2 prolongation
  return ws_spw ? ws_spw : (kind == 0 ? 2 : 1);
}

// resident CTAs per SM of the warp-streamed kernels (set by tma_prepare),
// [stages - 1]
static int ws_occ_resid[2] = {1, 1}, ws_occ_prolong[2] = {1, 1};

// CTAs per plane: fill the resident slots once (no tail wave), at most one
// warp per chunk, and at most `cap` warps per plane (partial-sum slots)
static unsigned ws_ctas(int occ, long nplanes, long nq, long cap) {
  long slots = (long)num_sms() * occ;
  long per = slots / (nplanes > 0 ? nplanes : 1);
  long maxw = nq < cap ? nq : cap;
  if (per * WS_NW > maxw) per = maxw / WS_NW;
  if (per < 1) per = 1;
  return (unsigned)per;
}

template <int SPW>
static int ws_prepare() {
  SP_CUDA(cudaFuncSetAttribute(k_ws_resid<0, true, SPW>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem(SPW)));
  SP_CUDA(cudaFuncSetAttribute(k_ws_resid<0, false, SPW>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem(SPW)));
  SP_CUDA(cudaFuncSetAttribute(k_ws_resid<1, false, SPW>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem(SPW)));
  SP_CUDA(cudaFuncSetAttribute(k_ws_prolong<true, SPW>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, ws_psmem(SPW)));
  SP_CUDA(cudaFuncSetAttribute(k_ws_prolong<false, SPW>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, ws_psmem(SPW)));
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &ws_occ_resid[SPW - 1], k_ws_resid<0, true, SPW>, WS_NW * 32, ws_smem(SPW)));
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &ws_occ_prolong[SPW - 1], k_ws_prolong<true, SPW>, WS_NW * 32, ws_psmem(SPW)));
  if (ws_occ_resid[SPW - 1] < 1) ws_occ_resid[SPW - 1] = 1;
  if (ws_occ_prolong[SPW - 1] < 1) ws_occ_prolong[SPW - 1] = 1;
  return 0;
}

// one-time kernel attributes (called at hierarchy / strip-group creation,
// never inside a stream capture)
int tma_prepare() {
  static bool done = false;
  if (done) return 0;
  SP_TRY(ws_prepare<1>());
  SP_TRY(ws_prepare<2>());
  SP_CUDA(cudaFuncSetAttribute(k_resid_tma<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               SMEM));
  SP_CUDA(cudaFuncSetAttribute(k_resid_tma<0, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  SP_CUDA(cudaFuncSetAttribute(k_resid_tma<1, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  SP_CUDA(cudaFuncSetAttribute(k_prolong_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               PSMEM));
  SP_CUDA(cudaFuncSetAttribute(k_prolong_tma<false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, PSMEM));
  done = true;
  return 0;
}

// TMA path: float levels with W % 16 == 0 (16-byte mask row pitch for the
// tensor map), W >= 128, 16-byte aligned buffers, and few enough CTAs per
// plane for the partial-sum slots
bool tma_prolong_ok(int H, int W) {
  // the coarse map's row pitch (W/2 floats) must be a multiple of 16 bytes
  return W % 16 == 0 && W >= TC && (W / 2) % 4 == 0 && encode_fn() != nullptr;
}

// strips (band-norm mode: no CTA-partial slots needed)
bool tma_view_ok(int W) { return W % 16 == 0 && W >= TC && encode_fn() != nullptr; }

bool tma_ok(int H, int W, size_t npart) {
  if (W % 16 != 0 || W < TC || !encode_fn()) return false;
  return (size_t)cdiv(W, TC) * cdiv(H, TR) <= npart;
}

// warp-streamed launch (k_ws_resid); npart: partial-sum slots per plane
template <int MODE, bool NORMS>
static int launch_ws(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
                     unsigned* counter, double* norms, float* rc, int C, int H, int W,
                     cudaStream_t s, int ntile, const int* active, size_t npart, size_t ps,
                     size_t cps) {
  if (!ps) ps = (size_t)H * W;
  if (!cps) cps = (size_t)((H + 1) / 2) * (W / 2);
  Maps mp;
  if (!make_maps(mp, u, b, m, C, H, W, ntile, ps)) {
    set_error("cuTensorMapEncodeTiled failed (%d x %d x %d)", C * ntile, H, W);
    return -1;
  }
  const long nz = (long)C * ntile, nq = (long)cdiv(W, TC) * cdiv(H, CR);
  const int spw = spw_for(MODE);
  const unsigned per = ws_ctas(ws_occ_resid[spw - 1], nz, nq, NORMS ? (long)npart : (1L << 30));
  dim3 grid(per, (unsigned)nz);
  SP_CUDA(launch_k(spw == 1 ? k_ws_resid<MODE, NORMS, 1> : k_ws_resid<MODE, NORMS, 2>, grid,
                   dim3(WS_NW * 32), ws_smem(spw), s, mp, r, partial, counter, norms, rc, C, H,
                   W, active, ps, cps, ws_pf));
  SP_CHECK_LAUNCH();
  return 0;
}

static bool ws_usable(size_t npart) { return ws_on && npart >= (size_t)WS_NW; }

int resid_tma(const float* u, const float* b, const uint8_t* m, float* r, double* partial,
              unsigned* counter, double* norms, int C, int H, int W, cudaStream_t s, int ntile,
              const int* active, double* bandcol, int band0, int nbt, size_t ps, size_t npart) {
  if (bandcol)
    return launch<0, true>(u, b, m, r, partial, counter, nullptr, nullptr, C, H, W, s, ntile,
                           active, bandcol, band0, nbt, ps);
  if (ws_usable(npart)) {
    if (norms)
      return launch_ws<0, true>(u, b, m, r, partial, counter, norms, nullptr, C, H, W, s, ntile,
                                active, npart, ps, 0);
    return launch_ws<0, false>(u, b, m, r, partial, counter, norms, nullptr, C, H, W, s, ntile,
                               active, npart, ps, 0);
  }
  if (norms)
    return launch<0, true>(u, b, m, r, partial, counter, norms, nullptr, C, H, W, s, ntile,
                           active);
  return launch<0, false>(u, b, m, r, partial, counter, norms, nullptr, C, H, W, s, ntile,
                          active);
}

int prolong_tma(const float* e, float* u, const float* b, const uint8_t* m, int C, int chh,
                int cww, int H, int W, int add, cudaStream_t s, int ntile, const int* active,
                size_t ps, size_t cps) {
  if (!ps) ps = (size_t)H * W;
  if (!cps) cps = (size_t)chh * cww;
  PMaps mp;
  const int nz = C * ntile;
  if ((add && !make_map(&mp.u, u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, W, H, nz, TC, CR, ps)) ||
      !make_map(&mp.m, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, H, ntile, TC, CR) ||
      !make_map(&mp.e, e, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cww, chh, nz, EW, EH, cps)) {
    set_error("cuTensorMapEncodeTiled failed (prolongation %d x %d x %d)", nz, H, W);
    return -1;
  }
  if (!add) mp.u = mp.m;  // unused
  if (ws_on) {
    const long nq = (long)cdiv(W, TC) * cdiv(H, CR);
    const int spw = spw_for(2);
    dim3 grid(ws_ctas(ws_occ_prolong[spw - 1], nz, nq, 1L << 30), (unsigned)nz);
    auto kern = spw == 1 ? (add ? k_ws_prolong<true, 1> : k_ws_prolong<false, 1>)
                         : (add ? k_ws_prolong<true, 2> : k_ws_prolong<false, 2>);
    SP_CUDA(launch_k(kern, grid, dim3(WS_NW * 32), ws_psmem(spw), s, mp, u, b, C, chh, cww, H,
                     W, active, ps, ws_pf));
    SP_CHECK_LAUNCH();
    return 0;
  }
  dim3 grid(cdiv(W, TC), cdiv(H, TR), (unsigned)nz);
  SP_CUDA(launch_k(add ? k_prolong_tma<true> : k_prolong_tma<false>, grid, dim3(CR * 32), PSMEM,
                   s, mp, u, b, m, C, chh, cww, H, W, active, ps));
  SP_CHECK_LAUNCH();
  return 0;
}

int resid_restrict_tma(const float* u, const float* b, const uint8_t* m, float* rc, int C,
                       int H, int W, cudaStream_t s, int ntile, const int* active, size_t ps,
                       size_t cps) {
  if (ws_on)
    return launch_ws<1, false>(u, b, m, nullptr, nullptr, nullptr, nullptr, rc, C, H, W, s,
                               ntile, active, 0, ps, cps);
  return launch<1, false>(u, b, m, nullptr, nullptr, nullptr, nullptr, rc, C, H, W, s, ntile,
                          active, nullptr, 0, 0, ps, cps);
}

}  // namespace sp
