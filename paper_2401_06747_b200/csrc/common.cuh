// common.cuh -- shared helpers for the sm_100a data-optimization kernels.
//
// All kernels are compiled with --fmad=false (see build.py): the reference
// kernels (numba_impl.py) never contract a*b+c, and the exact-parity kernels
// (stencils, transfers, geometry, dithering) rely on the same rounding.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

namespace sp {

// ---- error plumbing -------------------------------------------------------
void set_error(const char* fmt, ...);
const char* last_error();

#define SP_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::sp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                      cudaGetErrorString(_e));                                 \
      return -1;                                                               \
    }                                                                          \
  } while (0)

// kernels launched by this library (direct launches; graph replays add their
// node count) -- reported by bench.py as gpu_launches
void count_launches(long long n);
void count_work(int kind, long long px_cycles);

#define SP_CHECK_LAUNCH()                                                      \
  do {                                                                         \
    ::sp::count_launches(1);                                                   \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::sp::set_error("%s:%d launch: %s", __FILE__, __LINE__,                  \
                      cudaGetErrorString(_e));                                 \
      return -1;                                                               \
    }                                                                          \
  } while (0)

#define SP_TRY(expr)                                                           \
  do {                                                                         \
    int _rc = (expr);                                                          \
    if (_rc != 0) return _rc;                                                  \
  } while (0)

enum DType { SP_F32 = 0, SP_F64 = 1 };

// ---- programmatic dependent launch (coarse multigrid levels) ---------------
// On the small levels of a V-cycle every kernel is a few microseconds and the
// dependent-launch gap between consecutive kernels dominates.  Launched with
// programmatic stream serialization, a kernel is scheduled while its
// predecessor still runs and blocks in pdl_enter() until the predecessor has
// completed and its memory is visible; pdl_enter() then releases its own
// successor.  Kernels that may be launched this way call pdl_enter() before
// touching global memory (a no-op for ordinary launches).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// host side: PDL for the launches made while pdl_now() is set (solver.cu
// sets it for the levels >= sp_pdl_from_level of a V-cycle)
bool pdl_now();
void pdl_set(bool on);
int pdl_from_level(int v);  // solver.cu

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args... args) {
  if (!pdl_now()) {
    kern<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

inline unsigned cdiv(long a, long b) { return (unsigned)((a + b - 1) / b); }

// number of SMs of the current device (cached)
int num_sms();

// ---- device helpers ---------------------------------------------------------

// deterministic CTA-wide double sum: warp butterfly, then every thread adds
// the per-warp partials in warp order.  `scratch` holds >= nwarps doubles and
// must not be reused by the next call until after a __syncthreads() (callers
// alternate two scratch arrays).
template <int NT>
__device__ __forceinline__ double cta_sum(double v, double* scratch) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;  // 1-D or 2-D CTAs
  if ((tid & 31) == 0) scratch[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += scratch[w];
  return s;
}

// solver.py:134-139 _starts(dim, size, stride): min(i*stride, dim-size)
__host__ __device__ __forceinline__ int block_start(int k, int stride, int dim,
                                                    int size) {
  int s = k * stride;
  int lim = dim - size;
  return s < lim ? s : lim;
}

__host__ __device__ __forceinline__ int num_starts(int dim, int size, int stride) {
  if (dim <= size) return 1;
  return (dim - size + stride - 1) / stride + 1;
}

// keep freed stream-ordered memory in the device pool (the default release
// threshold of 0 hands it back to the driver at every synchronization, which
// makes every later scratch allocation pay a fresh mapping)
void retain_pool_memory();

// RAII stream-ordered scratch (cudaMallocAsync / cudaFreeAsync)
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  int alloc(size_t bytes) {
    retain_pool_memory();
    if (cudaMallocAsync(&p, bytes ? bytes : 16, s) != cudaSuccess) {
      set_error("cudaMallocAsync(%zu) failed", bytes);
      return -1;
    }
    return 0;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace sp
