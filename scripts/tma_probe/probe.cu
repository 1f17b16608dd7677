// standalone TMA probe: one 3-D box load via a __grid_constant__ tensor map
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct alignas(64) Maps { CUtensorMap a, b; };
template <typename T, int BW>
__global__ void k(const __grid_constant__ Maps mp, T* out, int x, int y, int which) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(BW * 4 * (int)sizeof(T)) : "memory");
    const CUtensorMap* m = which ? &mp.b : &mp.a;
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sa(sm)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(0), "r"(sa(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
  for (int i = threadIdx.x; i < BW * 4; i += blockDim.x) out[i] = ((T*)sm)[i];
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int W = 512, H = 64;
  float* f; uint8_t* m; float* of; uint8_t* om;
  cudaMalloc(&f, W * H * 4); cudaMalloc(&m, W * H); cudaMalloc(&of, 4096); cudaMalloc(&om, 4096);
  std::vector<float> hf(W * H); for (int i = 0; i < W * H; ++i) hf[i] = i;
  std::vector<uint8_t> hm(W * H); for (int i = 0; i < W * H; ++i) hm[i] = i & 0xff;
  cudaMemcpy(f, hf.data(), W * H * 4, cudaMemcpyHostToDevice); cudaMemcpy(m, hm.data(), W * H, cudaMemcpyHostToDevice);
  Maps mp;
  cuuint64_t dims[3] = {W, H, 1}; cuuint64_t st[2] = {W * 4, (cuuint64_t)W * H * 4}; cuuint32_t box[3] = {136, 4, 1}, es[3] = {1, 1, 1};
  int r1 = enc(&mp.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, f, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t st2[2] = {W, (cuuint64_t)W * H}; cuuint32_t box2[3] = {144, 4, 1};
  int r2 = enc(&mp.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, m, dims, st2, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", r1, r2);
  k<float, 136><<<1, 128, 8192>>>(mp, of, -4, -1, 0);
  printf("float map: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> o(544); cudaMemcpy(o.data(), of, 544 * 4, cudaMemcpyDeviceToHost);
  printf("  row0 %g %g %g %g | row1 %g %g %g\n", o[0], o[4], o[5], o[135], o[136], o[140], o[141]);
  int xs[4] = {0, 16, -16, -8};
  int ys[2] = {0, -1};
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 2; ++b) {
    k<uint8_t, 144><<<1, 128, 8192>>>(mp, om, xs[a], ys[b], 1);
    printf("u8 map x=%d y=%d: %s\n", xs[a], ys[b], cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
