// Minimal TMA probe: one warp loads a 16x8 u32 tile via cp.async.bulk.tensor and checks it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void k(const __grid_constant__ CUtensorMap tmap, uint32_t* out, int x0, int y0) {
  __shared__ __align__(128) uint32_t tile[128];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (VARIANT == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(512) : "memory");
    if (VARIANT == 0)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(tile)), "l"((uint64_t)&tmap), "r"(x0), "r"(y0), "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(tile)), "l"((uint64_t)&tmap), "r"(x0), "r"(y0), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 128; i += 32) out[i] = tile[i];
}

int main() {
  const int W = 160, H = 120, pitch = 160;
  std::vector<uint32_t> h(pitch * H);
  for (int y = 0; y < H; y++) for (int x = 0; x < W; x++) h[y * pitch + x] = y * 1000 + x;
  uint32_t *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 512);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t gd[2] = {W, H}; cuuint64_t gs[1] = {pitch * 4}; cuuint32_t bx[2] = {16, 8}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int v = 0; v < 2; v++) {
    if (v == 0) k<0><<<1, 32>>>(m, o, 71, 16); else k<1><<<1, 32>>>(m, o, 72, 16);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t res[128]; cudaMemcpy(res, o, 512, cudaMemcpyDeviceToHost);
    printf("variant %d: %s  first %u last %u (expect %u %u)\n", v, cudaGetErrorString(e), res[0], res[127], 16*1000+71+v, 23*1000+86+v);
    if (e != cudaSuccess) break;
  }
  return 0;
}
