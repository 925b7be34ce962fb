// TMA load-throughput probe (profiling aid, not part of the library).
// 128 CTAs each stream 64 tiles of 64 tokens x 128 bf16 (16 KB) from a
// [128][4096][128] bf16 tensor into shared memory, NS tiles in flight:
//   il    : the fused kernels' 4-D interleaved box {8, 64, 16, 1} (16 B rows)
//   sw128 : two 2-D boxes {64, 64} with SWIZZLE_128B (128 B rows)
//   bulk  : one contiguous 16 KB cp.async.bulk (upper bound)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int UNITS = 128, L = 4096, D = 128, C = 64, TILE = C * D * 2, NS = 4;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap m, const uint8_t* g, int ntiles, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[NS];
  const int unit = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  auto issue = [&](int t) {
    const int s = t % NS;
    uint8_t* dst = smem + s * TILE;
    expect_tx(&full[s], TILE);
    if (MODE == 0) {
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(su32(dst)), "l"(&m), "r"(0), "r"(t * C), "r"(0), "r"(unit), "r"(su32(&full[s])) : "memory");
    } else if (MODE == 1) {
      for (int h = 0; h < 2; ++h)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(dst + h * TILE / 2)), "l"(&m), "r"(h * 64), "r"(t * C), "r"(unit), "r"(su32(&full[s])) : "memory");
    } else {
      const uint8_t* src = g + ((size_t)unit * L + (size_t)t * C) * D * 2;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(dst)), "l"(src), "r"(TILE), "r"(su32(&full[s])) : "memory");
    }
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < NS && t < ntiles; ++t) issue(t);
  for (int t = 0; t < ntiles; ++t) {
    mbar_wait(&full[t % NS], (t / NS) & 1);
    acc += (float)smem[(t % NS) * TILE + threadIdx.x * 16];
    __syncthreads();
    if (threadIdx.x == 0 && t + NS < ntiles) issue(t + NS);
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  uint8_t* g;
  float* sink;
  const size_t bytes = (size_t)UNITS * L * D * 2;
  CK(cudaMalloc(&g, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(g, 1, bytes));
  CUtensorMap mil, msw;
  {
    cuuint64_t dims[4] = {8, (cuuint64_t)L, (cuuint64_t)(D / 8), (cuuint64_t)UNITS};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, 16, (cuuint64_t)L * D * 2};
    cuuint32_t box[4] = {8, (cuuint32_t)C, (cuuint32_t)(D / 8), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mil, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc il\n"); return 1; }
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)L, (cuuint64_t)UNITS};
    cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)L * D * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)C, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&msw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc sw\n"); return 1; }
  }
  const int smem = NS * TILE;
  CK(cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"il (16 B rows)", "sw128 (128 B rows)", "bulk (contiguous)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) probe<0><<<UNITS, 128, smem>>>(mil, g, L / C, sink);
      if (mode == 1) probe<1><<<UNITS, 128, smem>>>(msw, g, L / C, sink);
      if (mode == 2) probe<2><<<UNITS, 128, smem>>>(mil, g, L / C, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 3)
        printf("%-20s %8.1f us  %7.0f GB/s  %6.0f ns per tile per CTA (NS=%d in flight)\n", names[mode], ms * 1e3,
               bytes / (ms * 1e-3) / 1e9, ms * 1e6 / (L / C), NS);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
