// mma_probe.cu -- TEST-ONLY probe of the tcgen05 operand conventions used by
// the product kernels (tc_common.cuh): K-major / MN-major IL tiles, M=64 and
// M=128 accumulators (TMEM lane mapping), negated A, accumulate-into-D.
// D = init + (neg ? -1 : 1) * A @ B^T-convention below, fp32 accumulate.
//   A logical [M][K], B logical [N][K]  (D[m][n] = sum_k A[m][k] B[n][k])
#include "../../paper_2406_06484_b200/csrc/tc_common.cuh"

using namespace dn::tc;

__global__ void probe_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, const float* Dinit,
                             float* D, int M, int N, int K, int a_mn, int b_mn, int neg_a,
                             int lane_off) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 2;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // A tile: K-major -> rows M, cols K ; MN-major -> rows K, cols M
  for (int e = tid; e < M * K; e += blockDim.x) {
    int m = e / K, k = e % K;
    uint32_t off = a_mn ? il_off(k, m, K) : il_off(m, k, M);
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int n = e / K, k = e % K;
    uint32_t off = b_mn ? il_off(k, n, K) : il_off(n, k, N);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[e];
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  // preload D (lane mapping: M=128 row m -> lane m; M=64 row m -> lane 32*(m/16) + m%16)
  if (Dinit) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      int m = (M == 128) ? tid : ((lane >= lane_off && lane < lane_off + 16) ? warp * 16 + lane - lane_off : -1);
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(m >= 0 ? Dinit[m * N + c0 + j] : 0.f);
      tmem_st16(taddr(tm, warp * 32, c0), r);
    }
    tmem_st_wait();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t id = idesc_bf16(M, N, a_mn, b_mn, neg_a);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint64_t ad = a_mn ? desc_mn(a0, K, k0) : desc_k(a0, M, k0);
      uint64_t bd = b_mn ? desc_mn(b0, K, k0) : desc_k(b0, N, k0);
      mma_bf16(tm + ((uint32_t)lane_off << 16), ad, bd, id, (Dinit != nullptr || k0 > 0) ? 1u : 0u);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr(tm, warp * 32, c0), r);
    tmem_ld_wait();
    int m = (M == 128) ? tid : ((lane >= lane_off && lane < lane_off + 16) ? warp * 16 + lane - lane_off : -1);
    if (m >= 0)
      for (int j = 0; j < 16; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" int probe_mma(const void* A, const void* B, const float* Dinit, float* D, int M, int N,
                         int K, int a_mn, int b_mn, int neg_a, int lane_off) {
  size_t smem = (size_t)(M + N) * K * 2;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_kernel<<<1, 128, smem>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, Dinit, D, M,
                                 N, K, a_mn, b_mn, neg_a, lane_off);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}


// A (M=128 x K, bf16) staged in TMEM columns [256, 256 + K/2): lane m holds
// row m, column 256 + k/2 holds (A[m][k], A[m][k+1]) packed (low = even k).
__global__ void probe_ts_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int N,
                                int K, int b_mn) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* sB = smem;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < N * K; e += blockDim.x) {
    int n = e / K, k = e % K;
    uint32_t off = b_mn ? il_off(k, n, K) : il_off(n, k, N);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[e];
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  for (int c0 = 0; c0 < K / 2; c0 += 16) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 h;
      h.x = A[tid * K + 2 * (c0 + j)];
      h.y = A[tid * K + 2 * (c0 + j) + 1];
      r[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st16(taddr(tm, warp * 32, 256 + c0), r);
  }
  tmem_st_wait();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t id = idesc_bf16(128, N, false, b_mn);
    const uint32_t b0 = smem_u32(sB);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint64_t bd = b_mn ? desc_mn(b0, K, k0) : desc_k(b0, N, k0);
      mma_bf16_ts(tm, tm + 256 + k0 / 2, bd, id, k0 > 0 ? 1u : 0u);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr(tm, warp * 32, c0), r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = __uint_as_float(r[j]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" int probe_mma_ts(const void* A, const void* B, float* D, int N, int K, int b_mn) {
  size_t smem = (size_t)N * K * 2;
  cudaFuncSetAttribute(probe_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_ts_kernel<<<1, 128, smem>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, N, K,
                                    b_mn);
  return (int)cudaDeviceSynchronize();
}


// TMEM -> register read throughput: each warp of the CTA repeatedly loads
// `ncols` 32-bit columns of its 32-lane quadrant (32x32b.x16 shape).
__global__ void tmem_bw_kernel(long long* out, int iters, int ncols) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c0 = 0; c0 < ncols; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(taddr(tm, (warp & 3) * 32, c0), r);
      tmem_ld_wait();
      acc += r[0] ^ r[7] ^ r[15];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" long long probe_tmem_bw(int nthreads, int iters, int ncols) {
  long long* d;
  long long h[2];
  cudaMalloc(&d, 16);
  tmem_bw_kernel<<<1, nthreads>>>(d, iters, ncols);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h[0];
}


// tcgen05.mma issue/execute throughput from SWIZZLE_NONE IL tiles: one thread
// issues `n` MMAs of shape M x N x 16 (A K-major or MN-major, B K-major or
// MN-major), then waits on a commit.  Returns cycles.
__global__ void mma_tput_kernel(long long* out, int M, int N, int n, int a_mn, int b_mn) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 64 * 1024 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = 0;
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_bf16(M, N, a_mn, b_mn);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    // A tile: M rows x 128 K (K-major) or 128 rows (K) x M cols (MN-major)
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const int k0 = (i % 8) * 16;
      uint64_t ad = a_mn ? desc_mn(a0, 128, k0) : desc_k(a0, M, k0);
      uint64_t bd = b_mn ? desc_mn(b0, 128, k0) : desc_k(b0, N, k0);
      mma_bf16(tm, ad, bd, id, 1);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" long long probe_mma_tput(int M, int N, int n, int a_mn, int b_mn, long long* issue) {
  long long* d;
  long long h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mma_tput_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_tput_kernel<<<1, 128, 65536>>>(d, M, N, n, a_mn, b_mn);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  *issue = h[0];
  return h[1];
}


// MMA issue-pattern variants (see test_mma_issue_patterns).
__device__ __forceinline__ void mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ int lane_of(int tid) { return tid & 31; }

__global__ void mma_issue_kernel(long long* out, int variant, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 64 * 1024 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = 0;
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) { mbar_init(&bar, variant >= 3 ? variant - 1 : 1); mbar_fence_init(); }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  const uint32_t id = idesc_bf16(128, 64, false, false);
  const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
  long long t0 = 0, t1 = 0;
  if (variant == 0 && tid == 0) {         // per-iteration descriptors, lane 0 only
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k0 = 0; k0 < 128; k0 += 16)
        mma_bf16(tm, desc_k(a0, 128, k0), desc_k(b0, 64, k0), id, 1);
    t1 = clock64();
    mma_commit(&bar);
  } else if (variant == 1 && tid == 0) {  // precomputed descriptors, lane 0 only
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { ad[k] = desc_k(a0, 128, 16 * k); bd[k] = desc_k(b0, 64, 16 * k); }
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_bf16(tm, ad[k], bd[k], id, 1);
    t1 = clock64();
    mma_commit(&bar);
  } else if (variant >= 3 && warp < variant - 1 && lane_of(tid) == 0) {
    // variant 3/4/5: 2/3/4 warps issue concurrently into disjoint TMEM columns
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { ad[k] = desc_k(a0, 128, 16 * k); bd[k] = desc_k(b0, 64, 16 * k); }
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_bf16(tm + 64 * warp, ad[k], bd[k], id, 1);
    t1 = clock64();
    mma_commit(&bar);
  } else if (variant == 2 && warp == 0) {  // whole warp, elect.sync inside the asm
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { ad[k] = desc_k(a0, 128, 16 * k); bd[k] = desc_k(b0, 64, 16 * k); }
    __syncwarp();
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_elect(tm, ad[k], bd[k], id, 1);
    t1 = clock64();
    if (tid == 0) mma_commit(&bar);
  }
  if (tid == 0) {
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" long long probe_mma_issue(int variant, int reps, long long* issue) {
  long long* d;
  long long h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mma_issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_issue_kernel<<<1, 128, 65536>>>(d, variant, reps);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  *issue = h[0];
  return h[1];
}


// Throughput of a batch resembling the backward's M5: alternating M=64
// accumulators at lane offsets 0 / 16 and N in {64, 128}; one thread issues.
__global__ void mma_batch_kernel(long long* out, int N, int lane16, int n) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 64 * 1024 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = 0;
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_bf16(64, N, false, true);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { ad[k] = desc_k(a0, 64, 16 * k); bd[k] = desc_mn(b0, 128, 16 * k); }
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const uint32_t d = tm + ((lane16 && (i & 8)) ? (16u << 16) : 0u);
      mma_bf16(d, ad[i & 7], bd[i & 7], id, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" long long probe_mma_batch(int N, int lane16, int n) {
  long long* d;
  long long h = 0;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mma_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_batch_kernel<<<1, 128, 65536>>>(d, N, lane16, n);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

// SWIZZLE_128B ("SW") operand tiles (tc_common.cuh sw_off / desc_k_sw /
// desc_mn_sw): sw bit 0 = A in the SW layout, bit 1 = B; M=128 or 64.
__global__ void probe_sw_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int M,
                                int N, int K, int a_mn, int b_mn, int sw) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* sA = smem;
  uint8_t* sB = smem + ((M * K * 2 + 1023) / 1024) * 1024;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const bool swa = sw & 1, swb = sw & 2;
  for (int e = tid; e < M * K; e += blockDim.x) {
    int m = e / K, k = e % K;
    uint32_t off = a_mn ? (swa ? sw_off(k, m, K) : il_off(k, m, K))
                        : (swa ? sw_off(m, k, M) : il_off(m, k, M));
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int n = e / K, k = e % K;
    uint32_t off = b_mn ? (swb ? sw_off(k, n, K) : il_off(k, n, K))
                        : (swb ? sw_off(n, k, N) : il_off(n, k, N));
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[e];
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_bf16(M, N, a_mn, b_mn, false);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint64_t ad = a_mn ? (swa ? desc_mn_sw(a0, K, k0) : desc_mn(a0, K, k0))
                         : (swa ? desc_k_sw(a0, M, k0) : desc_k(a0, M, k0));
      uint64_t bd = b_mn ? (swb ? desc_mn_sw(b0, K, k0) : desc_mn(b0, K, k0))
                         : (swb ? desc_k_sw(b0, N, k0) : desc_k(b0, N, k0));
      mma_bf16(tm, ad, bd, id, k0 > 0 ? 1u : 0u);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr(tm, warp * 32, c0), r);
    tmem_ld_wait();
    int m = (M == 128) ? tid : (lane < 16 ? warp * 16 + lane : -1);
    if (m >= 0)
      for (int j = 0; j < 16; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" int probe_mma_sw(const void* A, const void* B, float* D, int M, int N, int K, int a_mn,
                            int b_mn, int sw) {
  size_t smem = ((size_t)(M * K * 2 + 1023) / 1024) * 1024 + (size_t)N * K * 2;
  cudaFuncSetAttribute(probe_sw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_sw_kernel<<<1, 128, smem>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, M, N, K,
                                    a_mn, b_mn, sw);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
