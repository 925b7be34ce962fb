// tc_fwd.cu -- fused sm_100a forward of the chunkwise DeltaNet layer:
// TMA-staged bf16 Q/K/V chunk tiles, tcgen05 MMAs with fp32 accumulators in
// TMEM, the intra-chunk triangular inverse by forward substitution in shared
// memory, and the fp32 state H = S^T held in TMEM across all chunks.
//
// Per (b, h) unit one CTA walks the L/C chunks (§3.2; Listing 1
// lines 1108-1117).  Per chunk t, with raw (un-normalised) bf16 tiles Q, K, V
// and s_i = 1/max(||k_i||, eps), r_i = 1/max(||q_i||, eps) (R9; identity
// when L2 normalisation is off):
//   G_qk = Q K^T, G_kk = K K^T                         tcgen05, M=64
//   L = tril(diag(beta s) G_kk diag(s), -1)            Eq. 10 (l2-normalised)
//   X = (I + L)^{-1}                                   forward substitution
//   T' = X diag(beta s), T'' = X diag(beta)
//       (so W = T' K = X diag(beta) K_hat and U = T'' V, Eq. 11)
//   W^T = K^T T'^T, U^T = V^T T''^T                    tcgen05, M=128
//   U'^T = U^T - H^T W^T                               tcgen05, negated A
//   Z = diag(s) U'                                      (K_hat^T U' = K^T Z)
//   O = diag(r) (Q H + tril(Q K^T) Z)                  Eq. 9, M=64
//   H^T += Z^T K                                       Eq. 8, M=128
// Algebra of the folded normalisation: DESIGN.md §Forward kernel.
#include <cudaTypedefs.h>
#include <stdio.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

using namespace tc;

constexpr int C = 64, DK = 128, DV = 128, NT = 128;
constexpr int LS = 68;  // row stride (floats) of the fp32 substitution buffers

// dynamic shared memory map (bytes)
constexpr int OFF_Q = 0;                     // Q   IL R=64  x 128    16 KB
constexpr int OFF_K = OFF_Q + C * DK * 2;    // K   IL R=64  x 128    16 KB
constexpr int OFF_V = OFF_K + C * DK * 2;    // V   IL R=64  x 128    16 KB
constexpr int OFF_T = OFF_V + C * DV * 2;    // T'  IL R=64  x 64      8 KB
constexpr int OFF_TU = OFF_T + C * C * 2;    // T'' IL R=64  x 64      8 KB
constexpr int OFF_A = OFF_TU + C * C * 2;    // A   IL R=64  x 64      8 KB
constexpr int OFF_W = OFF_A + C * C * 2;     // W^T IL R=128 x 64     16 KB
constexpr int OFF_H = OFF_W + DK * C * 2;    // H^T IL R=128 x 128    32 KB
constexpr int OFF_Z = OFF_H + DV * DK * 2;   // Z^T IL R=128 x 64     16 KB
constexpr int OFF_O = OFF_Z + DV * C * 2;    // O   IL R=64  x 128    16 KB
constexpr int OFF_L = OFF_O + C * DV * 2;    // L   fp32 [64][LS]
constexpr int OFF_X = OFF_L + C * LS * 4;    // X   fp32 [64][LS]
constexpr int OFF_B = OFF_X + C * LS * 4;    // beta, s, r  fp32 [3][64]
constexpr int SMEM_BYTES = OFF_B + 3 * C * 4;

// TMEM column map (512 columns allocated)
constexpr uint32_t TM_H = 0, TM_GQK = 128, TM_GKK = 192, TM_W = 256, TM_U = 320, TM_O = 384;

#ifdef DN_DEBUG
// Test-only intermediate dumps (tests/test_tc_debug.py builds with -DDN_DEBUG).
__device__ float* dn_dbg = nullptr;
__device__ int dn_dbg_chunk = 0;
enum { D_L = 0, D_X = 4096, D_GQK = 8192, D_W = 12288, D_U = 20480, D_UP = 28672,
       D_O = 36864, D_H = 45056, D_S = 61440, D_R = 61504, D_B = 61568 };
__device__ void dbg_smem(float* dst, const float* src, int rows, int cols, int stride) {
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x)
    dst[e] = src[(e / cols) * stride + e % cols];
}
__device__ void dbg_tmem(float* dst, uint32_t tm, uint32_t col, int ncols, int M) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < ncols; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr(tm, warp * 32, col + c0), r);
    tmem_ld_wait();
    const int row = M == 128 ? (int)threadIdx.x : (lane < 16 ? warp * 16 + lane : -1);
    if (row >= 0)
      for (int j = 0; j < 16; ++j) dst[row * ncols + c0 + j] = __uint_as_float(r[j]);
  }
}
#define DBG_ON (dn_dbg != nullptr && blockIdx.x == 0 && c == dn_dbg_chunk)
#define DBG(stmt) do { if (DBG_ON) { stmt; } } while (0)
#else
#define DBG(stmt) do { } while (0)
#endif

__global__ void __launch_bounds__(NT, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                  const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mO,
                  Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tslot;
  uint8_t* sQ = smem + OFF_Q;
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  uint8_t* sT = smem + OFF_T;
  uint8_t* sTu = smem + OFF_TU;
  uint8_t* sA = smem + OFF_A;
  uint8_t* sW = smem + OFF_W;
  uint8_t* sH = smem + OFF_H;
  uint8_t* sZ = smem + OFF_Z;
  uint8_t* sO = smem + OFF_O;
  float* Ls = reinterpret_cast<float*>(smem + OFF_L);
  float* Xs = reinterpret_cast<float*>(smem + OFF_X);
  float* sb = reinterpret_cast<float*>(smem + OFF_B);  // beta
  float* ss = sb + C;                                   // 1/||k||
  float* sr = ss + C;                                   // 1/||q||

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = blockIdx.x;
  const int L = a.L, NC = a.NC;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * L;
  uint8_t* states =
      (a.flags & DELTANET_SAVE_STATES) ? (uint8_t*)a.states + (size_t)unit * NC * (DK * DV * 2)
                                       : nullptr;

  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    mbar_fence_init();
    prefetch_tmap(&mQ);
    prefetch_tmap(&mK);
    prefetch_tmap(&mV);
    prefetch_tmap(&mO);
  }
  cta_sync();
  const uint32_t tm = tslot;
  uint32_t ph_tma = 0, ph_mma = 0;

  // ---- initial state: H^T row dv = tid (TMEM lane tid) from h0 [dk][dv]
  {
    const float* h0 = a.h0 ? a.h0 + (size_t)unit * DK * DV : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < DK; c0 += 16) {
      uint32_t r[16];
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        f[j] = h0 ? h0[(size_t)(c0 + j) * DV + tid] : 0.f;
        r[j] = __float_as_uint(f[j]);
      }
      tmem_st16(taddr(tm, warp * 32, TM_H + c0), r);
      il_store8(sH, DV, tid, c0, f);
      il_store8(sH, DV, tid, c0 + 8, f + 8);
    }
    tmem_st_wait();
  }
  fence_proxy_async();
  cta_sync();

  const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aT = smem_u32(sT),
                 aTu = smem_u32(sTu),
                 aA = smem_u32(sA), aW = smem_u32(sW), aH = smem_u32(sH), aZ = smem_u32(sZ);

#pragma unroll 1
  for (int c = 0; c < NC; ++c) {
    const int t0 = c * C;
    // ---- S0: TMA the chunk tiles; beta; save H_c (bf16 image) for the bwd
    if (tid == 0) {
      mbar_expect_tx(&bar_tma, 3 * C * DK * 2);
      tma_load_4d(sQ, &mQ, 0, t0, 0, unit, &bar_tma);
      tma_load_4d(sK, &mK, 0, t0, 0, unit, &bar_tma);
      tma_load_4d(sV, &mV, 0, t0, 0, unit, &bar_tma);
      if (states) {
        bulk_store(states + (size_t)c * DK * DV * 2, sH, DK * DV * 2);
        bulk_commit();
      }
    }
    if (tid < C) sb[tid] = (t0 + tid < L) ? __bfloat162float(beta[t0 + tid]) : 0.f;
    mbar_wait(&bar_tma, ph_tma);
    ph_tma ^= 1;

    // ---- S1: Gram MMAs (M=64, N=64, K=128) + row norms on CUDA cores
    if (tid == 0) {
      fence_after_sync();
      const uint32_t id = idesc_bf16(64, 64, false, false);
#pragma unroll
      for (int k0 = 0; k0 < DK; k0 += 16) {
        mma_bf16(tm + TM_GQK, desc_k(aQ, C, k0), desc_k(aK, C, k0), id, k0 > 0);
        mma_bf16(tm + TM_GKK, desc_k(aK, C, k0), desc_k(aK, C, k0), id, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    {
      // tid < 64: ||q_tid||;  tid >= 64: ||k_{tid-64}||  (fp32 from bf16)
      const int row = tid & 63;
      const uint8_t* tile = tid < 64 ? sQ : sK;
      float acc = 0.f;
#pragma unroll
      for (int g = 0; g < DK / 8; ++g) {
        uint4 v = *reinterpret_cast<const uint4*>(tile + il_off(row, g * 8, C));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          acc = fmaf(f.x, f.x, fmaf(f.y, f.y, acc));
        }
      }
      float inv = l2 ? 1.f / fmaxf(sqrtf(acc), a.eps) : 1.f;
      if (t0 + row >= L) inv = 0.f;  // padded token: exact zero contribution
      (tid < 64 ? sr : ss)[row] = inv;
    }
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1;
    cta_sync();

    // ---- S2: A = tril(Q K^T) (bf16, raw), L = beta_i s_i s_j (k_i.k_j), j < i
    {
      float f[64];
      const int i = warp * 16 + (lane & 15);  // M=64 accumulator row of this lane
      ld64(tm, warp, TM_GQK, f);
      if (lane < 16) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = (g * 8 + e <= i) ? f[g * 8 + e] : 0.f;
          il_store8(sA, C, i, g * 8, x);
        }
      }
      ld64(tm, warp, TM_GKK, f);
      if (lane < 16) {
        const float bi = sb[i] * ss[i];
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
          float4 v;
          v.x = (j + 0 < i) ? bi * ss[j + 0] * f[j + 0] : 0.f;
          v.y = (j + 1 < i) ? bi * ss[j + 1] * f[j + 1] : 0.f;
          v.z = (j + 2 < i) ? bi * ss[j + 2] * f[j + 2] : 0.f;
          v.w = (j + 3 < i) ? bi * ss[j + 3] * f[j + 3] : 0.f;
          *reinterpret_cast<float4*>(Ls + i * LS + j) = v;
        }
      }
    }
    __syncthreads();
    DBG(dbg_smem(dn_dbg + D_L, Ls, C, C, LS); dbg_tmem(dn_dbg + D_GQK, tm, TM_GQK, C, 64);
        dbg_smem(dn_dbg + D_S, ss, 1, C, C); dbg_smem(dn_dbg + D_R, sr, 1, C, C);
        dbg_smem(dn_dbg + D_B, sb, 1, C, C));

    // ---- S3: X = (I + L)^{-1}, two 32x32 diagonal blocks by column-parallel
    // forward substitution, then X21 = -X22 L21 X11.
    if (tid < 64) {
      const int b = tid >> 5, j = lane;
      const int o = 32 * b;
      float x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float acc = 0.f;
#pragma unroll
        for (int m = 0; m < i; m += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(Ls + (o + i) * LS + o + m);
          acc = fmaf(l4.x, x[m], acc);
          if (m + 1 < i) acc = fmaf(l4.y, x[m + 1], acc);
          if (m + 2 < i) acc = fmaf(l4.z, x[m + 2], acc);
          if (m + 3 < i) acc = fmaf(l4.w, x[m + 3], acc);
        }
        x[i] = (i == j) ? 1.f : ((i < j) ? 0.f : -acc);
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        Xs[(o + i) * LS + o + j] = x[i];
        Xs[(o + i) * LS + (32 - o) + j] = 0.f;  // upper block 0; lower-left overwritten below
      }
    }
    __syncthreads();
    {
      // Y = L21 X11 into Ls[0:32][32:64] (unused upper-right block of L)
      const int j = lane, i0 = warp * 8;
      float y[8];
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) y[ii] = 0.f;
#pragma unroll 4
      for (int m = 0; m < 32; ++m) {
        const float xm = Xs[m * LS + j];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) y[ii] = fmaf(Ls[(32 + i0 + ii) * LS + m], xm, y[ii]);
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) Ls[(i0 + ii) * LS + 32 + j] = y[ii];
    }
    __syncthreads();
    {
      // X21 = -X22 Y
      const int j = lane, i0 = warp * 8;
      float y[8];
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) y[ii] = 0.f;
#pragma unroll 4
      for (int m = 0; m < 32; ++m) {
        const float ym = Ls[m * LS + 32 + j];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) y[ii] = fmaf(Xs[(32 + i0 + ii) * LS + 32 + m], ym, y[ii]);
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) Xs[(32 + i0 + ii) * LS + j] = -y[ii];
    }
    __syncthreads();
    {
      // T'[i][j] = X[i][j] beta_j s_j, T''[i][j] = X[i][j] beta_j -> bf16 IL tiles
      const int i = tid >> 1, j0 = (tid & 1) * 32;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float x[8], y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = j0 + g * 8 + e;
          y[e] = Xs[i * LS + j] * sb[j];
          x[e] = y[e] * ss[j];
        }
        il_store8(sT, C, i, j0 + g * 8, x);
        il_store8(sTu, C, i, j0 + g * 8, y);
      }
    }
    DBG(dbg_smem(dn_dbg + D_X, Xs, C, C, LS));
    fence_proxy_async();
    cta_sync();

    // ---- S4: W^T = K^T T'^T, U^T = V^T T''^T  (M=128, N=64, K=64)
    if (tid == 0) {
      const uint32_t id = idesc_bf16(128, 64, true, false);
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16) {
        mma_bf16(tm + TM_W, desc_mn(aK, C, k0), desc_k(aT, C, k0), id, k0 > 0);
        mma_bf16(tm + TM_U, desc_mn(aV, C, k0), desc_k(aTu, C, k0), id, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1;
    fence_after_sync();

    DBG(dbg_tmem(dn_dbg + D_W, tm, TM_W, C, 128); dbg_tmem(dn_dbg + D_U, tm, TM_U, C, 128));
    // ---- S5: W^T (lane = dk) -> bf16 IL tile sW (row dk, cols = tokens)
    {
      float f[64];
      ld64(tm, warp, TM_W, f);
#pragma unroll
      for (int g = 0; g < 8; ++g) il_store8(sW, DK, tid, g * 8, f + g * 8);
    }
    fence_proxy_async();
    cta_sync();

    // ---- S6: U'^T = U^T - H^T W^T (M=128,N=64,K=128), O = Q H (M=64,N=128,K=128)
    if (tid == 0) {
      const uint32_t idn = idesc_bf16(128, 64, false, true, /*neg_a=*/true);
      const uint32_t ido = idesc_bf16(64, 128, false, false);
#pragma unroll
      for (int k0 = 0; k0 < DK; k0 += 16) {
        mma_bf16(tm + TM_U, desc_k(aH, DV, k0), desc_mn(aW, DK, k0), idn, 1);
        mma_bf16(tm + TM_O, desc_k(aQ, C, k0), desc_k(aH, DV, k0), ido, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1;
    fence_after_sync();

    DBG(dbg_tmem(dn_dbg + D_UP, tm, TM_U, C, 128));
    // ---- S7: Z^T[dv][t] = U'^T[dv][t] * s_t -> bf16 IL tile sZ (row dv)
    {
      float f[64];
      ld64(tm, warp, TM_U, f);
#pragma unroll
      for (int t = 0; t < 64; ++t) f[t] *= ss[t];
#pragma unroll
      for (int g = 0; g < 8; ++g) il_store8(sZ, DV, tid, g * 8, f + g * 8);
    }
    fence_proxy_async();
    cta_sync();

    // ---- S8: O += tril(QK^T) Z (M=64,N=128,K=64); H^T += Z^T K (M=128,N=128,K=64)
    if (tid == 0) {
      const uint32_t ido = idesc_bf16(64, 128, false, false);
      const uint32_t idh = idesc_bf16(128, 128, false, true);
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16) {
        mma_bf16(tm + TM_O, desc_k(aA, C, k0), desc_k(aZ, DV, k0), ido, 1);
        mma_bf16(tm + TM_H, desc_k(aZ, DV, k0), desc_mn(aK, C, k0), idh, 1);
      }
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1;
    fence_after_sync();

    DBG(dbg_tmem(dn_dbg + D_O, tm, TM_O, DV, 64); dbg_tmem(dn_dbg + D_H, tm, TM_H, DK, 128));
    // ---- S9: O rows * r -> bf16 -> TMA store; H^T -> bf16 sH (next chunk)
    if (tid == 0) bulk_wait_read0();  // previous O store and state save done reading smem
    __syncthreads();
    {
      const int i = warp * 16 + (lane & 15);
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float f[64];
        ld64(tm, warp, TM_O + 64 * half, f);
        if (lane < 16) {
          const float ri = sr[i];
#pragma unroll
          for (int e = 0; e < 64; ++e) f[e] *= ri;
#pragma unroll
          for (int g = 0; g < 8; ++g) il_store8(sO, C, i, 64 * half + g * 8, f + g * 8);
        }
      }
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float f[64];
        ld64(tm, warp, TM_H + 64 * half, f);
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sH, DV, tid, 64 * half + g * 8, f + g * 8);
      }
    }
    fence_proxy_async();
    cta_sync();
    if (tid == 0 && a.o) {
      tma_store_4d(&mO, sO, 0, t0, 0, unit);
      bulk_commit();
    }
  }

  // ---- final state hT [dk][dv] (fp32), lane dv = tid
  if (a.hT) {
    float* hT = a.hT + (size_t)unit * DK * DV;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      float f[64];
      ld64(tm, warp, TM_H + 64 * half, f);
#pragma unroll
      for (int e = 0; e < 64; ++e) hT[(size_t)(64 * half + e) * DV + tid] = f[e];
    }
  }
  if (tid == 0) bulk_wait0();
  cta_sync();
  if (warp == 0) tmem_dealloc<512>(tm);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

}  // namespace

// 4-D view {8 elems, L rows, D/8 column groups, B*H units} of a [B*H][L][D]
// bf16 tensor; a box {8, 64, D/8, 1} lands in smem as the IL layout (R=64).
bool make_il_map(CUtensorMap* m, const void* base, int BH, int L, int D, int rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {8, (cuuint64_t)L, (cuuint64_t)(D / 8), (cuuint64_t)BH};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, 16, (cuuint64_t)L * D * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)rows, (cuuint32_t)(D / 8), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tc_supported(const deltanet_desc* d) {
  return d->dtype == DELTANET_BF16 && d->chunk == C && d->Dk == DK && d->Dv == DV && d->L > 0;
}

size_t tc_scratch_bytes(const deltanet_desc*) { return 0; }  // states region only

// fwd: 1 kernel; bwd: 1 kernel, plus the state-recompute forward without SAVE_STATES
int tc_launch_count(const deltanet_desc* d, int which) {
  return which == 0 ? 1 : ((d->flags & DELTANET_SAVE_STATES) ? 1 : 2);
}

int tc_fwd(const Args& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap mQ, mK, mV, mO;
  if (!make_il_map(&mQ, a.q, BH, a.L, DK, C) || !make_il_map(&mK, a.k, BH, a.L, DK, C) ||
      !make_il_map(&mV, a.v, BH, a.L, DV, C) ||
      !make_il_map(&mO, a.o ? a.o : a.v, BH, a.L, DV, C))  // o == null: states only
    return DELTANET_ERR_CUDA;
  tc_fwd_kernel<<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}


}  // namespace dn

#ifdef DN_DEBUG
extern "C" int dn_debug_set(float* buf, int chunk) {
  if (cudaMemcpyToSymbol(dn::dn_dbg, &buf, sizeof(buf)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(dn::dn_dbg_chunk, &chunk, sizeof(int)) != cudaSuccess) return 1;
  return 0;
}
#endif
