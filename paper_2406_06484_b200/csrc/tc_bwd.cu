// tc_bwd.cu -- fused sm_100a backward of the chunkwise DeltaNet layer.
//
// The paper gives no backward (PAPER.md line 250 only says states are
// recomputed; reading R12).  This kernel evaluates the exact
// adjoint of Eq. 8-11 chunk by chunk in reverse (DESIGN.md §Backward,
// SURVEY App. A.2), one CTA per (b, h) unit, with dH = dl/dH_{t+1} held in
// TMEM (fp32, lanes = d_v) across chunks and the chunk-boundary states H_t
// read from the workspace image the forward wrote.
//
// Per chunk (q_hat, k_hat: L2-normalised rows, rounded to bf16 in smem):
//   recompute  A = tril(Q K^T), L = tril(diag(b) K K^T, -1), X = (I+L)^{-1},
//              T = X diag(b), W = T K, U = T V, U' = U - W H, R = V - K H
//   chain      dU' = K dH + A^T dO
//              dH <- dH + Q^T dO - W^T dU'
//   local      dA = tril(dO U'^T)          P = X^T dU'  (= dV_beta)
//              dX = (dU' R^T) diag(b)      Y = X^T dX,  G = tril(-Y X^T, -1)
//              dQ = dO H^T + dA K
//              dK = U' dH^T + dA^T Q - dV H^T + (diag(b) G + G^T diag(b)) K
//              dV = diag(b) P
//              dbeta = rowsum(P . R) + rowsum(G . K K^T)
//   then the L2-normalisation adjoint on dQ, dK (R9).
// (dK_beta = X^T dW = -P H^T, and rowsum(dK_beta . K) + rowsum(P . V) =
//  rowsum(P . R) -- DESIGN.md §Backward.)
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

using namespace tc;

constexpr int C = 64, D = 128, NT = 128;
constexpr int LS = 68;
constexpr uint32_t LO16 = 16u << 16;  // TMEM lane offset 16 (second M=64 accumulator)

// ---- shared memory map (bytes); regions reused by lifetime
constexpr int OFF_Q = 0;          // q_hat  IL R=64 x 128   (whole chunk)
constexpr int OFF_K = 16384;      // k_hat  IL R=64 x 128   (whole chunk)
constexpr int OFF_DO = 32768;     // dO     IL R=64 x 128   (whole chunk)
constexpr int OFF_H = 49152;      // H^T    IL R=128 x 128  (-> dq staging)
constexpr int OFF_DH = 81920;     // dH^T   IL R=128 x 128  (-> dk staging)
constexpr int OFF_UP = 114688;    // U'^T   IL R=128 x 64
constexpr int OFF_X = 131072;     // X      IL R=64 x 64
constexpr int OFF_W = 139264;     // W^T    IL R=128 x 64
constexpr int OFF_V = 155648;     // V      IL R=64 x 128   (-> dV staging)
constexpr int OFF_S = 172032;     // region S (51200 B), see below
constexpr int S_L = OFF_S;                // Ls fp32 | dU'^T | Y, Mg
constexpr int S_X = OFF_S + 17408;        // Xs fp32 | R    | G fp32
constexpr int S_T = OFF_S + 34816;        // T      | dA
constexpr int S_A = OFF_S + 43008;        // A      | dX
constexpr int OFF_B = OFF_S + 51200;      // 6 x 64 floats
constexpr int SMEM_BYTES = OFF_B + 6 * C * 4;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

// ---- TMEM column map (512 columns)
constexpr uint32_t TM_DH = 0;                       // dH^T, M=128
constexpr uint32_t TM_GKK = 128, TM_Y = 128 | LO16; // M=64 pair
constexpr uint32_t TM_GQK = 192, TM_DA = 192, TM_GB = 192, TM_DX = 192 | LO16;
constexpr uint32_t TM_W = 256, TM_DU = 256, TM_U = 320;   // M=128 (B1-B3)
constexpr uint32_t TM_P = 256, TM_DK = 256 | LO16;        // M=64 pair, 128 cols (B4-)
constexpr uint32_t TM_R = 384, TM_DQ = 384;               // M=64, 128 cols

__global__ void __launch_bounds__(NT, 1)
    tc_bwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                  const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mDO,
                  const __grid_constant__ CUtensorMap mDQ, const __grid_constant__ CUtensorMap mDK,
                  const __grid_constant__ CUtensorMap mDV, Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tslot;
  uint8_t *sQ = smem + OFF_Q, *sK = smem + OFF_K, *sDO = smem + OFF_DO, *sH = smem + OFF_H,
          *sDH = smem + OFF_DH, *sUP = smem + OFF_UP, *sX = smem + OFF_X, *sW = smem + OFF_W,
          *sV = smem + OFF_V;
  float* Ls = reinterpret_cast<float*>(smem + S_L);
  float* Xs = reinterpret_cast<float*>(smem + S_X);
  uint8_t* sT = smem + S_T;
  uint8_t* sA = smem + S_A;
  uint8_t* sDUP = smem + S_L;  // after the substitution
  uint8_t* sR = smem + S_X;
  uint8_t* sDA = smem + S_T;
  uint8_t* sDX = smem + S_A;
  uint8_t* sY = smem + S_L;          // after B4
  uint8_t* sMG = smem + S_L + 8192;  // after B4
  float* Gs = reinterpret_cast<float*>(smem + S_X);  // after B4
  uint8_t* sDV = sV;
  uint8_t* sDQo = sH;
  uint8_t* sDKo = sDH;
  float* sb = reinterpret_cast<float*>(smem + OFF_B);  // beta
  float* sr = sb + C;                                   // 1/max(||q||,eps) (0: padded)
  float* ss = sr + C;                                   // 1/max(||k||,eps)
  float* nq = ss + C;                                   // ||q||
  float* nk = nq + C;                                   // ||k||
  float* sdb = nk + C;                                  // dbeta partial

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r64 = warp * 16 + (lane & 15);  // M=64 accumulator row of this lane
  const bool lo = lane < 16;                // lane+0 accumulator (else lane+16)
  const int unit = blockIdx.x;
  const int L = a.L, NC = a.NC;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const float eps = a.eps;
  const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * L;
  __nv_bfloat16* dbeta = (__nv_bfloat16*)a.dbeta + (size_t)unit * L;
  const uint8_t* states = (const uint8_t*)a.states + (size_t)unit * NC * (D * D * 2);

  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    mbar_fence_init();
  }
  cta_sync();
  const uint32_t tm = tslot;
  uint32_t ph_tma = 0, ph_mma = 0;
  auto mma_wait = [&]() {
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1;
    fence_after_sync();
  };

  // dH^T <- dhT^T (lane dv = tid)
  {
    const float* dhT = a.dhT ? a.dhT + (size_t)unit * D * D : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(dhT ? dhT[(size_t)(c0 + j) * D + tid] : 0.f);
      tmem_st16(taddr(tm, warp * 32, TM_DH + c0), r);
    }
    tmem_st_wait();
  }
  cta_sync();

  const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aDO = smem_u32(sDO), aH = smem_u32(sH),
                 aDH = smem_u32(sDH), aUP = smem_u32(sUP), aX = smem_u32(sX),
                 aW = smem_u32(sW), aV = smem_u32(sV), aT = smem_u32(sT), aA = smem_u32(sA),
                 aDUP = smem_u32(sDUP), aR = smem_u32(sR), aDA = smem_u32(sDA),
                 aDX = smem_u32(sDX), aY = smem_u32(sY), aMG = smem_u32(sMG),
                 aDV = smem_u32(sDV);

#pragma unroll 1
  for (int c = NC - 1; c >= 0; --c) {
    const int t0 = c * C;
    // ---------------- L0: loads (previous chunk's stores must be done reading smem)
    if (tid == 0) {
      bulk_wait_read0();
      mbar_expect_tx(&bar_tma, 4 * C * D * 2 + D * D * 2);
      tma_load_4d(sQ, &mQ, 0, t0, 0, unit, &bar_tma);
      tma_load_4d(sK, &mK, 0, t0, 0, unit, &bar_tma);
      tma_load_4d(sV, &mV, 0, t0, 0, unit, &bar_tma);
      tma_load_4d(sDO, &mDO, 0, t0, 0, unit, &bar_tma);
      bulk_load(sH, states + (size_t)c * D * D * 2, D * D * 2, &bar_tma);
    }
    __syncthreads();
    if (tid < C) sb[tid] = (t0 + tid < L) ? __bfloat162float(beta[t0 + tid]) : 0.f;
    {  // L1: dH^T (dl/dH_{c+1}) -> bf16 image for this chunk's MMAs
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float f[64];
        ld64(tm, warp, TM_DH + 64 * half, f);
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sDH, D, tid, 64 * half + g * 8, f + g * 8);
      }
    }
    mbar_wait(&bar_tma, ph_tma);
    ph_tma ^= 1;
    {  // normalise q (tid < 64) / k (tid >= 64) rows in place (R9)
      const int row = tid & 63;
      uint8_t* tile = tid < 64 ? sQ : sK;
      float acc = 0.f;
#pragma unroll
      for (int g = 0; g < D / 8; ++g) {
        float x[8];
        il_load8(tile, C, row, g * 8, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(x[e], x[e], acc);
      }
      const float n = sqrtf(acc);
      float inv = l2 ? 1.f / fmaxf(n, eps) : 1.f;
      if (t0 + row >= L) inv = 0.f;
      if (l2) {
#pragma unroll
        for (int g = 0; g < D / 8; ++g) {
          float x[8];
          il_load8(tile, C, row, g * 8, x);
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] *= inv;
          il_store8(tile, C, row, g * 8, x);
        }
      }
      (tid < 64 ? sr : ss)[row] = inv;
      (tid < 64 ? nq : nk)[row] = n;
    }
    fence_proxy_async();
    cta_sync();

    // ---------------- B1: Gram (M=64): Q K^T, K K^T
    if (tid == 0) {
      const uint32_t id = idesc_bf16(64, 64, false, false);
#pragma unroll
      for (int k0 = 0; k0 < D; k0 += 16) {
        mma_bf16(tm + TM_GQK, desc_k(aQ, C, k0), desc_k(aK, C, k0), id, k0 > 0);
        mma_bf16(tm + TM_GKK, desc_k(aK, C, k0), desc_k(aK, C, k0), id, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      float f[64];
      ld64(tm, warp, TM_GQK, f);
      if (lo) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = (g * 8 + e <= r64) ? f[g * 8 + e] : 0.f;
          il_store8(sA, C, r64, g * 8, x);
        }
      }
      ld64(tm, warp, TM_GKK, f);
      if (lo) {
        const float bi = sb[r64];
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
          float4 v;
          v.x = (j + 0 < r64) ? bi * f[j + 0] : 0.f;
          v.y = (j + 1 < r64) ? bi * f[j + 1] : 0.f;
          v.z = (j + 2 < r64) ? bi * f[j + 2] : 0.f;
          v.w = (j + 3 < r64) ? bi * f[j + 3] : 0.f;
          *reinterpret_cast<float4*>(Ls + r64 * LS + j) = v;
        }
      }
    }
    __syncthreads();
    // substitution X = (I + L)^{-1} (same blocking as the forward kernel)
    if (tid < 64) {
      const int b = tid >> 5, j = lane, o = 32 * b;
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
        Xs[(o + i) * LS + (32 - o) + j] = 0.f;
      }
    }
    __syncthreads();
    {
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
    {  // X -> bf16 sX;  T = X diag(beta) -> bf16 sT
      const int i = tid >> 1, j0 = (tid & 1) * 32;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float x[8], y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = j0 + g * 8 + e;
          x[e] = Xs[i * LS + j];
          y[e] = x[e] * sb[j];
        }
        il_store8(sX, C, i, j0 + g * 8, x);
        il_store8(sT, C, i, j0 + g * 8, y);
      }
    }
    fence_proxy_async();
    cta_sync();

    // ---------------- B1b: W^T = K^T T^T, U^T = V^T T^T (M=128, N=64, K=64)
    if (tid == 0) {
      const uint32_t id = idesc_bf16(128, 64, true, false);
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16) {
        mma_bf16(tm + TM_W, desc_mn(aK, C, k0), desc_k(aT, C, k0), id, k0 > 0);
        mma_bf16(tm + TM_U, desc_mn(aV, C, k0), desc_k(aT, C, k0), id, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      float f[64];
      ld64(tm, warp, TM_W, f);
#pragma unroll
      for (int g = 0; g < 8; ++g) il_store8(sW, D, tid, g * 8, f + g * 8);
    }
    fence_proxy_async();
    cta_sync();

    // ---------------- B2: U' = U - W H ; K H (for R) ; dU'^T = dH^T K^T + dO^T A
    if (tid == 0) {
      const uint32_t idn = idesc_bf16(128, 64, false, true, true);
      const uint32_t idr = idesc_bf16(64, 128, false, false);
      const uint32_t idd = idesc_bf16(128, 64, false, false);
      const uint32_t ida = idesc_bf16(128, 64, true, true);
#pragma unroll
      for (int k0 = 0; k0 < D; k0 += 16) {
        mma_bf16(tm + TM_U, desc_k(aH, D, k0), desc_mn(aW, D, k0), idn, 1);
        mma_bf16(tm + TM_R, desc_k(aK, C, k0), desc_k(aH, D, k0), idr, k0 > 0);
        mma_bf16(tm + TM_DU, desc_k(aDH, D, k0), desc_k(aK, C, k0), idd, k0 > 0);
      }
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16)
        mma_bf16(tm + TM_DU, desc_mn(aDO, C, k0), desc_mn(aA, C, k0), ida, 1);
      mma_commit(&bar_mma);
    }
    mma_wait();
    {  // B3: U'^T, dU'^T -> bf16 (rows d_v);  R = V - K H -> bf16 (rows t)
      float f[64];
      ld64(tm, warp, TM_U, f);
#pragma unroll
      for (int g = 0; g < 8; ++g) il_store8(sUP, D, tid, g * 8, f + g * 8);
      ld64(tm, warp, TM_DU, f);
#pragma unroll
      for (int g = 0; g < 8; ++g) il_store8(sDUP, D, tid, g * 8, f + g * 8);
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        ld64(tm, warp, TM_R + 64 * half, f);
        if (lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float v8[8];
            il_load8(sV, C, r64, 64 * half + g * 8, v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) v8[e] -= f[g * 8 + e];
            il_store8(sR, C, r64, 64 * half + g * 8, v8);
          }
        }
      }
    }
    fence_proxy_async();
    cta_sync();

    // ---------------- B4: dA, P, dX, dH update, dK += U' dH^T
    if (tid == 0) {
      const uint32_t id_da = idesc_bf16(64, 64, false, true);
      const uint32_t id_p = idesc_bf16(64, 128, true, false);
      const uint32_t id_dx = idesc_bf16(64, 64, true, false);
      const uint32_t id_h1 = idesc_bf16(128, 128, true, true);
      const uint32_t id_h2 = idesc_bf16(128, 128, false, false, true);
      const uint32_t id_dk = idesc_bf16(64, 128, true, true);
#pragma unroll
      for (int k0 = 0; k0 < D; k0 += 16) {
        mma_bf16(tm + TM_DA, desc_k(aDO, C, k0), desc_mn(aUP, D, k0), id_da, k0 > 0);
        mma_bf16(tm + TM_DX, desc_mn(aDUP, D, k0), desc_k(aR, C, k0), id_dx, k0 > 0);
        mma_bf16(tm + TM_DK, desc_mn(aUP, D, k0), desc_mn(aDH, D, k0), id_dk, k0 > 0);
      }
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16) {
        mma_bf16(tm + TM_P, desc_mn(aX, C, k0), desc_k(aDUP, D, k0), id_p, k0 > 0);
        mma_bf16(tm + TM_DH, desc_mn(aDO, C, k0), desc_mn(aQ, C, k0), id_h1, 1);
        mma_bf16(tm + TM_DH, desc_k(aDUP, D, k0), desc_k(aW, D, k0), id_h2, 1);
      }
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      float f[64];
      ld64(tm, warp, TM_DA, f);  // lanes<16: dA row r64; lanes>=16: dX' row r64
      if (lo) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = (g * 8 + e <= r64) ? f[g * 8 + e] : 0.f;
          il_store8(sDA, C, r64, g * 8, x);
        }
      } else {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = f[g * 8 + e] * sb[g * 8 + e];
          il_store8(sDX, C, r64, g * 8, x);
        }
      }
      float db = 0.f;
      const float bt = sb[r64];
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float p[64];
        ld64(tm, warp, TM_P + 64 * half, p);  // lanes<16: P row
        ld64(tm, warp, TM_R + 64 * half, f);  // lanes<16: (K H) row
        if (lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float v8[8], dv8[8];
            il_load8(sV, C, r64, 64 * half + g * 8, v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              db = fmaf(p[g * 8 + e], v8[e] - f[g * 8 + e], db);  // P . R
              dv8[e] = bt * p[g * 8 + e];
            }
            il_store8(sDV, C, r64, 64 * half + g * 8, dv8);
          }
        }
      }
      if (lo) sdb[r64] = db;
    }
    fence_proxy_async();
    cta_sync();
    if (tid == 0) {
      tma_store_4d(&mDV, sDV, 0, t0, 0, unit);
      bulk_commit();
    }

    // ---------------- B5: dQ = dO H^T + dA K ; dK += dA^T Q - dV H^T ; Y = X^T dX
    if (tid == 0) {
      const uint32_t id_q1 = idesc_bf16(64, 128, false, true);
      const uint32_t id_k1 = idesc_bf16(64, 128, true, true);
      const uint32_t id_k2 = idesc_bf16(64, 128, false, true, true);
      const uint32_t id_y = idesc_bf16(64, 64, true, true);
#pragma unroll
      for (int k0 = 0; k0 < D; k0 += 16) {
        mma_bf16(tm + TM_DQ, desc_k(aDO, C, k0), desc_mn(aH, D, k0), id_q1, k0 > 0);
        mma_bf16(tm + TM_DK, desc_k(aDV, C, k0), desc_mn(aH, D, k0), id_k2, 1);
      }
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16) {
        mma_bf16(tm + TM_DQ, desc_k(aDA, C, k0), desc_mn(aK, C, k0), id_q1, 1);
        mma_bf16(tm + TM_DK, desc_mn(aDA, C, k0), desc_mn(aQ, C, k0), id_k1, 1);
        mma_bf16(tm + TM_Y, desc_mn(aX, C, k0), desc_mn(aDX, C, k0), id_y, k0 > 0);
      }
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      // lanes<16: dq_hat row -> L2 adjoint -> dq staging; lanes>=16: Y row -> sY
      float f[64];
      float dot = 0.f;
      const float inv = sr[r64];
      const bool big = l2 && nq[r64] >= eps;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        ld64(tm, warp, TM_DQ + 64 * half, f);
        if (lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float q8[8];
            il_load8(sQ, C, r64, 64 * half + g * 8, q8);
#pragma unroll
            for (int e = 0; e < 8; ++e) dot = fmaf(q8[e], f[g * 8 + e], dot);
          }
        }
      }
      if (!big) dot = 0.f;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        ld64(tm, warp, TM_DQ + 64 * half, f);
        if (lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float q8[8];
            il_load8(sQ, C, r64, 64 * half + g * 8, q8);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              q8[e] = l2 ? inv * (f[g * 8 + e] - q8[e] * dot) : f[g * 8 + e];
            il_store8(sDQo, C, r64, 64 * half + g * 8, q8);
          }
        }
      }
      ld64(tm, warp, TM_GKK, f);  // lanes>=16 see Y (TM_Y = TM_GKK | lane 16)
      if (!lo) {
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sY, C, r64, g * 8, f + g * 8);
      }
    }
    fence_proxy_async();
    cta_sync();
    if (tid == 0) {
      tma_store_4d(&mDQ, sDQo, 0, t0, 0, unit);
      bulk_commit();
      // ---------------- B7: G = -Y X^T (M=64, N=64, K=64)
      const uint32_t id_g = idesc_bf16(64, 64, false, false, true);
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16)
        mma_bf16(tm + TM_GB, desc_k(aY, C, k0), desc_k(aX, C, k0), id_g, k0 > 0);
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      // lanes<16: G row -> Gs (strict lower); dbeta += rowsum(G . K K^T)
      float g64[64], kk[64];
      ld64(tm, warp, TM_GB, g64);
      ld64(tm, warp, TM_GKK, kk);
      if (lo) {
        float db = sdb[r64];
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
          float4 v;
          v.x = (j + 0 < r64) ? g64[j + 0] : 0.f;
          v.y = (j + 1 < r64) ? g64[j + 1] : 0.f;
          v.z = (j + 2 < r64) ? g64[j + 2] : 0.f;
          v.w = (j + 3 < r64) ? g64[j + 3] : 0.f;
          db = fmaf(v.x, kk[j], fmaf(v.y, kk[j + 1], fmaf(v.z, kk[j + 2], fmaf(v.w, kk[j + 3], db))));
          *reinterpret_cast<float4*>(Gs + r64 * LS + j) = v;
        }
        if (t0 + r64 < L) dbeta[t0 + r64] = __float2bfloat16_rn(db);
      }
    }
    __syncthreads();
    {  // Mg[i][j] = b_i G[i][j] + b_j G[j][i]  -> bf16 (row i, 32 columns per thread)
      const int i = tid >> 1, j0 = (tid & 1) * 32;
      const float bi = sb[i];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = j0 + g * 8 + e;
          x[e] = bi * Gs[i * LS + j] + sb[j] * Gs[j * LS + i];
        }
        il_store8(sMG, C, i, j0 + g * 8, x);
      }
    }
    fence_proxy_async();
    cta_sync();
    // ---------------- B9: dK += Mg K
    if (tid == 0) {
      const uint32_t id_m = idesc_bf16(64, 128, false, true);
#pragma unroll
      for (int k0 = 0; k0 < C; k0 += 16)
        mma_bf16(tm + TM_DK, desc_k(aMG, C, k0), desc_mn(aK, C, k0), id_m, 1);
      mma_commit(&bar_mma);
    }
    mma_wait();
    {
      // lanes>=16: dk_hat row -> L2 adjoint -> dk staging
      float f[64];
      float dot = 0.f;
      const float inv = ss[r64];
      const bool big = l2 && nk[r64] >= eps;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        ld64(tm, warp, TM_P + 64 * half, f);  // lanes>=16 read TM_DK
        if (!lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float k8[8];
            il_load8(sK, C, r64, 64 * half + g * 8, k8);
#pragma unroll
            for (int e = 0; e < 8; ++e) dot = fmaf(k8[e], f[g * 8 + e], dot);
          }
        }
      }
      if (!big) dot = 0.f;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        ld64(tm, warp, TM_P + 64 * half, f);
        if (!lo) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float k8[8];
            il_load8(sK, C, r64, 64 * half + g * 8, k8);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              k8[e] = l2 ? inv * (f[g * 8 + e] - k8[e] * dot) : f[g * 8 + e];
            il_store8(sDKo, C, r64, 64 * half + g * 8, k8);
          }
        }
      }
    }
    fence_proxy_async();
    cta_sync();
    if (tid == 0) {
      tma_store_4d(&mDK, sDKo, 0, t0, 0, unit);
      bulk_commit();
    }
  }

  // dh0 = dH (orientation [dk][dv]; lane dv = tid)
  if (a.dh0) {
    float* dh0 = a.dh0 + (size_t)unit * D * D;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      float f[64];
      ld64(tm, warp, TM_DH + 64 * half, f);
#pragma unroll
      for (int e = 0; e < 64; ++e) dh0[(size_t)(64 * half + e) * D + tid] = f[e];
    }
  }
  if (tid == 0) bulk_wait0();
  cta_sync();
  if (warp == 0) tmem_dealloc<512>(tm);
}

}  // namespace

int tc_fwd(const Args& a, cudaStream_t s);

int tc_bwd(const Args& a0, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr = true;
  }
  Args a = a0;
  if (!(a.flags & DELTANET_SAVE_STATES)) {
    // recompute the chunk states with the forward kernel (no O store)
    Args f = a0;
    f.flags |= DELTANET_SAVE_STATES;
    f.o = nullptr;
    f.hT = nullptr;
    int rc = tc_fwd(f, s);
    if (rc) return rc;
  }
  const int BH = a.B * a.H;
  CUtensorMap mQ, mK, mV, mDO, mDQ, mDK, mDV;
  if (!make_il_map(&mQ, a.q, BH, a.L, D, C) || !make_il_map(&mK, a.k, BH, a.L, D, C) ||
      !make_il_map(&mV, a.v, BH, a.L, D, C) || !make_il_map(&mDO, a.dO, BH, a.L, D, C) ||
      !make_il_map(&mDQ, a.dq, BH, a.L, D, C) || !make_il_map(&mDK, a.dk, BH, a.L, D, C) ||
      !make_il_map(&mDV, a.dv, BH, a.L, D, C))
    return DELTANET_ERR_CUDA;
  tc_bwd_kernel<<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

}  // namespace dn
