// tc_split.cu -- the tcgen05 "split" path of the chunkwise DeltaNet layer for
// head dims whose per-unit working set does not fit one SM (d = 256: the fp32
// state alone is 256 KB = all of TMEM; BASELINE configs[3]), and for d = 64.
// (d = 128 runs the fused one-CTA-per-unit kernels of tc_fwd.cu / tc_bwd.cu;
// DELTANET_FORCE_SPLIT selects this path there too, for cross-checking.)
//
// Same mathematics as the fused kernels (§3.2 Eq. 8-11, lines
// 166-182; backward = the exact adjoint, R12 / §4.2), decomposed
// FLA-style into chunk-parallel and state-chain kernels:
//
//   sp_prep_kernel      one CTA per (unit, chunk), chunk-parallel: q, k row
//                       norms and q_hat, k_hat (bf16, to the workspace), the
//                       Gram pair Q_hat K_hat^T | K_hat K_hat^T (tcgen05),
//                       A = tril(Q_hat K_hat^T), L = tril(diag(beta) K_hat
//                       K_hat^T, -1), X = (I + L)^{-1} (forward substitution,
//                       tc_common.cuh), T = X diag(beta), W^T = K_hat^T T^T
//                       (tcgen05; W = T K_hat, Eq. 11).
//   sp_fwd_chain_kernel one CTA per (unit, 64-column block j of d_v): the
//                       columns of the state evolve independently (S is
//                       d_v x d_k; H = S^T), so H_j^T (64 x d_k fp32) stays in
//                       TMEM across the chunks:
//                         U_j^T  = V_j^T T^T                 (Eq. 11)
//                         U'_j^T = U_j^T - H_j^T W^T         (Eq. 8-9)
//                         O_j    = Q_hat H_j + A U'_j        (Eq. 9)
//                         H_j^T += U'_j^T K_hat              (Eq. 8)
//   sp_bwd_chain_kernel one CTA per (unit, d_v block j), reverse over chunks:
//                       dH_j^T (dl/dH, 64 x d_k fp32) in TMEM,
//                         dU'_j^T = dH_j^T K_hat^T + dO_j^T A
//                         P_j = X^T dU'_j,  dV_j = diag(beta) P_j   (output)
//                         R_j = V_j - K_hat H_j,  rowsum(P_j . R_j) (dbeta part)
//                         dH_j^T += dO_j^T Q_hat - dV_j^T K_hat
//   sp_bwd_local_kernel one CTA per (unit, chunk), chunk-parallel, looping
//                       over the d_v blocks v for the d_v contractions:
//                         dA = tril(dO U'^T), dX = dU' R^T diag(beta),
//                         dQ_hat = dO H^T + dA K_hat,
//                         dK_hat = U' dH^T - dV H^T + dA^T Q_hat + (G1 + G1^T) K_hat,
//                         Y = X^T dX, G = -Y X^T, G1 = diag(beta) tril(G, -1),
//                         dbeta = rowsum(P . R) + rowsum(tril(G,-1) . K_hat K_hat^T),
//                       then the L2-normalisation adjoint (R9) on dq, dk.
//
// Every operand tile is the IL layout of tc_common.cuh (TMA boxes for the
// [B,H,L,d] tensors, bulk copies of smem images for the records); every
// accumulator with a 64-row side is an M = 64 tcgen05 accumulator (rows in
// TMEM lanes 0-15 of each 32-lane quadrant, a second one at lane offset 16).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

using namespace tc;

constexpr int C = 64, LS = 68;
constexpr uint32_t LO16 = 16u << 16;
constexpr int BLK = C * 64 * 2;  // 64 x 64 bf16 IL tile (8 KB)

#ifdef DN_TIMING
// Test-only phase stamps (tools/sp_timeline.py, -DDN_TIMING): clock64 of CTA
// (0, 0) of the chain kernels per chunk iteration (32 slots), and of CTA
// (NC / 2, 0) of the local kernel per sub-step.
__device__ long long* sp_tim = nullptr;
__device__ int sp_tim_kernel = 0;  // 1 fwd chain, 2 bwd chain, 3 bwd local
#define SPT(K, it, slot)                                                                 \
  do {                                                                                   \
    if (sp_tim != nullptr && sp_tim_kernel == (K) && blockIdx.y == 0 &&                  \
        blockIdx.x == ((K) == 3 ? gridDim.x / 2 : 0))                                    \
      sp_tim[(size_t)(it) * 32 + (slot)] = clock64();                                    \
  } while (0)
#else
#define SPT(K, it, slot) do { } while (0)
#endif

template <int D>
struct SP {
  static constexpr int NB = D / 64;        // d_v blocks
  static constexpr int TILE = C * D * 2;   // 64 x D bf16
  static constexpr int WT = D * C * 2;     // W^T image, D x 64
  static constexpr int HIMG = 64 * D * 2;  // H_j^T image, 64 x D
  // per (unit, chunk) record written by the prep kernel
  static constexpr int R1_X = 0, R1_T = BLK, R1_A = 2 * BLK, R1_N = 3 * BLK;
  static constexpr int R1_W = 3 * BLK + 512;
  static constexpr int R1_BYTES = R1_W + WT;
  // per (unit, chunk, d_v block) record (fwd chain: U'; bwd chain: dU', R, db, dH)
  static constexpr int R2_U = 0, R2_DU = BLK, R2_R = 2 * BLK, R2_DB = 3 * BLK;
  static constexpr int R2_DH = 3 * BLK + 256;
  static constexpr int R2_BYTES = R2_DH + HIMG;
};

// workspace layout of the split path (after the states region, which holds
// the H_j^T images [unit][chunk][block], 64 x D bf16 each)
struct SpLayout {
  // normalised q, k as per-(unit, chunk) IL smem images (64 x D bf16 each):
  // one contiguous bulk copy per tile (a [B,H,L,D] TMA box moves 16 B rows)
  uint8_t *qh, *kh;
  uint8_t *rec1, *rec2;
};
template <int D>
__host__ __device__ inline SpLayout sp_layout(const Args& a) {
  SpLayout s;
  const size_t qk = (size_t)a.B * a.H * a.NC * SP<D>::TILE;
  uint8_t* base = reinterpret_cast<uint8_t*>(a.scratch);
  s.qh = base;
  s.kh = base + qk;
  s.rec1 = base + 2 * qk;
  s.rec2 = s.rec1 + (size_t)a.B * a.H * a.NC * SP<D>::R1_BYTES;
  return s;
}

__device__ __forceinline__ void ld16(uint32_t tm, int wq, uint32_t col, float (&f)[16]) {
  uint32_t r[16];
  tmem_ld16(taddr(tm, wq * 32, col), r);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void ld32f(uint32_t tm, int wq, uint32_t col, float (&f)[32]) {
  uint32_t r[2][16];
  tmem_ld16(taddr(tm, wq * 32, col), r[0]);
  tmem_ld16(taddr(tm, wq * 32, col + 16), r[1]);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) f[16 * i + j] = __uint_as_float(r[i][j]);
}

// 8 fp32 -> 8 bf16 (16 B) to global memory
__device__ __forceinline__ void stg8(void* dst, const float* x) {
  uint4 v;
  v.x = pack_bf16(x[0], x[1]);
  v.y = pack_bf16(x[2], x[3]);
  v.z = pack_bf16(x[4], x[5]);
  v.w = pack_bf16(x[6], x[7]);
  *reinterpret_cast<uint4*>(dst) = v;
}

// SIMT (256 threads, named barrier 1) -> control thread hand-off
__device__ __forceinline__ void hand_off(uint64_t* bar, int tid) {
  fence_proxy_async();
  fence_before_sync();
  grp_sync<256>(1);
  if (tid == 0) mbar_arrive(bar);
}

// ============================================================== prep kernel
template <int D>
__global__ void __launch_bounds__(288, 2)
    sp_prep_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                   Args a) {
  using S = SP<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + S::TILE;
  float* LX = reinterpret_cast<float*>(sK + S::TILE);  // [64][LS]
  float* part = LX + C * LS;                            // [2 tiles][4][64] sums of squares
  float* vb = part + 2 * 4 * C;                         // beta [64]
  float* nrm = vb + C;                                  // record: ||k|| [64] | ||q|| [64]
  uint8_t* sT = reinterpret_cast<uint8_t*>(nrm + 2 * C);
  uint8_t* sA = sT + BLK;
  uint8_t* sX = sA + BLK;
  // the W^T image reuses the q_hat tile once the Gram product and the q_hat
  // store have read it (q_free): 108 KB at d = 256, two CTAs per SM
  uint8_t* sW = sQ;
  static_assert(SP<D>::WT == SP<D>::TILE, "W^T image over the q tile");
  __shared__ uint64_t ld_full, norm_done, g_done, t_ready, w_done, w_img, q_free;
  __shared__ uint32_t tslot;
  constexpr uint32_t TM_G = 0, TM_W = 64;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x, unit = blockIdx.y, t0 = c * C;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const SpLayout ly = sp_layout<D>(a);
  uint8_t* rec = ly.rec1 + ((size_t)unit * a.NC + c) * S::R1_BYTES;

  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 256) {
    mbar_init(&ld_full, 1);
    mbar_init(&norm_done, 1);
    mbar_init(&g_done, 1);
    mbar_init(&t_ready, 1);
    mbar_init(&w_done, 1);
    mbar_init(&w_img, 1);
    mbar_init(&q_free, 1);
    mbar_fence_init();
    mbar_expect_tx(&ld_full, 2 * S::TILE);
    tma_load_4d(sQ, &mQ, 0, t0, 0, unit, &ld_full);
    tma_load_4d(sK, &mK, 0, t0, 0, unit, &ld_full);
  }
  cta_sync();
  const uint32_t tm = tslot;

  if (warp == 8) {
    if (lane == 0) {
      const uint32_t aq = smem_u32(sQ), ak = smem_u32(sK), at = smem_u32(sT);
      mbar_wait(&norm_done, 0);
      const size_t img = ((size_t)unit * a.NC + c) * S::TILE;
      bulk_store(ly.qh + img, sQ, S::TILE);
      bulk_store(ly.kh + img, sK, S::TILE);
      bulk_commit();
      fence_after_sync();
      const uint32_t idg = idesc_bf16(64, 64, false, false);
#pragma unroll 4
      for (int k0 = 0; k0 < D; k0 += 16) {
        mma_bf16(tm + TM_G, desc_k(aq, C, k0), desc_k(ak, C, k0), idg, k0 > 0);
        mma_bf16(tm + TM_G + LO16, desc_k(ak, C, k0), desc_k(ak, C, k0), idg, k0 > 0);
      }
      mma_commit(&g_done);
      bulk_wait_read0();  // q_hat / k_hat stores have read the tiles
      mbar_wait(&g_done, 0);
      mbar_arrive(&q_free);
      mbar_wait(&t_ready, 0);
      fence_after_sync();
      // W^T = K_hat^T T^T: M = d_k (128-row accumulators; M = 64 at d = 64)
      constexpr int MW = D >= 128 ? 128 : 64;
      const uint32_t idw = idesc_bf16(MW, 64, true, false);
#pragma unroll
      for (int h = 0; h < D / MW; ++h)
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_W + 64 * h, desc_mn(ak, C, k0, MW * h), desc_k(at, C, k0), idw, k0 > 0);
      mma_commit(&w_done);
      bulk_store(rec + S::R1_X, sX, BLK);
      bulk_store(rec + S::R1_T, sT, BLK);
      bulk_store(rec + S::R1_A, sA, BLK);
      bulk_store(rec + S::R1_N, nrm, 2 * C * 4);
      bulk_commit();
      mbar_wait(&w_img, 0);
      bulk_store(rec + S::R1_W, sW, S::WT);
      bulk_commit();
      bulk_wait0();
    }
    __syncwarp();
  } else {
    // ---------------- SIMT warps 0-7
    const int w = tid & 127, wq = w >> 5, half = tid >> 7;
    const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * a.L;
    if (tid < C) vb[tid] = (t0 + tid < a.L) ? __bfloat162float(beta[t0 + tid]) : 0.f;
    mbar_wait(&ld_full, 0);
    {  // row sums of squares: thread = (row, column quarter) of q and of k
      const int row = tid & 63, qt = tid >> 6;
      constexpr int QC = D / 4;
      float sq = 0.f, sk = 0.f;
#pragma unroll 4
      for (int g = 0; g < QC / 8; ++g) {
        float x[8], y[8];
        il_load8(sQ, C, row, qt * QC + g * 8, x);
        il_load8(sK, C, row, qt * QC + g * 8, y);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          sq = fmaf(x[e], x[e], sq);
          sk = fmaf(y[e], y[e], sk);
        }
      }
      part[qt * C + row] = sq;
      part[4 * C + qt * C + row] = sk;
      grp_sync<256>(1);
      // s_i, r_i = 1 / max(||x_i||, eps) (R9); padded tokens -> 0 (zero rows)
      const int tq = row;  // this thread's row again (scales its own quarter)
      const float nq = sqrtf((part[tq] + part[C + tq]) + (part[2 * C + tq] + part[3 * C + tq]));
      const float nk = sqrtf((part[4 * C + tq] + part[5 * C + tq]) +
                             (part[6 * C + tq] + part[7 * C + tq]));
      float r = l2 ? 1.f / fmaxf(nq, a.eps) : 1.f, s = l2 ? 1.f / fmaxf(nk, a.eps) : 1.f;
      if (t0 + tq >= a.L) r = s = 0.f;
      if (qt == 0) {
        nrm[tq] = nk;
        nrm[C + tq] = nq;
      }
#pragma unroll 4
      for (int g = 0; g < QC / 8; ++g) {
        float x[8], y[8];
        il_load8(sQ, C, row, qt * QC + g * 8, x);
        il_load8(sK, C, row, qt * QC + g * 8, y);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          x[e] *= r;
          y[e] *= s;
        }
        il_store8(sQ, C, row, qt * QC + g * 8, x);
        il_store8(sK, C, row, qt * QC + g * 8, y);
      }
    }
    hand_off(&norm_done, tid);
    mbar_wait(&g_done, 0);
    fence_after_sync();
    {
      // Gram read-out (lanes < 16: Q_hat K_hat^T row i, lanes >= 16: K_hat
      // K_hat^T row i; this warpgroup's 32 columns), lane pairs trade halves
      float f[32];
      ld32f(tm, wq, TM_G + 32 * half, f);
      const int i = wq * 16 + (lane & 15), h = 32 * half;
      const bool lo = lane < 16;
      float x[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = __shfl_xor_sync(0xffffffffu, lo ? f[16 + e] : f[e], 16);
      const int c0 = h + (lo ? 0 : 16);
      // A = tril(Q_hat K_hat^T), inclusive (R4)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        float a8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float qk = lo ? f[g * 8 + e] : x[g * 8 + e];
          a8[e] = (c0 + g * 8 + e <= i) ? qk : 0.f;
        }
        il_store8(sA, C, i, c0 + g * 8, a8);
      }
      // L = beta_i (k_hat_i . k_hat_j), j < i (Eq. 10)
      const float bi = vb[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = c0 + 4 * q;
        float kk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) kk[e] = lo ? x[4 * q + e] : f[16 + 4 * q + e];
        float4 v;
        v.x = (j + 0 < i) ? bi * kk[0] : 0.f;
        v.y = (j + 1 < i) ? bi * kk[1] : 0.f;
        v.z = (j + 2 < i) ? bi * kk[2] : 0.f;
        v.w = (j + 3 < i) ? bi * kk[3] : 0.f;
        *reinterpret_cast<float4*>(LX + i * LS + j) = v;
      }
    }
    fence_before_sync();
    grp_sync<256>(1);
    ut_inverse_inplace<LS, 256>(LX, tid, 1);
    {  // T = X diag(beta) (bf16), X (bf16 record); thread: row i, 16-column quarter
      const int i = tid & 63, j0 = (tid >> 6) * 16;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        float x[8], y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = j0 + g * 8 + e;
          x[e] = (j <= i) ? LX[i * LS + j] : 0.f;
          y[e] = x[e] * vb[j];
        }
        il_store8(sX, C, i, j0 + g * 8, x);
        il_store8(sT, C, i, j0 + g * 8, y);
      }
    }
    hand_off(&t_ready, tid);
    mbar_wait(&w_done, 0);
    mbar_wait(&q_free, 0);
    fence_after_sync();
    // W^T read-out -> bf16 image IL R = D (row = d_k)
    if (D >= 128) {
      constexpr int NA = D / 128;  // 128-row accumulators
#pragma unroll
      for (int item = half; item < 2 * NA; item += 2) {
        const int acc = item >> 1, ch = item & 1;
        float f[32];
        ld32f(tm, wq, TM_W + 64 * acc + 32 * ch, f);
        const int row = 128 * acc + 32 * wq + lane;
#pragma unroll
        for (int g = 0; g < 4; ++g) il_store8(sW, D, row, 32 * ch + g * 8, f + g * 8);
      }
    } else {  // M = 64: rows in lanes 0-15; warpgroups split the columns
      float f[32];
      ld32f(tm, wq, TM_W + 32 * half, f);
      if (lane < 16) {
        const int row = 16 * wq + lane;
#pragma unroll
        for (int g = 0; g < 4; ++g) il_store8(sW, D, row, 32 * half + g * 8, f + g * 8);
      }
    }
    hand_off(&w_img, tid);
  }
  cta_sync();
  if (warp == 0) tmem_dealloc<256>(tm);
}

template <int D>
__host__ __device__ constexpr int prep_smem() {
  return 2 * SP<D>::TILE + (C * LS + 2 * 4 * C + C + 2 * C) * 4 + 3 * BLK;
}

// ============================================================ fwd chain kernel
template <int D>
__host__ __device__ constexpr int fchain_smem() {
  return SP<D>::TILE * 3 + 2 * BLK + SP<D>::WT + 2 * BLK + SP<D>::HIMG + BLK;
}

template <int D>
__global__ void __launch_bounds__(288, 1)
    sp_fwd_chain_kernel(const __grid_constant__ CUtensorMap mV64, Args a) {
  using S = SP<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sKb = sQ + S::TILE;  // 2 slots
  uint8_t* sV = sKb + 2 * S::TILE;
  uint8_t* sT = sV + BLK;
  uint8_t* sW = sT + BLK;
  uint8_t* sAb = sW + S::WT;    // 2 slots
  uint8_t* sH = sAb + 2 * BLK;
  uint8_t* sZ = sH + S::HIMG;
  __shared__ uint64_t q_full, vt_full, w_full, k_full[2], a_full[2];
  __shared__ uint64_t up_done, q_done, ho_done, h_img, z_ready;
  __shared__ uint32_t tslot;
  // H_j^T (64 x D fp32): d_k columns [0, D/2) in lanes 0-15 of each quadrant
  // (lane offset 0), [D/2, D) in lanes 16-31 (offset 16), so every lane of a
  // warp converts state; U'^T (offset 0) and O (offset 16) share 64 columns
  constexpr int HD = D / 2;
  constexpr uint32_t TM_H = 0, TM_U = HD, TM_O = HD | LO16;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.x, unit = blockIdx.y, NC = a.NC;
  const bool rec = (a.flags & DELTANET_SAVE_STATES) != 0;
  const SpLayout ly = sp_layout<D>(a);
  auto r1 = [&](int c) { return ly.rec1 + ((size_t)unit * NC + c) * S::R1_BYTES; };
  auto r2 = [&](int c) { return ly.rec2 + (((size_t)unit * NC + c) * S::NB + j) * S::R2_BYTES; };
  uint8_t* himg = reinterpret_cast<uint8_t*>(a.states);
  auto rh = [&](int c) { return himg + (((size_t)unit * NC + c) * S::NB + j) * S::HIMG; };

  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 256) {
    mbar_init(&q_full, 1);
    mbar_init(&vt_full, 1);
    mbar_init(&w_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&k_full[b], 1);
      mbar_init(&a_full[b], 1);
    }
    mbar_init(&up_done, 1);
    mbar_init(&q_done, 1);
    mbar_init(&ho_done, 1);
    mbar_init(&h_img, 1);
    mbar_init(&z_ready, 1);
    mbar_fence_init();
  }
  cta_sync();
  const uint32_t tm = tslot;

  if (warp == 8) {
    if (lane == 0) {
      auto load_q = [&](int c) {
        mbar_expect_tx(&q_full, S::TILE);
        bulk_load(sQ, ly.qh + ((size_t)unit * NC + c) * S::TILE, S::TILE, &q_full);
      };
      auto load_vtw = [&](int c) {
        mbar_expect_tx(&vt_full, 2 * BLK);
        tma_load_4d(sV, &mV64, 0, c * C, 8 * j, unit, &vt_full);
        bulk_load(sT, r1(c) + S::R1_T, BLK, &vt_full);
        mbar_expect_tx(&w_full, S::WT);
        bulk_load(sW, r1(c) + S::R1_W, S::WT, &w_full);
      };
      auto load_ka = [&](int c) {
        const int b = c & 1;
        mbar_expect_tx(&k_full[b], S::TILE);
        bulk_load(sKb + b * S::TILE, ly.kh + ((size_t)unit * NC + c) * S::TILE, S::TILE,
                  &k_full[b]);
        mbar_expect_tx(&a_full[b], BLK);
        bulk_load(sAb + b * BLK, r1(c) + S::R1_A, BLK, &a_full[b]);
      };
      if (NC > 0) {
        load_q(0);
        load_vtw(0);
        load_ka(0);
        if (NC > 1) load_ka(1);
      }
      const uint32_t aQ = smem_u32(sQ), aV = smem_u32(sV), aT = smem_u32(sT),
                     aW = smem_u32(sW), aH = smem_u32(sH), aZ = smem_u32(sZ);
      const uint32_t id_u = idesc_bf16(64, 64, true, false);
      const uint32_t id_up = idesc_bf16(64, 64, false, true, true);
      const uint32_t id_o = idesc_bf16(64, 64, false, false);
      const uint32_t id_h = idesc_bf16(64, HD, false, true);
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        const int kb = c & 1;
        const uint32_t ph = c & 1, kph = (c >> 1) & 1;
        const uint32_t aK = smem_u32(sKb + kb * S::TILE), aA = smem_u32(sAb + kb * BLK);
        mbar_wait(&h_img, ph);  // sH = bf16 H_c (this block)
        SPT(1, c, 0);
        mbar_wait(&vt_full, ph);
        mbar_wait(&w_full, ph);
        mbar_wait(&q_full, ph);
        fence_after_sync();
        SPT(1, c, 1);
        // U^T = V_j^T T^T ; U'^T = U^T - H_j^T W^T
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_U, desc_mn(aV, C, k0), desc_k(aT, C, k0), id_u, k0 > 0);
#pragma unroll 4
        for (int k0 = 0; k0 < D; k0 += 16)
          mma_bf16(tm + TM_U, desc_k(aH, 64, k0), desc_mn(aW, D, k0), id_up, 1);
        mma_commit(&up_done);
        // O = Q_hat H_j
#pragma unroll 4
        for (int k0 = 0; k0 < D; k0 += 16)
          mma_bf16(tm + TM_O, desc_k(aQ, C, k0), desc_k(aH, 64, k0), id_o, k0 > 0);
        mma_commit(&q_done);
        // the next chunk's V / T / W as soon as U' has read them, its Q as
        // soon as O = Q H has (both complete before Z is converted: the
        // state update below queues behind O = Q H on the tensor pipe anyway)
        mbar_wait(&up_done, ph);
        if (c + 1 < NC) load_vtw(c + 1);
        mbar_wait(&q_done, ph);
        if (c + 1 < NC) load_q(c + 1);
        mbar_wait(&z_ready, ph);
        SPT(1, c, 2);
        mbar_wait(&k_full[kb], kph);
        mbar_wait(&a_full[kb], kph);
        fence_after_sync();
        SPT(1, c, 3);
        // H_j^T += U'_j^T K_hat (two d_k halves at lane offsets 0 / 16) ;
        // O += A U'_j
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_H + (h ? LO16 : 0), desc_k(aZ, 64, k0), desc_mn(aK, C, k0, HD * h),
                     id_h, 1);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_O, desc_k(aA, C, k0), desc_k(aZ, 64, k0), id_o, 1);
        mma_commit(&ho_done);
        SPT(1, c, 4);
        mbar_wait(&ho_done, ph);
        SPT(1, c, 5);
        if (c + 2 < NC) load_ka(c + 2);
      }
    }
    __syncwarp();
  } else {
    // ---------------- SIMT warps 0-7.  Every record and O go to global memory
    // straight from registers (coalesced 16 B stores; no smem staging to wait
    // for).  Lanes 0-15 of each quadrant hold the
    // rows of the offset-0 accumulators, lanes 16-31 those at offset 16; for
    // H, lane half hh = lane >> 4 holds d_k columns [hh D/2, hh D/2 + D/2)
    // and warpgroup wg a quarter of them
    const int w = tid & 127, wq = w >> 5, wg = tid >> 7;
    const bool lo = lane < 16;
    const int r16 = 16 * wq + (lane & 15);
    constexpr int QC = D / 4;                       // H columns per thread
    const int tcol = wg * QC;                       // TMEM column (within TM_H)
    const int gcol = (lo ? 0 : HD) + wg * QC;       // d_k column
    {  // H_j^T[dv][dk] = h0[dk][64 j + dv] -> TMEM (fp32) and the bf16 image
      const float* h0 = a.h0 ? a.h0 + (size_t)unit * D * D : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < QC; c0 += 16) {
        uint32_t r[16];
        float f[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          f[e] = h0 ? h0[(size_t)(gcol + c0 + e) * D + 64 * j + r16] : 0.f;
          r[e] = __float_as_uint(f[e]);
        }
        tmem_st16(taddr(tm, wq * 32, TM_H + tcol + c0), r);
        il_store8(sH, 64, r16, gcol + c0, f);
        il_store8(sH, 64, r16, gcol + c0 + 8, f + 8);
        if (rec && NC > 0) {
          stg8(rh(0) + il_off(r16, gcol + c0, 64), f);
          stg8(rh(0) + il_off(r16, gcol + c0 + 8, 64), f + 8);
        }
      }
      tmem_st_wait();
    }
    hand_off(&h_img, tid);
    __nv_bfloat16* const obase =
        a.o ? reinterpret_cast<__nv_bfloat16*>(a.o) + (size_t)unit * a.L * D + 64 * j : nullptr;
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const uint32_t ph = c & 1;
      mbar_wait(&up_done, ph);
      if (tid == 0) SPT(1, c, 8);
      fence_after_sync();
      if (tid == 0) SPT(1, c, 9);
      {  // U'^T (lanes < 16: row dv) -> bf16 sZ (IL R = 64, row dv, col token);
        // its record is stored after the hand-off (off the chain)
        float f[32];
        ld32f(tm, wq, TM_U + 32 * wg, f);
        if (lo) {
#pragma unroll
          for (int g = 0; g < 4; ++g) il_store8(sZ, 64, r16, 32 * wg + g * 8, f + g * 8);
        }
        hand_off(&z_ready, tid);
        if (lo && rec) {
          uint8_t* rz = r2(c) + S::R2_U;
#pragma unroll
          for (int g = 0; g < 4; ++g) stg8(rz + il_off(r16, 32 * wg + g * 8, 64), f + g * 8);
        }
      }
      if (tid == 0) SPT(1, c, 10);
      mbar_wait(&ho_done, ph);
      if (tid == 0) SPT(1, c, 11);
      fence_after_sync();
      if (tid == 0) SPT(1, c, 12);
      // H_{c+1}^T -> bf16 image (all lanes)
#pragma unroll
      for (int c0 = 0; c0 < QC; c0 += 16) {
        float f[16];
        ld16(tm, wq, TM_H + tcol + c0, f);
        il_store8(sH, 64, r16, gcol + c0, f);
        il_store8(sH, 64, r16, gcol + c0 + 8, f + 8);
      }
      float fo[32];  // O (lanes >= 16: token row), read before the next O = Q H
      ld32f(tm, wq, TM_U + 32 * wg, fo);
      hand_off(&h_img, tid);
      if (tid == 0) SPT(1, c, 13);
      if (rec && c + 1 < NC) {  // the H_{c+1} record: this thread's image chunks
        uint8_t* hr = rh(c + 1);
#pragma unroll
        for (int c0 = 0; c0 < QC; c0 += 8)
          *reinterpret_cast<uint4*>(hr + il_off(r16, gcol + c0, 64)) =
              *reinterpret_cast<const uint4*>(sH + il_off(r16, gcol + c0, 64));
      }
      const int tok = c * C + r16;
      if (!lo && obase && tok < a.L) {
#pragma unroll
        for (int g = 0; g < 4; ++g) stg8(obase + (size_t)tok * D + 32 * wg + g * 8, fo + g * 8);
      }
    }
    if (a.hT) {  // hT[dk][64 j + dv]
      fence_after_sync();
      float* hT = a.hT + (size_t)unit * D * D;
#pragma unroll 1
      for (int c0 = 0; c0 < QC; c0 += 16) {
        float f[16];
        ld16(tm, wq, TM_H + tcol + c0, f);
#pragma unroll
        for (int e = 0; e < 16; ++e) hT[(size_t)(gcol + c0 + e) * D + 64 * j + r16] = f[e];
      }
    }
  }
  cta_sync();
  if (warp == 0) tmem_dealloc<256>(tm);
}

// ============================================================ bwd chain kernel
template <int D>
__host__ __device__ constexpr int bchain_smem() {
  // K[2] Q | dO[2] A X V | Hf dH | dU' dV | beta [64] db [2][64]
  return 3 * SP<D>::TILE + 5 * BLK + 2 * SP<D>::HIMG + 2 * BLK + 3 * C * 4;
}

template <int D>
__global__ void __launch_bounds__(288, 1)
    sp_bwd_chain_kernel(const __grid_constant__ CUtensorMap mV64,
                        const __grid_constant__ CUtensorMap mDO64, Args a) {
  using S = SP<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sKb = smem;  // 2 slots
  uint8_t* sQ = sKb + 2 * S::TILE;
  uint8_t* sDOb = sQ + S::TILE;  // 2 slots
  uint8_t* sA = sDOb + 2 * BLK;
  uint8_t* sX = sA + BLK;
  uint8_t* sV = sX + BLK;
  uint8_t* sHf = sV + BLK;
  uint8_t* sDH = sHf + S::HIMG;
  uint8_t* sDU = sDH + S::HIMG;
  uint8_t* sDV = sDU + BLK;
  float* vb = reinterpret_cast<float*>(sDV + BLK);
  float* dbp = vb + C;  // [2][64]
  __shared__ uint64_t k_full[2], do_full[2], a_full, x_full, v_full, hf_full, q_full;
  __shared__ uint64_t du_done, r_done, p_done, dh_done, dh_img, du_ready, dv_ready, rr_ready;
  __shared__ uint32_t tslot;
  // dH_j^T (64 x D fp32) split by d_k halves over the lane offsets 0 / 16 as
  // in the forward chain; dU'^T (offset 0) | R' = K_hat H_j (offset 16) share
  // 64 columns, P (offset 16) 64 more
  constexpr int HD = D / 2;
  constexpr uint32_t TM_DH = 0, TM_DU = HD, TM_R = HD | LO16, TM_P = (HD + 64) | LO16;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.x, unit = blockIdx.y, NC = a.NC;
  const SpLayout ly = sp_layout<D>(a);
  auto r1 = [&](int c) { return ly.rec1 + ((size_t)unit * NC + c) * S::R1_BYTES; };
  auto r2 = [&](int c) { return ly.rec2 + (((size_t)unit * NC + c) * S::NB + j) * S::R2_BYTES; };
  const uint8_t* himg = reinterpret_cast<const uint8_t*>(a.states);
  auto rh = [&](int c) { return himg + (((size_t)unit * NC + c) * S::NB + j) * S::HIMG; };

  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 256) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&k_full[b], 1);
      mbar_init(&do_full[b], 1);
    }
    mbar_init(&a_full, 1);
    mbar_init(&x_full, 1);
    mbar_init(&v_full, 1);
    mbar_init(&hf_full, 1);
    mbar_init(&q_full, 1);
    mbar_init(&du_done, 1);
    mbar_init(&r_done, 1);
    mbar_init(&p_done, 1);
    mbar_init(&dh_done, 1);
    mbar_init(&dh_img, 1);
    mbar_init(&du_ready, 1);
    mbar_init(&dv_ready, 1);
    mbar_init(&rr_ready, 1);
    mbar_fence_init();
  }
  cta_sync();
  const uint32_t tm = tslot;

  if (warp == 8) {
    if (lane == 0) {
      // slots by iteration parity: chunk c = NC-1-it uses slot it & 1
      auto load_kdo = [&](int c, int slot) {
        mbar_expect_tx(&k_full[slot], S::TILE);
        bulk_load(sKb + slot * S::TILE, ly.kh + ((size_t)unit * NC + c) * S::TILE, S::TILE,
                  &k_full[slot]);
        mbar_expect_tx(&do_full[slot], BLK);
        tma_load_4d(sDOb + slot * BLK, &mDO64, 0, c * C, 8 * j, unit, &do_full[slot]);
      };
      auto load_a = [&](int c) {
        mbar_expect_tx(&a_full, BLK);
        bulk_load(sA, r1(c) + S::R1_A, BLK, &a_full);
      };
      auto load_x = [&](int c) {
        mbar_expect_tx(&x_full, BLK);
        bulk_load(sX, r1(c) + S::R1_X, BLK, &x_full);
      };
      auto load_hf = [&](int c) {
        mbar_expect_tx(&hf_full, S::HIMG);
        bulk_load(sHf, rh(c), S::HIMG, &hf_full);
      };
      auto load_v = [&](int c) {
        mbar_expect_tx(&v_full, BLK);
        tma_load_4d(sV, &mV64, 0, c * C, 8 * j, unit, &v_full);
      };
      auto load_q = [&](int c) {
        mbar_expect_tx(&q_full, S::TILE);
        bulk_load(sQ, ly.qh + ((size_t)unit * NC + c) * S::TILE, S::TILE, &q_full);
      };
      if (NC > 0) {
        load_kdo(NC - 1, 0);
        load_a(NC - 1);
        load_hf(NC - 1);
        load_x(NC - 1);
        load_v(NC - 1);
        load_q(NC - 1);
        if (NC > 1) load_kdo(NC - 2, 1);
      }
      const uint32_t aQ = smem_u32(sQ), aA = smem_u32(sA), aX = smem_u32(sX),
                     aHf = smem_u32(sHf), aDH = smem_u32(sDH), aDU = smem_u32(sDU),
                     aDV = smem_u32(sDV);
      const uint32_t id_du1 = idesc_bf16(64, 64, false, false);
      const uint32_t id_du2 = idesc_bf16(64, 64, true, true);
      const uint32_t id_p = idesc_bf16(64, 64, true, false);
      const uint32_t id_dh = idesc_bf16(64, HD, true, true);
      const uint32_t id_dhn = idesc_bf16(64, HD, true, true, true);
#pragma unroll 1
      for (int it = 0; it < NC; ++it) {
        const int c = NC - 1 - it, kb = it & 1;
        const uint32_t ph = it & 1, kph = (it >> 1) & 1;
        const uint32_t aK = smem_u32(sKb + kb * S::TILE), aDO = smem_u32(sDOb + kb * BLK);
        mbar_wait(&dh_img, ph);  // sDH = bf16 dl/dH_{c+1} (this block)
        SPT(2, it, 0);
        mbar_wait(&k_full[kb], kph);
        mbar_wait(&do_full[kb], kph);
        mbar_wait(&a_full, ph);
        fence_after_sync();
        SPT(2, it, 1);
        // dU'^T = dH^T K_hat^T + dO^T A   (the chain)
#pragma unroll 4
        for (int k0 = 0; k0 < D; k0 += 16)
          mma_bf16(tm + TM_DU, desc_k(aDH, 64, k0), desc_k(aK, C, k0), id_du1, k0 > 0);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_DU, desc_mn(aDO, C, k0), desc_mn(aA, C, k0), id_du2, 1);
        mma_commit(&du_done);
        if (it >= 1) {  // the previous chunk's R phase has read V and R' (rr_ready):
          // this chunk's forward H_j and V (R' of this chunk comes after its dH update)
          mbar_wait(&rr_ready, ph ^ 1);
          SPT(2, it, 5);
          load_hf(c);
          load_v(c);
        }
        mbar_wait(&du_ready, ph);  // dU'^T in smem (du_done seen by the SIMT warps)
        SPT(2, it, 2);
        if (c > 0) load_a(c - 1);
        mbar_wait(&x_full, ph);
        fence_after_sync();
        // P = X^T dU'_j (the chain), then R' = K_hat H_j (forward H_j; off it)
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_P, desc_mn(aX, C, k0), desc_k(aDU, 64, k0), id_p, k0 > 0);
        mma_commit(&p_done);
        mbar_wait(&dv_ready, ph);  // dV staged (P read)
        SPT(2, it, 3);
        if (c > 0) load_x(c - 1);
        mbar_wait(&q_full, ph);
        fence_after_sync();
        SPT(2, it, 4);
        // dH_j^T += dO_j^T Q_hat - dV_j^T K_hat  (two d_k halves)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t d = tm + TM_DH + (h ? LO16 : 0);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(d, desc_mn(aDO, C, k0), desc_mn(aQ, C, k0, HD * h), id_dh, 1);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(d, desc_mn(aDV, C, k0), desc_mn(aK, C, k0, HD * h), id_dhn, 1);
        }
        mma_commit(&dh_done);
        // R' = K_hat H_j (forward H_j) for R and dbeta: off the chain, after it
        mbar_wait(&hf_full, ph);
        fence_after_sync();
#pragma unroll 4
        for (int k0 = 0; k0 < D; k0 += 16)
          mma_bf16(tm + TM_R, desc_k(aK, C, k0), desc_k(aHf, 64, k0), id_du1, k0 > 0);
        mma_commit(&r_done);
        mbar_wait(&dh_done, ph);
        SPT(2, it, 6);
        if (c > 0) load_q(c - 1);
        if (c > 1) load_kdo(c - 2, kb);
      }
    }
    __syncwarp();
  } else {
    const int w = tid & 127, wq = w >> 5, wg = tid >> 7;
    const bool lo = lane < 16;
    const int r16 = 16 * wq + (lane & 15);
    constexpr int QC = D / 4;
    const int tcol = wg * QC, gcol = (lo ? 0 : HD) + wg * QC;
    const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * a.L;
    // every record and dV go to global memory straight from registers
    // (coalesced 16 B stores; nothing staged for a bulk store to drain)
    __nv_bfloat16* const dvbase = reinterpret_cast<__nv_bfloat16*>(a.dv) +
                                  (size_t)unit * a.L * D + 64 * j;
    {  // dH_j^T[dv][dk] = dhT[dk][64 j + dv]; its image is the record of chunk NC-1
      const float* dhT = a.dhT ? a.dhT + (size_t)unit * D * D : nullptr;
      uint8_t* hr = NC > 0 ? r2(NC - 1) + S::R2_DH : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < QC; c0 += 16) {
        uint32_t r[16];
        float f[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          f[e] = dhT ? dhT[(size_t)(gcol + c0 + e) * D + 64 * j + r16] : 0.f;
          r[e] = __float_as_uint(f[e]);
        }
        tmem_st16(taddr(tm, wq * 32, TM_DH + tcol + c0), r);
        il_store8(sDH, 64, r16, gcol + c0, f);
        il_store8(sDH, 64, r16, gcol + c0 + 8, f + 8);
        if (hr) {
          stg8(hr + il_off(r16, gcol + c0, 64), f);
          stg8(hr + il_off(r16, gcol + c0 + 8, 64), f + 8);
        }
      }
      tmem_st_wait();
    }
    hand_off(&dh_img, tid);
#pragma unroll 1
    for (int it = 0; it < NC; ++it) {
      const int c = NC - 1 - it, t0 = c * C;
      const uint32_t ph = it & 1;
      if (tid < C) vb[tid] = (t0 + tid < a.L) ? __bfloat162float(beta[t0 + tid]) : 0.f;
      mbar_wait(&du_done, ph);
      if (tid == 0) SPT(2, it, 8);
      fence_after_sync();
      if (tid == 0) SPT(2, it, 9);
      {  // dU'^T (lanes < 16: row dv) -> bf16 operand; the record after the hand-off
        float f[32];
        ld32f(tm, wq, TM_DU + 32 * wg, f);
        if (lo) {
#pragma unroll
          for (int g = 0; g < 4; ++g) il_store8(sDU, 64, r16, 32 * wg + g * 8, f + g * 8);
        }
        hand_off(&du_ready, tid);
        if (lo) {
          uint8_t* rd = r2(c) + S::R2_DU;
#pragma unroll
          for (int g = 0; g < 4; ++g) stg8(rd + il_off(r16, 32 * wg + g * 8, 64), f + g * 8);
        }
      }
      if (tid == 0) SPT(2, it, 10);
      mbar_wait(&p_done, ph);
      fence_after_sync();
      if (tid == 0) SPT(2, it, 11);
      float p[32];  // P (lanes >= 16: token row r16), kept for dbeta
      {  // dV = diag(beta) P -> bf16 operand; the dv output after the hand-off
        ld32f(tm, wq, HD + 64 + 32 * wg, p);
        const float bt = lo ? 0.f : vb[r16];
        if (!lo) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float d8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) d8[e] = bt * p[g * 8 + e];
            il_store8(sDV, C, r16, 32 * wg + g * 8, d8);
          }
        }
        hand_off(&dv_ready, tid);
        const int tok = t0 + r16;
        if (!lo && tok < a.L) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<uint4*>(dvbase + (size_t)tok * D + 32 * wg + g * 8) =
                *reinterpret_cast<const uint4*>(sDV + il_off(r16, 32 * wg + g * 8, C));
        }
      }
      if (tid == 0) SPT(2, it, 12);
      mbar_wait(&dh_done, ph);
      if (tid == 0) SPT(2, it, 15);
      fence_after_sync();
      if (tid == 0) SPT(2, it, 16);
      // dl/dH_c image (the next chunk's operand); the record of chunk c-1 is
      // copied out of it after the hand-off
#pragma unroll
      for (int c0 = 0; c0 < QC; c0 += 16) {
        float f[16];
        ld16(tm, wq, TM_DH + tcol + c0, f);
        il_store8(sDH, 64, r16, gcol + c0, f);
        il_store8(sDH, 64, r16, gcol + c0 + 8, f + 8);
      }
      hand_off(&dh_img, tid);
      if (tid == 0) SPT(2, it, 17);
      if (c > 0) {
        uint8_t* hr = r2(c - 1) + S::R2_DH;
#pragma unroll
        for (int c0 = 0; c0 < QC; c0 += 8)
          *reinterpret_cast<uint4*>(hr + il_off(r16, gcol + c0, 64)) =
              *reinterpret_cast<const uint4*>(sDH + il_off(r16, gcol + c0, 64));
      }
      mbar_wait(&r_done, ph);
      mbar_wait(&v_full, ph);
      fence_after_sync();
      if (tid == 0) SPT(2, it, 13);
      {  // R = V_j - K_hat H_j (record) ; rowsum(P . R) (lanes >= 16)
        float rp[32];
        ld32f(tm, wq, HD + 32 * wg, rp);
        if (!lo) {
          uint8_t* rr = r2(c) + S::R2_R;
          float db = 0.f;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float v8[8], r8[8];
            il_load8(sV, C, r16, 32 * wg + g * 8, v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              r8[e] = v8[e] - rp[g * 8 + e];
              db = fmaf(p[g * 8 + e], r8[e], db);
            }
            stg8(rr + il_off(r16, 32 * wg + g * 8, C), r8);
          }
          dbp[wg * C + r16] = db;
        }
      }
      hand_off(&rr_ready, tid);
      if (tid == 0) SPT(2, it, 14);
      if (tid < C)  // rowsum(P_j . R_j) of this block (dbeta part 1)
        reinterpret_cast<float*>(r2(c) + S::R2_DB)[tid] = dbp[tid] + dbp[C + tid];
    }
    if (a.dh0) {
      fence_after_sync();
      float* dh0 = a.dh0 + (size_t)unit * D * D;
#pragma unroll 1
      for (int c0 = 0; c0 < QC; c0 += 16) {
        float f[16];
        ld16(tm, wq, TM_DH + tcol + c0, f);
#pragma unroll
        for (int e = 0; e < 16; ++e) dh0[(size_t)(gcol + c0 + e) * D + 64 * j + r16] = f[e];
      }
    }
  }
  cta_sync();
  if (warp == 0) tmem_dealloc<256>(tm);
}

// ============================================================ bwd local kernel
// The d_v loop runs in sub-steps (block v, d_k half h): the five 64 x 64
// tiles of block v (dO, U', dU', R, dV) and the d_k half h of the H^T and
// dH^T images of block v, each double-buffered, so the next sub-step's loads
// overlap this one's products.
template <int D>
struct BL {
  static constexpr int DH = D >= 128 ? 128 : D;    // d_k columns per image half
  static constexpr int HALVES = D / DH;
  static constexpr int IH = 64 * DH * 2;           // image half (bytes)
  static constexpr int SSET = 5 * BLK;             // dO U' dU' R dV
  static constexpr int ISET = 2 * IH;              // H^T half, dH^T half
  static constexpr int LOOP = 2 * SSET + 2 * ISET;
  static constexpr int REG = LOOP > 2 * SP<D>::TILE ? LOOP : 2 * SP<D>::TILE;
};
template <int D>
__host__ __device__ constexpr int blocal_smem() {
  return BL<D>::REG + 5 * BLK + (C * 4) * 10;
}

template <int D>
__global__ void __launch_bounds__(288, 1)
    sp_bwd_local_kernel(const __grid_constant__ CUtensorMap mDO64,
                        const __grid_constant__ CUtensorMap mDV64,
                        const __grid_constant__ CUtensorMap mDQ,
                        const __grid_constant__ CUtensorMap mDK, Args a) {
  using S = SP<D>;
  using Bl = BL<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  auto sset = [&](int b) { return smem + b * Bl::SSET; };  // + 0 dO, 1 U', 2 dU', 3 R, 4 dV (x BLK)
  auto iset = [&](int b) { return smem + 2 * Bl::SSET + b * Bl::ISET; };  // + 0 H^T, IH dH^T
  // q_hat / k_hat land in loop buffers as they retire (the S buffer of block
  // NB-2 and the image buffer of sub-step NS-2), or in the buffers a single
  // block never uses (NB = 1); dq / dk are staged there in place
  constexpr int NSS = S::NB * Bl::HALVES;
  static_assert(Bl::SSET >= S::TILE && Bl::ISET >= S::TILE, "q_hat / k_hat in the loop buffers");
  uint8_t* sQ = S::NB > 1 ? sset((S::NB - 2) & 1) : sset(1);
  uint8_t* sK = NSS > 1 ? iset((NSS - 2) & 1) : iset(1);
  uint8_t* sX = smem + Bl::REG;
  uint8_t* sDA = sX + BLK;
  uint8_t* sDX = sDA + BLK;
  uint8_t* sY = sDX + BLK;
  uint8_t* sG1 = sY + BLK;
  float* vb = reinterpret_cast<float*>(sG1 + BLK);  // beta [64]
  float* nrm = vb + C;                              // ||k|| | ||q||  [128]
  float* db2 = nrm + 2 * C;                         // [2][64]
  float* dot = db2 + 2 * C;                         // [2 (q|k)][2 wg][64]
  __shared__ uint64_t x_full, s_full[2], i_full[2], i_done[2], v_all, qh_full, kh_full, dax_ready,
      y_done, y_ready, kk_done, g_done, g1_ready, k_done, epi_done;
  __shared__ uint32_t tslot;
  constexpr uint32_t TM_DQ = 0, TM_DK = LO16, TM_DA = D, TM_DX = D | LO16, TM_Y = D,
                     TM_G = D | LO16, TM_KK = (D + 64) | LO16;
  constexpr int TMC = D + 128 <= 256 ? 256 : 512;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x, unit = blockIdx.y, NC = a.NC, t0 = c * C;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const SpLayout ly = sp_layout<D>(a);
  const uint8_t* rec1 = ly.rec1 + ((size_t)unit * NC + c) * S::R1_BYTES;
  auto r2 = [&](int v) { return ly.rec2 + (((size_t)unit * NC + c) * S::NB + v) * S::R2_BYTES; };
  const uint8_t* himg = reinterpret_cast<const uint8_t*>(a.states);
  auto rh = [&](int v) { return himg + (((size_t)unit * NC + c) * S::NB + v) * S::HIMG; };

  if (tid == 0) SPT(3, 8, 2);
  if (warp == 0) tmem_alloc<TMC>(&tslot);
  if (tid == 256) {
    mbar_init(&x_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&i_full[b], 1);
      mbar_init(&i_done[b], 1);
    }
    mbar_init(&v_all, 1);
    mbar_init(&qh_full, 1);
    mbar_init(&kh_full, 1);
    mbar_init(&dax_ready, 1);
    mbar_init(&y_done, 1);
    mbar_init(&y_ready, 1);
    mbar_init(&kk_done, 1);
    mbar_init(&g_done, 1);
    mbar_init(&g1_ready, 1);
    mbar_init(&k_done, 1);
    mbar_init(&epi_done, 1);
    mbar_fence_init();
  }
  cta_sync();
  const uint32_t tm = tslot;

  if (warp == 8) {
    if (lane == 0) {
      mbar_expect_tx(&x_full, BLK + 2 * C * 4);
      bulk_load(sX, rec1 + S::R1_X, BLK, &x_full);
      bulk_load(nrm, rec1 + S::R1_N, 2 * C * 4, &x_full);
      constexpr int NS = S::NB * Bl::HALVES;  // sub-steps (v, h)
      auto load_s = [&](int v) {
        const int b = v & 1;
        uint8_t* st = sset(b);
        mbar_expect_tx(&s_full[b], Bl::SSET);
        tma_load_4d(st, &mDO64, 0, t0, 8 * v, unit, &s_full[b]);
        tma_load_4d(st + 4 * BLK, &mDV64, 0, t0, 8 * v, unit, &s_full[b]);
        bulk_load(st + BLK, r2(v) + S::R2_U, BLK, &s_full[b]);
        bulk_load(st + 2 * BLK, r2(v) + S::R2_DU, BLK, &s_full[b]);
        bulk_load(st + 3 * BLK, r2(v) + S::R2_R, BLK, &s_full[b]);
      };
      auto load_i = [&](int ss) {  // H^T and dH^T images of block v, d_k half h
        const int v = ss / Bl::HALVES, h = ss % Bl::HALVES, b = ss & 1;
        uint8_t* it = iset(b);
        mbar_expect_tx(&i_full[b], Bl::ISET);
        bulk_load(it, rh(v) + h * Bl::IH, Bl::IH, &i_full[b]);
        bulk_load(it + Bl::IH, r2(v) + S::R2_DH + h * Bl::IH, Bl::IH, &i_full[b]);
      };
      auto load_qh = [&]() {
        mbar_expect_tx(&qh_full, S::TILE);
        bulk_load(sQ, ly.qh + ((size_t)unit * NC + c) * S::TILE, S::TILE, &qh_full);
      };
      auto load_kh = [&]() {
        mbar_expect_tx(&kh_full, S::TILE);
        bulk_load(sK, ly.kh + ((size_t)unit * NC + c) * S::TILE, S::TILE, &kh_full);
      };
      load_s(0);
      load_i(0);
      if (S::NB > 1) load_s(1);
      if (NS > 1) load_i(1);
      if (S::NB == 1) load_qh();
      if (NS == 1) load_kh();
      const uint32_t id_a = idesc_bf16(64, 64, false, true);           // dA = dO U'^T
      const uint32_t id_x = idesc_bf16(64, 64, true, false);           // dX' = dU' R^T
      const uint32_t id_q = idesc_bf16(64, Bl::DH, false, true);       // dQ += dO H^T
      const uint32_t id_k = idesc_bf16(64, Bl::DH, true, true);        // dK += U' dH^T
      const uint32_t id_kn = idesc_bf16(64, Bl::DH, false, true, true);  // dK -= dV H^T
#pragma unroll 1
      for (int ss = 0; ss < NS; ++ss) {
        const int v = ss / Bl::HALVES, h = ss % Bl::HALVES;
        SPT(3, ss, 0);
        mbar_wait(&s_full[v & 1], (v >> 1) & 1);
        mbar_wait(&i_full[ss & 1], (ss >> 1) & 1);
        fence_after_sync();
        SPT(3, ss, 1);
        const uint8_t* st = sset(v & 1);
        const uint8_t* it = iset(ss & 1);
        const uint32_t aDO = smem_u32(st), aU = smem_u32(st + BLK), aDU = smem_u32(st + 2 * BLK),
                       aR = smem_u32(st + 3 * BLK), aDV = smem_u32(st + 4 * BLK),
                       aH = smem_u32(it), aDH = smem_u32(it + Bl::IH);
        const uint32_t cq = TM_DQ + Bl::DH * h, ck = TM_DK + Bl::DH * h;
#pragma unroll
        for (int k0 = 0; k0 < 64; k0 += 16) {
          const uint32_t acc = (v > 0 || k0 > 0) ? 1u : 0u;
          if (h == 0) {
            mma_bf16(tm + TM_DA, desc_k(aDO, C, k0), desc_mn(aU, 64, k0), id_a, acc);
            mma_bf16(tm + TM_DX, desc_mn(aDU, 64, k0), desc_k(aR, C, k0), id_x, acc);
          }
          mma_bf16(tm + cq, desc_k(aDO, C, k0), desc_mn(aH, 64, k0), id_q, acc);
          mma_bf16(tm + ck, desc_mn(aU, 64, k0), desc_mn(aDH, 64, k0), id_k, acc);
          mma_bf16(tm + ck, desc_k(aDV, C, k0), desc_mn(aH, 64, k0), id_kn, 1);
        }
        mma_commit(&i_done[ss & 1]);
        SPT(3, ss, 2);
        if (ss >= 1) {  // sub-step ss-1 retired: refill its buffers
          const int pv = (ss - 1) / Bl::HALVES, ph = (ss - 1) % Bl::HALVES;
          mbar_wait(&i_done[(ss - 1) & 1], ((ss - 1) >> 1) & 1);
          if (ss + 1 < NS) load_i(ss + 1);
          if (ph == Bl::HALVES - 1 && pv + 2 < S::NB) load_s(pv + 2);
          if (ph == Bl::HALVES - 1 && pv == S::NB - 2) load_qh();  // its S buffer retired
          if (ss - 1 == NS - 2) load_kh();                         // its image buffer retired
        }
      }
      mma_commit(&v_all);  // the SIMT warps wait for the whole d_v loop
      mbar_wait(&v_all, 0);
      SPT(3, 8, 0);
      const uint32_t aX = smem_u32(sX), aDA = smem_u32(sDA), aDX = smem_u32(sDX),
                     aY = smem_u32(sY), aG1 = smem_u32(sG1), aQ = smem_u32(sQ),
                     aK = smem_u32(sK);
      mbar_wait(&x_full, 0);
      mbar_wait(&dax_ready, 0);
      fence_after_sync();
      {  // Y = X^T dX
        const uint32_t id = idesc_bf16(64, 64, true, true);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_Y, desc_mn(aX, C, k0), desc_mn(aDX, C, k0), id, k0 > 0);
        mma_commit(&y_done);
      }
      mbar_wait(&qh_full, 0);
      mbar_wait(&kh_full, 0);
      fence_after_sync();
      {  // K_hat K_hat^T ; dQ += dA K_hat ; dK += dA^T Q_hat
        const uint32_t id = idesc_bf16(64, 64, false, false);
#pragma unroll 4
        for (int k0 = 0; k0 < D; k0 += 16)
          mma_bf16(tm + TM_KK, desc_k(aK, C, k0), desc_k(aK, C, k0), id, k0 > 0);
        mma_commit(&kk_done);
        const uint32_t idq = idesc_bf16(64, D, false, true), idk = idesc_bf16(64, D, true, true);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16) {
          mma_bf16(tm + TM_DQ, desc_k(aDA, C, k0), desc_mn(aK, C, k0), idq, 1);
          mma_bf16(tm + TM_DK, desc_mn(aDA, C, k0), desc_mn(aQ, C, k0), idk, 1);
        }
      }
      mbar_wait(&y_ready, 0);
      fence_after_sync();
      {  // G = -Y X^T
        const uint32_t id = idesc_bf16(64, 64, false, false, true);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_G, desc_k(aY, C, k0), desc_k(aX, C, k0), id, k0 > 0);
        mma_commit(&g_done);
      }
      mbar_wait(&g1_ready, 0);
      fence_after_sync();
      {  // dK += G1 K_hat + G1^T K_hat
        const uint32_t id = idesc_bf16(64, D, false, true), idt = idesc_bf16(64, D, true, true);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16) {
          mma_bf16(tm + TM_DK, desc_k(aG1, C, k0), desc_mn(aK, C, k0), id, 1);
          mma_bf16(tm + TM_DK, desc_mn(aG1, C, k0), desc_mn(aK, C, k0), idt, 1);
        }
        mma_commit(&k_done);
      }
      mbar_wait(&epi_done, 0);
      SPT(3, 8, 1);
      tma_store_4d(&mDQ, sQ, 0, t0, 0, unit);
      tma_store_4d(&mDK, sK, 0, t0, 0, unit);
      bulk_commit();
      bulk_wait0();
    }
    __syncwarp();
  } else {
    const int w = tid & 127, wq = w >> 5, wg = tid >> 7;
    const bool lo = lane < 16;
    const int r16 = 16 * wq + (lane & 15);
    const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * a.L;
    if (tid < C) vb[tid] = (t0 + tid < a.L) ? __bfloat162float(beta[t0 + tid]) : 0.f;
    float db1 = 0.f;  // sum_v rowsum(P_v . R_v) (bwd chain records), loads in flight now
    if (tid < C) {
#pragma unroll
      for (int v = 0; v < S::NB; ++v) db1 += reinterpret_cast<const float*>(r2(v) + S::R2_DB)[tid];
    }
    mbar_wait(&x_full, 0);
    if (tid == 0) SPT(3, 9, 0);
    mbar_wait(&v_all, 0);
    fence_after_sync();
    if (tid == 0) SPT(3, 9, 1);
    grp_sync<256>(1);  // beta visible
    {  // lanes < 16: dA row (masked j <= i); lanes >= 16: dX row = dX' diag(beta)
      float f[32];
      ld32f(tm, wq, TM_DA + 32 * wg, f);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int jj = 32 * wg + g * 8 + e;
          x[e] = lo ? ((jj <= r16) ? f[g * 8 + e] : 0.f) : f[g * 8 + e] * vb[jj];
        }
        il_store8(lo ? sDA : sDX, C, r16, 32 * wg + g * 8, x);
      }
    }
    hand_off(&dax_ready, tid);
    if (tid == 0) SPT(3, 9, 2);
    mbar_wait(&y_done, 0);
    fence_after_sync();
    {  // Y (lanes < 16) -> bf16
      float f[32];
      ld32f(tm, wq, TM_Y + 32 * wg, f);
      if (lo) {
#pragma unroll
        for (int g = 0; g < 4; ++g) il_store8(sY, C, r16, 32 * wg + g * 8, f + g * 8);
      }
    }
    hand_off(&y_ready, tid);
    if (tid == 0) SPT(3, 9, 3);
    mbar_wait(&g_done, 0);
    mbar_wait(&kk_done, 0);
    if (tid == 0) SPT(3, 9, 4);
    fence_after_sync();
    {  // lanes >= 16: G row i and K_hat K_hat^T row i
      float gg[32], kk[32];
      ld32f(tm, wq, D + 32 * wg, gg);
      ld32f(tm, wq, D + 64 + 32 * wg, kk);
      if (!lo) {
        const float bi = vb[r16];
        float d2 = 0.f;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float y[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int jj = 32 * wg + g * 8 + e;
            const float gv = (jj < r16) ? gg[g * 8 + e] : 0.f;
            d2 = fmaf(gv, kk[g * 8 + e], d2);
            y[e] = bi * gv;
          }
          il_store8(sG1, C, r16, 32 * wg + g * 8, y);
        }
        db2[wg * C + r16] = d2;
      }
    }
    hand_off(&g1_ready, tid);
    if (tid < C && t0 + tid < a.L) {  // dbeta = sum_v rowsum(P_v . R_v) + rowsum(G . K K^T)
      const float db = db1 + (db2[tid] + db2[C + tid]);
      reinterpret_cast<__nv_bfloat16*>(a.dbeta)[(size_t)unit * a.L + t0 + tid] =
          __float2bfloat16_rn(db);
    }
    if (tid == 0) SPT(3, 9, 5);
    mbar_wait(&k_done, 0);
    fence_after_sync();
    if (tid == 0) SPT(3, 9, 6);
    {
      // dq (lanes < 16, TM_DQ) / dk (lanes >= 16, TM_DK) rows: L2 adjoint
      // dx = inv (dx_hat - x_hat (x_hat . dx_hat)) when ||x|| >= eps (R9)
      constexpr int HC = D / 2;
      uint8_t* tile = lo ? sQ : sK;
      float dt = 0.f;
#pragma unroll 1
      for (int c0 = wg * HC; c0 < wg * HC + HC; c0 += 32) {
        float f[32];
        ld32f(tm, wq, c0, f);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float x8[8];
          il_load8(tile, C, r16, c0 + g * 8, x8);
#pragma unroll
          for (int e = 0; e < 8; ++e) dt = fmaf(x8[e], f[g * 8 + e], dt);
        }
      }
      dot[(lo ? 0 : 2 * C) + wg * C + r16] = dt;
      grp_sync<256>(1);
      const float* dd = dot + (lo ? 0 : 2 * C);
      dt = dd[r16] + dd[C + r16];
      const float n = nrm[(lo ? C : 0) + r16];
      float inv = l2 ? 1.f / fmaxf(n, a.eps) : 1.f;
      if (t0 + r16 >= a.L) inv = 0.f;
      if (!(l2 && n >= a.eps)) dt = 0.f;
#pragma unroll 1
      for (int c0 = wg * HC; c0 < wg * HC + HC; c0 += 32) {
        float f[32];
        ld32f(tm, wq, c0, f);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float x8[8];
          il_load8(tile, C, r16, c0 + g * 8, x8);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            x8[e] = l2 ? inv * (f[g * 8 + e] - x8[e] * dt) : f[g * 8 + e];
          il_store8(tile, C, r16, c0 + g * 8, x8);
        }
      }
    }
    hand_off(&epi_done, tid);
    if (tid == 0) SPT(3, 9, 7);
  }
  cta_sync();
  if (warp == 0) tmem_dealloc<TMC>(tm);
}

// ------------------------------------------------------------------ host side
// 4-D view {8, L, D/8, BH} of a [BH][L][D] bf16 tensor with a box of
// `cg` column groups (cg = D/8: whole rows; 8: one 64-column block)
bool make_map(CUtensorMap* m, const void* base, int BH, int L, int D, int cg) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {8, (cuuint64_t)L, (cuuint64_t)(D / 8), (cuuint64_t)BH};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, 16, (cuuint64_t)L * D * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)C, (cuuint32_t)cg, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
int set_attrs() {
  static PerDevice attr;
  if (attr.done()) return DELTANET_OK;
  if (cudaFuncSetAttribute(sp_prep_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           prep_smem<D>()) != cudaSuccess ||
      cudaFuncSetAttribute(sp_fwd_chain_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           fchain_smem<D>()) != cudaSuccess ||
      cudaFuncSetAttribute(sp_bwd_chain_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bchain_smem<D>()) != cudaSuccess ||
      cudaFuncSetAttribute(sp_bwd_local_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           blocal_smem<D>()) != cudaSuccess)
    return DELTANET_ERR_CUDA;
  attr.mark();
  return DELTANET_OK;
}

template <int D>
int sp_fwd_t(const Args& a0, cudaStream_t s) {
  static_assert(prep_smem<D>() <= 232448 - 1024 && fchain_smem<D>() <= 232448 - 1024 &&
                    bchain_smem<D>() <= 232448 - 1024 && blocal_smem<D>() <= 232448 - 1024,
                "shared memory budget");
  if (int rc = set_attrs<D>()) return rc;
  Args a = a0;
  const int BH = a.B * a.H;
  const SpLayout ly = sp_layout<D>(a);
  CUtensorMap mQ, mK, mV64;
  if (!make_map(&mQ, a.q, BH, a.L, D, D / 8) || !make_map(&mK, a.k, BH, a.L, D, D / 8) ||
      !make_map(&mV64, a.v, BH, a.L, D, 8))
    return DELTANET_ERR_CUDA;
  if (a.NC > 0)
    sp_prep_kernel<D><<<dim3(a.NC, BH), 288, prep_smem<D>(), s>>>(mQ, mK, a);
  sp_fwd_chain_kernel<D><<<dim3(SP<D>::NB, BH), 288, fchain_smem<D>(), s>>>(mV64, a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

template <int D>
int sp_bwd_t(const Args& a0, cudaStream_t s) {
  if (int rc = set_attrs<D>()) return rc;
  Args a = a0;
  if (!(a.flags & DELTANET_SAVE_STATES)) {  // recompute the forward's records (no O)
    Args f = a0;
    f.flags |= DELTANET_SAVE_STATES;
    f.o = nullptr;
    f.hT = nullptr;
    if (int rc = sp_fwd_t<D>(f, s)) return rc;
  }
  const int BH = a.B * a.H;
  const SpLayout ly = sp_layout<D>(a);
  CUtensorMap mV64, mDO64, mDV64, mDQ, mDK;
  if (!make_map(&mV64, a.v, BH, a.L, D, 8) || !make_map(&mDO64, a.dO, BH, a.L, D, 8) ||
      !make_map(&mDV64, a.dv, BH, a.L, D, 8) || !make_map(&mDQ, a.dq, BH, a.L, D, D / 8) ||
      !make_map(&mDK, a.dk, BH, a.L, D, D / 8))
    return DELTANET_ERR_CUDA;
  sp_bwd_chain_kernel<D><<<dim3(SP<D>::NB, BH), 288, bchain_smem<D>(), s>>>(mV64, mDO64, a);
  if (a.NC > 0)
    sp_bwd_local_kernel<D><<<dim3(a.NC, BH), 288, blocal_smem<D>(), s>>>(mDO64, mDV64,
                                                                        mDQ, mDK, a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

}  // namespace

// d_k = d_v = D in {64, 128, 256}, C = 64, bf16, ungated
bool sp_supported(const deltanet_desc* d) {
  return d->dtype == DELTANET_BF16 && d->chunk == C && d->Dk == d->Dv &&
         (d->Dk == 64 || d->Dk == 128 || d->Dk == 256) && !(d->flags & DELTANET_GATED);
}

size_t sp_scratch_bytes(const deltanet_desc* d) {
  const int D = d->Dk;
  const size_t BH = (size_t)d->B * d->H, NC = (size_t)(d->L + C - 1) / C;
  const size_t qk = BH * NC * (size_t)C * D * 2;  // q_hat / k_hat images
  size_t r1 = 0, r2 = 0;
  switch (D) {
    case 64: r1 = SP<64>::R1_BYTES; r2 = SP<64>::NB * (size_t)SP<64>::R2_BYTES; break;
    case 128: r1 = SP<128>::R1_BYTES; r2 = SP<128>::NB * (size_t)SP<128>::R2_BYTES; break;
    default: r1 = SP<256>::R1_BYTES; r2 = SP<256>::NB * (size_t)SP<256>::R2_BYTES; break;
  }
  return 2 * qk + BH * NC * (r1 + r2);
}

int sp_launch_count(const deltanet_desc* d, int which) {
  const int f = d->L > 0 ? 2 : 1;
  if (which == 0) return f;
  const int b = d->L > 0 ? 2 : 1;
  return (d->flags & DELTANET_SAVE_STATES) ? b : b + f;
}

int sp_fwd(const Args& a, cudaStream_t s) {
  switch (a.Dk) {
    case 64: return sp_fwd_t<64>(a, s);
    case 128: return sp_fwd_t<128>(a, s);
    case 256: return sp_fwd_t<256>(a, s);
  }
  return DELTANET_ERR_UNSUPPORTED;
}

int sp_bwd(const Args& a, cudaStream_t s) {
  switch (a.Dk) {
    case 64: return sp_bwd_t<64>(a, s);
    case 128: return sp_bwd_t<128>(a, s);
    case 256: return sp_bwd_t<256>(a, s);
  }
  return DELTANET_ERR_UNSUPPORTED;
}

}  // namespace dn

#ifdef DN_TIMING
extern "C" int sp_timing_set(long long* buf, int kernel) {
  return cudaMemcpyToSymbol(dn::sp_tim, &buf, sizeof(buf)) != cudaSuccess ||
         cudaMemcpyToSymbol(dn::sp_tim_kernel, &kernel, sizeof(int)) != cudaSuccess;
}
#endif
