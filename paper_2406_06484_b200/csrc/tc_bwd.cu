// tc_bwd.cu -- fused sm_100a backward of the chunkwise DeltaNet layer.
//
// The paper gives no backward (PAPER.md line 250 only says states are
// recomputed; reading R12).  This kernel evaluates the exact
// adjoint of Eq. 8-11 chunk by chunk in reverse (DESIGN.md §4.2,
// SURVEY App. A.2), one CTA per (b, h) unit, with dH = dl/dH_{t+1} held in
// TMEM (fp32, lanes = d_v) across chunks.  The forward's per-chunk record
// (H_t, X, Z^T = (diag(s) U')^T; tc_common.cuh REC_*) is read back, so the
// UT substitution and the W / U / U' products are not recomputed.
//
// Per chunk (q_hat = diag(r) q, k_hat = diag(s) k: L2-normalised rows):
//   recompute  A = tril(Q_hat K_hat^T), R = V - K_hat H, U' = diag(1/s) Z
//   chain      dU' = K_hat dH + A^T dO
//              dH <- dH + Q_hat^T dO - W^T dU',  W^T dU' = K_hat^T diag(b) X^T dU' = K_hat^T dV
//   local      dA = tril(dO U'^T)          P = X^T dU'  (= dV_beta)
//              dX = (dU' R^T) diag(b)      Y = X^T dX,  G = tril(-Y X^T, -1)
//              dQ = dO H^T + dA K_hat
//              dK = U' dH^T + dA^T Q_hat - dV H^T + (G1 + G1^T) K_hat,  G1 = diag(b) G
//              dV = diag(b) P
//              dbeta = rowsum(P . R) + rowsum(G . K_hat K_hat^T)
//   then the L2-normalisation adjoint on dQ, dK (R9).
// (dK_beta = X^T dW = -P H^T, and rowsum(dK_beta . K) + rowsum(P . V) =
//  rowsum(P . R) -- DESIGN.md §4.2.)
//
// The first products of a chunk (K K^T, Q K^T, dH^T K^T, K H) run on the RAW
// bf16 q / k tiles as they land, so they overlap the previous chunk's
// epilogues; the row scales enter exactly in the conversions:
//   A_m = tril(diag(r) Q K^T)  (M2 operand; A = A_m diag(s)),
//   dU'^T = (dH^T K^T + dO^T A_m) diag(s),  R = V - diag(s) (K H),
// q and k are normalised in place afterwards for the remaining products.
//
// 320 threads: warps 0-7 run the SIMT phases (split by columns between the
// two warpgroups, both see all 128 TMEM lanes); warp 8 issues every MMA and
// warp 9 every TMA load and store, both driven by mbarrier hand-offs (a
// single issuer would sit blocked on a full MMA queue while a load waits).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

using namespace tc;

constexpr int C = 64, D = 128, NT = 320;  // warps 0-7 SIMT, 8 MMA issuer, 9 TMA
constexpr uint32_t LO16 = 16u << 16;  // TMEM lane offset 16 (second M=64 accumulator)
constexpr int TILE = C * D * 2;       // 16 KB
constexpr int HALF_ROWS = 64 * 16;    // byte offset of row 64 in an IL R=128 tile

// ---- shared memory map (bytes); regions reused by lifetime
constexpr int OFF_QU0 = 0;                  // QU slot 0 (see OFF_QU1)
constexpr int OFF_K = OFF_QU0 + TILE;        // 2 slots: k (raw, then k_hat), chunk parity
constexpr int OFF_DO = OFF_K + 2 * TILE;    // dO     IL R=64 x 128
constexpr int OFF_V = OFF_DO + TILE;        // V -> dV staging
constexpr int OFF_H = OFF_V + TILE;         // H^T    IL R=128 x 128
constexpr int OFF_DH = OFF_H + D * D * 2;   // dH^T   IL R=128 x 128
constexpr int OFF_X = OFF_DH + D * D * 2;   // X      IL R=64 x 64 (record)
constexpr int OFF_Z = OFF_X + C * C * 2;    // Z^T (record) -> U'^T in place
constexpr int OFF_R = OFF_Z + TILE;         // R -> Y [0,8K) + G1 [8K,16K)
// QU slots alternate by chunk parity: q (raw -> q_hat -> dq staging in place)
// of chunk c in one, dU'^T of chunk c then q of chunk c-1 in the other
constexpr int OFF_QU1 = OFF_R + TILE;
constexpr int OFF_A = OFF_QU1 + TILE;       // A_m -> dX -> dA
constexpr int OFF_VEC = OFF_A + C * C * 2;  // beta, r, s, nq, nk, db1[2], db2[2], dot[2], dotq[2], (4 spare)
// gated: gate vectors of the chunk and the dl/dG partials
constexpr int OFF_GV = OFF_VEC + 17 * C * 4;  // gG, gam, gD [64] each
// colT1[4][64] colT2[4][64] pkh[2][64] DD[2][64] rowT1[2][64] tq[2][64] dG[64] hdot[8] gCn
constexpr int OFF_GP = OFF_GV + 3 * C * 4;
constexpr int GP_FLOATS = 4 * C + 4 * C + 2 * C + 2 * C + 2 * C + 2 * C + C + 8 + 8;
constexpr int OFF_N = OFF_GP + GP_FLOATS * 4;  // record row norms [||k|| | ||q||] fp32
constexpr int SMEM_BYTES = OFF_N + 2 * C * 4;
static_assert(SMEM_BYTES <= 232448 - 1024, "shared memory budget");

// ---- TMEM column map (512 columns)
constexpr uint32_t TM_DH = 0;                            // dH^T, M=128
constexpr uint32_t TM_G = 128;                           // raw Q K^T | K_hat K_hat^T (lane+16)
constexpr uint32_t TM_DK = 192, TM_DQ = 192 | LO16;      // dK | dQ  (M=64, 128 cols)
constexpr uint32_t TM_DU = 320;                          // dU'^T, M=128 (M1-P3)
constexpr uint32_t TM_DX = 320, TM_GB = 320;             // dX' (M3-P5), G (M6-P7)
constexpr uint32_t TM_P = 384;                           // P[:, :64] | P[:, 64:] (M3-P5)
constexpr uint32_t TM_DA = 384, TM_Y = 384 | LO16;       // dA | Y (M5-P6)
constexpr uint32_t TM_KH = 448;                          // (K H)[:, :64] | [:, 64:], raw K

enum { BAR_SIMT = 1 };
// issuer -> SIMT: MMA commits and TMA arrivals
enum { MB_AL, MB_R, MB_DU, MB_P, MB_DH, MB_A, MB_LD, MB_GB, MB_K, MB_MAIN, MB_QL, MB_KL0, MB_KL1, MB_DHK,
       MB_P1, MB_N };
// SIMT -> issuer hand-offs (SG_STG: issuer -> SIMT, staging regions free)
enum { SG_DHI, SG_A, SG_P3, SG_P5, SG_P6, SG_P7, SG_P8, SG_STG, SG_RFREE, SG_P5A, SG_N };

__device__ __forceinline__ void ld32(uint32_t tm, int wwarp, uint32_t col, float (&f)[32]) {
  uint32_t r[2][16];
  tmem_ld16(taddr(tm, wwarp * 32, col), r[0]);
  tmem_ld16(taddr(tm, wwarp * 32, col + 16), r[1]);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) f[16 * i + j] = __uint_as_float(r[i][j]);
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// reduce-scatter across N lanes (N = 32, or 16 within each half-warp): on
// return lane l holds the sum over the N lanes of v[l % N]
template <int N>
__device__ __forceinline__ float reduce_scatter(float (&v)[N], int lane) {
#pragma unroll
  for (int m = N / 2; m >= 1; m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? v[i] : v[i + m];
      const float keep = up ? v[i + m] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  return v[0];
}
// Gamma(i, j) = e^{G_i - G_j} for j <= i; 1 above the diagonal (masked by
// index, not by clamping the exponent: g > 0 is allowed)
__device__ __forceinline__ float gamma_ij(const float* gG, int i, int j) {
  return __expf(j <= i ? gG[i] - gG[j] : 0.f);
}
// Two 32-column loads behind one wait (the TMEM load latency is paid once)
__device__ __forceinline__ void ld32x2(uint32_t tm, int wwarp, uint32_t ca, float (&fa)[32],
                                       uint32_t cb, float (&fb)[32]) {
  uint32_t r[4][16];
  tmem_ld16(taddr(tm, wwarp * 32, ca), r[0]);
  tmem_ld16(taddr(tm, wwarp * 32, ca + 16), r[1]);
  tmem_ld16(taddr(tm, wwarp * 32, cb), r[2]);
  tmem_ld16(taddr(tm, wwarp * 32, cb + 16), r[3]);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    fa[j] = __uint_as_float(r[0][j]);
    fa[16 + j] = __uint_as_float(r[1][j]);
    fb[j] = __uint_as_float(r[2][j]);
    fb[16 + j] = __uint_as_float(r[3][j]);
  }
}
__device__ __forceinline__ void ld16f(uint32_t tm, int wwarp, uint32_t col, float (&f)[16]) {
  uint32_t r[16];
  tmem_ld16(taddr(tm, wwarp * 32, col), r);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(r[j]);
}

#ifdef DN_TIMING
// Test-only phase timestamps of CTA 0 (tests/test_tc_timing.py, -DDN_TIMING):
// slots 0-15 by SIMT threads 0 / 128, slots 16-31 by the issuer.
__device__ long long* dn_tim_bwd = nullptr;
#define BSTAMP(slot)                                                        \
  do {                                                                      \
    if (dn_tim_bwd != nullptr && blockIdx.x == 0 && (tid & 127) == 0)       \
      dn_tim_bwd[(size_t)it * 32 + (slot)] = clock64();                     \
  } while (0)
#define ISTAMP(slot)                                                         \
  do {                                                                       \
    if (dn_tim_bwd != nullptr && blockIdx.x == 0)                            \
      dn_tim_bwd[(size_t)it * 32 + (slot)] = clock64();                      \
  } while (0)
// per-CTA [globaltimer start, end, smid] after the CTA-0 stamps
#define CTA_STAMP(k, v)                                                      \
  do {                                                                       \
    if (dn_tim_bwd != nullptr) dn_tim_bwd[(size_t)a.NC * 32 + blockIdx.x * 4 + (k)] = (v); \
  } while (0)
__device__ __forceinline__ long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return (long long)t;
}
__device__ __forceinline__ long long smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#else
#define BSTAMP(slot) do { } while (0)
#define ISTAMP(slot) do { } while (0)
#define CTA_STAMP(k, v) do { } while (0)
#endif

// SIMT -> issuer hand-off: operand tiles written by the 256 SIMT threads
// become visible to the tensor core / TMA (async proxy), TMEM reads are
// ordered before the issuer's next tcgen05 op, then one arrival.
__device__ __forceinline__ void simt_signal(uint64_t* bar, int tid) {
  fence_proxy_async();
  fence_before_sync();
  grp_sync<256>(BAR_SIMT);
  if (tid == 0) mbar_arrive(bar);
}

// SEG1 = pass 1 of the segment-parallel backward: only the
// dH chain of the segment, from dH = 0 at its end, down to its start (the
// segment-local dl/dH_start); no local gradients, no stores.
// GATED = Gated DeltaNet backward (R23, §4.9; the exact adjoint of
// tc_fwd_kernel<false, true>, oracle/forms.py gated_chunkwise_backward).  With
// the chunk's cumulative log-gate G, gamma = e^G, Gamma(i,j) = e^{G_i - G_j},
// D_j = e^{G_63 - G_j} (all formed from differences, never as ratios):
//   dU'^T = (dH^T K^T diag(D) + dO^T (Gamma . A_m)) diag(s)   [two accumulators]
//   R = V - diag(gamma s) K H,  sDV = diag(gamma) dV (dV itself stored from P5)
//   dK = diag(D) U' dH^T (rescaled in TMEM) - (gamma dV) H^T + dS^T Q_hat + ...
//   dS = Gamma . dA;  G1 = diag(beta) (Gamma . G)
//   dO is scaled by gamma in place once dA has read it (P6); then
//   dH += (gamma dO)^T Q_hat and dQ = (gamma dO) H^T + dS K_hat
//   dH <- gamma_63 dH rescaled in TMEM when its bf16 image is taken (P5b)
// and dl/dG_i = q_hat_i . (gamma dO H^T)_i + rowsum(T1)_i - colsum(T1)_i + rowsum(T2)_i - colsum(T2)_i
//   - beta_i gamma_i rowsum(P . K_hat H)_i - DD_i
//   + [i = 63] (sum_j DD_j + gamma_63 <dH, H_t>),
// T1 = dS . Q_hat K_hat^T, T2 = G1 . K_hat K_hat^T, DD_j = D_j k_hat_j . (U' dH^T)_j
// (the first term is read in P7 before dS K_hat accumulates into dQ, and the
// T1 row and column sums come from the same fp32 values, so their diagonal
// cancels exactly under fast decay); dg = reverse cumulative sum of dl/dG
// within the chunk.
template <bool SEG1, bool GATED = false>
__global__ void __launch_bounds__(NT, 1)
    tc_bwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                  const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mDO,
                  const __grid_constant__ CUtensorMap mDQ, const __grid_constant__ CUtensorMap mDK,
                  const __grid_constant__ CUtensorMap mDV, Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mb[MB_N], sg[SG_N];
  __shared__ uint32_t tslot;
  uint8_t *sDO = smem + OFF_DO, *sV = smem + OFF_V, *sH = smem + OFF_H,
          *sDH = smem + OFF_DH, *sX = smem + OFF_X, *sZ = smem + OFF_Z, *sR = smem + OFF_R,
          *sA = smem + OFF_A;
  auto qu = [&](int slot) { return smem + (slot ? OFF_QU1 : OFF_QU0); };
  uint8_t* sUP = sZ;               // U'^T (converted in place from the record's Z^T)
  uint8_t* sDV = sV;               // dV staging (in place over V)
  uint8_t* sDX = sA;               // dX after M2
  uint8_t* sDA = sA;               // dA after M5
  uint8_t* sY = sR;                // after M3
  uint8_t* sG1 = sR + 8192;
  float* sb = reinterpret_cast<float*>(smem + OFF_VEC);  // beta
  float* sr = sb + C;          // 1/max(||q||,eps) (0: padded)
  float* ss = sr + C;          // 1/max(||k||,eps)
  float* nq = ss + C;          // ||q||
  float* nk = nq + C;          // ||k||
  float* db1 = nk + C;         // [2][64] rowsum(P . R) partials
  float* db2 = db1 + 2 * C;    // [2][64] rowsum(G . K K^T) partials
  float* sdot = db2 + 2 * C;   // [2][64] dk-adjoint dot partials
  float* sdotq = sdot + 2 * C; // [2][64] dq-adjoint dot partials
  // gated only
  float* gG = reinterpret_cast<float*>(smem + OFF_GV);  // in-chunk cumulative log-gate
  float* gam = gG + C;         // e^G
  float* gD = gam + C;         // e^{G_63 - G}
  float* colT1 = reinterpret_cast<float*>(smem + OFF_GP);  // [4 warps][64]
  float* colT2 = colT1 + 4 * C;  // [4 warps][64]
  float* pkh = colT2 + 4 * C;    // [2][64] rowsum(P . K_hat H) partials
  float* ddp = pkh + 2 * C;      // [2][64] k_hat . (U' dH^T) partials
  float* rowT1 = ddp + 2 * C;    // [2][64] rowsum(T1) partials
  float* tqp = rowT1 + 2 * C;    // [2][64] q_hat . (gamma dO H^T) partials
  float* dGs = tqp + 2 * C;      // [64] dl/dG of the chunk
  float* hdot = dGs + C;         // [8] <dH image, H_t> per warp
  float* gCn = hdot + 8;         // e^{G_63} of the next chunk processed (c - 1)
  static_assert(!(SEG1 && GATED), "the gated backward runs one CTA per unit");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = (tid >> 7) & 1, w = tid & 127, wwarp = w >> 5;
  const int r64 = wwarp * 16 + (lane & 15);  // M=64 accumulator row of this lane
  const bool lo = lane < 16;
  // segment of this CTA (tc_fwd.cu): local chunk c is global chunk cbase + c,
  // token T0 + c*C; L counts tokens from T0
  const int nseg = a.nseg > 1 ? a.nseg : 1;
  const int unit = blockIdx.x / nseg, seg = blockIdx.x % nseg;
  const int cbase = nseg > 1 ? seg * a.seg_len : 0;
  const int NC = nseg > 1 ? min(a.seg_len, a.NC - cbase) : a.NC;
  const int T0 = cbase * C;
  const int L = a.L - T0;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const bool comp = (a.flags & DELTANET_COMPENSATED) != 0;  // DESIGN.md R19
  const float eps = a.eps;
  const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * a.L + T0;
  __nv_bfloat16* dbeta = (__nv_bfloat16*)a.dbeta + (size_t)unit * a.L + T0;
  const uint8_t* states = (const uint8_t*)a.states + ((size_t)unit * a.NC + cbase) * (D * D * 2);
  const uint8_t* recs = (const uint8_t*)a.scratch + ((size_t)unit * a.NC + cbase) * REC_BYTES;

  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    CTA_STAMP(0, gtimer());
    CTA_STAMP(2, smid());
    for (int i = 0; i < MB_N; ++i) mbar_init(&mb[i], 1);
    for (int i = 0; i < SG_N; ++i) mbar_init(&sg[i], 1);
    mbar_fence_init();
    prefetch_tmap(&mQ);
    prefetch_tmap(&mK);
    prefetch_tmap(&mV);
    prefetch_tmap(&mDO);
    prefetch_tmap(&mDQ);
    prefetch_tmap(&mDK);
    prefetch_tmap(&mDV);
  }
  cta_sync();
  const uint32_t tm = tslot;

  if (warp == 9) {
    // =====================================================================
    // TMA warp (lane 0): every load and store.  Chunk c-1's tiles are loaded
    // as their regions retire during chunk c: K at the start of chunk c
    // (double-buffered), dO / V / H / Z after M5 (MB_LD), X after G (MB_GB),
    // Q after M3 (into the dU'^T slot).  SG_STG tells the SIMT warps that the
    // dq staging (the other q slot) has been read out.
    // =====================================================================
    if (lane == 0) {
      // SEG1 reads only dO and X besides q, k
      constexpr uint32_t MAIN_BYTES = 2 * C * 4 +  // the record's row norms
          (SEG1 ? TILE + C * C * 2 : 3 * TILE + D * D * 2 + C * C * 2);  // dO V Z | H | X
      auto load_k = [&](int c, int slot) {  // own barrier per slot (one phase per use)
        mbar_expect_tx(&mb[MB_KL0 + slot], TILE);
        tma_load_4d(smem + OFF_K + slot * TILE, &mK, 0, T0 + c * C, 0, unit, &mb[MB_KL0 + slot]);
      };
      auto load_rest = [&](int c) {  // dO, V, H_t, Z^T (opens the MB_MAIN phase, X included)
        mbar_expect_tx(&mb[MB_MAIN], MAIN_BYTES);
        tma_load_4d(sDO, &mDO, 0, T0 + c * C, 0, unit, &mb[MB_MAIN]);
        bulk_load(smem + OFF_N, recs + (size_t)c * REC_BYTES + REC_N, 2 * C * 4, &mb[MB_MAIN]);
        if (!SEG1) {
          tma_load_4d(sV, &mV, 0, T0 + c * C, 0, unit, &mb[MB_MAIN]);
          bulk_load(sH, states + (size_t)c * D * D * 2, D * D * 2, &mb[MB_MAIN]);
          bulk_load(sZ, recs + (size_t)c * REC_BYTES + REC_Z, D * C * 2, &mb[MB_MAIN]);
        }
      };
      auto load_x = [&](int c) {
        bulk_load(sX, recs + (size_t)c * REC_BYTES + REC_X, C * C * 2, &mb[MB_MAIN]);
      };
      auto load_a = [&](int c) {  // the forward's A into sA (free once M6 / M7 are done)
        mbar_expect_tx(&mb[MB_AL], C * C * 2);
        bulk_load(sA, recs + (size_t)c * REC_BYTES + REC_A, C * C * 2, &mb[MB_AL]);
      };
      auto load_q = [&](int c, int slot) {
        mbar_expect_tx(&mb[MB_QL], TILE);
        tma_load_4d(qu(slot), &mQ, 0, T0 + c * C, 0, unit, &mb[MB_QL]);
      };
      if (NC > 0) {
        load_k(NC - 1, 0);
        load_rest(NC - 1);
        load_x(NC - 1);
        load_a(NC - 1);
        load_q(NC - 1, 0);
      }
      mbar_arrive(&sg[SG_STG]);
#pragma unroll 1
      for (int it = 0; it < NC; ++it) {
        const int c = NC - 1 - it, t0 = T0 + c * C;
        const uint32_t ph = it & 1;
        if (it > 0) {  // tail of chunk c+1: its epilogue read q_hat / k_hat
          mbar_wait(&sg[SG_P8], ph ^ 1);
          if (!SEG1) {  // dq / dk were staged in place over q_hat / k_hat of chunk c+1
            tma_store_4d(&mDQ, qu((it + 1) & 1), 0, t0 + C, 0, unit);
            tma_store_4d(&mDK, smem + OFF_K + ((it + 1) & 1) * TILE, 0, t0 + C, 0, unit);
            bulk_commit();
          }
          bulk_wait_read0();           // both read out: the q slot takes dU'^T (P3),
          mbar_arrive(&sg[SG_STG]);    // the k slot chunk c-1's k
          if (c > 0) load_k(c - 1, (it + 1) & 1);
        } else if (c > 0) {
          load_k(c - 1, 1);
        }
        if (c > 0) {  // q of chunk c-1 into the slot of dU'^T (last read by M3)
          mbar_wait(&mb[MB_P], ph);
          load_q(c - 1, (it + 1) & 1);
        }
        mbar_wait(&sg[SG_P5], ph);
        if (!SEG1 && !GATED) {
          tma_store_4d(&mDV, sDV, 0, t0, 0, unit);
          bulk_commit();
        }
        if (GATED) {  // sDV holds gamma dV (the operands'); dV itself was staged in
          // the R slot, free between M3 and P6's Y: store it, then hand the slot back
          tma_store_4d(&mDV, sR, 0, t0, 0, unit);
          bulk_commit();
          bulk_wait_read0();
          mbar_arrive(&sg[SG_RFREE]);
        }
        if (c > 0) {
          mbar_wait(&mb[MB_LD], ph);  // dO, H^T, U' read by M5; V once dV is read out
          bulk_wait_read0();
          load_rest(c - 1);
          mbar_wait(&mb[MB_GB], ph);  // X read by G
          load_x(c - 1);
          mbar_wait(&mb[SEG1 ? MB_GB : MB_K], ph);  // dA (in sA) read by M6 (SEG1: A by M2)
          load_a(c - 1);
        }
      }
      if (NC > 0) {
        mbar_wait(&sg[SG_P8], (NC - 1) & 1);
        if (!SEG1) {
          tma_store_4d(&mDQ, qu((NC - 1) & 1), 0, T0, 0, unit);
          tma_store_4d(&mDK, smem + OFF_K + ((NC - 1) & 1) * TILE, 0, T0, 0, unit);
          bulk_commit();
        }
      }
      bulk_wait0();
    }
    __syncwarp();
  } else if (warp == 8) {
    // =====================================================================
    // MMA warp (lane 0): every tcgen05.mma.  Software-pipelined: chunk c-1's
    // first products are issued as soon as its tiles land, under chunk c's
    // epilogues.
    // =====================================================================
    if (lane == 0) {
      const uint32_t aDO = smem_u32(sDO), aH = smem_u32(sH),
                     aDH = smem_u32(sDH), aX = smem_u32(sX), aA = smem_u32(sA),
                     aR = smem_u32(sR), aDA = smem_u32(sDA),
                     aDX = smem_u32(sDX), aY = smem_u32(sY), aG1 = smem_u32(sG1),
                     aDV = smem_u32(sDV), aUP = smem_u32(sUP);
#pragma unroll 1
      for (int it = 0; it < NC; ++it) {
        const int ks = it & 1;
        const uint32_t ph = it & 1;
        const uint32_t aK = smem_u32(smem + OFF_K + ks * TILE);
        const uint32_t aQ = smem_u32(qu(ks)), aDUP = smem_u32(qu(ks ^ 1));

        // M1a (raw k): dH^T K^T | K H.  TMEM DU / KH were released by the
        // previous chunk's P7 / P5 (waited below in program order).
        mbar_wait(&mb[MB_KL0 + ks], (it >> 1) & 1);
        mbar_wait(&mb[MB_MAIN], ph);
        mbar_wait(&sg[SG_DHI], ph);
        fence_after_sync();
        ISTAMP(16);
        {
          const uint32_t idg = idesc_bf16(64, 64, false, false);
          // K H first (the SIMT warps wait on it for R)
          if (!SEG1) {
#pragma unroll
            for (int k0 = 0; k0 < D; k0 += 16) {
              mma_bf16(tm + TM_KH, desc_k(aK, C, k0), desc_k(aH, D, k0), idg, k0 > 0);
              mma_bf16(tm + TM_KH + LO16, desc_k(aK, C, k0), desc_k(aH + HALF_ROWS, D, k0), idg,
                       k0 > 0);
            }
          }
          mma_commit(&mb[MB_R]);
        }
        ISTAMP(17);
        ISTAMP(18);
        {
          // dH^T K^T (P3 reads it after M2's MB_DU).  Q K^T is not formed:
          // the forward's A comes with the record (load_a).
          const uint32_t idd = idesc_bf16(128, 64, false, false);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DU, desc_k(aDH, D, k0), desc_k(aK, C, k0), idd, k0 > 0);
          mma_commit(&mb[MB_DHK]);  // the last reader of the raw k tile (P3 normalises it)
        }
        ISTAMP(19);

        // M2: dU'^T += dO^T A_m
        mbar_wait(&sg[SG_A], ph);
        fence_after_sync();
        ISTAMP(20);
        {
          const uint32_t ida = idesc_bf16(128, 64, true, true);
#pragma unroll
          // gated: its own accumulator (TM_P, free until M3); P3 adds
          // diag(D) times the dH^T K^T term
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + (GATED ? TM_P : TM_DU), desc_mn(aDO, C, k0), desc_mn(aA, C, k0), ida,
                     GATED ? k0 > 0 : 1);
          mma_commit(&mb[MB_DU]);
        }
        if (!GATED && !SEG1) {
          // M2b: dQ = dO H^T now, under P3 (the tensor pipe would idle there;
          // TM_DQ was read by P8 of chunk c+1, which precedes SG_A of chunk c)
          const uint32_t id_q = idesc_bf16(64, 128, false, true);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DQ, desc_k(aDO, C, k0), desc_mn(aH, D, k0), id_q, k0 > 0);
        }

        // M3: P = X^T dU' (two N=64 halves), dX' = dU' R^T
        // M4a: dH += Q_hat^T dO ; dK = U' dH^T (dH image of chunk c+1) ; K_hat K_hat^T
        mbar_wait(&sg[SG_P3], ph);
        fence_after_sync();
        ISTAMP(21);
        if (GATED) {
          // dK = U' dH^T first: P5 takes k_hat . (U' dH^T) and rescales it by D
          // before M5 accumulates (MB_P covers it); dH += (gamma dO)^T Q_hat
          // waits for P6 (dO scaled in place)
          const uint32_t id_k1 = idesc_bf16(64, 128, true, true);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DK, desc_mn(aUP, D, k0), desc_mn(aDH, D, k0), id_k1, k0 > 0);
          const uint32_t idp = idesc_bf16(64, 64, true, false);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16) {
            mma_bf16(tm + TM_P, desc_mn(aX, C, k0), desc_k(aDUP, D, k0), idp, k0 > 0);
            mma_bf16(tm + TM_P + LO16, desc_mn(aX, C, k0), desc_k(aDUP + HALF_ROWS, D, k0), idp,
                     k0 > 0);
          }
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DX, desc_mn(aDUP, D, k0), desc_k(aR, C, k0), idp, k0 > 0);
          const uint32_t idg = idesc_bf16(64, 64, false, false);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_G + LO16, desc_k(aK, C, k0), desc_k(aK, C, k0), idg, k0 > 0);
          mma_commit(&mb[MB_P]);
        } else {
          const uint32_t idp = idesc_bf16(64, 64, true, false);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16) {
            mma_bf16(tm + TM_P, desc_mn(aX, C, k0), desc_k(aDUP, D, k0), idp, k0 > 0);
            mma_bf16(tm + TM_P + LO16, desc_mn(aX, C, k0), desc_k(aDUP + HALF_ROWS, D, k0), idp,
                     k0 > 0);
          }
          mma_commit(&mb[MB_P1]);  // P alone: P5 starts on dV while dX' runs
          if (!SEG1) {
#pragma unroll
            for (int k0 = 0; k0 < D; k0 += 16)
              mma_bf16(tm + TM_DX, desc_mn(aDUP, D, k0), desc_k(aR, C, k0), idp, k0 > 0);
          }
          mma_commit(&mb[MB_P]);
          const uint32_t id1 = idesc_bf16(128, 128, true, true);
          const uint32_t id_k1 = idesc_bf16(64, 128, true, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_DH, desc_mn(aDO, C, k0), desc_mn(aQ, C, k0), id1, 1);
          if (!SEG1) {
#pragma unroll
            for (int k0 = 0; k0 < D; k0 += 16)
              mma_bf16(tm + TM_DK, desc_mn(aUP, D, k0), desc_mn(aDH, D, k0), id_k1, k0 > 0);
            // K_hat K_hat^T (k normalised in P3) for the dbeta term of P7
            const uint32_t idg = idesc_bf16(64, 64, false, false);
#pragma unroll
            for (int k0 = 0; k0 < D; k0 += 16)
              mma_bf16(tm + TM_G + LO16, desc_k(aK, C, k0), desc_k(aK, C, k0), idg, k0 > 0);
          }
        }
        ISTAMP(22);

        // M4b: dH -= W^T dU' = K_hat^T dV  (W = X diag(b) K_hat, dV = diag(b) X^T dU')
        // M5: dA, Y | dK -= dV H^T (ungated: dQ = dO H^T was M2b)
        // (ungated full backward: M4b as soon as dV is staged, SG_P5A, so
        // the dH update overlaps P5's dX conversion)
        mbar_wait(&sg[(!GATED && !SEG1) ? SG_P5A : SG_P5], ph);
        fence_after_sync();
        ISTAMP(23);
        {
          const uint32_t id2 = idesc_bf16(128, 128, true, true, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_DH, desc_mn(aDV, C, k0), desc_mn(aK, C, k0), id2, 1);
          if (!GATED) mma_commit(&mb[MB_DH]);
          if (SEG1) {  // the chain is all: dO, X and the q / k slots are free
            mma_commit(&mb[MB_LD]);
            mma_commit(&mb[MB_GB]);
            continue;
          }
          if (!GATED) {  // dX staged (Y reads it)
            mbar_wait(&sg[SG_P5], ph);
            fence_after_sync();
          }
          const uint32_t id_da = idesc_bf16(64, 64, false, true);
          const uint32_t id_y = idesc_bf16(64, 64, true, true);
          const uint32_t id_k2 = idesc_bf16(64, 128, false, true, true);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DA, desc_k(aDO, C, k0), desc_mn(aUP, D, k0), id_da, k0 > 0);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_Y, desc_mn(aX, C, k0), desc_mn(aDX, C, k0), id_y, k0 > 0);
          mma_commit(&mb[MB_A]);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DK, desc_k(aDV, C, k0), desc_mn(aH, D, k0), id_k2, 1);
          if (!GATED) mma_commit(&mb[MB_LD]);
        }
        ISTAMP(24);

        // M6: G = -Y X^T first (the SIMT warps wait on it) ; dQ += dA K_hat ;
        // dK += dA^T Q_hat
        mbar_wait(&sg[SG_P6], ph);
        fence_after_sync();
        ISTAMP(25);
        if (GATED) {  // dO now holds gamma dO
          const uint32_t id1 = idesc_bf16(128, 128, true, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_DH, desc_mn(aDO, C, k0), desc_mn(aQ, C, k0), id1, 1);
          mma_commit(&mb[MB_DH]);
          const uint32_t id_q = idesc_bf16(64, 128, false, true);
#pragma unroll
          for (int k0 = 0; k0 < D; k0 += 16)
            mma_bf16(tm + TM_DQ, desc_k(aDO, C, k0), desc_mn(aH, D, k0), id_q, k0 > 0);
          mma_commit(&mb[MB_LD]);
        }
        {
          const uint32_t id_q = idesc_bf16(64, 128, false, true);
          const uint32_t id_k = idesc_bf16(64, 128, true, true);
          const uint32_t id_g = idesc_bf16(64, 64, false, false, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_GB, desc_k(aY, C, k0), desc_k(aX, C, k0), id_g, k0 > 0);
          mma_commit(&mb[MB_GB]);
          if (!GATED) {  // (gated: after P7, which reads TM_DQ = (gamma dO) H^T)
#pragma unroll
            for (int k0 = 0; k0 < C; k0 += 16) {
              mma_bf16(tm + TM_DQ, desc_k(aDA, C, k0), desc_mn(aK, C, k0), id_q, 1);
              mma_bf16(tm + TM_DK, desc_mn(aDA, C, k0), desc_mn(aQ, C, k0), id_k, 1);
            }
          }
        }
        ISTAMP(26);

        // M7: dK += (G1 + G1^T) K_hat
        mbar_wait(&sg[SG_P7], ph);
        fence_after_sync();
        ISTAMP(27);
        if (GATED) {  // M6's dQ += dS K_hat ; dK += dS^T Q_hat
          const uint32_t id_q = idesc_bf16(64, 128, false, true);
          const uint32_t id_k = idesc_bf16(64, 128, true, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16) {
            mma_bf16(tm + TM_DQ, desc_k(aDA, C, k0), desc_mn(aK, C, k0), id_q, 1);
            mma_bf16(tm + TM_DK, desc_mn(aDA, C, k0), desc_mn(aQ, C, k0), id_k, 1);
          }
        }
        {
          const uint32_t id_m = idesc_bf16(64, 128, false, true);
          const uint32_t id_mt = idesc_bf16(64, 128, true, true);
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16) {
            mma_bf16(tm + TM_DK, desc_k(aG1, C, k0), desc_mn(aK, C, k0), id_m, 1);
            mma_bf16(tm + TM_DK, desc_mn(aG1, C, k0), desc_mn(aK, C, k0), id_mt, 1);
          }
          mma_commit(&mb[MB_K]);
        }
      }
    }
    __syncwarp();
  } else {
    // =====================================================================
    // SIMT warps 0-7 (two warpgroups; phases split columns between them)
    // =====================================================================
    // gated: log-gates of the chunk processed next, rows (lane, 32 + lane) in
    // warps 0-1, read one chunk ahead; e^{G_63} of the last chunk rescales dhT
    const float* gsrc = GATED ? a.g + (size_t)unit * a.L + T0 : nullptr;
    auto gload = [&](int cc, int j) {
      return (GATED && cc >= 0 && cc * C + j < L) ? gsrc[cc * C + j] : 0.f;
    };
    float ga = 0.f, gb = 0.f;
    if (GATED) {
      if (tid < C) {
        ga = gload(NC - 1, lane);
        gb = gload(NC - 1, 32 + lane);
      }
      if (tid < 32) {
        const float t = warp_sum(ga) + warp_sum(gb);
        if (tid == 0) gCn[0] = __expf(t);
      }
      grp_sync<256>(BAR_SIMT);
    }
    {
      // dH^T <- dhT^T in TMEM (lane dv = w; columns split by warpgroup) and
      // its bf16 image for the first chunk (gated: TMEM holds e^{G_63} dhT)
      // the cotangent at this segment's end: dhT for the last segment, the
      // scanned dl/dH for the others (pass 3), zero in pass 1
      const float* dhT = SEG1 ? nullptr
                         : (seg < nseg - 1) ? a.hseg + ((size_t)unit * nseg + seg) * D * D
                         : a.dhT ? a.dhT + (size_t)unit * D * D : nullptr;
#pragma unroll 1
      for (int c0 = 64 * wg; c0 < 64 * wg + 64; c0 += 16) {
        uint32_t r[16];
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          f[j] = dhT ? dhT[(size_t)(c0 + j) * D + w] : 0.f;
          r[j] = __float_as_uint(GATED ? f[j] * gCn[0] : f[j]);
        }
        tmem_st16(taddr(tm, wwarp * 32, TM_DH + c0), r);
        il_store8(sDH, D, w, c0, f);
        il_store8(sDH, D, w, c0 + 8, f + 8);
      }
      tmem_st_wait();
      simt_signal(&sg[SG_DHI], tid);
    }

    // beta of the next chunk is read from global one chunk ahead
    float bnext = (tid < C && NC > 0 && (NC - 1) * C + tid < L)
                      ? __bfloat162float(beta[(NC - 1) * C + tid])
                      : 0.f;
#pragma unroll 1
    for (int it = 0; it < NC; ++it) {
      const int c = NC - 1 - it, t0 = c * C, ks = it & 1;
      const uint32_t ph = it & 1;
      uint8_t* sK = smem + OFF_K + ks * TILE;
      uint8_t* sQ = qu(ks);         // q -> q_hat -> dq staging
      uint8_t* sDUP = qu(ks ^ 1);   // dU'^T
      uint32_t qkg[8];              // gated: Gamma . Q_hat K_hat^T of P2 (bf16 pairs, for P6)

      // ================= P1: k norms ; U' ; R = V - diag(s) K H ; q norms
      BSTAMP(0);
      if (tid < C) sb[tid] = bnext;
      if (GATED && tid < C) {
        // G = in-chunk inclusive cumsum of g; gamma = e^G; D = e^{G_63 - G}
        float x = tid < 32 ? ga : gb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const float tot0 = warp_sum(ga), tot1 = warp_sum(gb);
        const float Gi = x + (tid >= 32 ? tot0 : 0.f);
        gG[tid] = Gi;
        gam[tid] = __expf(Gi);
        gD[tid] = __expf((tot0 + tot1) - Gi);
        ga = gload(c - 1, lane);  // next chunk processed (summed in P3)
        gb = gload(c - 1, 32 + lane);
      }
      mbar_wait(&mb[MB_KL0 + ks], (it >> 1) & 1);
      mbar_wait(&mb[MB_MAIN], ph);
      // row norms of k and q from the forward's record (REC_N): s, r and the
      // norms the L2 adjoint needs, no pass over the tiles
      if (tid < 2 * C) {
        const int row = tid & (C - 1);
        const float n = reinterpret_cast<const float*>(smem + OFF_N)[tid];
        float inv = l2 ? 1.f / fmaxf(n, eps) : 1.f;
        if (t0 + row >= L) inv = 0.f;
        (tid < C ? ss : sr)[row] = inv;
        (tid < C ? nk : nq)[row] = n;
      }
      grp_sync<256>(BAR_SIMT);
      BSTAMP(1);
      if (GATED) {  // <dH image (dl/dH_{t+1}), H_t>: both bf16 IL R=128 images
        float hd = 0.f;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
          const int off = (tid + 256 * k8) * 16;
          float x8[8], y8[8];
          unpack8(*reinterpret_cast<const uint4*>(sH + off), x8);
          unpack8(*reinterpret_cast<const uint4*>(sDH + off), y8);
#pragma unroll
          for (int e = 0; e < 8; ++e) hd = fmaf(x8[e], y8[e], hd);
        }
        hd = warp_sum(hd);
        if (lane == 0) hdot[warp] = hd;
      }
      if (l2 && !SEG1 && !comp) {  // U'^T[dv][t] = Z^T[dv][t] * max(|k_t|, eps)  (row dv = w)
        // (with DELTANET_COMPENSATED the record holds U'^T itself; R19)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int col = 32 * wg + g * 8;
          float z8[8];
          il_load8(sUP, D, w, col, z8);
          const float4 n0 = *reinterpret_cast<const float4*>(nk + col);
          const float4 n1 = *reinterpret_cast<const float4*>(nk + col + 4);
          const float nn[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) z8[e] *= fmaxf(nn[e], eps);
          il_store8(sUP, D, w, col, z8);
        }
      }
      if (!SEG1) {  // (SEG1 needs no R)
        mbar_wait(&mb[MB_R], ph);
        fence_after_sync();
        BSTAMP(2);
        {
          // (K H) row r64: lanes < 16 hold columns [0,64), lanes >= 16 [64,128);
          // this warpgroup takes 32 of each half
          float f[32];
          ld32(tm, wwarp, TM_KH + 32 * wg, f);
          const float si = GATED ? ss[r64] * gam[r64] : ss[r64];  // gated: R = V - gamma K_hat H
          const int c0 = (lo ? 0 : 64) + 32 * wg;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float v8[8];
            il_load8(sV, C, r64, c0 + g * 8, v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) v8[e] = fmaf(-si, f[g * 8 + e], v8[e]);
            il_store8(sR, C, r64, c0 + g * 8, v8);
          }
        }
      }
      mbar_wait(&mb[MB_QL], ph);
      BSTAMP(3);

      // ================= P2: A_m = diag(r) A, A = tril(Q K^T) (gated: Gamma . A)
      // from the forward's record, scaled in place (thread: row r64, 16 columns)
      mbar_wait(&mb[MB_AL], ph);
      BSTAMP(4);
      {
        const float ri = sr[r64];
        const int c0 = 32 * wg + (lo ? 0 : 16);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float a8[8];
          il_load8(sA, C, r64, c0 + g * 8, a8);
#pragma unroll
          for (int e = 0; e < 8; ++e) a8[e] *= ri;
          if (GATED) {  // Gamma . Q_hat K_hat^T of this lane's 16 columns (T1 of P6)
#pragma unroll
            for (int e = 0; e < 8; e += 2)
              qkg[g * 4 + e / 2] = pack_bf16(a8[e] * ss[c0 + g * 8 + e],
                                             a8[e + 1] * ss[c0 + g * 8 + e + 1]);
          }
          il_store8(sA, C, r64, c0 + g * 8, a8);
        }
      }
      simt_signal(&sg[SG_A], tid);

      // ================= P3: q_hat, k_hat in place ; dU' = (..) diag(s) -> bf16
      if (wg == 1) mbar_wait(&mb[MB_DHK], ph);  // dH^T K^T has read the raw k tile
      if (l2) {  // no MMA reads raw q; dH^T K^T and K H have read raw k (MB_DHK);
        // thread: row w & 63 of q (wg0) or k (wg1), one column half
        const int row = w & 63;
        uint8_t* tile = wg == 0 ? sQ : sK;
        const float inv = (wg == 0 ? sr : ss)[row];
#pragma unroll
        for (int g = 8 * (w >> 6); g < 8 * (w >> 6) + 8; ++g) {
          float x[8];
          il_load8(tile, C, row, g * 8, x);
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] *= inv;
          il_store8(tile, C, row, g * 8, x);
        }
      }
      mbar_wait(&sg[SG_STG], ph);  // the dU' slot (dq staging of chunk c+1) read out
      mbar_wait(&mb[MB_DU], ph);
      fence_after_sync();
      BSTAMP(5);
      if (GATED && tid < 32) {  // e^{G_63} of chunk c-1 (P5b rescales dH by it)
        const float t = warp_sum(ga) + warp_sum(gb);
        if (tid == 0) gCn[0] = __expf(t);
      }
      {  // dU'^T (lane d_v = w) * s_j -> bf16
        float f[32];
        ld32(tm, wwarp, TM_DU + 32 * wg, f);
        if (GATED) {  // dU'^T = dH^T K^T diag(D) (TM_DU) + dO^T (Gamma . A_m) (TM_P)
          float p[32];
          ld32(tm, wwarp, TM_P + 32 * wg, p);
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = fmaf(f[e], gD[32 * wg + e], p[e]);
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4) {  // vector broadcast loads of s
          const float4 s4 = *reinterpret_cast<const float4*>(ss + 32 * wg + e);
          f[e] *= s4.x;
          f[e + 1] *= s4.y;
          f[e + 2] *= s4.z;
          f[e + 3] *= s4.w;
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) il_store8(sDUP, D, w, 32 * wg + g * 8, f + g * 8);
      }
      simt_signal(&sg[SG_P3], tid);
      BSTAMP(6);

      // ================= P5: P, R -> dV, dbeta part ; dX  (SEG1: dV only)
      if (tid < C && c > 0) bnext = __bfloat162float(beta[t0 - C + tid]);
      mbar_wait(&mb[(!GATED && !SEG1) ? MB_P1 : MB_P], ph);  // (ungated: P; dX' below)
      fence_after_sync();
      BSTAMP(7);
      if (SEG1) {  // dV = diag(beta) P only (the chain's K_hat^T dV)
        float p[32];
        ld32(tm, wwarp, TM_P + 32 * wg, p);
        const float bt = sb[r64];
        const int c0 = (lo ? 0 : 64) + 32 * wg;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float dv8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) dv8[e] = bt * p[g * 8 + e];
          il_store8(sDV, C, r64, c0 + g * 8, dv8);
        }
      } else {
        if (GATED) {
          // dK = U' dH^T (lanes < 16; lanes >= 16 carry TM_DQ's stale rows
          // back unchanged): DD partial k_hat . (U' dH^T), then rows * D
          float f[64];
          ld64(tm, wwarp, TM_DK + 64 * wg, f);
          float dd = 0.f;
          if (lo) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              float x8[8];
              il_load8(sK, C, r64, 64 * wg + g * 8, x8);
#pragma unroll
              for (int e = 0; e < 8; ++e) dd = fmaf(x8[e], f[g * 8 + e], dd);
            }
            ddp[wg * C + r64] = dd;
          }
          const float sc = lo ? gD[r64] : 1.f;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t r[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(f[16 * q4 + j] * sc);
            tmem_st16(taddr(tm, wwarp * 32, TM_DK + 64 * wg + 16 * q4), r);
          }
          tmem_st_wait();
        }
        BSTAMP(31);
        {
          // lanes < 16: columns [0,64), lanes >= 16: [64,128) of row r64, for
          // both P (TM_P) and K H (TM_KH); 32 of each half per warpgroup
          float p[32], f[32];
          // (gated: both behind one wait; the ungated kernel measured faster
          // with two -- DESIGN.md §11)
          if (GATED) {
            ld32x2(tm, wwarp, TM_P + 32 * wg, p, TM_KH + 32 * wg, f);
          } else {
            ld32(tm, wwarp, TM_P + 32 * wg, p);
            ld32(tm, wwarp, TM_KH + 32 * wg, f);
          }
          const float bt = sb[r64], si = ss[r64];
          const float gi = GATED ? gam[r64] : 1.f;
          const int c0 = (lo ? 0 : 64) + 32 * wg;
          float db = 0.f, pk = 0.f;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float v8[8], dv8[8];
            il_load8(sV, C, r64, c0 + g * 8, v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float kh = si * f[g * 8 + e];  // (K_hat H)[r64][.]
              const float rr = fmaf(-gi, kh, v8[e]);
              db = fmaf(p[g * 8 + e], rr, db);  // P . R
              if (GATED) pk = fmaf(p[g * 8 + e], kh, pk);
              dv8[e] = bt * p[g * 8 + e];
            }
            if (GATED) {  // dV staged in the R slot (TMA-stored); the operand tile takes gamma dV
              il_store8(sR, C, r64, c0 + g * 8, dv8);
#pragma unroll
              for (int e = 0; e < 8; ++e) dv8[e] *= gi;
            }
            il_store8(sDV, C, r64, c0 + g * 8, dv8);
          }
          db += __shfl_xor_sync(0xffffffffu, db, 16);
          if (lo) db1[wg * C + r64] = db;
          if (GATED) {
            pk += __shfl_xor_sync(0xffffffffu, pk, 16);
            if (lo) pkh[wg * C + r64] = pk;
          }
        }
        if (!GATED) {  // dV staged: M4b (the dH update) can start; then dX'
          simt_signal(&sg[SG_P5A], tid);
          mbar_wait(&mb[MB_P], ph);
          fence_after_sync();
        }
        // dX = dX' diag(beta) (lanes < 16: dX' rows), 16 columns at a time
        auto dx16 = [&](int cc, const float (&f)[16]) {
          const int col = 32 * wg + 16 * cc;
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = __shfl_xor_sync(0xffffffffu, f[8 + e], 16);
          if (lo) {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = f[e];
          }
          const int c8 = col + (lo ? 0 : 8);
          const float4 b0 = *reinterpret_cast<const float4*>(sb + c8);
          const float4 b1 = *reinterpret_cast<const float4*>(sb + c8 + 4);
          x[0] *= b0.x; x[1] *= b0.y; x[2] *= b0.z; x[3] *= b0.w;
          x[4] *= b1.x; x[5] *= b1.y; x[6] *= b1.z; x[7] *= b1.w;
          il_store8(sDX, C, r64, c8, x);
        };
        if (GATED) {  // both halves behind one TMEM wait
          float fdx[32];
          ld32(tm, wwarp, TM_DX + 32 * wg, fdx);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            float f[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) f[e] = fdx[16 * cc + e];
            dx16(cc, f);
          }
        } else {
#pragma unroll 1
          for (int cc = 0; cc < 2; ++cc) {
            float f[16];
            ld16f(tm, wwarp, TM_DX + 32 * wg + 16 * cc, f);
            dx16(cc, f);
          }
        }
      }
      simt_signal(&sg[SG_P5], tid);
      BSTAMP(8);

      // ================= P5b (under M5): dH image for chunk c-1 (gated:
      // after P6, since dH += (gamma dO)^T Q_hat needs dO scaled; TMEM dH is
      // then rescaled by e^{G_63} of chunk c-1)
      auto dh_image = [&]() {
        mbar_wait(&mb[MB_DH], ph);  // M4 done; dK = U' dH^T done reading the old image
        fence_after_sync();
        float f[64];
        ld64(tm, wwarp, TM_DH + 64 * wg, f);
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sDH, D, w, 64 * wg + g * 8, f + g * 8);
        if (GATED) {
          const float sc = gCn[0];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t r[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(f[16 * q4 + j] * sc);
            tmem_st16(taddr(tm, wwarp * 32, TM_DH + 64 * wg + 16 * q4), r);
          }
          tmem_st_wait();
        }
        simt_signal(&sg[SG_DHI], tid);
      };
      if (!GATED && c > 0) dh_image();
      BSTAMP(9);
      if (SEG1) {  // pass 1 stops at the chain; the TMA warp reloads the k slot
        simt_signal(&sg[SG_P8], tid);
        continue;
      }

      // ================= P6: dA -> bf16 (masked) | Y -> bf16
      mbar_wait(&mb[MB_A], ph);
      if (GATED) mbar_wait(&sg[SG_RFREE], ph);  // dV read out of the R slot (sY)
      fence_after_sync();
      BSTAMP(10);
      {
        float f[32];
        ld32(tm, wwarp, TM_DA + 32 * wg, f);  // lanes<16: dA row, lanes>=16: Y row
        // gated: T1 = dS . Q_hat K_hat^T = dA . qkg (P2).  Lane pairs split the
        // row's 32 columns as in P2 (lo: first 16, hi: last 16; the hi lane
        // takes its dA values from the lo lane), so every lane sums 16 values.
        if (GATED) {
          float t1[16];
          const int cb = 32 * wg + (lo ? 0 : 16);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float dap = __shfl_xor_sync(0xffffffffu, f[16 + e], 16);
            const float da = lo ? f[e] : dap;
            const uint32_t u = qkg[e / 2];
            const float qv = __uint_as_float((e & 1) ? (u & 0xffff0000u) : (u << 16));
            t1[e] = (cb + e <= r64) ? da * qv : 0.f;
          }
          float rt = 0.f;
#pragma unroll
          for (int e = 0; e < 16; ++e) rt += t1[e];
          rt += __shfl_xor_sync(0xffffffffu, rt, 16);
          if (lo) rowT1[wg * C + r64] = rt;
          // this warp's 16 rows summed per column: lane gets column cb + (lane & 15)
          const float cs = reduce_scatter<16>(t1, lane);
          colT1[wwarp * C + cb + (lane & 15)] = cs;
        }
        float err[4] = {0.f, 0.f, 0.f, 0.f};  // DELTANET_COMPENSATED: dA rows
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = 32 * wg + g * 8 + e;
            float v = f[g * 8 + e];
            if (GATED) {  // dS = Gamma . dA (branch-free: Y rows keep their value)
              const float gm = gamma_ij(gG, r64, j);
              v *= lo ? gm : 1.f;
            }
            x[e] = (!lo || j <= r64) ? v : 0.f;
          }
          if (comp && lo) {  // dQ = dA K_hat sums dA over j: carry the bf16
            // rounding error along j (4 interleaved 8-column blocks)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float xv = x[e] + err[g];
              x[e] = __bfloat162float(__float2bfloat16_rn(xv));
              err[g] = xv - x[e];
            }
          }
          il_store8(lo ? sDA : sY, C, r64, 32 * wg + g * 8, x);
        }
        BSTAMP(28);
        if (GATED) {
          // dO <- diag(gamma) dO in place (dA has read it: MB_A): thread = row
          // tid & 63, column quarter tid >> 6
          const int row = tid & 63, qt = tid >> 6;
          const float gr = gam[row];
#pragma unroll
          for (int g = 4 * qt; g < 4 * qt + 4; ++g) {
            float x8[8];
            il_load8(sDO, C, row, g * 8, x8);
#pragma unroll
            for (int e = 0; e < 8; ++e) x8[e] *= gr;
            il_store8(sDO, C, row, g * 8, x8);
          }
        }
      }
      simt_signal(&sg[SG_P6], tid);
      BSTAMP(11);
      if (GATED && c > 0) dh_image();

      // ================= P7: G1 = diag(b) G, dbeta part 2
      mbar_wait(&mb[MB_GB], ph);
      fence_after_sync();
      BSTAMP(12);
      {
        // lanes < 16 hold the G row (TM_GB), lanes >= 16 the K_hat K_hat^T row
        // (TM_G + 16); each lane pair splits every 16 columns 8 / 8
        float d2 = 0.f, t2[16];
        const float bi = sb[r64];
        // gated: G and K_hat K_hat^T columns [32 wg, 32 wg + 32) behind one wait
        float g32[32], k32[32];
        if (GATED) ld32x2(tm, wwarp, TM_GB + 32 * wg, g32, TM_G + 32 * wg, k32);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int col = 32 * wg + 16 * cc;
          float g16[16], k16[16], x[8];
          if (GATED) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              g16[e] = g32[16 * cc + e];
              k16[e] = k32[16 * cc + e];
            }
          } else {
            ld16f(tm, wwarp, TM_GB + col, g16);
            ld16f(tm, wwarp, TM_G + col, k16);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = __shfl_xor_sync(0xffffffffu, lo ? g16[8 + e] : k16[e], 16);
          const int c8 = col + (lo ? 0 : 8);
          float y[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = c8 + e;
            const float gr = lo ? g16[e] : x[e];
            const float kk = lo ? x[e] : k16[8 + e];
            float gv = (j < r64) ? gr : 0.f;
            if (GATED) gv *= gamma_ij(gG, r64, j);  // Gamma . G
            d2 = fmaf(gv, kk, d2);
            y[e] = bi * gv;
            if (GATED) t2[cc * 8 + e] = y[e] * kk;  // T2 = G1 . K_hat K_hat^T
          }
          il_store8(sG1, C, r64, c8, y);
        }
        d2 += __shfl_xor_sync(0xffffffffu, d2, 16);
        if (lo) db2[wg * C + r64] = d2;
        if (GATED) {  // column sums over this warp's 16 rows (lanes of equal lane >> 4)
          const float cs = reduce_scatter<16>(t2, lane);
          const int vi = lane & 15;
          colT2[wwarp * C + 32 * wg + 16 * (vi >> 3) + (lo ? 0 : 8) + (vi & 7)] = cs;
          // TM_DQ holds (gamma dO) H^T only (dS K_hat is issued after this
          // phase): lanes >= 16 take q_hat . (gamma dO H^T) of row r64
          float f[64];
          ld64(tm, wwarp, TM_DK + 64 * wg, f);
          if (!lo) {
            float tq = 0.f;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              float x8[8];
              il_load8(sQ, C, r64, 64 * wg + g * 8, x8);
#pragma unroll
              for (int e = 0; e < 8; ++e) tq = fmaf(x8[e], f[g * 8 + e], tq);
            }
            tqp[wg * C + r64] = tq;
          }
        }
      }
      simt_signal(&sg[SG_P7], tid);
      BSTAMP(13);
      if (wg == 0 && lo && t0 + r64 < L)
        dbeta[t0 + r64] = __float2bfloat16_rn(db1[r64] + db1[C + r64] + db2[r64] + db2[C + r64]);

      // ================= P8: dq / dk epilogue (lanes >= 16: dq_hat row, lanes
      // < 16: dk_hat row; columns split by warpgroup; row dots combined)
      mbar_wait(&mb[MB_K], ph);
      fence_after_sync();
      BSTAMP(14);
      {
        // each thread keeps the bf16 chunks it read and overwrites exactly
        // those (in-place staging)
        float f[64];
        ld64(tm, wwarp, TM_DK + 64 * wg, f);
        uint8_t* tile = lo ? sK : sQ;
        uint4 raw[8];
        float dot = 0.f;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          raw[g] = *reinterpret_cast<const uint4*>(tile + il_off(r64, 64 * wg + g * 8, C));
          float x8[8];
          unpack8(raw[g], x8);
#pragma unroll
          for (int e = 0; e < 8; ++e) dot = fmaf(x8[e], f[g * 8 + e], dot);
        }
        (lo ? sdot : sdotq)[wg * C + r64] = dot;
        grp_sync<256>(BAR_SIMT);
        const float* dd = lo ? sdot : sdotq;
        dot = dd[r64] + dd[C + r64];
        if (!(l2 && (lo ? nk : nq)[r64] >= eps)) dot = 0.f;
        const float inv = (lo ? ss : sr)[r64];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float x8[8];
          unpack8(raw[g], x8);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            x8[e] = l2 ? inv * (f[g * 8 + e] - x8[e] * dot) : f[g * 8 + e];
          il_store8(tile, C, r64, 64 * wg + g * 8, x8);
        }
      }
      if (GATED && warp == 0) {
        // dl/dG of rows lane and 32 + lane (partials of P1-P8), then dg =
        // reverse cumulative sum within the chunk
        auto dGrow = [&](int i, float& DDi) {
          DDi = gD[i] * (ddp[i] + ddp[C + i]);
          const float ct1 = (colT1[i] + colT1[C + i]) + (colT1[2 * C + i] + colT1[3 * C + i]);
          const float ct2 = (colT2[i] + colT2[C + i]) + (colT2[2 * C + i] + colT2[3 * C + i]);
          return (tqp[i] + tqp[C + i]) + (rowT1[i] + rowT1[C + i]) - ct1 +
                 sb[i] * (db2[i] + db2[C + i]) - ct2 - sb[i] * gam[i] * (pkh[i] + pkh[C + i]) -
                 DDi;
        };
        float DD0, DD1;
        const float d0 = dGrow(lane, DD0);
        float d1 = dGrow(32 + lane, DD1);
        const float sDD = warp_sum(DD0 + DD1);
        const float shd = warp_sum(lane < 8 ? hdot[lane] : 0.f);
        if (lane == 31) d1 += sDD + gam[C - 1] * shd;
        float s1 = d1, s0 = d0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y1 = __shfl_down_sync(0xffffffffu, s1, o);
          const float y0 = __shfl_down_sync(0xffffffffu, s0, o);
          if (lane + o < 32) {
            s1 += y1;
            s0 += y0;
          }
        }
        s0 += __shfl_sync(0xffffffffu, s1, 0);  // + all of rows 32..63
        float* dg = a.dg + (size_t)unit * a.L + T0 + t0;
        if (t0 + lane < L) dg[lane] = s0;
        if (t0 + 32 + lane < L) dg[32 + lane] = s1;
      }
      simt_signal(&sg[SG_P8], tid);
      BSTAMP(15);
    }

    // dh0 = dH (orientation [dk][dv]; lane dv = w, columns split): segment 0's
    // (pass 3); pass 1 writes the segment-local dl/dH_start instead
    float* dho = SEG1 ? a.hloc + ((size_t)unit * nseg + seg) * D * D
                 : (seg == 0 && a.dh0) ? a.dh0 + (size_t)unit * D * D : nullptr;
    if (SEG1 && NC > 0) mbar_wait(&mb[MB_DH], (NC - 1) & 1);  // the last chunk's dH update
    if (dho) {
      fence_after_sync();
      float f[64];
      ld64(tm, wwarp, TM_DH + 64 * wg, f);
#pragma unroll
      for (int e = 0; e < 64; ++e) dho[(size_t)(64 * wg + e) * D + w] = f[e];
    }
  }
  cta_sync();
  if (tid == 0) CTA_STAMP(1, gtimer());
  if (warp == 0) tmem_dealloc<512>(tm);
}

// Pass 2 of the segment-parallel backward: the cotangent at each segment's
// end, dl/dH_end(s-1) = dl/dH_start(s) = Psi_s dl/dH_end(s) + dH_loc(s), from
// dl/dH_end(S-1) = dhT (H = S^T, [dk][dv]; Psi from the forward's pass 1 --
// the backward's per-chunk maps are the transposes of the forward's).  A CTA
// scans one 16-column block; fp32.
__global__ void __launch_bounds__(256) seg_scan_bwd_kernel(Args a) {
  extern __shared__ __align__(16) float scan_sm[];
  float* Ps = scan_sm;  // Psi_s, row stride PSI_LD (tc_common.cuh stage_psi)
  float(*Hs)[16] = reinterpret_cast<float(*)[16]>(scan_sm + D * PSI_LD);
  const int unit = blockIdx.x, j0 = blockIdx.y * 16, nseg = a.nseg;
  const int tid = threadIdx.x, i = tid >> 1, jj = (tid & 1) * 8;
  for (int e = tid; e < D * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    Hs[r][cc] = a.dhT ? a.dhT[(size_t)unit * D * D + (size_t)r * D + j0 + cc] : 0.f;
  }
  for (int sg = nseg - 1; sg >= 1; --sg) {
    const float* hl = a.hloc + ((size_t)unit * nseg + sg) * D * D + (size_t)i * D + j0 + jj;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = hl[e];
    stage_psi(Ps, a.psi + ((size_t)unit * nseg + sg) * D * D, tid);
#pragma unroll 8
    for (int r = 0; r < D; ++r) {
      const float pv = Ps[i * PSI_LD + r];  // Psi[i][r]
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(pv, Hs[r][jj + e], acc[e]);
    }
    __syncthreads();
    float* out = a.hseg + ((size_t)unit * nseg + sg - 1) * D * D + (size_t)i * D + j0 + jj;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      Hs[i][jj + e] = acc[e];
      out[e] = acc[e];
    }
  }
}
constexpr int SEG_SCAN_BWD_SMEM = PSI_SMEM;

}  // namespace

int tc_fwd(const Args& a, cudaStream_t s);

int tc_bwd(const Args& a0, cudaStream_t s) {
  static PerDevice attr;
  if (!attr.done()) {
    if (cudaFuncSetAttribute(tc_bwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_bwd_kernel<false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr.mark();
  }
  Args a = a0;
  if (!(a.flags & DELTANET_SAVE_STATES)) {
    // recompute the chunk states (and the segment transitions) with the
    // forward kernel (no O store)
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
  const int nseg = tc_seg_setup(a);
  if (a.flags & DELTANET_GATED) {  // one CTA per unit (tc_fwd_segments: 1 when gated)
    if (nseg > 1 || !a.g || !a.dg) return DELTANET_ERR_INVALID_ARG;
    tc_bwd_kernel<false, true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  if (nseg <= 1) {
    tc_bwd_kernel<false><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  // segment-parallel backward, with the forward's Psi
  tc_bwd_kernel<true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
  {
    static PerDevice sattr;
    if (!sattr.done()) {
      if (cudaFuncSetAttribute(seg_scan_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               SEG_SCAN_BWD_SMEM) != cudaSuccess)
        return DELTANET_ERR_CUDA;
      sattr.mark();
    }
  }
  seg_scan_bwd_kernel<<<dim3(BH, D / 16), 256, SEG_SCAN_BWD_SMEM, s>>>(a);
  tc_bwd_kernel<false><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

// Context parallelism: the local cotangent chain of this call's sequence from
// dl/dH_end = 0 (pass 1 with one segment per unit, or S segments composed
// with the forward's segment transitions); needs the forward's per-chunk
// records (and segment Psi) in the workspace (deltanet_fwd with SAVE_STATES)
int tc_bwd_transition(const Args& a0, float* dhloc, cudaStream_t s) {
  Args a = a0;
  const int BH = a.B * a.H;
  CUtensorMap mQ, mK, mV, mDO, mDQ, mDK, mDV;
  if (!make_il_map(&mQ, a.q, BH, a.L, D, C) || !make_il_map(&mK, a.k, BH, a.L, D, C) ||
      !make_il_map(&mV, a.v, BH, a.L, D, C) || !make_il_map(&mDO, a.dO, BH, a.L, D, C) ||
      !make_il_map(&mDQ, a.q, BH, a.L, D, C) || !make_il_map(&mDK, a.k, BH, a.L, D, C) ||
      !make_il_map(&mDV, a.v, BH, a.L, D, C))
    return DELTANET_ERR_CUDA;
  static PerDevice attr;
  if (!attr.done()) {
    if (cudaFuncSetAttribute(tc_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr.mark();
  }
  const int nseg = tc_seg_setup(a);
  if (nseg <= 1) {
    a.nseg = 1;
    a.hloc = dhloc;
    tc_bwd_kernel<true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  tc_bwd_kernel<true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mDO, mDQ, mDK, mDV, a);
  if (cudaGetLastError() != cudaSuccess) return DELTANET_ERR_CUDA;
  return cp_compose_bwd(a, dhloc, s);
}

}  // namespace dn

#ifdef DN_TIMING
extern "C" int dn_timing_set_bwd(long long* buf) {
  return cudaMemcpyToSymbol(dn::dn_tim_bwd, &buf, sizeof(buf)) != cudaSuccess;
}
#endif
