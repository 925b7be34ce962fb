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
// Algebra of the folded normalisation: DESIGN.md §4.1.
//
// Warp specialisation: warps 0-7 ("prep") run the
// state-independent part of chunk t+1 (row norms and L from G_kk, the
// substitution, T', T'') while warps 8-11 ("state") run chunk t's chain
// conversions (W^T, A from G_qk, Z, H^T) and the output epilogue.  Warp 12
// issues the prep MMAs (the two Gram halves, W, U) and the V loads; warp 13
// issues the chain MMAs, the O store, the record copies and the next Q/K
// loads, so no compute warp ever stalls on an MMA issue queue.  Q, K, V and
// O are SW (SWIZZLE_128B) tiles, moved by TMA boxes of 128 B rows
// (tc_common.cuh sw_off).  Q, A and the U accumulator are double-buffered by
// chunk parity, K has three slots; mbarriers hand every buffer over
// (full/empty, *_done/*_free/*_ready).
#include <cudaTypedefs.h>
#include <stdio.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

using namespace tc;

constexpr int C = 64, DK = 128, DV = 128, NT = 448;  // 8 prep + 4 state + 2 MMA warps
constexpr int NP = 256;  // prep threads
constexpr int LS = 68;  // row stride (floats) of the fp32 substitution buffer

// dynamic shared memory map (bytes)
constexpr int TILE = C * DK * 2;                 // 16 KB chunk tile
constexpr int NQB = 2;                           // Q slots (chunk c in slot c % NQB)
constexpr int OFF_Q = 0;                         // Q[NQB] IL R=64 x 128
constexpr int OFF_K = OFF_Q + NQB * TILE;        // K[2]  IL R=64 x 128
constexpr int OFF_V = OFF_K + 2 * TILE;          // V     IL R=64 x 128
constexpr int OFF_T = OFF_V + TILE;              // T'    IL R=64 x 64
constexpr int OFF_TU = OFF_T + C * C * 2;        // T''   IL R=64 x 64
constexpr int OFF_A = OFF_TU + C * C * 2;        // A[2]  IL R=64 x 64
constexpr int OFF_W = OFF_A + 2 * C * C * 2;     // W^T[2] IL R=128 x 64 (outside SEG1: W^T | K slot 2)
constexpr int OFF_H = OFF_W + 2 * DK * C * 2;    // H^T   IL R=128 x 128
constexpr int OFF_Z = OFF_H + DV * DK * 2;       // Z^T   IL R=128 x 64  | O staging
constexpr int OFF_L = OFF_Z + DV * C * 2;        // L -> X fp32 [64][LS]
// per-chunk vectors [2][beta, s, 1/s, G, gamma, D][64] (G, gamma, D: gated only)
constexpr int NVEC = 6;
constexpr int OFF_VEC = OFF_L + C * LS * 4 + 2 * 128 * 4;  // (LX, partial norms) | vectors
constexpr int SMEM_BYTES = OFF_VEC + 2 * NVEC * C * 4;
static_assert(SMEM_BYTES <= 232448 - 1024, "shared memory budget");
static_assert(REC_Z == C * C * 2 && REC_N == C * C * 2 + DV * C * 2 &&
                  REC_A == REC_N + 2 * C * 4 && REC_BYTES == REC_A + C * C * 2, "record");

// Prep record of the segmented forward: pass 1 stores, per
// chunk, the bf16 IL images of T' and T'' and the fp32 row scales s, 1/s;
// pass 3 loads them with one bulk copy each instead of redoing the Gram
// conversion, the substitution and the T writes (bit-identical operands).
constexpr int PREC_T = 0, PREC_S = 2 * C * C * 2, PREC_BYTES = PREC_S + 2 * C * 4;

// TMEM column map (512 columns)
constexpr uint32_t LO16 = 16u << 16;
constexpr uint32_t TM_H = 0;                     // H^T  M=128, 128 cols (S)
constexpr uint32_t TM_O = 128;                   // O    M=64,  128 cols (S)
constexpr uint32_t TM_U1 = 256;                  // U^T  buffer 1, M=128, 64 cols
constexpr uint32_t TM_G = 320;                   // G_qk lane+0 | G_kk lane+16 (P)
constexpr uint32_t TM_W = 384;                   // W^T  M=128, 64 cols (P)
constexpr uint32_t TM_U0 = 448;                  // U^T  buffer 0
__device__ __forceinline__ uint32_t tm_u(int b) { return b ? TM_U1 : TM_U0; }

enum { BAR_P = 1, BAR_S = 2 };  // named barriers of the two warpgroups

// 32 fp32 columns [col, col+32) of this warp's 32 TMEM lanes
__device__ __forceinline__ void ld32_cols(uint32_t tm, int warp, uint32_t col, float (&f)[32]) {
  uint32_t r[2][16];
  tmem_ld16(taddr(tm, warp * 32, col), r[0]);
  tmem_ld16(taddr(tm, warp * 32, col + 16), r[1]);
  tmem_ld_wait();
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    f[e] = __uint_as_float(r[0][e]);
    f[16 + e] = __uint_as_float(r[1][e]);
  }
}

#ifdef DN_DEBUG
// Test-only intermediate dumps (tests/test_tc_debug.py builds with -DDN_DEBUG).
__device__ float* dn_dbg = nullptr;
__device__ int dn_dbg_chunk = 0;
enum { D_L = 0, D_X = 4096, D_GQK = 8192, D_W = 12288, D_U = 20480, D_UP = 28672,
       D_O = 36864, D_H = 45056, D_S = 61440, D_R = 61504, D_B = 61568 };
__device__ void dbg_smem(float* dst, const float* src, int rows, int cols, int stride, int w) {
  for (int e = w; e < rows * cols; e += 128) {
    const int i = e / cols, j = e % cols;
    // the substitution buffer keeps scratch above the diagonal
    dst[e] = (stride == LS && j > i && rows == cols) ? 0.f : src[i * stride + j];
  }
}
__device__ void dbg_tmem(float* dst, uint32_t tm, uint32_t col, int ncols, int M, int w) {
  const int warp = w >> 5, lane = w & 31;
  for (int c0 = 0; c0 < ncols; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr(tm, warp * 32, col + c0), r);
    tmem_ld_wait();
    const int row = M == 128 ? w : (lane < 16 ? warp * 16 + lane : -1);
    if (row >= 0)
      for (int j = 0; j < 16; ++j) dst[row * ncols + c0 + j] = __uint_as_float(r[j]);
  }
}
#define DBG_ON (dn_dbg != nullptr && blockIdx.x == 0 && c == dn_dbg_chunk)
#define DBG(stmt) do { if (DBG_ON) { stmt; } } while (0)
#else
#define DBG(stmt) do { } while (0)
#endif

#ifdef DN_TIMING
// Test-only phase timestamps of CTA 0 (tests/test_tc_timing.py, -DDN_TIMING).
__device__ long long* dn_tim = nullptr;
#define TSTAMP(slot)                                                       \
  do {                                                                     \
    if (dn_tim != nullptr && blockIdx.x == 0 && (tid == 0 || tid == NP))   \
      dn_tim[(size_t)c * 32 + (slot)] = clock64();                         \
  } while (0)
#define TSTAMP_PTR(slot) \
  ((dn_tim != nullptr && blockIdx.x == 0) ? dn_tim + (size_t)c * 32 + (slot) : nullptr)
#define TSTAMP1(slot)                                                      \
  do {                                                                     \
    if (dn_tim != nullptr && blockIdx.x == 0) dn_tim[(size_t)c * 32 + (slot)] = clock64(); \
  } while (0)
// stamp filed under another chunk (load issue times, by target chunk)
#define TSTAMPC(cc, slot)                                                  \
  do {                                                                     \
    if (dn_tim != nullptr && blockIdx.x == 0 && (cc) < NC) dn_tim[(size_t)(cc) * 32 + (slot)] = clock64(); \
  } while (0)
#else
#define TSTAMPC(cc, slot) do { } while (0)
#define TSTAMP1(slot) do { } while (0)
#define TSTAMP(slot) do { } while (0)
#define TSTAMP_PTR(slot) nullptr
#endif

// SEG1 = pass 1 of the segment-parallel forward: from a zero
// state, the segment's end state H_loc and its transition
// Psi = prod_c (I - W_c^T K_hat_c) (H^T_end = H^T_start Psi + H^T_loc); no O.
// GATED = Gated DeltaNet (R23, §4.9): per chunk, with the in-chunk
// cumulative log-gate G, gamma = e^G, Gamma(i,j) = e^{G_i - G_j},
// D_j = e^{G_63 - G_j}: A and L carry Gamma, T' carries gamma
// (W = X diag(beta gamma) K_hat), Q rows are scaled by gamma in place before
// O = Q H, H is rescaled by gamma_63 in TMEM, and the state update takes
// Z_h = diag(s D) U' from TMEM (bf16 pairs) while O takes Z = diag(s) U'.
// PRE = pass 3 of the segmented forward with pass 1's prep records (T', T'',
// s, 1/s per chunk): the prep warps only load them.
template <bool SEG1, bool GATED = false, bool COMP = false, bool PRE = false>
__global__ void __launch_bounds__(NT, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                  const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mO,
                  Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // mbarriers (DESIGN.md §4.1 "fwd pipeline")
  // Q double-buffered by chunk parity; K in NKB slots (3 outside SEG1: the
  // third slot is W^T's second buffer, W^T then being single-buffered), so
  // K of chunk c+3 loads when chunk c's chain ends and Q of chunk c+2 as
  // soon as O = Q H has read Q (q_done): the next Grams never wait on HBM
  constexpr int NKB = SEG1 ? 2 : 3;
  __shared__ uint64_t q_full[NQB], k_full[3], v_full[2], bar_full[2], bar_empty[2], q_done;
  // Gram: gk_done / gk_free for K K^T (lanes 16-31 of each quadrant), g_done /
  // g_free for Q K^T (lanes 0-15); the two halves are issued and released apart
  __shared__ uint64_t gk_done, gk_free, g_done, g_free, t_ready, w_done, wu_done, w_free;  // prep side
  __shared__ uint64_t pr_full;  // pass 3: the chunk's prep record has landed
  __shared__ uint64_t up_done, z_free, z_ready, ho_done, h_ready, st_free;  // state side
  // q_read: the state warpgroup's norm pass has finished reading Q[b] (the
  // chain warp may then overwrite the slot with Q of chunk c+2; ADVICE r1:
  // q_done alone does not order those generic-proxy reads before the TMA)
  __shared__ uint64_t q_read;
  // u_read: all 128 state threads have read U' of the chunk out of TMEM (the
  // ungated U' record is formed after z_ready); the U buffer is released
  // (bar_empty) only after it
  __shared__ uint64_t u_read;
  __shared__ uint32_t tslot;

  // SW tiles need 1024 B alignment (the swizzle acts on absolute address bits)
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int w = tid & 127;            // thread index inside a 128-thread group
  const int wwarp = w >> 5;           // TMEM lane quadrant of this warp
  const int half = (tid >> 7) & 1;    // prep: which column half this thread handles
  // segment of this CTA: chunks [cbase, cbase + NC) of unit; local chunk c is
  // global chunk cbase + c (token T0 + c*C); L counts tokens from T0
  const int nseg = a.nseg > 1 ? a.nseg : 1;
  const int unit = blockIdx.x / nseg, seg = blockIdx.x % nseg;
  const int cbase = nseg > 1 ? seg * a.seg_len : 0;
  const int NC = nseg > 1 ? min(a.seg_len, a.NC - cbase) : a.NC;
  const int T0 = cbase * C;
  const int L = a.L - T0;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;

  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&v_full[b], 1);
      mbar_init(&bar_full[b], 1);
      mbar_init(&bar_empty[b], 1);
    }
    for (int b = 0; b < 3; ++b) mbar_init(&k_full[b], 1);
    for (int b = 0; b < NQB; ++b) mbar_init(&q_full[b], 1);
    mbar_init(&q_done, 1);
    mbar_init(&g_done, 1);
    mbar_init(&gk_done, 1);
    mbar_init(&gk_free, 1);
    mbar_init(&pr_full, 1);
    mbar_init(&g_free, 1);
    mbar_init(&t_ready, 1);
    mbar_init(&w_done, 1);
    mbar_init(&wu_done, 1);
    mbar_init(&w_free, 1);
    mbar_init(&up_done, 1);
    mbar_init(&z_free, 1);
    mbar_init(&z_ready, 1);
    mbar_init(&ho_done, 1);
    mbar_init(&h_ready, 1);
    mbar_init(&st_free, 1);
    mbar_init(&q_read, 1);
    mbar_init(&u_read, 128);
    mbar_fence_init();
    prefetch_tmap(&mQ);
    prefetch_tmap(&mK);
    prefetch_tmap(&mV);
    prefetch_tmap(&mO);
  }
  cta_sync();
  const uint32_t tm = tslot;
  auto sQ = [&](int b) { return smem + OFF_Q + b * TILE; };
  // K slot b (0..NKB-1); slot 2 is the memory of W^T[1]
  auto sK = [&](int b) { return b < 2 ? smem + OFF_K + b * TILE : smem + OFF_W + DK * C * 2; };
  auto sA = [&](int b) { return smem + OFF_A + b * C * C * 2; };
  auto sW = [&](int) { return smem + OFF_W + (SEG1 ? 1 : 0) * DK * C * 2; };
  static_assert(TILE == DK * C * 2, "K slot 2 spans W^T[1]");
  auto vec = [&](int b) { return reinterpret_cast<float*>(smem + OFF_VEC) + b * NVEC * C; };
  uint8_t* sV = smem + OFF_V;
  uint8_t* sT = smem + OFF_T;
  uint8_t* sTu = smem + OFF_TU;
  uint8_t* sH = smem + OFF_H;
  uint8_t* sZ = smem + OFF_Z;
  // pass 1 with prep records also writes the X and ||k|| records (pass 3 then
  // takes T', T'' and s from its prep record and writes neither)
  uint8_t* recs = ((!SEG1 || a.prec) && (a.flags & DELTANET_SAVE_STATES))
                      ? reinterpret_cast<uint8_t*>(a.scratch) +
                            ((size_t)unit * a.NC + cbase) * REC_BYTES
                      : nullptr;
  uint8_t* const prec =
      a.prec ? a.prec + ((size_t)unit * a.NC + cbase) * PREC_BYTES : nullptr;
  constexpr bool pre = PRE;  // pass 3 from prep records
  // compensated mode: A = tril(Q K^T) is formed by the prep warps from a
  // joint Gram commit (its state warpgroup carries the rounding chains and is
  // the busier side there)
  constexpr bool APREP = COMP && !SEG1;
  // SEG1: the Psi image [dk][dk] bf16 (IL R=128) over A[0], A[1], W[0]; W in W[1]
  uint8_t* sPsi = smem + OFF_A;
  static_assert(OFF_W == OFF_A + 2 * C * C * 2 && 2 * C * C * 2 + DK * C * 2 == DK * DK * 2,
                "Psi image spans A[0..1] and W[0]");
  uint8_t* sO = sZ;
  float* LX = reinterpret_cast<float*>(smem + OFF_L);

  if (warp < 8) {
    // =====================================================================
    // Prep warps 0-7 (256 threads): prep of chunk c (state independent).
    // Every row-wise phase is split in two column halves (`half`), so each
    // SM sub-partition runs two prep warps and hides the other's latency.
    // =====================================================================
    const __nv_bfloat16* beta = (const __nv_bfloat16*)a.beta + (size_t)unit * a.L + T0;
    // beta is prefetched into a register one chunk ahead (global latency)
    uint16_t bnext = (w < C && w < L) ? ldg_u16(beta + w) : (uint16_t)0;  // raw bf16 bits
    // gated: own log-gate and the warp-0 counterpart (lane), one chunk ahead
    const float* gsrc = GATED ? a.g + (size_t)unit * a.L + T0 : nullptr;
    float gnext = 0.f, g0next = 0.f;
    if (GATED) {
      gnext = (w < C && w < L) ? gsrc[w] : 0.f;
      g0next = (lane < L) ? gsrc[lane] : 0.f;
    }
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const int b = c & 1, t0 = c * C;
      float* vb = vec(b);  // beta, s, -, G, gamma, D of this chunk
      const float bval = bf16_bits(bnext);
      bnext = (w < C && t0 + C + w < L) ? ldg_u16(beta + t0 + C + w) : (uint16_t)0;
      float gval = 0.f, g0val = 0.f;
      if (GATED) {
        gval = gnext;
        g0val = g0next;
        gnext = (w < C && t0 + C + w < L) ? gsrc[t0 + C + w] : 0.f;
        g0next = (t0 + C + lane < L) ? gsrc[t0 + C + lane] : 0.f;
      }
      TSTAMP(0);
      if (c >= 2) mbar_wait(&bar_empty[b], ((c >> 1) - 1) & 1);  // chain c-2 released b
      TSTAMP(1);
      if (half == 0 && w < C) vb[w] = bval;
      if (pre) {
        // pass 3: T', T'' and s, 1/s from pass 1's prep record (T' / T'' of
        // chunk c-1 are free once its W/U products completed)
        if (tid == 0) {
          if (c >= 1) mbar_wait(&wu_done, (c - 1) & 1);
          mbar_expect_tx(&pr_full, 2 * C * C * 2 + 2 * C * 4);
          bulk_load(sT, prec + (size_t)c * PREC_BYTES + PREC_T, 2 * C * C * 2, &pr_full);
          bulk_load(vb + C, prec + (size_t)c * PREC_BYTES + PREC_S, 2 * C * 4, &pr_full);
        }
        mbar_wait(&pr_full, c & 1);
        grp_sync<NP>(BAR_P);  // beta written by every thread that holds one
        if (tid == 0) mbar_arrive(&t_ready);
        continue;
      }
      if (GATED && half == 0 && w < C) {
        // G_w = sum_{j <= w} g_j: warp inclusive scan + warp 0's total
        float x = gval, t0s = g0val;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
          t0s += __shfl_xor_sync(0xffffffffu, t0s, o);
        }
        vb[3 * C + w] = x + (w >= 32 ? t0s : 0.f);
      }
      TSTAMP(2);
      // The Gram pair is split (K K^T first, Q K^T later): L and the
      // substitution need only K K^T; A = tril(Q K^T) is formed by the state
      // warpgroup just before the chain needs it.
      mbar_wait(&gk_done, c & 1);
      fence_after_sync();
      TSTAMP(3);
      const int i = wwarp * 16 + (lane & 15), h = 32 * half;
      // lane pair (lo: G_qk row i, hi: G_kk row i) trades halves, so both
      // lanes write 16 columns of L, with no divergence
      const bool lo = lane < 16;
      const int c0 = h + (lo ? 0 : 16);
      // gated: Gamma(i, j) = e^{G_i - G_j} for the 16 columns [c0, c0+16) of this lane
      // (masked by index, not clamped: with g > 0 allowed, G_i - G_j may be
      // positive for j <= i; j > i is masked by the callers)
      auto gamma16 = [&](float (&gam16)[16]) {
        const float Gi = vb[3 * C + i];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 g4 = *reinterpret_cast<const float4*>(vb + 3 * C + c0 + 4 * q);
          const int j = c0 + 4 * q;
          gam16[4 * q + 0] = __expf(j + 0 <= i ? Gi - g4.x : 0.f);
          gam16[4 * q + 1] = __expf(j + 1 <= i ? Gi - g4.y : 0.f);
          gam16[4 * q + 2] = __expf(j + 2 <= i ? Gi - g4.z : 0.f);
          gam16[4 * q + 3] = __expf(j + 3 <= i ? Gi - g4.w : 0.f);
        }
      };
      {
        // S2a: this half's 32 columns; lanes >= 16 hold G_kk rows (lanes < 16:
        // the G_qk half, possibly still in flight -- not used here)
        float f[32];
        ld32_cols(tm, wwarp, TM_G + 32 * half, f);
        // s_i = 1/max(||k_i||, eps) from the Gram diagonal (fp32 sum of exact
        // bf16 products; R9).  r (for q) is computed by the state warpgroup.
        if (!lo && (i >> 5) == half) {
          // d = f[i - h] by a 5-level select tree (no dynamic register
          // indexing, no 32-step dependent chain)
          const int k = i - h;
          float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
          for (int e = 0; e < 16; ++e) t16[e] = (k & 16) ? f[16 + e] : f[e];
#pragma unroll
          for (int e = 0; e < 8; ++e) t8[e] = (k & 8) ? t16[8 + e] : t16[e];
#pragma unroll
          for (int e = 0; e < 4; ++e) t4[e] = (k & 4) ? t8[4 + e] : t8[e];
#pragma unroll
          for (int e = 0; e < 2; ++e) t2[e] = (k & 2) ? t4[2 + e] : t4[e];
          const float d = (k & 1) ? t2[1] : t2[0];
          const float nrm = sqrtf(d);
          float inv = l2 ? 1.f / fmaxf(nrm, a.eps) : 1.f;
          if (t0 + i >= L) inv = 0.f;  // padded token: exact zero contribution
          vb[C + i] = inv;
          vb[2 * C + i] = l2 ? fmaxf(nrm, a.eps) : 1.f;  // 1 / s (compensated rounding of Z)
          // ||k_i|| for the backward's record (it then needs no norm pass)
          if (recs) reinterpret_cast<float*>(recs + (size_t)c * REC_BYTES + REC_N)[i] = nrm;
        }
        TSTAMP(21);
        grp_sync<NP>(BAR_P);  // beta, s (and G) visible
        TSTAMP(22);
        if (GATED && half == 0 && w < C) {  // read after later syncs (T', state WG)
          const float Gw = vb[3 * C + w];
          vb[4 * C + w] = __expf(Gw);
          vb[5 * C + w] = __expf(vb[3 * C + C - 1] - Gw);
        }
        // lo lanes take G_kk columns [h, h+16) from their hi partner
        float x[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __shfl_xor_sync(0xffffffffu, f[e], 16);
        float gam16[16];
        if (GATED) gamma16(gam16);
        {  // L = beta_i s_i s_j (k_i . k_j), j < i
          const float bi = vb[i] * vb[C + i];
          float4 s4[4];  // all loads first: no smem aliasing stalls
#pragma unroll
          for (int q = 0; q < 4; ++q) s4[q] = *reinterpret_cast<const float4*>(vb + C + c0 + 4 * q);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = c0 + 4 * q;
            float kk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              kk[e] = lo ? x[4 * q + e] : f[16 + 4 * q + e];
              if (GATED) kk[e] *= gam16[4 * q + e];
            }
            float4 v;
            v.x = (j + 0 < i) ? bi * s4[q].x * kk[0] : 0.f;
            v.y = (j + 1 < i) ? bi * s4[q].y * kk[1] : 0.f;
            v.z = (j + 2 < i) ? bi * s4[q].z * kk[2] : 0.f;
            v.w = (j + 3 < i) ? bi * s4[q].w * kk[3] : 0.f;
            *reinterpret_cast<float4*>(LX + i * LS + j) = v;
          }
        }
        if (APREP) {  // A = tril(Q K^T) (raw, inclusive, R4; gated: Gamma . A) and its record
          float xa[16];  // hi lanes: G_qk columns [h+16, h+32) from the lo partner
#pragma unroll
          for (int e = 0; e < 16; ++e) xa[e] = __shfl_xor_sync(0xffffffffu, f[16 + e], 16);
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            float a8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float qk = lo ? f[g * 8 + e] : xa[g * 8 + e];
              if (GATED) qk *= gam16[g * 8 + e];
              a8[e] = (c0 + g * 8 + e <= i) ? qk : 0.f;
            }
            il_store8(sA(b), C, i, c0 + g * 8, a8);
            if (recs) il_store8(recs + (size_t)c * REC_BYTES + REC_A, C, i, c0 + g * 8, a8);
          }
        }
      }
      TSTAMP(23);
      fence_before_sync();
      grp_sync<NP>(BAR_P);
      DBG(dbg_smem(dn_dbg + D_L, LX, C, C, LS, w); dbg_smem(dn_dbg + D_S, vb + C, 1, C, C, w);
          dbg_smem(dn_dbg + D_B, vb, 1, C, C, w); fence_before_sync(); grp_sync<NP>(BAR_P));
      if (tid == 0) mbar_arrive(&gk_free);  // G_kk may be overwritten (next chunk's K K^T)
      TSTAMP(4);
      ut_inverse_inplace<LS, NP>(LX, tid, BAR_P, TSTAMP_PTR(10));
      TSTAMP(5);
      DBG(dbg_smem(dn_dbg + D_X, LX, C, C, LS, w));
      TSTAMP(9);
      {
        // T'[i][j] = X[i][j] beta_j s_j, T''[i][j] = X[i][j] beta_j  (j <= i).
        // (T' / T'' of chunk c-1 are free once its W/U products completed.)
        // Lanes map to consecutive rows (conflict-free IL stores); each thread
        // handles one 16-column quarter of its row.
        if (c >= 1) mbar_wait(&wu_done, (c - 1) & 1);
        TSTAMP(15);
        const int i = tid & 63, j0 = (tid >> 6) * 16;
        uint4 xrec[2];  // the X record, stored once T is handed over
        uint4 trec[2], turec[2];  // SEG1 with prep records: T', T'' segments
        float4 x4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x4[q] = *reinterpret_cast<const float4*>(LX + i * LS + j0 + 4 * q);
        // beta_j, s_j (and gamma_j) of the 16 columns: vector broadcast loads
        float4 b4[4], s4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          b4[q] = *reinterpret_cast<const float4*>(vb + j0 + 4 * q);
          s4[q] = *reinterpret_cast<const float4*>(vb + C + j0 + 4 * q);
          if (GATED) {
            const float4 g4 = *reinterpret_cast<const float4*>(vb + 4 * C + j0 + 4 * q);
            s4[q].x *= g4.x; s4[q].y *= g4.y; s4[q].z *= g4.z; s4[q].w *= g4.w;
          }
        }
        auto el = [](const float4& v, int r) { return r == 0 ? v.x : r == 1 ? v.y : r == 2 ? v.z : v.w; };
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float x[8], y[8], xs[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = j0 + g * 8 + e, q = 2 * g + e / 4, r = e % 4;
            const float xm = (j <= i) ? el(x4[q], r) : 0.f;
            xs[e] = xm;
            y[e] = xm * el(b4[q], r);
            x[e] = y[e] * el(s4[q], r);  // gated: W = X diag(beta gamma) K_hat
          }
          il_store8(sT, C, i, j0 + g * 8, x);
          il_store8(sTu, C, i, j0 + g * 8, y);
          if (SEG1) {
            trec[g] = make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]),
                                 pack_bf16(x[6], x[7]));
            turec[g] = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]),
                                  pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
          }
          xrec[g].x = pack_bf16(xs[0], xs[1]);
          xrec[g].y = pack_bf16(xs[2], xs[3]);
          xrec[g].z = pack_bf16(xs[4], xs[5]);
          xrec[g].w = pack_bf16(xs[6], xs[7]);
        }
        fence_proxy_async();
        grp_sync<NP>(BAR_P);
        TSTAMP(31);
        if (tid == 0) mbar_arrive(&t_ready);
        if (SEG1 && prec) {  // pass 1: the prep record for pass 3 (T', T'' images; s, 1/s)
          uint8_t* pr = prec + (size_t)c * PREC_BYTES;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            *reinterpret_cast<uint4*>(pr + PREC_T + il_off(i, j0 + g * 8, C)) = trec[g];
            *reinterpret_cast<uint4*>(pr + PREC_T + C * C * 2 + il_off(i, j0 + g * 8, C)) = turec[g];
          }
          if (tid < 2 * C) reinterpret_cast<float*>(pr + PREC_S)[tid] = vb[C + tid];
        }
        if (recs) {  // the X record from registers (IL image, 16 B per row), off the hand-over
#pragma unroll
          for (int g = 0; g < 2; ++g)
            *reinterpret_cast<uint4*>(recs + (size_t)c * REC_BYTES + REC_X +
                                      il_off(i, j0 + g * 8, C)) = xrec[g];
        }
      }
      TSTAMP(6);
      TSTAMP(7);
      TSTAMP(8);
    }
  } else if (warp < 12) {
    // =====================================================================
    // Warpgroup S (warps 8-11): state chain conversions + output epilogue
    // =====================================================================
    float* qn2 = LX + C * LS;  // [2][64] partial ||q||^2 (region after LX)
    constexpr bool comp = COMP;  // DELTANET_COMPENSATED (R19): its own instantiation
    {  // initial state: H^T row dv = w (TMEM lane w) from h0 [dk][dv] (segment
      // starts after the first: the scanned state; SEG1: zero)
      const float* h0 = SEG1 ? nullptr
                        : (seg > 0 && a.hseg) ? a.hseg + ((size_t)unit * nseg + seg) * DK * DV
                        : a.h0 ? a.h0 + (size_t)unit * DK * DV : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < DK; c0 += 16) {
        uint32_t r[16];
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          f[j] = h0 ? h0[(size_t)(c0 + j) * DV + w] : 0.f;
          r[j] = __float_as_uint(f[j]);
        }
        tmem_st16(taddr(tm, wwarp * 32, TM_H + c0), r);
        il_store8(sH, DV, w, c0, f);
        il_store8(sH, DV, w, c0 + 8, f + 8);
      }
      if (SEG1) {  // Psi = I: TMEM (fp32, lane = row a = w) and the bf16 image
#pragma unroll 1
        for (int c0 = 0; c0 < DK; c0 += 16) {
          uint32_t r[16];
          float f[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            f[j] = (c0 + j == w) ? 1.f : 0.f;
            r[j] = __float_as_uint(f[j]);
          }
          tmem_st16(taddr(tm, wwarp * 32, TM_O + c0), r);
          il_store8(sPsi, DK, w, c0, f);
          il_store8(sPsi, DK, w, c0 + 8, f + 8);
        }
      }
      tmem_st_wait();
    }
    fence_proxy_async();
    fence_before_sync();
    wg_sync(BAR_S);
    if (w == 0) mbar_arrive(&h_ready);
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const int b = c & 1;
      const float* vb = vec(b);
      TSTAMP(16);
      // W^T of this chunk (lane = dk) -> bf16 IL tile sW(b) (row dk, cols =
      // tokens); the prep warps only hand over T (t_ready), so the W/U
      // products and this conversion are off the prep's critical path
      mbar_wait(&w_done, c & 1);
      fence_after_sync();
      DBG(mbar_wait(&wu_done, c & 1); fence_after_sync();
          dbg_tmem(dn_dbg + D_W, tm, TM_W, C, 128, w);
          dbg_tmem(dn_dbg + D_U, tm, tm_u(b), C, 128, w));
      {
        float f[64];
        ld64(tm, wwarp, TM_W, f);
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sW(b), DK, w, g * 8, f + g * 8);
      }
      // r_i = 1/max(||q_i||, eps) for this lane's output row (R9): partial sums
      // of squares over column halves (thread w: row w & 63, half w >> 6).
      // Gated: the same pass scales the raw Q rows by gamma in place (O = Q H
      // then carries diag(gamma)), so it runs before bar_full releases Q.
      float ri = 0.f;
      auto norms = [&]() {
        const int row = w & 63, hh = w >> 6;
        float x[DK / 2];
#pragma unroll
        for (int g = 0; g < DK / 16; ++g) sw_load8(sQ(c % NQB), C, row, DK / 2 * hh + g * 8, x + 8 * g);
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int e = 0; e < DK / 2; e += 2) {
          acc0 = fmaf(x[e], x[e], acc0);
          acc1 = fmaf(x[e + 1], x[e + 1], acc1);
        }
        qn2[hh * C + row] = acc0 + acc1;
        if (GATED) {
          const float gr = vb[4 * C + row];
#pragma unroll
          for (int e = 0; e < DK / 2; ++e) x[e] *= gr;
#pragma unroll
          for (int g = 0; g < DK / 16; ++g) sw_store8(sQ(c % NQB), C, row, DK / 2 * hh + g * 8, x + 8 * g);
        }
        wg_sync(BAR_S);
        if (w == 0) mbar_arrive(&q_read);  // every thread's reads of sQ(b) are done
        const int i = wwarp * 16 + (lane & 15);
        const float nrm = sqrtf(qn2[i] + qn2[C + i]);
        ri = l2 ? 1.f / fmaxf(nrm, a.eps) : 1.f;
        if (c * C + i >= L) ri = 0.f;
        if (recs && lane < 16)  // ||q_i|| for the backward's record
          reinterpret_cast<float*>(recs + (size_t)c * REC_BYTES + REC_N)[C + i] = nrm;
        DBG(if (lane < 16) dn_dbg[D_R + i] = ri);
      };
      if (GATED) norms();
      fence_proxy_async();
      fence_before_sync();
      wg_sync(BAR_S);
      if (w == 0) {
        // U^T[b] complete before the chain uses it; waited before w_free is
        // released so that wu_done cannot run a phase ahead of this wait
        // (SEG1: TM_W then holds T1 = Psi W^T until the Psi update: w_free
        // comes after ho_done)
        mbar_wait(&wu_done, c & 1);
        if (!SEG1) mbar_arrive(&w_free);
        mbar_arrive(&bar_full[b]);
      }
      if (!SEG1 && !GATED) norms();
      if (!SEG1 && !APREP) {
        // A = tril(Q K^T), raw (inclusive, R4; gated: Gamma . A) -> sA(b), the
        // operand of this chunk's O += A Z, and the backward's A record.  Done
        // here (the state warpgroup waits for the U' product anyway) rather than
        // by the prep warps, whose chunk loop is the forward's critical path.
        // G_qk row i sits in lanes < 16 of each quadrant; lo lanes write columns
        // [0, 32) of it, their hi partners [32, 64).
        mbar_wait(&g_done, c & 1);
        fence_after_sync();
        DBG(dbg_tmem(dn_dbg + D_GQK, tm, TM_G, C, 64, w));
        float f[64];
        ld64(tm, wwarp, TM_G, f);
        const bool lo = lane < 16;
        const int i = wwarp * 16 + (lane & 15), c0 = lo ? 0 : 32;
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __shfl_xor_sync(0xffffffffu, f[32 + e], 16);
        const float Gi = GATED ? vb[3 * C + i] : 0.f;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float a8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = c0 + g * 8 + e;
            float qk = lo ? f[g * 8 + e] : x[g * 8 + e];
            // gated: Gamma(i, j) = e^{G_i - G_j}, masked by index (not clamped:
            // g > 0 is allowed)
            if (GATED) qk *= __expf(j <= i ? Gi - vb[3 * C + j] : 0.f);
            a8[e] = (j <= i) ? qk : 0.f;
          }
          il_store8(sA(b), C, i, c0 + g * 8, a8);
          if (recs) il_store8(recs + (size_t)c * REC_BYTES + REC_A, C, i, c0 + g * 8, a8);
        }
      }
      mbar_wait(&up_done, c & 1);
      mbar_wait(&z_free, c & 1);
      fence_after_sync();
      TSTAMP(17);
      DBG(dbg_tmem(dn_dbg + D_UP, tm, tm_u(b), C, 128, w));
      if (!comp) {  // Z^T[dv][t] = U'^T[dv][t] * s_t -> bf16 IL tile (row dv)
        float f[64];
        ld64(tm, wwarp, tm_u(b), f);
#pragma unroll
        for (int t = 0; t < 64; ++t) f[t] *= vb[C + t];
#pragma unroll
        for (int g = 0; g < 8; ++g) il_store8(sZ, DV, w, g * 8, f + g * 8);
        if (GATED) {  // Z_h^T = Z^T diag(D) as bf16 pairs over U's first 32 TMEM columns
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t r[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int t = 32 * h2 + 2 * j;
              r[j] = pack_bf16(f[t] * vb[5 * C + t], f[t + 1] * vb[5 * C + t + 1]);
            }
            tmem_st16(taddr(tm, wwarp * 32, tm_u(b) + 16 * h2), r);
          }
        }
      } else {
        // DELTANET_COMPENSATED (R19): Z (the operand of H += K^T Z
        // and O += A Z) and U' (the backward's record) are rounded to bf16
        // with the rounding error carried along the token axis, so prefix
        // sums over tokens carry ~sqrt(4) roundings instead of sqrt(C)
        // rounding errors are carried (in U' units: Z = s U', and the s_t of
        // neighbouring tokens may differ by orders of magnitude) along
        // 8-token blocks, four interleaved per 32-token half (ILP; DESIGN.md
        // R19).  Only Z is on the state chain; the ungated U' record is
        // formed after z_ready.
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float f[32];
          ld32_cols(tm, wwarp, tm_u(b) + 32 * h2, f);
          float ez[4] = {0.f, 0.f, 0.f, 0.f}, eu[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
              const int i = 8 * blk + e, t = 32 * h2 + i;
              const float st = vb[C + t], nt = vb[2 * C + t];  // s_t, 1 / s_t
              const float u = f[i];
              const float xz = u + ez[blk];
              f[i] = __bfloat162float(__float2bfloat16_rn(xz * st));
              ez[blk] = fmaf(-f[i], nt, xz);
              if (st == 0.f) f[i] = 0.f;  // padded token: exact zero
              if (GATED && recs) {  // gated: the U' record inline (U's TMEM columns
                // 0-31 take Z_h below)
                const float xu = u + eu[blk];
                const float ru = __bfloat162float(__float2bfloat16_rn(xu));
                eu[blk] = xu - ru;
                *reinterpret_cast<__nv_bfloat16*>(recs + (size_t)c * REC_BYTES + REC_Z +
                                                  il_off(w, t, DV)) =
                    __float2bfloat16_rn(st == 0.f ? 0.f : ru);
              }
            }
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) il_store8(sZ, DV, w, 32 * h2 + g * 8, f + g * 8);
          if (GATED) {  // Z_h = Z diag(D) as bf16 pairs into U's columns [16 h2, 16 h2 + 16)
            // (this half of U' is in registers; the other half lies in columns >= 32)
            uint32_t zh[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int t = 32 * h2 + 2 * j;
              zh[j] = pack_bf16(f[2 * j] * vb[5 * C + t], f[2 * j + 1] * vb[5 * C + t + 1]);
            }
            tmem_st16(taddr(tm, wwarp * 32, tm_u(b) + 16 * h2), zh);
          }
        }
      }
      {
        if (GATED) {
          // (Z_h^T = Z^T diag(D) is in U's first 32 TMEM columns, the A operand
          // of H^T += Z_h^T K); H^T *= gamma_63 in TMEM
          const float gC = vb[4 * C + C - 1];
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            float hf[64];
            ld64(tm, wwarp, TM_H + 64 * hh, hf);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint32_t r[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(hf[16 * q4 + j] * gC);
              tmem_st16(taddr(tm, wwarp * 32, TM_H + 64 * hh + 16 * q4), r);
            }
          }
          tmem_st_wait();
        }
      }
      if (SEG1) {
        // T1 = Psi W^T (TM_W, lane = row a, cols = tokens) -> -T1 diag(s) as
        // bf16 pairs in TM_W's first 32 columns: the A operand (from TMEM) of
        // Psi += (-T1 diag(s)) K = Psi - Psi W^T K_hat
        float f[64];
        ld64(tm, wwarp, TM_W, f);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t r[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int t = 32 * h2 + 2 * j;
            r[j] = pack_bf16(-f[t] * vb[C + t], -f[t + 1] * vb[C + t + 1]);
          }
          tmem_st16(taddr(tm, wwarp * 32, TM_W + 16 * h2), r);
        }
        tmem_st_wait();
      }
      fence_proxy_async();
      fence_before_sync();
      wg_sync(BAR_S);
      if (w == 0) {
        mbar_arrive(&z_ready);
        if (!SEG1 && !APREP) mbar_arrive(&g_free);  // G_qk read: the next chunk's Q K^T may land
      }
      TSTAMP(18);
      mbar_wait(&ho_done, c & 1);
      mbar_wait(&st_free, c & 1);
      fence_after_sync();
      TSTAMP(19);
      DBG(dbg_tmem(dn_dbg + D_O, tm, TM_O, DV, 64, w); dbg_tmem(dn_dbg + D_H, tm, TM_H, DK, 128, w));
      {
        // H^T -> bf16 sH (operand of the next chunk) first: it is on the chain
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          float f[64];
          ld64(tm, wwarp, TM_H + 64 * half, f);
#pragma unroll
          for (int g = 0; g < 8; ++g) il_store8(sH, DV, w, 64 * half + g * 8, f + g * 8);
        }
        if (SEG1) {  // Psi (TM_O, lane = row a) -> bf16 image (row a) for the next T1
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            float f[64];
            ld64(tm, wwarp, TM_O + 64 * half, f);
#pragma unroll
            for (int g = 0; g < 8; ++g) il_store8(sPsi, DK, w, 64 * half + g * 8, f + g * 8);
          }
        } else {
          // O rows * r -> bf16 -> staging (IL R=64, row = token)
          const int i = wwarp * 16 + (lane & 15);
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            float f[64];
            ld64(tm, wwarp, TM_O + 64 * half, f);
            if (lane < 16) {
#pragma unroll
              for (int e = 0; e < 64; ++e) f[e] *= ri;
#pragma unroll
              for (int g = 0; g < 8; ++g) sw_store8(sO, C, i, 64 * half + g * 8, f + g * 8);
            }
          }
        }
      }
      fence_proxy_async();
      fence_before_sync();
      wg_sync(BAR_S);
      if (w == 0) {
        if (SEG1) mbar_arrive(&w_free);  // T1 consumed by the Psi update (ho_done)
        mbar_arrive(&h_ready);
      }
      if (!GATED && recs && comp) {
        // the backward's U'^T record (IL R = 128 x 64), off the state chain
        // (after h_ready, where this warpgroup would wait for the prep's next
        // W^T anyway): U' is still in TMEM -- the chain warp releases the U
        // buffer (bar_empty) only after u_read -- rounded with the error
        // carried along the tokens
        fence_after_sync();
        uint8_t* rz = recs + (size_t)c * REC_BYTES + REC_Z;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float f[32];
          ld32_cols(tm, wwarp, tm_u(b) + 32 * h2, f);
          float eu[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
              const int i = 8 * blk + e;
              const float xu = f[i] + eu[blk];
              f[i] = __bfloat162float(__float2bfloat16_rn(xu));
              eu[blk] = xu - f[i];
              if (vb[C + 32 * h2 + i] == 0.f) f[i] = 0.f;
            }
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 v;
            v.x = pack_bf16(f[g * 8 + 0], f[g * 8 + 1]);
            v.y = pack_bf16(f[g * 8 + 2], f[g * 8 + 3]);
            v.z = pack_bf16(f[g * 8 + 4], f[g * 8 + 5]);
            v.w = pack_bf16(f[g * 8 + 6], f[g * 8 + 7]);
            *reinterpret_cast<uint4*>(rz + il_off(w, 32 * h2 + g * 8, DV)) = v;
          }
        }
      }
      if (comp) {  // every state thread: its U' reads are complete
        fence_before_sync();
        mbar_arrive(&u_read);
      }
      TSTAMP(20);
    }
    // final state hT [dk][dv] (fp32), lane dv = w: the last segment's; SEG1
    // writes the segment-local end state and Psi instead
    float* hout = SEG1 ? a.hloc + ((size_t)unit * nseg + seg) * DK * DV
                  : (seg == nseg - 1) ? a.hT : nullptr;
    if (!SEG1 && hout) hout += (size_t)unit * DK * DV;
    if (SEG1) {
      fence_after_sync();
      float* psi = a.psi + ((size_t)unit * nseg + seg) * DK * DK;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float f[64];
        ld64(tm, wwarp, TM_O + 64 * half, f);
#pragma unroll
        for (int e = 0; e < 64; ++e) psi[(size_t)w * DK + 64 * half + e] = f[e];
      }
    }
    if (hout) {
      fence_after_sync();
      float* hT = hout;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float f[64];
        ld64(tm, wwarp, TM_H + 64 * half, f);
#pragma unroll
        for (int e = 0; e < 64; ++e) hT[(size_t)(64 * half + e) * DV + w] = f[e];
      }
    }
  } else if (warp == 12) {
    // =====================================================================
    // Warp 12: prep MMA issue + TMA loads of V (and of Q/K for chunks 0, 1)
    // =====================================================================
    if (lane == 0) {
      for (int c = 0; c < NQB && c < NC && !SEG1; ++c) {  // (SEG1 needs no Q)
        mbar_expect_tx(&q_full[c], TILE);
        tma_load_sw(sQ(c), &mQ, T0 + c * C, unit, &q_full[c]);
      }
      for (int c = 0; c < NKB && c < NC; ++c) {
        mbar_expect_tx(&k_full[c], TILE);
        tma_load_sw(sK(c), &mK, T0 + c * C, unit, &k_full[c]);
      }
      mbar_expect_tx(&v_full[0], TILE);
      tma_load_sw(sV, &mV, T0, unit, &v_full[0]);
      const uint32_t idg = idesc_bf16(64, 64, false, false);
      const uint32_t idw = idesc_bf16(128, 64, true, false);
      const uint32_t at = smem_u32(sT), atu = smem_u32(sTu), av = smem_u32(sV);
      auto gram_k = [&](int c) {  // G_kk -> lanes 16-31 of each quadrant (APREP: and G_qk)
        const uint32_t ak = smem_u32(sK(c % NKB)), aq = smem_u32(sQ(c % NQB));
        mbar_wait(&k_full[c % NKB], (c / NKB) & 1);
        if (APREP) mbar_wait(&q_full[c % NQB], (c / NQB) & 1);
        fence_after_sync();
#pragma unroll
        for (int k0 = 0; k0 < DK; k0 += 16) {
          mma_bf16(tm + TM_G + LO16, desc_k_sw(ak, C, k0), desc_k_sw(ak, C, k0), idg, k0 > 0);
          if (APREP) mma_bf16(tm + TM_G, desc_k_sw(aq, C, k0), desc_k_sw(ak, C, k0), idg, k0 > 0);
        }
        mma_commit(&gk_done);
      };
      auto gram_q = [&](int c) {  // G_qk -> lanes 0-15 of each quadrant
        const uint32_t aq = smem_u32(sQ(c % NQB)), ak = smem_u32(sK(c % NKB));
        mbar_wait(&q_full[c % NQB], (c / NQB) & 1);
        mbar_wait(&k_full[c % NKB], (c / NKB) & 1);
        fence_after_sync();
        TSTAMP1(28);
#pragma unroll
        for (int k0 = 0; k0 < DK; k0 += 16)
          mma_bf16(tm + TM_G, desc_k_sw(aq, C, k0), desc_k_sw(ak, C, k0), idg, k0 > 0);
        mma_commit(&g_done);
      };
      if (NC > 0) {
        if (!pre) gram_k(0);  // (pass 3 from prep records needs no K K^T)
        if (!SEG1 && !APREP) gram_q(0);
      }
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        const int b = c & 1;
        const uint32_t ak = smem_u32(sK(c % NKB));
        // the next chunk's Gram halves as soon as the prep has read this
        // chunk's (gk_free after L; g_free once the state warpgroup has formed A)
        // and their tiles have
        // landed (K K^T then runs under this chunk's substitution) -- but
        // never ahead of this chunk's W/U products: if T is ready first, the
        // remaining halves wait until after them
        bool pk = !pre && c + 1 < NC, pq = !SEG1 && !APREP && c + 1 < NC;
        bool kfree = false;
        while (true) {
          if (pk) {
            if (!kfree) kfree = mbar_test(&gk_free, c & 1);
            if (kfree && mbar_test(&k_full[(c + 1) % NKB], ((c + 1) / NKB) & 1) &&
                (!APREP || mbar_test(&q_full[(c + 1) % NQB], ((c + 1) / NQB) & 1))) {
              gram_k(c + 1);
              pk = false;
            }
          }
          if (mbar_test(&t_ready, c & 1)) break;
        }
        TSTAMP1(24);
        if (c >= 1) mbar_wait(&w_free, (c - 1) & 1);
        TSTAMP1(25);
        if (c >= 2) mbar_wait(&bar_empty[b], ((c >> 1) - 1) & 1);  // U[b] consumed
        TSTAMP1(26);
        mbar_wait(&v_full[b], (c >> 1) & 1);
        TSTAMP1(27);
        fence_after_sync();
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + TM_W, desc_mn_sw(ak, C, k0), desc_k(at, C, k0), idw, k0 > 0);
        mma_commit(&w_done);
#pragma unroll
        for (int k0 = 0; k0 < C; k0 += 16)
          mma_bf16(tm + tm_u(b), desc_mn_sw(av, C, k0), desc_k(atu, C, k0), idw, k0 > 0);
        mma_commit(&wu_done);
        if (pk) {
          mbar_wait(&gk_free, c & 1);
          gram_k(c + 1);
        }
        mbar_wait(&wu_done, c & 1);
        if (c + 1 < NC) {  // V (and T, T'') free again: prefetch the next chunk's V
          const int nb = (c + 1) & 1;
          mbar_expect_tx(&v_full[nb], TILE);
          tma_load_sw(sV, &mV, T0 + (c + 1) * C, unit, &v_full[nb]);
        }
        if (pq) {  // the state warpgroup has read this chunk's G_qk (g_free, with z_ready)
          mbar_wait(&g_free, c & 1);
          gram_q(c + 1);
        }
      }
    }
    __syncwarp();
  } else {
    // =====================================================================
    // Warp 13: state-chain MMA issue, state save, O store, next Q/K loads
    // =====================================================================
    if (lane == 0) {
      void* const o_out = SEG1 ? nullptr : a.o;
      uint8_t* states = (!SEG1 && (a.flags & DELTANET_SAVE_STATES))
                            ? (uint8_t*)a.states + ((size_t)unit * a.NC + cbase) * (DK * DV * 2)
                            : nullptr;
      const uint32_t aPsi = smem_u32(sPsi);
      const uint32_t idt = idesc_bf16(128, 64, false, true);    // T1 = Psi W^T
      const uint32_t idp = idesc_bf16(128, 128, false, true);   // Psi += (-T1 s) K
      const uint32_t aH = smem_u32(sH), aZ = smem_u32(sZ);
      const uint32_t idn = idesc_bf16(128, 64, false, true, /*neg_a=*/true);
      const uint32_t ido = idesc_bf16(64, 128, false, false);
      const uint32_t idh = idesc_bf16(128, 128, false, true);
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        const int b = c & 1;
        const uint32_t aw = smem_u32(sW(b)), aq = smem_u32(sQ(c % NQB)), aa = smem_u32(sA(b)),
                       ak = smem_u32(sK(c % NKB));
        mbar_wait(&bar_full[b], (c >> 1) & 1);
        mbar_wait(&h_ready, c & 1);  // sH = bf16 image of H_c; sO = O of chunk c-1
        if (c >= 1 && o_out) {
          tma_store_sw(&mO, sO, T0 + (c - 1) * C, unit);
          bulk_commit();
        }
        if (states) {  // save H_c (bf16 smem image) for the backward
          bulk_store(states + (size_t)c * DK * DV * 2, sH, DK * DV * 2);
          bulk_commit();
        }
        fence_after_sync();
        // U'^T = U^T - H^T W^T (M=128,N=64,K=128); O = Q H (M=64,N=128,K=128)
#pragma unroll
        for (int k0 = 0; k0 < DK; k0 += 16)
          mma_bf16(tm + tm_u(b), desc_k(aH, DV, k0), desc_mn(aw, DK, k0), idn, 1);
        if (SEG1) {  // T1 = Psi W^T (M=128 a, N=64 t, K=128 dk) into TM_W
#pragma unroll
          for (int k0 = 0; k0 < DK; k0 += 16)
            mma_bf16(tm + TM_W, desc_k(aPsi, DK, k0), desc_mn(aw, DK, k0), idt, k0 > 0);
        }
        mma_commit(&up_done);
        if (!SEG1) {
#pragma unroll
          for (int k0 = 0; k0 < DK; k0 += 16)
            mma_bf16(tm + TM_O, desc_k_sw(aq, C, k0), desc_k(aH, DV, k0), ido, k0 > 0);
        }
        mma_commit(&q_done);  // Q[b] read by the tensor core (norm reads: q_read)
        // the O store of chunk c-1 must finish reading sO (= sZ) before Z is written
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(1) : "memory");
        if (!states) bulk_wait_read0();
        mbar_arrive(&z_free);
        mbar_wait(&q_done, c & 1);
        if (!SEG1 && c + NQB < NC) {  // Q of chunk c+NQB into the slot O = Q H has released
          if (!SEG1) mbar_wait(&q_read, c & 1);  // ... and the norm pass (SEG1 has none)
          const int qs = c % NQB;
          mbar_expect_tx(&q_full[qs], TILE);
          tma_load_sw(sQ(qs), &mQ, T0 + (c + NQB) * C, unit, &q_full[qs]);
          TSTAMPC(c + NQB, 29);
        }
        mbar_wait(&z_ready, c & 1);
        fence_after_sync();
        if (states && !COMP) {
          // Z^T of this chunk for the backward (read out before st_free); with
          // DELTANET_COMPENSATED the state warpgroup stores U'^T instead
          bulk_store(reinterpret_cast<uint8_t*>(a.scratch) +
                         ((size_t)unit * a.NC + cbase + c) * REC_BYTES + REC_Z,
                     sZ, DV * C * 2);
          bulk_commit();
        }
        // H^T += Z^T K (M=128,N=128,K=64); O += tril(QK^T) Z (M=64,N=128,K=64)
        // (gated: H^T += Z_h^T K with Z_h^T from TMEM)
        if (GATED) {
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16_ts(tm + TM_H, tm + tm_u(b) + k0 / 2, desc_mn_sw(ak, C, k0), idh, 1);
        } else {
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_H, desc_k(aZ, DV, k0), desc_mn_sw(ak, C, k0), idh, 1);
        }
        if (SEG1) {  // Psi += (-T1 diag(s)) K, A from TMEM (bf16 pairs in TM_W)
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16_ts(tm + TM_O, tm + TM_W + k0 / 2, desc_mn_sw(ak, C, k0), idp, 1);
        } else {
#pragma unroll
          for (int k0 = 0; k0 < C; k0 += 16)
            mma_bf16(tm + TM_O, desc_k(aa, C, k0), desc_k(aZ, DV, k0), ido, 1);
        }
        mma_commit(&ho_done);
        mbar_wait(&ho_done, c & 1);
        if (c + NKB < NC) {  // K of chunk c+NKB into this chunk's K slot
          const int ks = c % NKB;
          mbar_expect_tx(&k_full[ks], TILE);
          tma_load_sw(sK(ks), &mK, T0 + (c + NKB) * C, unit, &k_full[ks]);
          TSTAMPC(c + NKB, 30);
        }
        bulk_wait_read0();  // state save done reading sH
        mbar_arrive(&st_free);
        // (after st_free: the state warpgroup reads U' for its record after
        // h_ready, which follows its st_free wait)
        // DELTANET_COMPENSATED: the state warpgroup reads U[b] and vec[b] for
        // the U' record after h_ready; otherwise its U' reads precede z_ready
        if (COMP) mbar_wait(&u_read, c & 1);
        mbar_arrive(&bar_empty[b]);  // A[b], vec[b] and U[b] are free for chunk c+2
      }
      // O of the last chunk
      mbar_wait(&h_ready, NC & 1);
      if (o_out && NC > 0) {
        tma_store_sw(&mO, sO, T0 + (NC - 1) * C, unit);
        bulk_commit();
      }
      bulk_wait0();
    }
    __syncwarp();
  }
  cta_sync();
  if (warp == 0) tmem_dealloc<512>(tm);
}

// Pass 2 of the segment-parallel forward: per unit, the states at the segment
// starts, H_start(s+1) = Psi_s^T H_start(s) + H_loc(s) (H = S^T, [dk][dv]),
// from H_start(0) = h0.  The columns of H evolve independently: a CTA scans
// one 16-column block; fp32 throughout.
__global__ void __launch_bounds__(256) seg_scan_kernel(Args a) {
  extern __shared__ __align__(16) float scan_sm[];
  float* Ps = scan_sm;  // Psi_s, row stride PSI_LD (tc_common.cuh stage_psi)
  float(*Hs)[16] = reinterpret_cast<float(*)[16]>(scan_sm + DK * PSI_LD);
  const int unit = blockIdx.x, j0 = blockIdx.y * 16, nseg = a.nseg;
  const int tid = threadIdx.x, i = tid >> 1, jj = (tid & 1) * 8;
  for (int e = tid; e < DK * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    Hs[r][cc] = a.h0 ? a.h0[(size_t)unit * DK * DV + (size_t)r * DV + j0 + cc] : 0.f;
  }
  for (int sg = 0; sg + 1 < nseg; ++sg) {
    const float* hl = a.hloc + ((size_t)unit * nseg + sg) * DK * DV + (size_t)i * DV + j0 + jj;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = hl[e];
    stage_psi(Ps, a.psi + ((size_t)unit * nseg + sg) * DK * DK, tid);
#pragma unroll 8
    for (int r = 0; r < DK; ++r) {
      const float pv = Ps[r * PSI_LD + i];  // Psi[r][i]
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(pv, Hs[r][jj + e], acc[e]);
    }
    __syncthreads();
    float* out = a.hseg + ((size_t)unit * nseg + sg + 1) * DK * DV + (size_t)i * DV + j0 + jj;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      Hs[i][jj + e] = acc[e];
      out[e] = acc[e];
    }
  }
}

// Context-parallel scan (deltanet_state_scan): parts p of the sequence with
// transitions Psi_p [Dk][Dk] and local states loc_p [Dk][Dv] (gathered over
// ranks).  Forward: out = fold_{p < part} (H <- Psi_p^T H + loc_p) from h_edge;
// reverse: out = fold_{p > part, descending} (G <- Psi_p G + loc_p) from
// h_edge.  A CTA owns one 16-column block of one unit; fp32.
struct ScanArgs {
  int units, nparts, part, reverse;
  const float *psi, *loc, *edge;
  float* out;
};
__global__ void __launch_bounds__(256) cp_scan_kernel(ScanArgs sa) {
  extern __shared__ __align__(16) float scan_sm[];
  float* Ps = scan_sm;
  float(*Hs)[16] = reinterpret_cast<float(*)[16]>(scan_sm + DK * PSI_LD);
  const int unit = blockIdx.x, j0 = blockIdx.y * 16;
  const int tid = threadIdx.x, i = tid >> 1, jj = (tid & 1) * 8;
  for (int e = tid; e < DK * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    Hs[r][cc] = sa.edge ? sa.edge[(size_t)unit * DK * DV + (size_t)r * DV + j0 + cc] : 0.f;
  }
  const int n = sa.reverse ? sa.nparts - 1 - sa.part : sa.part;
  for (int step = 0; step < n; ++step) {
    const int p = sa.reverse ? sa.nparts - 1 - step : step;
    const float* lc = sa.loc + ((size_t)p * sa.units + unit) * DK * DV + (size_t)i * DV + j0 + jj;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = lc[e];
    stage_psi(Ps, sa.psi + ((size_t)p * sa.units + unit) * DK * DK, tid);
#pragma unroll 8
    for (int r = 0; r < DK; ++r) {
      const float pv = sa.reverse ? Ps[i * PSI_LD + r] : Ps[r * PSI_LD + i];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(pv, Hs[r][jj + e], acc[e]);
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) Hs[i][jj + e] = acc[e];
  }
  __syncthreads();
  for (int e = tid; e < DK * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    sa.out[(size_t)unit * DK * DV + (size_t)r * DV + j0 + cc] = Hs[r][cc];
  }
}

// Composition of a unit's S segment transitions (context parallelism with
// the segment-parallel pass 1), fp32:
//   fwd: Psi = Psi_0 Psi_1 ... Psi_{S-1} (blockIdx.y < 8: column block),
//        Hloc = fold_s (H <- Psi_s^T H + hloc_s) from 0 (blockIdx.y >= 8);
//   bwd: dHloc = fold_{s = S-1..0} (G <- Psi_s G + dhloc_s) from 0.
__global__ void __launch_bounds__(256) cp_compose_kernel(int nseg, int bwd, const float* psi_s,
                                                         const float* loc_s, float* psi_out,
                                                         float* loc_out) {
  extern __shared__ __align__(16) float scan_sm[];
  float* Ps = scan_sm;
  float(*Xs)[16] = reinterpret_cast<float(*)[16]>(scan_sm + DK * PSI_LD);
  const int unit = blockIdx.x;
  const bool do_psi = !bwd && blockIdx.y < DK / 16;
  const int j0 = (do_psi ? blockIdx.y : blockIdx.y - (bwd ? 0 : DK / 16)) * 16;
  const int tid = threadIdx.x, i = tid >> 1, jj = (tid & 1) * 8;
  const float* P = psi_s + (size_t)unit * nseg * DK * DK;
  const float* H = loc_s + (size_t)unit * nseg * DK * DV;
  for (int e = tid; e < DK * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    Xs[r][cc] = do_psi ? P[(size_t)(nseg - 1) * DK * DK + (size_t)r * DK + j0 + cc] : 0.f;
  }
  const int n = do_psi ? nseg - 1 : nseg;
  for (int step = 0; step < n; ++step) {
    // fwd Psi: s = S-2 .. 0 (X <- Psi_s X); fwd Hloc: s = 0 .. S-1 (Psi_s^T);
    // bwd: s = S-1 .. 0 (Psi_s)
    const int sg = do_psi ? nseg - 2 - step : bwd ? nseg - 1 - step : step;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      acc[e] = do_psi ? 0.f : H[(size_t)sg * DK * DV + (size_t)i * DV + j0 + jj + e];
    stage_psi(Ps, P + (size_t)sg * DK * DK, tid);
    const bool tr = !do_psi && !bwd;
#pragma unroll 8
    for (int r = 0; r < DK; ++r) {
      const float pv = tr ? Ps[r * PSI_LD + i] : Ps[i * PSI_LD + r];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(pv, Xs[r][jj + e], acc[e]);
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) Xs[i][jj + e] = acc[e];
  }
  __syncthreads();
  float* out = do_psi ? psi_out + (size_t)unit * DK * DK : loc_out + (size_t)unit * DK * DV;
  for (int e = tid; e < DK * 16; e += blockDim.x) {
    const int r = e / 16, cc = e % 16;
    out[(size_t)r * DK + j0 + cc] = Xs[r][cc];
  }
}

// transition of an empty sequence: Psi = I, loc = 0 (psi or loc may be null)
__global__ void cp_empty_kernel(int units, float* psi, float* loc) {
  const size_t n = (size_t)units * DK * DK;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)((e / DK) % DK), c = (int)(e % DK);
    if (psi) psi[e] = r == c ? 1.f : 0.f;
    if (loc) loc[e] = 0.f;  // DK == DV
  }
}

}  // namespace

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


// 4-D view {8 elems, L rows, D/8 column groups, B*H units} of a [B*H][L][D]
// bf16 tensor; a box {8, rows, D/8, 1} lands in smem as the IL layout (R=rows).
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

bool make_sw_map(CUtensorMap* m, const void* base, int BH, int L, int D, int rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)L, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)L * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tc_supported(const deltanet_desc* d) {
  return d->dtype == DELTANET_BF16 && d->chunk == C && d->Dk == DK && d->Dv == DV && d->L > 0;
}

// gated DeltaNet (R23) on the tcgen05 kernels, forward and backward
//
bool tc_gated_supported(const deltanet_desc*) { return true; }

// per-chunk records [X | Z^T | row norms] the backward reads (tc_common.cuh REC_*)
namespace {
int sm_count() {  // per device (a process may drive several GPUs)
  static std::atomic<int> cache[64];
  const int dev = cur_device();
  int n = cache[dev].load();
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;  // B200
    }
    cache[dev].store(n);
  }
  return n;
}
size_t round256(size_t x) { return (x + 255) & ~(size_t)255; }
size_t rec_bytes(int B, int H, int L) {
  return (size_t)B * H * ((size_t)(L + C - 1) / C) * REC_BYTES;
}
}  // namespace

// dynamic shared memory opt-in of the scan kernels outside tc_fwd (per device)
int scan_attrs() {
  static PerDevice attr;
  if (attr.done()) return DELTANET_OK;
  if (cudaFuncSetAttribute(seg_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PSI_SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(cp_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PSI_SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(cp_compose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PSI_SMEM) != cudaSuccess)
    return DELTANET_ERR_CUDA;
  attr.mark();
  return DELTANET_OK;
}

// Sequence segments per unit of the tcgen05 forward: when
// B*H units leave SMs idle, each unit's chunks are split over up to
// SMs / units CTAs (segments of >= 8 chunks, at most 16).
int tc_fwd_segments(const deltanet_desc* d) {
  if (d->flags & (DELTANET_NO_SEGMENTS | DELTANET_GATED)) return 1;  // gated: one CTA per unit
  const int units = d->B * d->H, NCk = (d->L + C - 1) / C;
  if (units <= 0) return 1;
  int n = sm_count() / units;
  n = n < NCk / 8 ? n : NCk / 8;
  n = n < 16 ? n : 16;
  if (n < 3) return 1;  // passes 1 + 3 cost about two forwards: pays from 3 segments
  const int seg_len = (NCk + n - 1) / n;
  return (NCk + seg_len - 1) / seg_len;
}

// per-chunk records [X | Z^T] the backward reads (24 KB per chunk per unit),
// then the segment scratch (H_loc, Psi, H_start per (unit, segment))
size_t tc_scratch_bytes(const deltanet_desc* d) {
  const int nseg = tc_fwd_segments(d);
  const size_t seg = nseg > 1 ? (size_t)d->B * d->H * nseg * (2 * DK * DV + DK * DK) * 4 : 0;
  const size_t prec = nseg > 1 ? (size_t)d->B * d->H * ((d->L + C - 1) / C) * PREC_BYTES : 0;
  return round256(rec_bytes(d->B, d->H, d->L)) + round256(seg) + prec;
}

// fwd: 1 kernel (3 when segmented); bwd: 1 kernel (3 when segmented), plus
// the state-recompute forward without SAVE_STATES
int tc_launch_count(const deltanet_desc* d, int which) {
  const int f = tc_fwd_segments(d) > 1 ? 3 : 1;
  return which == 0 ? f : ((d->flags & DELTANET_SAVE_STATES) ? f : 2 * f);
}

// Segment layout shared by the forward and the backward: nseg, seg_len and
// the scratch after the records (H_loc | Psi | H_start per (unit, segment);
// the backward reuses H_loc and H_start for dl/dH).  Returns nseg.
int tc_seg_setup(Args& a) {
  deltanet_desc d;
  d.B = a.B; d.H = a.H; d.L = a.L; d.Dk = a.Dk; d.Dv = a.Dv; d.chunk = a.C;
  d.dtype = DELTANET_BF16; d.flags = a.flags; d.l2_eps = a.eps;
  const int nseg = tc_fwd_segments(&d);
  a.nseg = nseg > 1 ? nseg : 1;
  if (nseg <= 1) return 1;
  const int BH = a.B * a.H;
  a.seg_len = (a.NC + nseg - 1) / nseg;
  float* base = (float*)((char*)a.scratch + round256(rec_bytes(a.B, a.H, a.L)));
  a.hloc = base;
  a.psi = a.hloc + (size_t)BH * nseg * DK * DV;
  a.hseg = a.psi + (size_t)BH * nseg * DK * DK;
  // prep records of pass 1 for pass 3 (forward, with the per-chunk records)
  a.prec = (a.flags & DELTANET_SAVE_STATES)
               ? (uint8_t*)base + round256((size_t)BH * nseg * (2 * DK * DV + DK * DK) * 4)
               : nullptr;
  return nseg;
}

int tc_fwd(const Args& a0, cudaStream_t s) {
  static PerDevice attr;
  if (!attr.done()) {
    if (cudaFuncSetAttribute(tc_fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_fwd_kernel<false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_fwd_kernel<false, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_fwd_kernel<false, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(tc_fwd_kernel<false, false, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess ||
        scan_attrs() != DELTANET_OK)
      return DELTANET_ERR_CUDA;
    attr.mark();
  }
  Args a = a0;
  const int BH = a.B * a.H;
  CUtensorMap mQ, mK, mV, mO;
  if (!make_sw_map(&mQ, a.q, BH, a.L, DK, C) || !make_sw_map(&mK, a.k, BH, a.L, DK, C) ||
      !make_sw_map(&mV, a.v, BH, a.L, DV, C) ||
      !make_sw_map(&mO, a.o ? a.o : a.v, BH, a.L, DV, C))  // o == null: states only
    return DELTANET_ERR_CUDA;
  const int nseg = tc_seg_setup(a);
  const bool comp = (a.flags & DELTANET_COMPENSATED) != 0;  // DESIGN.md R19
  if (a.g) {  // gated DeltaNet (R23): one CTA per unit
    if (comp) tc_fwd_kernel<false, true, true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
    else tc_fwd_kernel<false, true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  if (nseg <= 1) {
    if (comp) tc_fwd_kernel<false, false, true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
    else tc_fwd_kernel<false><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  if (comp) a.prec = nullptr;  // (the compensated pass 3 redoes its prep)
  tc_fwd_kernel<true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);   // pass 1
  seg_scan_kernel<<<dim3(BH, DV / 16), 256, PSI_SMEM, s>>>(a);              // pass 2
  if (comp) tc_fwd_kernel<false, false, true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
  else if (a.prec)  // pass 3 from pass 1's prep records
    tc_fwd_kernel<false, false, false, true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
  else tc_fwd_kernel<false><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);  // pass 3
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

// Context parallelism (include/deltanet.h): the transition of this call's
// whole sequence: pass 1 of the segment machinery, one segment per unit, or,
// when the units leave SMs idle, S segments per unit composed by
// cp_compose_kernel (a.scratch = the workspace's segment scratch)
int tc_fwd_transition(const Args& a0, float* psi, float* hloc, cudaStream_t s) {
  Args a = a0;
  const int BH = a.B * a.H;
  CUtensorMap mQ, mK, mV, mO;
  if (!make_sw_map(&mQ, a.q, BH, a.L, DK, C) || !make_sw_map(&mK, a.k, BH, a.L, DK, C) ||
      !make_sw_map(&mV, a.v, BH, a.L, DV, C) || !make_sw_map(&mO, a.v, BH, a.L, DV, C))
    return DELTANET_ERR_CUDA;
  static PerDevice attr;
  if (!attr.done()) {
    if (cudaFuncSetAttribute(tc_fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr.mark();
  }
  a.o = nullptr;
  a.hT = nullptr;
  a.h0 = nullptr;
  const int nseg = a.scratch ? tc_seg_setup(a) : 1;
  a.prec = nullptr;  // no pass 3 here
  if (nseg <= 1) {
    a.nseg = 1;
    a.hloc = hloc;
    a.psi = psi;
    tc_fwd_kernel<true><<<BH, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
  } else {
    if (int rc = scan_attrs()) return rc;
    tc_fwd_kernel<true><<<BH * nseg, NT, SMEM_BYTES, s>>>(mQ, mK, mV, mO, a);
    cp_compose_kernel<<<dim3(BH, 2 * DK / 16), 256, PSI_SMEM, s>>>(nseg, 0, a.psi, a.hloc, psi,
                                                                    hloc);
  }
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int cp_compose_bwd(const Args& a, float* dhloc, cudaStream_t s) {
  if (int rc = scan_attrs()) return rc;
  cp_compose_kernel<<<dim3(a.B * a.H, DV / 16), 256, PSI_SMEM, s>>>(a.nseg, 1, a.psi, a.hloc, nullptr,
                                                             dhloc);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int cp_empty(int units, float* psi, float* loc, cudaStream_t s) {
  cp_empty_kernel<<<4 * 148, 256, 0, s>>>(units, psi, loc);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int cp_scan(int units, int nparts, int part, int reverse, const float* psi, const float* loc,
            const float* edge, float* out, cudaStream_t s) {
  ScanArgs sa{units, nparts, part, reverse, psi, loc, edge, out};
  if (int rc = scan_attrs()) return rc;
  cp_scan_kernel<<<dim3(units, DV / 16), 256, PSI_SMEM, s>>>(sa);
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

#ifdef DN_TIMING
extern "C" int dn_timing_set(long long* buf) {
  return cudaMemcpyToSymbol(dn::dn_tim, &buf, sizeof(buf)) != cudaSuccess;
}
#endif
