// tc_common.cuh -- sm_100a primitives: tcgen05 MMA/TMEM, mbarrier, TMA.
//
// Operand layout of the tensor-core tiles ("IL"; the forward's Q, K, V and
// O tiles use the SW layout further below instead,
// SWIZZLE_NONE canonical layout): a logical R x Cc bf16 matrix X (row-major,
// columns contiguous) is stored as core matrices of 8 rows x 16 bytes:
//     byte offset of X[r][c] = ((c / 8) * R + r) * 16 + (c % 8) * 2
// i.e. [Cc/8 column groups][R rows][8 elements].  The same tile serves as
//   - a K-major operand whose M/N index is the row r (reduction over c):
//       SBO = 128 B (next 8 rows), LBO = R*16 B (next 8 columns),
//       K-step of 16 columns = +2*R*16 B;
//   - an MN-major operand whose M/N index is the column c (reduction over r):
//       SBO = R*16 B (next 8 columns), LBO = 128 B (next 8 rows),
//       K-step of 16 rows = +256 B.
// (Canonical forms from CuTe's UMMA::make_umma_desc, mma_traits_sm100.hpp.)
// A TMA box {8 elements, R rows, Cc/8 groups} writes exactly this layout.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dn {
namespace tc {

// Per-chunk record the tcgen05 forward writes (with DELTANET_SAVE_STATES)
// for the backward, next to H_t: images of X = (I+L)^{-1} (bf16, IL R=64 x
// 64, exactly lower-triangular) and Z^T = (diag(s) U')^T (IL R=128 x 64) --
// with DELTANET_COMPENSATED U'^T itself, rounded with the error carried
// along the tokens (R19).  Offsets in bytes.  (W is not needed: the backward
// uses W^T dU' = K_hat^T diag(beta) X^T dU' = K_hat^T dV.)
constexpr int REC_X = 0, REC_Z = 64 * 64 * 2;
constexpr int REC_N = REC_Z + 128 * 64 * 2;  // fp32 row norms [||k|| (64) | ||q|| (64)]
constexpr int REC_A = REC_N + 2 * 64 * 4;     // A = tril(Q K^T) (gated: Gamma . A), raw, bf16 IL 64x64
constexpr int REC_BYTES = REC_A + 64 * 64 * 2;  // 32.5 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ------------------------------------------------------------------ UMMA
// Shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // descriptor version (Blackwell)
  return d;                 // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE
}
// K-major view of an IL tile with R rows (M/N = rows), at K offset k0 (cols).
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int R, int k0) {
  return sdesc(base + (uint32_t)(k0 / 8) * R * 16, (uint32_t)R * 16, 128);
}
// MN-major view of an IL tile with R rows (M/N = columns, starting at col
// group n0/8), at K offset k0 (rows).
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int R, int k0, int n0 = 0) {
  return sdesc(base + (uint32_t)(n0 / 8) * R * 16 + (uint32_t)k0 * 16, 128, (uint32_t)R * 16);
}

// ---- "SW" tiles: the SWIZZLE_128B canonical layout, which a TMA box with
// 128 B rows writes directly (8x fewer TMA requests than the IL box's 16 B
// rows; tools/probes/tma_probe.cu).  A logical R x Cc bf16 matrix (Cc a
// multiple of 64) is stored as Cc/64 column blocks of R rows x 128 B; inside
// a block, row r is at r*128 and its 16 B chunk j at chunk (j ^ (r & 7)):
//     byte offset of X[r][c] = (c/64)*R*128 + r*128 + (((c%64)/8) ^ (r%8))*16 + (c%8)*2
// Tiles are 1024 B aligned (the swizzle XORs absolute address bits [4,7)
// with [7,10)).  The same tile serves as
//   - a K-major operand (M/N = row r, reduction over c): SBO = 1024 B (next 8
//     rows), K-step of 16 columns = +32 B inside a block (next block at 64);
//   - an MN-major operand (M/N = column c, reduction over r): LBO = R*128 B
//     (next 64-column block), SBO = 1024 B (next 8 rows), K-step of 16 rows
//     = +2048 B.
__host__ __device__ __forceinline__ uint32_t sw_off(int r, int c, int R) {
  return (uint32_t)((c >> 6) * R * 128 + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + (c & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = sdesc(saddr, lbo, sbo);
  d |= (uint64_t)2u << 61;  // layout type SWIZZLE_128B (sm_100 encoding)
  return d;
}
__device__ __forceinline__ uint64_t desc_k_sw(uint32_t base, int R, int k0) {
  return sdesc_sw128(base + (uint32_t)(k0 >> 6) * R * 128 + (uint32_t)(k0 & 63) * 2, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mn_sw(uint32_t base, int R, int k0, int n0 = 0) {
  return sdesc_sw128(base + (uint32_t)(n0 >> 6) * R * 128 + (uint32_t)k0 * 128, (uint32_t)R * 128,
                     1024);
}

// Instruction descriptor, kind::f16, A/B bf16, D fp32.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn,
                                                  bool neg_a = false) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (neg_a ? (1u << 13) : 0u) |
         (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier when all previously issued tcgen05.mma of this
// thread complete (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Make generic-proxy shared-memory writes visible to the async proxy
// (tensor core / TMA reads).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ TMEM
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%"
      "14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%"
      "13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// TMEM address of (lane, column) relative to an allocation base.
__device__ __forceinline__ uint32_t taddr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking probe of an mbarrier phase (true once the phase completed).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ------------------------------------------------------------------ TMA / bulk
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* smem_src, int c0,
                                             int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::
          "l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(smem_src))
      : "memory");
}
// A chunk tile [rows tokens][128 columns] of a [BH][L][128] bf16 tensor as a
// SW tile (two 64-column boxes of a make_sw_map map), and its store.
__device__ __forceinline__ void tma_load_sw(void* smem_dst, const CUtensorMap* map, int t,
                                            int unit, uint64_t* bar, int rows = 64) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst) + h * rows * 128),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(64 * h), "r"(t), "r"(unit), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_sw(const CUtensorMap* map, const void* smem_src, int t,
                                             int unit, int rows = 64) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(64 * h), "r"(t), "r"(unit), "r"(smem_u32(smem_src) + h * rows * 128)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// L2 prefetch of a TMA tile (no shared memory, no completion): a later
// tma_load_4d of the same box then hits L2 instead of waiting on HBM
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2,
                                                int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// L2 prefetch of a contiguous global range (bytes: a multiple of 16)
__device__ __forceinline__ void bulk_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------------------ packing
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Byte offset of element (r, c) in an IL tile of R rows.
__host__ __device__ __forceinline__ uint32_t il_off(int r, int c, int R) {
  return (uint32_t)(((c >> 3) * R + r) * 16 + (c & 7) * 2);
}
// Store 8 consecutive columns [c0, c0+8) of row r (c0 % 8 == 0) as one 16 B chunk.
__device__ __forceinline__ void il_store8(uint8_t* tile, int R, int r, int c0, const float* x) {
  uint4 v;
  v.x = pack_bf16(x[0], x[1]);
  v.y = pack_bf16(x[2], x[3]);
  v.z = pack_bf16(x[4], x[5]);
  v.w = pack_bf16(x[6], x[7]);
  *reinterpret_cast<uint4*>(tile + il_off(r, c0, R)) = v;
}

// Store / load 8 consecutive columns [c0, c0+8) of row r (c0 % 8 == 0) of a SW tile.
__device__ __forceinline__ void sw_store8(uint8_t* tile, int R, int r, int c0, const float* x) {
  uint4 v;
  v.x = pack_bf16(x[0], x[1]);
  v.y = pack_bf16(x[2], x[3]);
  v.z = pack_bf16(x[4], x[5]);
  v.w = pack_bf16(x[6], x[7]);
  *reinterpret_cast<uint4*>(tile + sw_off(r, c0, R)) = v;
}
__device__ __forceinline__ void sw_load8(const uint8_t* tile, int R, int r, int c0, float* x) {
  const uint4 v = *reinterpret_cast<const uint4*>(tile + sw_off(r, c0, R));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 f = __bfloat1622float2(h[e]);
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}

// ------------------------------------------------------------------ CTA helpers
__device__ __forceinline__ void cta_sync() {
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
}

// Load 64 fp32 columns [col, col+64) of this warp's 32 TMEM lanes.
__device__ __forceinline__ void ld64(uint32_t tm, int warp, uint32_t col, float (&f)[64]) {
  uint32_t r[4][16];
#pragma unroll
  for (int i = 0; i < 4; ++i) tmem_ld16(taddr(tm, warp * 32, col + 16 * i), r[i]);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) f[16 * i + j] = __uint_as_float(r[i][j]);
}

// Read 8 bf16 of row r, columns [c0, c0+8) of an IL tile as fp32.
__device__ __forceinline__ void il_load8(const uint8_t* tile, int R, int r, int c0, float* x) {
  uint4 v = *reinterpret_cast<const uint4*>(tile + il_off(r, c0, R));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 f = __bfloat1622float2(h[e]);
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}

}  // namespace tc

// host: 4-D TMA view of a [B*H][L][D] bf16 tensor whose box {8, rows, D/8, 1}
// lands in shared memory as the IL layout with R = rows (tc_fwd.cu).
bool make_il_map(CUtensorMap* m, const void* base, int BH, int L, int D, int rows);
// 3-D view {D, L, B*H} of a [B*H][L][D] bf16 tensor (D = 128); a box {64,
// rows, 1} lands in smem as one 64-column block of a SW tile (SWIZZLE_128B)
bool make_sw_map(CUtensorMap* m, const void* base, int BH, int L, int D, int rows);
// cuTensorMapEncodeTiled through the runtime's driver entry point (tc_fwd.cu)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

}  // namespace dn

namespace dn {
namespace tc {

// Unpack one 16 B chunk (8 bf16) to fp32.
__device__ __forceinline__ void unpack8(const uint4& v, float* x) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 f = __bfloat1622float2(h[e]);
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}

// Named barrier over one 128-thread warpgroup (ids 1.. ; 0 is __syncthreads).
__device__ __forceinline__ void wg_sync(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// Named barrier over NTH threads (NTH = 128 or 256).
template <int NTH>
__device__ __forceinline__ void grp_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NTH) : "memory");
}

// Warp-level tensor-core product D(16x8) += A(16x8) B(8x8), tf32 inputs
// (cvt.rna from fp32), fp32 accumulate.  Fragments (g = lane/4, t = lane%4):
// a = {A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4]}, b = {B[t][g], B[t+4][g]},
// d = {D[g][2t], D[g][2t+1], D[g+8][2t], D[g+8][2t+1]}.
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], const float (&a)[4],
                                                const float (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(to_tf32(a[0])), "r"(to_tf32(a[1])), "r"(to_tf32(a[2])), "r"(to_tf32(a[3])),
        "r"(to_tf32(b[0])), "r"(to_tf32(b[1])));
}

// One 16x8 tile of P = A B (K = 8 * KSTEPS) from fp32 row-major smem, by one
// warp.  A(r, k) = LX[(ar + r) * LS + ac + k], B(k, n) = LX[(br + k) * LS + bc + n];
// a_lower / b_lower mask A / B to their lower triangle relative to the given
// diagonal offsets (entries above it hold scratch).
template <int LS, int KSTEPS>
__device__ __forceinline__ void tile_mma(const float* LX, int ar, int ac, int br, int bc,
                                         bool a_lower, int a_diag, bool b_lower, int b_diag,
                                         int lane, float (&d)[4]) {
  const int g = lane >> 2, t = lane & 3;
  d[0] = d[1] = d[2] = d[3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
    const int k0 = 8 * ks;
    float a[4], b[2];
    a[0] = LX[(ar + g) * LS + ac + k0 + t];
    a[1] = LX[(ar + g + 8) * LS + ac + k0 + t];
    a[2] = LX[(ar + g) * LS + ac + k0 + t + 4];
    a[3] = LX[(ar + g + 8) * LS + ac + k0 + t + 4];
    b[0] = LX[(br + k0 + t) * LS + bc + g];
    b[1] = LX[(br + k0 + t + 4) * LS + bc + g];
    if (a_lower) {  // A(r, k) = 0 for k - r > a_diag
      a[0] = (k0 + t - g <= a_diag) ? a[0] : 0.f;
      a[1] = (k0 + t - g - 8 <= a_diag) ? a[1] : 0.f;
      a[2] = (k0 + t + 4 - g <= a_diag) ? a[2] : 0.f;
      a[3] = (k0 + t + 4 - g - 8 <= a_diag) ? a[3] : 0.f;
    }
    if (b_lower) {  // B(k, n) = 0 for n - k > b_diag
      b[0] = (g - (k0 + t) <= b_diag) ? b[0] : 0.f;
      b[1] = (g - (k0 + t + 4) <= b_diag) ? b[1] : 0.f;
    }
    mma_tf32_16x8x8(d, a, b);
  }
}

// X = (I + L)^{-1} for a 64x64 strictly-lower L, in place in LX (fp32,
// row stride LSTRIDE floats), by 256 threads (wtid) that share named barrier
// bar_id.
// Level 1: forward substitution on the eight 8x8
// diagonal blocks, one warp per block, column-parallel in registers, then
// 8 -> 16 merges X21 = -X22 (L21 X11) in fp32 by all 256 threads.
// Levels 2-3: merge blocks pairwise, X21 = -X22 (L21 X11), for 16 -> 32 -> 64,
// as warp-level tf32 tensor-core products (mma.sync m16n8k8; R20:
// tf32 operand rounding, 2^-11, is below the bf16 rounding X then gets).
// On return the lower triangle and diagonal of LX hold X; entries above the
// diagonal hold scratch (callers mask j > i).
template <int LSTRIDE, int NTH = 256>
__device__ __forceinline__ void ut_inverse_inplace(float* LX, int wtid, int bar_id,
                                                   long long* stamps = nullptr) {
  static_assert(NTH == 256, "the tensor-core merges assume 8 warps");
  constexpr int LS = LSTRIDE;
  const int lane = wtid & 31, wwarp = wtid >> 5;
  const int g = lane >> 2, t = lane & 3;
  static_assert(LS >= 68, "level 1b keeps its 8x8 products in the row padding (cols 64-67)");
  {  // level 1a: the eight 8x8 diagonal blocks, warp q = block, column j = lane (< 8)
    const int o = 8 * wwarp, j = lane & 7;
    // All loads first (branch-free, so they can all be in flight), then the
    // dependent chain; x_i = [i == j] - [i > j] * sum_m L_im x_m.
    float4 l4[8][2];
#pragma unroll
    for (int i = 1; i < 8; ++i)
#pragma unroll
      for (int m = 0; m < i; m += 4)
        l4[i][m / 4] = *reinterpret_cast<const float4*>(LX + (o + i) * LS + o + m);
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int m = 0; m < i; m += 4) {
        const float4 l = l4[i][m / 4];
        a0 = fmaf(l.x, x[m], a0);
        if (m + 1 < i) a1 = fmaf(l.y, x[m + 1], a1);
        if (m + 2 < i) a2 = fmaf(l.z, x[m + 2], a2);
        if (m + 3 < i) a3 = fmaf(l.w, x[m + 3], a3);
      }
      const float eq = (i == j) ? 1.f : 0.f, gt = (i > j) ? 1.f : 0.f;
      x[i] = fmaf(-gt, (a0 + a1) + (a2 + a3), eq);
    }
    __syncwarp();
    if (lane < 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) LX[(o + i) * LS + o + j] = x[i];
    }
  }
  grp_sync<NTH>(bar_id);
  {  // level 1b: 8 -> 16 merges, warps 2p, 2p+1 on the 16x16 block p (offset
    // o = 16p); thread (r, c) of the 8x8 products.  Y = L21 X11 goes to the
    // row padding (cols 64-67 of rows o .. o+15), then X21 = -X22 Y.  The
    // block's upper-right 8x8 already holds zeros (L is strictly lower).
    const int o = 16 * (wwarp >> 1), idx = ((wwarp & 1) << 5) | lane, r = idx >> 3, c = idx & 7;
    float* ys = LX + o * LS + 64;  // Y[r][c] at ys[(idx >> 2) * LS + (idx & 3)]
    float y = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m)  // X11(m, c) = 0 for m < c (stored zeros)
      y = fmaf(LX[(o + 8 + r) * LS + o + m], LX[(o + m) * LS + o + c], y);
    ys[(idx >> 2) * LS + (idx & 3)] = y;
    grp_sync<NTH>(bar_id);
    float z = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m) {  // X22(r, m) = 0 for m > r (stored zeros)
      const int ym = m * 8 + c;
      z = fmaf(LX[(o + 8 + r) * LS + o + 8 + m], ys[(ym >> 2) * LS + (ym & 3)], z);
    }
    LX[(o + 8 + r) * LS + o + c] = -z;  // L21 was read above (before the sync)
  }
  grp_sync<NTH>(bar_id);
  if (stamps && wtid == 0) stamps[0] = clock64();
  // level 2 (warps 0-3): pair p at offset o = 32p, column tile n0 = 8 * (w & 1)
  const int o2 = 32 * ((wwarp >> 1) & 1), n2 = 8 * (wwarp & 1);
  if (wwarp < 4) {  // Y = L21 X11 -> LX[o:o+16][o+16:o+32] (scratch)
    float d[4];
    // X11 is a level-1 block: zero above its diagonal, no mask needed
    tile_mma<LS, 2>(LX, o2 + 16, o2, o2, o2 + n2, false, 0, false, 0, lane, d);
    LX[(o2 + g) * LS + o2 + 16 + n2 + 2 * t] = d[0];
    LX[(o2 + g) * LS + o2 + 16 + n2 + 2 * t + 1] = d[1];
    LX[(o2 + g + 8) * LS + o2 + 16 + n2 + 2 * t] = d[2];
    LX[(o2 + g + 8) * LS + o2 + 16 + n2 + 2 * t + 1] = d[3];
  }
  grp_sync<NTH>(bar_id);
  if (stamps && wtid == 0) stamps[1] = clock64();
  if (wwarp < 4) {  // X21 = -X22 Y -> LX[o+16:o+32][o:o+16]
    float d[4];
    tile_mma<LS, 2>(LX, o2 + 16, o2 + 16, o2, o2 + 16 + n2, true, 0, false, 0, lane, d);
    LX[(o2 + 16 + g) * LS + o2 + n2 + 2 * t] = -d[0];
    LX[(o2 + 16 + g) * LS + o2 + n2 + 2 * t + 1] = -d[1];
    LX[(o2 + 16 + g + 8) * LS + o2 + n2 + 2 * t] = -d[2];
    LX[(o2 + 16 + g + 8) * LS + o2 + n2 + 2 * t + 1] = -d[3];
  }
  grp_sync<NTH>(bar_id);
  if (stamps && wtid == 0) stamps[2] = clock64();
  // level 3 (8 warps): row tile r0 = 16 * (w >> 2), column tile n0 = 8 * (w & 3)
  const int r3 = 16 * (wwarp >> 2), n3 = 8 * (wwarp & 3);
  {  // Y = L21 X11 -> LX[0:32][32:64] (scratch)
    float d[4];
    // X11(m, j) = 0 for j > m (its upper-right block holds level-2 scratch)
    tile_mma<LS, 4>(LX, 32 + r3, 0, 0, n3, false, 0, true, -n3, lane, d);
    LX[(r3 + g) * LS + 32 + n3 + 2 * t] = d[0];
    LX[(r3 + g) * LS + 32 + n3 + 2 * t + 1] = d[1];
    LX[(r3 + g + 8) * LS + 32 + n3 + 2 * t] = d[2];
    LX[(r3 + g + 8) * LS + 32 + n3 + 2 * t + 1] = d[3];
  }
  grp_sync<NTH>(bar_id);
  if (stamps && wtid == 0) stamps[3] = clock64();
  {  // X21 = -X22 Y -> LX[32:64][0:32]
    float d[4];
    // X22(i, m) = 0 for m > i (its upper-right block holds level-2 scratch)
    tile_mma<LS, 4>(LX, 32 + r3, 32, 0, 32 + n3, true, r3, false, 0, lane, d);
    LX[(32 + r3 + g) * LS + n3 + 2 * t] = -d[0];
    LX[(32 + r3 + g) * LS + n3 + 2 * t + 1] = -d[1];
    LX[(32 + r3 + g + 8) * LS + n3 + 2 * t] = -d[2];
    LX[(32 + r3 + g + 8) * LS + n3 + 2 * t + 1] = -d[3];
  }
  grp_sync<NTH>(bar_id);
  if (stamps && wtid == 0) stamps[4] = clock64();
}

}  // namespace tc
}  // namespace dn

namespace dn {
namespace tc {

// D[tmem] (+)= A[tmem] * B[smem]: A (bf16, K-major) read from TMEM -- lane =
// row m, each 32-bit column holds two consecutive k; a K=16 step spans 8
// columns.  Pinned by tests/test_tc_probe.py::test_mma_a_from_tmem.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

}  // namespace tc
}  // namespace dn

namespace dn {
namespace tc {

// Segment / context-parallel scans (tc_fwd.cu, tc_bwd.cu): stage a 128 x 128
// fp32 matrix (64 KB, global) in shared memory with row stride 129 floats
// (conflict-free reads along rows and along columns), 256 threads with all
// of their 16 float4 loads in flight; the scans are latency-bound otherwise.
constexpr int PSI_LD = 129;
constexpr int PSI_SMEM = (128 * PSI_LD + 128 * 16) * 4;  // + the 128 x 16 state block
__device__ __forceinline__ void stage_psi(float* Ps, const float* psi, int tid) {
  float4 v[16];
  const float4* src = reinterpret_cast<const float4*>(psi);
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = src[tid + 256 * q];
  __syncthreads();  // the previous step's readers of Ps (and writers of the state) are done
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int f = (tid + 256 * q) * 4, row = f >> 7, col = f & 127;
    float* d = Ps + row * PSI_LD + col;
    d[0] = v[q].x;
    d[1] = v[q].y;
    d[2] = v[q].z;
    d[3] = v[q].w;
  }
  __syncthreads();
}

}  // namespace tc
}  // namespace dn

