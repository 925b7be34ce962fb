// common.cuh -- shared device helpers and launch arguments of libdeltanet.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/deltanet.h"

namespace dn {

// Current device ordinal (0 if the query fails), for per-device host caches.
inline int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d & 63;
}

// One-time setup flags kept per device: kernel attributes such as the
// dynamic shared-memory opt-in belong to a device context, so a process that
// drives several GPUs must set them on each.  Concurrent first calls may both
// run the (idempotent) setup.
struct PerDevice {
  std::atomic<unsigned long long> bits{0};
  bool done() const { return (bits.load() >> cur_device()) & 1ull; }
  void mark() { bits.fetch_or(1ull << cur_device()); }
};

// All tensor arguments of one fwd or bwd call (see include/deltanet.h).
struct Args {
  int B, H, L, Dk, Dv, C, NC;
  unsigned flags;
  float eps;
  const void *q, *k, *v, *beta;
  const float* h0;
  void* o;
  float* hT;
  const void* dO;
  const float* dhT;
  void *dq, *dk, *dv, *dbeta;
  float* dh0;
  void* states;    // [B*H][NC][Dk][Dv] of the I/O dtype (H_t before chunk t)
  float* scratch;  // path-specific scratch
  // sequence segments of the tcgen05 forward (tc_fwd.cu):
  // nseg CTAs per unit, seg_len chunks each (nseg <= 1: one CTA per unit)
  int nseg, seg_len;
  float* hseg;  // [B*H][nseg][Dk][Dv] state at each segment start (pass 3 input)
  float* hloc;  // [B*H][nseg][Dk][Dv] segment-local end state from zero (pass 1)
  float* psi;   // [B*H][nseg][Dk][Dk] segment transition (pass 1)
  // [B*H][NC] per-chunk prep records [T' | T'' | s | 1/s] written by pass 1
  // and read by pass 3 instead of redoing the substitution (tc_fwd.cu PREC_*)
  uint8_t* prec;
  // Gated DeltaNet (R23): log-decay g [B*H][L]
  // fp32 (null = ungated) and its gradient
  const float* g;
  float* dg;
};

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
// Prefetch of a bf16 scalar one chunk ahead: the raw bits stay in a register
// and are widened at the use site.  (With `x = __bfloat162float(*p)` the
// compiler places the widening right after the load, so the warp waits out
// the full global latency there -- ~1.2 k cycles per chunk on the forward's
// prep warps, measured.)
__device__ __forceinline__ uint16_t ldg_u16(const void* p) {
  uint16_t v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float bf16_bits(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }

template <typename T>
__device__ __forceinline__ void stf(T* p, float x);
template <>
__device__ __forceinline__ void stf<float>(float* p, float x) { *p = x; }
template <>
__device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, float x) {
  *p = __float2bfloat16_rn(x);
}

// SIMT path entry points (simt.cu)
int simt_fwd(const Args& a, int dtype, cudaStream_t s);
int simt_bwd(const Args& a, int dtype, cudaStream_t s);
size_t simt_scratch_floats_per_unit(int L, int Dk, int Dv, int C);

// recurrent (token-by-token) inference path (recurrent.cu)
int rec_fwd(const Args& a, int dtype, cudaStream_t s);

// layer prologue (prologue.cu)
size_t prologue_workspace_bytes(const deltanet_desc* d);
int prologue_fwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                 const void* xb, const float* wq, const float* wk, const float* wv, void* q,
                 void* k, void* v, void* beta, cudaStream_t s);
int prologue_bwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                 const void* xb, const float* wq, const float* wk, const float* wv,
                 const void* dq, const void* dk, const void* dv, const void* dbeta, void* dxq,
                 void* dxk, void* dxv, void* dxb, float* dwq, float* dwk, float* dwv,
                 void* ws, cudaStream_t s);

// tcgen05 path entry points (tc_fwd.cu / tc_bwd.cu)
bool tc_supported(const deltanet_desc* d);
bool tc_gated_supported(const deltanet_desc* d);
size_t tc_scratch_bytes(const deltanet_desc* d);
int tc_fwd(const Args& a, cudaStream_t s);
int tc_bwd(const Args& a, cudaStream_t s);
int tc_launch_count(const deltanet_desc* d, int which);
int tc_fwd_segments(const deltanet_desc* d);
int tc_seg_setup(Args& a);
int tc_fwd_transition(const Args& a, float* psi, float* hloc, cudaStream_t s);
int tc_bwd_transition(const Args& a, float* dhloc, cudaStream_t s);
int cp_empty(int units, float* psi, float* loc, cudaStream_t s);
int cp_compose_bwd(const Args& a, float* dhloc, cudaStream_t s);
int cp_scan(int units, int nparts, int part, int reverse, const float* psi, const float* loc,
            const float* edge, float* out, cudaStream_t s);

// tcgen05 split path (tc_split.cu)
bool sp_supported(const deltanet_desc* d);
size_t sp_scratch_bytes(const deltanet_desc* d);
int sp_launch_count(const deltanet_desc* d, int which);
int sp_fwd(const Args& a, cudaStream_t s);
int sp_bwd(const Args& a, cudaStream_t s);

}  // namespace dn
