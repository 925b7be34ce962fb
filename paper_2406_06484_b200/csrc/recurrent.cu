// recurrent.cu -- token-by-token (recurrent-form) DeltaNet forward for
// inference / decode (the paper's recurrent baseline of
// fig:kernel_speed).
//
// The delta rule of PAPER.md §2.2, in the kernel orientation
// H = S^T [Dk][Dv] (R2):
//   u_j = sum_i k_i H[i][j],  H[i][j] -= beta (u_j - v_j) k_i,  o_j = sum_i q_i H[i][j]
// with q, k optionally L2-normalised (R9).  Column j of H evolves
// independently of the other columns given the token stream, so the state is
// split by columns across threads and CTAs: a CTA owns VB <= 64 columns of one
// (b, h) unit, a thread owns RPT <= 64 rows of one column in registers (TPC
// threads per column, adjacent lanes, combined with shuffles).  Gated
// DeltaNet (R23): H <- alpha (H - beta k (k^T H)) + beta k v^T, i.e.
// H[i][j] = alpha H[i][j] - beta (alpha u_j - v_j) k_i.  Tokens are
// staged through shared memory 32 at a time (q, k normalised there).  fp32
// state and arithmetic; bf16 or fp32 I/O.  Latency-bound on the per-token
// dependency (two TPC-lane reductions per token) at long L; HBM-bound on the
// state read/write at decode lengths.
#include "common.cuh"

namespace dn {
namespace {

constexpr int TB = 32;  // tokens staged per block

template <int DK>
struct RecShape {
  static constexpr int TPC = DK >= 128 ? DK / 64 : 1;  // threads per column
  static constexpr int RPT = DK / TPC;                 // rows per thread (<= 64)
  // smem row of q / k: a 4-float pad between 64-row segments so the TPC
  // segments of one warp-wide float4 load fall in different banks
  static constexpr int KS = DK + (TPC > 1 ? 4 * TPC : 0);
  __host__ __device__ static constexpr int idx(int i) { return TPC > 1 ? i + (i / 64) * 4 : i; }
};

template <typename T, int DK>
__global__ void __launch_bounds__(256) rec_fwd_kernel(Args a, int VB) {
  using S = RecShape<DK>;
  extern __shared__ __align__(16) float sm[];
  float* sk = sm;                    // [TB][KS]
  float* sq = sk + TB * S::KS;       // [TB][KS]
  float* sv = sq + TB * S::KS;       // [TB][VB]
  float* so = sv + TB * VB;          // [TB][VB]
  float* sb = so + TB * VB;          // [TB]
  float* sa = sb + TB;               // [TB] alpha = exp(g) (1 without a gate)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int unit = blockIdx.x, c0 = blockIdx.y * VB;
  const int col = tid / S::TPC, seg = tid % S::TPC;
  const int L = a.L, Dv = a.Dv;
  const bool l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  const T* q = (const T*)a.q + (size_t)unit * L * DK;
  const T* k = (const T*)a.k + (size_t)unit * L * DK;
  const T* v = (const T*)a.v + (size_t)unit * L * Dv;
  const T* beta = (const T*)a.beta + (size_t)unit * L;
  T* o = (T*)a.o + (size_t)unit * L * Dv;
  const float* gg = a.g ? a.g + (size_t)unit * L : nullptr;

  float h[S::RPT];
  {
    const float* h0 = a.h0 ? a.h0 + (size_t)unit * DK * Dv : nullptr;
#pragma unroll
    for (int r = 0; r < S::RPT; ++r)
      h[r] = h0 ? h0[(size_t)(seg * S::RPT + r) * Dv + c0 + col] : 0.f;
  }

  for (int t0 = 0; t0 < L; t0 += TB) {
    const int nt = min(TB, L - t0);
    __syncthreads();  // previous block's so / sk / sq consumed
    for (int e = tid; e < nt * DK; e += blockDim.x) {
      const int t = e / DK, i = e % DK;
      sk[t * S::KS + S::idx(i)] = ldf(k + (size_t)(t0 + t) * DK + i);
      sq[t * S::KS + S::idx(i)] = ldf(q + (size_t)(t0 + t) * DK + i);
    }
    for (int e = tid; e < nt * VB; e += blockDim.x) {
      const int t = e / VB, j = e % VB;
      sv[t * VB + j] = ldf(v + (size_t)(t0 + t) * Dv + c0 + j);
    }
    if (tid < nt) {
      sb[tid] = ldf(beta + t0 + tid);
      sa[tid] = gg ? __expf(gg[t0 + tid]) : 1.f;
    }
    __syncthreads();
    if (l2) {  // x <- x / max(||x||, eps), one warp per (token, tensor)
      for (int p = warp; p < 2 * nt; p += nwarp) {
        float* row = (p < nt ? sk : sq) + (p % nt) * S::KS;
        float acc = 0.f;
        for (int i = lane; i < DK; i += 32) acc = fmaf(row[S::idx(i)], row[S::idx(i)], acc);
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
        const float inv = 1.f / fmaxf(sqrtf(acc), a.eps);
        for (int i = lane; i < DK; i += 32) row[S::idx(i)] *= inv;
      }
      __syncthreads();
    }
    if (col < VB) {
      // u_t = k_t . h before token t's update; one fused pass per token then
      // applies the update and forms o_t = q_t . h and u_{t+1} = k_{t+1} . h
      float u;
      {
        const float* kr = sk + S::idx(seg * S::RPT);
        float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
#pragma unroll
        for (int r = 0; r < S::RPT; r += 4) {
          const float4 k4 = *reinterpret_cast<const float4*>(kr + r);
          u0 = fmaf(k4.x, h[r], u0);
          u1 = fmaf(k4.y, h[r + 1], u1);
          u2 = fmaf(k4.z, h[r + 2], u2);
          u3 = fmaf(k4.w, h[r + 3], u3);
        }
        u = (u0 + u1) + (u2 + u3);
#pragma unroll
        for (int m = 1; m < S::TPC; m <<= 1) u += __shfl_xor_sync(0xffffffffu, u, m);
      }
      for (int t = 0; t < nt; ++t) {
        const float* kr = sk + t * S::KS + S::idx(seg * S::RPT);
        const float* qr = sq + t * S::KS + S::idx(seg * S::RPT);
        const float* kn = (t + 1 < nt) ? kr + S::KS : kr;  // k_{t+1} (dummy at the block end)
        const float al = sa[t];
        const float cc = sb[t] * (al * u - sv[t * VB + col]);
        float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f, n3 = 0.f;
#pragma unroll
        for (int r = 0; r < S::RPT; r += 4) {
          const float4 k4 = *reinterpret_cast<const float4*>(kr + r);
          const float4 q4 = *reinterpret_cast<const float4*>(qr + r);
          const float4 n4 = *reinterpret_cast<const float4*>(kn + r);
          h[r] = fmaf(-cc, k4.x, al * h[r]);
          h[r + 1] = fmaf(-cc, k4.y, al * h[r + 1]);
          h[r + 2] = fmaf(-cc, k4.z, al * h[r + 2]);
          h[r + 3] = fmaf(-cc, k4.w, al * h[r + 3]);
          o0 = fmaf(q4.x, h[r], o0);
          o1 = fmaf(q4.y, h[r + 1], o1);
          o2 = fmaf(q4.z, h[r + 2], o2);
          o3 = fmaf(q4.w, h[r + 3], o3);
          n0 = fmaf(n4.x, h[r], n0);
          n1 = fmaf(n4.y, h[r + 1], n1);
          n2 = fmaf(n4.z, h[r + 2], n2);
          n3 = fmaf(n4.w, h[r + 3], n3);
        }
        float ov = (o0 + o1) + (o2 + o3);
        u = (n0 + n1) + (n2 + n3);
#pragma unroll
        for (int m = 1; m < S::TPC; m <<= 1) {
          ov += __shfl_xor_sync(0xffffffffu, ov, m);
          u += __shfl_xor_sync(0xffffffffu, u, m);
        }
        if (seg == 0) so[t * VB + col] = ov;
      }
    }
    __syncthreads();
    for (int e = tid; e < nt * VB; e += blockDim.x) {
      const int t = e / VB, j = e % VB;
      stf(o + (size_t)(t0 + t) * Dv + c0 + j, so[t * VB + j]);
    }
  }
  if (a.hT && col < VB) {
    float* hT = a.hT + (size_t)unit * DK * Dv;
#pragma unroll
    for (int r = 0; r < S::RPT; ++r) hT[(size_t)(seg * S::RPT + r) * Dv + c0 + col] = h[r];
  }
}

template <typename T, int DK>
int launch(const Args& a, cudaStream_t s) {
  using S = RecShape<DK>;
  const int VB = a.Dv < 64 ? a.Dv : 64;
  const int threads = VB * S::TPC;  // 16..256, a multiple of 16
  const int nthreads = (threads + 31) / 32 * 32;
  const size_t smem = (size_t)(2 * TB * S::KS + 2 * TB * VB + 2 * TB) * sizeof(float);
  static PerDevice attr;  // per template instance: the largest (VB = 64) footprint
  if (!attr.done()) {
    const size_t smax = (size_t)(2 * TB * S::KS + 2 * TB * 64 + 2 * TB) * sizeof(float);
    if (cudaFuncSetAttribute(rec_fwd_kernel<T, DK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smax) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    attr.mark();
  }
  dim3 grid(a.B * a.H, a.Dv / VB);
  rec_fwd_kernel<T, DK><<<grid, nthreads, smem, s>>>(a, VB);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

template <typename T>
int dispatch(const Args& a, cudaStream_t s) {
  switch (a.Dk) {
    case 16: return launch<T, 16>(a, s);
    case 32: return launch<T, 32>(a, s);
    case 64: return launch<T, 64>(a, s);
    case 128: return launch<T, 128>(a, s);
    case 256: return launch<T, 256>(a, s);
  }
  return DELTANET_ERR_UNSUPPORTED;
}

}  // namespace

int rec_fwd(const Args& a, int dtype, cudaStream_t s) {
  return dtype == DELTANET_FP32 ? dispatch<float>(a, s) : dispatch<__nv_bfloat16>(a, s);
}

}  // namespace dn
