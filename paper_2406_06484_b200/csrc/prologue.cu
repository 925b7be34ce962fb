// prologue.cu -- the DeltaNet layer prologue in front of the chunkwise kernel
// (SURVEY §8(f) f1): short causal depthwise convolution (width 4) after the
// q/k/v projections (§3.4, kernel size 4 P:822), SiLU
// feature map on q and k (the L2 normalisation itself is fused into
// the chunkwise kernels), beta = sigmoid(W_beta x), and the layout
// change from the projections' token-major [B, L, H, D] to the kernels'
// [B, H, L, D].  Forward and backward; both HBM-bound elementwise passes.
//
//   y[t] = sum_{j<4} w[c][j] x[t-3+j]   (x[t<0] = 0),   out = act(y)
//   act = SiLU for q, k; identity for v (or SiLU with DELTANET_PROLOGUE_SILU_V)
//
// Tiling: a thread owns 4 consecutive channels (8 B of bf16) and a run of
// RUN = 64 tokens, sliding a 4-token window with UNR = 8 tokens' loads in
// flight; a warp covers 128 channels of its run (one 256 B row per token), a
// CTA is 8 runs = 256 threads over 512 tokens of one (b, h, tensor).  (Four
// channels rather than eight keep the backward under 128 registers: at 255
// it ran one CTA per SM, 23 % of HBM.)  The
// backward recomputes y, forms dy = dout * act'(y), dx[t] = sum_j w[j]
// dy[t+3-j], and per-CTA partial dw sums that a second kernel reduces in a
// fixed order (deterministic, no atomics).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace dn {
namespace {

constexpr int RUN = 64, RUNS = 8, TT = RUN * RUNS;  // tokens per thread / CTA
constexpr int NCG = 32;  // channel groups of 4 per pass: one warp covers 128 channels
constexpr int UNR = 8;   // tokens whose loads are in flight per thread

// 4 consecutive channels as raw words (bf16: 8 B, fp32: 16 B), so that UNR
// tokens' loads can be in flight before any is unpacked
template <typename T>
struct Raw4;
template <>
struct Raw4<__nv_bfloat16> {
  uint2 w;
};
template <>
struct Raw4<float> {
  float4 w;
};
template <typename T>
__device__ __forceinline__ void load_raw(const T* p, Raw4<T>& r);
template <>
__device__ __forceinline__ void load_raw<__nv_bfloat16>(const __nv_bfloat16* p,
                                                        Raw4<__nv_bfloat16>& r) {
  r.w = *reinterpret_cast<const uint2*>(p);
}
template <>
__device__ __forceinline__ void load_raw<float>(const float* p, Raw4<float>& r) {
  r.w = *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void unpack(const Raw4<__nv_bfloat16>& r, float (&x)[4]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.w);
  const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
}
__device__ __forceinline__ void unpack(const Raw4<float>& r, float (&x)[4]) {
  x[0] = r.w.x; x[1] = r.w.y; x[2] = r.w.z; x[3] = r.w.w;
}
template <typename T>
__device__ __forceinline__ void load4(const T* p, float (&x)[4]) {
  Raw4<T> r;
  load_raw(p, r);
  unpack(r, x);
}
template <typename T>
__device__ __forceinline__ void store4(T* p, const float (&x)[4]);
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, const float (&x)[4]) {
  uint2 v;
  __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]), b = __floats2bfloat162_rn(x[2], x[3]);
  v.x = *reinterpret_cast<uint32_t*>(&a);
  v.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = v;
}
template <>
__device__ __forceinline__ void store4<float>(float* p, const float (&x)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
}

// fast reciprocal: an IEEE division here was most of the instruction count
__device__ __forceinline__ float sigm(float y) { return __frcp_rn(1.f + __expf(-y)); }

struct ProArgs {
  int B, H, L, Dk, Dv, silu_v, ntile;
  const void *xq, *xk, *xv, *xb;
  const float *wq, *wk, *wv;
  void *q, *k, *v, *beta;                 // fwd outputs / bwd cotangents (dq ...)
  void *dxq, *dxk, *dxv, *dxb;            // bwd outputs
  float *dwq, *dwk, *dwv;                 // bwd outputs [H*D][4]
  float* part;                            // bwd scratch: [3][B*ntile][H*Dmax][4]
};

// tensor z (0 q, 1 k, 2 v) of a ProArgs
struct Tz {
  const void* x;
  const float* w;
  void* y;
  void* dx;
  float* dw;
  int D;
  bool silu;
};
__device__ __forceinline__ Tz pick(const ProArgs& a, int z) {
  if (z == 0) return {a.xq, a.wq, a.q, a.dxq, a.dwq, a.Dk, true};
  if (z == 1) return {a.xk, a.wk, a.k, a.dxk, a.dwk, a.Dk, true};
  return {a.xv, a.wv, a.v, a.dxv, a.dwv, a.Dv, a.silu_v != 0};
}

// grid (ntile, B*H, 4): z < 3 conv + activation of q / k / v, z == 3 beta.
// A warp is one token run over 128 channels (lane = channel group of 4:
// 256 B per token row, coalesced); the 8 warps take consecutive runs.
template <typename T>
__global__ void __launch_bounds__(256, 2) prologue_fwd_kernel(ProArgs a) {
  const int tile = blockIdx.x, bh = blockIdx.y, z = blockIdx.z;
  const int b = bh / a.H, h = bh % a.H, H = a.H, L = a.L;
  const int t_begin = tile * TT;
  if (z == 3) {  // beta[b, h, t] = sigmoid(xb[b, t, h])
    for (int t = t_begin + threadIdx.x; t < min(L, t_begin + TT); t += blockDim.x)
      stf((T*)a.beta + ((size_t)b * H + h) * L + t,
          sigm(ldf((const T*)a.xb + ((size_t)b * L + t) * H + h)));
    return;
  }
  const Tz tz = pick(a, z);
  const int D = tz.D;
  const int run = threadIdx.x / NCG;  // token run
  const int t0 = t_begin + run * RUN;
  if (t0 >= L) return;
  for (int cg = threadIdx.x % NCG; 4 * cg < D; cg += NCG) {  // D = 256: two passes
  const int c = h * D + 4 * cg;  // first channel of this thread
  const T* x = (const T*)tz.x + (size_t)b * L * H * D + c;   // token stride H * D
  T* y = (T*)tz.y + ((size_t)b * H + h) * L * D + 4 * cg;     // token stride D
  float w[4][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float4 w4 = *reinterpret_cast<const float4*>(tz.w + (size_t)(c + e) * 4);
    w[e][0] = w4.x; w[e][1] = w4.y; w[e][2] = w4.z; w[e][3] = w4.w;
  }
  float win[3][4];  // x[t-3], x[t-2], x[t-1]
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int t = t0 - 3 + j;
    if (t >= 0) {
      load4(x + (size_t)t * H * D, win[j]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) win[j][e] = 0.f;
    }
  }
  const int t1 = min(L, t0 + RUN);
  for (int tb = t0; tb < t1; tb += UNR) {
    Raw4<T> raw[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (tb + u < t1) load_raw(x + (size_t)(tb + u) * H * D, raw[u]);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (tb + u >= t1) break;
      float xt[4], o[4];
      unpack(raw[u], xt);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float yy = fmaf(w[e][0], win[0][e],
                              fmaf(w[e][1], win[1][e], fmaf(w[e][2], win[2][e], w[e][3] * xt[e])));
        o[e] = tz.silu ? yy * sigm(yy) : yy;
        win[0][e] = win[1][e];
        win[1][e] = win[2][e];
        win[2][e] = xt[e];
      }
      store4(y + (size_t)(tb + u) * D, o);
    }
  }
  }
}

// backward: dy = dout * act'(y); dx[t] = sum_j w[j] dy[t+3-j]; partial dw.
template <typename T>
__global__ void __launch_bounds__(256, 2) prologue_bwd_kernel(ProArgs a) {
  __shared__ float red[RUNS][NCG * 16 + 4];  // [run][cg*16 + e*4 + j]
  const int tile = blockIdx.x, bh = blockIdx.y, z = blockIdx.z;
  const int b = bh / a.H, h = bh % a.H, H = a.H, L = a.L;
  const int t_begin = tile * TT;
  if (z == 3) {  // dxb[b, t, h] = dbeta * beta (1 - beta)
    for (int t = t_begin + threadIdx.x; t < min(L, t_begin + TT); t += blockDim.x) {
      const float s = sigm(ldf((const T*)a.xb + ((size_t)b * L + t) * H + h));
      const float g = ldf((const T*)a.beta + ((size_t)b * H + h) * L + t);
      stf((T*)a.dxb + ((size_t)b * L + t) * H + h, g * s * (1.f - s));
    }
    return;
  }
  const Tz tz = pick(a, z);
  const int D = tz.D;
  const int run = threadIdx.x / NCG;
  const int t0 = t_begin + run * RUN;
  const int npass = D > 4 * NCG ? D / (4 * NCG) : 1;  // 32 channel groups per pass
  for (int pass = 0; pass < npass; ++pass) {
  const int cg = threadIdx.x % NCG + NCG * pass;
  const bool active = 4 * cg < D && t0 < L;
  float dw[4][4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) dw[e][j] = 0.f;
  if (active) {
    const int c = h * D + 4 * cg;
    const T* x = (const T*)tz.x + (size_t)b * L * H * D + c;
    const T* g = (const T*)tz.y + ((size_t)b * H + h) * L * D + 4 * cg;  // dout
    T* dx = (T*)tz.dx + (size_t)b * L * H * D + c;
    float w[4][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 w4 = *reinterpret_cast<const float4*>(tz.w + (size_t)(c + e) * 4);
      w[e][0] = w4.x; w[e][1] = w4.y; w[e][2] = w4.z; w[e][3] = w4.w;
    }
    float xw[4][4];   // x[t-3..t]
    float dyw[3][4];  // dy[t-3], dy[t-2], dy[t-1]
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int t = t0 - 3 + j;
      if (t >= 0) {
        load4(x + (size_t)t * H * D, xw[j + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) xw[j + 1][e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) dyw[j][e] = 0.f;
    }
    const int t1 = min(L, t0 + RUN);
    const int tend = min(L, t1 + 3);  // dy needed up to t1 + 2 for dx[t1 - 1]
    for (int tb = t0; tb < tend; tb += UNR) {
    Raw4<T> rx[UNR], rg[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (tb + u < tend) {
        load_raw(x + (size_t)(tb + u) * H * D, rx[u]);
        load_raw(g + (size_t)(tb + u) * D, rg[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = tb + u;
      if (t >= tend) break;
      float xt[4], gt[4], dyt[4];
      unpack(rx[u], xt);
      unpack(rg[u], gt);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xw[0][e] = xw[1][e];
        xw[1][e] = xw[2][e];
        xw[2][e] = xw[3][e];
        xw[3][e] = xt[e];
        const float yy = fmaf(w[e][0], xw[0][e],
                              fmaf(w[e][1], xw[1][e], fmaf(w[e][2], xw[2][e], w[e][3] * xw[3][e])));
        float dyy = gt[e];
        if (tz.silu) {
          const float s = sigm(yy);
          dyy *= s * (1.f + yy * (1.f - s));
        }
        dyt[e] = dyy;
        if (t < t1) {  // this thread's own tokens contribute to dw
#pragma unroll
          for (int j = 0; j < 4; ++j) dw[e][j] = fmaf(dyy, xw[j][e], dw[e][j]);
        }
      }
      // dx[t-3] = w3 dy[t-3] + w2 dy[t-2] + w1 dy[t-1] + w0 dy[t]
      if (t - 3 >= t0) {
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          o[e] = fmaf(w[e][3], dyw[0][e],
                      fmaf(w[e][2], dyw[1][e], fmaf(w[e][1], dyw[2][e], w[e][0] * dyt[e])));
        store4(dx + (size_t)(t - 3) * H * D, o);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        dyw[0][e] = dyw[1][e];
        dyw[1][e] = dyw[2][e];
        dyw[2][e] = dyt[e];
      }
    }
    }
    // tail: tokens whose dy window runs past L (dy[t >= L] = 0)
    for (int s = max(t0, tend - 3); s < t1; ++s) {
      // after the loop dyw holds dy[tend-3], dy[tend-2], dy[tend-1]
      const int k0 = s - (tend - 3);  // 0, 1 or 2: position of dy[s] in dyw
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // dy[s + 3 - j] at dyw index k0 + 3 - j (< 3)
          const int idx = k0 + 3 - j;  // selects, not a dynamic register index
          const float dv = idx == 0 ? dyw[0][e] : idx == 1 ? dyw[1][e] : idx == 2 ? dyw[2][e] : 0.f;
          acc = fmaf(w[e][j], dv, acc);
        }
        o[e] = acc;
      }
      store4(dx + (size_t)s * H * D, o);
    }
  }
  // per-CTA dw partial: sum over the 8 runs in a fixed order
  __syncthreads();  // the previous pass finished reading red
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[run][(cg % NCG) * 16 + e * 4 + j] = dw[e][j];
  __syncthreads();
  for (int i = threadIdx.x; i < NCG * 16; i += blockDim.x) {
    const int cgi = i / 16 + NCG * pass;
    if (4 * cgi >= D) continue;
    float s = 0.f;
    for (int r = 0; r < RUNS; ++r) s += red[r][i];
    // part[z][b * ntile + tile][h * D + 4 cgi + e][j]
    const int Dm = a.Dk > a.Dv ? a.Dk : a.Dv;
    const size_t slot = ((size_t)z * a.B * a.ntile + (size_t)b * a.ntile + tile);
    a.part[(slot * H * Dm + (size_t)h * D + 4 * cgi) * 4 + (i % 16)] = s;
  }
  }
}

// dw[z][c][j] = sum over (b, tile) of the partials, fixed order
__global__ void prologue_dw_reduce(ProArgs a) {
  const int z = blockIdx.y;
  const int D = z == 2 ? a.Dv : a.Dk;
  const int Dm = a.Dk > a.Dv ? a.Dk : a.Dv;
  float* dw = z == 0 ? a.dwq : z == 1 ? a.dwk : a.dwv;
  const int n = a.H * D * 4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int h = i / (D * 4), r = i % (D * 4);
    float s = 0.f;
    for (int p = 0; p < a.B * a.ntile; ++p)
      s += a.part[(((size_t)z * a.B * a.ntile + p) * a.H * Dm + (size_t)h * D) * 4 + r];
    dw[i] = s;
  }
}

// ---- bf16, D = 128 forward: token rows staged by TMA (the register path
// above keeps too few bytes in flight to reach HBM speed, 2.5 TB/s).  A CTA
// owns TILE_T tokens of one (b, h, tensor); a ring of NBUF stages of ST
// token rows (256 B each) is loaded two stages ahead, stage -1 being the
// 3-token window before the tile (zero-filled by TMA before t = 0).  Warp w
// computes tokens [8w, 8w + 8) of a stage, lane = 4 channels.
constexpr int ST = 64, NBUF = 4, TILE_T = 1024, DT = 128, DHF = DT / 2;
constexpr int TMA_SMEM = NBUF * ST * DHF * 2;  // 32 KB: several CTAs per SM

// grid (B*H, tiles, 3 tensors x 2 channel halves); lane = 2 channels of the
// half (128 B rows), warp w = tokens [8w, 8w + 8) of a stage
__global__ void __launch_bounds__(256) prologue_fwd_tma_kernel(
    const __grid_constant__ CUtensorMap mxq, const __grid_constant__ CUtensorMap mxk,
    const __grid_constant__ CUtensorMap mxv, ProArgs a) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ uint64_t full[NBUF];
  // consecutive CTAs are the heads of one batch row and token tile, so the
  // token rows they share ([B,L,H,D]) are read together
  const int bh = blockIdx.x, tile = blockIdx.y, z = blockIdx.z >> 1, half = blockIdx.z & 1;
  const int b = bh / a.H, h = bh % a.H, H = a.H, L = a.L;
  const int t_begin = tile * TILE_T;
  const int nst = (min(TILE_T, L - t_begin) + ST - 1) / ST;
  const CUtensorMap* mx = z == 0 ? &mxq : z == 1 ? &mxk : &mxv;
  const Tz tz = pick(a, z);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int SB = ST * DHF * 2;
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) tc::mbar_init(&full[i], 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(mx);
  }
  __syncthreads();
  auto issue = [&](int s) {  // stage s -> buffer (s + 1) % NBUF
    uint64_t* bar = &full[(s + 1) % NBUF];
    tc::mbar_expect_tx(bar, SB);
    tc::tma_load_4d(sbuf + ((s + 1) % NBUF) * SB, mx, h * DT + half * DHF, t_begin + s * ST, b, 0,
                    bar);
  };
  if (tid == 0)
    for (int s = -1; s <= 1 && s < nst; ++s) issue(s);
  const int c = h * DT + half * DHF + 2 * lane;
  float w[2][4];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float4 w4 = *reinterpret_cast<const float4*>(tz.w + (size_t)(c + e) * 4);
    w[e][0] = w4.x; w[e][1] = w4.y; w[e][2] = w4.z; w[e][3] = w4.w;
  }
  __nv_bfloat16* y = (__nv_bfloat16*)tz.y + ((size_t)b * H + h) * L * DT + half * DHF + 2 * lane;
  auto row = [&](int s, int r, float (&x)[2]) {  // row r (may be < 0: previous stage)
    const int bi = (r < 0 ? s : s + 1) % NBUF, rr = r < 0 ? r + ST : r;
    const float2 f = __bfloat1622float2(
        *reinterpret_cast<const __nv_bfloat162*>(sbuf + (size_t)bi * SB + rr * DHF * 2 + 4 * lane));
    x[0] = f.x;
    x[1] = f.y;
  };
#pragma unroll 1
  for (int s = 0; s < nst; ++s) {
    if (tid == 0 && s + 2 < nst) issue(s + 2);  // its buffer held stage s - 2 (synced below)
    tc::mbar_wait(&full[s % NBUF], (s >> 2) & 1);            // stage s - 1 (window)
    tc::mbar_wait(&full[(s + 1) % NBUF], ((s + 1) >> 2) & 1);  // stage s
    const int r0 = 8 * warp;
    float win[3][2];
#pragma unroll
    for (int j = 0; j < 3; ++j) row(s, r0 - 3 + j, win[j]);
    float xt[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) row(s, r0 + u, xt[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t_begin + s * ST + r0 + u;
      float o[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float yy = fmaf(w[e][0], win[0][e],
                              fmaf(w[e][1], win[1][e], fmaf(w[e][2], win[2][e], w[e][3] * xt[u][e])));
        o[e] = tz.silu ? yy * sigm(yy) : yy;
        win[0][e] = win[1][e];
        win[1][e] = win[2][e];
        win[2][e] = xt[u][e];
      }
      if (t < L)
        *reinterpret_cast<__nv_bfloat162*>(y + (size_t)t * DT) = __floats2bfloat162_rn(o[0], o[1]);
    }
    __syncthreads();  // every warp is done with stage s - 1's buffer
  }
}

// beta[b, h, t] = sigmoid(xb[b, t, h]): thread per (b, t, h), reads contiguous
template <typename T>
__global__ void prologue_beta_kernel(ProArgs a) {
  const size_t n = (size_t)a.B * a.L * a.H;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int h = (int)(i % a.H);
    const size_t bt = i / a.H;
    const int t = (int)(bt % a.L), b = (int)(bt / a.L);
    stf((T*)a.beta + ((size_t)b * a.H + h) * a.L + t, sigm(ldf((const T*)a.xb + i)));
  }
}

// ---- bf16, D = 128 backward, TMA-staged like the forward, on 64-channel
// halves (a CTA per (b, h, tensor, half, tile); lane = 2 channels, 128 B
// rows) so that stages stay small (8 KB) and ~6 CTAs share an SM: stages of
// STB rows of x (token-major) and dout ([B,H,L,D]) in a ring of NBUF; stage
// -1 is the window before the tile, stage nst the 3-row look-ahead after it.
// Warp w owns rows [8w, 8w + 8) of a stage: it slides over rows 8w - 3 ..
// 8w + 10, forming dy = dout act'(y) for rows 8w .. 8w + 10 (3 recomputed
// by the next warp too) and dx for its own rows; dw partials stay in
// registers over the tile, then reduce over the warps in a fixed order into
// part[z][b * ntile + tile] (TILE_T tiles).
constexpr int STB = 32, NWB = 4, RPW = STB / NWB, DH = DT / 2;  // 4 warps of 8 rows, 64 channels
constexpr int TMA_SMEM_B = NBUF * 2 * STB * DH * 2;  // 32 KB

__global__ void __launch_bounds__(32 * NWB) prologue_bwd_tma_kernel(
    const __grid_constant__ CUtensorMap mxq, const __grid_constant__ CUtensorMap mxk,
    const __grid_constant__ CUtensorMap mxv, const __grid_constant__ CUtensorMap mgq,
    const __grid_constant__ CUtensorMap mgk, const __grid_constant__ CUtensorMap mgv, ProArgs a) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ uint64_t full[NBUF];
  // grid (B*H, tiles, 3 tensors x 2 channel halves)
  const int bh = blockIdx.x, tile = blockIdx.y, z = blockIdx.z >> 1, half = blockIdx.z & 1;
  const int b = bh / a.H, h = bh % a.H, H = a.H, L = a.L;
  const int t_begin = tile * TILE_T;
  const int nst = (min(TILE_T, L - t_begin) + STB - 1) / STB;
  const CUtensorMap* mx = z == 0 ? &mxq : z == 1 ? &mxk : &mxv;
  const CUtensorMap* mg = z == 0 ? &mgq : z == 1 ? &mgk : &mgv;
  const Tz tz = pick(a, z);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int SB = STB * DH * 2;  // bytes of one tile of a stage
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) tc::mbar_init(&full[i], 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(mx);
    tc::prefetch_tmap(mg);
  }
  __syncthreads();
  auto buf = [&](int s) { return sbuf + ((s + 1) % NBUF) * 2 * SB; };  // [x | dout]
  auto issue = [&](int s) {
    uint64_t* bar = &full[(s + 1) % NBUF];
    tc::mbar_expect_tx(bar, 2 * SB);
    tc::tma_load_4d(buf(s), mx, h * DT + half * DH, t_begin + s * STB, b, 0, bar);
    tc::tma_load_4d(buf(s) + SB, mg, half * DH, t_begin + s * STB, bh, 0, bar);
  };
  if (tid == 0)
    for (int s = -1; s <= 1 && s <= nst; ++s) issue(s);
  const int c = h * DT + half * DH + 2 * lane;  // first of this lane's two channels
  float w[2][4], dw[2][4];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float4 w4 = *reinterpret_cast<const float4*>(tz.w + (size_t)(c + e) * 4);
    w[e][0] = w4.x; w[e][1] = w4.y; w[e][2] = w4.z; w[e][3] = w4.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) dw[e][j] = 0.f;
  }
  __nv_bfloat16* dx = (__nv_bfloat16*)tz.dx + (size_t)b * L * H * DT + c;  // token stride H*D
  auto ld = [&](int s, int r, int part, float (&x)[2]) {  // row r of stage s (r may leave it)
    const int ss = r < 0 ? s - 1 : r >= STB ? s + 1 : s;
    const int rr = r < 0 ? r + STB : r >= STB ? r - STB : r;
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(
        buf(ss) + part * SB + rr * DH * 2 + 4 * lane));
    x[0] = f.x;
    x[1] = f.y;
  };
#pragma unroll 1
  for (int s = 0; s < nst; ++s) {
    if (tid == 0 && s + 2 <= nst) issue(s + 2);  // into stage s - 2's buffer (synced below)
    tc::mbar_wait(&full[s % NBUF], (s >> 2) & 1);
    tc::mbar_wait(&full[(s + 1) % NBUF], ((s + 1) >> 2) & 1);
    tc::mbar_wait(&full[(s + 2) % NBUF], ((s + 2) >> 2) & 1);
    const int r0 = RPW * warp;
    float xw[4][2], dyw[3][2];
#pragma unroll
    for (int j = 0; j < 3; ++j) ld(s, r0 - 3 + j, 0, xw[j + 1]);
#pragma unroll
    for (int u = 0; u < RPW + 3; ++u) {  // row r0 + u
      float xt[2], gt[2], dyt[2];
      ld(s, r0 + u, 0, xt);
      ld(s, r0 + u, 1, gt);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        xw[0][e] = xw[1][e];
        xw[1][e] = xw[2][e];
        xw[2][e] = xw[3][e];
        xw[3][e] = xt[e];
        const float yy = fmaf(w[e][0], xw[0][e],
                              fmaf(w[e][1], xw[1][e], fmaf(w[e][2], xw[2][e], w[e][3] * xw[3][e])));
        float dyy = gt[e];
        if (tz.silu) {
          const float sg = sigm(yy);
          dyy *= sg * (1.f + yy * (1.f - sg));
        }
        dyt[e] = dyy;
        if (u < RPW) {
#pragma unroll
          for (int j = 0; j < 4; ++j) dw[e][j] = fmaf(dyy, xw[j][e], dw[e][j]);
        }
      }
      if (u >= 3) {  // dx of own row r0 + u - 3 = w3 dy[.] + w2 dy[+1] + w1 dy[+2] + w0 dy[+3]
        const int t = t_begin + s * STB + r0 + u - 3;
        float o[2];
#pragma unroll
        for (int e = 0; e < 2; ++e)
          o[e] = fmaf(w[e][3], dyw[0][e],
                      fmaf(w[e][2], dyw[1][e], fmaf(w[e][1], dyw[2][e], w[e][0] * dyt[e])));
        if (t < L)
          *reinterpret_cast<__nv_bfloat162*>(dx + (size_t)t * H * DT) = __floats2bfloat162_rn(o[0], o[1]);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        dyw[0][e] = dyw[1][e];
        dyw[1][e] = dyw[2][e];
        dyw[2][e] = dyt[e];
      }
    }
    __syncthreads();  // every warp is done with stage s - 1's buffer
  }
  // dw partial of the tile: warps summed in a fixed order (the ring is free)
  float* red = reinterpret_cast<float*>(sbuf);  // [NWB warps][32 lanes * 8]
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[warp * 256 + lane * 8 + e * 4 + j] = dw[e][j];
  __syncthreads();
  for (int i = tid; i < 256; i += 32 * NWB) {
    float sum = 0.f;
    for (int r = 0; r < NWB; ++r) sum += red[r * 256 + i];
    const int Dm = a.Dk > a.Dv ? a.Dk : a.Dv;
    const size_t slot = ((size_t)z * a.B * a.ntile + (size_t)b * a.ntile + tile);
    // i = (channel within the half) * 4 + tap
    a.part[(slot * H * Dm + (size_t)h * DT + half * DH) * 4 + i] = sum;
  }
}

// dxb[b, t, h] = dbeta[b, h, t] * beta (1 - beta), beta = sigmoid(xb[b, t, h])
template <typename T>
__global__ void prologue_beta_bwd_kernel(ProArgs a) {
  const size_t n = (size_t)a.B * a.L * a.H;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int h = (int)(i % a.H);
    const size_t bt = i / a.H;
    const int t = (int)(bt % a.L), b = (int)(bt / a.L);
    const float sg = sigm(ldf((const T*)a.xb + i));
    const float g = ldf((const T*)a.beta + ((size_t)b * a.H + h) * a.L + t);
    stf((T*)a.dxb + i, g * sg * (1.f - sg));
  }
}

// [B*H][L][D] contiguous bf16 (the cotangents dq, dk, dv) viewed as
// {D, L, B*H, 1}, box {D/2, STB} (one channel half)
bool make_head_map(CUtensorMap* m, const void* base, int BH, int L) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)DT, (cuuint64_t)L, (cuuint64_t)BH, 1};
  cuuint64_t strides[3] = {(cuuint64_t)DT * 2, (cuuint64_t)L * DT * 2, (cuuint64_t)BH * L * DT * 2};
  cuuint32_t box[4] = {(cuuint32_t)DH, (cuuint32_t)STB, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [B][L][H*D] token-major bf16 input viewed as {H*D, L, B, 1}, box {D, ST}
bool make_rows_map(CUtensorMap* m, const void* base, int B, int L, int HD, int rows = ST,
                   int cols = DT) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)HD, (cuuint64_t)L, (cuuint64_t)B, 1};
  cuuint64_t strides[3] = {(cuuint64_t)HD * 2, (cuuint64_t)L * HD * 2, (cuuint64_t)B * L * HD * 2};
  cuuint32_t box[4] = {(cuuint32_t)cols, (cuuint32_t)rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

ProArgs make(const deltanet_desc* d) {
  ProArgs a;
  memset(&a, 0, sizeof a);
  a.B = d->B; a.H = d->H; a.L = d->L; a.Dk = d->Dk; a.Dv = d->Dv;
  a.silu_v = (d->flags & DELTANET_PROLOGUE_SILU_V) ? 1 : 0;
  a.ntile = (d->L + TT - 1) / TT;
  return a;
}

}  // namespace

size_t prologue_workspace_bytes(const deltanet_desc* d) {
  const size_t ntile = (size_t)(d->L + TT - 1) / TT;
  const size_t Dm = d->Dk > d->Dv ? d->Dk : d->Dv;
  return 3 * (size_t)d->B * ntile * d->H * Dm * 4 * sizeof(float);
}

int prologue_fwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                 const void* xb, const float* wq, const float* wk, const float* wv, void* q,
                 void* k, void* v, void* beta, cudaStream_t s) {
  ProArgs a = make(d);
  a.xq = xq; a.xk = xk; a.xv = xv; a.xb = xb; a.wq = wq; a.wk = wk; a.wv = wv;
  a.q = q; a.k = k; a.v = v; a.beta = beta;
  if (d->dtype == DELTANET_BF16 && d->Dk == DT && d->Dv == DT && d->L > 0) {
    static PerDevice attr;
    if (!attr.done()) {
      if (cudaFuncSetAttribute(prologue_fwd_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               TMA_SMEM) != cudaSuccess)
        return DELTANET_ERR_CUDA;
      attr.mark();
    }
    CUtensorMap mq, mk, mv;
    const int HD = d->H * DT;
    if (!make_rows_map(&mq, xq, d->B, d->L, HD, ST, DHF) ||
        !make_rows_map(&mk, xk, d->B, d->L, HD, ST, DHF) ||
        !make_rows_map(&mv, xv, d->B, d->L, HD, ST, DHF))
      return DELTANET_ERR_CUDA;
    dim3 grid(a.B * a.H, (d->L + TILE_T - 1) / TILE_T, 6);
    prologue_fwd_tma_kernel<<<grid, 256, TMA_SMEM, s>>>(mq, mk, mv, a);
    prologue_beta_kernel<__nv_bfloat16><<<296, 256, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  dim3 grid(a.ntile, a.B * a.H, 4);
  if (d->dtype == DELTANET_FP32)
    prologue_fwd_kernel<float><<<grid, 256, 0, s>>>(a);
  else
    prologue_fwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int prologue_bwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                 const void* xb, const float* wq, const float* wk, const float* wv,
                 const void* dq, const void* dk, const void* dv, const void* dbeta, void* dxq,
                 void* dxk, void* dxv, void* dxb, float* dwq, float* dwk, float* dwv,
                 void* ws, cudaStream_t s) {
  ProArgs a = make(d);
  a.xq = xq; a.xk = xk; a.xv = xv; a.xb = xb; a.wq = wq; a.wk = wk; a.wv = wv;
  a.q = const_cast<void*>(dq); a.k = const_cast<void*>(dk); a.v = const_cast<void*>(dv);
  a.beta = const_cast<void*>(dbeta);
  a.dxq = dxq; a.dxk = dxk; a.dxv = dxv; a.dxb = dxb;
  a.dwq = dwq; a.dwk = dwk; a.dwv = dwv;
  a.part = (float*)ws;
  if (d->dtype == DELTANET_BF16 && d->Dk == DT && d->Dv == DT && d->L > 0) {
    static PerDevice attr;
    if (!attr.done()) {
      if (cudaFuncSetAttribute(prologue_bwd_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               TMA_SMEM_B) != cudaSuccess)
        return DELTANET_ERR_CUDA;
      attr.mark();
    }
    CUtensorMap mxq, mxk, mxv, mgq, mgk, mgv;
    const int HD = d->H * DT, BH = d->B * d->H;
    if (!make_rows_map(&mxq, xq, d->B, d->L, HD, STB, DH) ||
        !make_rows_map(&mxk, xk, d->B, d->L, HD, STB, DH) ||
        !make_rows_map(&mxv, xv, d->B, d->L, HD, STB, DH) || !make_head_map(&mgq, dq, BH, d->L) ||
        !make_head_map(&mgk, dk, BH, d->L) || !make_head_map(&mgv, dv, BH, d->L))
      return DELTANET_ERR_CUDA;
    a.ntile = (d->L + TILE_T - 1) / TILE_T;  // <= the workspace's (512-token) tile count
    dim3 grid(BH, a.ntile, 6);
    prologue_bwd_tma_kernel<<<grid, 32 * NWB, TMA_SMEM_B, s>>>(mxq, mxk, mxv, mgq, mgk, mgv, a);
    prologue_beta_bwd_kernel<__nv_bfloat16><<<296, 256, 0, s>>>(a);
    prologue_dw_reduce<<<dim3(16, 3), 256, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
  }
  dim3 grid(a.ntile, a.B * a.H, 4);
  if (d->dtype == DELTANET_FP32)
    prologue_bwd_kernel<float><<<grid, 256, 0, s>>>(a);
  else
    prologue_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a);
  prologue_dw_reduce<<<dim3(16, 3), 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

}  // namespace dn
