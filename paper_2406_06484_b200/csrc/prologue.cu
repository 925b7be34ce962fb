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
// Tiling: a thread owns 8 consecutive channels (one 16 B bf16 vector) and a
// run of RUN = 32 tokens, sliding a 4-token window; a CTA is 16 channel
// groups x 16 runs = 256 threads over 512 tokens of one (b, h, tensor).  The
// backward recomputes y, forms dy = dout * act'(y), dx[t] = sum_j w[j]
// dy[t+3-j], and per-CTA partial dw sums that a second kernel reduces in a
// fixed order (deterministic, no atomics).
#include "common.cuh"

namespace dn {
namespace {

constexpr int RUN = 32, RUNS = 16, TT = RUN * RUNS;  // tokens per thread / CTA

template <typename T>
__device__ __forceinline__ void store8(T* p, const float (&x)[8]);
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float (&x)[8]) {
  uint4 v;
  uint32_t* u = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
    u[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = v;
}
template <>
__device__ __forceinline__ void store8<float>(float* p, const float (&x)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(x[4], x[5], x[6], x[7]);
}

// 8 elements as raw 16 B words (bf16: one uint4, fp32: two), so that several
// tokens' loads can be in flight before any is unpacked
template <typename T>
struct Raw8 {
  uint4 w[sizeof(T) / 2];
};
template <typename T>
__device__ __forceinline__ void load_raw(const T* p, Raw8<T>& r) {
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 2); ++i) r.w[i] = reinterpret_cast<const uint4*>(p)[i];
}
template <typename T>
__device__ __forceinline__ void unpack(const Raw8<T>& r, float (&x)[8]);
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const Raw8<__nv_bfloat16>& r, float (&x)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.w[0]);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void unpack<float>(const Raw8<float>& r, float (&x)[8]) {
  const float* f = reinterpret_cast<const float*>(&r.w[0]);
#pragma unroll
  for (int e = 0; e < 8; ++e) x[e] = f[e];
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&x)[8]) {
  Raw8<T> r;
  load_raw(p, r);
  unpack(r, x);
}

constexpr int UNR = 4;  // tokens loaded ahead per iteration

__device__ __forceinline__ float sigm(float y) { return 1.f / (1.f + __expf(-y)); }

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

// grid (ntile, B*H, 4): z < 3 conv + activation of q / k / v, z == 3 beta
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
  const int run = threadIdx.x / RUNS;  // token run
  const int t0 = t_begin + run * RUN;
  if (t0 >= L) return;
  // channel groups of 8: 16 per pass (D = 256 takes two passes)
  for (int cg = threadIdx.x % RUNS; 8 * cg < D; cg += RUNS) {
  const int c = h * D + 8 * cg;  // first channel of this thread
  const T* x = (const T*)tz.x + (size_t)b * L * H * D + c;   // token stride H * D
  T* y = (T*)tz.y + ((size_t)b * H + h) * L * D + 8 * cg;     // token stride D
  float w[8][4];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) w[e][j] = tz.w[(size_t)(c + e) * 4 + j];
  float win[3][8];  // x[t-3], x[t-2], x[t-1]
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int t = t0 - 3 + j;
    if (t >= 0) {
      load8(x + (size_t)t * H * D, win[j]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) win[j][e] = 0.f;
    }
  }
  const int t1 = min(L, t0 + RUN);
  for (int tb = t0; tb < t1; tb += UNR) {
    Raw8<T> raw[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (tb + u < t1) load_raw(x + (size_t)(tb + u) * H * D, raw[u]);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (tb + u >= t1) break;
      float xt[8], o[8];
      unpack(raw[u], xt);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float yy = fmaf(w[e][0], win[0][e],
                              fmaf(w[e][1], win[1][e], fmaf(w[e][2], win[2][e], w[e][3] * xt[e])));
        o[e] = tz.silu ? yy * sigm(yy) : yy;
        win[0][e] = win[1][e];
        win[1][e] = win[2][e];
        win[2][e] = xt[e];
      }
      store8(y + (size_t)(tb + u) * D, o);
    }
  }
  }
}

// backward: dy = dout * act'(y); dx[t] = sum_j w[j] dy[t+3-j]; partial dw.
template <typename T>
__global__ void __launch_bounds__(256) prologue_bwd_kernel(ProArgs a) {
  __shared__ float red[RUNS][RUNS * 8 * 4 + 4];  // [run][cg*32 + e*4 + j]
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
  const int run = threadIdx.x / RUNS;
  const int t0 = t_begin + run * RUN;
  const int npass = D > 8 * RUNS ? D / (8 * RUNS) : 1;  // 16 channel groups per pass
  for (int pass = 0; pass < npass; ++pass) {
  const int cg = threadIdx.x % RUNS + RUNS * pass;
  const bool active = 8 * cg < D && t0 < L;
  float dw[8][4];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) dw[e][j] = 0.f;
  if (active) {
    const int c = h * D + 8 * cg;
    const T* x = (const T*)tz.x + (size_t)b * L * H * D + c;
    const T* g = (const T*)tz.y + ((size_t)b * H + h) * L * D + 8 * cg;  // dout
    T* dx = (T*)tz.dx + (size_t)b * L * H * D + c;
    float w[8][4];
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int j = 0; j < 4; ++j) w[e][j] = tz.w[(size_t)(c + e) * 4 + j];
    float xw[4][8];   // x[t-3..t]
    float dyw[3][8];  // dy[t-3], dy[t-2], dy[t-1]
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int t = t0 - 3 + j;
      if (t >= 0) {
        load8(x + (size_t)t * H * D, xw[j + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xw[j + 1][e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) dyw[j][e] = 0.f;
    }
    const int t1 = min(L, t0 + RUN);
    const int tend = min(L, t1 + 3);  // dy needed up to t1 + 2 for dx[t1 - 1]
    for (int tb = t0; tb < tend; tb += UNR) {
    Raw8<T> rx[UNR], rg[UNR];
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
      float xt[8], gt[8], dyt[8];
      unpack(rx[u], xt);
      unpack(rg[u], gt);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
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
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          o[e] = fmaf(w[e][3], dyw[0][e],
                      fmaf(w[e][2], dyw[1][e], fmaf(w[e][1], dyw[2][e], w[e][0] * dyt[e])));
        store8(dx + (size_t)(t - 3) * H * D, o);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
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
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // dy[s + 3 - j] at dyw index k0 + 3 - j (< 3)
          const int idx = k0 + 3 - j;  // selects, not a dynamic register index
          const float dv = idx == 0 ? dyw[0][e] : idx == 1 ? dyw[1][e] : idx == 2 ? dyw[2][e] : 0.f;
          acc = fmaf(w[e][j], dv, acc);
        }
        o[e] = acc;
      }
      store8(dx + (size_t)s * H * D, o);
    }
  }
  // per-CTA dw partial: sum over the 16 runs in a fixed order
  __syncthreads();  // the previous pass finished reading red
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[run][(cg % RUNS) * 32 + e * 4 + j] = dw[e][j];
  __syncthreads();
  for (int i = threadIdx.x; i < RUNS * 32; i += blockDim.x) {
    const int cgi = i / 32 + RUNS * pass;
    if (8 * cgi >= D) continue;
    float s = 0.f;
    for (int r = 0; r < RUNS; ++r) s += red[r][i];
    // part[z][b * ntile + tile][h * D + 8 cgi + e][j]
    const int Dm = a.Dk > a.Dv ? a.Dk : a.Dv;
    const size_t slot = ((size_t)z * a.B * a.ntile + (size_t)b * a.ntile + tile);
    a.part[(slot * H * Dm + (size_t)h * D + 8 * cgi) * 4 + (i % 32)] = s;
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
  dim3 grid(a.ntile, a.B * a.H, 4);
  if (d->dtype == DELTANET_FP32)
    prologue_bwd_kernel<float><<<grid, 256, 0, s>>>(a);
  else
    prologue_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a);
  prologue_dw_reduce<<<dim3(16, 3), 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

}  // namespace dn
