// simt.cu -- generic CUDA-core path of the chunkwise DeltaNet layer.
//
// One CTA per (b, h) unit walks the chunks of PAPER.md §3.2 exactly as
// Listing 1 (lines 1085-1118) does, in fp32 FFMA arithmetic: per chunk the
// UT transform (Eq. 10-11; forward substitution, line 249), then
// Eq. 8-9 (lines 166-168).  The backward is the chunked reverse sweep of
// DESIGN.md §Backward (the paper gives none; reading R12), with the chunk
// states H_t taken from the workspace (written by the forward) or
// recomputed by a forward sweep inside the same kernel.
//
// This path serves fp32 I/O (tensor-core tf32 cannot meet the 1e-4 bar;
// SURVEY App. B) and every shape the tcgen05 path does not cover.
// Intermediates live in a per-unit global scratch (L2-resident); it is a
// correctness path, not the throughput path.
//
// Gated DeltaNet (R23; oracle/forms.py gated_chunkwise_*): with
// the in-chunk cumulative log-gate G, gamma_i = e^{G_i}, Gamma(i,r) =
// e^{G_i - G_r} (r <= i), D_i = e^{G_{C-1} - G_i}, the chunk step becomes
// X = (I + tril(diag(beta)(Gamma . KK^T), -1))^{-1}, W = X diag(beta gamma) K,
// O = diag(gamma) Q H + (Gamma . tril(QK^T)) U', H <- gamma_C H + (D K)^T U';
// without a gate every factor is exactly 1 and the code skips them.
#include "common.cuh"

namespace dn {
namespace {

struct Scratch {
  float *nq, *nk;             // [L] raw row norms
  float *H, *dH;              // [Dk*Dv]
  float *KK, *A, *Ti, *dA, *dTi, *Gb;  // [C*C]
  float *W, *dqh, *dkh, *dW, *dKb;     // [C*Dk]
  float *U, *dUp, *dVb;                // [C*Dv]
  float *Gc, *dG, *tmp;                // [C] gate: cumulative log-gate, dl/dG, row temp
};

__host__ __device__ inline size_t scratch_floats(int L, int Dk, int Dv, int C) {
  return 2 * (size_t)L + 2 * (size_t)Dk * Dv + 6 * (size_t)C * C +
         5 * (size_t)C * Dk + 3 * (size_t)C * Dv + 3 * (size_t)C + 1;
}

__device__ Scratch carve(float* base, int L, int Dk, int Dv, int C) {
  Scratch s;
  float* p = base;
  s.nq = p; p += L;
  s.nk = p; p += L;
  s.H = p; p += (size_t)Dk * Dv;
  s.dH = p; p += (size_t)Dk * Dv;
  s.KK = p; p += C * C;
  s.A = p; p += C * C;
  s.Ti = p; p += C * C;
  s.dA = p; p += C * C;
  s.dTi = p; p += C * C;
  s.Gb = p; p += C * C;
  s.W = p; p += (size_t)C * Dk;
  s.dqh = p; p += (size_t)C * Dk;
  s.dkh = p; p += (size_t)C * Dk;
  s.dW = p; p += (size_t)C * Dk;
  s.dKb = p; p += (size_t)C * Dk;
  s.U = p; p += (size_t)C * Dv;
  s.dUp = p; p += (size_t)C * Dv;
  s.dVb = p; p += (size_t)C * Dv;
  s.Gc = p; p += C;
  s.dG = p; p += C;
  s.tmp = p; p += C + 1;
  return s;
}

template <typename T>
struct Unit {
  const T *q, *k, *v, *beta, *dO;
  const float* g;  // log-gate of this unit, null = ungated
  int L, Dk, Dv, C;
  bool l2;
  float eps;
  Scratch s;
  // q_hat, k_hat: L2-normalised rows (§3.3; R9),
  // zero past the end (padding, R14).
  __device__ float qh(int t, int m) const {
    if (t >= L) return 0.f;
    float x = ldf(q + (size_t)t * Dk + m);
    return l2 ? x / fmaxf(s.nq[t], eps) : x;
  }
  __device__ float kh(int t, int m) const {
    if (t >= L) return 0.f;
    float x = ldf(k + (size_t)t * Dk + m);
    return l2 ? x / fmaxf(s.nk[t], eps) : x;
  }
  __device__ float vv(int t, int j) const {
    return t < L ? ldf(v + (size_t)t * Dv + j) : 0.f;
  }
  __device__ float bb(int t) const { return t < L ? ldf(beta + t) : 0.f; }
  __device__ float dd(int t, int j) const {
    return t < L ? ldf(dO + (size_t)t * Dv + j) : 0.f;
  }
  // gate factors of the current chunk (s.Gc filled by chunk_gates)
  __device__ float gam(int i) const { return g ? __expf(s.Gc[i]) : 1.f; }
  __device__ float Gam(int i, int r) const {
    return g ? (r <= i ? __expf(s.Gc[i] - s.Gc[r]) : 0.f) : (r <= i ? 1.f : 0.f);
  }
  __device__ float Dn(int i) const { return g ? __expf(s.Gc[C - 1] - s.Gc[i]) : 1.f; }
};

// s.Gc[i] = sum_{j <= i} g[t0 + j] (padding: g = 0)
template <typename T>
__device__ void chunk_gates(const Unit<T>& u, int t0) {
  if (!u.g) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    float acc = 0.f;
    for (int i = 0; i < u.C; ++i) {
      acc += (t0 + i < u.L) ? u.g[t0 + i] : 0.f;
      u.s.Gc[i] = acc;
    }
  }
  __syncthreads();
}

template <typename T>
__device__ void row_norms(Unit<T>& u) {
  for (int t = threadIdx.x; t < u.L; t += blockDim.x) {
    float sq = 0.f, sk = 0.f;
    for (int m = 0; m < u.Dk; ++m) {
      float a = ldf(u.q + (size_t)t * u.Dk + m);
      float b = ldf(u.k + (size_t)t * u.Dk + m);
      sq = fmaf(a, a, sq);
      sk = fmaf(b, b, sk);
    }
    u.s.nq[t] = sqrtf(sq);
    u.s.nk[t] = sqrtf(sk);
  }
}

// Per-chunk state-independent part: KK = K K^T (full), A = tril(Q K^T)
// (inclusive, R4), Ti = (I + tril(diag(beta) K K^T, -1))^{-1} by forward
// substitution (Eq. 10; line 249), W = Ti (beta K), U = Ti (beta V) (Eq. 11).
template <typename T>
__device__ void chunk_ut(const Unit<T>& u, int t0) {
  const int C = u.C, Dk = u.Dk, Dv = u.Dv;
  const Scratch& s = u.s;
  chunk_gates(u, t0);
  for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
    int i = e / C, j = e % C;
    float kk = 0.f, qk = 0.f;
    for (int m = 0; m < Dk; ++m) {
      float kj = u.kh(t0 + j, m);
      kk = fmaf(u.kh(t0 + i, m), kj, kk);
      qk = fmaf(u.qh(t0 + i, m), kj, qk);
    }
    s.KK[e] = kk;
    s.A[e] = (j <= i) ? qk * u.Gam(i, j) : 0.f;
  }
  __syncthreads();
  // column j of Ti: x_i = delta_ij - sum_{j<=m<i} beta_i KK[i][m] x_m
  for (int j = threadIdx.x; j < C; j += blockDim.x) {
    for (int i = 0; i < C; ++i) {
      float x = (i == j) ? 1.f : 0.f;
      if (i > j) {
        const float bi = u.bb(t0 + i);
        for (int m = j; m < i; ++m)
          x = fmaf(-bi * s.KK[i * C + m] * u.Gam(i, m), s.Ti[m * C + j], x);
      }
      s.Ti[i * C + j] = (i < j) ? 0.f : x;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < C * Dk; e += blockDim.x) {
    int i = e / Dk, m = e % Dk;
    float w = 0.f;
    for (int r = 0; r <= i; ++r)
      w = fmaf(s.Ti[i * C + r] * u.bb(t0 + r) * u.gam(r), u.kh(t0 + r, m), w);
    s.W[e] = w;
  }
  for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
    int i = e / Dv, j = e % Dv;
    float x = 0.f;
    for (int r = 0; r <= i; ++r) x = fmaf(s.Ti[i * C + r] * u.bb(t0 + r), u.vv(t0 + r, j), x);
    s.U[e] = x;
  }
  __syncthreads();
}

// U' = U - W H  (Listing 1), in place in s.U.
template <typename T>
__device__ void chunk_uprime(const Unit<T>& u) {
  const int C = u.C, Dk = u.Dk, Dv = u.Dv;
  const Scratch& s = u.s;
  for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
    int i = e / Dv, j = e % Dv;
    float x = s.U[e];
    for (int m = 0; m < Dk; ++m) x = fmaf(-s.W[i * Dk + m], s.H[m * Dv + j], x);
    s.U[e] = x;
  }
  __syncthreads();
}

template <typename T>
__device__ void load_state(const Unit<T>& u, const T* st) {
  for (int e = threadIdx.x; e < u.Dk * u.Dv; e += blockDim.x) u.s.H[e] = ldf(st + e);
  __syncthreads();
}

// Forward sweep of one unit.  o may be null (state recompute only).
template <typename T>
__device__ void unit_forward(const Unit<T>& u, const float* h0, T* o, float* hT,
                             T* states, int NC) {
  const int C = u.C, Dk = u.Dk, Dv = u.Dv, L = u.L;
  const Scratch& s = u.s;
  for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) s.H[e] = h0 ? h0[e] : 0.f;
  __syncthreads();
  for (int c = 0; c < NC; ++c) {
    const int t0 = c * C;
    if (states) {
      T* st = states + (size_t)c * Dk * Dv;
      for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) stf(st + e, s.H[e]);
      // Use exactly the stored (rounded) state, so fwd and bwd see the same H_t.
      __syncthreads();
      for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) s.H[e] = ldf(st + e);
    }
    __syncthreads();
    chunk_ut(u, t0);
    chunk_uprime(u);
    if (o) {
      // O = Q H + tril(Q K^T) U'   (Eq. 9; Listing 1)
      for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
        int i = e / Dv, j = e % Dv;
        if (t0 + i >= L) continue;
        float x = 0.f;
        for (int m = 0; m < Dk; ++m) x = fmaf(u.qh(t0 + i, m), s.H[m * Dv + j], x);
        x *= u.gam(i);
        for (int r = 0; r <= i; ++r) x = fmaf(s.A[i * C + r], s.U[r * Dv + j], x);
        stf(o + (size_t)(t0 + i) * Dv + j, x);
      }
      __syncthreads();  // O reads H_t; the update below overwrites it
    }
    // H += K^T U'   (Eq. 8; Listing 1)
    // gated: H <- gamma_C H + (D K)^T U'
    const float gC = u.gam(C - 1);
    for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) {
      int m = e / Dv, j = e % Dv;
      float x = s.H[e] * gC;
      for (int r = 0; r < C; ++r) x = fmaf(u.kh(t0 + r, m) * u.Dn(r), s.U[r * Dv + j], x);
      s.H[e] = x;
    }
    __syncthreads();
  }
  if (hT)
    for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) hT[e] = s.H[e];
}

template <typename T>
__global__ void __launch_bounds__(256) simt_fwd_kernel(Args a) {
  const size_t unit = blockIdx.x;
  Unit<T> u;
  u.q = (const T*)a.q + unit * a.L * a.Dk;
  u.k = (const T*)a.k + unit * a.L * a.Dk;
  u.v = (const T*)a.v + unit * a.L * a.Dv;
  u.beta = (const T*)a.beta + unit * a.L;
  u.dO = nullptr;
  u.g = a.g ? a.g + unit * a.L : nullptr;
  u.L = a.L; u.Dk = a.Dk; u.Dv = a.Dv; u.C = a.C;
  u.l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  u.eps = a.eps;
  u.s = carve(a.scratch + unit * scratch_floats(a.L, a.Dk, a.Dv, a.C), a.L, a.Dk, a.Dv, a.C);
  row_norms(u);
  __syncthreads();
  const size_t SS = (size_t)a.Dk * a.Dv;
  T* states = (a.flags & DELTANET_SAVE_STATES) ? (T*)a.states + unit * a.NC * SS : nullptr;
  unit_forward(u, a.h0 ? a.h0 + unit * SS : nullptr, (T*)a.o + unit * a.L * a.Dv,
               a.hT ? a.hT + unit * SS : nullptr, states, a.NC);
}

// Chunked reverse sweep.
template <typename T>
__global__ void __launch_bounds__(256) simt_bwd_kernel(Args a) {
  const size_t unit = blockIdx.x;
  const int C = a.C, Dk = a.Dk, Dv = a.Dv, L = a.L;
  Unit<T> u;
  u.q = (const T*)a.q + unit * L * Dk;
  u.k = (const T*)a.k + unit * L * Dk;
  u.v = (const T*)a.v + unit * L * Dv;
  u.beta = (const T*)a.beta + unit * L;
  u.dO = (const T*)a.dO + unit * L * Dv;
  u.g = a.g ? a.g + unit * L : nullptr;
  u.L = L; u.Dk = Dk; u.Dv = Dv; u.C = C;
  u.l2 = (a.flags & DELTANET_L2NORM_QK) != 0;
  u.eps = a.eps;
  u.s = carve(a.scratch + unit * scratch_floats(L, Dk, Dv, C), L, Dk, Dv, C);
  const Scratch& s = u.s;
  const size_t SS = (size_t)Dk * Dv;
  T* states = (T*)a.states + unit * a.NC * SS;
  row_norms(u);
  __syncthreads();
  if (!(a.flags & DELTANET_SAVE_STATES))
    unit_forward(u, a.h0 ? a.h0 + unit * SS : nullptr, (T*)nullptr, nullptr, states, a.NC);
  __syncthreads();
  for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x)
    s.dH[e] = a.dhT ? a.dhT[unit * SS + e] : 0.f;
  __syncthreads();
  T* dq = (T*)a.dq + unit * L * Dk;
  T* dk = (T*)a.dk + unit * L * Dk;
  T* dv = (T*)a.dv + unit * L * Dv;
  T* dbeta = (T*)a.dbeta + unit * L;

  for (int c = a.NC - 1; c >= 0; --c) {
    const int t0 = c * C;
    load_state(u, states + (size_t)c * SS);
    chunk_ut(u, t0);
    chunk_uprime(u);  // s.U = U'
    // 1. dU' = K dH + A^T dO ;  2. dA = tril(dO U'^T)
    for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
      int i = e / Dv, j = e % Dv;
      float x = 0.f;
      for (int m = 0; m < Dk; ++m) x = fmaf(u.kh(t0 + i, m), s.dH[m * Dv + j], x);
      x *= u.Dn(i);
      for (int r = i; r < C; ++r) x = fmaf(s.A[r * C + i], u.dd(t0 + r, j), x);
      s.dUp[e] = x;
    }
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
      int i = e / C, r = e % C;
      float x = 0.f;
      if (r <= i)
        for (int j = 0; j < Dv; ++j) x = fmaf(u.dd(t0 + i, j), s.U[r * Dv + j], x);
      s.dA[e] = x;
    }
    __syncthreads();
    // 3. dQ = dO H^T + dA K ; 4. dK = U' dH^T + dA^T Q ; 5. dW = -dU' H^T
    for (int e = threadIdx.x; e < C * Dk; e += blockDim.x) {
      int i = e / Dk, m = e % Dk;
      float xq = 0.f, xk = 0.f, xw = 0.f;
      for (int j = 0; j < Dv; ++j) {
        float h = s.H[m * Dv + j];
        xq = fmaf(u.dd(t0 + i, j), h, xq);
        xk = fmaf(s.U[i * Dv + j], s.dH[m * Dv + j], xk);
        xw = fmaf(-s.dUp[i * Dv + j], h, xw);
      }
      xq *= u.gam(i);
      xk *= u.Dn(i);
      for (int r = 0; r <= i; ++r) xq = fmaf(s.dA[i * C + r] * u.Gam(i, r), u.kh(t0 + r, m), xq);
      for (int r = i; r < C; ++r) xk = fmaf(s.dA[r * C + i] * u.Gam(r, i), u.qh(t0 + r, m), xk);
      s.dqh[e] = xq;
      s.dkh[e] = xk;
      s.dW[e] = xw;
    }
    __syncthreads();
    if (u.g) {
      // gate, part 1 (dl/dG_i, G the cumulative log-gate): from gamma in
      // diag(gamma) Q H, from D in (D K)^T U', from Gamma in A, and
      // gamma_C <dH, H> from gamma_C H
      for (int i = threadIdx.x; i < C; i += blockDim.x) {
        float qo = 0.f, dd = 0.f;
        for (int m = 0; m < Dk; ++m) {
          float ph = 0.f, pu = 0.f;
          for (int j = 0; j < Dv; ++j) {
            ph = fmaf(u.dd(t0 + i, j), s.H[m * Dv + j], ph);
            pu = fmaf(s.U[i * Dv + j], s.dH[m * Dv + j], pu);
          }
          qo = fmaf(u.qh(t0 + i, m), ph, qo);
          dd = fmaf(u.kh(t0 + i, m), pu, dd);
        }
        float row = 0.f, col = 0.f;
        for (int r = 0; r <= i; ++r) row = fmaf(s.dA[i * C + r], s.A[i * C + r], row);
        for (int r = i; r < C; ++r) col = fmaf(s.dA[r * C + i], s.A[r * C + i], col);
        const float dD = dd * u.Dn(i);
        s.dG[i] = u.gam(i) * qo - dD + row - col;
        s.tmp[i] = dD;
      }
      if (threadIdx.x == 0) s.tmp[C] = 0.f;
      __syncthreads();
      float part = 0.f;
      for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) part = fmaf(s.dH[e], s.H[e], part);
      for (int m = 16; m > 0; m >>= 1) part += __shfl_xor_sync(0xffffffffu, part, m);
      if ((threadIdx.x & 31) == 0) atomicAdd(&s.tmp[C], part);
      __syncthreads();
      if (threadIdx.x == 0) {
        float x = u.gam(C - 1) * s.tmp[C];
        for (int i = 0; i < C; ++i) x += s.tmp[i];
        s.dG[C - 1] += x;
      }
      __syncthreads();
    }
    // 6. dH += Q^T dO - W^T dU'   (gated: dH <- gamma_C dH + (gamma Q)^T dO - W^T dU')
    const float gC = u.gam(C - 1);
    for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) {
      int m = e / Dv, j = e % Dv;
      float x = s.dH[e] * gC;
      for (int i = 0; i < C; ++i)
        x = fmaf(u.qh(t0 + i, m) * u.gam(i), u.dd(t0 + i, j),
                 fmaf(-s.W[i * Dk + m], s.dUp[i * Dv + j], x));
      s.dH[e] = x;
    }
    // 7. dTi = dW (beta K)^T + dU' (beta V)^T
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
      int i = e / C, r = e % C;
      float x = 0.f;
      for (int m = 0; m < Dk; ++m) x = fmaf(s.dW[i * Dk + m], u.kh(t0 + r, m), x);
      x *= u.gam(r);
      for (int j = 0; j < Dv; ++j) x = fmaf(s.dUp[i * Dv + j], u.vv(t0 + r, j), x);
      s.dTi[e] = x * u.bb(t0 + r);
    }
    __syncthreads();
    // 8/9. dKb = Ti^T dW, dVb = Ti^T dU' ; 13a. tmp = Ti^T dTi (into dA)
    for (int e = threadIdx.x; e < C * Dk; e += blockDim.x) {
      int r = e / Dk, m = e % Dk;
      float x = 0.f;
      for (int i = r; i < C; ++i) x = fmaf(s.Ti[i * C + r], s.dW[i * Dk + m], x);
      s.dKb[e] = x;
    }
    for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
      int r = e / Dv, j = e % Dv;
      float x = 0.f;
      for (int i = r; i < C; ++i) x = fmaf(s.Ti[i * C + r], s.dUp[i * Dv + j], x);
      s.dVb[e] = x;
    }
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
      int i = e / C, r = e % C;
      float x = 0.f;
      for (int p = i; p < C; ++p) x = fmaf(s.Ti[p * C + i], s.dTi[p * C + r], x);
      s.dA[e] = x;
    }
    __syncthreads();
    // 13b. Gb = tril(-(Ti^T dTi) Ti^T, -1)
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
      int i = e / C, r = e % C;
      float x = 0.f;
      if (r < i)
        for (int p = 0; p <= r; ++p) x = fmaf(-s.dA[i * C + p], s.Ti[r * C + p], x);
      s.Gb[e] = x;
    }
    // 11. dV = beta dVb (final)
    for (int e = threadIdx.x; e < C * Dv; e += blockDim.x) {
      int i = e / Dv, j = e % Dv;
      if (t0 + i < L) stf(dv + (size_t)(t0 + i) * Dv + j, u.bb(t0 + i) * s.dVb[e]);
    }
    __syncthreads();
    // 10/15. dK += beta dKb + (beta Gb) K + (beta Gb)^T K
    for (int e = threadIdx.x; e < C * Dk; e += blockDim.x) {
      int i = e / Dk, m = e % Dk;
      const float bi = u.bb(t0 + i);
      float x = s.dkh[e] + bi * u.gam(i) * s.dKb[e];
      for (int r = 0; r < i; ++r)
        x = fmaf(bi * s.Gb[i * C + r] * u.Gam(i, r), u.kh(t0 + r, m), x);
      for (int r = i + 1; r < C; ++r)
        x = fmaf(u.bb(t0 + r) * s.Gb[r * C + i] * u.Gam(r, i), u.kh(t0 + r, m), x);
      s.dkh[e] = x;
    }
    // 12/14. dbeta = rowsum(dKb . K) + rowsum(dVb . V) + rowsum(Gb . KK)
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
      if (t0 + i >= L) continue;
      float rk = 0.f, x = 0.f;
      for (int m = 0; m < Dk; ++m) rk = fmaf(s.dKb[i * Dk + m], u.kh(t0 + i, m), rk);
      for (int j = 0; j < Dv; ++j) x = fmaf(s.dVb[i * Dv + j], u.vv(t0 + i, j), x);
      x = fmaf(u.gam(i), rk, x);
      for (int r = 0; r < i; ++r) x = fmaf(s.Gb[i * C + r] * u.Gam(i, r), s.KK[i * C + r], x);
      stf(dbeta + t0 + i, x);
    }
    if (u.g) {
      // gate, part 2: gamma in W's diag(beta gamma), Gamma in the UT matrix;
      // then dg = reverse cumulative sum of dl/dG within the chunk
      for (int i = threadIdx.x; i < C; i += blockDim.x) {
        const float bi = u.bb(t0 + i);
        float rk = 0.f, row = 0.f, col = 0.f;
        for (int m = 0; m < Dk; ++m) rk = fmaf(s.dKb[i * Dk + m], u.kh(t0 + i, m), rk);
        for (int r = 0; r < i; ++r)
          row = fmaf(bi * s.Gb[i * C + r] * u.Gam(i, r), s.KK[i * C + r], row);
        for (int r = i + 1; r < C; ++r)
          col = fmaf(u.bb(t0 + r) * s.Gb[r * C + i] * u.Gam(r, i), s.KK[r * C + i], col);
        s.dG[i] += bi * u.gam(i) * rk + row - col;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        float acc = 0.f;
        for (int i = C - 1; i >= 0; --i) {
          acc += s.dG[i];
          if (t0 + i < L && a.dg) a.dg[unit * L + t0 + i] = acc;
        }
      }
    }
    __syncthreads();
    // L2-norm adjoint (R9): dx = (dxh - xh (xh . dxh)) / ||x|| if ||x|| >= eps
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
      const int t = t0 + i;
      if (t >= L) continue;
      if (u.l2) {
        float sq = 0.f, sk = 0.f;
        for (int m = 0; m < Dk; ++m) {
          sq = fmaf(u.qh(t, m), s.dqh[i * Dk + m], sq);
          sk = fmaf(u.kh(t, m), s.dkh[i * Dk + m], sk);
        }
        const float nq = s.nq[t], nk = s.nk[t];
        for (int m = 0; m < Dk; ++m) {
          float gq = nq >= u.eps ? (s.dqh[i * Dk + m] - u.qh(t, m) * sq) / nq
                                 : s.dqh[i * Dk + m] / u.eps;
          float gk = nk >= u.eps ? (s.dkh[i * Dk + m] - u.kh(t, m) * sk) / nk
                                 : s.dkh[i * Dk + m] / u.eps;
          stf(dq + (size_t)t * Dk + m, gq);
          stf(dk + (size_t)t * Dk + m, gk);
        }
      } else {
        for (int m = 0; m < Dk; ++m) {
          stf(dq + (size_t)t * Dk + m, s.dqh[i * Dk + m]);
          stf(dk + (size_t)t * Dk + m, s.dkh[i * Dk + m]);
        }
      }
    }
    __syncthreads();
  }
  if (a.dh0)
    for (int e = threadIdx.x; e < Dk * Dv; e += blockDim.x) a.dh0[unit * SS + e] = s.dH[e];
}

}  // namespace

size_t simt_scratch_floats_per_unit(int L, int Dk, int Dv, int C) {
  return scratch_floats(L, Dk, Dv, C);
}

int simt_fwd(const Args& a, int dtype, cudaStream_t s) {
  const unsigned units = (unsigned)(a.B * a.H);
  if (units == 0) return DELTANET_OK;
  if (dtype == DELTANET_FP32)
    simt_fwd_kernel<float><<<units, 256, 0, s>>>(a);
  else
    simt_fwd_kernel<__nv_bfloat16><<<units, 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int simt_bwd(const Args& a, int dtype, cudaStream_t s) {
  const unsigned units = (unsigned)(a.B * a.H);
  if (units == 0) return DELTANET_OK;
  if (dtype == DELTANET_FP32)
    simt_bwd_kernel<float><<<units, 256, 0, s>>>(a);
  else
    simt_bwd_kernel<__nv_bfloat16><<<units, 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DELTANET_OK : DELTANET_ERR_CUDA;
}

}  // namespace dn
