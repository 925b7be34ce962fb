/*
 * deltanet.h -- C ABI of the B200 (sm_100a) DeltaNet chunkwise delta-rule
 * layer library, libdeltanet.so.  Forward and backward of one layer over
 * q, k, v, beta of shape [B, H, L, d].
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md, arXiv 2406.06484):
 *   per (b, h) unit, with q, k optionally L2-normalised (§3.3),
 *     S_t = S_{t-1} - beta_t (S_{t-1} k_t - v_t) k_t^T,  o_t = S_t q_t
 *   (§2.2 lines 82-97), evaluated by the chunkwise-parallel algorithm of §3.2:
 *   per chunk of C tokens the UT transform (Eq. 10-11)
 *     T = (I + tril(diag(beta) K K^T, -1))^{-1} diag(beta),  W = T K,  U = T V
 *   then the state recurrence and output (Eq. 8-9)
 *     S <- S + (U - W S^T)^T K,   O = Q S^T + (Q K^T (.) M)(U - W S^T)
 *   with M the inclusive causal mask (Listing 1; R4).
 *   The backward (not given in the paper; R12) is the exact
 *   adjoint of that map.
 *
 * Conventions
 *  - Every tensor pointer is DEVICE memory owned by the caller, contiguous,
 *    row-major, 16-byte aligned (MISALIGNED otherwise).  The library never
 *    allocates or frees, never synchronises the host, and keeps no mutable
 *    global state except once-per-device kernel attributes; calls on
 *    different streams are independent.
 *  - Layouts: q, k [B,H,L,Dk]; v, o, dO [B,H,L,Dv]; beta [B,H,L];
 *    states h0, hT, dhT, dh0 [B,H,Dk,Dv] in the orientation H = S^T
 *    (R2; Listing 1's S).  I/O tensors have the descriptor dtype;
 *    states are always fp32.  Accumulation is always fp32.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Errors: argument errors are detected before any launch and nothing is
 *    written; a launch failure returns DELTANET_ERR_CUDA; asynchronous device
 *    faults surface at the caller's next synchronisation.  No exception
 *    crosses the ABI.
 *  - L need not be a multiple of chunk: the tail chunk is processed with the
 *    missing tokens treated as beta = 0, zero rows (an exact no-op; R14).
 */
#ifndef DELTANET_H
#define DELTANET_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DELTANET_ABI_VERSION 8

typedef enum {
  DELTANET_BF16 = 0, /* bf16 I/O, fp32 accumulation (BASELINE.json north_star) */
  DELTANET_FP32 = 1  /* fp32 I/O, fp32 CUDA-core arithmetic (parity mode)     */
} deltanet_dtype;

enum {
  /* q <- q / max(||q||_2, eps), same for k, inside the kernel (§3.3
   * lines 329-331; R9/R10).  Gradients are w.r.t. the RAW q, k. */
  DELTANET_L2NORM_QK = 1u << 0,
  /* fwd: write the chunk-boundary states H_t into the workspace so the bwd
   * does not recompute them (§3.2 line 250 recomputes them; we
   * store them -- DESIGN.md "Differences from the paper").  The tcgen05
   * path also stores a 32.5 KB per-chunk record (X, Z^T, the q/k row
   * norms, A = tril(QK^T)) so the bwd skips the UT
   * substitution, the norm passes and the QK^T product.
   * bwd: the workspace holds what a fwd with this flag over the same inputs
   * and the same desc wrote. */
  DELTANET_SAVE_STATES = 1u << 1,
  /* run the generic CUDA-core (SIMT) kernels even where the tcgen05 path
   * applies, and allow bf16 descriptors outside the tcgen05 shapes (without
   * this flag those are DELTANET_ERR_UNSUPPORTED: the CUDA-core kernels run
   * 10^3-10^4x below the tensor-core roofline, so they are never chosen
   * silently).  fp32 I/O always runs on them.  No CPU fallback exists. */
  DELTANET_FORCE_SIMT = 1u << 2,
  /* layer prologue only: SiLU on v as well (the paper states SiLU for q, k
   * only; R22) */
  DELTANET_PROLOGUE_SILU_V = 1u << 3,
  /* tcgen05 forward: never split a unit's sequence into segments processed
   * by several CTAs (the segment-parallel forward, is used
   * automatically when B*H is small against the SM count) */
  DELTANET_NO_SEGMENTS = 1u << 4,
  /* Gated DeltaNet (set internally by the deltanet_gated_* calls; set it in
   * the descriptor passed to deltanet_workspace_bytes / deltanet_path /
   * deltanet_launch_count to query the gated calls) */
  DELTANET_GATED = 1u << 5,
  /* run the tcgen05 "split" kernels (chunk-parallel prep + per-d_v-block
   * state chains + chunk-parallel local gradients) at
   * Dk = Dv = 128 too, where the fused one-CTA-per-unit kernels are the
   * default (cross-checking and measurement).  Dk = Dv in {64, 256} always
   * run the split kernels. */
  DELTANET_FORCE_SPLIT = 1u << 6,
  /* fused tcgen05 kernels (d = 128): round the bf16 operands that are
   * summed over tokens (Z = diag(s) U' in the forward, the U' record and dA
   * in the backward) with the rounding error carried along the token axis
   * (compensated rounding).  Prefix sums then carry ~2 roundings instead of
   * ~sqrt(C); it matters where those sums telescope (e.g. many identical
   * keys with beta = 1, R19) and costs ~7% of a fwd+bwd step.
   * Set it for both deltanet_fwd and deltanet_bwd (the record differs). */
  DELTANET_COMPENSATED = 1u << 7
};

typedef struct {
  int B, H, L;      /* batch, heads, sequence length (>= 0)                  */
  int Dk, Dv;       /* head dims, each in {16, 32, 64, 128, 256}             */
  int chunk;        /* C in {16, 32, 64, 128}             */
  int dtype;        /* deltanet_dtype                                        */
  unsigned flags;   /* DELTANET_* bits                                       */
  float l2_eps;     /* eps of the L2 normalisation; <= 0 selects 1e-6 (R9)   */
} deltanet_desc;

/* Error codes. */
#define DELTANET_OK 0
#define DELTANET_ERR_INVALID_ARG 1 /* null required pointer, negative size   */
#define DELTANET_ERR_UNSUPPORTED 2 /* Dk/Dv/chunk/dtype outside the table, or
                                      bf16 outside the tcgen05 shapes without
                                      DELTANET_FORCE_SIMT                     */
#define DELTANET_ERR_MISALIGNED 3  /* a pointer not 16-byte aligned          */
#define DELTANET_ERR_CUDA 4        /* cudaGetLastError() after a launch      */
#define DELTANET_ERR_WORKSPACE 5   /* workspace NULL or smaller than needed  */

/* Bytes of device workspace both deltanet_fwd and deltanet_bwd need for this
 * descriptor (the chunk-boundary states, B*H*ceil(L/C)*Dk*Dv elements of the
 * I/O dtype, plus kernel scratch).  0 for an invalid descriptor. */
size_t deltanet_workspace_bytes(const deltanet_desc* d);

/* Forward.  q, k, v, beta: inputs; h0: nullable initial state (else 0);
 * o: output [B,H,L,Dv]; hT: nullable final state; workspace: device buffer
 * of at least deltanet_workspace_bytes(d) bytes (states are written there
 * when DELTANET_SAVE_STATES is set). */
int deltanet_fwd(const deltanet_desc* d, const void* q, const void* k,
                 const void* v, const void* beta, const float* h0, void* o,
                 float* hT, void* workspace, size_t workspace_bytes,
                 void* stream);

/* Backward.  dO: cotangent of o; dhT: nullable cotangent of hT (else 0).
 * Outputs dq, dk [B,H,L,Dk], dv [B,H,L,Dv], dbeta [B,H,L] in the I/O dtype
 * (w.r.t. the raw inputs), dh0 nullable [B,H,Dk,Dv] fp32.  With
 * DELTANET_SAVE_STATES the workspace must hold the states written by a
 * deltanet_fwd over the same inputs; otherwise they are recomputed. */
int deltanet_bwd(const deltanet_desc* d, const void* q, const void* k,
                 const void* v, const void* beta, const float* h0,
                 const void* dO, const float* dhT, void* dq, void* dk,
                 void* dv, void* dbeta, float* dh0, void* workspace,
                 size_t workspace_bytes, void* stream);

/* Forward + backward of HOST-resident tensors (the same layouts, in pinned
 * host memory for copy/compute overlap): the B*H (b, h) units are cut into
 * `slabs` consecutive unit ranges (each a descriptor with B = units, H = 1)
 * that flow through a three-stream pipeline inside the library --
 * H2D of slab i+1, deltanet_fwd + deltanet_bwd (with
 * DELTANET_SAVE_STATES) of slab i, D2H of slab i-1 -- through two
 * ping-pong device buffers carved from dev_buffer (at least
 * deltanet_fwd_bwd_host_device_bytes(d, slabs) bytes).  Writes o, dq, dk,
 * dv, dbeta (host); h0 / hT / dh0 are not exposed here (zero / unused).
 * Asynchronous: `stream` (the caller's) is made to wait for the last
 * read-out, so a synchronisation of it makes the host outputs valid; the
 * internal streams and events are created and released per call.  Same
 * error codes; WORKSPACE if dev_buffer is missing or small. */
int deltanet_fwd_bwd_host(const deltanet_desc* d, const void* q,
                          const void* k, const void* v, const void* beta,
                          const void* dO, void* o, void* dq, void* dk, void* dv,
                          void* dbeta, int slabs, void* dev_buffer,
                          size_t dev_bytes, void* stream);

/* Device bytes deltanet_fwd_bwd_host needs for this descriptor and slab
 * count (slabs > B*H counts as B*H); 0 for an invalid descriptor. */
size_t deltanet_fwd_bwd_host_device_bytes(const deltanet_desc* d, int slabs);

/* Recurrent (token-by-token) form, for inference / decode:
 * the delta rule of PAPER.md §2.2 applied one token at a time,
 *   S_t = S_{t-1} - beta_t (S_{t-1} k_t - v_t) k_t^T,  o_t = S_t q_t,
 * in the kernel orientation H = S^T, fp32 state, with q, k L2-normalised
 * under DELTANET_L2NORM_QK.  Same tensors and layouts as
 * deltanet_fwd; d->chunk is ignored and no workspace is used.  h0 nullable
 * (zeros); hT nullable; h0 == hT is allowed (in-place state update, the
 * decode loop).  No backward (inference only).  Same error codes. */
int deltanet_recurrent_fwd(const deltanet_desc* d, const void* q,
                           const void* k, const void* v, const void* beta,
                           const float* h0, void* o, float* hT, void* stream);

/* Layer prologue: the steps in front of the chunkwise
 * kernel in a DeltaNet layer.  After the q/k/v projections a causal depthwise
 * short convolution of width 4 (§3.4), the SiLU
 * feature map on q and k (their L2 normalisation is fused into the
 * chunkwise kernels), beta = sigmoid(W_beta x):
 *   y[t] = sum_{j<4} w[c][j] x[t-3+j]  (x[t<0] = 0);  q = SiLU(y_q),
 *   k = SiLU(y_k), v = y_v (SiLU too with DELTANET_PROLOGUE_SILU_V),
 *   beta = sigmoid(xb).
 * Inputs in the projections' token-major layout: xq, xk [B, L, H, Dk],
 * xv [B, L, H, Dv], xb [B, L, H] (I/O dtype); weights wq, wk [H*Dk][4],
 * wv [H*Dv][4] fp32 (channel c = h*D + d).  Outputs in the deltanet_fwd
 * layout: q, k [B,H,L,Dk], v [B,H,L,Dv], beta [B,H,L].  d->chunk ignored. */
int deltanet_prologue_fwd(const deltanet_desc* d, const void* xq,
                          const void* xk, const void* xv, const void* xb,
                          const float* wq, const float* wk, const float* wv,
                          void* q, void* k, void* v, void* beta, void* stream);

/* Device workspace deltanet_prologue_bwd needs (per-block partial sums of
 * the weight gradients; 0 for an invalid descriptor). */
size_t deltanet_prologue_workspace_bytes(const deltanet_desc* d);

/* Backward of the prologue: dq, dk, dv, dbeta are the cotangents of its
 * outputs (what deltanet_bwd returns); writes dxq, dxk, dxv, dxb (layouts of
 * xq ... xb) and overwrites dwq, dwk, dwv (fp32, reduced over B and L in a
 * fixed order: deterministic). */
int deltanet_prologue_bwd(const deltanet_desc* d, const void* xq,
                          const void* xk, const void* xv, const void* xb,
                          const float* wq, const float* wk, const float* wv,
                          const void* dq, const void* dk, const void* dv,
                          const void* dbeta, void* dxq, void* dxk, void* dxv,
                          void* dxb, float* dwq, float* dwk, float* dwv,
                          void* workspace, size_t workspace_bytes, void* stream);

/* ---- Gated DeltaNet (R23) ----
 * The recurrence of PAPER.md Table tab:overview,
 *   S_t = S_{t-1} (alpha_t (I - beta_t k_t k_t^T)) + beta_t v_t k_t^T,
 *   o_t = S_t q_t,   alpha_t = exp(g_t),
 * with g [B,H,L] the per-token log-decay, fp32 whatever the I/O dtype
 * (g <= 0 for a decay; any finite g is accepted).  Same tensors, layouts,
 * flags and error codes as deltanet_fwd / deltanet_bwd plus g and dg
 * ([B,H,L] fp32, the gradient w.r.t. g).  The workspace must be at least
 * deltanet_workspace_bytes of the descriptor with DELTANET_GATED set.
 * g = NULL is the ungated layer. */
int deltanet_gated_fwd(const deltanet_desc* d, const void* q, const void* k,
                       const void* v, const void* beta, const float* g,
                       const float* h0, void* o, float* hT, void* workspace,
                       size_t workspace_bytes, void* stream);

int deltanet_gated_bwd(const deltanet_desc* d, const void* q, const void* k,
                       const void* v, const void* beta, const float* g,
                       const float* h0, const void* dO, const float* dhT,
                       void* dq, void* dk, void* dv, void* dbeta, float* dg,
                       float* dh0, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Recurrent (token-by-token) gated forward for inference / decode; as
 * deltanet_recurrent_fwd plus g (nullable). */
int deltanet_gated_recurrent_fwd(const deltanet_desc* d, const void* q,
                                 const void* k, const void* v,
                                 const void* beta, const float* g,
                                 const float* h0, void* o, float* hT,
                                 void* stream);

/* ---- Context parallelism ----
 * A sequence split into P consecutive parts (one per GPU, or per call) is
 * processed part-locally, with the parts' boundary states stitched by the
 * affine composition of the per-chunk state update (§3.2 Eq. 8,
 * line 166: S_{t+1} = S_t (I - W_t^T K_t) + U_t^T K_t).  Over a part p the
 * composition is, in the orientation H = S^T,
 *   H_end = Psi_p^T H_start + Hloc_p,   Psi_p = prod_t (I - W_t^T K_t) [Dk,Dk]
 * (the product over the part's chunks in order; Hloc_p the part's end state
 * from H_start = 0), and the backward's cotangent chain is its adjoint,
 *   dH_start = Psi_p dH_end + dHloc_p
 * (dHloc_p = dl/dH_start of the part with dH_end = 0).  A context-parallel
 * fwd is: deltanet_fwd_transition on each part; gather (Psi, Hloc) of all
 * parts (e.g. NCCL all_gather); deltanet_state_scan(part, reverse=0) gives
 * the part's H_start; deltanet_fwd with h0 = H_start.  The bwd:
 * deltanet_bwd_transition; gather dHloc; deltanet_state_scan(reverse=1)
 * gives dhT of the part; deltanet_bwd with h0 = H_start, dhT = that.
 * These three calls need the tcgen05 path's shapes (bf16, Dk = Dv = 128,
 * chunk 64, no DELTANET_FORCE_SIMT; else UNSUPPORTED); L = 0 is allowed
 * (Psi = I, Hloc = 0).  Psi and the states are fp32; a part's Psi, Hloc,
 * dHloc have the layout [B,H,128,128] (row i of Psi = row i of the matrix). */

/* Psi [B,H,Dk,Dk] and Hloc [B,H,Dk,Dv] of this call's sequence.  One
 * launch, or (when B*H leaves SMs idle, as deltanet_fwd's segments) the
 * segment-parallel pass 1 plus a composition launch; the workspace
 * (deltanet_workspace_bytes(d)) holds the segment scratch.  Nothing the
 * backward needs is written there. */
int deltanet_fwd_transition(const deltanet_desc* d, const void* q,
                            const void* k, const void* v, const void* beta,
                            float* psi, float* hloc, void* workspace,
                            size_t workspace_bytes, void* stream);

/* dHloc [B,H,Dk,Dv] of this call's sequence for the cotangent dO.  The
 * workspace (deltanet_workspace_bytes(d)) must hold what deltanet_fwd with
 * DELTANET_SAVE_STATES wrote over the same q, k, v, beta (any h0) when the
 * flag is set (its per-chunk records and, when segmented, its segment
 * transitions); without the flag they are recomputed into it. */
int deltanet_bwd_transition(const deltanet_desc* d, const void* q,
                            const void* k, const void* v, const void* beta,
                            const void* dO, float* dhloc, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Boundary state of part `part` of nparts from the gathered transitions
 * psi_all [nparts][B,H,Dk,Dk] and loc_all [nparts][B,H,Dk,Dv] (fp32):
 *   reverse = 0: out = H_start(part) = fold over p = 0 .. part-1 of
 *                H <- Psi_p^T H + Hloc_p, from H = edge (h0; NULL = 0);
 *   reverse = 1: out = dH_end(part) = fold over p = nparts-1 down to part+1
 *                of G <- Psi_p G + dHloc_p, from G = edge (dhT; NULL = 0).
 * out [B,H,Dk,Dv] may alias edge.  fp32 CUDA-core arithmetic. */
int deltanet_state_scan(const deltanet_desc* d, int nparts, int part,
                        int reverse, const float* psi_all,
                        const float* loc_all, const float* edge, float* out,
                        void* stream);

/* Which kernel family a descriptor dispatches to: 1 = fused tcgen05/TMEM/TMA
 * sm_100a kernels (one CTA per (b, h) unit), 2 = split tcgen05 kernels
 * (DESIGN.md §4.10), 0 = CUDA-core (SIMT) path, -1 = unsupported descriptor.
 * The fused path serves bf16 I/O with chunk = 64 and Dk = Dv = 128
 * (ungated and gated; BASELINE configs 1, 2, 4 and the target); the split
 * path bf16, chunk = 64, ungated, Dk = Dv in {64, 256} (configs 3) and, with
 * DELTANET_FORCE_SPLIT, 128.  fp32 I/O and (with DELTANET_FORCE_SIMT only)
 * other bf16 shapes run on the CUDA-core kernels; any other bf16 descriptor
 * is -1 (UNSUPPORTED). */
int deltanet_path(const deltanet_desc* d);

/* Number of kernel launches deltanet_fwd (which=0), deltanet_bwd (which=1),
 * deltanet_recurrent_fwd (2), deltanet_prologue_fwd (3),
 * deltanet_prologue_bwd (4), deltanet_fwd_transition (5),
 * deltanet_bwd_transition (6) or deltanet_state_scan (7) issues for this
 * descriptor (launch accounting). */
int deltanet_launch_count(const deltanet_desc* d, int which);

/* Human-readable message for an error code (static storage). */
const char* deltanet_strerror(int code);

/* DELTANET_ABI_VERSION of the loaded library. */
int deltanet_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DELTANET_H */
