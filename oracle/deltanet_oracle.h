/*
 * deltanet_oracle.h -- fp64 CPU oracle for the DeltaNet delta-rule layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2406_06484_b200/), and the product path never loads it.
 *
 * What it computes is the plain definition of the method, token by token
 * (§2.2, lines 82-97):
 *     S_t = S_{t-1} - beta_t (S_{t-1} k_t - v_t) k_t^T,      o_t = S_t q_t
 * with the keys/queries L2-normalised first when requested (§3.3,
 * lines 329-331; eps reading R9 in DESIGN.md).  The chunkwise algorithm of
 * §3.2 reaches this exact result in real arithmetic, so no chunk size
 * appears here.  The backward is reverse-mode through the same recurrence
 * (the paper gives none -- DESIGN.md reading R12), with S_{t-1} recomputed
 * from checkpoints every 64 tokens.
 *
 * Layouts (all row-major, fp64, caller-owned host memory):
 *   q, k  [B,H,L,Dk]      v, o, dO  [B,H,L,Dv]      beta  [B,H,L]
 *   h0, hT, dhT, dh0  [B,H,Dk,Dv]   -- the kernel orientation H = S^T
 * Nullable: h0 (zero), hT, dhT (zero), dh0.
 *
 * Gated DeltaNet (PAPER.md Table tab:overview):
 *     S_t = S_{t-1} (alpha_t (I - beta_t k_t k_t^T)) + beta_t v_t k_t^T
 * with alpha_t = exp(g_t), g [B,H,L] the log-decay (R23); the
 * gated entry points take g (NULL = ungated, alpha = 1) and return dg.
 * Returns 0 on success, 1 on an invalid argument (nothing written).
 */
#ifndef DELTANET_ORACLE_H
#define DELTANET_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int B, H, L, Dk, Dv;
  int l2norm;      /* 1: q,k <- x / max(||x||_2, eps) before the recurrence */
  double eps;      /* 1e-6 (R9) */
  int nthreads;    /* <=0: one */
} dn_oracle_desc;

int dn_oracle_fwd(const dn_oracle_desc* d, const double* q, const double* k,
                  const double* v, const double* beta, const double* h0,
                  double* o, double* hT);

int dn_oracle_bwd(const dn_oracle_desc* d, const double* q, const double* k,
                  const double* v, const double* beta, const double* h0,
                  const double* dO, const double* dhT, double* dq, double* dk,
                  double* dv, double* dbeta, double* dh0);

int dn_oracle_gated_fwd(const dn_oracle_desc* d, const double* q, const double* k,
                        const double* v, const double* beta, const double* g,
                        const double* h0, double* o, double* hT);

int dn_oracle_gated_bwd(const dn_oracle_desc* d, const double* q, const double* k,
                        const double* v, const double* beta, const double* g,
                        const double* h0, const double* dO, const double* dhT,
                        double* dq, double* dk, double* dv, double* dbeta,
                        double* dg, double* dh0);

#ifdef __cplusplus
}
#endif
#endif
