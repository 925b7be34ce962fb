/*
 * deltanet_oracle.c -- plain, slow, fp64 CPU oracle.  TEST INFRASTRUCTURE
 * ONLY (see deltanet_oracle.h).  Every step cites the passage it follows.
 *
 * Paper notation (§2.2): the state S is d_v x d_k and o_t = S_t q_t.
 * The boundary uses H = S^T (reading R2); we convert at the edges.
 */
#include "deltanet_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define CKPT 64 /* checkpoint interval of the backward (SURVEY §8c memory scheme) */

typedef struct {
  const dn_oracle_desc* d;
  const double *q, *k, *v, *beta, *g, *h0, *dO, *dhT;
  double *o, *hT, *dq, *dk, *dv, *dbeta, *dg, *dh0;
  int worker, nworkers, bwd;
  int status;
} job_t;

/* PAPER.md §3.3: k_t = phi(x)/||phi(x)||_2 (same for q).
 * Reading R9: divide by max(||x||_2, eps). */
static void l2_normalize(const double* x, double* y, int n, double eps,
                         double* norm_out) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * x[i];
  double nrm = sqrt(s);
  double den = (nrm >= eps) ? nrm : eps;
  for (int i = 0; i < n; ++i) y[i] = x[i] / den;
  if (norm_out) *norm_out = nrm;
}

/* Adjoint of y = x / max(||x||, eps):
 *   ||x|| >= eps: dx = (dy - y (y . dy)) / ||x||        (textbook)
 *   ||x|| <  eps: dx = dy / eps                          (constant divisor) */
static void l2_normalize_adjoint(const double* y, const double* dy, double nrm,
                                 double eps, double* dx, int n) {
  if (nrm >= eps) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += y[i] * dy[i];
    for (int i = 0; i < n; ++i) dx[i] = (dy[i] - y[i] * s) / nrm;
  } else {
    for (int i = 0; i < n; ++i) dx[i] = dy[i] / eps;
  }
}

/* One delta-rule step, §2.2 line 86:
 *   S_t = S_{t-1} - beta_t (S_{t-1} k_t - v_t) k_t^T
 * and its gated form (Gated DeltaNet, PAPER.md Table tab:overview):
 *   S_t = S_{t-1} (alpha_t (I - beta_t k_t k_t^T)) + beta_t v_t k_t^T
 *       = alpha_t S_{t-1} + beta_t (v_t - alpha_t S_{t-1} k_t) k_t^T
 * (alpha_t = 1 is the ungated step, bit for bit).  S is Dv x Dk row-major;
 * r (scratch, Dv) receives v_t - alpha_t S_{t-1} k_t. */
static void delta_step(double* S, const double* kt, const double* vt,
                       double bt, double at, double* r, int Dk, int Dv) {
  for (int i = 0; i < Dv; ++i) {
    double sk = 0.0;
    for (int j = 0; j < Dk; ++j) sk += S[(size_t)i * Dk + j] * kt[j];
    r[i] = vt[i] - at * sk;
  }
  for (int i = 0; i < Dv; ++i)
    for (int j = 0; j < Dk; ++j)
      S[(size_t)i * Dk + j] = at * S[(size_t)i * Dk + j] + bt * r[i] * kt[j];
}

/* alpha_t = exp(g_t) (g = log-decay, R23); 1 without a gate */
static double gate(const double* g, int t) { return g ? exp(g[t]) : 1.0; }

/* o_t = S_t q_t  (§2.2 line 97). */
static void readout(const double* S, const double* qt, double* ot, int Dk,
                    int Dv) {
  for (int i = 0; i < Dv; ++i) {
    double s = 0.0;
    for (int j = 0; j < Dk; ++j) s += S[(size_t)i * Dk + j] * qt[j];
    ot[i] = s;
  }
}

/* Normalised (or copied) rows of one unit: xh[L][n], norms[L]. */
static void prep_rows(const double* x, double* xh, double* norms, int L, int n,
                      int l2, double eps) {
  for (int t = 0; t < L; ++t) {
    if (l2)
      l2_normalize(x + (size_t)t * n, xh + (size_t)t * n, n, eps, norms + t);
    else {
      memcpy(xh + (size_t)t * n, x + (size_t)t * n, sizeof(double) * n);
      norms[t] = 0.0;
    }
  }
}

static void unit_fwd(const dn_oracle_desc* d, size_t u, const job_t* J,
                     double* work) {
  const int L = d->L, Dk = d->Dk, Dv = d->Dv;
  const double* q = J->q + u * (size_t)L * Dk;
  const double* k = J->k + u * (size_t)L * Dk;
  const double* v = J->v + u * (size_t)L * Dv;
  const double* beta = J->beta + u * (size_t)L;
  const double* gg = J->g ? J->g + u * (size_t)L : NULL;
  double* o = J->o + u * (size_t)L * Dv;

  double* S = work;                          /* Dv*Dk */
  double* qh = S + (size_t)Dv * Dk;          /* Dk */
  double* kh = qh + Dk;                      /* Dk */
  double* r = kh + Dk;                       /* Dv */

  /* S_0 = h0^T, else zero (Listing 1 line 1108 starts from zeros). */
  for (int i = 0; i < Dv; ++i)
    for (int j = 0; j < Dk; ++j)
      S[(size_t)i * Dk + j] =
          J->h0 ? J->h0[u * (size_t)Dk * Dv + (size_t)j * Dv + i] : 0.0;

  for (int t = 0; t < L; ++t) {
    if (d->l2norm) {
      l2_normalize(q + (size_t)t * Dk, qh, Dk, d->eps, NULL);
      l2_normalize(k + (size_t)t * Dk, kh, Dk, d->eps, NULL);
    } else {
      memcpy(qh, q + (size_t)t * Dk, sizeof(double) * Dk);
      memcpy(kh, k + (size_t)t * Dk, sizeof(double) * Dk);
    }
    delta_step(S, kh, v + (size_t)t * Dv, beta[t], gate(gg, t), r, Dk, Dv);
    readout(S, qh, o + (size_t)t * Dv, Dk, Dv);
  }
  if (J->hT)
    for (int i = 0; i < Dv; ++i)
      for (int j = 0; j < Dk; ++j)
        J->hT[u * (size_t)Dk * Dv + (size_t)j * Dv + i] = S[(size_t)i * Dk + j];
}

/* Reverse mode through the recurrence (reading R12; derivation in
 * SURVEY App. A.1).  With dS = dl/dS_t, for t = L..1:
 *   dS += do_t q_t^T;  dq_t = S_t^T do_t;  g = dS k_t;  r = v_t - S_{t-1} k_t
 *   dv_t = beta_t g;   dbeta_t = g . r;   dk_t = beta_t (dS^T r - S_{t-1}^T g)
 *   dS <- dS - beta_t g k_t^T                                  (= dl/dS_{t-1})
 * Gated step (S_t = a S_{t-1} + beta r k^T, r = v - a S_{t-1} k, a = alpha_t):
 * the same with r = v_t - a S_{t-1} k_t,  dk_t = beta_t (dS^T r - a S_{t-1}^T g),
 *   dalpha_t = <dS, S_{t-1}> - beta_t g . (S_{t-1} k_t),  dg_t = a dalpha_t,
 *   dS <- a (dS - beta_t g k_t^T).
 */
static void unit_bwd(const dn_oracle_desc* d, size_t u, const job_t* J,
                     double* work) {
  const int L = d->L, Dk = d->Dk, Dv = d->Dv;
  const size_t SS = (size_t)Dv * Dk;
  const double* q = J->q + u * (size_t)L * Dk;
  const double* k = J->k + u * (size_t)L * Dk;
  const double* v = J->v + u * (size_t)L * Dv;
  const double* beta = J->beta + u * (size_t)L;
  const double* dO = J->dO + u * (size_t)L * Dv;
  double* dq = J->dq + u * (size_t)L * Dk;
  double* dk = J->dk + u * (size_t)L * Dk;
  double* dv = J->dv + u * (size_t)L * Dv;
  double* dbeta = J->dbeta + u * (size_t)L;
  const double* gg = J->g ? J->g + u * (size_t)L : NULL;
  double* dgg = J->dg ? J->dg + u * (size_t)L : NULL;

  const int nseg = (L + CKPT - 1) / CKPT;
  double* ck = work;                          /* (nseg+1) * SS checkpoints */
  double* seg = ck + (size_t)(nseg + 1) * SS; /* (CKPT+1) * SS local states */
  double* dS = seg + (size_t)(CKPT + 1) * SS; /* SS */
  double* qh = dS + SS;                       /* L*Dk */
  double* kh = qh + (size_t)L * Dk;           /* L*Dk */
  double* qn = kh + (size_t)L * Dk;           /* L */
  double* kn = qn + L;                        /* L */
  double* r = kn + L;                         /* Dv */
  double* g = r + Dv;                         /* Dv */
  double* dqh = g + Dv;                       /* Dk */
  double* dkh = dqh + Dk;                     /* Dk */

  prep_rows(q, qh, qn, L, Dk, d->l2norm, d->eps);
  prep_rows(k, kh, kn, L, Dk, d->l2norm, d->eps);

  /* forward sweep: S_0 and every CKPT-th state */
  double* S = seg; /* scratch state for the sweep */
  for (int i = 0; i < Dv; ++i)
    for (int j = 0; j < Dk; ++j)
      S[(size_t)i * Dk + j] =
          J->h0 ? J->h0[u * SS + (size_t)j * Dv + i] : 0.0;
  memcpy(ck, S, sizeof(double) * SS);
  for (int t = 0; t < L; ++t) {
    delta_step(S, kh + (size_t)t * Dk, v + (size_t)t * Dv, beta[t], gate(gg, t), r, Dk, Dv);
    if ((t + 1) % CKPT == 0 || t + 1 == L)
      memcpy(ck + (size_t)((t + CKPT) / CKPT) * SS, S, sizeof(double) * SS);
  }

  /* dS <- dhT^T (or 0) */
  for (int i = 0; i < Dv; ++i)
    for (int j = 0; j < Dk; ++j)
      dS[(size_t)i * Dk + j] = J->dhT ? J->dhT[u * SS + (size_t)j * Dv + i] : 0.0;

  for (int m = nseg - 1; m >= 0; --m) {
    const int t0 = m * CKPT;
    const int t1 = (t0 + CKPT < L) ? t0 + CKPT : L;
    /* seg[s] = S_{t0+s}, s = 0..t1-t0 */
    memcpy(seg, ck + (size_t)m * SS, sizeof(double) * SS);
    for (int t = t0; t < t1; ++t) {
      memcpy(seg + (size_t)(t - t0 + 1) * SS, seg + (size_t)(t - t0) * SS,
             sizeof(double) * SS);
      delta_step(seg + (size_t)(t - t0 + 1) * SS, kh + (size_t)t * Dk,
                 v + (size_t)t * Dv, beta[t], gate(gg, t), r, Dk, Dv);
    }
    for (int t = t1 - 1; t >= t0; --t) {
      const double* St = seg + (size_t)(t - t0 + 1) * SS; /* S_t (after) */
      const double* Sp = seg + (size_t)(t - t0) * SS;     /* S_{t-1} */
      const double* qt = qh + (size_t)t * Dk;
      const double* kt = kh + (size_t)t * Dk;
      const double* vt = v + (size_t)t * Dv;
      const double* dot = dO + (size_t)t * Dv;
      const double bt = beta[t];
      const double at = gate(gg, t);
      /* dS += do_t q_t^T */
      for (int i = 0; i < Dv; ++i)
        for (int j = 0; j < Dk; ++j) dS[(size_t)i * Dk + j] += dot[i] * qt[j];
      /* dq_t = S_t^T do_t */
      for (int j = 0; j < Dk; ++j) {
        double s = 0.0;
        for (int i = 0; i < Dv; ++i) s += St[(size_t)i * Dk + j] * dot[i];
        dqh[j] = s;
      }
      /* g = dS k_t ; r = v_t - a S_{t-1} k_t ; dalpha_t */
      double da = 0.0;
      for (int i = 0; i < Dv; ++i) {
        double sg = 0.0, sk = 0.0;
        for (int j = 0; j < Dk; ++j) {
          sg += dS[(size_t)i * Dk + j] * kt[j];
          sk += Sp[(size_t)i * Dk + j] * kt[j];
          da += dS[(size_t)i * Dk + j] * Sp[(size_t)i * Dk + j];
        }
        g[i] = sg;
        r[i] = vt[i] - at * sk;
        da -= bt * sg * sk;
      }
      if (dgg) dgg[t] = at * da;
      /* dv_t = beta_t g ; dbeta_t = g . r */
      double gr = 0.0;
      for (int i = 0; i < Dv; ++i) {
        dv[(size_t)t * Dv + i] = bt * g[i];
        gr += g[i] * r[i];
      }
      dbeta[t] = gr;
      /* dk_t = beta_t (dS^T r - a S_{t-1}^T g) */
      for (int j = 0; j < Dk; ++j) {
        double s = 0.0;
        for (int i = 0; i < Dv; ++i)
          s += dS[(size_t)i * Dk + j] * r[i] - at * Sp[(size_t)i * Dk + j] * g[i];
        dkh[j] = bt * s;
      }
      /* dS <- a (dS - beta_t g k_t^T) */
      for (int i = 0; i < Dv; ++i)
        for (int j = 0; j < Dk; ++j)
          dS[(size_t)i * Dk + j] = at * (dS[(size_t)i * Dk + j] - bt * g[i] * kt[j]);
      /* chain through the L2 normalisation (R9) */
      if (d->l2norm) {
        l2_normalize_adjoint(qt, dqh, qn[t], d->eps, dq + (size_t)t * Dk, Dk);
        l2_normalize_adjoint(kt, dkh, kn[t], d->eps, dk + (size_t)t * Dk, Dk);
      } else {
        memcpy(dq + (size_t)t * Dk, dqh, sizeof(double) * Dk);
        memcpy(dk + (size_t)t * Dk, dkh, sizeof(double) * Dk);
      }
    }
  }
  if (J->dh0)
    for (int i = 0; i < Dv; ++i)
      for (int j = 0; j < Dk; ++j)
        J->dh0[u * SS + (size_t)j * Dv + i] = dS[(size_t)i * Dk + j];
}

static size_t work_doubles(const dn_oracle_desc* d, int bwd) {
  const size_t SS = (size_t)d->Dv * d->Dk;
  if (!bwd) return SS + 2 * (size_t)d->Dk + d->Dv;
  const size_t nseg = (size_t)(d->L + CKPT - 1) / CKPT;
  return (nseg + 1) * SS + (CKPT + 1) * SS + SS + 2 * (size_t)d->L * d->Dk +
         2 * (size_t)d->L + 2 * (size_t)d->Dv + 2 * (size_t)d->Dk;
}

static void* worker_main(void* arg) {
  job_t* J = (job_t*)arg;
  const dn_oracle_desc* d = J->d;
  double* work = (double*)malloc(sizeof(double) * work_doubles(d, J->bwd));
  if (!work) {
    J->status = 1;
    return NULL;
  }
  const size_t units = (size_t)d->B * d->H;
  for (size_t u = (size_t)J->worker; u < units; u += (size_t)J->nworkers) {
    if (J->bwd)
      unit_bwd(d, u, J, work);
    else
      unit_fwd(d, u, J, work);
  }
  free(work);
  J->status = 0;
  return NULL;
}

static int run(const job_t* proto) {
  const dn_oracle_desc* d = proto->d;
  int nw = d->nthreads > 0 ? d->nthreads : 1;
  const size_t units = (size_t)d->B * d->H;
  if ((size_t)nw > units) nw = (int)units;
  if (nw < 1) return 0;
  job_t* jobs = (job_t*)calloc((size_t)nw, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nw, sizeof(pthread_t));
  if (!jobs || !th) {
    free(jobs);
    free(th);
    return 1;
  }
  int rc = 0;
  for (int w = 0; w < nw; ++w) {
    jobs[w] = *proto;
    jobs[w].worker = w;
    jobs[w].nworkers = nw;
    if (nw == 1) {
      worker_main(&jobs[w]);
    } else if (pthread_create(&th[w], NULL, worker_main, &jobs[w]) != 0) {
      jobs[w].status = 1; /* run inline instead */
      worker_main(&jobs[w]);
    }
  }
  if (nw > 1)
    for (int w = 0; w < nw; ++w) pthread_join(th[w], NULL);
  for (int w = 0; w < nw; ++w) rc |= jobs[w].status;
  free(jobs);
  free(th);
  return rc;
}

static int bad_desc(const dn_oracle_desc* d) {
  return !d || d->B < 0 || d->H < 0 || d->L < 0 || d->Dk <= 0 || d->Dv <= 0 ||
         !(d->eps > 0.0);
}

int dn_oracle_gated_fwd(const dn_oracle_desc* d, const double* q, const double* k,
                        const double* v, const double* beta, const double* g,
                        const double* h0, double* o, double* hT) {
  if (bad_desc(d) || !q || !k || !v || !beta || !o) return 1;
  job_t J;
  memset(&J, 0, sizeof J);
  J.d = d; J.q = q; J.k = k; J.v = v; J.beta = beta; J.g = g; J.h0 = h0;
  J.o = o; J.hT = hT; J.bwd = 0;
  return run(&J);
}

int dn_oracle_fwd(const dn_oracle_desc* d, const double* q, const double* k,
                  const double* v, const double* beta, const double* h0,
                  double* o, double* hT) {
  return dn_oracle_gated_fwd(d, q, k, v, beta, NULL, h0, o, hT);
}

int dn_oracle_gated_bwd(const dn_oracle_desc* d, const double* q, const double* k,
                        const double* v, const double* beta, const double* g,
                        const double* h0, const double* dO, const double* dhT,
                        double* dq, double* dk, double* dv, double* dbeta,
                        double* dg, double* dh0) {
  if (bad_desc(d) || !q || !k || !v || !beta || !dO || !dq || !dk || !dv ||
      !dbeta || (g && !dg))
    return 1;
  job_t J;
  memset(&J, 0, sizeof J);
  J.d = d; J.q = q; J.k = k; J.v = v; J.beta = beta; J.g = g; J.h0 = h0;
  J.dO = dO; J.dhT = dhT; J.dq = dq; J.dk = dk; J.dv = dv; J.dbeta = dbeta;
  J.dg = dg; J.dh0 = dh0; J.bwd = 1;
  return run(&J);
}

int dn_oracle_bwd(const dn_oracle_desc* d, const double* q, const double* k,
                  const double* v, const double* beta, const double* h0,
                  const double* dO, const double* dhT, double* dq, double* dk,
                  double* dv, double* dbeta, double* dh0) {
  return dn_oracle_gated_bwd(d, q, k, v, beta, NULL, h0, dO, dhT, dq, dk, dv, dbeta,
                             NULL, dh0);
}
