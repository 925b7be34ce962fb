// abi.cu -- the extern "C" boundary of libdeltanet (include/deltanet.h):
// descriptor validation, workspace sizing, path selection and launch.
#include <string.h>

#include "common.cuh"

namespace {

bool pow2_in(int x, int lo, int hi) {
  if (x < lo || x > hi) return false;
  return (x & (x - 1)) == 0;
}

bool misaligned(const void* p) { return p && (((uintptr_t)p) & 15u) != 0; }

int validate(const deltanet_desc* d) {
  if (!d) return DELTANET_ERR_INVALID_ARG;
  if (d->B < 0 || d->H < 0 || d->L < 0) return DELTANET_ERR_INVALID_ARG;
  if (d->dtype != DELTANET_BF16 && d->dtype != DELTANET_FP32) return DELTANET_ERR_UNSUPPORTED;
  if (!pow2_in(d->Dk, 16, 256) || !pow2_in(d->Dv, 16, 256)) return DELTANET_ERR_UNSUPPORTED;
  if (!pow2_in(d->chunk, 16, 128)) return DELTANET_ERR_UNSUPPORTED;
  return DELTANET_OK;
}

// the recurrent form has no chunk: only shapes and dtype are checked
int validate_rec(const deltanet_desc* d) {
  if (!d) return DELTANET_ERR_INVALID_ARG;
  if (d->B < 0 || d->H < 0 || d->L < 0) return DELTANET_ERR_INVALID_ARG;
  if (d->dtype != DELTANET_BF16 && d->dtype != DELTANET_FP32) return DELTANET_ERR_UNSUPPORTED;
  if (!pow2_in(d->Dk, 16, 256) || !pow2_in(d->Dv, 16, 256)) return DELTANET_ERR_UNSUPPORTED;
  return DELTANET_OK;
}

// path choice (the gated forward and backward share the tcgen05 shapes):
// fused tcgen05 kernels at d = 128, split tcgen05 kernels at d in {64, 256}
// (or 128 with DELTANET_FORCE_SPLIT), CUDA-core kernels for fp32 / FORCE_SIMT
bool use_split(const deltanet_desc* d) {
  return !(d->flags & DELTANET_FORCE_SIMT) && dn::sp_supported(d) &&
         (d->Dk != 128 || (d->flags & DELTANET_FORCE_SPLIT));
}
bool use_tc(const deltanet_desc* d) {
  return !(d->flags & DELTANET_FORCE_SIMT) && !use_split(d) && dn::tc_supported(d) &&
         (!(d->flags & DELTANET_GATED) || dn::tc_gated_supported(d));
}

bool use_tc_bwd(const deltanet_desc* d) { return use_tc(d); }

// bf16 I/O runs on the tcgen05 kernels only: a bf16 descriptor outside their
// shapes is UNSUPPORTED unless the caller asks for the CUDA-core kernels
// explicitly (DELTANET_FORCE_SIMT) -- no silent 10^3-10^4x slower fallback.
// fp32 I/O (the 1e-4 parity mode) always runs on the CUDA-core kernels.
int validate_path(const deltanet_desc* d) {
  int rc = validate(d);
  if (rc) return rc;
  deltanet_desc e = *d;  // L = 0 (nothing to compute) keeps its shape's path
  if (e.L == 0) e.L = 1;
  if (e.dtype == DELTANET_BF16 && !(e.flags & DELTANET_FORCE_SIMT) && !use_tc(&e) &&
      !use_split(&e))
    return DELTANET_ERR_UNSUPPORTED;
  return DELTANET_OK;
}

size_t elem_bytes(const deltanet_desc* d) { return d->dtype == DELTANET_FP32 ? 4 : 2; }

size_t states_bytes(const deltanet_desc* d) {
  const size_t NC = (size_t)(d->L + d->chunk - 1) / d->chunk;
  return (size_t)d->B * d->H * NC * d->Dk * d->Dv * elem_bytes(d);
}

size_t round_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t scratch_bytes(const deltanet_desc* d) {
  const size_t simt = (size_t)d->B * d->H *
                      dn::simt_scratch_floats_per_unit(d->L, d->Dk, d->Dv, d->chunk) *
                      sizeof(float);
  if (use_split(d)) return dn::sp_scratch_bytes(d);
  if (!use_tc(d)) return simt;
  const size_t tc = dn::tc_scratch_bytes(d);
  return tc;
}

dn::Args make_args(const deltanet_desc* d, void* ws) {
  dn::Args a;
  memset(&a, 0, sizeof a);
  a.B = d->B; a.H = d->H; a.L = d->L; a.Dk = d->Dk; a.Dv = d->Dv; a.C = d->chunk;
  a.NC = (d->L + d->chunk - 1) / d->chunk;
  a.flags = d->flags;
  a.eps = d->l2_eps > 0.f ? d->l2_eps : 1e-6f;
  a.states = ws;
  a.scratch = (float*)((char*)ws + round_up(states_bytes(d)));
  return a;
}

// context parallelism: transitions exist
// on the tcgen05 path's shapes; L = 0 is the identity map
int validate_cp(const deltanet_desc* d) {
  int rc = validate(d);
  if (rc) return rc;
  if (d->flags & (DELTANET_FORCE_SIMT | DELTANET_GATED | DELTANET_FORCE_SPLIT))
    return DELTANET_ERR_UNSUPPORTED;
  deltanet_desc e = *d;
  e.L = 1;
  return dn::tc_supported(&e) ? DELTANET_OK : DELTANET_ERR_UNSUPPORTED;
}

// host-buffer pipeline (deltanet_fwd_bwd_host): per-slab buffer sizes
struct SlabLayout {
  int rows;          // (b, h) units per slab (the last may have fewer)
  size_t in_bytes;   // q k v dO beta of one slab
  size_t out_bytes;  // o dq dk dv dbeta of one slab
  size_t ws_bytes;   // fwd/bwd workspace of one (full) slab
};

SlabLayout slab_layout(const deltanet_desc* d, int slabs) {
  // units are independent and contiguous ([B*H][L][D]): a slab is a unit
  // range, run as a descriptor with B = units, H = 1
  SlabLayout sl;
  const int units = d->B * d->H;
  sl.rows = (units + slabs - 1) / slabs;
  deltanet_desc e = *d;
  e.B = sl.rows;
  e.H = 1;
  e.flags |= DELTANET_SAVE_STATES;
  const size_t eb = elem_bytes(d), per_row_tok = (size_t)d->L;
  const size_t qk = per_row_tok * d->Dk * eb, vv = per_row_tok * d->Dv * eb,
               bb = per_row_tok * eb;
  sl.in_bytes = round_up(sl.rows * qk) * 2 + round_up(sl.rows * vv) * 2 + round_up(sl.rows * bb);
  sl.out_bytes = sl.in_bytes;  // o dq dk dv dbeta have the shapes of v q k dO beta
  // the shared workspace must fit every slab's descriptor: a short last slab
  // can pick more sequence segments (more segment scratch) than a full one
  // (ADVICE r1), so size it for the larger of the two
  sl.ws_bytes = round_up(deltanet_workspace_bytes(&e));
  const int last = units - (units - 1) / sl.rows * sl.rows;
  if (units > 0 && last != sl.rows) {
    e.B = last;
    const size_t wl = round_up(deltanet_workspace_bytes(&e));
    if (wl > sl.ws_bytes) sl.ws_bytes = wl;
  }
  return sl;
}

}  // namespace

extern "C" {

size_t deltanet_workspace_bytes(const deltanet_desc* d) {
  if (validate_path(d) != DELTANET_OK) return 0;
  return round_up(states_bytes(d)) + round_up(scratch_bytes(d));
}

int deltanet_path(const deltanet_desc* d) {
  if (validate_path(d) != DELTANET_OK) return -1;
  deltanet_desc e = *d;
  if (e.L == 0) e.L = 1;
  return use_split(&e) ? 2 : use_tc(&e) ? 1 : 0;
}

int deltanet_launch_count(const deltanet_desc* d, int which) {
  if (which >= 2 && which <= 4) {  // recurrent fwd, prologue fwd / bwd
    if (validate_rec(d) != DELTANET_OK) return -1;
    if ((size_t)d->B * d->H == 0 || (which >= 3 && d->L == 0)) return 0;
    return which == 4 ? 2 : 1;
  }
  if (which >= 5 && which <= 7) {  // context-parallel transitions, scan
    if (validate_cp(d) != DELTANET_OK) return -1;
    if ((size_t)d->B * d->H == 0) return 0;
    if (which == 7 || d->L == 0) return 1;
    const int tr = dn::tc_fwd_segments(d) > 1 ? 2 : 1;  // pass 1 (+ composition)
    if (which == 6 && !(d->flags & DELTANET_SAVE_STATES)) return tr + dn::tc_launch_count(d, 0);
    return tr;
  }
  if (validate_path(d) != DELTANET_OK) return -1;
  if ((size_t)d->B * d->H == 0) return 0;
  if (use_split(d)) return dn::sp_launch_count(d, which);
  if (which == 1 ? use_tc_bwd(d) : use_tc(d)) return dn::tc_launch_count(d, which);
  return 1;
}

static int fwd_impl(const deltanet_desc* d, const void* q, const void* k, const void* v,
                    const void* beta, const float* g, const float* h0, void* o, float* hT,
                    void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_path(d);
  if (rc) return rc;
  const size_t units = (size_t)d->B * d->H;
  const bool tokens = units && d->L > 0;  // L = 0: token tensors may be empty (null)
  if (tokens && (!q || !k || !v || !beta || !o)) return DELTANET_ERR_INVALID_ARG;
  if (misaligned(q) || misaligned(k) || misaligned(v) || misaligned(beta) || misaligned(h0) ||
      misaligned(o) || misaligned(hT) || misaligned(workspace))
    return DELTANET_ERR_MISALIGNED;
  const size_t need = deltanet_workspace_bytes(d);
  if (units && (!workspace || workspace_bytes < need)) return DELTANET_ERR_WORKSPACE;
  if (!units) return DELTANET_OK;
  dn::Args a = make_args(d, workspace);
  a.q = q; a.k = k; a.v = v; a.beta = beta; a.h0 = h0; a.o = o; a.hT = hT; a.g = g;
  cudaStream_t s = (cudaStream_t)stream;
  if (use_split(d)) return dn::sp_fwd(a, s);
  return use_tc(d) ? dn::tc_fwd(a, s) : dn::simt_fwd(a, d->dtype, s);
}

int deltanet_fwd(const deltanet_desc* d, const void* q, const void* k, const void* v,
                 const void* beta, const float* h0, void* o, float* hT, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (d && (d->flags & DELTANET_GATED)) return DELTANET_ERR_INVALID_ARG;
  return fwd_impl(d, q, k, v, beta, nullptr, h0, o, hT, workspace, workspace_bytes, stream);
}

int deltanet_gated_fwd(const deltanet_desc* d, const void* q, const void* k, const void* v,
                       const void* beta, const float* g, const float* h0, void* o, float* hT,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!d) return DELTANET_ERR_INVALID_ARG;
  deltanet_desc e = *d;
  if (g) e.flags |= DELTANET_GATED;
  return fwd_impl(&e, q, k, v, beta, g, h0, o, hT, workspace, workspace_bytes, stream);
}

static int bwd_impl(const deltanet_desc* d, const void* q, const void* k, const void* v,
                    const void* beta, const float* g, const float* h0, const void* dO,
                    const float* dhT, void* dq, void* dk, void* dv, void* dbeta, float* dg,
                    float* dh0, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_path(d);
  if (rc) return rc;
  const size_t units = (size_t)d->B * d->H;
  const bool tokens = units && d->L > 0;
  if (tokens && (!q || !k || !v || !beta || !dO || !dq || !dk || !dv || !dbeta || (g && !dg)))
    return DELTANET_ERR_INVALID_ARG;
  if (misaligned(q) || misaligned(k) || misaligned(v) || misaligned(beta) || misaligned(h0) ||
      misaligned(dO) || misaligned(dhT) || misaligned(dq) || misaligned(dk) || misaligned(dv) ||
      misaligned(dbeta) || misaligned(dh0) || misaligned(workspace))
    return DELTANET_ERR_MISALIGNED;
  const size_t need = deltanet_workspace_bytes(d);
  if (units && (!workspace || workspace_bytes < need)) return DELTANET_ERR_WORKSPACE;
  if (!units) return DELTANET_OK;
  dn::Args a = make_args(d, workspace);
  a.q = q; a.k = k; a.v = v; a.beta = beta; a.h0 = h0; a.dO = dO; a.dhT = dhT;
  a.dq = dq; a.dk = dk; a.dv = dv; a.dbeta = dbeta; a.dh0 = dh0; a.g = g; a.dg = dg;
  cudaStream_t s = (cudaStream_t)stream;
  if (use_split(d)) return dn::sp_bwd(a, s);
  if (use_tc_bwd(d)) return dn::tc_bwd(a, s);
  // the SIMT backward cannot read states saved by a tcgen05 forward (their
  // layout is the bf16 operand image): it recomputes them
  if (use_tc(d)) a.flags &= ~DELTANET_SAVE_STATES;
  return dn::simt_bwd(a, d->dtype, s);
}

int deltanet_bwd(const deltanet_desc* d, const void* q, const void* k, const void* v,
                 const void* beta, const float* h0, const void* dO, const float* dhT, void* dq,
                 void* dk, void* dv, void* dbeta, float* dh0, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (d && (d->flags & DELTANET_GATED)) return DELTANET_ERR_INVALID_ARG;
  return bwd_impl(d, q, k, v, beta, nullptr, h0, dO, dhT, dq, dk, dv, dbeta, nullptr, dh0,
                  workspace, workspace_bytes, stream);
}

int deltanet_gated_bwd(const deltanet_desc* d, const void* q, const void* k, const void* v,
                       const void* beta, const float* g, const float* h0, const void* dO,
                       const float* dhT, void* dq, void* dk, void* dv, void* dbeta, float* dg,
                       float* dh0, void* workspace, size_t workspace_bytes, void* stream) {
  if (!d) return DELTANET_ERR_INVALID_ARG;
  deltanet_desc e = *d;
  if (g) e.flags |= DELTANET_GATED;
  return bwd_impl(&e, q, k, v, beta, g, h0, dO, dhT, dq, dk, dv, dbeta, dg, dh0, workspace,
                  workspace_bytes, stream);
}

int deltanet_recurrent_fwd(const deltanet_desc* d, const void* q, const void* k, const void* v,
                           const void* beta, const float* h0, void* o, float* hT,
                           void* stream) {
  return deltanet_gated_recurrent_fwd(d, q, k, v, beta, nullptr, h0, o, hT, stream);
}

int deltanet_gated_recurrent_fwd(const deltanet_desc* d, const void* q, const void* k,
                                 const void* v, const void* beta, const float* g,
                                 const float* h0, void* o, float* hT, void* stream) {
  int rc = validate_rec(d);
  if (rc) return rc;
  const size_t units = (size_t)d->B * d->H;
  if (units && d->L > 0 && (!q || !k || !v || !beta || !o)) return DELTANET_ERR_INVALID_ARG;
  if (misaligned(q) || misaligned(k) || misaligned(v) || misaligned(beta) || misaligned(h0) ||
      misaligned(o) || misaligned(hT))
    return DELTANET_ERR_MISALIGNED;
  if (!units) return DELTANET_OK;
  dn::Args a;
  memset(&a, 0, sizeof a);
  a.B = d->B; a.H = d->H; a.L = d->L; a.Dk = d->Dk; a.Dv = d->Dv;
  a.flags = d->flags;
  a.eps = d->l2_eps > 0.f ? d->l2_eps : 1e-6f;
  a.q = q; a.k = k; a.v = v; a.beta = beta; a.h0 = h0; a.o = o; a.hT = hT; a.g = g;
  return dn::rec_fwd(a, d->dtype, (cudaStream_t)stream);
}

size_t deltanet_prologue_workspace_bytes(const deltanet_desc* d) {
  if (validate_rec(d) != DELTANET_OK) return 0;
  return dn::prologue_workspace_bytes(d);
}

int deltanet_prologue_fwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                          const void* xb, const float* wq, const float* wk, const float* wv,
                          void* q, void* k, void* v, void* beta, void* stream) {
  int rc = validate_rec(d);
  if (rc) return rc;
  if ((size_t)d->B * d->H == 0 || d->L == 0) return DELTANET_OK;
  if (!xq || !xk || !xv || !xb || !wq || !wk || !wv || !q || !k || !v || !beta)
    return DELTANET_ERR_INVALID_ARG;
  if (misaligned(xq) || misaligned(xk) || misaligned(xv) || misaligned(wq) || misaligned(wk) ||
      misaligned(wv) || misaligned(q) || misaligned(k) || misaligned(v))
    return DELTANET_ERR_MISALIGNED;
  return dn::prologue_fwd(d, xq, xk, xv, xb, wq, wk, wv, q, k, v, beta, (cudaStream_t)stream);
}

int deltanet_prologue_bwd(const deltanet_desc* d, const void* xq, const void* xk, const void* xv,
                          const void* xb, const float* wq, const float* wk, const float* wv,
                          const void* dq, const void* dk, const void* dv, const void* dbeta,
                          void* dxq, void* dxk, void* dxv, void* dxb, float* dwq, float* dwk,
                          float* dwv, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_rec(d);
  if (rc) return rc;
  if ((size_t)d->B * d->H == 0) return DELTANET_OK;
  if (!dwq || !dwk || !dwv) return DELTANET_ERR_INVALID_ARG;
  if (d->L > 0 && (!xq || !xk || !xv || !xb || !wq || !wk || !wv || !dq || !dk || !dv ||
                   !dbeta || !dxq || !dxk || !dxv || !dxb))
    return DELTANET_ERR_INVALID_ARG;
  if (misaligned(xq) || misaligned(xk) || misaligned(xv) || misaligned(wq) || misaligned(wk) ||
      misaligned(wv) || misaligned(dq) || misaligned(dk) || misaligned(dv) || misaligned(dxq) ||
      misaligned(dxk) || misaligned(dxv) || misaligned(workspace))
    return DELTANET_ERR_MISALIGNED;
  if (d->L == 0) {  // no tokens: zero weight gradients
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(dwq, 0, (size_t)d->H * d->Dk * 4 * sizeof(float), s) != cudaSuccess ||
        cudaMemsetAsync(dwk, 0, (size_t)d->H * d->Dk * 4 * sizeof(float), s) != cudaSuccess ||
        cudaMemsetAsync(dwv, 0, (size_t)d->H * d->Dv * 4 * sizeof(float), s) != cudaSuccess)
      return DELTANET_ERR_CUDA;
    return DELTANET_OK;
  }
  if (!workspace || workspace_bytes < dn::prologue_workspace_bytes(d))
    return DELTANET_ERR_WORKSPACE;
  return dn::prologue_bwd(d, xq, xk, xv, xb, wq, wk, wv, dq, dk, dv, dbeta, dxq, dxk, dxv, dxb,
                          dwq, dwk, dwv, workspace, (cudaStream_t)stream);
}

// ---- host-buffer pipeline (include/deltanet.h deltanet_fwd_bwd_host) ----
size_t deltanet_fwd_bwd_host_device_bytes(const deltanet_desc* d, int slabs) {
  if (validate_path(d) != DELTANET_OK || slabs < 1) return 0;
  const int units = d->B * d->H;
  if (slabs > units) slabs = units > 0 ? units : 1;
  const SlabLayout sl = slab_layout(d, slabs);
  return 2 * (sl.in_bytes + sl.out_bytes) + sl.ws_bytes;
}

int deltanet_fwd_bwd_host(const deltanet_desc* d, const void* q, const void* k, const void* v,
                          const void* beta, const void* dO, void* o, void* dq, void* dk,
                          void* dv, void* dbeta, int slabs, void* dev_buffer,
                          size_t dev_bytes, void* stream) {
  int rc = validate_path(d);
  if (rc) return rc;
  if (slabs < 1) return DELTANET_ERR_INVALID_ARG;
  const size_t units = (size_t)d->B * d->H;
  if (!units || d->L == 0) return DELTANET_OK;
  if (!q || !k || !v || !beta || !dO || !o || !dq || !dk || !dv || !dbeta)
    return DELTANET_ERR_INVALID_ARG;
  if (misaligned(dev_buffer)) return DELTANET_ERR_MISALIGNED;
  if ((size_t)slabs > units) slabs = (int)units;
  if (!dev_buffer || dev_bytes < deltanet_fwd_bwd_host_device_bytes(d, slabs))
    return DELTANET_ERR_WORKSPACE;
  const SlabLayout sl = slab_layout(d, slabs);
  slabs = (int)((units + sl.rows - 1) / sl.rows);
  cudaStream_t user = (cudaStream_t)stream;
  cudaStream_t sin = nullptr, scmp = nullptr, sout = nullptr;
  cudaEvent_t ev_entry = nullptr, ev_done = nullptr, ev_in[2] = {}, ev_cmp[2] = {},
              ev_out[2] = {};
  bool ok = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&scmp, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_entry, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) == cudaSuccess;
  for (int b = 0; b < 2 && ok; ++b)
    ok = cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_cmp[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming) == cudaSuccess;
  // the device buffer may still be in use by earlier work on the caller's stream
  ok = ok && cudaEventRecord(ev_entry, user) == cudaSuccess &&
       cudaStreamWaitEvent(sin, ev_entry, 0) == cudaSuccess &&
       cudaStreamWaitEvent(scmp, ev_entry, 0) == cudaSuccess &&
       cudaStreamWaitEvent(sout, ev_entry, 0) == cudaSuccess;
  const size_t eb = elem_bytes(d), per_row_tok = (size_t)d->L;  // per unit
  const size_t rq = per_row_tok * d->Dk * eb, rv = per_row_tok * d->Dv * eb,
               rb = per_row_tok * eb;
  char* base = (char*)dev_buffer;
  void* wsb = base + 2 * (sl.in_bytes + sl.out_bytes);
  for (int i = 0; i < slabs && ok; ++i) {
    const int b = i & 1, r0 = i * sl.rows;
    const int nr = ((size_t)r0 + sl.rows <= units) ? sl.rows : (int)units - r0;
    // slab buffers (ping-pong by slab parity): q k v dO beta | o dq dk dv dbeta
    char* io = base + (size_t)b * (sl.in_bytes + sl.out_bytes);
    char* iq = io;
    char* ik = iq + round_up(sl.rows * rq);
    char* iv = ik + round_up(sl.rows * rq);
    char* ido = iv + round_up(sl.rows * rv);
    char* ib = ido + round_up(sl.rows * rv);
    char* oo = io + sl.in_bytes;
    char* odq = oo + round_up(sl.rows * rv);
    char* odk = odq + round_up(sl.rows * rq);
    char* odv = odk + round_up(sl.rows * rq);
    char* odb = odv + round_up(sl.rows * rv);
    const size_t fq = (size_t)r0 * rq, fv = (size_t)r0 * rv, fb = (size_t)r0 * rb;
    const size_t nq = (size_t)nr * rq, nv = (size_t)nr * rv, nb = (size_t)nr * rb;
    // slab i's inputs once slab i-2's outputs have been read out of buffer b
    if (i >= 2) ok = cudaStreamWaitEvent(sin, ev_out[b], 0) == cudaSuccess;
    ok = ok &&
         cudaMemcpyAsync(iq, (const char*)q + fq, nq, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
         cudaMemcpyAsync(ik, (const char*)k + fq, nq, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
         cudaMemcpyAsync(iv, (const char*)v + fv, nv, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
         cudaMemcpyAsync(ido, (const char*)dO + fv, nv, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
         cudaMemcpyAsync(ib, (const char*)beta + fb, nb, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
         cudaEventRecord(ev_in[b], sin) == cudaSuccess &&
         cudaStreamWaitEvent(scmp, ev_in[b], 0) == cudaSuccess;
    if (!ok) break;
    deltanet_desc e = *d;
    e.B = nr;
    e.H = 1;
    e.flags |= DELTANET_SAVE_STATES;
    rc = fwd_impl(&e, iq, ik, iv, ib, nullptr, nullptr, oo, nullptr, wsb, sl.ws_bytes, scmp);
    if (!rc)
      rc = bwd_impl(&e, iq, ik, iv, ib, nullptr, nullptr, ido, nullptr, odq, odk, odv, odb,
                    nullptr, nullptr, wsb, sl.ws_bytes, scmp);
    if (rc) break;
    ok = cudaEventRecord(ev_cmp[b], scmp) == cudaSuccess &&
         cudaStreamWaitEvent(sout, ev_cmp[b], 0) == cudaSuccess &&
         cudaMemcpyAsync((char*)o + fv, oo, nv, cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
         cudaMemcpyAsync((char*)dq + fq, odq, nq, cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
         cudaMemcpyAsync((char*)dk + fq, odk, nq, cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
         cudaMemcpyAsync((char*)dv + fv, odv, nv, cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
         cudaMemcpyAsync((char*)dbeta + fb, odb, nb, cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
         cudaEventRecord(ev_out[b], sout) == cudaSuccess;
  }
  // the caller's stream resumes after the last read-out (sout is in order)
  const bool tail = cudaEventRecord(ev_done, sout) == cudaSuccess &&
                    cudaStreamWaitEvent(user, ev_done, 0) == cudaSuccess;
  ok = ok && tail;
  for (int b = 0; b < 2; ++b) {
    if (ev_in[b]) cudaEventDestroy(ev_in[b]);
    if (ev_cmp[b]) cudaEventDestroy(ev_cmp[b]);
    if (ev_out[b]) cudaEventDestroy(ev_out[b]);
  }
  if (ev_entry) cudaEventDestroy(ev_entry);
  if (ev_done) cudaEventDestroy(ev_done);
  if (sin) cudaStreamDestroy(sin);
  if (scmp) cudaStreamDestroy(scmp);
  if (sout) cudaStreamDestroy(sout);
  if (rc) return rc;
  return ok ? DELTANET_OK : DELTANET_ERR_CUDA;
}

int deltanet_fwd_transition(const deltanet_desc* d, const void* q, const void* k, const void* v,
                            const void* beta, float* psi, float* hloc, void* workspace,
                            size_t workspace_bytes, void* stream) {
  int rc = validate_cp(d);
  if (rc) return rc;
  const size_t units = (size_t)d->B * d->H;
  if (!units) return DELTANET_OK;
  if (!psi || !hloc || (d->L > 0 && (!q || !k || !v || !beta))) return DELTANET_ERR_INVALID_ARG;
  if (misaligned(q) || misaligned(k) || misaligned(v) || misaligned(beta) || misaligned(psi) ||
      misaligned(hloc) || misaligned(workspace))
    return DELTANET_ERR_MISALIGNED;
  cudaStream_t s = (cudaStream_t)stream;
  if (d->L == 0) return dn::cp_empty((int)units, psi, hloc, s);
  if (!workspace || workspace_bytes < deltanet_workspace_bytes(d)) return DELTANET_ERR_WORKSPACE;
  dn::Args a = make_args(d, workspace);
  a.q = q; a.k = k; a.v = v; a.beta = beta;
  return dn::tc_fwd_transition(a, psi, hloc, s);
}

int deltanet_bwd_transition(const deltanet_desc* d, const void* q, const void* k, const void* v,
                            const void* beta, const void* dO, float* dhloc, void* workspace,
                            size_t workspace_bytes, void* stream) {
  int rc = validate_cp(d);
  if (rc) return rc;
  const size_t units = (size_t)d->B * d->H;
  if (!units) return DELTANET_OK;
  if (!dhloc || (d->L > 0 && (!q || !k || !v || !beta || !dO))) return DELTANET_ERR_INVALID_ARG;
  if (misaligned(q) || misaligned(k) || misaligned(v) || misaligned(beta) || misaligned(dO) ||
      misaligned(dhloc) || misaligned(workspace))
    return DELTANET_ERR_MISALIGNED;
  cudaStream_t s = (cudaStream_t)stream;
  if (d->L == 0) return dn::cp_empty((int)units, nullptr, dhloc, s);
  if (!workspace || workspace_bytes < deltanet_workspace_bytes(d)) return DELTANET_ERR_WORKSPACE;
  dn::Args a = make_args(d, workspace);
  a.q = q; a.k = k; a.v = v; a.beta = beta; a.dO = dO;
  if (!(d->flags & DELTANET_SAVE_STATES)) {  // records of this shard (X is independent of h0)
    dn::Args f = a;
    f.flags |= DELTANET_SAVE_STATES;
    f.o = nullptr;
    f.hT = nullptr;
    rc = dn::tc_fwd(f, s);
    if (rc) return rc;
  }
  return dn::tc_bwd_transition(a, dhloc, s);
}

int deltanet_state_scan(const deltanet_desc* d, int nparts, int part, int reverse,
                        const float* psi_all, const float* loc_all, const float* edge, float* out,
                        void* stream) {
  int rc = validate_cp(d);
  if (rc) return rc;
  if (nparts < 1 || part < 0 || part >= nparts || (reverse != 0 && reverse != 1))
    return DELTANET_ERR_INVALID_ARG;
  const size_t units = (size_t)d->B * d->H;
  if (!units) return DELTANET_OK;
  if (!out || (nparts > 1 && (!psi_all || !loc_all))) return DELTANET_ERR_INVALID_ARG;
  if (misaligned(psi_all) || misaligned(loc_all) || misaligned(edge) || misaligned(out))
    return DELTANET_ERR_MISALIGNED;
  return dn::cp_scan((int)units, nparts, part, reverse, psi_all, loc_all, edge, out,
                     (cudaStream_t)stream);
}

const char* deltanet_strerror(int code) {
  switch (code) {
    case DELTANET_OK: return "ok";
    case DELTANET_ERR_INVALID_ARG: return "invalid argument (null pointer or negative size)";
    case DELTANET_ERR_UNSUPPORTED: return "unsupported descriptor (dtype, Dk/Dv, or chunk)";
    case DELTANET_ERR_MISALIGNED: return "tensor pointer not 16-byte aligned";
    case DELTANET_ERR_CUDA: return "CUDA launch failed";
    case DELTANET_ERR_WORKSPACE: return "workspace missing or too small";
    default: return "unknown deltanet error code";
  }
}

int deltanet_abi_version(void) { return DELTANET_ABI_VERSION; }

}  // extern "C"
