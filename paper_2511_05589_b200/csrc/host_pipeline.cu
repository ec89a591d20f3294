// host_pipeline.cu — the host-buffer drop-in for grpo_step_loss
// (grpo.hpp:117-185): host arrays in, host loss/counts/dlogits out.
//
// A workspace owns every device buffer the call needs (no allocation on the
// hot path) and three streams. Logits flow through two chunk buffers:
//
//   h2d stream   : copy chunk c      -> lbuf[c%2]              (after fused(c-2))
//   compute      : fused(lbuf[c%2])  -> dbuf[c%2]              (after h2d(c), d2h(c-2))
//   d2h stream   : dbuf[c%2]         -> host dlogits chunk c   (after fused(c))
//
// so the PCIe copies in both directions overlap the kernel. Per-token
// metadata goes up once per call on the compute stream; advantages are
// computed on the device when the caller passes rewards.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/copris_b200.h"
#include "internal.hpp"
#include "kernels.cuh"

using namespace copris_b200;

struct copris_workspace {
  copris_ctx* ctx = nullptr;
  int64_t chunk_rows = 0;
  int32_t vocab = 0;
  int32_t in_dtype = 0, out_dtype = 0;
  size_t in_es = 0, out_es = 0;
  int64_t max_tokens = 0, max_traj = 0;
  void* lbuf[2] = {nullptr, nullptr};
  void* dbuf[2] = {nullptr, nullptr};
  int32_t* target = nullptr;
  uint32_t* stage = nullptr;
  float* blp = nullptr;
  float* ref_lp = nullptr;
  int64_t* tok_off = nullptr;
  int32_t* tok_traj = nullptr;
  double* adv = nullptr;
  double* rewards = nullptr;
  int64_t* group_off = nullptr;
  float* cur_lp = nullptr;
  double* obj = nullptr;
  uint8_t* flags = nullptr;
  double* out4 = nullptr;
  double* h_out4 = nullptr;  // pinned
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {}, meta_done = nullptr;
};

namespace {

size_t esize(int32_t dt) { return dt == COPRIS_BF16 ? 2 : 4; }

void release(copris_workspace* w) {
  for (int i = 0; i < 2; ++i) {
    cudaFree(w->lbuf[i]);
    cudaFree(w->dbuf[i]);
    if (w->h2d_done[i]) cudaEventDestroy(w->h2d_done[i]);
    if (w->comp_done[i]) cudaEventDestroy(w->comp_done[i]);
    if (w->d2h_done[i]) cudaEventDestroy(w->d2h_done[i]);
  }
  if (w->meta_done) cudaEventDestroy(w->meta_done);
  void* bufs[] = {w->target, w->stage, w->blp, w->ref_lp, w->tok_off, w->tok_traj, w->adv,
                  w->rewards, w->group_off, w->cur_lp, w->obj, w->flags, w->out4};
  for (void* b : bufs) cudaFree(b);
  if (w->h_out4) cudaFreeHost(w->h_out4);
  if (w->s_h2d) cudaStreamDestroy(w->s_h2d);
  if (w->s_comp) cudaStreamDestroy(w->s_comp);
  if (w->s_d2h) cudaStreamDestroy(w->s_d2h);
}

// Copies rows [r0, r0+n) of a host [* x ld] matrix into a packed device chunk.
cudaError_t copy_rows_h2d(void* dst, const void* src, int64_t ld, int64_t r0, int64_t n,
                          int32_t vocab, size_t es, cudaStream_t s) {
  const char* base = static_cast<const char*>(src) + r0 * ld * es;
  if (ld == vocab) return cudaMemcpyAsync(dst, base, n * vocab * es, cudaMemcpyHostToDevice, s);
  return cudaMemcpy2DAsync(dst, vocab * es, base, ld * es, vocab * es, n, cudaMemcpyHostToDevice, s);
}

cudaError_t copy_rows_d2h(void* dst, int64_t ld, int64_t r0, const void* src, int64_t n,
                          int32_t vocab, size_t es, cudaStream_t s) {
  char* base = static_cast<char*>(dst) + r0 * ld * es;
  if (ld == vocab) return cudaMemcpyAsync(base, src, n * vocab * es, cudaMemcpyDeviceToHost, s);
  return cudaMemcpy2DAsync(base, ld * es, src, vocab * es, vocab * es, n, cudaMemcpyDeviceToHost, s);
}

#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

}  // namespace

extern "C" {

int copris_workspace_create(copris_ctx* ctx, int64_t chunk_rows, int32_t vocab,
                            int32_t logits_dtype, int32_t dlogits_dtype, int64_t max_tokens,
                            int64_t max_traj, copris_workspace** out) {
  if (!ctx || !out) return fail(COPRIS_E_INVALID, "null argument");
  *out = nullptr;
  if (chunk_rows < 1 || vocab < 1 || max_tokens < 1 || max_traj < 1)
    return fail(COPRIS_E_INVALID, "workspace sizes must be >= 1");
  if ((logits_dtype != COPRIS_BF16 && logits_dtype != COPRIS_F32) ||
      (dlogits_dtype != COPRIS_BF16 && dlogits_dtype != COPRIS_F32))
    return fail(COPRIS_E_INVALID, "unknown dtype");
  DeviceGuard g(ctx->device);
  auto* w = new copris_workspace{};
  w->ctx = ctx;
  w->chunk_rows = chunk_rows;
  w->vocab = vocab;
  w->in_dtype = logits_dtype;
  w->out_dtype = dlogits_dtype;
  w->in_es = esize(logits_dtype);
  w->out_es = esize(dlogits_dtype);
  w->max_tokens = max_tokens;
  w->max_traj = max_traj;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](auto** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  };
  for (int i = 0; i < 2; ++i) {
    alloc(&w->lbuf[i], chunk_rows * vocab * w->in_es);
    alloc(&w->dbuf[i], chunk_rows * vocab * w->out_es);
  }
  alloc(&w->target, max_tokens * 4);
  alloc(&w->stage, max_tokens * 4);
  alloc(&w->blp, max_tokens * 4);
  alloc(&w->ref_lp, max_tokens * 4);
  alloc(&w->tok_traj, max_tokens * 4);
  alloc(&w->cur_lp, max_tokens * 4);
  alloc(&w->obj, max_tokens * 8);
  alloc(&w->flags, max_tokens);
  alloc(&w->tok_off, (max_traj + 1) * 8);
  alloc(&w->adv, max_traj * 8);
  alloc(&w->rewards, max_traj * 8);
  alloc(&w->group_off, (max_traj + 1) * 8);
  alloc(&w->out4, 4 * 8);
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&w->h_out4), 4 * 8, cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->s_h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->s_comp, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->s_d2h, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&w->h2d_done[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->comp_done[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->d2h_done[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->meta_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    release(w);
    delete w;
    return cuda_fail(e, "copris_workspace_create");
  }
  *out = w;
  return COPRIS_OK;
}

int copris_workspace_destroy(copris_workspace* ws) {
  if (!ws) return COPRIS_OK;
  DeviceGuard g(ws->ctx->device);
  cudaDeviceSynchronize();
  release(ws);
  delete ws;
  return COPRIS_OK;
}

int copris_grpo_step_loss_host(copris_ctx* ctx, copris_workspace* w, const copris_host_batch* b,
                               const copris_loss_cfg* cfg_in, copris_host_result* out) {
  NvtxRange nv("copris_grpo_step_loss_host");
  if (!ctx || !w || !b || !cfg_in || !out) return fail(COPRIS_E_INVALID, "null argument");
  if (w->ctx != ctx) return fail(COPRIS_E_INVALID, "workspace belongs to another context");
  // grpo.hpp:120-133 order: empty batch, then per-item checks, then no tokens
  if (b->n_traj == 0) return fail(COPRIS_E_CONFIG, "grpo_step_loss requires a non-empty batch");
  if (b->n_tok == 0) return fail(COPRIS_E_CONFIG, "grpo_step_loss batch has no tokens");
  if (b->n_traj < 0 || b->n_tok < 0) return fail(COPRIS_E_INVALID, "negative size");
  if (b->n_tok > w->max_tokens || b->n_traj > w->max_traj)
    return fail(COPRIS_E_INVALID, "batch exceeds the workspace capacity");
  if (b->vocab != w->vocab || b->logits_dtype != w->in_dtype)
    return fail(COPRIS_E_INVALID, "batch vocab/dtype differs from the workspace");
  if (out->dlogits && out->dlogits_dtype != w->out_dtype)
    return fail(COPRIS_E_INVALID, "dlogits dtype differs from the workspace");
  if (!b->logits || !b->tok_off || !b->target || !b->stage || !b->buffered_lp)
    return fail(COPRIS_E_INVALID, "null batch pointer");
  if (b->ld < b->vocab || (out->dlogits && out->ld_dlogits < b->vocab))
    return fail(COPRIS_E_INVALID, "ld must be >= vocab");
  if (b->tok_off[0] != 0 || b->tok_off[b->n_traj] != b->n_tok)
    return fail(COPRIS_E_CONTRACT, "log-prob vectors must align with token count");
  if (!b->adv) {
    if (!b->rewards || !b->group_off) return fail(COPRIS_E_INVALID, "need adv or rewards+group_off");
    if (b->group_off[b->n_groups] != b->n_traj)
      return fail(COPRIS_E_CONTRACT, "groups must cover the batch");
    for (int64_t g = 0; g < b->n_groups; ++g)
      if (b->group_off[g + 1] - b->group_off[g] < 2)
        return fail(COPRIS_E_CONFIG, "advantage group size must be >= 2");
  }
  copris_loss_cfg cfg = *cfg_in;
  if (cfg.total_tokens == 0) cfg.total_tokens = b->n_tok;
  // every argument check runs BEFORE the first copy is enqueued: an error
  // return must not leave DMA reading the caller's (pinned) host buffers
  if (!b->adv && !(b->adv_epsilon > 0.0)) return fail(COPRIS_E_CONFIG, "grpo.adv_epsilon must be > 0");
  if (cfg.clip_low <= 0.0 || cfg.clip_high <= 0.0)  // grpo.hpp:21-22
    return fail(COPRIS_E_CONFIG, "grpo.clip_low and grpo.clip_high must be > 0");
  if (cfg.kl_coeff < 0.0) return fail(COPRIS_E_CONFIG, "grpo.kl_coeff must be >= 0");
  if (cfg.kl_coeff > 0.0 && !b->ref_lp)  // grpo.hpp:126-127
    return fail(COPRIS_E_CONTRACT, "reference log-probs required when kl_coeff > 0");
  if (cfg.behav_mode != COPRIS_BEHAV_RECOMPUTED && cfg.behav_mode != COPRIS_BEHAV_RECORDED)
    return fail(COPRIS_E_INVALID, "behav_mode must be COPRIS_BEHAV_RECOMPUTED or _RECORDED");
  if (cfg.total_tokens < b->n_tok) return fail(COPRIS_E_CONTRACT, "log-prob vectors must align with token count");

  DeviceGuard g(ctx->device);
  // past this point work is in flight: a failing call drains all three
  // streams before it returns (the caller may free its buffers right after)
  struct Drain {
    copris_workspace* w;
    bool armed = true;
    ~Drain() {
      if (!armed) return;
      cudaStreamSynchronize(w->s_h2d);
      cudaStreamSynchronize(w->s_comp);
      cudaStreamSynchronize(w->s_d2h);
    }
  } drain{w};
  const int64_t T = b->n_tok, n = b->n_traj;
  cudaStream_t sc = w->s_comp;
  // per-token / per-trajectory metadata
  CK(cudaMemcpyAsync(w->target, b->target, T * 4, cudaMemcpyHostToDevice, sc));
  CK(cudaMemcpyAsync(w->stage, b->stage, T * 4, cudaMemcpyHostToDevice, sc));
  CK(cudaMemcpyAsync(w->blp, b->buffered_lp, T * 4, cudaMemcpyHostToDevice, sc));
  if (b->ref_lp) CK(cudaMemcpyAsync(w->ref_lp, b->ref_lp, T * 4, cudaMemcpyHostToDevice, sc));
  CK(cudaMemcpyAsync(w->tok_off, b->tok_off, (n + 1) * 8, cudaMemcpyHostToDevice, sc));
  CK(launch_token_traj(w->tok_off, n, w->tok_traj, sc));
  if (b->adv) {
    CK(cudaMemcpyAsync(w->adv, b->adv, n * 8, cudaMemcpyHostToDevice, sc));
  } else {
    CK(cudaMemcpyAsync(w->rewards, b->rewards, n * 8, cudaMemcpyHostToDevice, sc));
    CK(cudaMemcpyAsync(w->group_off, b->group_off, (b->n_groups + 1) * 8, cudaMemcpyHostToDevice, sc));
    CK(launch_group_advantages(w->rewards, w->group_off, b->n_groups, b->adv_epsilon, w->adv, sc));
  }

  copris_loss_batch lb{};
  lb.ld = b->vocab;
  lb.logits_dtype = b->logits_dtype;
  lb.vocab = b->vocab;
  lb.target = w->target;
  lb.stage = w->stage;
  lb.buffered_lp = w->blp;
  lb.ref_lp = b->ref_lp ? w->ref_lp : nullptr;
  lb.tok_traj = w->tok_traj;
  lb.adv = w->adv;
  lb.cur_stage = b->cur_stage;
  copris_loss_out lo{};
  lo.ld_dlogits = b->vocab;
  lo.dlogits_dtype = w->out_dtype;
  lo.cur_lp = w->cur_lp;
  lo.obj = w->obj;
  lo.flags = w->flags;

  const int64_t nchunks = (T + w->chunk_rows - 1) / w->chunk_rows;
  for (int64_t c = 0; c < nchunks; ++c) {
    NvtxRange nvc("chunk: h2d -> fused -> d2h");
    const int i = static_cast<int>(c & 1);
    const int64_t r0 = c * w->chunk_rows;
    const int64_t rows = std::min(w->chunk_rows, T - r0);
    // lbuf[i] is free once fused(c-2) has consumed it
    if (c >= 2) CK(cudaStreamWaitEvent(w->s_h2d, w->comp_done[i], 0));
    CK(copy_rows_h2d(w->lbuf[i], b->logits, b->ld, r0, rows, b->vocab, w->in_es, w->s_h2d));
    CK(cudaEventRecord(w->h2d_done[i], w->s_h2d));
    CK(cudaStreamWaitEvent(sc, w->h2d_done[i], 0));
    if (out->dlogits && c >= 2) CK(cudaStreamWaitEvent(sc, w->d2h_done[i], 0));
    lb.logits = w->lbuf[i];
    lb.n_rows = rows;
    lb.row_base = r0;
    lo.dlogits = out->dlogits ? w->dbuf[i] : nullptr;
    int rc = copris_is_loss_fused(ctx, &lb, &cfg, &lo, sc);
    if (rc) return rc;
    CK(cudaEventRecord(w->comp_done[i], sc));
    if (out->dlogits) {
      CK(cudaStreamWaitEvent(w->s_d2h, w->comp_done[i], 0));
      CK(copy_rows_d2h(out->dlogits, out->ld_dlogits, r0, w->dbuf[i], rows, b->vocab, w->out_es,
                       w->s_d2h));
      CK(cudaEventRecord(w->d2h_done[i], w->s_d2h));
    }
  }
  CK(launch_reduce(w->obj, w->flags, T, w->out4, ctx->d_scratch, ctx->num_sms, sc));
  CK(cudaMemcpyAsync(w->h_out4, w->out4, 4 * 8, cudaMemcpyDeviceToHost, sc));
  if (out->cur_lp) CK(cudaMemcpyAsync(out->cur_lp, w->cur_lp, T * 4, cudaMemcpyDeviceToHost, sc));
  CK(cudaStreamSynchronize(w->s_h2d));
  CK(cudaStreamSynchronize(w->s_d2h));
  drain.armed = false;  // every stream is idle from here on
  int rc = copris_ctx_check(ctx, sc);  // syncs sc, maps device-detected violations
  if (rc) return rc;
  const double* o4 = w->h_out4;
  out->objective = o4[0];
  out->loss = -o4[0] * (1.0 / static_cast<double>(cfg.total_tokens));  // grpo.hpp:183
  out->token_count = static_cast<int64_t>(o4[1]);
  out->stale_tokens = static_cast<int64_t>(o4[2]);
  out->clipped_tokens = static_cast<int64_t>(o4[3]);
  return COPRIS_OK;
}

}  // extern "C"
