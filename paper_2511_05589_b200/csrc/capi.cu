// capi.cu — the C-ABI (include/copris_b200.h): argument validation with the
// reference's exception semantics, context/device handling and dispatch to the
// sm_100a kernels in kernels.cu. No CPU compute path exists behind any entry.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/copris_b200.h"
#include "internal.hpp"
#include "lmhead.cuh"
#include "kernels.cuh"

using namespace copris_b200;

namespace copris_b200 {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(COPRIS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

DeviceGuard::DeviceGuard(int dev) {
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != dev) cudaSetDevice(dev);
}

DeviceGuard::~DeviceGuard() {
  int cur = -1;
  if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
}

}  // namespace copris_b200

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool valid_dtype(int32_t d) { return d == COPRIS_BF16 || d == COPRIS_F32; }

// grpo.hpp:120-133 / trainer.hpp:21-48 style validation shared by the loss
// entry points. Returns COPRIS_OK or an error with the reference's message.
int validate_loss(const copris_ctx* ctx, const copris_loss_batch* b, const copris_loss_cfg* c,
                  const copris_loss_out* o) {
  if (!ctx || !b || !c || !o) return fail(COPRIS_E_INVALID, "null argument");
  if (c->total_tokens <= 0) return fail(COPRIS_E_CONFIG, "grpo_step_loss batch has no tokens");
  if (c->clip_low <= 0.0 || c->clip_high <= 0.0)  // grpo.hpp:21-22
    return fail(COPRIS_E_CONFIG, "grpo.clip_low and grpo.clip_high must be > 0");
  if (c->kl_coeff < 0.0) return fail(COPRIS_E_CONFIG, "grpo.kl_coeff must be >= 0");
  if (c->kl_coeff > 0.0 && !b->ref_lp)  // grpo.hpp:126-127
    return fail(COPRIS_E_CONTRACT, "reference log-probs required when kl_coeff > 0");
  if (c->behav_mode != COPRIS_BEHAV_RECOMPUTED && c->behav_mode != COPRIS_BEHAV_RECORDED)
    return fail(COPRIS_E_INVALID, "behav_mode must be COPRIS_BEHAV_RECOMPUTED or _RECORDED");
  if (b->n_rows < 0 || b->row_base < 0) return fail(COPRIS_E_INVALID, "negative row range");
  // with a mask total_tokens counts the unmasked tokens only
  if (!b->loss_mask && b->row_base + b->n_rows > c->total_tokens)
    return fail(COPRIS_E_CONTRACT, "log-prob vectors must align with token count");
  if (b->n_rows == 0) return COPRIS_OK;
  if (b->vocab < 1) return fail(COPRIS_E_CONFIG, "policy.vocab must leave room for answer tokens plus EOS");
  if (b->ld < b->vocab) return fail(COPRIS_E_INVALID, "ld must be >= vocab");
  if (!valid_dtype(b->logits_dtype)) return fail(COPRIS_E_INVALID, "unknown logits dtype");
  if (!b->logits || !b->target || !b->stage || !b->buffered_lp || !b->tok_traj || !b->adv)
    return fail(COPRIS_E_INVALID, "null batch pointer");
  if (!o->obj || !o->flags) return fail(COPRIS_E_INVALID, "null output pointer (obj/flags)");
  if (o->dlogits) {
    if (!valid_dtype(o->dlogits_dtype)) return fail(COPRIS_E_INVALID, "unknown dlogits dtype");
    if (o->ld_dlogits < b->vocab) return fail(COPRIS_E_INVALID, "ld_dlogits must be >= vocab");
  }
  return COPRIS_OK;
}

LossParams make_params(const copris_ctx* ctx, const copris_loss_batch* b, const copris_loss_cfg* c,
                       const copris_loss_out* o) {
  LossParams p{};
  p.logits = b->logits;
  p.ld = b->ld;
  p.vocab = b->vocab;
  p.cur_stage = static_cast<int32_t>(b->cur_stage);
  p.n_rows = b->n_rows;
  p.row_base = b->row_base;
  p.target = b->target;
  p.stage = b->stage;
  p.buffered_lp = b->buffered_lp;
  p.ref_lp = c->kl_coeff > 0.0 ? b->ref_lp : nullptr;
  p.tok_traj = b->tok_traj;
  p.adv = b->adv;
  p.loss_mask = b->loss_mask;
  p.clamp_lo = 1.0 - c->clip_low;   // grpo.hpp:149 bounds, same fp64 ops
  p.clamp_hi = 1.0 + c->clip_high;
  p.kl_coeff = c->kl_coeff;
  p.entropy_coeff = c->entropy_coeff;
  p.inv_t = 1.0 / static_cast<double>(c->total_tokens);  // grpo.hpp:135
  p.is_enabled = c->is_enabled;
  p.behav_mode = c->behav_mode;
  p.dlogits = o->dlogits;
  p.ld_d = o->ld_dlogits;
  p.cur_lp = o->cur_lp;
  p.lse = o->lse;
  p.behav = o->behav;
  p.obj = o->obj;
  p.coef = o->coef;
  p.flags = o->flags;
  p.err = ctx->d_err;
  p.trace = ctx->d_trace;
  p.row_ctr = ctx->d_rowctr;
  p.out4 = o->out4;
  p.red_scratch = ctx->d_scratch;
  p.red_n = b->row_base + b->n_rows;
  return p;
}

DType dt(int32_t d) { return d == COPRIS_BF16 ? DType::BF16 : DType::F32; }

}  // namespace

extern "C" {

int copris_abi_version(void) { return COPRIS_B200_ABI_VERSION; }

const char* copris_last_error(void) { return g_err.c_str(); }

int copris_ctx_create(int device, copris_ctx** out) {
  if (!out) return fail(COPRIS_E_INVALID, "null out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(COPRIS_E_INVALID, "device out of range");
  DeviceGuard g(device);
  cudaDeviceProp prop{};
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10)
    return fail(COPRIS_E_CUDA, "copris_b200 kernels are built for sm_100a (Blackwell B200)");
  auto* ctx = new copris_ctx{};
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->tuning = tuning_from_env();  // the only environment read: launches use this copy
  e = cudaMalloc(&ctx->d_err, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_err, 0, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_rowctr, sizeof(unsigned long long));
  // the claim counter starts at 0; every launch that claims rows leaves it at 0
  // again (the TMA kernel's last CTA resets it, reduce.cuh end_of_launch; in
  // the pair family the last cluster whose row claim comes back empty)
  if (e == cudaSuccess) e = cudaMemset(ctx->d_rowctr, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_scratch, reduce_scratch_bytes());
  if (e == cudaSuccess) e = cudaMemset(ctx->d_scratch, 0, reduce_scratch_bytes());
  if (e == cudaSuccess && ctx->tuning.trace) {
    e = cudaMalloc(&ctx->d_trace, sizeof(long long) * kTraceCtas * kTraceSlots);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_trace, 0, sizeof(long long) * kTraceCtas * kTraceSlots);
  }
  if (e != cudaSuccess) {
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_rowctr);
    cudaFree(ctx->d_scratch);
    cudaFree(ctx->d_trace);
    delete ctx;
    return cuda_fail(e, "copris_ctx_create");
  }
  *out = ctx;
  return COPRIS_OK;
}

int copris_ctx_destroy(copris_ctx* ctx) {
  if (!ctx) return COPRIS_OK;
  DeviceGuard g(ctx->device);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_rowctr);
  cudaFree(ctx->d_scratch);
  cudaFree(ctx->d_trace);
  delete ctx;
  return COPRIS_OK;
}

int copris_ctx_check(copris_ctx* ctx, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaStreamSynchronize(as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  uint32_t err = 0;
  e = cudaMemcpy(&err, ctx->d_err, sizeof(err), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read error word");
  if (err == 0) return COPRIS_OK;
  cudaMemset(ctx->d_err, 0, sizeof(uint32_t));
  if (err & ERR_TOKEN_OOV) return fail(COPRIS_E_CONTRACT, "token out of vocabulary");
  if (err & ERR_NONFINITE_ADV) return fail(COPRIS_E_CONTRACT, "advantage must be finite");
  if (err & ERR_NONFINITE_LP) return fail(COPRIS_E_CONTRACT, "token_ratio requires finite log-probs");
  if (err & ERR_NOT_TERMINATED)
    return fail(COPRIS_E_CONTRACT, "terminal_reward requires a terminated trajectory");
  if (err & ERR_EMPTY_TERMINATED)
    return fail(COPRIS_E_CONTRACT, "terminated trajectory cannot be empty");
  return fail(COPRIS_E_CUDA, "unknown device error");
}

int copris_logprob_gather(copris_ctx* ctx, const void* logits, int64_t ld, int32_t dtype,
                          const int32_t* target, int64_t n_tok, int32_t vocab, float* out_lp,
                          float* out_lse, void* stream) {
  NvtxRange nv("copris_logprob_gather");
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_tok < 0) return fail(COPRIS_E_INVALID, "negative n_tok");
  if (n_tok == 0) return COPRIS_OK;  // test_policy.cpp:151-155
  if (!logits || !target || !out_lp) return fail(COPRIS_E_INVALID, "null pointer");
  if (!valid_dtype(dtype)) return fail(COPRIS_E_INVALID, "unknown logits dtype");
  if (vocab < 1 || ld < vocab) return fail(COPRIS_E_INVALID, "bad vocab/ld");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_logprob_gather(logits, ld, dt(dtype), target, n_tok, vocab, out_lp,
                                        out_lse, ctx->d_err, ctx->d_rowctr, ctx->d_scratch,
                                        ctx->num_sms, ctx->tuning, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "logprob_gather launch");
}

int32_t copris_lmhead_num_vtiles(int32_t vocab) {
  return vocab > 0 ? lmhead_num_vtiles(vocab) : 0;
}

int copris_lmhead_logits(copris_ctx* ctx, const void* hidden, int64_t ld_hidden,
                         const void* weight, int64_t ld_weight, int64_t n_rows,
                         int32_t hidden_dim, int32_t vocab, const int32_t* target, void* logits,
                         int64_t ld_logits, float* partials, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_rows < 0) return fail(COPRIS_E_INVALID, "negative n_rows");
  if (n_rows == 0) return COPRIS_OK;
  if (!hidden || !weight || !logits || (partials && !target))
    return fail(COPRIS_E_INVALID, "null pointer");
  if (vocab < 1 || hidden_dim < 1) return fail(COPRIS_E_INVALID, "bad vocab/hidden_dim");
  if (ld_hidden < hidden_dim || ld_weight < hidden_dim || ld_hidden % 8 || ld_weight % 8)
    return fail(COPRIS_E_INVALID, "hidden/weight row strides must be >= hidden_dim and 16-byte aligned");
  if (ld_logits < vocab || ld_logits % 8) return fail(COPRIS_E_INVALID, "bad ld_logits");
  if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(weight) |
       reinterpret_cast<uintptr_t>(logits)) & 15)
    return fail(COPRIS_E_INVALID, "hidden/weight/logits must be 16-byte aligned");
  if (n_rows > INT32_MAX || vocab > INT32_MAX - 256) return fail(COPRIS_E_INVALID, "too many rows");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_lmhead_fwd(hidden, ld_hidden, weight, ld_weight, n_rows, hidden_dim, vocab,
                                    target, logits, ld_logits, partials, ctx->num_sms,
                                    ctx->tuning, as_stream(stream), &ctx->last);
  if (e == cudaErrorInvalidValue && !partials)
    return fail(COPRIS_E_INVALID, "logits-only mode needs the CTA-pair kernel with TMA stores (vocab % 8 == 0)");
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "lmhead_logits launch");
}

int copris_lse_merge(copris_ctx* ctx, const float* partials, int32_t n_vt, const void* logits,
                     int64_t ld, const int32_t* target, int64_t n_rows, int32_t vocab,
                     float* out_lp, float* out_lse, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_rows < 0) return fail(COPRIS_E_INVALID, "negative n_rows");
  if (n_rows == 0) return COPRIS_OK;
  if (!partials || !logits || !target || !out_lp) return fail(COPRIS_E_INVALID, "null pointer");
  if (vocab < 1 || ld < vocab) return fail(COPRIS_E_INVALID, "bad vocab/ld");
  if (n_vt != lmhead_num_vtiles(vocab)) return fail(COPRIS_E_INVALID, "n_vt does not match vocab");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_lse_merge(partials, n_vt, logits, ld, target, n_rows, vocab, out_lp,
                                   out_lse, ctx->d_err, ctx->num_sms, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "lse_merge launch");
}

int32_t copris_lmhead_dhidden_splits(copris_ctx* ctx, int64_t n_rows, int32_t hidden_dim) {
  if (!ctx || n_rows < 1 || hidden_dim < 1) return 0;
  return gemm_nt_splits(n_rows, hidden_dim, ctx->num_sms, ctx->tuning);
}

int copris_lmhead_dhidden(copris_ctx* ctx, const void* dlogits, int64_t ld_dlogits,
                          const void* weight_t, int64_t ld_weight_t, int64_t n_rows,
                          int32_t hidden_dim, int32_t vocab, void* dhidden, int64_t ld_dhidden,
                          float* work, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_rows < 0) return fail(COPRIS_E_INVALID, "negative n_rows");
  if (n_rows == 0) return COPRIS_OK;
  if (!dlogits || !weight_t || !dhidden || !work) return fail(COPRIS_E_INVALID, "null pointer");
  if (vocab < 1 || hidden_dim < 4 || hidden_dim % 4) return fail(COPRIS_E_INVALID, "bad vocab/hidden_dim");
  if (ld_dlogits < vocab || ld_weight_t < vocab || ld_dlogits % 8 || ld_weight_t % 8 ||
      ld_dhidden < hidden_dim || ld_dhidden % 4)
    return fail(COPRIS_E_INVALID, "bad row strides");
  if ((reinterpret_cast<uintptr_t>(dlogits) | reinterpret_cast<uintptr_t>(weight_t)) & 15 ||
      reinterpret_cast<uintptr_t>(dhidden) & 7 || reinterpret_cast<uintptr_t>(work) & 15)
    return fail(COPRIS_E_INVALID, "misaligned operand");
  if (n_rows > INT32_MAX) return fail(COPRIS_E_INVALID, "too many rows");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_gemm_nt_bf16(dlogits, ld_dlogits, weight_t, ld_weight_t, n_rows, hidden_dim,
                                      vocab, dhidden, ld_dhidden, work,
                                      gemm_nt_splits(n_rows, hidden_dim, ctx->num_sms, ctx->tuning),
                                      ctx->num_sms, ctx->tuning, as_stream(stream), &ctx->last);
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "lmhead_dhidden launch");
}

int copris_lmhead_dweight(copris_ctx* ctx, const void* dlogits, int64_t ld_dlogits,
                          const void* hidden, int64_t ld_hidden, int64_t n_rows,
                          int32_t hidden_dim, int32_t vocab, float* dweight, int64_t ld_dweight,
                          void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_rows < 0) return fail(COPRIS_E_INVALID, "negative n_rows");
  if (n_rows == 0) return COPRIS_OK;
  if (!dlogits || !hidden || !dweight) return fail(COPRIS_E_INVALID, "null pointer");
  if (vocab < 1 || hidden_dim < 1 || vocab > INT32_MAX - 256 || hidden_dim > INT32_MAX - 256)
    return fail(COPRIS_E_INVALID, "bad vocab/hidden_dim");
  if (ld_dlogits < vocab || ld_hidden < hidden_dim || ld_dlogits % 8 || ld_hidden % 8 ||
      ld_dweight < hidden_dim || ld_dweight % 4)
    return fail(COPRIS_E_INVALID, "bad row strides");
  if ((reinterpret_cast<uintptr_t>(dlogits) | reinterpret_cast<uintptr_t>(hidden) |
       reinterpret_cast<uintptr_t>(dweight)) & 15)
    return fail(COPRIS_E_INVALID, "misaligned operand");
  if (n_rows > INT32_MAX) return fail(COPRIS_E_INVALID, "too many rows");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_gemm_tn_acc_f32(dlogits, ld_dlogits, hidden, ld_hidden, n_rows, vocab,
                                         hidden_dim, dweight, ld_dweight, ctx->num_sms,
                                         ctx->tuning, as_stream(stream), &ctx->last);
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "lmhead_dweight launch");
}

int copris_expand_segments(copris_ctx* ctx, const int64_t* seg_off, const uint32_t* seg_ver,
                           int64_t n_seg, uint32_t* out_stage, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_seg < 0) return fail(COPRIS_E_INVALID, "negative n_seg");
  if (n_seg == 0) return COPRIS_OK;
  if (!seg_off || !seg_ver || !out_stage) return fail(COPRIS_E_INVALID, "null pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_expand_segments(seg_off, seg_ver, n_seg, out_stage, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "expand_segments launch");
}

int copris_behaviour_concat(copris_ctx* ctx, const uint32_t* stage, uint32_t cur_stage,
                            const float* buffered_lp, const float* cur_lp, int32_t is_enabled,
                            int32_t behav_mode, int64_t n_tok, float* out_behav,
                            uint8_t* out_flags, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_tok < 0) return fail(COPRIS_E_INVALID, "negative n_tok");
  if (n_tok == 0) return COPRIS_OK;
  if (!stage || !buffered_lp || !cur_lp || !out_behav) return fail(COPRIS_E_INVALID, "null pointer");
  if (behav_mode != COPRIS_BEHAV_RECOMPUTED && behav_mode != COPRIS_BEHAV_RECORDED)
    return fail(COPRIS_E_INVALID, "behav_mode must be COPRIS_BEHAV_RECOMPUTED or _RECORDED");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_behaviour(stage, cur_stage, buffered_lp, cur_lp, is_enabled, behav_mode,
                                   n_tok, out_behav, out_flags, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "behaviour_concat launch");
}

int copris_terminal_rewards(copris_ctx* ctx, const int32_t* tokens, const int64_t* tok_off,
                            int64_t n_traj, const uint8_t* terminated,
                            const int32_t* answer_target, int32_t eos_token, double* out_reward,
                            void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_traj < 0) return fail(COPRIS_E_INVALID, "negative n_traj");
  if (n_traj == 0) return COPRIS_OK;
  if (!tokens || !tok_off || !terminated || !answer_target || !out_reward)
    return fail(COPRIS_E_INVALID, "null pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_terminal_rewards(tokens, tok_off, n_traj, terminated, answer_target,
                                          eos_token, out_reward, ctx->d_err, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "terminal_rewards launch");
}

int copris_group_advantages(copris_ctx* ctx, const double* rewards,
                            const int64_t* group_off_host, const int64_t* group_off,
                            int64_t n_groups, double adv_epsilon, double* out_adv, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_groups < 0) return fail(COPRIS_E_INVALID, "negative n_groups");
  if (n_groups == 0) return COPRIS_OK;
  if (!rewards || !group_off_host || !group_off || !out_adv)
    return fail(COPRIS_E_INVALID, "null pointer");
  if (!(adv_epsilon > 0.0)) return fail(COPRIS_E_CONFIG, "grpo.adv_epsilon must be > 0");
  for (int64_t g = 0; g < n_groups; ++g)  // grpo.hpp:54
    if (group_off_host[g + 1] - group_off_host[g] < 2)
      return fail(COPRIS_E_CONFIG, "advantage group size must be >= 2");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_group_advantages(rewards, group_off, n_groups, adv_epsilon, out_adv,
                                          as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "group_advantages launch");
}

int copris_token_traj(copris_ctx* ctx, const int64_t* tok_off, int64_t n_traj, int64_t n_tok,
                      int32_t* out_tok_traj, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_traj < 0 || n_tok < 0) return fail(COPRIS_E_INVALID, "negative size");
  if (n_traj == 0 || n_tok == 0) return COPRIS_OK;
  if (!tok_off || !out_tok_traj) return fail(COPRIS_E_INVALID, "null pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_token_traj(tok_off, n_traj, out_tok_traj, as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "token_traj launch");
}

int copris_is_loss_fused(copris_ctx* ctx, const copris_loss_batch* batch,
                         const copris_loss_cfg* cfg, const copris_loss_out* out, void* stream) {
  NvtxRange nv("copris_is_loss_fused");
  int rc = validate_loss(ctx, batch, cfg, out);
  if (rc) return rc;
  if (!out->cur_lp) return fail(COPRIS_E_INVALID, "null output pointer (cur_lp)");
  if (batch->n_rows == 0) return COPRIS_OK;
  DeviceGuard g(ctx->device);
  LossParams p = make_params(ctx, batch, cfg, out);
  cudaError_t e = launch_fused(p, dt(batch->logits_dtype), dt(out->dlogits_dtype), ctx->num_sms,
                               ctx->tuning, as_stream(stream), &ctx->last);
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "is_loss_fused launch");
}

int copris_is_loss_bwd(copris_ctx* ctx, const copris_loss_batch* batch,
                       const copris_loss_cfg* cfg, const float* cur_lp, const float* lse,
                       const float* behav, const copris_loss_out* out, void* stream) {
  NvtxRange nv("copris_is_loss_bwd");
  int rc = validate_loss(ctx, batch, cfg, out);
  if (rc) return rc;
  if (!cur_lp || !lse || !behav) return fail(COPRIS_E_INVALID, "null cur_lp/lse/behav input");
  if (batch->n_rows == 0) return COPRIS_OK;
  DeviceGuard g(ctx->device);
  LossParams p = make_params(ctx, batch, cfg, out);
  p.in_cur_lp = cur_lp;
  p.in_lse = lse;
  p.in_behav = behav;
  p.cur_lp = nullptr;
  p.lse = nullptr;
  p.behav = nullptr;
  cudaError_t e = launch_bwd(p, dt(batch->logits_dtype), dt(out->dlogits_dtype), ctx->num_sms,
                             as_stream(stream), &ctx->last);
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "is_loss_bwd launch");
}

int copris_loss_reduce(copris_ctx* ctx, const double* obj, const uint8_t* flags, int64_t n_tok,
                       double* out4, void* stream) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (n_tok < 0) return fail(COPRIS_E_INVALID, "negative n_tok");
  if (!out4 || (n_tok > 0 && (!obj || !flags))) return fail(COPRIS_E_INVALID, "null pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_reduce(obj, flags, n_tok, out4, ctx->d_scratch, ctx->num_sms,
                                as_stream(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "loss_reduce launch");
}

/* Introspection (not part of the reference surface): what the last loss
 * launch on this context ran. kernel_name is a static string. */
int copris_ctx_last_launch(const copris_ctx* ctx, int* cluster, int* grid, int* num_sms,
                           const char** kernel_name) {
  if (!ctx) return fail(COPRIS_E_INVALID, "null ctx");
  if (cluster) *cluster = ctx->last.cluster;
  if (grid) *grid = ctx->last.grid;
  if (num_sms) *num_sms = ctx->num_sms;
  if (kernel_name) *kernel_name = ctx->last.kernel ? ctx->last.kernel : "";
  return COPRIS_OK;
}

int copris_ctx_last_fused_reduce(const copris_ctx* ctx) { return ctx ? ctx->last.reduced : 0; }

int copris_ctx_set_option(copris_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return fail(COPRIS_E_INVALID, "null argument");
  if (!tuning_set(ctx->tuning, name, value))
    return fail(COPRIS_E_INVALID, std::string("unknown option or value out of range: ") + name);
  if (ctx->tuning.trace && !ctx->d_trace) {
    DeviceGuard g(ctx->device);
    cudaError_t e = cudaMalloc(&ctx->d_trace, sizeof(long long) * kTraceCtas * kTraceSlots);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_trace, 0, sizeof(long long) * kTraceCtas * kTraceSlots);
    if (e != cudaSuccess) return cuda_fail(e, "trace buffer");
  }
  return COPRIS_OK;
}

int copris_ctx_get_option(const copris_ctx* ctx, const char* name, int64_t* value) {
  if (!ctx || !name || !value) return fail(COPRIS_E_INVALID, "null argument");
  if (!tuning_get(ctx->tuning, name, value)) return fail(COPRIS_E_INVALID, std::string("unknown option: ") + name);
  return COPRIS_OK;
}

int copris_ctx_trace_read(copris_ctx* ctx, long long* host, int n) {
  if (!ctx || !host) return fail(COPRIS_E_INVALID, "null argument");
  if (!ctx->d_trace) return fail(COPRIS_E_INVALID, "tracing is off (set COPRIS_TRACE=1 before creating the context)");
  DeviceGuard g(ctx->device);
  const int cap = kTraceCtas * kTraceSlots;
  cudaError_t e = cudaMemcpy(host, ctx->d_trace, sizeof(long long) * (n < cap ? n : cap), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(ctx->d_trace, 0, sizeof(long long) * cap);
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "trace read");
}

}  // extern "C"
