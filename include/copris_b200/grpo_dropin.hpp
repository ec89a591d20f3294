// grpo_dropin.hpp — C++ drop-in for the reference's grpo_step_loss
// (/root/reference/proj/include/copris/grpo.hpp:117-185) over the C-ABI.
//
// Header-only and templated on the caller's types, so it needs no reference
// header itself: a maintainer includes it next to copris/grpo.hpp and replaces
//
//     GrpoStepResult res = grpo_step_loss(params_, items, cfg_.clip);      // trainer.hpp:176
// with
//     GrpoStepResult res = gpu_.grpo_step_loss<GrpoStepResult, ContractViolation, ConfigError>(
//         params_, std::span<const GrpoItem>(items), cfg_.clip);
//
// where `gpu_` is a copris_b200::DropIn member. Semantics are the reference's:
// the stored log-probs are taken verbatim from each GrpoItem (COPRIS_BEHAV_RECORDED,
// which already carries the IS-off substitution of trainer.hpp:149), the token
// mean uses the batch's own token count, the gradient comes back shaped like
// PolicyParams::logits, and violations throw the caller's exception types with
// the reference's messages. The tabular policy of the reference is adapted by
// gathering the (class, position) rows of every token into a dense [T x V]
// matrix and scatter-adding the per-token dlogits rows back in batch order
// (SURVEY.md Appendix A.7); a transformer trainer passes its LM-head logits
// straight to copris_is_loss_fused instead.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "copris_b200.h"

namespace copris_b200 {

template <class ContractViolation, class ConfigError>
inline void throw_status(int rc) {
  if (rc == COPRIS_OK) return;
  const std::string msg = copris_last_error();
  if (rc == COPRIS_E_CONTRACT) throw ContractViolation(msg);
  if (rc == COPRIS_E_CONFIG) throw ConfigError(msg);
  throw std::runtime_error("copris_b200: " + msg);
}

class DropIn {
 public:
  explicit DropIn(int device = 0) {
    if (copris_ctx_create(device, &ctx_) != COPRIS_OK)
      throw std::runtime_error(std::string("copris_ctx_create: ") + copris_last_error());
  }
  ~DropIn() {
    if (ws_) copris_workspace_destroy(ws_);
    if (ctx_) copris_ctx_destroy(ctx_);
  }
  DropIn(const DropIn&) = delete;
  DropIn& operator=(const DropIn&) = delete;

  // grpo_step_loss(params, batch, cfg) with the reference's types:
  //   Params: .shape{num_classes,horizon,vocab}, .logits (double [Q*H*V]), .row_offset
  //   Item:   .traj->{question.class_id, tokens.tokens}, .advantage, .stored_lp, .ref_lp
  //   Clip:   .clip_low, .clip_high, .kl_coeff, .entropy_coeff
  template <class Result, class ContractViolation, class ConfigError, class Params, class Item,
            class Clip>
  Result grpo_step_loss(const Params& params, std::span<const Item> batch, const Clip& cfg) {
    if (batch.empty()) throw ConfigError("grpo_step_loss requires a non-empty batch");
    const int V = params.shape.vocab;
    size_t T = 0;
    for (const auto& it : batch) {
      if (it.traj == nullptr) throw ContractViolation("batch item missing trajectory");
      const size_t n = it.traj->tokens.tokens.size();
      if (it.stored_lp.size() != n) throw ContractViolation("log-prob vectors must align with token count");
      if (cfg.kl_coeff != 0.0 && it.ref_lp.size() != n)
        throw ContractViolation("reference log-probs required when kl_coeff > 0");
      T += n;
    }
    if (T == 0) throw ConfigError("grpo_step_loss batch has no tokens");
    ensure(T, batch.size(), V);
    // gather rows and per-token records (batch order)
    std::vector<int64_t> tok_off(batch.size() + 1, 0);
    size_t t = 0;
    for (size_t i = 0; i < batch.size(); ++i) {
      const auto& it = batch[i];
      const auto& toks = it.traj->tokens.tokens;
      for (size_t pos = 0; pos < toks.size(); ++pos, ++t) {
        const double* row = params.logits.data() +
                            params.shape.row_offset(it.traj->question.class_id, static_cast<int>(pos));
        float* dst = logits_.data() + t * V;
        for (int k = 0; k < V; ++k) dst[k] = static_cast<float>(row[k]);
        target_[t] = toks[pos];
        stage_[t] = 0;
        blp_[t] = static_cast<float>(it.stored_lp[pos]);
        if (cfg.kl_coeff != 0.0) ref_[t] = static_cast<float>(it.ref_lp[pos]);
      }
      adv_[i] = it.advantage;
      tok_off[i + 1] = static_cast<int64_t>(t);
    }
    copris_host_batch hb{};
    hb.logits = logits_.data();
    hb.ld = V;
    hb.logits_dtype = COPRIS_F32;
    hb.vocab = V;
    hb.n_tok = static_cast<int64_t>(T);
    hb.n_traj = static_cast<int64_t>(batch.size());
    hb.tok_off = tok_off.data();
    hb.target = target_.data();
    hb.stage = stage_.data();
    hb.buffered_lp = blp_.data();
    hb.ref_lp = cfg.kl_coeff != 0.0 ? ref_.data() : nullptr;
    hb.adv = adv_.data();
    hb.cur_stage = 1;  // every token "stale": behaviour = stored_lp verbatim
    copris_loss_cfg lc{};
    lc.clip_low = cfg.clip_low;
    lc.clip_high = cfg.clip_high;
    lc.kl_coeff = cfg.kl_coeff;
    lc.entropy_coeff = cfg.entropy_coeff;
    lc.is_enabled = 1;
    lc.behav_mode = COPRIS_BEHAV_RECORDED;
    lc.total_tokens = 0;
    copris_host_result hr{};
    hr.dlogits = dlogits_.data();
    hr.ld_dlogits = V;
    hr.dlogits_dtype = COPRIS_F32;
    throw_status<ContractViolation, ConfigError>(copris_grpo_step_loss_host(ctx_, ws_, &hb, &lc, &hr));
    // scatter-add the per-token rows into the table gradient, batch order
    Result out;
    out.loss = hr.loss;
    out.token_count = T;
    out.grad.assign(params.logits.size(), 0.0);
    t = 0;
    for (const auto& it : batch) {
      const auto& toks = it.traj->tokens.tokens;
      for (size_t pos = 0; pos < toks.size(); ++pos, ++t) {
        double* g = out.grad.data() +
                    params.shape.row_offset(it.traj->question.class_id, static_cast<int>(pos));
        const float* d = dlogits_.data() + t * V;
        for (int k = 0; k < V; ++k) g[k] += d[k];
      }
    }
    return out;
  }

  copris_ctx* ctx() const { return ctx_; }

 private:
  void ensure(size_t T, size_t n, int V) {
    if (ws_ && T <= cap_tok_ && n <= cap_traj_ && V == vocab_) {
      resize_host(T, n, V);
      return;
    }
    if (ws_) copris_workspace_destroy(ws_);
    ws_ = nullptr;
    cap_tok_ = std::max<size_t>(T, 2 * cap_tok_);
    cap_traj_ = std::max<size_t>(n, 2 * cap_traj_);
    vocab_ = V;
    const int64_t chunk = static_cast<int64_t>(std::min<size_t>(cap_tok_, 4096));
    if (copris_workspace_create(ctx_, chunk, V, COPRIS_F32, COPRIS_F32,
                                static_cast<int64_t>(cap_tok_), static_cast<int64_t>(cap_traj_),
                                &ws_) != COPRIS_OK)
      throw std::runtime_error(std::string("copris_workspace_create: ") + copris_last_error());
    resize_host(T, n, V);
  }
  void resize_host(size_t T, size_t n, int V) {
    logits_.resize(T * V);
    dlogits_.resize(T * V);
    target_.resize(T);
    stage_.resize(T);
    blp_.resize(T);
    ref_.resize(T);
    adv_.resize(n);
  }

  copris_ctx* ctx_ = nullptr;
  copris_workspace* ws_ = nullptr;
  size_t cap_tok_ = 0, cap_traj_ = 0;
  int vocab_ = 0;
  std::vector<float> logits_, dlogits_, blp_, ref_;
  std::vector<int32_t> target_;
  std::vector<uint32_t> stage_;
  std::vector<double> adv_;
};

// Drop-in for AdamOptimizer (grpo.hpp:205-235): replaces
//     adam_.update(params_, res.grad);                                      // trainer.hpp:177
// with
//     gpu_adam_.update<ContractViolation, ConfigError>(params_, res.grad);
// The moments live on the device (copris_adam_host); each update is one
// blocking call that leaves params.logits updated and bumps params.version by
// exactly 1, as the reference does.
class AdamDropIn {
 public:
  // `Cfg` is the reference's AdamConfig (.lr, .beta1, .beta2, .eps, .weight_decay).
  template <class Cfg>
  AdamDropIn(copris_ctx* ctx, const Cfg& c) : ctx_(ctx) {
    cfg_ = copris_adam_cfg{c.lr, c.beta1, c.beta2, c.eps, c.weight_decay};
  }
  ~AdamDropIn() {
    if (opt_) copris_adam_host_destroy(opt_);
  }
  AdamDropIn(const AdamDropIn&) = delete;
  AdamDropIn& operator=(const AdamDropIn&) = delete;

  template <class ContractViolation, class ConfigError, class Params>
  void update(Params& params, std::span<const double> grad) {
    if (grad.size() != params.logits.size()) throw ContractViolation("gradient shape mismatch");
    const int64_t n = static_cast<int64_t>(grad.size());
    if (!opt_) throw_status<ContractViolation, ConfigError>(copris_adam_host_create(ctx_, n, &cfg_, &opt_));
    throw_status<ContractViolation, ConfigError>(
        copris_adam_host_update(opt_, params.logits.data(), grad.data(), n));
    params.version += 1;
  }

 private:
  copris_ctx* ctx_;
  copris_adam_cfg cfg_{};
  copris_adam_host* opt_ = nullptr;
};

}  // namespace copris_b200
